// Library-level C ABI helpers.
#include "common.cuh"

extern "C" int fkv_version(void) { return 1; }

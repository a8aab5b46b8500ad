// K3: gather the selected K/V rows of every (request, KV head) into the
// ragged, page-aligned, pre-swizzled cache of one GPU.
//
// No reference implementation exists.  Traffic is the
// algorithmic minimum: each selected row is read once (256 B, contiguous)
// and written once; a warp moves two rows per instruction pair with 16-byte
// vector loads/stores (lane = one 16-B chunk), the store address applying
// the cache swizzle (chunk c of row r at c ^ (r & 7)) -- still one
// contiguous 256-B row per half-warp, so stores stay fully coalesced.
//
// A destination segment is (source head bh, logical token range [lo, hi) of
// that head's selection, first cache row row0): TP=1 caches use one segment
// per head; a rank of an AHA plan compacts only the head copies it owns
// (DP copies = sub-ranges), reading the same offsets/idx.
#include <cuda_runtime.h>

#include "common.cuh"

namespace fkv {
namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads)
    compact_kernel(const uint4* __restrict__ k_src, const uint4* __restrict__ v_src, int T,
                   const int64_t* __restrict__ offsets, const int32_t* __restrict__ idx,
                   const int32_t* __restrict__ seg_bh, const int32_t* __restrict__ seg_lo,
                   const int32_t* __restrict__ seg_hi, const int64_t* __restrict__ seg_row0,
                   int zero_pad, uint4* __restrict__ k_dst, uint4* __restrict__ v_dst) {
  const int s = blockIdx.x;
  const int bh = seg_bh[s];
  const int lo = seg_lo[s], hi = seg_hi[s];
  const int64_t row0 = seg_row0[s];
  const int n = hi - lo;
  const int rows = zero_pad ? (n + FKV_PAGE - 1) / FKV_PAGE * FKV_PAGE : n;
  const int32_t* sel = idx + offsets[bh] + lo;
  const int64_t src_base = static_cast<int64_t>(bh) * T;  // row index of (b, h, token 0)
  const int half = threadIdx.x >> 4;                        // 16 half-warps per CTA
  const int c = threadIdx.x & 15;                           // 16-byte chunk of the row
  for (int r = half; r < rows; r += kThreads / 16) {
    const int64_t dst = row0 + r;
    const int64_t o = dst * 16 + (c ^ static_cast<int>(dst & 7));
    if (r < n) {
      const int64_t src = (src_base + sel[r]) * 16 + c;
      const uint4 kv = __ldg(k_src + src);
      const uint4 vv = __ldg(v_src + src);
      k_dst[o] = kv;
      v_dst[o] = vv;
    } else {
      const uint4 z = make_uint4(0, 0, 0, 0);
      k_dst[o] = z;
      v_dst[o] = z;
    }
  }
}

}  // namespace
}  // namespace fkv

extern "C" int fkv_compact(const void* k_src, const void* v_src, int32_t T, int32_t n_segments,
                           const int64_t* offsets, const int32_t* idx, const int32_t* seg_bh,
                           const int32_t* seg_lo, const int32_t* seg_hi, const int64_t* seg_row0,
                           int32_t zero_pad, void* k_dst, void* v_dst, void* stream) {
  using namespace fkv;
  if (n_segments < 0 || T < 0) return set_error(FKV_ERR_INVALID, "fkv_compact: bad sizes");
  if (n_segments == 0) return FKV_OK;
  if (!k_src || !v_src || !offsets || !idx || !seg_bh || !seg_lo || !seg_hi || !seg_row0 ||
      !k_dst || !v_dst)
    return set_error(FKV_ERR_INVALID, "fkv_compact: null pointer");
  if ((reinterpret_cast<uintptr_t>(k_src) | reinterpret_cast<uintptr_t>(v_src) |
       reinterpret_cast<uintptr_t>(k_dst) | reinterpret_cast<uintptr_t>(v_dst)) & 15)
    return set_error(FKV_ERR_INVALID, "fkv_compact: buffers must be 16-byte aligned");
  compact_kernel<<<n_segments, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(k_src), static_cast<const uint4*>(v_src), T, offsets, idx, seg_bh,
      seg_lo, seg_hi, seg_row0, zero_pad, static_cast<uint4*>(k_dst), static_cast<uint4*>(v_dst));
  return cuda_check(cudaGetLastError(), "compact launch");
}

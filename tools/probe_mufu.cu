// MUFU ex2 throughput on this GPU: every thread runs 8 independent chains of
// ex2.approx.ftz.f32, timed with events.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* out, int iters) {
  float x[8];
  for (int j = 0; j < 8; ++j) x[j] = -1e-3f * (threadIdx.x + j);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[j]));
  float s = 0.f;
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.f) out[0] = s;
}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* d;
  cudaMalloc(&d, 4);
  const int iters = 4096, blocks = sms * 4, threads = 512;
  k<<<blocks, threads>>>(d, 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<blocks, threads>>>(d, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double ops = double(blocks) * threads * iters * 8;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"ex2_per_s\": %.4e, \"per_sm_per_clk_at_max_clock\": %.2f, \"sms\": %d, \"ms\": %.3f}\n",
         ops / (ms * 1e-3), ops / (ms * 1e-3) / sms / (clk * 1e3), sms, ms);
  return 0;
}

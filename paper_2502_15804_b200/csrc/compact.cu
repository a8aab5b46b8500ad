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

constexpr int kRowsPerCta = 64;  // 16 half-warps x 4 rows

// grid = (row blocks, segments): CTA (x, s) moves rows [64x, 64x+64) of
// segment s, so even a handful of long segments spreads over every SM.
__global__ void __launch_bounds__(kThreads)
    compact_kernel(const uint4* __restrict__ k_src, const uint4* __restrict__ v_src, int T,
                   const int64_t* __restrict__ offsets, const int32_t* __restrict__ idx,
                   const int32_t* __restrict__ seg_bh, const int32_t* __restrict__ seg_lo,
                   const int32_t* __restrict__ seg_hi, const int64_t* __restrict__ seg_row0,
                   int zero_pad, uint4* __restrict__ k_dst, uint4* __restrict__ v_dst) {
  const int s = blockIdx.y;
  const int lo = seg_lo[s], hi = seg_hi[s];
  const int n = hi - lo;
  const int rows = zero_pad ? (n + FKV_PAGE - 1) / FKV_PAGE * FKV_PAGE : n;
  const int r_begin = blockIdx.x * kRowsPerCta;
  if (r_begin >= rows) return;
  const int bh = seg_bh[s];
  const int64_t row0 = seg_row0[s];
  const int32_t* sel = idx + offsets[bh] + lo;
  const int64_t src_base = static_cast<int64_t>(bh) * T;  // row index of (b, h, token 0)
  const int half = threadIdx.x >> 4;                        // 16 half-warps per CTA
  const int c = threadIdx.x & 15;                           // 16-byte chunk of the row
  const int r_end = min(rows, r_begin + kRowsPerCta);
  // issue every load of this CTA's rows before any store (4 rows per half-warp in flight)
  uint4 kv[4], vv[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int r = r_begin + half + 16 * u;
    if (r < min(r_end, n)) {
      const int64_t src = (src_base + __ldg(sel + r)) * 16 + c;
      kv[u] = __ldg(k_src + src);
      vv[u] = __ldg(v_src + src);
    } else {
      kv[u] = vv[u] = make_uint4(0, 0, 0, 0);
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int r = r_begin + half + 16 * u;
    if (r < r_end) {
      const int64_t dst = row0 + r;
      const int64_t o = dst * 16 + (c ^ static_cast<int>(dst & 7));
      k_dst[o] = kv[u];
      v_dst[o] = vv[u];
    }
  }
}

}  // namespace
}  // namespace fkv

extern "C" int fkv_compact(const void* k_src, const void* v_src, int32_t T, int32_t n_segments,
                           const int64_t* offsets, const int32_t* idx, const int32_t* seg_bh,
                           const int32_t* seg_lo, const int32_t* seg_hi, const int64_t* seg_row0,
                           int32_t zero_pad, int32_t max_tokens, void* k_dst, void* v_dst,
                           void* stream) {
  using namespace fkv;
  if (n_segments < 0 || T < 0 || max_tokens < 0)
    return set_error(FKV_ERR_INVALID, "fkv_compact: bad sizes");
  max_tokens = (max_tokens + FKV_PAGE - 1) / FKV_PAGE * FKV_PAGE;  // padding rows too
  if (max_tokens == 0) max_tokens = FKV_PAGE;
  if (n_segments == 0) return FKV_OK;
  if (!k_src || !v_src || !offsets || !idx || !seg_bh || !seg_lo || !seg_hi || !seg_row0 ||
      !k_dst || !v_dst)
    return set_error(FKV_ERR_INVALID, "fkv_compact: null pointer");
  if ((reinterpret_cast<uintptr_t>(k_src) | reinterpret_cast<uintptr_t>(v_src) |
       reinterpret_cast<uintptr_t>(k_dst) | reinterpret_cast<uintptr_t>(v_dst)) & 15)
    return set_error(FKV_ERR_INVALID, "fkv_compact: buffers must be 16-byte aligned");
  // rows per segment are bounded by the host's layout; size the grid for the longest
  dim3 grid((max_tokens + kRowsPerCta - 1) / kRowsPerCta, n_segments);
  compact_kernel<<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(k_src), static_cast<const uint4*>(v_src), T, offsets, idx, seg_bh,
      seg_lo, seg_hi, seg_row0, zero_pad, static_cast<uint4*>(k_dst), static_cast<uint4*>(v_dst));
  return cuda_check(cudaGetLastError(), "compact launch");
}

// ---------------------------------------------------------------- append ----
// Decode-time growth of the compressed cache: every segment that owns the end
// of its head's token axis (a whole head, or the last AHA-DP copy) gets the
// step's new K/V row.  One half-warp per segment: the 256-B row is stored
// swizzled at cache row row0[s] + len[s] (the segment's reserved headroom),
// then lane 0 bumps len[s] and the n_tok of the segment's last piece in the
// decode work table, so the next fkv_decode sees the token with no host
// round trip.  A segment at capacity is left unchanged and flagged in
// *overflow (the host re-lays the cache out).
namespace fkv {
namespace {
__global__ void __launch_bounds__(256)
    append_kernel(const uint4* __restrict__ k_new, const uint4* __restrict__ v_new,
                  const int32_t* __restrict__ src_row, const int64_t* __restrict__ seg_row0,
                  int32_t* __restrict__ seg_len, const int32_t* __restrict__ seg_cap,
                  int32_t* __restrict__ work_ntok, const int32_t* __restrict__ last_piece,
                  int n_segments, int32_t* __restrict__ overflow, uint4* __restrict__ k_dst,
                  uint4* __restrict__ v_dst) {
  const int s = blockIdx.x * 16 + (threadIdx.x >> 4);
  const int c = threadIdx.x & 15;
  if (s >= n_segments) return;
  const int src = src_row[s];
  if (src < 0) return;  // this segment does not own the end of its head
  const int len = seg_len[s];
  if (len >= seg_cap[s]) {
    if (c == 0) atomicAdd(overflow, 1);
    return;
  }
  const uint4 kv = __ldg(k_new + static_cast<int64_t>(src) * 16 + c);
  const uint4 vv = __ldg(v_new + static_cast<int64_t>(src) * 16 + c);
  const int64_t dst = seg_row0[s] + len;
  const int64_t o = dst * 16 + (c ^ static_cast<int>(dst & 7));
  k_dst[o] = kv;
  v_dst[o] = vv;
  if (c == 0) {
    seg_len[s] = len + 1;
    work_ntok[static_cast<int64_t>(last_piece[s]) * 8] += 1;  // fkv_work_t.n_tok (int32 #2)
  }
}
}  // namespace
}  // namespace fkv

extern "C" int fkv_append(const void* k_new, const void* v_new, const int32_t* src_row,
                          const int64_t* seg_row0, int32_t* seg_len, const int32_t* seg_cap,
                          void* work, const int32_t* last_piece, int32_t n_segments,
                          int32_t* overflow, void* k_dst, void* v_dst, void* stream) {
  using namespace fkv;
  if (n_segments < 0) return set_error(FKV_ERR_INVALID, "fkv_append: bad sizes");
  if (n_segments == 0) return FKV_OK;
  if (!k_new || !v_new || !src_row || !seg_row0 || !seg_len || !seg_cap || !work || !last_piece ||
      !overflow || !k_dst || !v_dst)
    return set_error(FKV_ERR_INVALID, "fkv_append: null pointer");
  if ((reinterpret_cast<uintptr_t>(k_new) | reinterpret_cast<uintptr_t>(v_new) |
       reinterpret_cast<uintptr_t>(k_dst) | reinterpret_cast<uintptr_t>(v_dst)) & 15)
    return set_error(FKV_ERR_INVALID, "fkv_append: buffers must be 16-byte aligned");
  append_kernel<<<(n_segments + 15) / 16, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(k_new), static_cast<const uint4*>(v_new), src_row, seg_row0, seg_len,
      seg_cap, static_cast<int32_t*>(work) + 2, last_piece, n_segments, overflow,
      static_cast<uint4*>(k_dst), static_cast<uint4*>(v_dst));
  return cuda_check(cudaGetLastError(), "append launch");
}

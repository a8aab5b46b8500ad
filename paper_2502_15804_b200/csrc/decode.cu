// K4 + K5(local): split-KV decode attention over the ragged, swizzled,
// page-aligned compressed cache, and the log-sum-exp merge.
//
// No reference implementation exists; the reference only models
// this kernel's time as c0 + c1*B + c2*C + c3*B*C (pkg/src/headbalance/latency.py:85-91).
//
// Design:
//  * one CTA = 4 warps = one work item (a chunk of one segment); each warp
//    owns every 4th 16-token tile of the chunk and runs its own 3-stage TMA
//    bulk-copy ring (cp.async.bulk + mbarrier): no CTA barrier in the loop;
//  * the cache rows are stored pre-swizzled in HBM, so a 1-D bulk copy lands
//    a bank-conflict-free tile for ldmatrix -- no tensor map, no address math;
//  * GQA: every K/V tile is read once for all G query heads.  S^T = K Q^T
//    (m16n8k16: 16 tokens x 8 heads, no padding waste for G=8), online
//    softmax per head column (warp-shuffle max), P^T via movmatrix, then
//    O^T += V^T P^T with ldmatrix.trans on the V tile;
//  * 4 warp partials merge through shared memory into one (o, lse) partial
//    per item; K5 merges items of a segment (and, after the all-gather,
//    DP copies of a head) by log-sum-exp.
#include <cuda_bf16.h>
#include <math_constants.h>

#include "common.cuh"

namespace fkv {
namespace {

constexpr int kWarps = 4;
constexpr int kStages = 3;
constexpr int kTileTok = 16;
constexpr int kTileBytes = kTileTok * FKV_HEAD_DIM * 2;  // 4 KiB per K or V tile
constexpr int kWarpSmem = kStages * 2 * kTileBytes;      // 24 KiB
constexpr int kSmemBytes = kWarps * kWarpSmem;           // 96 KiB
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

template <int G>
__global__ void __launch_bounds__(kWarps * 32, 2)
    decode_partial_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ kc,
                          const __nv_bfloat16* __restrict__ vc, const int64_t* __restrict__ seg_row0,
                          const int32_t* __restrict__ seg_len, const int32_t* __restrict__ seg_qrow,
                          const int32_t* __restrict__ item_seg, const int32_t* __restrict__ item_t0,
                          const int32_t* __restrict__ item_t1, float scale_log2,
                          float* __restrict__ part_o, float* __restrict__ part_lse) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[kWarps][kStages];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int item = blockIdx.x;
  const int seg = item_seg[item];
  const int t0 = item_t0[item];
  const int t1 = min(item_t1[item], seg_len[seg]);
  const int64_t row0 = seg_row0[seg];
  const __nv_bfloat16* kseg = kc + row0 * FKV_HEAD_DIM;
  const __nv_bfloat16* vseg = vc + row0 * FKV_HEAD_DIM;

  const int n_tiles = t1 > t0 ? (t1 - t0 + kTileTok - 1) / kTileTok : 0;
  const int my_tiles = n_tiles > warp ? (n_tiles - warp + kWarps - 1) / kWarps : 0;
  uint8_t* wsm = smem + warp * kWarpSmem;

  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[warp][s], 1);
    fence_mbar_init();
  }
  __syncwarp();

  auto issue = [&](int i) {  // lane 0 only: tile i of this warp into stage i % kStages
    const int s = i % kStages;
    const int ts = t0 + kTileTok * (warp + kWarps * i);
    uint8_t* dst = wsm + s * 2 * kTileBytes;
    mbar_arrive_expect_tx(&bars[warp][s], 2 * kTileBytes);
    bulk_g2s(dst, kseg + static_cast<int64_t>(ts) * FKV_HEAD_DIM, kTileBytes, &bars[warp][s]);
    bulk_g2s(dst + kTileBytes, vseg + static_cast<int64_t>(ts) * FKV_HEAD_DIM, kTileBytes,
             &bars[warp][s]);
  };
  if (lane == 0)
    for (int i = 0; i < my_tiles && i < kStages; ++i) issue(i);

  // Q^T as the B operand (k = head_dim, n = query head of the group), kept in
  // registers for the whole item.
  uint32_t qb[8][2];
  {
    const int n = lane >> 2;
    const int kq = 2 * (lane & 3);
    if (n < G) {
      const __nv_bfloat16* qr = q + static_cast<int64_t>(seg_qrow[seg] + n) * FKV_HEAD_DIM;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        qb[kk][0] = *reinterpret_cast<const uint32_t*>(qr + 16 * kk + kq);
        qb[kk][1] = *reinterpret_cast<const uint32_t*>(qr + 16 * kk + 8 + kq);
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) qb[kk][0] = qb[kk][1] = 0u;
    }
  }

  float m0 = -CUDART_INF_F, m1 = -CUDART_INF_F;  // running max (log2 domain), heads h0, h1
  float l0 = 0.f, l1 = 0.f;                      // thread-partial denominators
  float acc[8][4];
#pragma unroll
  for (int dt = 0; dt < 8; ++dt) acc[dt][0] = acc[dt][1] = acc[dt][2] = acc[dt][3] = 0.f;

  const int mi = lane >> 3, ri = lane & 7;
  for (int i = 0; i < my_tiles; ++i) {
    const int s = i % kStages;
    mbar_wait(&bars[warp][s], (i / kStages) & 1);
    const uint32_t kt = smem_u32(wsm + s * 2 * kTileBytes);
    const uint32_t vt = kt + kTileBytes;
    const int tok_base = t0 + kTileTok * (warp + kWarps * i);

    // S^T[16 tok x 8 heads] = K_tile . Q^T
    float sc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t a0, a1, a2, a3;
      ldmatrix_x4(kt + swz_off(ri + 8 * (mi & 1), 2 * kk + (mi >> 1)), a0, a1, a2, a3);
      mma_bf16_16816(sc, a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
    }
    const int ta = tok_base + (lane >> 2);
    const float s0 = ta < t1 ? sc[0] * scale_log2 : -CUDART_INF_F;
    const float s1 = ta < t1 ? sc[1] * scale_log2 : -CUDART_INF_F;
    const float s2 = ta + 8 < t1 ? sc[2] * scale_log2 : -CUDART_INF_F;
    const float s3 = ta + 8 < t1 ? sc[3] * scale_log2 : -CUDART_INF_F;
    float mx0 = fmaxf(s0, s2), mx1 = fmaxf(s1, s3);
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
    }
    const float nm0 = fmaxf(m0, mx0), nm1 = fmaxf(m1, mx1);
    const float r0 = nm0 == -CUDART_INF_F ? 0.f : nm0;
    const float r1 = nm1 == -CUDART_INF_F ? 0.f : nm1;
    const float c0 = fast_exp2(m0 - r0), c1 = fast_exp2(m1 - r1);
    const float p0 = fast_exp2(s0 - r0), p1 = fast_exp2(s1 - r1);
    const float p2 = fast_exp2(s2 - r0), p3 = fast_exp2(s3 - r1);
    l0 = l0 * c0 + p0 + p2;
    l1 = l1 * c1 + p1 + p3;
    m0 = nm0;
    m1 = nm1;
#pragma unroll
    for (int dt = 0; dt < 8; ++dt) {
      acc[dt][0] *= c0;
      acc[dt][1] *= c1;
      acc[dt][2] *= c0;
      acc[dt][3] *= c1;
    }
    // P^T fragments (k = token, n = head) from the S^T accumulator layout
    const uint32_t pb0 = movmatrix_trans(pack_bf16x2(p0, p1));
    const uint32_t pb1 = movmatrix_trans(pack_bf16x2(p2, p3));
    // O^T[128 d x 8 heads] += V^T . P^T
#pragma unroll
    for (int dt = 0; dt < 8; ++dt) {
      uint32_t a0, a1, a2, a3;
      ldmatrix_x4_trans(vt + swz_off(ri + 8 * (mi >> 1), 2 * dt + (mi & 1)), a0, a1, a2, a3);
      mma_bf16_16816(acc[dt], a0, a1, a2, a3, pb0, pb1);
    }
    __syncwarp();
    if (lane == 0 && i + kStages < my_tiles) issue(i + kStages);
  }

#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, off);
    l1 += __shfl_xor_sync(0xffffffffu, l1, off);
  }

  // ---- per-warp partial -> own smem region (all its copies have landed)
  float* wo = reinterpret_cast<float*>(wsm);  // [G][128]
  float* wm = wo + G * FKV_HEAD_DIM;          // [8]
  float* wl = wm + 8;                         // [8]
  const int h0 = 2 * (lane & 3), h1 = h0 + 1;
  const int dr = lane >> 2;
#pragma unroll
  for (int dt = 0; dt < 8; ++dt) {
    if (h0 < G) {
      wo[h0 * FKV_HEAD_DIM + 16 * dt + dr] = acc[dt][0];
      wo[h0 * FKV_HEAD_DIM + 16 * dt + dr + 8] = acc[dt][2];
    }
    if (h1 < G) {
      wo[h1 * FKV_HEAD_DIM + 16 * dt + dr] = acc[dt][1];
      wo[h1 * FKV_HEAD_DIM + 16 * dt + dr + 8] = acc[dt][3];
    }
  }
  if (lane < 4) {
    if (h0 < G) { wm[h0] = m0; wl[h0] = l0; }
    if (h1 < G) { wm[h1] = m1; wl[h1] = l1; }
  }
  __syncthreads();

  // ---- cross-warp log-sum-exp combine: thread = one head_dim column
  const int d = threadIdx.x;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    float M = -CUDART_INF_F;
#pragma unroll
    for (int w = 0; w < kWarps; ++w)
      M = fmaxf(M, reinterpret_cast<const float*>(smem + w * kWarpSmem)[G * FKV_HEAD_DIM + g]);
    float L = 0.f, o = 0.f;
    if (M != -CUDART_INF_F) {
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        const float* b = reinterpret_cast<const float*>(smem + w * kWarpSmem);
        const float f = fast_exp2(b[G * FKV_HEAD_DIM + g] - M);
        L += b[G * FKV_HEAD_DIM + 8 + g] * f;
        o += b[g * FKV_HEAD_DIM + d] * f;
      }
    }
    const int64_t orow = static_cast<int64_t>(item) * G + g;
    part_o[orow * FKV_HEAD_DIM + d] = L > 0.f ? o / L : 0.f;
    if (d == 0) part_lse[orow] = L > 0.f ? (M + log2f(L)) * kLn2 : -CUDART_INF_F;
  }
}

template <int G>
__global__ void __launch_bounds__(128)
    merge_lse_kernel(const float* __restrict__ part_o, const float* __restrict__ part_lse,
                     const int32_t* __restrict__ grp_ptr, const int32_t* __restrict__ src_idx,
                     const int32_t* __restrict__ out_row, __nv_bfloat16* __restrict__ out_bf16,
                     float* __restrict__ out_f32, float* __restrict__ out_lse) {
  const int grp = blockIdx.x;
  const int d = threadIdx.x;
  const int i0 = grp_ptr[grp], i1 = grp_ptr[grp + 1];
  const int64_t row = out_row[grp];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    float M = -CUDART_INF_F;
    for (int i = i0; i < i1; ++i) M = fmaxf(M, part_lse[static_cast<int64_t>(src_idx[i]) * G + g]);
    float S = 0.f, o = 0.f;
    if (M != -CUDART_INF_F) {
      for (int i = i0; i < i1; ++i) {
        const int64_t r = static_cast<int64_t>(src_idx[i]) * G + g;
        const float w = __expf(part_lse[r] - M);
        S += w;
        o += w * part_o[r * FKV_HEAD_DIM + d];
      }
    }
    const float ov = S > 0.f ? o / S : 0.f;
    if (out_bf16) out_bf16[(row + g) * FKV_HEAD_DIM + d] = __float2bfloat16_rn(ov);
    if (out_f32) out_f32[(row + g) * FKV_HEAD_DIM + d] = ov;
    if (out_lse && d == 0) out_lse[row + g] = S > 0.f ? M + __logf(S) : -CUDART_INF_F;
  }
}

template <int G>
int launch_decode(const void* q, const void* k, const void* v, const int64_t* seg_row0,
                  const int32_t* seg_len, const int32_t* seg_qrow, const int32_t* item_seg,
                  const int32_t* item_t0, const int32_t* item_t1, int n_items, float sm_scale,
                  float* part_o, float* part_lse, cudaStream_t st) {
  static bool configured = false;  // idempotent; attribute set is per-function
  if (!configured) {
    if (int rc = cuda_check(cudaFuncSetAttribute(decode_partial_kernel<G>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 kSmemBytes),
                            "decode smem attribute"))
      return rc;
    configured = true;
  }
  decode_partial_kernel<G><<<n_items, kWarps * 32, kSmemBytes, st>>>(
      static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k),
      static_cast<const __nv_bfloat16*>(v), seg_row0, seg_len, seg_qrow, item_seg, item_t0,
      item_t1, sm_scale * kLog2e, part_o, part_lse);
  return cuda_check(cudaGetLastError(), "decode_partial launch");
}

}  // namespace
}  // namespace fkv

extern "C" int fkv_decode_partial(const void* q, const void* k, const void* v,
                                  const int64_t* seg_row0, const int32_t* seg_len,
                                  const int32_t* seg_qrow, const int32_t* item_seg,
                                  const int32_t* item_t0, const int32_t* item_t1, int32_t n_items,
                                  int32_t group, float sm_scale, float* part_o, float* part_lse,
                                  void* stream) {
  using namespace fkv;
  if (n_items < 0) return set_error(FKV_ERR_INVALID, "n_items < 0");
  if (n_items == 0) return FKV_OK;
  if (!q || !k || !v || !seg_row0 || !seg_len || !seg_qrow || !item_seg || !item_t0 || !item_t1 ||
      !part_o || !part_lse)
    return set_error(FKV_ERR_INVALID, "fkv_decode_partial: null pointer");
  if ((reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15)
    return set_error(FKV_ERR_INVALID, "fkv_decode_partial: cache not 16-byte aligned");
  auto st = static_cast<cudaStream_t>(stream);
  switch (group) {
    case 4:
      return launch_decode<4>(q, k, v, seg_row0, seg_len, seg_qrow, item_seg, item_t0, item_t1,
                              n_items, sm_scale, part_o, part_lse, st);
    case 8:
      return launch_decode<8>(q, k, v, seg_row0, seg_len, seg_qrow, item_seg, item_t0, item_t1,
                              n_items, sm_scale, part_o, part_lse, st);
    default:
      return set_error(FKV_ERR_INVALID, "fkv_decode_partial: group must be 4 or 8");
  }
}

extern "C" int fkv_merge_lse(const float* part_o, const float* part_lse, const int32_t* grp_ptr,
                             const int32_t* src_idx, const int32_t* out_row, int32_t n_groups,
                             int32_t group, void* out_bf16, float* out_f32, float* out_lse,
                             void* stream) {
  using namespace fkv;
  if (n_groups < 0) return set_error(FKV_ERR_INVALID, "n_groups < 0");
  if (n_groups == 0) return FKV_OK;
  if (!part_o || !part_lse || !grp_ptr || !src_idx || !out_row || (!out_bf16 && !out_f32))
    return set_error(FKV_ERR_INVALID, "fkv_merge_lse: null pointer");
  auto st = static_cast<cudaStream_t>(stream);
  auto ob = static_cast<__nv_bfloat16*>(out_bf16);
  switch (group) {
    case 4:
      merge_lse_kernel<4><<<n_groups, 128, 0, st>>>(part_o, part_lse, grp_ptr, src_idx, out_row,
                                                    ob, out_f32, out_lse);
      break;
    case 8:
      merge_lse_kernel<8><<<n_groups, 128, 0, st>>>(part_o, part_lse, grp_ptr, src_idx, out_row,
                                                    ob, out_f32, out_lse);
      break;
    default:
      return set_error(FKV_ERR_INVALID, "fkv_merge_lse: group must be 4 or 8");
  }
  return cuda_check(cudaGetLastError(), "merge_lse launch");
}

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

struct DecodeParams {
  const __nv_bfloat16* q;
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  const int64_t* seg_row0;
  const int32_t* seg_len;
  const int32_t* seg_qrow;
  const int32_t* seg_out_row;
  const int32_t* seg_item_ptr;
  const int32_t* item_seg;
  const int32_t* item_t0;
  const int32_t* item_t1;
  float scale_log2;
  float* part;        // [n_items, G, FKV_REC] partial records (multi-item segments)
  int32_t* counters;  // [n_seg] arrival counters, zero between launches (self-resetting)
  __nv_bfloat16* out_bf16;
  float* out_rec;
  float* out_lse;
};

template <int G>
__global__ void __launch_bounds__(kWarps * 32, 2) decode_kernel(const DecodeParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[kWarps][kStages];
  __shared__ int s_last;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int item = blockIdx.x;
  const int seg = p.item_seg[item];
  const int t0 = p.item_t0[item];
  const int t1 = min(p.item_t1[item], p.seg_len[seg]);
  const int64_t row0 = p.seg_row0[seg];
  const __nv_bfloat16* kseg = p.k + row0 * FKV_HEAD_DIM;
  const __nv_bfloat16* vseg = p.v + row0 * FKV_HEAD_DIM;

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
      const __nv_bfloat16* qr = p.q + static_cast<int64_t>(p.seg_qrow[seg] + n) * FKV_HEAD_DIM;
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
    const float s0 = ta < t1 ? sc[0] * p.scale_log2 : -CUDART_INF_F;
    const float s1 = ta < t1 ? sc[1] * p.scale_log2 : -CUDART_INF_F;
    const float s2 = ta + 8 < t1 ? sc[2] * p.scale_log2 : -CUDART_INF_F;
    const float s3 = ta + 8 < t1 ? sc[3] * p.scale_log2 : -CUDART_INF_F;
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
  float on[G], ls[G];
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
    on[g] = L > 0.f ? o / L : 0.f;
    ls[g] = L > 0.f ? (M + log2f(L)) * kLn2 : -CUDART_INF_F;
  }

  const bool fused = p.out_bf16 || p.out_rec || p.out_lse;
  const int i0 = p.seg_item_ptr[seg];
  const int n_it = p.seg_item_ptr[seg + 1] - i0;
  if (!fused || n_it > 1) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float* rec = p.part + (static_cast<int64_t>(item) * G + g) * FKV_REC;
      rec[d] = on[g];
      if (d == 0) rec[FKV_HEAD_DIM] = ls[g];
    }
  }
  if (!fused) return;
  if (n_it > 1) {
    // last-arriving CTA of the segment merges every chunk's record (K5 fused)
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&p.counters[seg], 1) == n_it - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // Latency-tolerant merge: all (item, head) lse values are fetched in one
    // parallel round trip, weights are formed in shared memory, then every
    // thread streams its head_dim column of all records with independent loads.
    float* s_w = reinterpret_cast<float*>(smem);  // [n_it][G] weights (stage buffers are free)
    float* s_lse = s_w + n_it * G;                // [G] merged lse
    for (int x = threadIdx.x; x < n_it * G; x += blockDim.x)
      s_w[x] = __ldcg(p.part + (static_cast<int64_t>(i0) * G + x) * FKV_REC + FKV_HEAD_DIM);
    __syncthreads();
    if (threadIdx.x < G) {
      const int g = threadIdx.x;
      float M = -CUDART_INF_F;
      for (int i = 0; i < n_it; ++i) M = fmaxf(M, s_w[i * G + g]);
      float S = 0.f;
      if (M != -CUDART_INF_F)
        for (int i = 0; i < n_it; ++i) S += __expf(s_w[i * G + g] - M);
      const float inv = S > 0.f ? 1.f / S : 0.f;
      for (int i = 0; i < n_it; ++i)
        s_w[i * G + g] = M != -CUDART_INF_F ? __expf(s_w[i * G + g] - M) * inv : 0.f;
      s_lse[g] = S > 0.f ? M + __logf(S) : -CUDART_INF_F;
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < G; ++g) on[g] = 0.f;
    const float* base = p.part + static_cast<int64_t>(i0) * G * FKV_REC + d;
#pragma unroll 2
    for (int i = 0; i < n_it; ++i) {
      float v[G];
#pragma unroll
      for (int g = 0; g < G; ++g) v[g] = __ldcg(base + (i * G + g) * FKV_REC);
#pragma unroll
      for (int g = 0; g < G; ++g) on[g] = fmaf(s_w[i * G + g], v[g], on[g]);
    }
#pragma unroll
    for (int g = 0; g < G; ++g) ls[g] = s_lse[g];
    if (threadIdx.x == 0) p.counters[seg] = 0;  // ready for the next launch / graph replay
  }
  const int64_t orow = p.seg_out_row[seg];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (p.out_bf16) p.out_bf16[(orow + g) * FKV_HEAD_DIM + d] = __float2bfloat16_rn(on[g]);
    if (p.out_rec) {
      p.out_rec[(orow + g) * FKV_REC + d] = on[g];
      if (d == 0) p.out_rec[(orow + g) * FKV_REC + FKV_HEAD_DIM] = ls[g];
    }
    if (p.out_lse && d == 0) p.out_lse[orow + g] = ls[g];
  }
}

// K5 standalone (after the all-gather): warp g of the CTA merges head g of
// one output group in a single online-LSE pass; lane = 4 head_dim columns.
template <int G>
__global__ void __launch_bounds__(G * 32)
    merge_lse_kernel(const float* __restrict__ part, const int32_t* __restrict__ grp_ptr,
                     const int32_t* __restrict__ src_idx, const int32_t* __restrict__ out_row,
                     __nv_bfloat16* __restrict__ out_bf16, float* __restrict__ out_rec,
                     float* __restrict__ out_lse) {
  const int grp = blockIdx.x;
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = grp_ptr[grp], i1 = grp_ptr[grp + 1];
  float m = -CUDART_INF_F, S = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = i0; i < i1; ++i) {
    const float* rec = part + (static_cast<int64_t>(src_idx[i]) * G + g) * FKV_REC;
    const float l = rec[FKV_HEAD_DIM];
    if (l == -CUDART_INF_F) continue;
    const float4 o = reinterpret_cast<const float4*>(rec)[lane];
    const float nm = fmaxf(m, l);
    const float a = __expf(m - nm), b = __expf(l - nm);
    S = S * a + b;
    acc.x = acc.x * a + o.x * b;
    acc.y = acc.y * a + o.y * b;
    acc.z = acc.z * a + o.z * b;
    acc.w = acc.w * a + o.w * b;
    m = nm;
  }
  const float inv = S > 0.f ? 1.f / S : 0.f;
  acc.x *= inv;
  acc.y *= inv;
  acc.z *= inv;
  acc.w *= inv;
  const float lse = S > 0.f ? m + __logf(S) : -CUDART_INF_F;
  const int64_t row = static_cast<int64_t>(out_row[grp]) + g;
  if (out_bf16) {
    __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(out_bf16 + row * FKV_HEAD_DIM) + 2 * lane;
    ob[0] = __floats2bfloat162_rn(acc.x, acc.y);
    ob[1] = __floats2bfloat162_rn(acc.z, acc.w);
  }
  if (out_rec) {
    reinterpret_cast<float4*>(out_rec + row * FKV_REC)[lane] = acc;
    if (lane == 0) out_rec[row * FKV_REC + FKV_HEAD_DIM] = lse;
  }
  if (out_lse && lane == 0) out_lse[row] = lse;
}

template <int G>
int launch_decode(const DecodeParams& p, int n_items, cudaStream_t st) {
  static bool configured = false;  // attribute set is per-function, idempotent
  if (!configured) {
    if (int rc = cuda_check(cudaFuncSetAttribute(decode_kernel<G>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 kSmemBytes),
                            "decode smem attribute"))
      return rc;
    configured = true;
  }
  decode_kernel<G><<<n_items, kWarps * 32, kSmemBytes, st>>>(p);
  return cuda_check(cudaGetLastError(), "decode launch");
}

}  // namespace
}  // namespace fkv

extern "C" int fkv_decode(const void* q, const void* k, const void* v, const int64_t* seg_row0,
                          const int32_t* seg_len, const int32_t* seg_qrow,
                          const int32_t* seg_out_row, const int32_t* seg_item_ptr,
                          const int32_t* item_seg, const int32_t* item_t0, const int32_t* item_t1,
                          int32_t n_items, int32_t group, float sm_scale, float* part,
                          int32_t* counters, void* out_bf16, float* out_rec, float* out_lse,
                          void* stream) {
  using namespace fkv;
  if (n_items < 0) return set_error(FKV_ERR_INVALID, "n_items < 0");
  if (n_items == 0) return FKV_OK;
  const bool fused = out_bf16 || out_rec || out_lse;
  if (!q || !k || !v || !seg_row0 || !seg_len || !seg_qrow || !item_seg || !item_t0 || !item_t1 ||
      !part || (fused && (!seg_out_row || !seg_item_ptr || !counters)))
    return set_error(FKV_ERR_INVALID, "fkv_decode: null pointer");
  if ((reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15)
    return set_error(FKV_ERR_INVALID, "fkv_decode: cache not 16-byte aligned");
  DecodeParams p{static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k),
                 static_cast<const __nv_bfloat16*>(v), seg_row0, seg_len, seg_qrow, seg_out_row,
                 seg_item_ptr, item_seg, item_t0, item_t1, sm_scale * kLog2e, part, counters,
                 static_cast<__nv_bfloat16*>(out_bf16), out_rec, out_lse};
  auto st = static_cast<cudaStream_t>(stream);
  switch (group) {
    case 4: return launch_decode<4>(p, n_items, st);
    case 8: return launch_decode<8>(p, n_items, st);
    default: return set_error(FKV_ERR_INVALID, "fkv_decode: group must be 4 or 8");
  }
}

extern "C" int fkv_merge_lse(const float* part, const int32_t* grp_ptr, const int32_t* src_idx,
                             const int32_t* out_row, int32_t n_groups, int32_t group,
                             void* out_bf16, float* out_rec, float* out_lse, void* stream) {
  using namespace fkv;
  if (n_groups < 0) return set_error(FKV_ERR_INVALID, "n_groups < 0");
  if (n_groups == 0) return FKV_OK;
  if (!part || !grp_ptr || !src_idx || !out_row || (!out_bf16 && !out_rec && !out_lse))
    return set_error(FKV_ERR_INVALID, "fkv_merge_lse: null pointer");
  auto st = static_cast<cudaStream_t>(stream);
  auto ob = static_cast<__nv_bfloat16*>(out_bf16);
  switch (group) {
    case 4:
      merge_lse_kernel<4><<<n_groups, 4 * 32, 0, st>>>(part, grp_ptr, src_idx, out_row, ob, out_rec,
                                                    out_lse);
      break;
    case 8:
      merge_lse_kernel<8><<<n_groups, 8 * 32, 0, st>>>(part, grp_ptr, src_idx, out_row, ob, out_rec,
                                                    out_lse);
      break;
    default:
      return set_error(FKV_ERR_INVALID, "fkv_merge_lse: group must be 4 or 8");
  }
  return cuda_check(cudaGetLastError(), "merge_lse launch");
}

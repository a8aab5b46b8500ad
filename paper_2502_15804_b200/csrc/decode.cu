// K4 + fused K5: warp-persistent split-KV decode attention over the ragged,
// swizzled, page-aligned compressed cache, with the log-sum-exp merges.
//
// No reference implementation exists; the reference only models
// this kernel's time as c0 + c1*B + c2*C + c3*B*C (pkg/src/headbalance/latency.py:85-91).
//
// Design:
//  * every warp is an independent persistent worker with a static, host-built
//    schedule: the concatenated 16-token tile stream of all segments is cut
//    into equal ranges, one per worker warp (so every warp streams the same
//    number of bytes), and a warp never synchronises with the other warps of
//    its CTA -- no block barriers anywhere;
//  * each warp runs its own S-stage TMA bulk-copy ring (cp.async.bulk +
//    mbarrier, 16-token K+V tiles of 8 KiB) that streams ACROSS item
//    boundaries: the producer lane lands the first tiles of the next item
//    while the warp is still finishing the current one;
//  * the cache rows are stored pre-swizzled in HBM, so a 1-D bulk copy lands
//    a bank-conflict-free tile for ldmatrix -- no tensor map, no address math;
//  * GQA: every K/V tile is read once for all G query heads.  S^T = K Q^T
//    (m16n8k16: 16 tokens x 8 heads, no padding waste for G=8), online
//    softmax per head column (warp-shuffle max), P^T via movmatrix, then
//    O^T += V^T P^T with ldmatrix.trans on the V tile;
//  * an item's (o, lse) goes straight from registers to its output rows when
//    the segment is one item; otherwise to a partial record, and the last
//    warp to finish one of the segment's items merges them (K5 fused).
#include <cuda_bf16.h>
#include <math_constants.h>

#include "common.cuh"

namespace fkv {
namespace {

constexpr int kWarps = 4;
constexpr int kRingStages = 12;  // per CTA: split over the active warps (12/6/4/3 each)
constexpr int kTileTok = 16;
constexpr int kTileBytes = kTileTok * FKV_HEAD_DIM * 2;  // 4 KiB per K or V tile
constexpr int kSmemBytes = kRingStages * 2 * kTileBytes;  // 96 KiB per CTA
constexpr int kMergeMax = 32;                            // max items per segment (host-enforced)
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
  const int32_t* warp_ptr;   // worker w processes work_list[warp_ptr[w] .. warp_ptr[w+1])
  const int32_t* work_list;  // item ids grouped by worker
  int n_items, n_seg, n_workers;
  float scale_log2;
  float* part;        // [n_items, G, FKV_REC] partial records (multi-item segments)
  int32_t* counters;  // [n_seg] segment arrival counters; zero between launches
  __nv_bfloat16* out_bf16;
  float* out_rec[FKV_MAX_PEERS];  // record destinations: local slots, or every peer's
  int n_rec;                      // receive block for this rank (fused NVLink all-gather)
  float* out_lse;
  int32_t* sig_done;              // warps-finished counter (local), zero between launches
  int32_t* sig_flag[FKV_MAX_PEERS];  // per peer: flags[tp] in that peer's memory
  int n_sig, my_rank;
};

__device__ __forceinline__ void put_rec(const DecodeParams& p, int64_t idx, float v) {
#pragma unroll 1
  for (int j = 0; j < p.n_rec; ++j) p.out_rec[j][idx] = v;
}

__device__ __forceinline__ void put_rec4(const DecodeParams& p, int64_t row, int lane, float4 v) {
#pragma unroll 1
  for (int j = 0; j < p.n_rec; ++j) reinterpret_cast<float4*>(p.out_rec[j] + row * FKV_REC)[lane] = v;
}

__device__ __forceinline__ int n_tiles_of(const DecodeParams& p, int it, int& t0, int& t1,
                                          int& seg) {
  seg = p.item_seg[it];
  t0 = p.item_t0[it];
  t1 = min(p.item_t1[it], p.seg_len[seg]);
  return t1 > t0 ? (t1 - t0 + kTileTok - 1) / kTileTok : 0;
}

template <int G>
__global__ void __launch_bounds__(kWarps * 32, 2) decode_kernel(const DecodeParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[kRingStages];
  __shared__ float scratch[kWarps][kMergeMax * 8];

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // a short schedule leaves warps idle: the active warps split the CTA's 12
  // ring stages, so a lone worker keeps 96 KiB in flight instead of 24 KiB
  const int kStages = kRingStages / static_cast<int>(blockDim.x >> 5);
  uint8_t* ring = smem + warp * kStages * 2 * kTileBytes;
  uint64_t* wbars = bars + warp * kStages;
  // worker ids are spread over CTAs first so a short schedule still uses every SM
  const int worker = warp * gridDim.x + blockIdx.x;
  const int w_beg = worker < p.n_workers ? p.warp_ptr[worker] : 0;
  const int w_end = worker < p.n_workers ? p.warp_ptr[worker + 1] : 0;

  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&wbars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();

  auto item_at = [&](int ord) -> int { return w_beg + ord < w_end ? p.work_list[w_beg + ord] : -1; };

  int p_ord = 0, p_t = 0;  // producer cursor: item ordinal, tile within item
  int p_nt = -1;           // cached tile count / row of the producer's item (-1: reload)
  int64_t p_row = 0;
  uint32_t p_seq = 0, c_seq = 0;
  bool p_done = false;
  auto refill = [&]() {
    while (!p_done && p_seq - c_seq < kStages) {
      if (p_nt < 0) {
        const int it = item_at(p_ord);
        if (it < 0) {
          p_done = true;
          break;
        }
        int t0, t1, seg;
        p_nt = n_tiles_of(p, it, t0, t1, seg);
        p_row = p.seg_row0[seg] + t0;
      }
      if (p_t >= p_nt) {
        ++p_ord;
        p_t = 0;
        p_nt = -1;
        continue;
      }
      if (lane == 0) {
        const int s = p_seq % kStages;
        const int64_t row = p_row + kTileTok * p_t;
        uint8_t* dst = ring + s * 2 * kTileBytes;
        mbar_arrive_expect_tx(&wbars[s], 2 * kTileBytes);
        bulk_g2s(dst, p.k + row * FKV_HEAD_DIM, kTileBytes, &wbars[s]);
        bulk_g2s(dst + kTileBytes, p.v + row * FKV_HEAD_DIM, kTileBytes, &wbars[s]);
      }
      ++p_t;
      ++p_seq;
    }
  };
  refill();

  const int mi = lane >> 3, ri = lane & 7;
  const int h0 = 2 * (lane & 3), h1 = h0 + 1;
  const int dr = lane >> 2;
  const bool fused = p.out_bf16 || p.n_rec > 0 || p.out_lse;

  uint32_t qn[8][2];  // q fragments of the next item, loaded one item ahead
  auto load_q = [&](int it) {
    const int n = lane >> 2, kq = 2 * (lane & 3);
    if (it >= 0 && n < G) {
      const __nv_bfloat16* qr =
          p.q + static_cast<int64_t>(p.seg_qrow[p.item_seg[it]] + n) * FKV_HEAD_DIM;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        qn[kk][0] = __ldg(reinterpret_cast<const unsigned int*>(qr + 16 * kk + kq));
        qn[kk][1] = __ldg(reinterpret_cast<const unsigned int*>(qr + 16 * kk + 8 + kq));
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) qn[kk][0] = qn[kk][1] = 0u;
    }
  };
  // Programmatic dependent launch: everything above (barrier init, schedule
  // reads, the first K/V tiles in flight) touches only the static cache and
  // overlaps the previous kernel's tail; q and every global write come after
  // the previous grid has completed.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  load_q(item_at(0));

  for (int ord = 0;; ++ord) {
    const int it = item_at(ord);
    if (it < 0) break;
    int t0, t1, seg;
    const int nt = n_tiles_of(p, it, t0, t1, seg);

    // Q^T (B operand: k = head_dim, n = query head) was prefetched into qn
    uint32_t qb[8][2];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      qb[kk][0] = qn[kk][0];
      qb[kk][1] = qn[kk][1];
    }

    float m0 = -CUDART_INF_F, m1 = -CUDART_INF_F;  // running max (log2 domain), heads h0, h1
    float l0 = 0.f, l1 = 0.f;                      // thread-partial denominators
    float acc[8][4];
#pragma unroll
    for (int dt = 0; dt < 8; ++dt) acc[dt][0] = acc[dt][1] = acc[dt][2] = acc[dt][3] = 0.f;

    for (int i = 0; i < nt; ++i) {
      const int s = c_seq % kStages;
      mbar_wait(&wbars[s], (c_seq / kStages) & 1);
      const uint32_t kt = smem_u32(ring + s * 2 * kTileBytes);
      const uint32_t vt = kt + kTileBytes;

      // S^T[16 tok x 8 heads] = K_tile . Q^T, two independent accumulation chains
      float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int kk = 0; kk < 8; kk += 2) {
        uint32_t a0, a1, a2, a3, b0, b1, b2, b3;
        ldmatrix_x4(kt + swz_off(ri + 8 * (mi & 1), 2 * kk + (mi >> 1)), a0, a1, a2, a3);
        ldmatrix_x4(kt + swz_off(ri + 8 * (mi & 1), 2 * kk + 2 + (mi >> 1)), b0, b1, b2, b3);
        mma_bf16_16816(sa, a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
        mma_bf16_16816(sb, b0, b1, b2, b3, qb[kk + 1][0], qb[kk + 1][1]);
      }
      const int ta = t0 + kTileTok * i + (lane >> 2);
      const float s0 = ta < t1 ? (sa[0] + sb[0]) * p.scale_log2 : -CUDART_INF_F;
      const float s1 = ta < t1 ? (sa[1] + sb[1]) * p.scale_log2 : -CUDART_INF_F;
      const float s2 = ta + 8 < t1 ? (sa[2] + sb[2]) * p.scale_log2 : -CUDART_INF_F;
      const float s3 = ta + 8 < t1 ? (sa[3] + sb[3]) * p.scale_log2 : -CUDART_INF_F;
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
      ++c_seq;
      refill();
    }

    load_q(item_at(ord + 1));  // overlaps the epilogue below

    // ---- finalise this item from registers
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, off);
      l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f, inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
    const float lse0 = l0 > 0.f ? (m0 + log2f(l0)) * kLn2 : -CUDART_INF_F;
    const float lse1 = l1 > 0.f ? (m1 + log2f(l1)) * kLn2 : -CUDART_INF_F;
    const int i0 = p.seg_item_ptr[seg];
    const int n_it = p.seg_item_ptr[seg + 1] - i0;
    const int64_t orow = p.seg_out_row[seg];

    if (fused && n_it == 1) {
      // whole segment in one item: registers -> output rows
#pragma unroll
      for (int dt = 0; dt < 8; ++dt) {
        const int d0 = 16 * dt + dr;
        if (h0 < G) {
          if (p.out_bf16) {
            p.out_bf16[(orow + h0) * FKV_HEAD_DIM + d0] = __float2bfloat16_rn(acc[dt][0] * inv0);
            p.out_bf16[(orow + h0) * FKV_HEAD_DIM + d0 + 8] = __float2bfloat16_rn(acc[dt][2] * inv0);
          }
          if (p.n_rec) {
            put_rec(p, (orow + h0) * FKV_REC + d0, acc[dt][0] * inv0);
            put_rec(p, (orow + h0) * FKV_REC + d0 + 8, acc[dt][2] * inv0);
          }
        }
        if (h1 < G) {
          if (p.out_bf16) {
            p.out_bf16[(orow + h1) * FKV_HEAD_DIM + d0] = __float2bfloat16_rn(acc[dt][1] * inv1);
            p.out_bf16[(orow + h1) * FKV_HEAD_DIM + d0 + 8] = __float2bfloat16_rn(acc[dt][3] * inv1);
          }
          if (p.n_rec) {
            put_rec(p, (orow + h1) * FKV_REC + d0, acc[dt][1] * inv1);
            put_rec(p, (orow + h1) * FKV_REC + d0 + 8, acc[dt][3] * inv1);
          }
        }
      }
      if (lane < 4) {
        if (h0 < G) {
          if (p.n_rec) put_rec(p, (orow + h0) * FKV_REC + FKV_HEAD_DIM, lse0);
          if (p.out_lse) p.out_lse[orow + h0] = lse0;
        }
        if (h1 < G) {
          if (p.n_rec) put_rec(p, (orow + h1) * FKV_REC + FKV_HEAD_DIM, lse1);
          if (p.out_lse) p.out_lse[orow + h1] = lse1;
        }
      }
      continue;
    }

    // partial record of this item
    float* rec = p.part + static_cast<int64_t>(it) * G * FKV_REC;
#pragma unroll
    for (int dt = 0; dt < 8; ++dt) {
      const int d0 = 16 * dt + dr;
      if (h0 < G) {
        rec[h0 * FKV_REC + d0] = acc[dt][0] * inv0;
        rec[h0 * FKV_REC + d0 + 8] = acc[dt][2] * inv0;
      }
      if (h1 < G) {
        rec[h1 * FKV_REC + d0] = acc[dt][1] * inv1;
        rec[h1 * FKV_REC + d0 + 8] = acc[dt][3] * inv1;
      }
    }
    if (lane < 4) {
      if (h0 < G) rec[h0 * FKV_REC + FKV_HEAD_DIM] = lse0;
      if (h1 < G) rec[h1 * FKV_REC + FKV_HEAD_DIM] = lse1;
    }
    if (!fused) continue;

    // the last warp to finish one of the segment's items merges them all
    __threadfence();
    __syncwarp();
    int last = 0;
    if (lane == 0) last = atomicAdd(&p.counters[seg], 1) == n_it - 1;
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) continue;
    __threadfence();
    // All (item, head) lse values in one parallel round trip, weights in the
    // warp's scratch, then every lane streams its 4 head_dim columns of all
    // records with n_it*G independent 16-B loads.
    const float* base = p.part + static_cast<int64_t>(i0) * G * FKV_REC;
    float* sw = scratch[warp];
    for (int x = lane; x < n_it * G; x += 32) sw[x] = __ldcg(base + x * FKV_REC + FKV_HEAD_DIM);
    __syncwarp();
    float lse_g = -CUDART_INF_F;
    if (lane < G) {
      float M = -CUDART_INF_F;
      for (int i = 0; i < n_it; ++i) M = fmaxf(M, sw[i * G + lane]);
      float S = 0.f;
      if (M != -CUDART_INF_F)
        for (int i = 0; i < n_it; ++i) S += __expf(sw[i * G + lane] - M);
      const float inv = S > 0.f ? 1.f / S : 0.f;
      for (int i = 0; i < n_it; ++i)
        sw[i * G + lane] = M != -CUDART_INF_F ? __expf(sw[i * G + lane] - M) * inv : 0.f;
      lse_g = S > 0.f ? M + __logf(S) : -CUDART_INF_F;
    }
    __syncwarp();
    float4 o[G];
#pragma unroll
    for (int g = 0; g < G; ++g) o[g] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int i = 0; i < n_it; ++i) {
      float4 v4[G];
#pragma unroll
      for (int g = 0; g < G; ++g) v4[g] = __ldcg(reinterpret_cast<const float4*>(base + (i * G + g) * FKV_REC) + lane);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float w = sw[i * G + g];
        o[g].x = fmaf(w, v4[g].x, o[g].x);
        o[g].y = fmaf(w, v4[g].y, o[g].y);
        o[g].z = fmaf(w, v4[g].z, o[g].z);
        o[g].w = fmaf(w, v4[g].w, o[g].w);
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int64_t row = orow + g;
      if (p.out_bf16) {
        __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(p.out_bf16 + row * FKV_HEAD_DIM) + 2 * lane;
        ob[0] = __floats2bfloat162_rn(o[g].x, o[g].y);
        ob[1] = __floats2bfloat162_rn(o[g].z, o[g].w);
      }
      if (p.n_rec) put_rec4(p, row, lane, o[g]);
    }
    if (lane < G) {
      if (p.n_rec) put_rec(p, (orow + lane) * FKV_REC + FKV_HEAD_DIM, lse_g);
      if (p.out_lse) p.out_lse[orow + lane] = lse_g;
    }
    if (lane == 0) p.counters[seg] = 0;  // ready for the next launch / graph replay
  }

  // Fused all-gather completion: the last warp out publishes this rank's
  // records to every peer by bumping its flag there (system-scope release).
  if (p.n_sig > 0) {
    __threadfence_system();
    __syncwarp();
    if (lane == 0 &&
        atomicAdd(p.sig_done, 1) == static_cast<int>(gridDim.x * (blockDim.x >> 5)) - 1) {
      *p.sig_done = 0;
      __threadfence_system();
      for (int j = 0; j < p.n_sig; ++j) atomicAdd_system(p.sig_flag[j] + p.my_rank, 1);
    }
  }
}

// K5 standalone (after the all-gather): warp g of the CTA merges head g of
// one output group in a single online-LSE pass; lane = 4 head_dim columns.
template <int G>
__global__ void __launch_bounds__(G * 32)
    merge_lse_kernel(const float* __restrict__ part, const int32_t* __restrict__ grp_ptr,
                     const int32_t* __restrict__ src_idx, const int32_t* __restrict__ out_row,
                     __nv_bfloat16* __restrict__ out_bf16, float* __restrict__ out_rec,
                     float* __restrict__ out_lse, const int32_t* flags, int tp,
                     int32_t* consumed) {
  // Fused all-gather consumer: wait until every peer has published this
  // layer's records (their flag reached consumed+1), read them from L2.
  __shared__ int s_target;
  if (flags) {
    if (threadIdx.x == 0) {
      const int target = *reinterpret_cast<volatile int32_t*>(consumed) + 1;
      for (int r = 0; r < tp; ++r) {
        int v;
        do {
          asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(flags + r) : "memory");
          if (v < target) __nanosleep(32);
        } while (v < target);
      }
      s_target = target;
    }
    __syncthreads();
    __threadfence_system();
  }
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
  if (flags) {
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(consumed + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      consumed[1] = 0;
      atomicExch(consumed, s_target);  // this layer consumed: next wait targets +1
    }
  }
}

template <int G>
int launch_decode(const DecodeParams& p, cudaStream_t st) {
  static int grid_cap = 0;  // 2 persistent CTAs per SM
  if (!grid_cap) {
    if (int rc = cuda_check(cudaFuncSetAttribute(decode_kernel<G>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 kSmemBytes),
                            "decode smem attribute"))
      return rc;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_kernel<G>, kWarps * 32,
                                                  kSmemBytes);
    grid_cap = sms * (per_sm > 0 ? per_sm : 1);
  }
  // up to 2 CTAs per SM; 1-4 active warps per CTA (worker w -> CTA w % grid)
  const int grid = p.n_workers < grid_cap ? p.n_workers : grid_cap;
  const int wpc = (p.n_workers + grid - 1) / grid;  // 12 stages split 12/6/4/3
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(wpc * 32, 1, 1);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (see kernel)
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cuda_check(cudaLaunchKernelEx(&cfg, decode_kernel<G>, p), "decode launch");
}

}  // namespace
}  // namespace fkv

namespace fkv {
namespace {
int decode_entry(DecodeParams& p, int group, cudaStream_t st) {
  switch (group) {
    case 4: return launch_decode<4>(p, st);
    case 8: return launch_decode<8>(p, st);
    default: return set_error(FKV_ERR_INVALID, "fkv_decode: group must be 4 or 8");
  }
}
}  // namespace
}  // namespace fkv

extern "C" int fkv_decode(const void* q, const void* k, const void* v, const int64_t* seg_row0,
                          const int32_t* seg_len, const int32_t* seg_qrow,
                          const int32_t* seg_out_row, const int32_t* seg_item_ptr,
                          const int32_t* item_seg, const int32_t* item_t0, const int32_t* item_t1,
                          const int32_t* warp_ptr, const int32_t* work_list, int32_t n_workers,
                          int32_t n_items, int32_t n_seg, int32_t group, float sm_scale,
                          float* part, int32_t* counters, void* out_bf16, float* out_rec,
                          float* out_lse, void* stream) {
  return fkv_decode_exchange(q, k, v, seg_row0, seg_len, seg_qrow, seg_out_row, seg_item_ptr,
                             item_seg, item_t0, item_t1, warp_ptr, work_list, n_workers, n_items,
                             n_seg,
                             group, sm_scale, part, counters, out_bf16, out_rec ? &out_rec : nullptr,
                             out_rec ? 1 : 0, out_lse, nullptr, nullptr, 0, 0, stream);
}

extern "C" int fkv_decode_exchange(const void* q, const void* k, const void* v,
                                   const int64_t* seg_row0, const int32_t* seg_len,
                                   const int32_t* seg_qrow, const int32_t* seg_out_row,
                                   const int32_t* seg_item_ptr, const int32_t* item_seg,
                                   const int32_t* item_t0, const int32_t* item_t1,
                                   const int32_t* warp_ptr, const int32_t* work_list,
                                   int32_t n_workers, int32_t n_items,
                                   int32_t n_seg, int32_t group, float sm_scale, float* part,
                                   int32_t* counters, void* out_bf16, float* const* out_recs,
                                   int32_t n_rec, float* out_lse, int32_t* sig_done,
                                   int32_t* const* sig_flags, int32_t n_sig, int32_t my_rank,
                                   void* stream) {
  using namespace fkv;
  if (n_items < 0 || n_seg < 0) return set_error(FKV_ERR_INVALID, "fkv_decode: negative size");
  if (n_rec < 0 || n_rec > FKV_MAX_PEERS || n_sig < 0 || n_sig > FKV_MAX_PEERS)
    return set_error(FKV_ERR_INVALID, "fkv_decode: too many record destinations / peers");
  if (n_items == 0) return FKV_OK;
  if (!q || !k || !v || !seg_row0 || !seg_len || !seg_qrow || !seg_item_ptr || !item_seg ||
      !item_t0 || !item_t1 || !warp_ptr || !work_list || n_workers < 1 || !part || !counters ||
      ((out_bf16 || n_rec || out_lse) && !seg_out_row) || (n_rec && !out_recs) ||
      (n_sig && (!sig_done || !sig_flags)))
    return set_error(FKV_ERR_INVALID, "fkv_decode: null pointer");
  if ((reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15)
    return set_error(FKV_ERR_INVALID, "fkv_decode: cache not 16-byte aligned");
  DecodeParams p{};
  p.q = static_cast<const __nv_bfloat16*>(q);
  p.k = static_cast<const __nv_bfloat16*>(k);
  p.v = static_cast<const __nv_bfloat16*>(v);
  p.seg_row0 = seg_row0;
  p.seg_len = seg_len;
  p.seg_qrow = seg_qrow;
  p.seg_out_row = seg_out_row;
  p.seg_item_ptr = seg_item_ptr;
  p.item_seg = item_seg;
  p.item_t0 = item_t0;
  p.item_t1 = item_t1;
  p.warp_ptr = warp_ptr;
  p.work_list = work_list;
  p.n_items = n_items;
  p.n_seg = n_seg;
  p.n_workers = n_workers;
  p.scale_log2 = sm_scale * kLog2e;
  p.part = part;
  p.counters = counters;
  p.out_bf16 = static_cast<__nv_bfloat16*>(out_bf16);
  for (int j = 0; j < n_rec; ++j) p.out_rec[j] = out_recs[j];
  p.n_rec = n_rec;
  p.out_lse = out_lse;
  p.sig_done = sig_done;
  for (int j = 0; j < n_sig; ++j) p.sig_flag[j] = sig_flags[j];
  p.n_sig = n_sig;
  p.my_rank = my_rank;
  return decode_entry(p, group, static_cast<cudaStream_t>(stream));
}

extern "C" int fkv_merge_lse(const float* part, const int32_t* grp_ptr, const int32_t* src_idx,
                             const int32_t* out_row, int32_t n_groups, int32_t group,
                             void* out_bf16, float* out_rec, float* out_lse, void* stream) {
  return fkv_merge_wait(part, grp_ptr, src_idx, out_row, n_groups, group, out_bf16, out_rec,
                        out_lse, nullptr, 0, nullptr, stream);
}

extern "C" int fkv_merge_wait(const float* part, const int32_t* grp_ptr, const int32_t* src_idx,
                              const int32_t* out_row, int32_t n_groups, int32_t group,
                              void* out_bf16, float* out_rec, float* out_lse,
                              const int32_t* flags, int32_t tp, int32_t* consumed, void* stream) {
  using namespace fkv;
  if (flags && (!consumed || tp < 1 || tp > FKV_MAX_PEERS))
    return set_error(FKV_ERR_INVALID, "fkv_merge_wait: bad flags / consumed / tp");
  if (n_groups < 0) return set_error(FKV_ERR_INVALID, "n_groups < 0");
  if (n_groups == 0) return FKV_OK;
  if (!part || !grp_ptr || !src_idx || !out_row || (!out_bf16 && !out_rec && !out_lse))
    return set_error(FKV_ERR_INVALID, "fkv_merge_lse: null pointer");
  auto st = static_cast<cudaStream_t>(stream);
  auto ob = static_cast<__nv_bfloat16*>(out_bf16);
  switch (group) {
    case 4:
      merge_lse_kernel<4><<<n_groups, 4 * 32, 0, st>>>(part, grp_ptr, src_idx, out_row, ob, out_rec,
                                                       out_lse, flags, tp, consumed);
      break;
    case 8:
      merge_lse_kernel<8><<<n_groups, 8 * 32, 0, st>>>(part, grp_ptr, src_idx, out_row, ob, out_rec,
                                                       out_lse, flags, tp, consumed);
      break;
    default:
      return set_error(FKV_ERR_INVALID, "fkv_merge_lse: group must be 4 or 8");
  }
  return cuda_check(cudaGetLastError(), "merge_lse launch");
}

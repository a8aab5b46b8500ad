// K1: Ada-SnapKV observation-window scoring on the 5th-gen tensor cores.
//
// No reference implementation exists (the paper used KVPress
// SnapKV/AdaKV).  Definition (oracle/kv.py):
//   P[r,:]  = softmax_t(q_r . k_t / sqrt(d)), r = (g, i) over the G*w window
//             rows of one KV head, causal inside the window
//   raw[t]  = (1/G) sum_r P[r,t]              t < T - w
//   s[t]    = max(raw[t-3 .. t+3])            (pooling kernel below)
//
// Two tcgen05 passes over K, each CTA owning (request, KV head, key chunk):
//   pass 1  D[GW rows x 128 keys]   = Q_win . K_tile^T  -> per-row online max
//           and sum-exp with rows in TMEM lanes (thread-local reductions);
//   pass 2  D^T[128 keys x GW rows] = K_tile . Q_win^T  -> per-key column
//           sums of exp(s - m_r)/l_r with keys in TMEM lanes (thread-local).
// Q_win (GW = G*w = 128 or 256 rows) is TMA-loaded once per CTA and stays in
// shared memory; K tiles (128 keys x 128 d, 32 KiB) stream through a 3-stage
// TMA ring with 128-B swizzle; one elected thread issues
// tcgen05.mma.cta_group::1.kind::f16 (M=128, N=128 or GW, K=16) into a
// double-buffered fp32 TMEM accumulator; eight epilogue warps drain it with
// tcgen05.ld (warp e reads TMEM lanes 32*(e%4) and half e/4 of the columns).
// Warp roles: 0-7 epilogue, 8 TMA producer, 9 MMA issuer.  Grid: one wave
// of one CTA per SM ((Bt*Hkv) x chunks <= #SMs when possible).
// The second pass re-reads K mostly from L2 (a layer's K for one request is
// 32 MiB at 16k context, well inside the 126 MB L2).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include "common.cuh"

namespace fkv {
namespace {

constexpr int kBN = 128;                 // keys per tile
constexpr int kStages = 3;
constexpr int kTileBytes = kBN * 256;    // 128 keys x 128 d x bf16
constexpr int kEpiWarps = 8;
constexpr int kTmaWarp = kEpiWarps, kMmaWarp = kEpiWarps + 1;
constexpr int kThreads = 32 * (kEpiWarps + 2);
constexpr float kLog2e = 1.4426950408889634f;

struct ScoreParams {
  int T, window, group, hkv, n_chunks, tiles_per_chunk;
  int q_rows_per_req;  // Hq * w
  float scale_log2;    // log2(e) / sqrt(d)
  float* stats;        // [Bt*Hkv, n_chunks, GW, 2] (max, sum) in log2 units
  float* raw;          // [Bt*Hkv, T - w]
  float* scores;       // pooled output (fused mode)
  int pool_r;          // pooling radius (pool_k / 2)
  struct GridBar* gridbar;  // fused mode: zeroed counter + generation
};

// ------------------------------------------------------------ tcgen05 ----
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)),
               "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
}

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 32 consecutive fp32 TMEM columns of this thread's lane.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// Same, with an L2 eviction-priority policy (createpolicy): pass 1 keeps K in
// L2 for pass 2 (evict_last), pass 2 streams it out (evict_first).
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int x, int y,
                                                 uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t l2_policy(bool keep) {
  uint64_t pol;
  if (keep)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// K-major, 128-B swizzled UMMA shared-memory descriptor (rows of 128 B,
// 8-row core groups 1024 B apart).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3fff);
  d |= static_cast<uint64_t>(1) << 16;             // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;     // SBO
  d |= static_cast<uint64_t>(1) << 46;             // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;             // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: BF16 x BF16 -> F32, both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

template <int GW>
struct __align__(1024) ScoreSmem {
  __nv_bfloat16 q[2][GW][64];                 // [d-half][row][64], 128-B swizzled by TMA
  __nv_bfloat16 k[kStages][2][kBN][64];
  uint64_t full[kStages], empty[kStages], tfull[2], tempty[2], qbar;
  uint32_t tmem_base;
  alignas(16) float bias[GW];  // pass 2: per query row, m_r + log2(G * l_r) (log2 units)
  float red[2][2][kBN];      // pass 2: [tile parity][column half][key] partial sums
  float ml[kBN][2];          // pass 1, GW=128: second column half's (max, sum) per row
};

struct GridBar {
  unsigned count, gen;
};

// Grid-wide barrier among the epilogue warps of co-resident CTAs (cooperative
// launch); the TMA and MMA warps keep streaming while the epilogue waits.
__device__ __forceinline__ void epi_grid_sync(GridBar* gb) {
  asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps));
  if (threadIdx.x == 0) {
    const unsigned g = *reinterpret_cast<volatile unsigned*>(&gb->gen);
    __threadfence();
    if (atomicAdd(&gb->count, 1) == gridDim.x * gridDim.y - 1) {
      gb->count = 0;
      __threadfence();
      atomicAdd(&gb->gen, 1);
    } else {
      while (*reinterpret_cast<volatile unsigned*>(&gb->gen) == g) __nanosleep(64);
    }
    __threadfence();
  }
  asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps));
}

// MODE 1: pass 1 only; MODE 2: pass 2 only; MODE 3: both passes + pooling in
// one cooperative launch (stats combined after a grid barrier, K re-read from
// L2, raw scores pooled after a second barrier).
template <int MODE, int GW>
__global__ void __launch_bounds__(kThreads, 1)
    score_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                 const ScoreParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  ScoreSmem<GW>& sm = *reinterpret_cast<ScoreSmem<GW>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  constexpr uint32_t kCols = 2 * GW;  // two accumulator buffers of GW fp32 columns
  constexpr bool kP1 = MODE != 2, kP2 = MODE != 1;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.y, chunk = blockIdx.x;
  const int b = bh / p.hkv, h = bh - b * p.hkv;
  const int n = p.T - p.window;
  const int nt1 = (p.T + kBN - 1) / kBN, nt2 = (n + kBN - 1) / kBN;
  const int a1 = chunk * p.tiles_per_chunk, e1 = kP1 ? min(a1 + p.tiles_per_chunk, nt1) : a1;
  const int a2 = chunk * p.tiles_per_chunk, e2 = kP2 ? min(a2 + p.tiles_per_chunk, nt2) : a2;
  const int n1 = max(e1 - a1, 0), n2 = max(e2 - a2, 0);  // tiles of each pass; iterations continue
  const int krow0 = bh * p.T;
  const int qrow0 = b * p.q_rows_per_req + h * GW;

  if (warp == kTmaWarp && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_q)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_k)) : "memory");
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.tfull[i], 1);
      mbar_init(&sm.tempty[i], kEpiWarps);
    }
    mbar_init(&sm.qbar, 1);
    fence_mbar_init();
  }
  if (warp == kMmaWarp) tmem_alloc(&sm.tmem_base, kCols);

  // combine every chunk's pass-1 statistics (log2 domain) into per-row biases
  auto combine_stats = [&]() {
    for (int r = threadIdx.x; r < GW; r += 32 * kEpiWarps) {
      float M = -CUDART_INF_F, L = 0.f;
      const float* st = p.stats + (static_cast<int64_t>(bh) * p.n_chunks) * GW * 2;
      for (int c = 0; c < p.n_chunks; ++c) {
        const float m = __ldcg(st + (c * GW + r) * 2), l = __ldcg(st + (c * GW + r) * 2 + 1);
        if (l <= 0.f) continue;
        const float nm = fmaxf(M, m);
        L = L * exp2f(M - nm) + l * exp2f(m - nm);
        M = nm;
      }
      // exp2(s*c - m) / (G*l) == exp2(s*c - bias): one FFMA + one MUFU per score
      sm.bias[r] = L > 0.f ? M + log2f(L * static_cast<float>(p.group)) : CUDART_INF_F;
    }
  };
  if (MODE == 2 && warp < kEpiWarps) combine_stats();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == kTmaWarp) {
    // ------------------------------------------------ TMA producer ----
    if (lane == 0 && n1 + n2 > 0) {
      mbar_arrive_expect_tx(&sm.qbar, GW * 256);
      for (int c = 0; c < 2; ++c)
        for (int rh = 0; rh < GW / 128; ++rh)
          tma_load_2d(&sm.q[c][rh * 128][0], &tm_q, 64 * c, qrow0 + 128 * rh, &sm.qbar);
      const uint64_t keep = l2_policy(true), stream = l2_policy(false);
      for (int it = 0; it < n1 + n2; ++it) {
        const bool p1 = it < n1;
        const int j = p1 ? a1 + it : a2 + (it - n1);
        const int s = it % kStages;
        mbar_wait(&sm.empty[s], ((it / kStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.full[s], kTileBytes);
        for (int c = 0; c < 2; ++c)
          tma_load_2d_hint(&sm.k[s][c][0][0], &tm_k, 64 * c, krow0 + j * kBN, &sm.full[s],
                           p1 ? keep : stream);
      }
    }
  } else if (warp == kMmaWarp) {
    // -------------------------------------------------- MMA issuer ----
    if (lane == 0 && n1 + n2 > 0) {
      mbar_wait(&sm.qbar, 0);
      constexpr uint32_t kIdesc1 = idesc_bf16(128, kBN);
      constexpr uint32_t kIdesc2 = idesc_bf16(128, GW);
      const uint32_t q_base = smem_u32(&sm.q[0][0][0]);
      for (int it = 0; it < n1 + n2; ++it) {
        const int s = it % kStages, buf = it & 1;
        mbar_wait(&sm.full[s], (it / kStages) & 1);
        mbar_wait(&sm.tempty[buf], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t k_base = smem_u32(&sm.k[s][0][0][0]);
        const uint32_t d_buf = tmem + buf * GW;
        const bool p1 = it < n1;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t koff = (kk >> 2) * (kBN * 128) + (kk & 3) * 32;
          const uint32_t qoff = (kk >> 2) * (GW * 128) + (kk & 3) * 32;
          if (p1) {
#pragma unroll
            for (int mh = 0; mh < GW / 128; ++mh)
              umma_bf16(d_buf + mh * kBN, sw128_desc(q_base + qoff + mh * 128 * 128),
                        sw128_desc(k_base + koff), kIdesc1, kk > 0);
          } else {
            umma_bf16(d_buf, sw128_desc(k_base + koff), sw128_desc(q_base + qoff), kIdesc2, kk > 0);
          }
        }
        umma_commit(&sm.empty[s]);
        umma_commit(&sm.tfull[buf]);
      }
    }
  } else {
    // ---------------------------------------------------- epilogue ----
    const int quad = warp & 3, half = warp >> 2;
    const uint32_t lane_base = static_cast<uint32_t>(32 * quad) << 16;
    if (kP1) {
      // GW=256: warp half = row half (one whole row per thread);
      // GW=128: warp half = column half (per-row partials, combined at the end)
      constexpr int MH = GW / 128;
      const int mh = MH == 2 ? half : 0;
      const int cb0 = MH == 2 ? 0 : 2 * half, cb1 = MH == 2 ? 4 : 2 * half + 2;
      const int r = mh * 128 + 32 * quad + lane;
      const int limit = min(p.T - 1, p.T - p.window + (r % p.window));  // last visible key
      float m = -CUDART_INF_F, l = 0.f;
      for (int it = 0; it < n1; ++it) {
        const int buf = it & 1;
        mbar_wait(&sm.tfull[buf], (it >> 1) & 1);
        tc_fence_after();
        const int ts = (a1 + it) * kBN;
#pragma unroll 1
        for (int cb = cb0; cb < cb1; ++cb) {
          float v[32];
          tmem_ld32(tmem + lane_base + buf * GW + mh * kBN + cb * 32, v);
          const int c0 = ts + cb * 32;
          float bmax = -CUDART_INF_F;
          if (c0 + 31 > limit) {  // only the window's tiles (and the tail) need masking
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              v[i] = c0 + i <= limit ? v[i] : -CUDART_INF_F;
              bmax = fmaxf(bmax, v[i]);
            }
            if (bmax == -CUDART_INF_F) continue;
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) bmax = fmaxf(bmax, v[i]);
          }
          // running max kept in raw-score units, exponents via one FFMA each
          const float nm = fmaxf(m, bmax);
          const float nms = nm * p.scale_log2;
          float acc = 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i) acc += fast_exp2(fmaf(v[i], p.scale_log2, -nms));
          l = l * fast_exp2((m - nm) * p.scale_log2) + acc;
          m = nm;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.tempty[buf]);
      }
      m = m == -CUDART_INF_F ? m : m * p.scale_log2;  // to log2 units
      if (MH == 1) {
        if (half == 1) {
          sm.ml[32 * quad + lane][0] = m;
          sm.ml[32 * quad + lane][1] = l;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps));
        if (half == 0) {
          const float m1 = sm.ml[32 * quad + lane][0], l1 = sm.ml[32 * quad + lane][1];
          const float nm = fmaxf(m, m1);
          if (nm != -CUDART_INF_F) {
            l = l * exp2f(m - nm) + l1 * exp2f(m1 - nm);
            m = nm;
          }
        }
      }
      if (MH == 2 || half == 0) {
        float* st = p.stats + ((static_cast<int64_t>(bh) * p.n_chunks + chunk) * GW + r) * 2;
        st[0] = m;
        st[1] = l;
      }
    }
    if (MODE == 3) {
      epi_grid_sync(p.gridbar);  // every chunk's statistics are in global memory
      combine_stats();
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps));
    }
    if (kP2) {
      const int key = 32 * quad + lane;
      for (int i2 = 0; i2 < n2; ++i2) {
        const int it = n1 + i2, buf = it & 1;
        mbar_wait(&sm.tfull[buf], (it >> 1) & 1);
        tc_fence_after();
        float acc = 0.f;
#pragma unroll 1
        for (int cb = half * (GW / 64); cb < (half + 1) * (GW / 64); ++cb) {
          float v[32];
          tmem_ld32(tmem + lane_base + buf * GW + cb * 32, v);
          const float4* b4 = reinterpret_cast<const float4*>(sm.bias + cb * 32);
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 bb = b4[i / 4];  // broadcast: every lane reads the same columns
            acc += fast_exp2(fmaf(v[i], p.scale_log2, -bb.x));
            acc += fast_exp2(fmaf(v[i + 1], p.scale_log2, -bb.y));
            acc += fast_exp2(fmaf(v[i + 2], p.scale_log2, -bb.z));
            acc += fast_exp2(fmaf(v[i + 3], p.scale_log2, -bb.w));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.tempty[buf]);
        sm.red[it & 1][half][key] = acc;
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps));
        const int t = (a2 + i2) * kBN + key;
        if (half == 0 && t < n)
          p.raw[static_cast<int64_t>(bh) * n + t] = acc + sm.red[it & 1][1][key];
      }
    }
    if (MODE == 3) {
      epi_grid_sync(p.gridbar);  // every raw column score is in global memory
      const float* rr = p.raw + static_cast<int64_t>(bh) * n;
      float* out = p.scores + static_cast<int64_t>(bh) * n;
      const int t_end = min(e2 * kBN, n);
      for (int t = a2 * kBN + threadIdx.x; t < t_end; t += 32 * kEpiWarps) {
        float mx = __ldcg(rr + t);
        const int lo = max(0, t - p.pool_r), hi = min(n - 1, t + p.pool_r);
        for (int u = lo; u <= hi; ++u) mx = fmaxf(mx, __ldcg(rr + u));
        out[t] = mx;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem, kCols);
  }
}

// Max-pool (kernel pool_k, stride 1, -inf padding) of the raw column scores.
__global__ void pool_kernel(const float* __restrict__ raw, float* __restrict__ out, int n,
                            int radius, int64_t total) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int64_t row = i / n;
  const int t = static_cast<int>(i - row * n);
  const float* r = raw + row * n;
  float m = r[t];
  const int lo = max(0, t - radius), hi = min(n - 1, t + radius);
  for (int u = lo; u <= hi; ++u) m = fmaxf(m, r[u]);
  out[i] = m;
}

// ------------------------------------------------------- host helpers ----
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(ptr);
  }
  return fn;
}

// rows x 128 bf16 matrix, box = 64 columns x box_rows rows, 128-B swizzle.
int make_map(CUtensorMap* map, const void* base, int64_t rows, int box_rows) {
  EncodeTiled enc = encoder();
  if (!enc) return set_error(FKV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {256};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(FKV_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return FKV_OK;
}

}  // namespace

// Key chunks per (request, KV head): one wave of one CTA per SM when the
// heads alone do not fill the GPU; never more chunks than tiles.
int score_chunks(int bh, int n_tiles) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
      sms = 148;
  }
  int c = sms / bh;
  if (c < 1) c = 1;
  return c > n_tiles ? n_tiles : c;
}

namespace {

template <int GW>
int launch_score(const CUtensorMap& tq, const CUtensorMap& tk, const ScoreParams& p, int batch_heads,
                 bool fused, cudaStream_t st) {
  const size_t smem = sizeof(ScoreSmem<GW>) + 1024;
  static bool configured = false;
  if (!configured) {
    for (auto fn : {score_kernel<1, GW>, score_kernel<2, GW>, score_kernel<3, GW>})
      if (int rc = cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   smem),
                              "score smem attribute"))
        return rc;
    configured = true;
  }
  dim3 grid(p.n_chunks, batch_heads);
  if (fused) {
    // one cooperative launch: both passes and the pooling (grid <= #SMs, 1 CTA/SM)
    if (int rc = cuda_check(cudaMemsetAsync(p.gridbar, 0, sizeof(GridBar), st), "gridbar reset"))
      return rc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cuda_check(cudaLaunchKernelEx(&cfg, score_kernel<3, GW>, tq, tk, p), "score fused launch");
  }
  score_kernel<1, GW><<<grid, kThreads, smem, st>>>(tq, tk, p);
  if (int rc = cuda_check(cudaGetLastError(), "score pass 1 launch")) return rc;
  score_kernel<2, GW><<<grid, kThreads, smem, st>>>(tq, tk, p);
  if (int rc = cuda_check(cudaGetLastError(), "score pass 2 launch")) return rc;
  const int n = p.T - p.window;
  const int64_t total = static_cast<int64_t>(batch_heads) * n;
  pool_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(p.raw, p.scores, n,
                                                                         p.pool_r, total);
  return cuda_check(cudaGetLastError(), "score pool launch");
}

}  // namespace
}  // namespace fkv

extern "C" int64_t fkv_score_workspace_bytes(int32_t batch, int32_t hkv, int32_t T, int32_t window,
                                             int32_t group) {
  const int gw = group * window;
  const int n_tiles = (T + fkv::kBN - 1) / fkv::kBN;
  const int bh = batch * hkv;
  const int chunks = fkv::score_chunks(bh > 0 ? bh : 1, n_tiles);
  const int64_t stats = static_cast<int64_t>(bh) * chunks * gw * 2 * 4;
  const int64_t raw = static_cast<int64_t>(bh) * (T - window) * 4;
  return stats + raw + 256;
}

extern "C" int fkv_snapkv_score(const void* q_win, const void* k, int32_t batch, int32_t hq,
                                int32_t hkv, int32_t T, int32_t window, int32_t pool_k,
                                float sm_scale, float* scores, void* workspace, void* stream) {
  using namespace fkv;
  if (!q_win || !k || !scores || !workspace)
    return set_error(FKV_ERR_INVALID, "fkv_snapkv_score: null pointer");
  if (batch < 1 || hkv < 1 || hq % hkv || T <= window || window < 1 || pool_k < 1 || !(pool_k & 1))
    return set_error(FKV_ERR_INVALID, "fkv_snapkv_score: bad sizes");
  const int group = hq / hkv;
  const int gw = group * window;
  if (gw != 128 && gw != 256)
    return set_error(FKV_ERR_INVALID, "fkv_snapkv_score: group * window must be 128 or 256");
  if (static_cast<int64_t>(batch) * hkv * T >= 0x7fffffffLL)
    return set_error(FKV_ERR_INVALID, "fkv_snapkv_score: Bt * Hkv * T too large");
  const int n_tiles = (T + kBN - 1) / kBN;
  const int bh = batch * hkv;
  int chunks = score_chunks(bh, n_tiles);
  const int tiles_per_chunk = (n_tiles + chunks - 1) / chunks;
  chunks = (n_tiles + tiles_per_chunk - 1) / tiles_per_chunk;

  CUtensorMap tq, tk;
  if (int rc = make_map(&tq, q_win, static_cast<int64_t>(batch) * hq * window, 128)) return rc;
  if (int rc = make_map(&tk, k, static_cast<int64_t>(batch) * hkv * T, kBN)) return rc;
  float* stats = static_cast<float*>(workspace);
  float* raw = stats + static_cast<int64_t>(bh) * chunks * gw * 2;
  auto* gridbar = reinterpret_cast<GridBar*>(
      (reinterpret_cast<uintptr_t>(raw + static_cast<int64_t>(bh) * (T - window)) + 15) & ~uintptr_t(15));
  ScoreParams p{T, window, group, hkv, chunks, tiles_per_chunk, hq * window,
                sm_scale * kLog2e, stats, raw, scores, pool_k / 2, gridbar};
  auto st = static_cast<cudaStream_t>(stream);
  // fused single launch whenever every CTA can be co-resident (1 CTA per SM)
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const bool fused = static_cast<int64_t>(bh) * chunks <= sms;
  return gw == 128 ? launch_score<128>(tq, tk, p, bh, fused, st)
                   : launch_score<256>(tq, tk, p, bh, fused, st);
}

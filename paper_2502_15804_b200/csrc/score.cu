// K1: Ada-SnapKV observation-window scoring on the 5th-gen tensor cores.
//
// No reference implementation exists (the paper used KVPress
// SnapKV/AdaKV).  Definition (oracle/kv.py):
//   P[r,:]  = softmax_t(q_r . k_t / sqrt(d)), r = (g, i) over the G*w window
//             rows of one KV head, causal inside the window
//   raw[t]  = (1/G) sum_r P[r,t]              t < T - w
//   s[t]    = max(raw[t-3 .. t+3])            (pooling kernel below)
//
// Two tcgen05 passes over K per work item (request, KV head, key chunk):
//   pass 1  D[GW rows x 128 keys]   = Q_win . K_tile^T  -> per-row online max
//           and sum-exp with rows in TMEM lanes (thread-local reductions,
//           one partial per column group, combined once per chunk);
//   pass 2  D^T[128 keys x GW rows] = K_tile . Q_win^T  -> per-key column
//           sums of exp(s - m_r)/l_r with keys in TMEM lanes (thread-local);
//           the four column groups (warps 4c..4c+3) store separate partial
//           sums, added by the pooling (no block barrier per tile).
// Q_win (GW = G*w = 128 or 256 rows) is TMA-loaded per item and stays in
// shared memory; K tiles (128 keys x 128 d, 32 KiB) stream through a 3-stage
// TMA ring with 128-B swizzle; one elected thread issues
// tcgen05.mma.cta_group::1.kind::f16 (M=128, N=128 or GW, K=16) into fp32
// TMEM accumulators (512 / GW buffers: all 512 columns); sixteen epilogue
// warps drain them with tcgen05.ld (warp e reads TMEM lanes 32*(e%4) and
// column group e/4) and hand each buffer back as soon as it is in registers.
// Warp roles: 0-15 epilogue, 16 TMA producer, 17 MMA issuer.
// One persistent cooperative launch at any batch (one CTA per SM): the
// Bt*Hkv*chunks items are dealt round robin (score_waves); pass 1 of every
// item, one grid barrier, pass 2 of every item, a second barrier, pooling,
// then the Ada split + top-k in the same launch (per chunk when every CTA
// holds one item, else the grid-wide search of gsel.cuh).  With one item
// per CTA the second pass re-reads K mostly from L2 (a layer's K for one
// request is 32 MiB at 16k context).
#include <cuda.h>

#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <type_traits>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include "common.cuh"
#include "gsel.cuh"

namespace fkv {
namespace {

constexpr int kBN = 128;                 // keys per tile
constexpr int kStages = 3;
constexpr int kTileBytes = kBN * 256;    // 128 keys x 128 d x bf16
// 16 epilogue warps: four per SM sub-partition, so one warp's TMEM-load wait
// is covered by the others' exponentials (the MUFU pipe is the bound)
constexpr int kEpiWarps = 16;
constexpr int kTmaWarp = kEpiWarps, kMmaWarp = kEpiWarps + 1;
constexpr int kThreads = 32 * (kEpiWarps + 2);
constexpr int kRawParts = 4;  // column partial sums per key written by pass 2 (one per column quarter)
// the selection phase runs on epilogue warps 0-7 (named barrier 2)
// Exponentials computed on the FMA pipe (poly_exp2) instead of the MUFU:
// 0 none, 1 one in four, 2 two in four, 3 one in eight (default; measured
// best: 128k 201.6 -> 194.3 us, 32k 76.3 -> 73.5, batch 4 at 32k 216.9 ->
// 207.2, 16k unchanged; one in four loses 4 % at batch 4 16k, two in four
// 10 % everywhere -- the FMA pipe then saturates)
#ifndef FKV_POLY_EXP
#define FKV_POLY_EXP 3
#endif
constexpr bool kPolyExp = FKV_POLY_EXP != 0;
constexpr bool kPolyExp2 = FKV_POLY_EXP == 2;
constexpr bool kPolyExp8 = FKV_POLY_EXP == 3;
constexpr int kSelWarps = 16, kSelThreads = 32 * kSelWarps;  // the selection: every epilogue warp
constexpr float kLog2e = 1.4426950408889634f;

struct ScoreParams {
  int T, window, group, hkv, n_chunks;  // key chunks per (request, KV head)
  int n_waves, bh_total;  // persistent schedule (score_waves): items per CTA, heads
  int q_rows_per_req;  // Hq * w
  float scale_log2;    // log2(e) / sqrt(d)
  float* stats;        // [Bt*Hkv, n_chunks, GW, 2] (max, sum) in log2 units
  float* raw;          // [kRawParts][Bt*Hkv, T - w] partial column sums
  float* scores;       // pooled output
  int pool_r;          // pooling radius (pool_k / 2)
  struct GridBar* gridbar;  // zeroed counter
  // selection after the scoring (fkv_snapkv_select); workspace parts zeroed per launch
  int sel_mode;        // 0 none, 1 per-chunk (one wave: select_phase), 2 grid search over the pooled scores
  int budget, floor_k, rest_total;  // B, f = floor(alpha (B - w)), R = Hkv (B - w - f)
  uint32_t* hist;      // sel_mode 1: [kSelPasses][Bt*Hkv][2][256] per-pass digit histograms (zeroed)
  int32_t* counts;     // sel_mode 1: [Bt*Hkv][n_chunks] int2 (chosen outright, ties at s*) per chunk
  int32_t* budgets;    // out [Bt, Hkv]
  int64_t* offsets;    // out [Bt*Hkv + 1]
  int32_t* idx;        // out [Bt*Hkv*budget]
  GSelParams gs;       // sel_mode 2
};

constexpr int kSelPasses = 4;            // 32-bit orderable scores, 8-bit digits (ties resolved by count)
constexpr int kSelMaxKeys = kStages * kTileBytes / 4;  // pooled f32 keys staged in the (idle) K ring
constexpr int kSelMaxHeads = 8;

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

// 32 consecutive fp32 TMEM columns of this thread's lane, no wait (pair
// with tmem_wait_ld: several loads in flight per wait).
__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// Wait, then pin the loaded registers behind the wait: the register uses have
// no data dependence on the wait otherwise and could be scheduled above it.
__device__ __forceinline__ void tmem_wait_ld(uint32_t (&a)[32], uint32_t (&b)[32]) {
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 32; ++i) asm volatile("" : "+r"(a[i]), "+r"(b[i]));
}

__device__ __forceinline__ void tmem_wait_ld(uint32_t (&a)[32]) {
  tmem_wait_ld();
#pragma unroll
  for (int i = 0; i < 32; ++i) asm volatile("" : "+r"(a[i]));
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
  uint64_t full[kStages], empty[kStages], tfull[512 / GW], tempty[512 / GW], qbar, qempty;
  uint32_t tmem_base;
  alignas(16) float bias[GW];  // pass 2: per query row, m_r + log2(G * l_r) (log2 units)
  float ml[4 * 128 * 2];     // pass 1: per-row (max, sum) partials of column groups 1..3 -> group 0
};
static_assert(offsetof(ScoreSmem<128>, k) == sizeof(ScoreSmem<128>::q) &&
                  offsetof(ScoreSmem<256>, k) == sizeof(ScoreSmem<256>::q),
              "Q_win and the K ring are contiguous (the grid select's key cache spans both)");

struct GridBar {
  unsigned count, gen;
};

// Grid-wide barrier among the epilogue warps of co-resident CTAs (cooperative
// launch); the TMA and MMA warps keep streaming while the epilogue waits.
// Monotonic counter (zeroed per launch): arrival k of every CTA lands in
// [k*N, (k+1)*N), so the k-th barrier's target is known up front and the
// arrival is a fire-and-forget release reduction (the poll is the only
// round trip).  `k` counts this CTA's barriers (thread 0's copy matters).
template <int BAR = 1, int NT = 32 * kEpiWarps>
__device__ __forceinline__ void epi_grid_sync(GridBar* gb, unsigned& k) {
  asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT));
  if (threadIdx.x == 0) {
    const unsigned target = ++k * (gridDim.x * gridDim.y);
    unsigned v;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&gb->count) : "memory");
    while (true) {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(&gb->count) : "memory");
      if (v >= target) break;
      __nanosleep(32);
    }
  }
  asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT));
}

// diagnostics: %globaltimer stamps of CTA (0,0) through the fused select
// (read with fkv__score_stamps; tools/probe_prefill_time.py)
__device__ unsigned long long g_sstamps[64];
__device__ __forceinline__ void sstamp(int i) {
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0 && i < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_sstamps[i] = t;
  }
}

__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps)); }
__device__ __forceinline__ void sel_sync() { asm volatile("bar.sync 2, %0;" ::"n"(kSelThreads)); }


// Scratch of the selection phase, placed in the (idle) Q_win region.
struct SelScratch {
  int32_t suf[kSelMaxHeads][256];  // per-head suffix counts of the current digit
  uint32_t hist[256], hist2[256];  // this chunk's digits: global search, floor search
  int32_t above[kSelMaxHeads], n_at[kSelMaxHeads];
  int32_t warp_tot[kSelWarps];
  int32_t dstar, exact;
  uint32_t fprefix, fmask;  // floor search of this CTA's head
  int32_t fexact, fabove;
};

__device__ __forceinline__ int32_t epi_count(bool pred, SelScratch& x) {
  const int tid = threadIdx.x;
  const uint32_t bal = __ballot_sync(0xffffffffu, pred);
  if ((tid & 31) == 0) x.warp_tot[tid >> 5] = __popc(bal);
  sel_sync();
  int32_t c = 0;
  for (int j = 0; j < kSelWarps; ++j) c += x.warp_tot[j];
  sel_sync();
  return c;
}

// Suffix counts of one global 256-bin histogram by one warp (8 bins per
// lane): s[j] = base + #keys in bins >= 8*lane + j; `up` = the count past the
// lane's last bin (base past bin 255).
__device__ __forceinline__ void warp_suffix8_of(const uint4 x0, const uint4 x1, int base, int (&s)[8], int& up) {
  const int lane = threadIdx.x & 31;
  const uint32_t h[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
  int run = 0;
#pragma unroll
  for (int j = 7; j >= 0; --j) {
    run += static_cast<int>(h[j]);
    s[j] = run;
  }
  int incl = run;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int v = __shfl_down_sync(0xffffffffu, incl, off);
    if (lane + off < 32) incl += v;
  }
  const int higher = incl - run + base;
#pragma unroll
  for (int j = 0; j < 8; ++j) s[j] += higher;
  up = __shfl_down_sync(0xffffffffu, s[0], 1);
  if (lane == 31) up = base;
}
__device__ __forceinline__ void warp_suffix8(const uint32_t* gh, int base, int (&s)[8], int& up) {
  const int lane = threadIdx.x & 31;
  warp_suffix8_of(__ldcg(reinterpret_cast<const uint4*>(gh + 8 * lane)),
                  __ldcg(reinterpret_cast<const uint4*>(gh + 8 * lane + 4)), base, s, up);
}

// Digit histograms of the pooled keys for the global search (keys matching
// (gp, gm), into h0) and the floor search ((fp, fm), into h1) at once.
__device__ __forceinline__ void epi_histogram2(const float* sp, int nk, bool ga, uint32_t gp, uint32_t gm,
                                               bool fa, uint32_t fp, uint32_t fm, int shift, uint32_t* h0,
                                               uint32_t* h1) {
  const int tid = threadIdx.x;
  (tid < 256 ? h0 : h1)[tid & 255] = 0;
  sel_sync();
  auto add = [&](uint32_t o) {
    const uint32_t d = (o >> shift) & 255u;
    if (ga && (o & gm) == gp) atomicAdd(&h0[d], 1u);
    if (fa && (o & fm) == fp) atomicAdd(&h1[d], 1u);
  };
  // four keys per 16-byte shared load (the staged keys start 16-byte aligned)
  const float4* s4 = reinterpret_cast<const float4*>(sp);
  const int n4 = nk >> 2;
#pragma unroll 2
  for (int j = tid; j < n4; j += kSelThreads) {
    const float4 v = s4[j];
    add(orderable(v.x));
    add(orderable(v.y));
    add(orderable(v.z));
    add(orderable(v.w));
  }
  if (tid < (nk & 3)) add(orderable(sp[4 * n4 + tid]));
  sel_sync();
}

// MODE 4, after pooling: Ada budget split + per-head top-k, grid-wide.  Same
// result as select.cu's grid_select_kernel (the standalone launch over
// pooled scores in HBM), here fused behind the scoring passes.
//
// Radix search over the 32-bit orderable score, MSB-first 8-bit digits: per
// digit each CTA histograms its own pooled keys into the per-(request, head)
// global histograms of that pass and, after a grid barrier, every CTA of the
// request evaluates G(d) = sum_h max(0, N_h(d) - floor) from all heads'
// histograms and takes the same d* = max{d : G(d) >= R} (the Ada split in
// its floor-free form, see select.cu).  The same passes run each head's own
// floor search (its f-th largest score), kept if the head ends below its
// floor; a head's global histogram is skipped once N_h < f is certain, its
// floor histogram once N_h >= f is, and one histogram serves both while
// they share a prefix.  Four passes fix the threshold score; ties at it are
// taken in the global tie order (head asc, token asc) -- or the head's token
// order for the floor -- from per-chunk tie counts, with no passes over the
// index bits.  One last barrier publishes per-chunk counts so every CTA
// writes its chosen tokens at the right place of the ascending index list.
template <class Smem>
__device__ void select_phase(const ScoreParams& p, Smem& sm, int b, int h, int bh, int chunk, int n,
                             int t_beg, int nk, const float* sp, unsigned& n_bar) {
  SelScratch& x = *reinterpret_cast<SelScratch*>(&sm.q[0][0][0]);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int HK = p.hkv, BH = p.bh_total;
  const int f = p.floor_k, R = p.rest_total;
  sstamp(1);
  if (tid < HK) x.above[tid] = 0, x.n_at[tid] = R > 0 ? n : 0;
  if (tid == 0) {
    x.fprefix = x.fmask = 0;
    x.fexact = f <= 0;
    x.fabove = 0;
  }
  sel_sync();
  uint32_t prefix = 0, mask = 0;
  bool exact = R <= 0;
  int dstar = 0;
  for (int pass = 0, shift = 24; pass < 4; ++pass, shift -= 8) {
    // global: N_h >= f still possible; floor: N_h < f still possible
    const bool ga = !exact && x.n_at[h] >= f;
    const bool fa = !x.fexact && (exact ? x.n_at[h] < f : x.above[h] < f);
    const bool same = ga && fa && prefix == x.fprefix && mask == x.fmask;
    uint32_t* gh = p.hist + (static_cast<int64_t>(pass) * BH + bh) * 512;
    if (ga || fa) {  // add my keys' digit histograms to this pass's global ones
      epi_histogram2(sp, nk, ga, prefix, mask, fa && !same, x.fprefix, x.fmask, shift, x.hist, x.hist2);
      if (tid < 256) {  // global histogram by threads 0..255, floor histogram by 256..511
        if (ga && x.hist[tid]) atomicAdd(gh + tid, x.hist[tid]);
      } else {
        const int d = tid - 256;
        const uint32_t fc = same ? x.hist[d] : (fa ? x.hist2[d] : 0u);
        if (fc) atomicAdd(gh + 256 + d, fc);
      }
    }
    sstamp(2 + 2 * pass);
    epi_grid_sync<2, kSelThreads>(p.gridbar, n_bar);  // fixed pass count: uniform across the grid
    sstamp(3 + 2 * pass);
    // decisions, one warp per histogram (8 bins per lane, no block-wide
    // scans): warp w -> suffix counts of head w's global histogram; warp 0
    // also runs my head's floor search (its floor histogram is the global one
    // while the two searches share a prefix)
    const uint32_t* gq = p.hist + (static_cast<int64_t>(pass) * BH + b * HK) * 512;
    // warp 0 loads my head's floor histogram together with its global one
    // (one L2 round trip for both)
    uint4 fx0 = make_uint4(0, 0, 0, 0), fx1 = fx0;
    if (fa && wid == 0) {
      const uint32_t* fg = same ? gh : gh + 256;
      fx0 = __ldcg(reinterpret_cast<const uint4*>(fg + 8 * lane));
      fx1 = __ldcg(reinterpret_cast<const uint4*>(fg + 8 * lane + 4));
    }
    if (!exact && wid < HK) {
      int sv[8], up;
      warp_suffix8(gq + wid * 512, x.above[wid], sv, up);
#pragma unroll
      for (int j = 0; j < 8; ++j) x.suf[wid][8 * lane + j] = sv[j];
    }
    if (fa && wid == 0) {  // my head's floor search: d* = max{d : S(d) >= f}
      int sv[8], up;
      warp_suffix8_of(fx0, fx1, x.fabove, sv, up);
      int c = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) c += sv[j] >= f;
      const int ds = __reduce_add_sync(0xffffffffu, c) - 1;
      int at = 0, nxt = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (8 * lane + j == ds) {
          at = sv[j];
          nxt = j < 7 ? sv[j + 1] : up;
        }
      at = __shfl_sync(0xffffffffu, at, ds >> 3);
      nxt = __shfl_sync(0xffffffffu, nxt, ds >> 3);
      if (lane == 0) {
        x.fprefix |= static_cast<uint32_t>(ds) << shift;
        x.fmask |= 255u << shift;
        x.fabove = nxt;
        x.fexact = at == f;
      }
    }
    sel_sync();
    sstamp(12 + 3 * pass);
    if (exact) continue;
    int32_t gd = 0;
    if (tid < 256)
      for (int hh = 0; hh < HK; ++hh) gd += max(0, x.suf[hh][tid] - f);
    const int32_t cnt = epi_count(tid < 256 && gd >= R, x);
    if (tid == cnt - 1) {
      x.dstar = cnt - 1;
      x.exact = gd == R;
    }
    sel_sync();
    dstar = x.dstar;
    exact = x.exact != 0;
    // n_at: keys with the decided digits >= prefix.d*; above: strictly above d*
    if (tid < HK) {
      x.n_at[tid] = x.suf[tid][dstar];
      x.above[tid] = dstar < 255 ? x.suf[tid][dstar + 1] : x.above[tid];
    }
    prefix |= static_cast<uint32_t>(dstar) << shift;
    mask |= 255u << shift;
    sel_sync();
    sstamp(13 + 3 * pass);
  }
  sstamp(30);
  const bool have_tau = R > 0;
  // Final per-head counts.  exact: every key with orderable(score) >= prefix
  // is in (N_h = n_at).  Otherwise s* = prefix is the full threshold score:
  // base_h = #(score > s*) = above, tied_h = n_at - above; walk the ties in
  // head order until G reaches R: heads before hstar take all their ties,
  // hstar takes its first kstar, later heads none.
  if (tid == 0) {
    int hstar = HK, kstar = 0;
    if (have_tau && !exact) {
      int need = R;
      for (int hh = 0; hh < HK; ++hh) need -= max(0, x.above[hh] - f);
      for (int hh = 0; hh < HK && need > 0; ++hh) {
        const int base = x.above[hh], tied = x.n_at[hh] - base;
        const int gain = max(0, base + tied - f) - max(0, base - f);
        if (gain >= need) {
          hstar = hh;
          kstar = max(0, f - base) + need;
          need = 0;
        } else {
          need -= gain;
        }
      }
      for (int hh = 0; hh < HK; ++hh)
        x.n_at[hh] = hh < hstar ? x.n_at[hh] : (hh == hstar ? x.above[hh] + kstar : x.above[hh]);
    }
    x.dstar = hstar;
    x.exact = kstar;
  }
  sel_sync();
  const int hstar = x.dstar, kstar = x.exact;
  const bool below = !have_tau || x.n_at[h] < f;
  auto budget_of = [&](int hh) {
    const int c = have_tau ? max(0, x.n_at[hh] - f) : 0;
    return p.window + f + c;
  };
  // keep rule of my head: kind 0 = above thr + ranked ties at thr (the first
  // ktie in order), 1 = o >= thr, 2 = nothing
  int kind = 2, ktie = 0;
  uint32_t thr = 0;
  if (below) {  // exactly its own top-f
    if (f > 0) {
      thr = x.fprefix;
      kind = x.fexact ? 1 : 0;
      ktie = x.fexact ? 0 : f - x.fabove;
    }
  } else if (exact) {
    thr = prefix;
    kind = 1;
  } else {
    thr = prefix;
    kind = 0;
    ktie = h < hstar ? 0x7fffffff : (h == hstar ? kstar : 0);
  }
  // class of key i: 1 = chosen outright, 2 = tie at thr taken by tie rank
  auto klass = [&](uint32_t o) -> int {
    if (kind == 2) return 0;
    if (kind == 1) return o >= thr;
    if (o != thr) return o > thr;
    return ktie == 0x7fffffff ? 1 : (ktie > 0 ? 2 : 0);
  };
  // per-warp (chosen outright, ties) counts of contiguous key segments (in
  // 4-key units: 16-byte shared loads), kept in x.suf for the writes; the
  // chunk's totals are published for the CTAs after it
  const float4* s4 = reinterpret_cast<const float4*>(sp);
  const int n4 = (nk + 3) >> 2, per4 = (n4 + kSelWarps - 1) / kSelWarps;
  const int v0 = min(n4, wid * per4), v1 = min(n4, v0 + per4);
  auto klass4 = [&](int j, int (&k)[4]) {  // unit j: keys 4j .. 4j+3 (those < nk)
    const float4 v = s4[j];
    const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int c = 0; c < 4; ++c) k[c] = 4 * j + c < nk ? klass(orderable(e[c])) : 0;
  };
  int32_t c1 = 0, c2 = 0;
#pragma unroll 2
  for (int j = v0 + lane; j < v1; j += 32) {
    int k[4];
    klass4(j, k);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      c1 += k[c] == 1;
      c2 += k[c] == 2;
    }
  }
  c1 = __reduce_add_sync(0xffffffffu, c1);
  c2 = __reduce_add_sync(0xffffffffu, c2);
  if (lane == 0) x.suf[0][wid] = c1, x.suf[1][wid] = c2;
  sel_sync();
  if (tid == 0) {
    int32_t a = 0, t2 = 0;
    for (int j = 0; j < kSelWarps; ++j) a += x.suf[0][j], t2 += x.suf[1][j];
    int2* cc = reinterpret_cast<int2*>(p.counts) + static_cast<int64_t>(bh) * p.n_chunks + chunk;
    *cc = make_int2(a, t2);
  }
  sstamp(31);
  epi_grid_sync<2, kSelThreads>(p.gridbar, n_bar);
  sstamp(32);
  // this chunk's position in the head's list, and its tie-rank origin
  int64_t pos = 0;
  int tie0 = 0;
  for (int c = lane; c < chunk; c += 32) {
    const int2 cc = __ldcg(reinterpret_cast<const int2*>(p.counts) + static_cast<int64_t>(bh) * p.n_chunks + c);
    pos += cc.x;
    tie0 += cc.y;
  }
  {
    // every warp computed the same partial sums per lane
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      pos += __shfl_xor_sync(0xffffffffu, pos, o);
      tie0 += __shfl_xor_sync(0xffffffffu, tie0, o);
    }
  }
  int64_t off = static_cast<int64_t>(b) * HK * p.budget;
  for (int hh = 0; hh < h; ++hh) off += budget_of(hh);
  const int bud = budget_of(h);
  int32_t* out = p.idx + off;
  // this warp's segment: chosen outright and ties of the segments before it
  int c1b = 0, tb = 0;
  for (int j = 0; j < wid; ++j) c1b += x.suf[0][j], tb += x.suf[1][j];
  int tie_run = tie0 + tb;  // tie rank of the warp's next tie in token order
  pos += c1b + min(tie_run, ktie);
  auto warp_excl = [&](int v, int& total) {  // exclusive prefix over lanes
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    total = __shfl_sync(0xffffffffu, incl, 31);
    return incl - v;
  };
  // no block barriers: each warp writes its own segment, 4 keys per lane
  for (int jb = v0; jb < v1; jb += 32) {
    const int j = jb + lane;
    int k[4] = {0, 0, 0, 0};
    if (j < v1) klass4(j, k);
    int t_all, n_all;
    int tr = tie_run + warp_excl((k[0] == 2) + (k[1] == 2) + (k[2] == 2) + (k[3] == 2), t_all);
    bool tk[4];
    int nt = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      tk[c] = k[c] == 1;
      if (k[c] == 2) tk[c] = tr++ < ktie;
      nt += tk[c];
    }
    int64_t q = pos + warp_excl(nt, n_all);
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (tk[c]) out[q++] = t_beg + 4 * j + c;
    pos += n_all;
    tie_run += t_all;
  }
  sstamp(33);
  if (chunk == 0) {
    for (int i = tid; i < p.window; i += kSelThreads) out[bud - p.window + i] = n + i;
    if (tid == 0) {
      p.budgets[bh] = bud;
      p.offsets[bh] = off;
      if (bh == BH - 1) p.offsets[BH] = off + bud;
    }
  }
}

// The epilogue warps as the 512 threads of the grid-wide select (gsel.cuh):
// named barrier 1 instead of __syncthreads.
struct EpiCx {
  int cta, ncta;
  __device__ void sync() const { epi_sync(); }
  __device__ int count(bool pred) const {
    int r;
    asm volatile("{\n.reg .pred q;\nsetp.ne.u32 q, %1, 0;\nbar.red.popc.u32 %0, 1, %2, q;\n}"
                 : "=r"(r)
                 : "r"(static_cast<int>(pred)), "n"(32 * kEpiWarps)
                 : "memory");
    return r;
  }
  __device__ void grid(unsigned* bar, unsigned& k) const { grid_sync_n(bar, k, ncta, [] { epi_sync(); }); }
};

// Grid-select state (sel_mode 2) at the start of the idle Q_win region, its
// key cache right after it through the (idle, contiguous) K ring.
__host__ __device__ constexpr int gsel_cache_off() { return (static_cast<int>(sizeof(GSelSmem)) + 15) & ~15; }
template <int GW>
__host__ __device__ constexpr int gsel_cache_keys() {
  return (GW * 256 + kStages * kTileBytes - gsel_cache_off()) / 4;
}

// One work item = key chunk `chunk` of (request, KV head) `bh`: tiles
// [a, e1) of pass 1 (all T keys) and [a, e2) of pass 2 (the T - w scored
// keys); chunks split a head's tiles as evenly as possible.  Items are dealt
// round robin: item w * grid + cta is the CTA's w-th.
struct Item {
  int bh, chunk, a, e1, e2;
  bool valid;
};
__device__ __forceinline__ Item score_item(const ScoreParams& p, int w) {
  Item it{};
  // 32-bit arithmetic: items < 2^31 and chunk * tiles < 2^31 (Bt*Hkv*T < 2^31 is checked on the host)
  const int i = (w * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  it.bh = i / p.n_chunks;
  it.chunk = i - it.bh * p.n_chunks;
  it.valid = it.bh < p.bh_total;
  const int nt1 = (p.T + kBN - 1) / kBN, nt2 = (p.T - p.window + kBN - 1) / kBN;
  it.a = it.chunk * nt1 / p.n_chunks;
  it.e1 = (it.chunk + 1) * nt1 / p.n_chunks;
  it.e2 = min(it.e1, nt2);
  if (!it.valid) it.e1 = it.e2 = it.a;
  return it;
}

// Persistent cooperative launch (one CTA per SM): every CTA runs pass 1 of
// each of its items, then one grid barrier (every chunk's row statistics are
// in global memory), then pass 2 of each item, a second barrier, the pooling
// of each item and (MODE 4) the Ada split + top-k -- per chunk in place
// (sel_mode 1: one item per CTA) or the grid-wide search over the pooled
// scores (sel_mode 2, gsel.cuh).  The TMA and MMA warps run ahead across
// items and passes; the Q_win tile is reloaded whenever the item changes,
// once the MMA warp has released it.  MODE 3: scores only; MODE 4: scores +
// selection.
template <int MODE, int GW, bool MULTI>
__global__ void __launch_bounds__(kThreads, 1)
    score_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                 const ScoreParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  ScoreSmem<GW>& sm = *reinterpret_cast<ScoreSmem<GW>*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  constexpr int NB = 512 / GW;           // accumulator buffers: all 512 TMEM columns
  constexpr uint32_t kCols = NB * GW;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  sstamp(0);
  unsigned n_bar = 0;  // grid barriers passed (epilogue thread 0)
  const int n = p.T - p.window;
  const int W = MULTI ? p.n_waves : 1;  // items per CTA (compile-time 1: straight-line passes)

  if (warp == kTmaWarp && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_q)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_k)) : "memory");
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    for (int i = 0; i < NB; ++i) {
      mbar_init(&sm.tfull[i], 1);
      mbar_init(&sm.tempty[i], kEpiWarps);
    }
    mbar_init(&sm.qbar, 1);
    mbar_init(&sm.qempty, 1);
    fence_mbar_init();
  }
  if (warp == kMmaWarp) tmem_alloc(&sm.tmem_base, kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == kTmaWarp) {
    // ------------------------------------------------ TMA producer ----
    if (lane == 0) {
      const uint64_t keep = l2_policy(true), stream = l2_policy(false);
      int g = 0, nq = 0;  // K tiles and Q_win loads issued
      int cur = -1;       // item whose Q_win is in shared memory
      for (int seg = 0; seg < 2 * W; ++seg) {  // pass 1 of every item, then pass 2
        const bool p1 = seg < W;
        const int w = p1 ? seg : seg - W;
        const Item itm = score_item(p, w);
        const int nt = p1 ? itm.e1 - itm.a : itm.e2 - itm.a;
        if (nt == 0) continue;
        if (cur != w) {
          const int b = itm.bh / p.hkv, h = itm.bh - b * p.hkv;
          const int qrow0 = b * p.q_rows_per_req + h * GW;
          if (nq > 0) mbar_wait(&sm.qempty, (nq - 1) & 1);  // the MMA warp is done with the last Q_win
          mbar_arrive_expect_tx(&sm.qbar, GW * 256);
          for (int c = 0; c < 2; ++c)
            for (int rh = 0; rh < GW / 128; ++rh)
              tma_load_2d(&sm.q[c][rh * 128][0], &tm_q, 64 * c, qrow0 + 128 * rh, &sm.qbar);
          ++nq;
          cur = w;
        }
        const int krow0 = itm.bh * p.T;
        for (int it = 0; it < nt; ++it, ++g) {
          const int s = g % kStages;
          mbar_wait(&sm.empty[s], ((g / kStages) & 1) ^ 1);
          mbar_arrive_expect_tx(&sm.full[s], kTileBytes);
          for (int c = 0; c < 2; ++c)
            tma_load_2d_hint(&sm.k[s][c][0][0], &tm_k, 64 * c, krow0 + (itm.a + it) * kBN, &sm.full[s],
                             p1 ? keep : stream);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // -------------------------------------------------- MMA issuer ----
    if (lane == 0) {
      constexpr uint32_t kIdesc1 = idesc_bf16(128, kBN);
      constexpr uint32_t kIdesc2 = idesc_bf16(128, GW);
      const uint32_t q_base = smem_u32(&sm.q[0][0][0]);
      int g = 0, nq = 0, cur = -1;
      // the same (pass, item) sequence as the producer; the Q_win tile is
      // released (qempty) before every change of item
      auto next_item = [&](int seg) {  // item of the next non-empty segment after seg, or -1
        for (int s2 = seg + 1; s2 < 2 * W; ++s2) {
          const int w2 = s2 < W ? s2 : s2 - W;
          const Item i2 = score_item(p, w2);
          if ((s2 < W ? i2.e1 : i2.e2) > i2.a) return w2;
        }
        return -1;
      };
      for (int seg = 0; seg < 2 * W; ++seg) {
        const bool p1 = seg < W;
        const int w = p1 ? seg : seg - W;
        const Item itm = score_item(p, w);
        const int nt = p1 ? itm.e1 - itm.a : itm.e2 - itm.a;
        if (nt == 0) continue;
        if (cur != w) {
          mbar_wait(&sm.qbar, nq & 1);
          ++nq;
          cur = w;
        }
        // one tile: wait for its K stage and a free accumulator buffer, issue
        // the 8 K=16 steps (pass 1: D = Q K^T per row half; pass 2: D^T = K Q^T)
        auto tile = [&](auto pass1) {
          const int s = g % kStages, buf = g % NB;
          mbar_wait(&sm.full[s], (g / kStages) & 1);
          mbar_wait(&sm.tempty[buf], ((g / NB) & 1) ^ 1);
          tc_fence_after();
          const uint32_t k_base = smem_u32(&sm.k[s][0][0][0]);
          const uint32_t d_buf = tmem + buf * GW;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t koff = (kk >> 2) * (kBN * 128) + (kk & 3) * 32;
            const uint32_t qoff = (kk >> 2) * (GW * 128) + (kk & 3) * 32;
            if constexpr (decltype(pass1)::value) {
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
          ++g;
        };
        if (p1)
          for (int it = 0; it < nt; ++it) tile(std::true_type{});
        else
          for (int it = 0; it < nt; ++it) tile(std::false_type{});
        const int nx = next_item(seg);
        if (nx >= 0 && nx != w) umma_commit(&sm.qempty);  // Q_win may be reloaded once these MMAs are done
      }
    }
  } else {
    // ---------------------------------------------------- epilogue ----
    // warp w reads TMEM lanes 32*(w%4) (its lane quarter) and column group
    // cs = w/4 of every accumulator buffer
    const int quad = warp & 3, cs = warp >> 2;
    const uint32_t lane_base = static_cast<uint32_t>(32 * quad) << 16;
    int g = 0;  // accumulator tiles consumed
    for (int w = 0; w < W; ++w) {
      const Item itm = score_item(p, w);
      const int bh = itm.bh, n1 = itm.e1 - itm.a;
      if (n1 > 0) {
        // rows in TMEM lanes: GW=128 -> one M=128 tile, each row's 128 keys in
        // four column groups of 32; GW=256 -> two M=128 tiles (row halves), each
        // row's keys in two column groups of 64.  Per-row partial (max, sum) of
        // each column group, combined by group 0 at the end.
        constexpr int MH = GW / 128, CG = 4 / MH, NCH = kBN / CG / 32;
        const int mh = MH == 2 ? cs >> 1 : 0, cg = MH == 2 ? cs & 1 : cs;
        const int r = mh * 128 + 32 * quad + lane;
        const int limit = min(p.T - 1, p.T - p.window + (r % p.window));  // last visible key
        float m = -CUDART_INF_F, l = 0.f;
        for (int it = 0; it < n1; ++it, ++g) {
          const int buf = g % NB;
          mbar_wait(&sm.tfull[buf], (g / NB) & 1);
          tc_fence_after();
          const uint32_t col = buf * GW + mh * kBN + cg * (NCH * 32);
          uint32_t ra[32], rb[32];
          tmem_ld32_nw(tmem + lane_base + col, ra);
          if constexpr (NCH == 2) {
            tmem_ld32_nw(tmem + lane_base + col + 32, rb);
            tmem_wait_ld(ra, rb);
          } else {
            tmem_wait_ld(ra);
          }
          tc_fence_before();  // the columns are in registers: the buffer goes back
          __syncwarp();       // to the MMA warp before the math
          if (lane == 0) mbar_arrive(&sm.tempty[buf]);
          constexpr int NV = NCH * 32;
          float v[NV];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(ra[i]);
          if constexpr (NCH == 2) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[32 + i] = __uint_as_float(rb[i]);
          }
          const int c0 = (itm.a + it) * kBN + cg * NV;
          float bmax = -CUDART_INF_F;
          if (c0 + NV - 1 > limit) {  // only the window's tiles (and the tail) need masking
#pragma unroll
            for (int i = 0; i < NV; ++i) {
              v[i] = c0 + i <= limit ? v[i] : -CUDART_INF_F;
              bmax = fmaxf(bmax, v[i]);
            }
            if (bmax == -CUDART_INF_F) continue;
          } else {
#pragma unroll
            for (int i = 0; i < NV; ++i) bmax = fmaxf(bmax, v[i]);
          }
          // running max kept in raw-score units, exponents via one FFMA each,
          // four independent sum chains
          const float nm = fmaxf(m, bmax);
          const float nms = nm * p.scale_log2;
          float e0 = 0.f, e1 = 0.f, e2 = 0.f, e3 = 0.f;
#pragma unroll
          for (int i = 0; i < NV; i += 4) {
            e0 += fast_exp2(fmaf(v[i], p.scale_log2, -nms));
            e1 += kPolyExp2 ? poly_exp2(fmaf(v[i + 1], p.scale_log2, -nms))
                            : fast_exp2(fmaf(v[i + 1], p.scale_log2, -nms));
            e2 += fast_exp2(fmaf(v[i + 2], p.scale_log2, -nms));
            e3 += kPolyExp && (!kPolyExp8 || ((i >> 2) & 1))
                      ? poly_exp2(fmaf(v[i + 3], p.scale_log2, -nms))  // off the MUFU
                           : fast_exp2(fmaf(v[i + 3], p.scale_log2, -nms));
          }
          l = l * fast_exp2((m - nm) * p.scale_log2) + ((e0 + e1) + (e2 + e3));
          m = nm;
        }
        m = m == -CUDART_INF_F ? m : m * p.scale_log2;  // to log2 units
        if (cg > 0) {
          sm.ml[(cg * GW + r) * 2] = m;
          sm.ml[(cg * GW + r) * 2 + 1] = l;
        }
        epi_sync();
        if (cg == 0) {
          for (int gg = 1; gg < CG; ++gg) {
            const float m1 = sm.ml[(gg * GW + r) * 2], l1 = sm.ml[(gg * GW + r) * 2 + 1];
            const float nm = fmaxf(m, m1);
            if (nm != -CUDART_INF_F) {
              l = l * exp2f(m - nm) + l1 * exp2f(m1 - nm);
              m = nm;
            }
          }
          float* st = p.stats + ((static_cast<int64_t>(bh) * p.n_chunks + itm.chunk) * GW + r) * 2;
          st[0] = m;
          st[1] = l;
        }
        if constexpr (MULTI) epi_sync();  // sm.ml is free for the next item
      }
    }
    sstamp(40);
    epi_grid_sync(p.gridbar, n_bar);  // every chunk's statistics are in global memory
    sstamp(41);
    for (int w = 0; w < W; ++w) {
      const Item itm = score_item(p, w);
      const int bh = itm.bh, n2 = itm.e2 - itm.a;
      if (n2 > 0) {
        // combine the head's chunk statistics (log2 domain) into per-row biases:
        // exp2(s*c - m) / (G*l) == exp2(s*c - bias), one FFMA + one MUFU per score
        for (int r = threadIdx.x; r < GW; r += 32 * kEpiWarps) {
          float M = -CUDART_INF_F, L = 0.f;
          const float* st = p.stats + (static_cast<int64_t>(bh) * p.n_chunks) * GW * 2;
          for (int c = 0; c < p.n_chunks; ++c) {
            const float mc = __ldcg(st + (c * GW + r) * 2), lc = __ldcg(st + (c * GW + r) * 2 + 1);
            if (lc <= 0.f) continue;
            const float nm = fmaxf(M, mc);
            L = L * exp2f(M - nm) + lc * exp2f(mc - nm);
            M = nm;
          }
          sm.bias[r] = L > 0.f ? M + log2f(L * static_cast<float>(p.group)) : CUDART_INF_F;
        }
        epi_sync();
        // keys in TMEM lanes, query rows in columns: warp (quad, cs) sums the
        // exponentials of rows [cs*GW/4, (cs+1)*GW/4) for its 32 keys; the four
        // column-group partials are added by the pooling
        constexpr int NC = GW / 128;  // 32-column chunks per warp
        const int key = 32 * quad + lane;
        for (int i2 = 0; i2 < n2; ++i2, ++g) {
          const int buf = g % NB;
          mbar_wait(&sm.tfull[buf], (g / NB) & 1);
          tc_fence_after();
          float acc = 0.f;
          auto chunk_sum = [&](const uint32_t (&rr)[32], int c) {
            const float4* b4 = reinterpret_cast<const float4*>(sm.bias + cs * (GW / 4) + c * 32);
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const float4 bb = b4[i / 4];  // broadcast: every lane reads the same columns
              acc += fast_exp2(fmaf(__uint_as_float(rr[i]), p.scale_log2, -bb.x));
              acc += kPolyExp2 ? poly_exp2(fmaf(__uint_as_float(rr[i + 1]), p.scale_log2, -bb.y))
                               : fast_exp2(fmaf(__uint_as_float(rr[i + 1]), p.scale_log2, -bb.y));
              acc += fast_exp2(fmaf(__uint_as_float(rr[i + 2]), p.scale_log2, -bb.z));
              acc += kPolyExp && (!kPolyExp8 || ((i >> 2) & 1))
                         ? poly_exp2(fmaf(__uint_as_float(rr[i + 3]), p.scale_log2, -bb.w))
                              : fast_exp2(fmaf(__uint_as_float(rr[i + 3]), p.scale_log2, -bb.w));
            }
          };
          uint32_t ra[32], rb[32];
          const uint32_t col = buf * GW + cs * (GW / 4);
          tmem_ld32_nw(tmem + lane_base + col, ra);
          if constexpr (NC == 2) {
            tmem_ld32_nw(tmem + lane_base + col + 32, rb);
            tmem_wait_ld(ra, rb);
          } else {
            tmem_wait_ld(ra);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.tempty[buf]);
          chunk_sum(ra, 0);
          if constexpr (NC == 2) chunk_sum(rb, 1);
          const int t = (itm.a + i2) * kBN + key;
          if (t < n) p.raw[(static_cast<int64_t>(cs) * p.bh_total + bh) * n + t] = acc;
        }
        epi_sync();  // sm.bias is free for the next item
      }
    }
    sstamp(42);
    epi_grid_sync(p.gridbar, n_bar);  // every raw column score is in global memory
    sstamp(43);
    // pooling of every item: the raw column sums (four partials added) of a
    // block of keys and its halo, staged in the (idle) Q_win region, then
    // max-pooled; one wave + per-chunk selection also stages the pooled keys
    // in the (idle) K ring
    float* sp = reinterpret_cast<float*>(&sm.k[0][0][0][0]);
    float* stg = reinterpret_cast<float*>(&sm.q[0][0][0]);
    constexpr int kStg = GW * 256 / 4;
    const int R = p.pool_r, blk = kStg - 2 * R;
    const int64_t part = static_cast<int64_t>(p.bh_total) * n;
    Item mine{};
    for (int w = 0; w < W; ++w) {
      const Item itm = score_item(p, w);
      if (itm.e2 <= itm.a) continue;
      const int bh = itm.bh;
      float* out = p.scores + static_cast<int64_t>(bh) * n;
      const float* rw = p.raw + static_cast<int64_t>(bh) * n;
      const int t_beg = itm.a * kBN, t_end = min(itm.e2 * kBN, n);
      for (int b0 = t_beg; b0 < t_end; b0 += blk) {
        const int b1 = min(b0 + blk, t_end);
        const int lo = b0 - R, cnt = b1 - b0 + 2 * R;
#pragma unroll 4
        for (int j = threadIdx.x; j < cnt; j += 32 * kEpiWarps) {
          const int x = lo + j;
          float v = -CUDART_INF_F;
          if (x >= 0 && x < n) {
            const float q0 = __ldcg(rw + x), q1 = __ldcg(rw + part + x);
            const float q2 = __ldcg(rw + 2 * part + x), q3 = __ldcg(rw + 3 * part + x);
            v = (q0 + q1) + (q2 + q3);
          }
          stg[j] = v;
        }
        epi_sync();
        for (int t = b0 + threadIdx.x; t < b1; t += 32 * kEpiWarps) {
          const float* wv = stg + (t - b0);  // taps t-R .. t+R
          float mx = wv[R];
          for (int j = 0; j <= 2 * R; ++j) mx = fmaxf(mx, wv[j]);
          out[t] = mx;
          if (MODE == 4 && p.sel_mode == 1) sp[t - t_beg] = mx;
        }
        epi_sync();
      }
    }
    if (MODE == 4 && p.sel_mode == 1) {
      // one wave, every CTA holds one chunk (possibly without scored keys) and
      // takes part in the selection's grid barriers
      mine = score_item(p, 0);
      if (warp < kSelWarps) {
        const int b = mine.bh / p.hkv, h = mine.bh - b * p.hkv;
        const int t_beg = mine.a * kBN, t_end = min(mine.e2 * kBN, n);
        select_phase(p, sm, b, h, mine.bh, mine.chunk, n, t_beg, max(t_end - t_beg, 0), sp, n_bar);
      }
    } else if (MODE == 4 && p.sel_mode == 2) {
      // every pooled score is in global memory: the grid-wide search over them,
      // its state in the Q_win region and its key cache in the K ring
      epi_grid_sync(p.gridbar, n_bar);
      static_assert(sizeof(GSelSmem) <= sizeof(sm.q), "grid-select state must fit in the Q_win region");
      uint8_t* base = reinterpret_cast<uint8_t*>(&sm.q[0][0][0]);
      gsel_body(p.gs, *reinterpret_cast<GSelSmem*>(base), reinterpret_cast<uint32_t*>(base + gsel_cache_off()),
                EpiCx{static_cast<int>(blockIdx.y * gridDim.x + blockIdx.x), static_cast<int>(gridDim.x * gridDim.y)});
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem, kCols);
  }
}

// ------------------------------------------------------- host helpers ----
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encoder() {
  // a driver entry point: the same for every device, resolved once
  static const EncodeTiled fn = []() -> EncodeTiled {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiled>(ptr);
    return nullptr;
  }();
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

// Persistent schedule of one scoring launch (one CTA per SM): each KV head
// cut into `chunks` key chunks, the bh * chunks items dealt round robin over
// `grid` CTAs, `waves` items per CTA at most.  The chunk count minimises the
// busiest CTA's tiles plus a per-item cost (Q_win reload, pipeline restart
// ~ 1.5 tiles), fewer chunks on ties; heads that fit one wave keep one item
// per CTA: batch 1 at 16k -> 16 chunks per head, batch 1 at 128k -> 18,
// batch 4 at 16k -> 4, batch 32 at 16k -> 4 (seven items per CTA).
struct Waves {
  int chunks, waves, grid;
};
Waves score_waves(int bh, int T) {
  static std::atomic<int> sms_of[kMaxDevices];
  const int sms = per_device(sms_of, sm_count);
  const int n_tiles = (T + kBN - 1) / kBN;
  static const int force_chunks = [] {  // tuning experiments: FKV_SCORE_CHUNKS
    const char* e = getenv("FKV_SCORE_CHUNKS");
    return e ? atoi(e) : 0;
  }();
  Waves best{1, 1, 1};
  double best_cost = 1e300;
  // heads that fit one wave stay in one (one item per CTA: the per-chunk
  // selection and no Q_win reloads): the most chunks that still fit
  const int one_wave = bh <= sms ? sms / bh : 0;
  for (int c = 1; c <= n_tiles && c <= 256; ++c) {
    if (force_chunks > 0 && c != force_chunks) continue;
    if (force_chunks == 0 && one_wave > 0 && c > one_wave) break;
    const int64_t items = static_cast<int64_t>(bh) * c;
    const int64_t waves = (items + sms - 1) / sms;
    const double cost = static_cast<double>(waves) * ((n_tiles + c - 1) / c + 1.5);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best.chunks = c;
      best.waves = static_cast<int>(waves);
      best.grid = static_cast<int>(items < sms ? items : sms);
    }
  }
  return best;
}

namespace {

template <int GW>
int launch_score(const CUtensorMap& tq, const CUtensorMap& tk, const ScoreParams& p, int grid, int mode,
                 cudaStream_t st, size_t reset_bytes) {
  const size_t smem = sizeof(ScoreSmem<GW>) + 1024;
  static std::atomic<int> ready[kMaxDevices];  // smem attributes set on this device
  const int rc0 = per_device(ready, [smem](int) {
    for (auto fn : {score_kernel<3, GW, false>, score_kernel<4, GW, false>, score_kernel<3, GW, true>,
                    score_kernel<4, GW, true>})
      if (int rc = cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   smem),
                              "score smem attribute"))
        return rc;
    return 1;
  });
  if (rc0 < 0) return rc0;
  // grid barrier counters (+ the selection's zeroed histograms right after them)
  if (int rc = cuda_check(cudaMemsetAsync(p.gridbar, 0, reset_bytes, st), "score workspace reset")) return rc;
  cudaLaunchConfig_t cfg = {};
  // one wave: a (chunks, heads) grid (measured: the same CTAs as a 1-D grid
  // stream K ~30 % faster -- block placement over the two dies)
  cfg.gridDim = p.n_waves == 1 && getenv("FKV_SCORE_1D") == nullptr ? dim3(p.n_chunks, p.bh_total, 1)
                                                                    : dim3(grid, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // grid barriers: every CTA co-resident (one per SM)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const bool multi = p.n_waves > 1;
  auto fn = mode == 4 ? (multi ? score_kernel<4, GW, true> : score_kernel<4, GW, false>)
                      : (multi ? score_kernel<3, GW, true> : score_kernel<3, GW, false>);
  return cuda_check(cudaLaunchKernelEx(&cfg, fn, tq, tk, p), "score launch");
}

// Workspace: stats | raw | gridbar | zeroed selection state | per-chunk counts | standalone select
struct ScoreLayout {
  Waves wv;
  int bh;
  int64_t stats, raw, gridbar, zero, zero_bytes1, zero_bytes2, counts, sel, total;
};

ScoreLayout score_layout(int batch, int hkv, int T, int window, int group) {
  ScoreLayout L{};
  const int gw = group * window;
  L.bh = batch * hkv;
  L.wv = score_waves(L.bh > 0 ? L.bh : 1, T);
  auto a16 = [](int64_t x) { return (x + 255) & ~int64_t(255); };
  const int64_t n = T - window;
  L.stats = 0;
  L.raw = a16(L.stats + static_cast<int64_t>(L.bh) * L.wv.chunks * gw * 2 * 4);
  L.gridbar = a16(L.raw + static_cast<int64_t>(L.bh) * n * 4 * kRawParts);  // column partials
  L.zero = L.gridbar + 256;
  // sel_mode 1: per-pass per-head digit histograms; sel_mode 2: the grid
  // search's barrier (256 B), three histogram buffers (two zeroed) and counts
  L.zero_bytes1 = static_cast<int64_t>(kSelPasses) * L.bh * 512 * 4;
  L.zero_bytes2 = 256 + static_cast<int64_t>(2) * L.bh * 512 * 4;
  const int64_t zone = std::max(L.zero_bytes1, 256 + static_cast<int64_t>(kGBufs) * L.bh * 512 * 4 +
                                                   static_cast<int64_t>(L.wv.grid) * 8);
  L.counts = a16(L.zero + zone);
  L.sel = a16(L.counts + static_cast<int64_t>(L.bh) * L.wv.chunks * 8);
  L.total = a16(L.sel + fkv_ada_select_workspace_bytes(batch, hkv, T - window));
  return L;
}

int score_common(const void* q_win, const void* k, int32_t batch, int32_t hq, int32_t hkv, int32_t T,
                 int32_t window, int32_t pool_k, float sm_scale, float* scores, void* workspace,
                 ScoreParams& p, ScoreLayout& L, CUtensorMap& tq, CUtensorMap& tk) {
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
  L = score_layout(batch, hkv, T, window, group);
  if (int rc = make_map(&tq, q_win, static_cast<int64_t>(batch) * hq * window, 128)) return rc;
  if (int rc = make_map(&tk, k, static_cast<int64_t>(batch) * hkv * T, kBN)) return rc;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  p = ScoreParams{};
  p.T = T;
  p.window = window;
  p.group = group;
  p.hkv = hkv;
  p.n_chunks = L.wv.chunks;
  p.n_waves = L.wv.waves;
  p.bh_total = L.bh;
  p.q_rows_per_req = hq * window;
  p.scale_log2 = sm_scale * kLog2e;
  p.stats = reinterpret_cast<float*>(ws + L.stats);
  p.raw = reinterpret_cast<float*>(ws + L.raw);
  p.scores = scores;
  p.pool_r = pool_k / 2;
  p.gridbar = reinterpret_cast<GridBar*>(ws + L.gridbar);
  p.hist = reinterpret_cast<uint32_t*>(ws + L.zero);
  p.counts = reinterpret_cast<int32_t*>(ws + L.counts);
  return FKV_OK;
}
}  // namespace
}  // namespace fkv

extern "C" int fkv__score_stamps(unsigned long long* host) {
  return fkv::cuda_check(cudaMemcpyFromSymbol(host, fkv::g_sstamps, sizeof(unsigned long long) * 64),
                         "score stamps");
}

extern "C" int64_t fkv_score_workspace_bytes(int32_t batch, int32_t hkv, int32_t T, int32_t window,
                                             int32_t group) {
  return fkv::score_layout(batch, hkv, T, window, group).total;
}

extern "C" int fkv_snapkv_score(const void* q_win, const void* k, int32_t batch, int32_t hq,
                                int32_t hkv, int32_t T, int32_t window, int32_t pool_k,
                                float sm_scale, float* scores, void* workspace, void* stream) {
  using namespace fkv;
  ScoreParams p;
  ScoreLayout L;
  CUtensorMap tq, tk;
  if (int rc = score_common(q_win, k, batch, hq, hkv, T, window, pool_k, sm_scale, scores, workspace,
                            p, L, tq, tk))
    return rc;
  auto st = static_cast<cudaStream_t>(stream);
  return p.group * window == 128 ? launch_score<128>(tq, tk, p, L.wv.grid, 3, st, 256)
                                 : launch_score<256>(tq, tk, p, L.wv.grid, 3, st, 256);
}

extern "C" int fkv_snapkv_select(const void* q_win, const void* k, int32_t batch, int32_t hq,
                                 int32_t hkv, int32_t T, int32_t window, int32_t pool_k,
                                 float sm_scale, int32_t budget, int32_t floor_k, float* scores,
                                 int32_t* budgets, int64_t* offsets, int32_t* idx, void* workspace,
                                 void* stream) {
  using namespace fkv;
  if (!budgets || !offsets || !idx) return set_error(FKV_ERR_INVALID, "fkv_snapkv_select: null pointer");
  const int n = T - window, sel = budget - window;
  if (sel < 0 || sel > n || floor_k < 0 || floor_k > sel)
    return set_error(FKV_ERR_INVALID, "fkv_snapkv_select: need 0 <= floor <= budget-window <= T-window");
  ScoreParams p;
  ScoreLayout L;
  CUtensorMap tq, tk;
  if (int rc = score_common(q_win, k, batch, hq, hkv, T, window, pool_k, sm_scale, scores, workspace,
                            p, L, tq, tk))
    return rc;
  auto st = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  const int max_chunk_keys = ((T + kBN - 1) / kBN + L.wv.chunks - 1) / L.wv.chunks * kBN;
  if (L.wv.waves == 1 && hkv <= kSelMaxHeads && max_chunk_keys <= kSelMaxKeys) {
    p.sel_mode = 1;  // every CTA selects within its own chunk
  } else if (hkv <= kGMaxHeads && L.bh <= (kGMaxPieces - 2) * L.wv.grid) {
    p.sel_mode = 2;  // grid-wide search over the pooled scores, same launch
  } else {           // two launches: scoring, then the standalone grid select (select.cu)
    if (int rc = p.group * window == 128 ? launch_score<128>(tq, tk, p, L.wv.grid, 3, st, 256)
                                         : launch_score<256>(tq, tk, p, L.wv.grid, 3, st, 256))
      return rc;
    return fkv_ada_select(scores, batch, hkv, n, budget, window, floor_k, budgets, offsets, idx, ws + L.sel,
                          stream);
  }
  p.budget = budget;
  p.floor_k = floor_k;
  p.rest_total = hkv * sel - hkv * floor_k;
  p.budgets = budgets;
  p.offsets = offsets;
  p.idx = idx;
  size_t reset = 256 + static_cast<size_t>(p.sel_mode == 1 ? L.zero_bytes1 : L.zero_bytes2);
  if (p.sel_mode == 2) {
    GSelParams& g = p.gs;
    g.scores = scores;
    g.hkv = hkv;
    g.n = n;
    g.window = window;
    g.f = floor_k;
    g.R = p.rest_total;
    g.budget = budget;
    g.select = 1;
    g.req0 = 0;
    g.bh_total = L.bh;
    g.total = static_cast<int64_t>(L.bh) * n;
    g.bar = reinterpret_cast<unsigned*>(ws + L.zero);
    g.hist = reinterpret_cast<uint32_t*>(ws + L.zero + 256);
    g.counts = reinterpret_cast<int2*>(ws + L.zero + 256 + static_cast<int64_t>(kGBufs) * L.bh * 512 * 4);
    g.budgets = budgets;
    g.offsets = offsets;
    g.idx = idx;
    const int64_t span_keys = (g.total + L.wv.grid - 1) / L.wv.grid + 1;
    // the CTA's keys fit in the (idle) Q_win + K ring after the select state
    g.cache = span_keys <= (p.group * window == 128 ? gsel_cache_keys<128>() : gsel_cache_keys<256>());
  }
  return p.group * window == 128 ? launch_score<128>(tq, tk, p, L.wv.grid, 4, st, reset)
                                 : launch_score<256>(tq, tk, p, L.wv.grid, 4, st, reset);
}

// A18 Ada budget split + K2 per-head top-k: the grid-wide radix search
// shared by select.cu (standalone launch over scores in HBM) and score.cu
// (persistent fused launch, after the scoring passes).  See select.cu for
// the algorithm and DESIGN.md "Algorithm definitions" for the tie rules.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace fkv {
namespace {

__device__ __forceinline__ uint32_t orderable(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// ------------------------------------------- A18 + K2, grid-wide search ----
// One cooperative launch for every (request, head).  The keys of all heads,
// laid end to end, are cut into equal contiguous ranges, one per persistent
// CTA (a range covers the tail of one head, whole heads, the head of
// another: its "pieces"), and an MSB-first radix search over the 32-bit
// orderable score (8-bit digits, four passes) runs for all requests at once:
// per pass every CTA adds its pieces' digit histograms into per-head global
// histograms, one grid barrier, and every CTA re-derives the decisions of
// the requests / heads it touches (identical on every CTA, no second
// barrier).
//
// Two searches per head:
//   global   the Ada split in its floor-free form: with N_h(tau) = #{keys of
//            head h >= tau} the non-floor picks of head h are
//            max(0, N_h - floor), so tau is the largest threshold with
//            G(tau) = sum_h max(0, N_h(tau) - floor) >= R (R = Hkv (B - w - f));
//   floor    the head's own f-th largest score, kept when it ends below its
//            floor (N_h < f: exactly its top-f).
// A head's global histogram is skipped once N_h < f is certain (it adds
// nothing to G), its floor histogram once N_h >= f is certain, and the two
// are one histogram while both searches share a prefix (always in pass 0).
// Four passes fix the threshold score s*; ties at s* are resolved in the
// global order (head asc, token asc) from per-piece tie counts, so no pass
// over the index bits is needed.  Per-CTA (chosen, tied) counts of the last
// piece meet after a fifth barrier and every CTA writes its chosen tokens in
// ascending order.  Same results as ada_budgets_kernel + topk_select_kernel
// (and the oracle).
constexpr int kGThreads = 512, kGWarps = kGThreads / 32;
constexpr int kGMaxHeads = 16;   // Hkv: one warp per head in the decisions
constexpr int kGMaxPieces = 16;  // heads touched per CTA
constexpr int kGBufs = 3;        // rotating per-pass histogram buffers
constexpr int kGMinKeys = 2048;  // keys per CTA, at least
constexpr int kGUnroll = 4;
constexpr int kGCacheBytes = 84 * 1024;  // key cache per CTA (two CTAs per SM still fit)

struct GSelParams {
  const float* scores;  // [BH, n] of this launch
  int hkv, n, window, f, R, budget;
  const int32_t* head_k;       // top-k mode: per-head budgets of this launch (incl. window); null = Ada
  const int32_t* budgets_all;  // top-k mode: all budgets (offsets are their exclusive prefix)
  int select;                  // 0: budgets only (Ada mode)
  int cache;                   // 1: the CTA's keys stay in shared memory after pass 0
  int req0, bh_total;   // first request of this launch; Bt*Hkv over all launches
  int64_t total;        // BH * n
  uint32_t* hist;       // [kGBufs][BH][2][256] (buffers 0, 1 zeroed by the host)
  int2* counts;         // [grid] (chosen outright, ties) of each CTA's last piece
  unsigned* bar;        // grid barrier counter (zeroed by the host)
  int32_t* budgets;     // [BH] of this launch
  int64_t* offsets;     // [BH (+1)] of this launch
  int32_t* idx;         // absolute
};

struct GReq {  // global search of one request
  uint32_t prefix, mask;
  int exact, hstar, kstar;
  int above[kGMaxHeads], n_at[kGMaxHeads];
};
struct GHead {  // floor search of one head (its own top-f; top-k mode: f = k)
  uint32_t prefix, mask;
  int exact, above, n_at, f;
};
struct GRule {  // final keep rule of one head: 0 = ties ranked, 1 = o >= prefix, 2 = none
  uint32_t prefix;
  int kind, ktie;
};

struct GSelSmem {
  uint32_t hist[2][256];
  int32_t suf[kGMaxHeads][256];
  GReq req[kGMaxPieces];
  GHead fl[kGMaxPieces];
  GRule rule[kGMaxPieces];
  uint8_t fact[kGMaxPieces];  // floor histogram built this pass
  int2 pc[kGMaxPieces][kGWarps];  // (chosen outright, ties) per piece and warp segment
  int64_t off[kGMaxPieces];       // index-list offset of each local head
  int32_t bud[kGMaxPieces];       // budget of each local head
  long long red[kGWarps];
  int32_t wt[2][kGWarps];
  int32_t tmp;
};

// diagnostics: %globaltimer stamps of CTA 0 (fkv__select_stamps)
__device__ unsigned long long g_gstamps[32];
__device__ __forceinline__ void gstamp(int cta, int i) {
  if (cta == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_gstamps[i] = t;
  }
}

// Grid barrier over a counter zeroed per launch: arrival k of every CTA
// lands in [k*N, (k+1)*N), so the k-th barrier's target is known up front
// and the arrival is a fire-and-forget release reduction -- the poll that
// follows it is the only round trip (a returning atomic costs one more).
// `sync` is the block barrier of the threads taking part.
template <class Sync>
__device__ __forceinline__ void grid_sync_n(unsigned* bar, unsigned& k, unsigned ncta, Sync&& sync) {
  sync();
  if (threadIdx.x == 0) {
    const unsigned target = ++k * ncta;
    unsigned v;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    while (true) {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if (v >= target) break;
      __nanosleep(32);
    }
  }
  sync();
}

// Suffix counts of one 256-bin histogram (8 bins per lane): s[j] = base +
// #keys in bins >= 8*lane + j; `up` = s of bin 8*lane + 8 (base past bin 255).
__device__ __forceinline__ void warp_suffix_of(const uint4 x0, const uint4 x1, int base, int (&s)[8], int& up) {
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
__device__ __forceinline__ void warp_suffix(const uint32_t* gh, int base, int (&s)[8], int& up) {
  const int lane = threadIdx.x & 31;
  warp_suffix_of(__ldcg(reinterpret_cast<const uint4*>(gh + 8 * lane)),
                 __ldcg(reinterpret_cast<const uint4*>(gh + 8 * lane + 4)), base, s, up);
}

__device__ __forceinline__ int rule_class(const GRule& r, uint32_t o) {
  if (r.kind == 2) return 0;
  if (r.kind == 1) return o >= r.prefix;
  return o > r.prefix ? 1 : (o == r.prefix ? 2 : 0);
}

// Piece [lo, hi) of a head's keys s[]: the 16-B aligned body [a, b) and the
// (at most 3 + 3) keys around it.
__device__ __forceinline__ void split_aligned(const float* s, int lo, int hi, int& a, int& b) {
  const int mis = static_cast<int>((reinterpret_cast<uintptr_t>(s + lo) >> 2) & 3);
  a = min(hi, lo + ((4 - mis) & 3));
  b = a + ((hi - a) & ~3);
}

// fn(valid, orderable key) over keys [lo, hi) by the whole CTA, every call
// warp-uniform; the body in float4 loads, kGUnroll of them in flight per
// thread.
template <class Fn>
__device__ __forceinline__ void for_keys(const float* s, int lo, int hi, Fn&& fn) {
  const int tid = threadIdx.x;
  int a, b;
  split_aligned(s, lo, hi, a, b);
  {
    const int nh = a - lo;
    const int i = tid < nh ? lo + tid : b + tid - nh;
    const bool in = tid < nh + (hi - b);
    fn(in, in ? orderable(__ldg(s + i)) : 0u, i);
  }
  const float4* v4 = reinterpret_cast<const float4*>(s + a);
  const int nv = (b - a) >> 2;
  for (int base = 0; base < nv; base += kGUnroll * kGThreads) {
    float4 x[kGUnroll];
#pragma unroll
    for (int u = 0; u < kGUnroll; ++u) {
      const int j = base + u * kGThreads + tid;
      x[u] = j < nv ? __ldg(v4 + j) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kGUnroll; ++u) {
      const int j = base + u * kGThreads + tid;
      const bool in = j < nv;
      fn(in, orderable(x[u].x), a + 4 * j);
      fn(in, orderable(x[u].y), a + 4 * j + 1);
      fn(in, orderable(x[u].z), a + 4 * j + 2);
      fn(in, orderable(x[u].w), a + 4 * j + 3);
    }
  }
}

// The A18 + K2 grid-wide search over the scores in p.scores, run by 512
// threads (threadIdx.x 0..511) of each of the cx.ncta CTAs taking part: the
// standalone select launch (grid_select_kernel) and the persistent fused
// scoring launch (score.cu, on its epilogue warps).  Cx supplies the CTA's
// index and count and its block / grid barriers.
template <class Cx>
__device__ void gsel_body(const GSelParams& p, GSelSmem& sm, uint32_t* skeys, const Cx& cx) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int HK = p.hkv, f = p.f, R = p.R, n = p.n;
  const int64_t k0 = static_cast<int64_t>(cx.cta) * p.total / cx.ncta;
  const int64_t k1 = static_cast<int64_t>(cx.cta + 1) * p.total / cx.ncta;
  const int bh_lo = static_cast<int>(k0 / n), rq_lo = bh_lo / HK;
  const int n_lh = k1 > k0 ? static_cast<int>((k1 - 1) / n) - bh_lo + 1 : 0;
  const int n_lr = k1 > k0 ? static_cast<int>((k1 - 1) / n) / HK - rq_lo + 1 : 0;
  const int64_t buf_words = p.total / n * 512;
  // piece of local head lh: keys [lo, hi) of head bh_lo + lh
  auto piece = [&](int lh, int& lo, int& hi) {
    const int64_t h0 = static_cast<int64_t>(bh_lo + lh) * n;
    lo = static_cast<int>(max(k0, h0) - h0);
    hi = static_cast<int>(min(k1, h0 + n) - h0);
  };

  for (int i = tid; i < n_lr * kGMaxHeads; i += kGThreads) {
    sm.req[i / kGMaxHeads].above[i % kGMaxHeads] = 0;
    sm.req[i / kGMaxHeads].n_at[i % kGMaxHeads] = R > 0 ? n : 0;
  }
  if (tid < n_lr) {
    GReq& r = sm.req[tid];
    r.prefix = r.mask = 0;
    r.exact = R <= 0;
    r.hstar = HK;
    r.kstar = 0;
  }
  if (tid < n_lh) {
    int fh = f;
    if (p.head_k) fh = min(max(p.head_k[bh_lo + tid] - p.window, 0), n);
    // no floor search: none to keep, all kept (prefix 0 takes every key), or budgets only
    sm.fl[tid] = GHead{0u, 0u, fh <= 0 || fh >= n || !p.select, 0, n, fh};
  }
  gstamp(cx.cta, 0);
  cx.sync();
  unsigned n_bar = 0;  // grid barriers passed (thread 0)

  for (int pass = 0, shift = 24; pass < 4; ++pass, shift -= 8) {
    uint32_t* hb = p.hist + (pass % kGBufs) * buf_words;
    gstamp(cx.cta, 23 + 2 * pass);
    // ---- my pieces' digit histograms into hb
    for (int lh = 0; lh < n_lh; ++lh) {
      const int bh = bh_lo + lh, h = bh % HK;
      const GReq& rq = sm.req[bh / HK - rq_lo];
      const GHead& fh = sm.fl[lh];
      // global: N_h >= f still possible; floor: N_h < f still possible
      const bool ga = !rq.exact && rq.n_at[h] >= f;
      const bool fa = !fh.exact && (rq.exact ? rq.n_at[h] < fh.f : rq.above[h] < fh.f);
      const bool same = ga && fa && rq.prefix == fh.prefix && rq.mask == fh.mask;
      if (tid == 0) sm.fact[lh] = fa;
      if (!ga && !fa) continue;
      (&sm.hist[0][0])[tid] = 0;
      cx.sync();
      int lo, hi;
      piece(lh, lo, hi);
      const float* s = p.scores + static_cast<int64_t>(bh) * n;
      const uint32_t gp = rq.prefix, gm = rq.mask, fp = fh.prefix, fm = fh.mask;
      uint32_t* skh = skeys + (static_cast<int64_t>(bh) * n - k0);  // this head's keys (p.cache)
      auto add = [&](bool in, uint32_t o, int i) {
        if (p.cache && pass == 0 && in) skh[i] = o;
        const uint32_t dig = (o >> shift) & 255u;
        const uint32_t dg = in && (o & gm) == gp ? dig : 256u;
        const uint32_t df = in && (o & fm) == fp ? dig : 256u;
        // plain shared atomics: measured on par with or faster than
        // warp-aggregated adds (match.any), also on pooled Ada-SnapKV scores
        // whose top byte takes few values
        if (ga && dg < 256u) atomicAdd(&sm.hist[0][dg], 1u);
        if (fa && !same && df < 256u) atomicAdd(&sm.hist[1][df], 1u);
      };
      if (p.cache && pass > 0) {  // keys from the shared-memory cache
        for (int base = lo; base < hi; base += kGThreads) {
          const int i = base + tid;
          const bool in = i < hi;
          add(in, in ? skh[i] : 0u, i);
        }
      } else {
        for_keys(s, lo, hi, add);
      }
      cx.sync();
      if (lh == 0) gstamp(cx.cta, 24 + 2 * pass);
      uint32_t* gh = hb + static_cast<int64_t>(bh) * 512;
      if (tid < 256) {
        const uint32_t c = sm.hist[0][tid];
        if (c) {
          if (ga) atomicAdd(gh + tid, c);
          if (same) atomicAdd(gh + 256 + tid, c);
        }
      } else if (fa && !same) {
        const uint32_t c = sm.hist[1][tid - 256];
        if (c) atomicAdd(gh + tid, c);
      }
      cx.sync();
    }
    gstamp(cx.cta, 1 + 3 * pass);
    cx.grid(p.bar, n_bar);
    gstamp(cx.cta, 2 + 3 * pass);
    // the buffer of pass + 2 was last read by pass - 1's decisions (before
    // this barrier) and is next written after the next one; the CTA holding
    // a head's first key clears it
    if (pass < 2) {
      uint32_t* zb = p.hist + ((pass + 2) % kGBufs) * buf_words;
      for (int lh = 0; lh < n_lh; ++lh) {
        int lo, hi;
        piece(lh, lo, hi);
        if (lo == 0) (zb + static_cast<int64_t>(bh_lo + lh) * 512)[tid] = 0;
      }
    }
    // my heads' floor histograms (one warp per local head), loaded now so the
    // round trip overlaps the global decisions' (both are L2 reads of this
    // pass's histograms)
    const bool fjob = wid < n_lh && sm.fact[wid];
    uint4 fx0 = make_uint4(0, 0, 0, 0), fx1 = fx0;
    if (fjob) {
      const uint32_t* fg = hb + static_cast<int64_t>(bh_lo + wid) * 512 + 256;
      fx0 = __ldcg(reinterpret_cast<const uint4*>(fg + 8 * lane));
      fx1 = __ldcg(reinterpret_cast<const uint4*>(fg + 8 * lane + 4));
    }
    // ---- global decisions of my requests: d* = max{d : G(d) >= R}
    for (int lr = 0; lr < n_lr; ++lr) {
      GReq& rq = sm.req[lr];
      if (rq.exact) continue;
      const int b = rq_lo + lr;
      if (wid < HK) {
        int sv[8], up;
        warp_suffix(hb + static_cast<int64_t>(b * HK + wid) * 512, rq.above[wid], sv, up);
#pragma unroll
        for (int j = 0; j < 8; ++j) sm.suf[wid][8 * lane + j] = sv[j];
      }
      cx.sync();
      int gd = 0;
      if (tid < 256)
        for (int h = 0; h < HK; ++h) gd += max(0, sm.suf[h][tid] - f);
      const int dstar = cx.count(tid < 256 && gd >= R) - 1;
      if (tid == dstar) sm.tmp = gd == R;
      cx.sync();
      if (tid < HK) {
        rq.n_at[tid] = sm.suf[tid][dstar];
        if (dstar < 255) rq.above[tid] = sm.suf[tid][dstar + 1];
      }
      if (tid == 0) {
        rq.prefix |= static_cast<uint32_t>(dstar) << shift;
        rq.mask |= 255u << shift;
        rq.exact = sm.tmp;
      }
      cx.sync();
    }
    gstamp(cx.cta, 3 + 3 * pass);
    // ---- floor decisions of my heads (one warp each): f-th largest
    for (int lh = wid; lh < n_lh; lh += kGWarps) {  // n_lh <= kGMaxPieces == kGWarps: one pass
      GHead& fh = sm.fl[lh];
      if (!sm.fact[lh]) continue;
      int sv[8], up;
      warp_suffix_of(fx0, fx1, fh.above, sv, up);
      int c = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) c += sv[j] >= fh.f;
      const int dstar = __reduce_add_sync(0xffffffffu, c) - 1;
      int at = 0, nxt = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (8 * lane + j == dstar) {
          at = sv[j];
          nxt = j < 7 ? sv[j + 1] : up;
        }
      at = __shfl_sync(0xffffffffu, at, dstar >> 3);
      nxt = __shfl_sync(0xffffffffu, nxt, dstar >> 3);
      if (lane == 0) {
        fh.n_at = at;
        fh.above = nxt;
        fh.prefix |= static_cast<uint32_t>(dstar) << shift;
        fh.mask |= 255u << shift;
        fh.exact = at == fh.f;
      }
    }
    cx.sync();
  }

  // ---- ties at s*: walk heads in order until G reaches R exactly
  if (tid < n_lr) {
    GReq& rq = sm.req[tid];
    if (R > 0 && !rq.exact) {
      int hstar = HK, kstar = 0, need = R;
      for (int h = 0; h < HK; ++h) need -= max(0, rq.above[h] - f);
      for (int h = 0; h < HK && need > 0; ++h) {
        const int base = rq.above[h];
        const int gain = max(0, rq.n_at[h] - f) - max(0, base - f);
        if (gain >= need) {
          hstar = h;
          kstar = max(0, f - base) + need;
          need = 0;
        } else {
          need -= gain;
        }
      }
      for (int h = 0; h < HK; ++h)
        rq.n_at[h] = h < hstar ? rq.n_at[h] : (h == hstar ? rq.above[h] + kstar : rq.above[h]);
      rq.hstar = hstar;
      rq.kstar = kstar;
    }
  }
  cx.sync();
  if (tid < n_lh) {
    const int bh = bh_lo + tid, h = bh % HK;
    const GReq& rq = sm.req[bh / HK - rq_lo];
    const GHead& fh = sm.fl[tid];
    GRule r;
    if (R <= 0 || rq.n_at[h] < f) {  // below the floor (or top-k mode): own top-f
      if (fh.f <= 0) r = GRule{0u, 2, 0};
      else if (fh.exact) r = GRule{fh.prefix, 1, 0};
      else r = GRule{fh.prefix, 0, fh.f - fh.above};
    } else if (rq.exact) {
      r = GRule{rq.prefix, 1, 0};
    } else {
      r = GRule{rq.prefix, 0, h < rq.hstar ? 0x7fffffff : (h == rq.hstar ? rq.kstar : 0)};
    }
    sm.rule[tid] = r;
  }
  cx.sync();
  // budgets and index-list offsets of my heads
  if (p.head_k) {  // top-k mode: exclusive prefix of the given budgets
    const int first = p.req0 * HK + bh_lo;
    long long part = 0;
    for (int i = tid; i < first; i += kGThreads) part += p.budgets_all[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) sm.red[wid] = part;
    cx.sync();
    if (tid == 0) {
      long long off = 0;
      for (int j = 0; j < kGWarps; ++j) off += sm.red[j];
      for (int lh = 0; lh < n_lh; ++lh) {
        sm.off[lh] = off;
        sm.bud[lh] = p.head_k[bh_lo + lh];
        off += sm.bud[lh];
      }
    }
  } else if (tid < n_lh) {  // Ada mode: request b starts at b * Hkv * budget
    const int bh = bh_lo + tid, b = bh / HK, h = bh - b * HK;
    const GReq& rq = sm.req[b - rq_lo];
    auto budget_of = [&](int hh) { return p.window + f + (R > 0 ? max(0, rq.n_at[hh] - f) : 0); };
    int64_t off = static_cast<int64_t>(p.req0 + b) * HK * p.budget;
    for (int hh = 0; hh < h; ++hh) off += budget_of(hh);
    sm.off[tid] = off;
    sm.bud[tid] = budget_of(h);
  }
  cx.sync();
  if (!p.select) {  // budgets only (uniform: no barrier follows)
    for (int lh = tid; lh < n_lh; lh += kGThreads) {
      int lo, hi;
      piece(lh, lo, hi);
      if (lo == 0) p.budgets[bh_lo + lh] = sm.bud[lh];
    }
    return;
  }

  // ---- per-warp-segment counts of every piece (warp w scans a contiguous
  // 1/16 of the piece's aligned body; warp 0 also the keys before it, the
  // last warp those after it); the last piece's total is published for the
  // CTAs after me.  Budgets, offsets and window tokens by the CTA holding a
  // head's first key.
  struct Seg {
    int lo, hi, a, b, v0, v1;
  };
  auto segment = [&](const float* s, int lo, int hi) {
    Seg g;
    g.lo = lo;
    g.hi = hi;
    split_aligned(s, lo, hi, g.a, g.b);
    const int nv = (g.b - g.a) >> 2, per = (nv + kGWarps - 1) / kGWarps;
    g.v0 = min(nv, wid * per);
    g.v1 = min(nv, g.v0 + per);
    return g;
  };
  for (int lh = 0; lh < n_lh; ++lh) {
    const int bh = bh_lo + lh;
    int lo, hi;
    piece(lh, lo, hi);
    const GRule r = sm.rule[lh];
    const float* s = p.scores + static_cast<int64_t>(bh) * n;
    int c1 = 0, c2 = 0;
    if (r.kind != 2) {
      const Seg g = segment(s, lo, hi);
      auto count = [&](uint32_t o) {
        const int k = rule_class(r, o);
        c1 += k == 1;
        c2 += k == 2;
      };
      const uint32_t* skh = skeys + (static_cast<int64_t>(bh) * n - k0);
      auto key = [&](int i) { return p.cache ? skh[i] : orderable(__ldg(s + i)); };
      if (wid == 0)
        for (int i = g.lo + lane; i < g.a; i += 32) count(key(i));
      const float4* v4 = reinterpret_cast<const float4*>(s + g.a);
#pragma unroll 4
      for (int j = g.v0 + lane; j < g.v1; j += 32) {
        if (p.cache) {
          const int i = g.a + 4 * j;
          count(skh[i]);
          count(skh[i + 1]);
          count(skh[i + 2]);
          count(skh[i + 3]);
        } else {
          const float4 x = __ldg(v4 + j);
          count(orderable(x.x));
          count(orderable(x.y));
          count(orderable(x.z));
          count(orderable(x.w));
        }
      }
      if (wid == kGWarps - 1)
        for (int i = g.b + lane; i < g.hi; i += 32) count(key(i));
    }
    c1 = __reduce_add_sync(0xffffffffu, c1);
    c2 = __reduce_add_sync(0xffffffffu, c2);
    if (lane == 0) sm.pc[lh][wid] = make_int2(c1, c2);
    if (lo == 0) {  // window tokens after the head's selected ones
      const int bud = sm.bud[lh];
      const int64_t off = sm.off[lh];
      const int kept = p.head_k ? sm.fl[lh].f : bud - p.window;
      for (int i = tid; i < p.window; i += kGThreads) p.idx[off + kept + i] = n + i;
      if (tid == 0) {
        if (!p.head_k) p.budgets[bh] = bud;
        p.offsets[bh] = off;
        if (p.req0 * HK + bh == p.bh_total - 1) p.offsets[bh + 1] = off + bud;
      }
    }
  }
  cx.sync();
  if (tid == 0 && n_lh > 0) {
    int x = 0, y = 0;
    for (int j = 0; j < kGWarps; ++j) x += sm.pc[n_lh - 1][j].x, y += sm.pc[n_lh - 1][j].y;
    p.counts[cx.cta] = make_int2(x, y);
  }
  gstamp(cx.cta, 20);
  cx.grid(p.bar, n_bar);
  gstamp(cx.cta, 21);

  // ---- chosen tokens of my pieces, ascending, at their place in the list;
  // each warp writes its own segment (no block barriers)
  const uint32_t lt = (1u << lane) - 1u;
  auto warp_excl = [&](int v, int& total) {  // exclusive prefix over lanes
    int incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    total = __shfl_sync(0xffffffffu, incl, 31);
    return incl - v;
  };
  for (int lh = 0; lh < n_lh; ++lh) {
    const int bh = bh_lo + lh;
    const GRule r = sm.rule[lh];
    if (r.kind == 2) continue;
    int lo, hi;
    piece(lh, lo, hi);
    int pos = 0, tie0 = 0;
    if (lo > 0) {  // earlier CTAs hold this head's keys [0, lo): their last pieces
      const int64_t h0 = static_cast<int64_t>(bh) * n;
      // first CTA c with c*total/grid <= h0 < (c+1)*total/grid
      const int c_first = static_cast<int>(((h0 + 1) * cx.ncta + p.total - 1) / p.total) - 1;
      for (int c = c_first + lane; c < static_cast<int>(cx.cta); c += 32) {
        const int2 cc = __ldcg(p.counts + c);
        pos += cc.x;
        tie0 += cc.y;
      }
      pos = __reduce_add_sync(0xffffffffu, pos);
      tie0 = __reduce_add_sync(0xffffffffu, tie0);
      pos += min(tie0, r.ktie);
    }
    // this warp's segment: chosen outright and ties of the segments before it
    int c1b = 0, tb = 0;
    for (int j = 0; j < wid; ++j) c1b += sm.pc[lh][j].x, tb += sm.pc[lh][j].y;
    int tie_run = tie0 + tb;
    pos += c1b + min(tie_run, r.ktie) - min(tie0, r.ktie);
    int32_t* out = p.idx + sm.off[lh];
    const float* s = p.scores + static_cast<int64_t>(bh) * n;
    const Seg g = segment(s, lo, hi);
    const uint32_t* skh = skeys + (static_cast<int64_t>(bh) * n - k0);
    auto emit_scalar = [&](int i0, int i1) {
      for (int base = i0; base < i1; base += 32) {
        const int i = base + lane;
        const int k = i < i1 ? rule_class(r, p.cache ? skh[i] : orderable(__ldg(s + i))) : 0;
        const uint32_t ties = __ballot_sync(0xffffffffu, k == 2);
        const bool take = k == 1 || (k == 2 && tie_run + __popc(ties & lt) < r.ktie);
        const uint32_t bal = __ballot_sync(0xffffffffu, take);
        if (take) out[pos + __popc(bal & lt)] = i;
        pos += __popc(bal);
        tie_run += __popc(ties);
      }
    };
    if (wid == 0) emit_scalar(g.lo, g.a);
    const float4* v4 = reinterpret_cast<const float4*>(s + g.a);
    for (int jb = g.v0; jb < g.v1; jb += 32) {
      const int j = jb + lane;
      int k[4] = {0, 0, 0, 0};
      if (j < g.v1) {
        if (p.cache) {
          const int i = g.a + 4 * j;
          k[0] = rule_class(r, skh[i]);
          k[1] = rule_class(r, skh[i + 1]);
          k[2] = rule_class(r, skh[i + 2]);
          k[3] = rule_class(r, skh[i + 3]);
        } else {
          const float4 x = __ldg(v4 + j);
          k[0] = rule_class(r, orderable(x.x));
          k[1] = rule_class(r, orderable(x.y));
          k[2] = rule_class(r, orderable(x.z));
          k[3] = rule_class(r, orderable(x.w));
        }
      }
      int t_all, n_all;
      int tr = tie_run + warp_excl((k[0] == 2) + (k[1] == 2) + (k[2] == 2) + (k[3] == 2), t_all);
      bool tk[4];
      int nt = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        tk[c] = k[c] == 1;
        if (k[c] == 2) tk[c] = tr++ < r.ktie;
        nt += tk[c];
      }
      int q = pos + warp_excl(nt, n_all);
      const int i0 = g.a + 4 * j;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (tk[c]) out[q++] = i0 + c;
      pos += n_all;
      tie_run += t_all;
    }
    if (wid == kGWarps - 1) emit_scalar(g.b, g.hi);
  }
  gstamp(cx.cta, 22);
}

}  // namespace
}  // namespace fkv

// A18 Ada cross-head budget split + K2 per-head top-k selection.
//
// No reference implementation exists (the paper used KVPress
// AdaKV).  Definitions and tie rules are fixed in DESIGN.md
// "Algorithm definitions" and restated in oracle/kv.py:
//   per-head order  (score desc, token asc)
//   global order    (score desc, head asc, token asc)
// Both are made total by a 64-bit composite key
//   key64 = orderable(score) << 32 | (0xffffffff - index)
// (index = token, or head * n + token for the global order), so a radix
// select over key64 returns exactly k elements and results are exact
// functions of the fp32 score tensor -- bit-exact against the oracle fed the
// same scores.
//
// Radix select: one CTA, MSB-first 8-bit digits, warp-aggregated
// shared-memory histograms (__match_any_sync: the top digits of float keys
// are nearly all equal, so naive per-thread atomics would serialise), early
// exit when the threshold bucket is taken whole.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace fkv {
namespace {

constexpr int kThreads = 1024;
constexpr uint64_t kNone = ~0ull;

__device__ __forceinline__ uint32_t orderable(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ uint64_t compose(float s, uint32_t index) {
  return (static_cast<uint64_t>(orderable(s)) << 32) | (0xffffffffu - index);
}

struct SelectSmem {
  uint32_t hist[256];
  uint32_t gh[256];  // cluster-summed histogram
  uint32_t count;
  uint32_t digit, above;
  uint32_t warp_tot[32];
  uint64_t tau_head[64];
  uint32_t count_head[64];
};

// Threshold tau such that exactly k of the valid elements have key >= tau
// (1 <= k <= #valid).  key_of(i, &key) -> valid.
template <class KeyOf>
__device__ uint64_t cta_select_kth(KeyOf key_of, int n, uint32_t k, SelectSmem& sm) {
  uint64_t prefix = 0, mask = 0;
  uint32_t need = k;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sm.hist[i] = 0;
    __syncthreads();
    for (int base = 0; base < n; base += blockDim.x) {
      const int i = base + threadIdx.x;
      uint64_t key = 0;
      const bool ok = i < n && key_of(i, key) && (key & mask) == prefix;
      const uint32_t d = ok ? static_cast<uint32_t>(key >> shift) & 255u : 256u;
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      if (ok && lane == __ffs(peers) - 1) atomicAdd(&sm.hist[d], __popc(peers));
    }
    __syncthreads();
    if (warp == 0) {
      // lane L owns bins [8L, 8L+8); find the bin holding the need-th largest
      uint32_t local = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) local += sm.hist[8 * lane + j];
      uint32_t incl = local;  // inclusive suffix sum over lanes >= this one
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t v = __shfl_down_sync(0xffffffffu, incl, off);
        if (lane + off < 32) incl += v;
      }
      const uint32_t suffix = incl - local;
      if (suffix < need && suffix + local >= need) {
        uint32_t acc = suffix;
        for (int j = 7; j >= 0; --j) {
          const uint32_t c = sm.hist[8 * lane + j];
          if (acc + c >= need) {
            sm.digit = 8 * lane + j;
            sm.above = acc;
            break;
          }
          acc += c;
        }
      }
    }
    __syncthreads();
    const uint32_t d = sm.digit;
    need -= sm.above;
    prefix |= static_cast<uint64_t>(d) << shift;
    mask |= 255ull << shift;
    const bool whole = sm.hist[d] == need;
    __syncthreads();
    if (whole) return prefix;
  }
  return prefix;
}

// Exclusive block scan of a 0/1 flag (one per thread), returns the total.
__device__ uint32_t block_flag_scan(bool flag, uint32_t& before, SelectSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t ballot = __ballot_sync(0xffffffffu, flag);
  const uint32_t in_warp = __popc(ballot & ((1u << lane) - 1u));
  if (lane == 0) sm.warp_tot[warp] = __popc(ballot);
  __syncthreads();
  uint32_t warp_base = 0, total = 0;
  const int nw = blockDim.x >> 5;
  for (int w = 0; w < nw; ++w) {
    const uint32_t t = sm.warp_tot[w];
    if (w < warp) warp_base += t;
    total += t;
  }
  __syncthreads();
  before = warp_base + in_warp;
  return total;
}

__device__ uint32_t block_sum(uint32_t v, SelectSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if (lane == 0) sm.warp_tot[warp] = v;
  __syncthreads();
  uint32_t total = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) total += sm.warp_tot[w];
  __syncthreads();
  return total;
}

// ---------------------------------------------------------------- A18 ----
// grid = Bt, one CTA per request.  scores f32 [Bt, Hkv, n] (pooled).
__global__ void __launch_bounds__(kThreads)
    ada_budgets_kernel(const float* __restrict__ scores, int hkv, int n, int window, int floor_k,
                       int rest_total, int32_t* __restrict__ budgets) {
  __shared__ SelectSmem sm;
  const int b = blockIdx.x;
  const float* s = scores + static_cast<int64_t>(b) * hkv * n;
  // phase 1: per-head floors (top floor_k by (score desc, token asc))
  for (int h = 0; h < hkv; ++h) {
    uint64_t tau = kNone;
    if (floor_k > 0) {
      const float* sh = s + static_cast<int64_t>(h) * n;
      tau = cta_select_kth(
          [&](int i, uint64_t& key) {
            key = compose(sh[i], static_cast<uint32_t>(i));
            return true;
          },
          n, static_cast<uint32_t>(floor_k), sm);
    }
    if (threadIdx.x == 0) sm.tau_head[h] = tau;
    __syncthreads();
  }
  auto in_floor = [&](int h, int t) -> bool {
    const uint64_t tau = sm.tau_head[h];
    return tau != kNone && compose(s[static_cast<int64_t>(h) * n + t], static_cast<uint32_t>(t)) >= tau;
  };
  // phase 2: global top rest_total over the non-floor elements
  const int total = hkv * n;
  uint64_t gtau = kNone;
  if (rest_total > 0) {
    gtau = cta_select_kth(
        [&](int i, uint64_t& key) {
          const int h = i / n, t = i - h * n;
          if (in_floor(h, t)) return false;
          key = compose(s[i], static_cast<uint32_t>(i));
          return true;
        },
        total, static_cast<uint32_t>(rest_total), sm);
  }
  // phase 3: per-head counts of globally chosen elements
  for (int h = 0; h < hkv; ++h) {
    uint32_t c = 0;
    if (gtau != kNone) {
      for (int t = threadIdx.x; t < n; t += blockDim.x) {
        const int i = h * n + t;
        if (!in_floor(h, t) && compose(s[i], static_cast<uint32_t>(i)) >= gtau) ++c;
      }
    }
    const uint32_t tot = block_sum(c, sm);
    if (threadIdx.x == 0) budgets[b * hkv + h] = window + floor_k + static_cast<int32_t>(tot);
  }
}

// ----------------------------------------------------------------- K2 ----
// grid = Bt * Hkv.  Writes offsets[bh] (exclusive prefix of budgets) and the
// selected tokens of head (b,h) ascending, then the window tokens n..n+w-1.
__global__ void __launch_bounds__(kThreads)
    topk_select_kernel(const float* __restrict__ scores, const int32_t* __restrict__ budgets,
                       int n, int window, int64_t* __restrict__ offsets,
                       int32_t* __restrict__ idx) {
  __shared__ SelectSmem sm;
  const int bh = blockIdx.x;
  // offset = sum of budgets before this head
  uint32_t part = 0;
  for (int j = threadIdx.x; j < bh; j += blockDim.x) part += static_cast<uint32_t>(budgets[j]);
  const int64_t off = block_sum(part, sm);
  if (threadIdx.x == 0) {
    offsets[bh] = off;
    if (bh == gridDim.x - 1) offsets[bh + 1] = off + budgets[bh];
  }
  const int k = budgets[bh] - window;
  const float* s = scores + static_cast<int64_t>(bh) * n;
  int32_t* out = idx + off;
  if (k > 0) {
    const uint64_t tau =
        k >= n ? 0ull
               : cta_select_kth(
                     [&](int i, uint64_t& key) {
                       key = compose(s[i], static_cast<uint32_t>(i));
                       return true;
                     },
                     n, static_cast<uint32_t>(k), sm);
    uint32_t written = 0;
    for (int base = 0; base < n; base += blockDim.x) {
      const int t = base + threadIdx.x;
      const bool take = t < n && compose(s[t], static_cast<uint32_t>(t)) >= tau;
      uint32_t before;
      const uint32_t tot = block_flag_scan(take, before, sm);
      if (take) out[written + before] = t;
      written += tot;
    }
  }
  for (int i = threadIdx.x; i < window; i += blockDim.x) out[max(k, 0) + i] = n + i;
}

// ------------------------------------------------ A18 + K2, one cluster ----
// One thread-block cluster per request, one CTA per KV head (cluster size =
// Hkv <= 8).  Each CTA stages its head's scores in shared memory when they
// fit; budgets, offsets (request b starts at b*Hkv*budget: every request
// keeps exactly Hkv*budget tokens) and the ascending index lists are written
// by the same launch.
constexpr int kStageLimit = 40 * 1024;  // scores staged in smem up to 160 KiB

// Ada split without materialising the floors: with N_h(tau) = #{t : gkey_h(t)
// >= tau}, the number of globally chosen (non-floor) elements of head h above
// tau is max(0, N_h(tau) - floor) (a head's floor is its own top-floor in the
// same order), so the global threshold is the largest tau with
// G(tau) = sum_h max(0, N_h(tau) - floor) >= R.  A cluster-wide MSB-first radix
// search finds it: per 8-bit digit every CTA (one head) builds its histogram,
// turns it into suffix counts S_h[d] = N_h(prefix.d...) and publishes them in
// shared memory; every CTA evaluates G[d] for all 256 digits from the
// peers' S arrays (DSMEM) and takes d* = max{d : G[d] >= R}.  Only heads that
// end below their floor (N_h(tau) < floor) need their own top-floor select.
__global__ void __launch_bounds__(kThreads)
    ada_select_kernel(const float* __restrict__ scores, int n, int window, int floor_k,
                      int rest_total, int budget, int32_t* __restrict__ budgets,
                      int64_t* __restrict__ offsets, int32_t* __restrict__ idx) {
  extern __shared__ __align__(16) uint8_t dyn[];
  __shared__ SelectSmem sm;
  __shared__ int32_t suffix[256];
  __shared__ int32_t s_budget;
  cg::cluster_group cluster = cg::this_cluster();
  const int hkv = static_cast<int>(cluster.num_blocks());
  const int h = static_cast<int>(cluster.block_rank());
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* src = scores + (static_cast<int64_t>(b) * hkv + h) * n;
  const bool staged = n <= kStageLimit;
  float* sv = reinterpret_cast<float*>(dyn);
  if (staged)
    for (int t = threadIdx.x; t < n; t += blockDim.x) sv[t] = src[t];
  __syncthreads();
  const float* s = staged ? sv : src;
  const uint32_t gbase = static_cast<uint32_t>(h) * n;

  // ---- cluster radix search for tau over the global keys of all heads
  uint64_t prefix = 0, mask = 0;
  int above = 0;          // this head's elements strictly above the current prefix range
  int n_at_tau = 0;       // N_h(tau) once found
  bool have_tau = rest_total > 0;
  if (have_tau) {
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += blockDim.x) sm.hist[i] = 0;
      __syncthreads();
      for (int base = 0; base < n; base += blockDim.x) {
        const int t = base + threadIdx.x;
        uint64_t key = t < n ? compose(s[t], gbase + t) : 0;
        const bool ok = t < n && (key & mask) == prefix;
        const uint32_t d = ok ? static_cast<uint32_t>(key >> shift) & 255u : 256u;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        if (ok && lane == __ffs(peers) - 1) atomicAdd(&sm.hist[d], __popc(peers));
      }
      __syncthreads();
      if (warp == 0) {  // suffix[d] = above + sum_{d' >= d} hist[d']
        uint32_t loc[8], run = 0;
#pragma unroll
        for (int j = 7; j >= 0; --j) {
          run += sm.hist[8 * lane + j];
          loc[j] = run;
        }
        uint32_t incl = run;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t v = __shfl_down_sync(0xffffffffu, incl, off);
          if (lane + off < 32) incl += v;
        }
        const uint32_t higher = incl - run;  // bins owned by higher lanes
#pragma unroll
        for (int j = 0; j < 8; ++j) suffix[8 * lane + j] = above + static_cast<int>(higher + loc[j]);
      }
      cluster.sync();  // every head's suffix counts are published
      bool ge = false;
      int gd = 0;
      if (threadIdx.x < 256) {
        for (int r = 0; r < hkv; ++r) {
          const int v = cluster.map_shared_rank(suffix, r)[threadIdx.x] - floor_k;
          gd += v > 0 ? v : 0;
        }
        ge = gd >= rest_total;
      }
      // G is non-increasing in d: d* = (#digits with G >= R) - 1
      const uint32_t cnt = block_sum(ge ? 1u : 0u, sm);
      const int dstar = static_cast<int>(cnt) - 1;
      if (threadIdx.x == dstar) {
        sm.digit = dstar;
        sm.above = gd == rest_total;  // exact: the whole bucket is taken
      }
      __syncthreads();
      const int d = static_cast<int>(sm.digit);
      const bool exact = sm.above != 0;
      n_at_tau = suffix[d];
      const int next_above = d < 255 ? suffix[d + 1] : above;
      prefix |= static_cast<uint64_t>(d) << shift;
      mask |= 255ull << shift;
      cluster.sync();  // peers are done reading `suffix` before it is rewritten
      if (exact) break;
      above = next_above;
    }
  }
  const uint64_t tau = prefix;
  const int c_h = have_tau ? (n_at_tau - floor_k > 0 ? n_at_tau - floor_k : 0) : 0;
  const bool below_floor = !have_tau || n_at_tau < floor_k;

  // heads that end below their floor keep exactly their own top-floor tokens
  uint64_t ltau = kNone;
  if (below_floor && floor_k > 0)
    ltau = cta_select_kth(
        [&](int i, uint64_t& key) {
          key = compose(s[i], static_cast<uint32_t>(i));
          return true;
        },
        n, static_cast<uint32_t>(floor_k), sm);
  auto chosen = [&](int t) -> bool {
    if (!below_floor) return compose(s[t], gbase + t) >= tau;
    return ltau != kNone && compose(s[t], static_cast<uint32_t>(t)) >= ltau;
  };

  // ---- budget, offsets within the request via DSMEM, ascending indices
  if (threadIdx.x == 0) s_budget = window + floor_k + c_h;
  cluster.sync();
  int64_t off = static_cast<int64_t>(b) * hkv * budget;
  for (int r = 0; r < h; ++r) off += *cluster.map_shared_rank(&s_budget, r);
  const int bh = b * hkv + h;
  if (threadIdx.x == 0) {
    budgets[bh] = s_budget;
    offsets[bh] = off;
    if (b == static_cast<int>(gridDim.y) - 1 && h == hkv - 1) offsets[bh + 1] = off + s_budget;
  }
  int32_t* out = idx + off;
  uint32_t written = 0;
  for (int base = 0; base < n; base += blockDim.x) {
    const int t = base + threadIdx.x;
    const bool take = t < n && chosen(t);
    uint32_t before;
    const uint32_t got = block_flag_scan(take, before, sm);
    if (take) out[written + before] = t;
    written += got;
  }
  for (int i = threadIdx.x; i < window; i += blockDim.x) out[s_budget - window + i] = n + i;
  cluster.sync();  // keep this CTA's shared memory alive until every peer is done reading it
}

}  // namespace
}  // namespace fkv

extern "C" int fkv_ada_budgets(const float* scores, int32_t batch, int32_t hkv, int32_t n,
                               int32_t budget, int32_t window, int32_t floor_k, int32_t* budgets,
                               void* stream) {
  using namespace fkv;
  if (!scores || !budgets) return set_error(FKV_ERR_INVALID, "fkv_ada_budgets: null pointer");
  if (batch < 0 || hkv < 1 || hkv > 64 || n < 0 || window < 0 || floor_k < 0)
    return set_error(FKV_ERR_INVALID, "fkv_ada_budgets: bad sizes");
  const int sel = budget - window;
  if (sel < 0 || sel > n || floor_k > sel)
    return set_error(FKV_ERR_INVALID, "fkv_ada_budgets: need 0 <= floor <= budget-window <= n");
  if (static_cast<int64_t>(hkv) * n >= 0x7fffffffLL)
    return set_error(FKV_ERR_INVALID, "fkv_ada_budgets: Hkv * n too large");
  if (batch == 0) return FKV_OK;
  const int rest = hkv * sel - hkv * floor_k;
  ada_budgets_kernel<<<batch, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      scores, hkv, n, window, floor_k, rest, budgets);
  return cuda_check(cudaGetLastError(), "ada_budgets launch");
}

extern "C" int fkv_topk_select(const float* scores, const int32_t* budgets, int32_t batch,
                               int32_t hkv, int32_t n, int32_t window, int64_t* offsets,
                               int32_t* idx, void* stream) {
  using namespace fkv;
  if (!scores || !budgets || !offsets || !idx)
    return set_error(FKV_ERR_INVALID, "fkv_topk_select: null pointer");
  if (batch < 0 || hkv < 1 || n < 0 || window < 0)
    return set_error(FKV_ERR_INVALID, "fkv_topk_select: bad sizes");
  if (batch == 0) return FKV_OK;
  topk_select_kernel<<<batch * hkv, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      scores, budgets, n, window, offsets, idx);
  return cuda_check(cudaGetLastError(), "topk_select launch");
}

extern "C" int fkv_ada_select(const float* scores, int32_t batch, int32_t hkv, int32_t n,
                              int32_t budget, int32_t window, int32_t floor_k, int32_t* budgets,
                              int64_t* offsets, int32_t* idx, void* stream) {
  using namespace fkv;
  if (!scores || !budgets || !offsets || !idx)
    return set_error(FKV_ERR_INVALID, "fkv_ada_select: null pointer");
  if (batch < 0 || hkv < 1 || hkv > 8 || n < 0 || window < 0 || floor_k < 0)
    return set_error(FKV_ERR_INVALID, "fkv_ada_select: bad sizes (Hkv must be 1..8)");
  const int sel = budget - window;
  if (sel < 0 || sel > n || floor_k > sel)
    return set_error(FKV_ERR_INVALID, "fkv_ada_select: need 0 <= floor <= budget-window <= n");
  if (static_cast<int64_t>(hkv) * n >= 0x7fffffffLL)
    return set_error(FKV_ERR_INVALID, "fkv_ada_select: Hkv * n too large");
  if (batch == 0) return FKV_OK;
  const int rest = hkv * sel - hkv * floor_k;
  const size_t smem = n <= kStageLimit ? static_cast<size_t>(n) * 4 : 16;
  static size_t configured = 0;
  if (smem > configured) {
    if (int rc = cuda_check(cudaFuncSetAttribute(ada_select_kernel,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem)),
                            "ada_select smem attribute"))
      return rc;
    configured = smem;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(hkv, batch, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = hkv;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cuda_check(cudaLaunchKernelEx(&cfg, ada_select_kernel, scores, n, window, floor_k, rest,
                                       budget, budgets, offsets, idx),
                    "ada_select launch");
}

// A18 Ada cross-head budget split + K2 per-head top-k selection.
//
// No reference implementation exists (the paper used KVPress
// AdaKV).  Definitions and tie rules are fixed in DESIGN.md
// "Algorithm definitions" and restated in oracle/kv.py:
//   per-head order  (score desc, token asc)
//   global order    (score desc, head asc, token asc)
// One grid-wide kernel serves the three entry points (fkv_ada_select,
// fkv_ada_budgets, fkv_topk_select): a radix search over the 32-bit
// orderable score finds the threshold score, and the keys tied at it are
// taken in the tie order above from per-range tie counts -- so results are
// exact functions of the fp32 score tensor, bit-exact against the oracle fed
// the same scores, without passes over the index bits.
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"
#include "gsel.cuh"

namespace fkv {
namespace {

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
struct KernelCx {  // the standalone launch: every thread of every CTA
  int cta, ncta;
  __device__ void sync() const { __syncthreads(); }
  __device__ int count(bool pred) const { return __syncthreads_count(pred); }
  __device__ void grid(unsigned* bar, unsigned& k) const {
    grid_sync_n(bar, k, ncta, [] { __syncthreads(); });
  }
};

__global__ void __launch_bounds__(kGThreads) grid_select_kernel(const GSelParams p) {
  __shared__ GSelSmem sm;
  extern __shared__ uint32_t skeys[];  // p.cache: orderable keys of [k0, k1)
  gsel_body(p, sm, skeys, KernelCx{static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x)});
}

int gsel_ctas() {
  static std::atomic<int> ctas[kMaxDevices];
  return per_device(ctas, [](int dev) {
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, grid_select_kernel, kGThreads, 0);
    occ = occ < 1 ? 1 : (occ > 2 ? 2 : occ);
    return sm_count(dev) * occ;
  });
}

// CTAs of a launch over `bh` heads of n keys.
int gsel_grid(int bh, int n) {
  const int64_t total = static_cast<int64_t>(bh) * n;
  static const int min_keys = [] {
    const char* e = getenv("FKV_GSEL_MIN_KEYS");  // tuning experiments
    return e ? atoi(e) : kGMinKeys;
  }();
  int64_t want = (total + min_keys - 1) / min_keys;
  // short heads: enough CTAs that no key range spans more than kGMaxPieces
  // heads (ranges of <= (kGMaxPieces - 2) * n keys); gsel_reqs_per_launch
  // keeps this within the co-resident grid
  const int64_t span = (bh + kGMaxPieces - 3) / (kGMaxPieces - 2);
  want = want > span ? want : span;
  const int ctas = gsel_ctas();
  return want < 1 ? 1 : (want > ctas ? ctas : static_cast<int>(want));
}

// Requests per launch: a CTA's key range spans at most kGMaxPieces heads.
int gsel_reqs_per_launch(int hkv) {
  const int r = (kGMaxPieces - 2) * gsel_ctas() / hkv;
  return r < 1 ? 1 : r;
}

}  // namespace
}  // namespace fkv

namespace fkv {
namespace {

// n == 0: nothing to rank -- every head keeps its window only.
__global__ void window_only_kernel(int bh_total, int window, const int32_t* head_k, int32_t* budgets,
                                   int64_t* offsets, int32_t* idx) {
  int64_t off = 0;
  for (int bh = 0; bh < bh_total; ++bh) {
    const int bud = head_k ? head_k[bh] : window;
    if (threadIdx.x == 0) {
      if (!head_k && budgets) budgets[bh] = bud;
      if (offsets) offsets[bh] = off;
    }
    if (idx)
      for (int i = threadIdx.x; i < window; i += blockDim.x) idx[off + i] = i;
    off += bud;
  }
  if (threadIdx.x == 0 && offsets) offsets[bh_total] = off;
}

// The three entry points: Ada split + selection (head_k null, select 1),
// Ada budgets only (select 0), per-head top-k of given budgets (head_k).
int grid_select(const float* scores, int batch, int hkv, int n, int budget, int window, int floor_k,
                const int32_t* head_k, int select, int32_t* budgets, int64_t* offsets, int32_t* idx,
                void* workspace, cudaStream_t st) {
  if (batch == 0) return FKV_OK;
  if (n == 0) {
    window_only_kernel<<<1, 32, 0, st>>>(batch * hkv, window, head_k, budgets, select ? offsets : nullptr,
                                         select ? idx : nullptr);
    return cuda_check(cudaGetLastError(), "window-only launch");
  }
  const int per = gsel_reqs_per_launch(hkv);
  const int sel = budget - window;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  for (int r0 = 0; r0 < batch; r0 += per) {
    const int reqs = batch - r0 < per ? batch - r0 : per;
    const int bh = reqs * hkv;
    GSelParams p{};
    p.scores = scores + static_cast<int64_t>(r0) * hkv * n;
    p.hkv = hkv;
    p.n = n;
    p.window = window;
    p.f = head_k ? 0 : floor_k;
    p.R = head_k ? 0 : hkv * sel - hkv * floor_k;
    p.budget = budget;
    p.head_k = head_k ? head_k + static_cast<int64_t>(r0) * hkv : nullptr;
    p.budgets_all = head_k;
    p.select = select;
    p.req0 = r0;
    p.bh_total = batch * hkv;
    p.total = static_cast<int64_t>(bh) * n;
    p.bar = reinterpret_cast<unsigned*>(ws);
    p.hist = reinterpret_cast<uint32_t*>(ws + 256);
    p.counts = reinterpret_cast<int2*>(ws + 256 + static_cast<int64_t>(kGBufs) * bh * 512 * 4);
    p.budgets = head_k ? nullptr : budgets + static_cast<int64_t>(r0) * hkv;
    p.offsets = offsets ? offsets + static_cast<int64_t>(r0) * hkv : nullptr;
    p.idx = idx;
    // barrier counter + the histogram buffers of passes 0 and 1
    if (int rc = cuda_check(cudaMemsetAsync(ws, 0, 256 + static_cast<size_t>(2) * bh * 512 * 4, st),
                            "select workspace reset"))
      return rc;
    const int grid = gsel_grid(bh, n);
    const int64_t span_keys = (p.total + grid - 1) / grid + 1;
    p.cache = span_keys * 4 <= kGCacheBytes;
    static std::atomic<int> ready[kMaxDevices];  // smem attribute set on this device
    const int rc0 = per_device(ready, [](int) {
      const int e = cuda_check(cudaFuncSetAttribute(grid_select_kernel,
                                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    kGCacheBytes),
                               "grid select smem attribute");
      return e < 0 ? e : 1;
    });
    if (rc0 < 0) return rc0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(kGThreads, 1, 1);
    cfg.dynamicSmemBytes = p.cache ? static_cast<size_t>(span_keys) * 4 : 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (int rc = cuda_check(cudaLaunchKernelEx(&cfg, grid_select_kernel, p), "grid select launch"))
      return rc;
  }
  return FKV_OK;
}

}  // namespace
}  // namespace fkv

extern "C" int fkv__select_stamps(unsigned long long* host) {
  return fkv::cuda_check(cudaMemcpyFromSymbol(host, fkv::g_gstamps, sizeof(unsigned long long) * 32),
                         "select stamps");
}

extern "C" int64_t fkv_ada_select_workspace_bytes(int32_t batch, int32_t hkv, int32_t n) {
  using namespace fkv;
  if (batch < 1 || hkv < 1) return 256;
  const int reqs = batch < gsel_reqs_per_launch(hkv) ? batch : gsel_reqs_per_launch(hkv);
  const int64_t hist = static_cast<int64_t>(kGBufs) * reqs * hkv * 512 * 4;
  return 256 + hist + static_cast<int64_t>(gsel_ctas()) * 8;
}

namespace {
int check_sizes(const char* fn, const float* scores, int batch, int hkv, int n, int window, void* workspace) {
  using namespace fkv;
  if ((!scores && n > 0) || !workspace) return set_error(FKV_ERR_INVALID, std::string(fn) + ": null pointer");
  if (batch < 0 || hkv < 1 || hkv > kGMaxHeads || n < 0 || window < 0)
    return set_error(FKV_ERR_INVALID, std::string(fn) + ": bad sizes (Hkv must be 1..16)");
  if (static_cast<int64_t>(hkv) * n >= 0x7fffffffLL)
    return set_error(FKV_ERR_INVALID, std::string(fn) + ": Hkv * n too large");
  return FKV_OK;
}
int check_ada(const char* fn, int n, int budget, int window, int floor_k) {
  using namespace fkv;
  const int sel = budget - window;
  if (floor_k < 0 || sel < 0 || sel > n || floor_k > sel)
    return set_error(FKV_ERR_INVALID, std::string(fn) + ": need 0 <= floor <= budget-window <= n");
  return FKV_OK;
}
}  // namespace

extern "C" int fkv_ada_budgets(const float* scores, int32_t batch, int32_t hkv, int32_t n,
                               int32_t budget, int32_t window, int32_t floor_k, int32_t* budgets,
                               void* workspace, void* stream) {
  using namespace fkv;
  if (!budgets) return set_error(FKV_ERR_INVALID, "fkv_ada_budgets: null pointer");
  if (int rc = check_sizes("fkv_ada_budgets", scores, batch, hkv, n, window, workspace)) return rc;
  if (int rc = check_ada("fkv_ada_budgets", n, budget, window, floor_k)) return rc;
  return grid_select(scores, batch, hkv, n, budget, window, floor_k, nullptr, 0, budgets, nullptr, nullptr,
                     workspace, static_cast<cudaStream_t>(stream));
}

extern "C" int fkv_topk_select(const float* scores, const int32_t* budgets, int32_t batch,
                               int32_t hkv, int32_t n, int32_t window, int64_t* offsets,
                               int32_t* idx, void* workspace, void* stream) {
  using namespace fkv;
  if (!budgets || !offsets || !idx) return set_error(FKV_ERR_INVALID, "fkv_topk_select: null pointer");
  if (int rc = check_sizes("fkv_topk_select", scores, batch, hkv, n, window, workspace)) return rc;
  return grid_select(scores, batch, hkv, n, 0, window, 0, budgets, 1, nullptr, offsets, idx, workspace,
                     static_cast<cudaStream_t>(stream));
}

extern "C" int fkv_ada_select(const float* scores, int32_t batch, int32_t hkv, int32_t n,
                              int32_t budget, int32_t window, int32_t floor_k, int32_t* budgets,
                              int64_t* offsets, int32_t* idx, void* workspace, void* stream) {
  using namespace fkv;
  if (!budgets || !offsets || !idx) return set_error(FKV_ERR_INVALID, "fkv_ada_select: null pointer");
  if (int rc = check_sizes("fkv_ada_select", scores, batch, hkv, n, window, workspace)) return rc;
  if (int rc = check_ada("fkv_ada_select", n, budget, window, floor_k)) return rc;
  return grid_select(scores, batch, hkv, n, budget, window, floor_k, nullptr, 1, budgets, offsets, idx,
                     workspace, static_cast<cudaStream_t>(stream));
}

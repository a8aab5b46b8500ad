// AHA placement planner (paper Alg. 1 + Alg. 2) as native host code.
//
// This is the B200 build's replacement for the reference's search-kernel
// plugin (pkg/src/headbalance/_kernel/__init__.py:49-57): the B&B is a
// sequential, branch-heavy CPU algorithm, so it stays on the host, in C++,
// behind the C ABI declared in include/fairkv.h.
//
// Parity contract: results are bit-identical to the reference's
// solve_equal_split / solve_free_split (pkg/src/headbalance/_kernel/reference.py:80-235,
// 238-340) *including node counts under truncation*.  That pins every float
// operation and its order: prefix sums accumulate left to right, guards are
// 1e-12*(1+|x|), bounds are evaluated in the reference's order, and this file
// is compiled with -ffp-contract=off (no FMA contraction; see build.py).
//
// Unlike the reference (which exposes only the per-scheme search), this file
// also runs the whole per-layer scheme loop (allocate.select_best,
// reference allocate.py:236-277) and the per-model layer loop with a thread
// pool (reference allocate.py:353-389 uses a process pool), so free-split
// TP=8 planning over 80 layers drops from minutes of Python to well under a
// second.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "fairkv.h"

namespace fkv {

// ---------------------------------------------------------------- errors --
static thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
const char* last_error() { return g_last_error.c_str(); }

namespace {

constexpr double kGuard = 1e-12;
constexpr double kInf = std::numeric_limits<double>::infinity();

inline double pad(double x) { return kGuard * (1.0 + std::fabs(x)); }

// Relabel group ids by first appearance -> restricted-growth string.
void to_rgs(const std::vector<int>& raw, int tp, std::vector<int>& rgs) {
  std::vector<int> relabel(tp, -1);
  int next = 0;
  rgs.resize(raw.size());
  for (size_t i = 0; i < raw.size(); ++i) {
    int g = raw[i];
    if (relabel[g] < 0) relabel[g] = next++;
    rgs[i] = relabel[g];
  }
}

struct Incumbent {
  bool found = false;
  double spread = 0.0;
  std::vector<int> rgs;
};

// Lowest-loaded-first greedy seed (reference.py:47-77).  Returns false when
// some copy has no admissible group.
bool greedy_seed(const double* w, const int* heads, int m, int tp, int k, int n_heads,
                 Incumbent& out) {
  std::vector<double> sums(tp, 0.0);
  std::vector<int> counts(tp, 0);
  // membership bitmap per group: head ids are < n_heads
  std::vector<uint8_t> member(static_cast<size_t>(tp) * n_heads, 0);
  std::vector<int> raw(m);
  for (int t = 0; t < m; ++t) {
    int pick = -1;
    for (int j = 0; j < tp; ++j) {
      if (counts[j] >= k || member[static_cast<size_t>(j) * n_heads + heads[t]]) continue;
      if (pick < 0 || sums[j] < sums[pick]) pick = j;
    }
    if (pick < 0) return false;
    sums[pick] += w[t];
    counts[pick] += 1;
    member[static_cast<size_t>(pick) * n_heads + heads[t]] = 1;
    raw[t] = pick;
  }
  double hi = sums[0], lo = sums[0];
  for (int j = 1; j < tp; ++j) {  // python max()/min() semantics on finite values
    hi = std::max(hi, sums[j]);
    lo = std::min(lo, sums[j]);
  }
  out.found = true;
  out.spread = hi - lo;
  to_rgs(raw, tp, out.rgs);
  return true;
}

// ------------------------------------------------------ equal-split B&B --
class EqualSplitSearch {
 public:
  EqualSplitSearch(const double* w, const int* heads, int m, int tp, double cutoff,
                   int64_t budget, double seed)
      : w_(w), heads_(heads), m_(m), tp_(tp), k_(m / tp), budget_(budget), seed_(seed),
        best_delta_(cutoff) {
    prefix_.assign(m + 1, 0.0);
    double acc = 0.0;
    for (int i = 0; i < m; ++i) {
      acc += w[i];
      prefix_[i + 1] = acc;
    }
    const double avg = prefix_[m] / tp;
    avg_up_ = avg + pad(avg);
    avg_dn_ = avg - pad(avg);
    int nh = 0;
    for (int i = 0; i < m; ++i) nh = std::max(nh, heads[i] + 1);
    same_after_.assign(m, 0);
    for (int t = m - 2; t >= 0; --t)
      if (heads[t + 1] == heads[t]) same_after_[t] = same_after_[t + 1] + 1;
    sums_.assign(tp, 0.0);
    counts_.assign(tp, 0);
    last_group_.assign(nh, -1);
    assign_.assign(m, 0);
  }

  void run() { dfs(0, 0); }

  int64_t nodes() const { return nodes_; }
  bool found() const { return found_; }
  double best_delta() const { return best_delta_; }
  const std::vector<int>& best_assign() const { return best_assign_; }

 private:
  // false <=> node budget exhausted (unwinds the whole search)
  bool dfs(int t, int opened) {
    if (nodes_ >= budget_) return false;
    ++nodes_;
    if (t == m_) {
      double hi = sums_[0], lo = sums_[0];
      for (int j = 1; j < tp_; ++j) {
        const double s = sums_[j];
        if (s > hi) hi = s;
        else if (s < lo) lo = s;
      }
      const double delta = hi - lo;
      if (delta < best_delta_ && delta <= seed_) {
        best_delta_ = delta;
        best_assign_ = assign_;
        found_ = true;
      }
      return true;
    }

    // completion lower bound: some group ends >= lb_max, some group <= ub_min
    double ub_min = avg_up_, lb_max = avg_dn_;
    for (int j = 0; j < tp_; ++j) {
      const bool open = j < opened;
      const double s = open ? sums_[j] : 0.0;
      const int need = open ? k_ - counts_[j] : k_;
      double hi = s + (prefix_[t + need] - prefix_[t]);
      hi += pad(hi);
      if (hi < ub_min) ub_min = hi;
      double lo = s + (prefix_[m_] - prefix_[m_ - need]);
      lo -= pad(lo);
      if (lo > lb_max) lb_max = lo;
      if (!open) break;  // all unopened groups look alike
    }
    const double lb = lb_max - ub_min;
    if (lb >= best_delta_ || lb > seed_) return true;

    const double wt = w_[t];
    const int h = heads_[t];
    const int trailing = same_after_[t];
    const int start = last_group_[h] + 1;
    const int limit = opened < tp_ ? opened : tp_ - 1;
    for (int j = start; j <= limit; ++j) {
      int cnt;
      double base;
      if (j < opened) {
        cnt = counts_[j];
        if (cnt >= k_) continue;
        base = sums_[j];
      } else {
        cnt = 0;
        base = 0.0;
      }
      if (trailing) {  // later copies of h need distinct, higher, non-full groups
        int avail = 0;
        for (int j2 = j + 1; j2 < tp_; ++j2)
          if (j2 >= opened || counts_[j2] < k_) ++avail;
        if (trailing > avail) continue;
      }
      const int fill = k_ - cnt - 1;
      double forced = base + wt + (prefix_[m_] - prefix_[m_ - fill]);
      forced -= pad(forced);
      const double branch_lb = forced - ub_min;
      if (branch_lb >= best_delta_ || branch_lb > seed_) continue;

      sums_[j] = base + wt;
      counts_[j] = cnt + 1;
      last_group_[h] = j;
      assign_[t] = j;
      const bool alive = dfs(t + 1, j == opened ? opened + 1 : opened);
      sums_[j] = base;
      counts_[j] = cnt;
      last_group_[h] = start - 1;
      if (!alive) return false;
    }
    return true;
  }

  const double* w_;
  const int* heads_;
  int m_, tp_, k_;
  int64_t budget_;
  double seed_;
  double best_delta_;
  double avg_up_ = 0, avg_dn_ = 0;
  bool found_ = false;
  int64_t nodes_ = 0;
  std::vector<double> prefix_, sums_;
  std::vector<int> same_after_, counts_, last_group_, assign_, best_assign_;
};

// ------------------------------------------------------- free-split B&B --
class FreeSplitSearch {
 public:
  FreeSplitSearch(const double* w, const int* heads, int m, int tp, double cutoff,
                  int64_t budget, double seed)
      : w_(w), heads_(heads), m_(m), tp_(tp), budget_(budget), seed_(seed), best_delta_(cutoff) {
    double total = 0.0;
    for (int i = 0; i < m; ++i) total += w[i];
    const double avg = total / tp;
    avg_up_ = avg + pad(avg);
    avg_dn_ = avg - pad(avg);
    int nh = 0;
    for (int i = 0; i < m; ++i) nh = std::max(nh, heads[i] + 1);
    same_after_.assign(m, 0);
    for (int t = m - 2; t >= 0; --t)
      if (heads[t + 1] == heads[t]) same_after_[t] = same_after_[t + 1] + 1;
    sums_.assign(tp, 0.0);
    last_group_.assign(nh, -1);
    assign_.assign(m, 0);
  }

  void run() { dfs(0, 0); }
  int64_t nodes() const { return nodes_; }
  bool found() const { return found_; }
  double best_delta() const { return best_delta_; }
  const std::vector<int>& best_assign() const { return best_assign_; }

 private:
  bool dfs(int t, int opened) {
    if (nodes_ >= budget_) return false;
    ++nodes_;
    if (t == m_) {
      if (opened < tp_) return true;
      double hi = sums_[0], lo = sums_[0];
      for (int j = 1; j < tp_; ++j) {
        const double s = sums_[j];
        if (s > hi) hi = s;
        else if (s < lo) lo = s;
      }
      const double delta = hi - lo;
      if (delta < best_delta_ && delta <= seed_) {
        best_delta_ = delta;
        best_assign_ = assign_;
        found_ = true;
      }
      return true;
    }
    if (m_ - t < tp_ - opened) return true;
    double cur_max = 0.0;
    for (int j = 0; j < opened; ++j)
      if (sums_[j] > cur_max) cur_max = sums_[j];
    const double lb_max = cur_max > avg_dn_ ? cur_max : avg_dn_;
    const double lb = lb_max - avg_up_;
    if (lb >= best_delta_ || lb > seed_) return true;

    const double wt = w_[t];
    const int h = heads_[t];
    const int trailing = same_after_[t];
    const int start = last_group_[h] + 1;
    const int limit = opened < tp_ ? opened : tp_ - 1;
    for (int j = start; j <= limit; ++j) {
      if (trailing > tp_ - 1 - j) continue;
      const int opened_next = j == opened ? opened + 1 : opened;
      if (m_ - t - 1 < tp_ - opened_next) continue;
      const double new_sum = sums_[j] + wt;
      const double branch_lb = new_sum - pad(new_sum) - avg_up_;
      if (branch_lb >= best_delta_ || branch_lb > seed_) continue;
      const double old = sums_[j];
      sums_[j] = new_sum;
      last_group_[h] = j;
      assign_[t] = j;
      const bool alive = dfs(t + 1, opened_next);
      sums_[j] = old;
      last_group_[h] = start - 1;
      if (!alive) return false;
    }
    return true;
  }

  const double* w_;
  const int* heads_;
  int m_, tp_;
  int64_t budget_;
  double seed_;
  double best_delta_;
  double avg_up_ = 0, avg_dn_ = 0;
  bool found_ = false;
  int64_t nodes_ = 0;
  std::vector<double> sums_;
  std::vector<int> same_after_, last_group_, assign_, best_assign_;
};

int check_copies(const double* w, const int32_t* heads, int m, int tp) {
  if (m < 0) return set_error(FKV_ERR_INVALID, "negative copy count");
  if (tp < 1) return set_error(FKV_ERR_INVALID, "tp must be >= 1");
  if (m > 0 && (!w || !heads)) return set_error(FKV_ERR_INVALID, "null weights/heads");
  for (int i = 0; i < m; ++i)
    if (heads[i] < 0) return set_error(FKV_ERR_INVALID, "negative head id");
  return 0;
}

}  // namespace

// Equal split with the reference's precedence on equal spreads:
// in-order B&B find, then hint, then greedy -- each only if strictly better.
int solve_equal(const double* w, const int32_t* heads, int m, int tp, double cutoff,
                int64_t node_budget, const double* hint_spread, const int32_t* hint_rgs,
                double* out_spread, int32_t* out_rgs, int64_t* out_nodes) {
  if (int rc = check_copies(w, heads, m, tp)) return rc;
  if (m % tp != 0) return set_error(FKV_ERR_INVALID, "copy count not divisible by tp");
  const int k = m / tp;
  std::vector<int> hv(heads, heads + m);
  int nh = 0;
  for (int i = 0; i < m; ++i) nh = std::max(nh, hv[i] + 1);

  Incumbent greedy;
  const bool have_greedy = greedy_seed(w, hv.data(), m, tp, k, nh, greedy);
  double seed = kInf;
  if (have_greedy && greedy.spread < seed) seed = greedy.spread;
  if (hint_spread && *hint_spread < seed) seed = *hint_spread;

  EqualSplitSearch s(w, hv.data(), m, tp, cutoff, node_budget, seed);
  s.run();

  bool have = false;
  double spread = 0.0;
  const int* src = nullptr;
  std::vector<int> tmp;
  if (s.found()) {
    have = true;
    spread = s.best_delta();
    src = s.best_assign().data();
  }
  if (hint_spread && *hint_spread < cutoff && (!have || *hint_spread < spread)) {
    have = true;
    spread = *hint_spread;
    tmp.assign(hint_rgs, hint_rgs + m);
    src = tmp.data();
  }
  if (have_greedy && greedy.spread < cutoff && (!have || greedy.spread < spread)) {
    have = true;
    spread = greedy.spread;
    src = greedy.rgs.data();
  }
  *out_nodes = s.nodes();
  if (!have) return 0;
  *out_spread = spread;
  for (int i = 0; i < m; ++i) out_rgs[i] = src[i];
  return 1;
}

int solve_free(const double* w, const int32_t* heads, int m, int tp, double cutoff,
               int64_t node_budget, const double* hint_spread, const int32_t* hint_rgs,
               double* out_spread, int32_t* out_rgs, int64_t* out_nodes) {
  if (int rc = check_copies(w, heads, m, tp)) return rc;
  *out_nodes = 0;
  if (m < tp) return 0;
  std::vector<int> hv(heads, heads + m);
  const double seed = hint_spread ? *hint_spread : kInf;
  FreeSplitSearch s(w, hv.data(), m, tp, cutoff, node_budget, seed);
  s.run();
  bool have = false;
  double spread = 0.0;
  const int* src = nullptr;
  std::vector<int> tmp;
  if (s.found()) {
    have = true;
    spread = s.best_delta();
    src = s.best_assign().data();
  }
  if (hint_spread && *hint_spread < cutoff && (!have || *hint_spread < spread)) {
    have = true;
    spread = *hint_spread;
    tmp.assign(hint_rgs, hint_rgs + m);
    src = tmp.data();
  }
  *out_nodes = s.nodes();
  if (!have) return 0;
  *out_spread = spread;
  for (int i = 0; i < m; ++i) out_rgs[i] = src[i];
  return 1;
}

// ------------------------------------------------- per-layer scheme loop --
namespace {

struct Scheme {
  std::vector<int> r;
  int total;
};

// Lexicographic odometer enumeration (reference schemes.py:64-96), then the
// planner's visit order: (total copies, replica vector) ascending
// (reference allocate.py:186-197).
int enumerate_ordered(int n, int ch_budget, int r_max, bool divisible, int tp, int64_t cap,
                      std::vector<Scheme>& out) {
  std::vector<int> vec(n, 1);
  int spent = 0;
  for (;;) {
    if (!divisible || (n + spent) % tp == 0) {
      if (static_cast<int64_t>(out.size()) >= cap) {
        char buf[160];
        std::snprintf(buf, sizeof buf, "more than %lld schemes for n=%d, ch_budget=%d, r_max=%d",
                      static_cast<long long>(cap), n, ch_budget, r_max);
        return set_error(FKV_ERR_SEARCH_SPACE, buf);
      }
      out.push_back({vec, n + spent});
    }
    int pos = n - 1;
    for (; pos >= 0; --pos) {
      if (vec[pos] < r_max && spent + 1 <= ch_budget) {
        ++vec[pos];
        ++spent;
        break;
      }
      spent -= vec[pos] - 1;
      vec[pos] = 1;
    }
    if (pos < 0) break;
  }
  std::stable_sort(out.begin(), out.end(), [](const Scheme& a, const Scheme& b) {
    if (a.total != b.total) return a.total < b.total;
    return a.r < b.r;
  });
  return 0;
}

struct LayerResult {
  double delta = 0.0;
  std::vector<int> replicas, heads_c, rgs;
};

int select_layer(const double* lw, int n, int tp, int ch_budget, int r_max, bool equal_split,
                 int64_t max_schemes, int64_t node_budget, LayerResult& res) {
  if (n < 1) return set_error(FKV_ERR_VALIDATION, "layer has no heads");
  if (tp < 1) return set_error(FKV_ERR_VALIDATION, "tp must be >= 1");
  std::vector<Scheme> schemes;
  if (int rc = enumerate_ordered(n, ch_budget, r_max, equal_split, tp, max_schemes, schemes))
    return rc;
  bool have = false;
  std::vector<double> wc;
  std::vector<int> hc;
  std::vector<int32_t> rgs;
  std::vector<std::pair<double, int>> copies;
  for (const Scheme& sc : schemes) {
    if (*std::max_element(sc.r.begin(), sc.r.end()) > tp) continue;
    // canonical copies: heaviest adjusted weight first, ties by head id
    // (reference allocate.py:85-98)
    copies.clear();
    for (int h = 0; h < n; ++h) {
      const double adj = lw[h] / sc.r[h];
      for (int c = 0; c < sc.r[h]; ++c) copies.emplace_back(adj, h);
    }
    std::stable_sort(copies.begin(), copies.end(), [](const auto& a, const auto& b) {
      if (a.first != b.first) return a.first > b.first;
      return a.second < b.second;
    });
    const int m = static_cast<int>(copies.size());
    wc.resize(m);
    hc.resize(m);
    for (int i = 0; i < m; ++i) {
      wc[i] = copies[i].first;
      hc[i] = copies[i].second;
    }
    // SHA hint only for the replication-free scheme (reference allocate.py:214-233,264-265)
    double hint_spread = 0.0;
    std::vector<int32_t> hint_rgs;
    const bool use_hint = equal_split && sc.total == n && n % tp == 0;
    if (use_hint) {
      const int kh = n / tp;
      std::vector<int> raw(m), r2;
      for (int i = 0; i < m; ++i) raw[i] = hc[i] / kh;
      to_rgs(raw, tp, r2);
      hint_rgs.assign(r2.begin(), r2.end());
      // heaviest-first fold per group == index order, copies are sorted desc
      std::vector<double> sums(tp, 0.0);
      std::vector<std::vector<double>> vals(tp);
      for (int i = 0; i < m; ++i) vals[r2[i]].push_back(wc[i]);
      for (int g = 0; g < tp; ++g) {
        std::stable_sort(vals[g].begin(), vals[g].end(), std::greater<double>());
        double acc = 0.0;
        for (double v : vals[g]) acc += v;
        sums[g] = acc;
      }
      hint_spread = *std::max_element(sums.begin(), sums.end()) -
                    *std::min_element(sums.begin(), sums.end());
    }
    const double cutoff = have ? res.delta : kInf;
    double spread = 0.0;
    int64_t nodes = 0;
    rgs.assign(m, 0);
    int rc = equal_split
                 ? solve_equal(wc.data(), hc.data(), m, tp, cutoff, node_budget,
                               use_hint ? &hint_spread : nullptr,
                               use_hint ? hint_rgs.data() : nullptr, &spread, rgs.data(), &nodes)
                 : solve_free(wc.data(), hc.data(), m, tp, cutoff, node_budget, nullptr, nullptr,
                              &spread, rgs.data(), &nodes);
    if (rc < 0) return rc;
    if (rc == 1) {
      have = true;
      res.delta = spread;
      res.replicas = sc.r;
      res.heads_c = hc;
      res.rgs.assign(rgs.begin(), rgs.end());
    }
  }
  if (!have) {
    char buf[200];
    std::snprintf(buf, sizeof buf,
                  "no feasible assignment of %d heads to %d GPUs (ch_budget=%d, r_max=%d)", n, tp,
                  ch_budget, r_max);
    return set_error(FKV_ERR_INFEASIBLE, buf);
  }
  return 0;
}

}  // namespace

int select_best(const double* lw, int n, int tp, int ch_budget, int r_max, int equal_split,
                int64_t max_schemes, int64_t node_budget, int32_t* out_replicas,
                int32_t* out_heads_c, int32_t* out_rgs, int32_t* out_m, double* out_delta) {
  if (!lw || !out_replicas || !out_heads_c || !out_rgs || !out_m || !out_delta)
    return set_error(FKV_ERR_INVALID, "null pointer argument");
  LayerResult r;
  if (int rc = select_layer(lw, n, tp, ch_budget, r_max, equal_split != 0, max_schemes,
                            node_budget, r))
    return rc;
  const int m = static_cast<int>(r.heads_c.size());
  *out_m = m;
  *out_delta = r.delta;
  for (int h = 0; h < n; ++h) out_replicas[h] = r.replicas[h];
  for (int i = 0; i < m; ++i) {
    out_heads_c[i] = r.heads_c[i];
    out_rgs[i] = r.rgs[i];
  }
  return 0;
}

int optimize_plan(const double* weights, int num_layers, int n, int tp, int ch_budget, int r_max,
                  int equal_split, int64_t max_schemes, int64_t node_budget, int workers,
                  int32_t* out_replicas, int32_t* out_heads_c, int32_t* out_rgs, int32_t* out_m,
                  double* out_delta) {
  if (num_layers < 1) return set_error(FKV_ERR_VALIDATION, "plan needs at least one layer");
  const int stride = n + ch_budget;  // max copies per layer
  std::vector<int> codes(num_layers, 0);
  std::vector<std::string> msgs(num_layers);
  std::atomic<int> next{0};
  auto worker = [&]() {
    for (;;) {
      const int l = next.fetch_add(1);
      if (l >= num_layers) return;
      int32_t m = 0;
      codes[l] = select_best(weights + static_cast<size_t>(l) * n, n, tp, ch_budget, r_max,
                             equal_split, max_schemes, node_budget,
                             out_replicas + static_cast<size_t>(l) * n,
                             out_heads_c + static_cast<size_t>(l) * stride,
                             out_rgs + static_cast<size_t>(l) * stride, &m, out_delta + l);
      out_m[l] = m;
      if (codes[l]) msgs[l] = last_error();
    }
  };
  const int nw = std::max(1, std::min(workers, num_layers));
  if (nw == 1) {
    worker();
  } else {
    std::vector<std::thread> pool;
    for (int i = 0; i < nw; ++i) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
  }
  for (int l = 0; l < num_layers; ++l)
    if (codes[l]) {
      // first failing layer in layer order, prefixed like reference allocate.py:379-386
      const std::string prefix =
          codes[l] == FKV_ERR_INFEASIBLE ? "layer " + std::to_string(l) + ": " : "";
      return set_error(codes[l], prefix + msgs[l]);
    }
  return 0;
}

}  // namespace fkv

// ------------------------------------------------------------- C ABI ----
extern "C" {

const char* fkv_last_error(void) { return fkv::last_error(); }

int fkv_solve_equal_split(const double* w, const int32_t* heads, int32_t m, int32_t tp,
                          double cutoff, int64_t node_budget, const double* hint_spread,
                          const int32_t* hint_rgs, double* out_spread, int32_t* out_rgs,
                          int64_t* out_nodes) {
  return fkv::solve_equal(w, heads, m, tp, cutoff, node_budget, hint_spread, hint_rgs, out_spread,
                          out_rgs, out_nodes);
}

int fkv_solve_free_split(const double* w, const int32_t* heads, int32_t m, int32_t tp,
                         double cutoff, int64_t node_budget, const double* hint_spread,
                         const int32_t* hint_rgs, double* out_spread, int32_t* out_rgs,
                         int64_t* out_nodes) {
  return fkv::solve_free(w, heads, m, tp, cutoff, node_budget, hint_spread, hint_rgs, out_spread,
                         out_rgs, out_nodes);
}

int fkv_select_best(const double* layer_weights, int32_t n, int32_t tp, int32_t ch_budget,
                    int32_t r_max, int32_t equal_split, int64_t max_schemes, int64_t node_budget,
                    int32_t* out_replicas, int32_t* out_heads_c, int32_t* out_rgs, int32_t* out_m,
                    double* out_delta) {
  return fkv::select_best(layer_weights, n, tp, ch_budget, r_max, equal_split, max_schemes,
                          node_budget, out_replicas, out_heads_c, out_rgs, out_m, out_delta);
}

int fkv_optimize_plan(const double* weights, int32_t num_layers, int32_t n, int32_t tp,
                      int32_t ch_budget, int32_t r_max, int32_t equal_split, int64_t max_schemes,
                      int64_t node_budget, int32_t workers, int32_t* out_replicas,
                      int32_t* out_heads_c, int32_t* out_rgs, int32_t* out_m, double* out_delta) {
  return fkv::optimize_plan(weights, num_layers, n, tp, ch_budget, r_max, equal_split, max_schemes,
                            node_budget, workers, out_replicas, out_heads_c, out_rgs, out_m,
                            out_delta);
}

}  // extern "C"

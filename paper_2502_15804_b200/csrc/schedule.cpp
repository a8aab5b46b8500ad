// K4 decode schedule planner (host): which CTA shape decodes a cache and the
// 32-byte piece descriptors every CTA reads (fkv_work_t tables).
//
// Native form of paper_2502_15804_b200/cache.py plan_schedule (and the
// plan_work / plan_work_solo / plan_work_whole / work_table it calls), which
// stays in Python as the checker: tests/test_schedule_native.py compares the
// two bit for bit on random caches and every schedule override.  Built once
// per cache at prefill (compaction) time; the Python planner costs 0.6-1.4
// ms per layer, this one tens of microseconds.  Compiled with
// -ffp-contract=off: the schedule choice model (whole_segments_win) is
// evaluated in the same double operations and order as the Python.
//
// The decode kernel has no reference counterpart; the schedule
// rules are documented in cache.py and DESIGN.md §4-5.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <string>
#include <utility>
#include <vector>

#include "fairkv.h"

namespace fkv {
int set_error(int code, const std::string& msg);

namespace {

using i64 = int64_t;
using V = std::vector<i64>;

constexpr i64 kTile = 16;
constexpr i64 kMaxItemsPerSegment = 32;  // FKV_MAX_PIECES
constexpr i64 kMaxWork = 32;             // FKV_MAX_WORK
constexpr i64 kHybridMinPieceTiles = 32;  // cache.py HYBRID_MIN_PIECE_TILES
constexpr double kHybridLoneTileUs = 0.045;  // cache.py HYBRID_LONE_TILE_US
constexpr i64 kLonePrefetchTiles = 28;       // cache.py LONE_PREFETCH_TILES
constexpr i64 kMinTilesPerWorker = 8;
constexpr i64 kMaxPiecesPerSegment = 4;
constexpr i64 kSoloMaxTilesPerCta = 19;
constexpr i64 kWideMaxSegments = 128;
constexpr i64 kWideMinMeanTiles = 6;
constexpr i64 kWideLongMaxSegments = 384;  // cache.py WIDE_LONG_MAX_SEGMENTS
constexpr i64 kWideLongMinMeanTiles = 40;  // cache.py WIDE_LONG_MIN_MEAN_TILES
constexpr i64 kPairPieceTilesWhole = 12;  // PAIR_PIECE_TILES in _whole_owners / _whole_cta_tiles
constexpr double kSplitUsPerMb = 0.165, kWholeMarginUs = 0.5, kWholeUsPerMb = 0.161;
constexpr double kWholeFullPerTileUs = 0.20;  // cache.py WHOLE_FULL_PER_TILE_US

struct PlanError {
  std::string msg;
};

// Python's -(-a // b) for b > 0 (ceil division, also for a < 0)
inline i64 ceil_div(i64 a, i64 b) {
  i64 q = a / b, r = a % b;
  if (r != 0 && ((r > 0) == (b > 0))) ++q;
  return q;
}

struct Plan {
  std::vector<int32_t> item_seg, t0, t1, seg_item_ptr, warp_ptr, work_list;
};

// numpy.argsort(key, kind="stable") for a descending key given as -key
template <class Key>
std::vector<i64> stable_order(i64 n, Key&& less) {
  std::vector<i64> o(n);
  std::iota(o.begin(), o.end(), 0);
  std::stable_sort(o.begin(), o.end(), less);
  return o;
}

// heapq of (load, worker) tuples: the least load, then the lowest worker id.
// Packed into one int64 key (load << 16 | worker; workers < 65536) so the
// heap compares one integer.
class MinHeap {
 public:
  explicit MinHeap(i64 workers) {
    h_.reserve(workers);
    for (i64 w = 0; w < workers; ++w) h_.push_back(w);  // load 0: already a heap in id order
  }
  std::pair<i64, i64> pop() {
    std::pop_heap(h_.begin(), h_.end(), std::greater<i64>());
    const i64 k = h_.back();
    h_.pop_back();
    return {k >> 16, k & 0xffff};
  }
  void push(i64 load, i64 w) {
    h_.push_back((load << 16) | w);
    std::push_heap(h_.begin(), h_.end(), std::greater<i64>());
  }

 private:
  std::vector<i64> h_;
};

// ---- cut of the concatenated tile stream (cache.py _cut_stream / _cut_stream_cost)
struct Cut {
  V seg, t0, t1, owner;
  i64 max_owner() const { return owner.empty() ? -1 : *std::max_element(owner.begin(), owner.end()); }
};

Cut cut_stream(const V& seg_len, const V& tiles, i64 per, i64 cap) {
  Cut c;
  i64 w = 0, used = 0, cnt = 0;
  for (size_t s = 0; s < seg_len.size(); ++s) {
    const i64 n = tiles[s];
    i64 t = 0;
    while (true) {
      if (cnt >= cap || (used >= per && n > t)) w += 1, used = 0, cnt = 0;
      const i64 take = std::min(n - t, per - used);
      c.seg.push_back(static_cast<i64>(s));
      c.t0.push_back(t * kTile);
      c.t1.push_back(std::min(seg_len[s], (t + take) * kTile));
      c.owner.push_back(w);
      used += take;
      cnt += 1;
      t += take;
      if (t >= n) break;
    }
  }
  return c;
}

Cut cut_stream_cost(const V& seg_len, const V& tiles, i64 C, i64 P, i64 cap) {
  Cut c;
  i64 w = 0, cost = 0, cnt = 0;
  for (size_t s = 0; s < seg_len.size(); ++s) {
    const i64 n = tiles[s];
    i64 t = 0;
    while (true) {
      if (cnt >= cap || (cnt > 0 && (C - cost - P < 1 || (n == t && C - cost - P < 0)))) w += 1, cost = 0, cnt = 0;
      const i64 take = std::min(n - t, std::max<i64>(C - cost - P, 1));
      c.seg.push_back(static_cast<i64>(s));
      c.t0.push_back(t * kTile);
      c.t1.push_back(std::min(seg_len[s], (t + take) * kTile));
      c.owner.push_back(w);
      cost += P + take;
      cnt += 1;
      t += take;
      if (t >= n) break;
    }
  }
  return c;
}

// Does cut_stream_cost(C) fit in W workers?  The same greedy walk without
// materialising the pieces, stopping at the first worker past W (the binary
// search over C probes this ~16 times per plan).
bool cut_fits(const V& seg_len, const V& tiles, i64 C, i64 P, i64 cap, i64 W) {
  i64 w = 0, cost = 0, cnt = 0;
  for (size_t s = 0; s < seg_len.size(); ++s) {
    const i64 n = tiles[s];
    i64 t = 0;
    while (true) {
      if (cnt >= cap || (cnt > 0 && (C - cost - P < 1 || (n == t && C - cost - P < 0)))) {
        if (++w >= W) return false;
        cost = 0, cnt = 0;
      }
      const i64 take = std::min(n - t, std::max<i64>(C - cost - P, 1));
      cost += P + take;
      cnt += 1;
      t += take;
      if (t >= n) break;
    }
  }
  return true;
}

// cache.py _pair_on_sms
V pair_on_sms(const V& owner, const V& t0s, const V& t1s, i64 sms, double pw) {
  const i64 busy = owner.empty() ? 0 : *std::max_element(owner.begin(), owner.end()) + 1;
  const i64 k = busy - sms;
  if (k <= 0) return owner;
  std::vector<double> w_tiles(busy, 0.0);
  for (size_t i = 0; i < owner.size(); ++i)  // np.bincount(weights=...): float adds in index order
    w_tiles[owner[i]] += static_cast<double>((t1s[i] - t0s[i] + kTile - 1) / kTile) + pw;
  // np.argsort(-w_tiles, kind="stable")
  auto order = stable_order(busy, [&](i64 a, i64 b) { return -w_tiles[a] < -w_tiles[b]; });
  V new_id(busy);
  for (i64 j = 0; j < sms - k; ++j) new_id[order[j]] = k + j;  // solo = order[:sms-k] -> arange(k, sms)
  const i64* paired = order.data() + (sms - k);
  for (i64 j = 0; j < k; ++j) {
    new_id[paired[j]] = j;
    new_id[paired[2 * k - 1 - j]] = j + sms;
  }
  V out(owner.size());
  for (size_t i = 0; i < owner.size(); ++i) out[i] = new_id[owner[i]];
  return out;
}

// shared tail of plan_work / plan_work_solo: pointers and the work list
Plan finish(i64 n_seg, const V& seg_i, const V& t0s, const V& t1s, const V& owner, bool whole_order) {
  Plan p;
  const i64 n = static_cast<i64>(seg_i.size());
  p.item_seg.resize(n);
  p.t0.resize(n);
  p.t1.resize(n);
  for (i64 i = 0; i < n; ++i) {
    p.item_seg[i] = static_cast<int32_t>(seg_i[i]);
    p.t0[i] = static_cast<int32_t>(t0s[i]);
    p.t1[i] = static_cast<int32_t>(t1s[i]);
  }
  p.seg_item_ptr.assign(n_seg + 1, 0);
  for (i64 i = 0; i < n; ++i) p.seg_item_ptr[seg_i[i] + 1] += 1;
  for (i64 s = 0; s < n_seg; ++s) p.seg_item_ptr[s + 1] += p.seg_item_ptr[s];
  const i64 busy = n ? *std::max_element(owner.begin(), owner.end()) + 1 : 1;
  p.warp_ptr.assign(busy + 1, 0);
  for (i64 i = 0; i < n; ++i) p.warp_ptr[owner[i] + 1] += 1;
  for (i64 w = 0; w < busy; ++w) p.warp_ptr[w + 1] += p.warp_ptr[w];
  std::vector<i64> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  if (whole_order) {  // np.argsort(owner, kind="stable")
    std::stable_sort(idx.begin(), idx.end(), [&](i64 a, i64 b) { return owner[a] < owner[b]; });
  } else {  // np.lexsort((arange, ~split, owner)): owner, split pieces first, index
    auto split = [&](i64 i) {
      const i64 s = seg_i[i];
      return p.seg_item_ptr[s + 1] - p.seg_item_ptr[s] > 1;
    };
    std::stable_sort(idx.begin(), idx.end(), [&](i64 a, i64 b) {
      if (owner[a] != owner[b]) return owner[a] < owner[b];
      const bool sa = split(a), sb = split(b);
      if (sa != sb) return sa;  // ~split: False (split) sorts first
      return a < b;
    });
  }
  p.work_list.resize(n);
  for (i64 i = 0; i < n; ++i) p.work_list[i] = static_cast<int32_t>(idx[i]);
  return p;
}

// cache.py plan_work
Plan plan_work(const V& seg_len, i64 n_workers, i64 chunk, i64 min_tiles, i64 P, i64 sms, bool sm_pairing,
               double pair_piece) {
  const i64 n_seg = static_cast<i64>(seg_len.size());
  V tiles(n_seg);
  i64 tsum = 0, longest = 0;
  for (i64 s = 0; s < n_seg; ++s) {
    tiles[s] = (seg_len[s] + kTile - 1) / kTile;
    tsum += tiles[s];
    longest = std::max(longest, tiles[s]);
  }
  const i64 W = std::max<i64>(1, n_workers);
  V seg_i, t0s, t1s, owner;
  if (chunk <= 0) {
    i64 per = std::max({ceil_div(tsum, W), min_tiles, static_cast<i64>(1)});
    const i64 avg = tsum / std::max<i64>(n_seg, 1);
    per = std::max(per, ceil_div(avg, kMaxPiecesPerSegment));
    per = std::max(per, ceil_div(longest, kMaxItemsPerSegment - 1));
    if (P > 0 && n_seg) {
      i64 lo = std::max(per + P, ceil_div(tsum + P * n_seg, W));
      i64 hi = std::max(lo, tsum + P * (n_seg + 1));
      i64 best = -1;
      while (lo <= hi) {
        const i64 C = (lo + hi) / 2;
        if (cut_fits(seg_len, tiles, C, P, kMaxWork, W)) {
          best = C;
          hi = C - 1;
        } else {
          lo = C + 1;
        }
      }
      if (best < 0)
        throw PlanError{std::to_string(n_seg) + " segments exceed one launch (" + std::to_string(W) +
                        " workers x " + std::to_string(kMaxWork) + " pieces)"};
      Cut cut = cut_stream_cost(seg_len, tiles, best, P, kMaxWork);
      seg_i = std::move(cut.seg), t0s = std::move(cut.t0), t1s = std::move(cut.t1), owner = std::move(cut.owner);
    } else {
      while (true) {
        Cut cut = cut_stream(seg_len, tiles, per, kMaxWork);
        seg_i = cut.seg, t0s = cut.t0, t1s = cut.t1, owner = cut.owner;
        if (owner.empty() || cut.max_owner() < W) break;
        if (per >= tsum)
          throw PlanError{std::to_string(n_seg) + " segments exceed one launch (" + std::to_string(W) +
                          " workers x " + std::to_string(kMaxWork) + " pieces)"};
        per *= 2;
      }
    }
  } else {
    i64 ch = std::max<i64>(1, ceil_div(chunk, kTile));
    ch = std::max(ch, ceil_div(longest, kMaxItemsPerSegment)) * kTile;
    V lens;
    for (i64 s = 0; s < n_seg; ++s) {
      const i64 cnt = std::max<i64>(1, ceil_div(seg_len[s], ch));
      for (i64 j = 0; j < cnt; ++j) {
        seg_i.push_back(s);
        const i64 a = j * ch, b = std::min(a + ch, seg_len[s]);
        t0s.push_back(a);
        t1s.push_back(b);
        lens.push_back(std::max<i64>(b - a, 0));
      }
    }
    i64 lsum = 0;
    for (i64 x : lens) lsum += x;
    const i64 per = std::max<i64>(1, ceil_div(lsum, W));
    owner.resize(lens.size());
    i64 cum = 0;
    std::vector<i64> cnt(W, 0);
    i64 maxcnt = 0;
    for (size_t i = 0; i < lens.size(); ++i) {
      owner[i] = std::min(cum / per, W - 1);
      cum += lens[i];
      maxcnt = std::max(maxcnt, ++cnt[owner[i]]);
    }
    if (!lens.empty() && maxcnt > kMaxWork) {
      i64 w = 0, used = 0, c = 0;
      for (size_t i = 0; i < lens.size(); ++i) {
        if (c >= kMaxWork || used >= per) w += 1, used = 0, c = 0;
        owner[i] = w;
        used += lens[i];
        c += 1;
      }
      if (w >= W)
        throw PlanError{std::to_string(lens.size()) + " pieces exceed one launch (" + std::to_string(W) +
                        " workers x " + std::to_string(kMaxWork) + " pieces)"};
    }
  }
  if (sms > 0 && sm_pairing) owner = pair_on_sms(owner, t0s, t1s, sms, pair_piece);
  return finish(n_seg, seg_i, t0s, t1s, owner, false);
}

// Python's round() (half to even) of j * n / k
inline i64 py_round_div(i64 num, i64 den) {
  return static_cast<i64>(std::nearbyint(static_cast<double>(num) / static_cast<double>(den)));
}

// cache.py plan_work_solo
Plan plan_work_solo(const V& seg_len, i64 n_workers, i64 piece_tiles, i64 whole_tiles) {
  const i64 n_seg = static_cast<i64>(seg_len.size());
  V tiles(n_seg);
  i64 total = 0;
  for (i64 s = 0; s < n_seg; ++s) tiles[s] = (seg_len[s] + kTile - 1) / kTile, total += tiles[s];
  const i64 W = std::max<i64>(1, n_workers);
  const i64 piece = std::max({piece_tiles, ceil_div(total, W), static_cast<i64>(1)});
  V seg_i, t0s, t1s;
  for (i64 s = 0; s < n_seg; ++s) {
    const i64 n = tiles[s];
    const i64 k = n <= whole_tiles ? 1 : std::min(kMaxItemsPerSegment, ceil_div(n, piece));
    for (i64 j = 0; j < k; ++j) {
      seg_i.push_back(s);
      t0s.push_back(py_round_div(j * n, k) * kTile);
      t1s.push_back(std::min(seg_len[s], py_round_div((j + 1) * n, k) * kTile));
    }
  }
  const i64 n_items = static_cast<i64>(seg_i.size());
  V owner(n_items);
  if (n_items <= W) {
    std::iota(owner.begin(), owner.end(), 0);
  } else {
    V size(n_items);
    for (i64 i = 0; i < n_items; ++i) size[i] = std::max<i64>(t1s[i] - t0s[i], 0);
    // np.lexsort((arange, -size)): size descending, index ascending
    auto order = stable_order(n_items, [&](i64 a, i64 b) { return size[a] > size[b]; });
    MinHeap heap(W);
    std::vector<i64> cnt(W, 0);
    for (i64 i : order) {
      const auto [load, w] = heap.pop();
      owner[i] = w;
      cnt[w] += 1;
      heap.push(load + size[i] + 1, w);
    }
    if (*std::max_element(cnt.begin(), cnt.end()) > kMaxWork)
      throw PlanError{"too many pieces for the per-warp schedule"};
    // np.unique(owner, return_inverse=True): rank among the used worker ids
    std::vector<i64> rank(W, -1);
    i64 r = 0;
    for (i64 w = 0; w < W; ++w)
      if (cnt[w]) rank[w] = r++;
    for (i64 i = 0; i < n_items; ++i) owner[i] = rank[owner[i]];
  }
  return finish(n_seg, seg_i, t0s, t1s, owner, false);
}

// cache.py _whole_owners
V whole_owners(const V& seg_tiles, i64 workers, i64 sms, double pair_piece) {
  const i64 n = static_cast<i64>(seg_tiles.size());
  V owner(n);
  if (n <= sms) {
    std::iota(owner.begin(), owner.end(), 0);
    return owner;
  }
  auto order = stable_order(n, [&](i64 a, i64 b) { return seg_tiles[a] > seg_tiles[b]; });
  MinHeap heap(workers);
  std::vector<char> used(workers, 0);
  for (i64 s : order) {
    const auto [load, w] = heap.pop();
    owner[s] = w;
    used[w] = 1;
    heap.push(load + seg_tiles[s] + (load ? kPairPieceTilesWhole : 0), w);
  }
  std::vector<i64> rank(workers, -1);
  i64 r = 0;
  for (i64 w = 0; w < workers; ++w)
    if (used[w]) rank[w] = r++;
  for (i64 i = 0; i < n; ++i) owner[i] = rank[owner[i]];
  V t0(n, 0), t1(n);
  for (i64 i = 0; i < n; ++i) t1[i] = seg_tiles[i] * kTile;
  return pair_on_sms(owner, t0, t1, sms, pair_piece);
}

// cache.py whole_segments_win
bool whole_segments_win(const V& seg_tiles, i64 workers, bool wide, i64 sms, double pair_piece) {
  const i64 n = static_cast<i64>(seg_tiles.size());
  if (!n || n > workers * kMaxWork) return false;
  const double s0 = wide ? 5.6 : 7.6, w0 = wide ? 3.3 : 2.6;
  double per_tile = (!wide && n >= 2 * workers) ? kWholeFullPerTileUs : (wide ? 0.104 : 0.285);
  if (wide && n <= 32 && *std::max_element(seg_tiles.begin(), seg_tiles.end()) <= kLonePrefetchTiles)
    per_tile = kHybridLoneTileUs;  // a few short segments, each held whole by its CTA's rings
  i64 tsum = 0;
  for (i64 t : seg_tiles) tsum += t;
  const double mb = static_cast<double>(tsum) * kTile * FKV_HEAD_DIM * 4 / 1e6;
  V owner = whole_owners(seg_tiles, workers, sms, pair_piece);
  const i64 busy = *std::max_element(owner.begin(), owner.end()) + 1;
  std::vector<double> tiles(busy, 0.0);
  std::vector<i64> cnt(busy, 0);
  for (i64 i = 0; i < n; ++i) tiles[owner[i]] += static_cast<double>(seg_tiles[i]), cnt[owner[i]] += 1;
  double crit = -1.0;
  for (i64 w = 0; w < busy; ++w)
    crit = std::max(crit, tiles[w] + static_cast<double>(std::max<i64>(cnt[w] - 1, 0) * kPairPieceTilesWhole));
  const double whole = w0 + std::max(per_tile * crit, kWholeUsPerMb * mb);
  return whole + kWholeMarginUs <= s0 + kSplitUsPerMb * mb;
}

// cache.py plan_work_hybrid: whole segments, the longest cut into equal
// pieces of <= T tiles (T the least >= kHybridMinPieceTiles whose pieces fit
// one per SM), one piece per CTA
Plan plan_work_hybrid(const V& seg_len, i64 sms, double per_tile_us, double min_saving_us) {
  const i64 n = static_cast<i64>(seg_len.size());
  V tiles(n);
  i64 hi = 1;
  for (i64 s = 0; s < n; ++s) {
    tiles[s] = std::max<i64>((seg_len[s] + kTile - 1) / kTile, 1);
    hi = std::max(hi, tiles[s]);
  }
  const i64 longest = hi;
  i64 lo = std::min(kHybridMinPieceTiles, hi);
  while (lo < hi) {
    const i64 T = (lo + hi) / 2;
    i64 pieces = 0;
    for (i64 t : tiles) pieces += ceil_div(t, T);
    if (pieces <= sms) hi = T;
    else lo = T + 1;
  }
  if (per_tile_us * static_cast<double>(longest - lo) <= min_saving_us) lo = longest;  // not worth its merges
  V seg_i, t0, t1, owner;
  for (i64 s = 0; s < n; ++s) {
    const i64 k = std::min(ceil_div(tiles[s], lo), kMaxItemsPerSegment);
    for (i64 j = 0; j < k; ++j) {
      const i64 b = std::min((j + 1) * tiles[s] / k * kTile, seg_len[s]);
      seg_i.push_back(s);
      t0.push_back(std::min(j * tiles[s] / k * kTile, b));
      t1.push_back(b);
      owner.push_back(static_cast<i64>(owner.size()));
    }
  }
  return finish(n, seg_i, t0, t1, owner, true);
}

// cache.py plan_work_whole
Plan plan_work_whole(const V& seg_len, i64 workers, i64 sms, double pair_piece) {
  const i64 n = static_cast<i64>(seg_len.size());
  V tiles(n);
  for (i64 s = 0; s < n; ++s) tiles[s] = (seg_len[s] + kTile - 1) / kTile;
  V owner = whole_owners(tiles, workers, sms, pair_piece);
  const i64 busy = *std::max_element(owner.begin(), owner.end()) + 1;
  std::vector<i64> cnt(busy, 0);
  for (i64 o : owner) cnt[o] += 1;
  if (*std::max_element(cnt.begin(), cnt.end()) > kMaxWork)
    throw PlanError{"too many segments per CTA for the whole-segment schedule"};
  V seg_i(n), t0(n, 0), t1(n);
  std::iota(seg_i.begin(), seg_i.end(), 0);
  for (i64 s = 0; s < n; ++s) t1[s] = seg_len[s];
  return finish(n, seg_i, t0, t1, owner, true);
}

// cache.py work_table -> tab [rows][K][8]
int work_table(const i64* seg_row0, const V& seg_len, const i64* seg_qrow, const i64* seg_out_row,
               const Plan& p, i64 solo_ctas, std::vector<int32_t>& tab, i64& rows_out, i64& K_out) {
  const i64 busy = static_cast<i64>(p.warp_ptr.size()) - 1;
  const i64 n = static_cast<i64>(p.work_list.size());
  std::vector<i64> w_of(n);  // np.repeat(arange(busy), counts): worker of list position i
  for (i64 w = 0; w < busy; ++w)
    for (i64 i = p.warp_ptr[w]; i < p.warp_ptr[w + 1]; ++i) w_of[i] = w;
  i64 rows;
  std::vector<i64> row_of(n), tag_of(n);
  if (solo_ctas > 0) {
    rows = std::min(solo_ctas, std::max<i64>(busy, 1));
    for (i64 i = 0; i < n; ++i) row_of[i] = w_of[i] % rows, tag_of[i] = w_of[i] / rows;
  } else {
    rows = std::max<i64>(busy, 1);
    for (i64 i = 0; i < n; ++i) row_of[i] = w_of[i], tag_of[i] = 0;
  }
  std::vector<i64> per_row(rows, 0);
  for (i64 i = 0; i < n; ++i) per_row[row_of[i]] += 1;
  const i64 K = std::max<i64>(1, n ? *std::max_element(per_row.begin(), per_row.end()) : 1);
  if (K > kMaxWork) throw PlanError{std::to_string(K) + " pieces on one CTA exceed FKV_MAX_WORK"};
  tab.assign(rows * K * 8, 0);
  std::vector<i64> next(rows, 0);  // pieces of a row in list (worker) order: stable by row
  for (i64 i = 0; i < n; ++i) {
    const i64 r = row_of[i], j = next[r]++;
    const i64 it = p.work_list[i];
    const i64 seg = p.item_seg[it];
    const i64 a = p.t0[it];
    const i64 b = std::min<i64>(p.t1[it], seg_len[seg]);
    const i64 row0 = seg_row0[seg] + a;
    int32_t* d = &tab[(r * K + j) * 8];
    d[0] = static_cast<int32_t>(static_cast<uint32_t>(row0 & 0xFFFFFFFF));
    d[1] = static_cast<int32_t>(row0 >> 32);
    d[2] = static_cast<int32_t>(std::max<i64>(b - a, 0));
    d[3] = static_cast<int32_t>(seg_qrow[seg]);
    d[4] = static_cast<int32_t>(seg_out_row[seg]);
    d[5] = static_cast<int32_t>(it);
    d[6] = p.seg_item_ptr[seg];
    d[7] = static_cast<int32_t>((p.seg_item_ptr[seg + 1] - p.seg_item_ptr[seg]) | (tag_of[i] << 16));
  }
  rows_out = rows;
  K_out = K;
  return 0;
}

// cache.py plan_schedule
int plan_schedule(const V& seg_len, const i64* seg_row0, const i64* seg_qrow, const i64* seg_out_row,
                  const fkv_sched_params& prm, Plan& plan, std::vector<int32_t>& tab, i64& rows, i64& K,
                  int& flags) {
  const i64 sms = prm.sms;
  const i64 solo_ctas = sms * prm.ctas_solo;
  const i64 n_seg = static_cast<i64>(seg_len.size());
  V seg_tiles(n_seg);
  i64 tiles = 0;
  for (i64 s = 0; s < n_seg; ++s) seg_tiles[s] = (seg_len[s] + kTile - 1) / kTile, tiles += seg_tiles[s];
  const int mode = prm.mode;  // 0 auto, 1 coop, 2 wide, 3 solo
  const bool small = tiles <= kSoloMaxTilesPerCta * solo_ctas && prm.solo_small;
  const double mean = n_seg ? static_cast<double>(tiles) / static_cast<double>(n_seg) : 0.0;
  const i64 warps = 4 * solo_ctas;
  const bool many_short = (n_seg >= warps && mean <= 24) || (n_seg >= 0.4 * warps && mean <= 12);
  const bool solo = mode == 3 || (mode == 0 && prm.chunk <= 0 && (small || many_short));
  if (solo) {
    i64 pt, wt;
    if (small || (mode == 3 && !many_short)) {
      const double x = std::nearbyint(1.5 * static_cast<double>(tiles) / static_cast<double>(warps));
      pt = wt = static_cast<i64>(std::min(std::max(x, 4.0), 8.0));
    } else {
      pt = wt = std::max<i64>(16, ceil_div(2 * tiles, warps));
    }
    if (prm.solo_piece >= 0) pt = prm.solo_piece;
    if (prm.solo_whole >= 0) wt = prm.solo_whole;
    try {
      plan = plan_work_solo(seg_len, warps, pt, wt);
      work_table(seg_row0, seg_len, seg_qrow, seg_out_row, plan, solo_ctas, tab, rows, K);
      flags = FKV_DECODE_SOLO;
      return 0;
    } catch (const PlanError&) {
      // too many pieces for the per-CTA tables: cooperative schedule
    }
  }
  const bool wide = mode == 2 || (mode != 1 && ((n_seg <= kWideMaxSegments && mean >= kWideMinMeanTiles) ||
                                                 (n_seg <= kWideLongMaxSegments && mean >= kWideLongMinMeanTiles)));
  flags = wide ? FKV_DECODE_WIDE : 0;
  const i64 workers = sms * (wide ? prm.ctas_wide : prm.ctas_coop);
  const i64 ctas_sm = std::max<i64>(1, workers / (sms * prm.ctas_wide));
  const i64 sms_eff = workers / ctas_sm;
  if (prm.chunk <= 0 && n_seg > 0 && n_seg <= workers * kMaxWork &&
      (prm.whole == 1 || (prm.whole < 0 && whole_segments_win(seg_tiles, workers, wide, sms_eff, prm.pair_piece)))) {
    // one CTA per SM: the longest segments cut when that pays for the merges
    const double per_tile = n_seg <= 32 ? kHybridLoneTileUs : (wide ? 0.104 : 0.285);  // WHOLE_MODEL
    plan = n_seg <= sms_eff ? plan_work_hybrid(seg_len, sms_eff, per_tile, prm.hybrid_saving_us)
                            : plan_work_whole(seg_len, workers, sms_eff, prm.pair_piece);
    work_table(seg_row0, seg_len, seg_qrow, seg_out_row, plan, 0, tab, rows, K);
    return 0;
  }
  plan = plan_work(seg_len, workers, prm.chunk, kMinTilesPerWorker, prm.piece_cost,
                   ctas_sm > 1 ? workers / ctas_sm : 0, prm.sm_pairing != 0, prm.pair_piece);
  work_table(seg_row0, seg_len, seg_qrow, seg_out_row, plan, 0, tab, rows, K);
  return 0;
}

}  // namespace
}  // namespace fkv

extern "C" int fkv_plan_schedule(const int64_t* seg_len, const int64_t* seg_row0, const int64_t* seg_qrow,
                                 const int64_t* seg_out_row, int32_t n_seg, const fkv_sched_params* prm,
                                 int32_t item_cap, int32_t worker_cap, int32_t table_cap, int32_t* item_seg,
                                 int32_t* item_t0, int32_t* item_t1, int32_t* seg_item_ptr, int32_t* warp_ptr,
                                 int32_t* work_list, int32_t* table, int32_t* out_sizes) {
  using namespace fkv;
  if (n_seg < 0 || !prm || !out_sizes || (n_seg && (!seg_len || !seg_row0 || !seg_qrow || !seg_out_row)))
    return set_error(FKV_ERR_INVALID, "fkv_plan_schedule: bad arguments");
  if (prm->sms < 1 || prm->ctas_coop < 1 || prm->ctas_wide < 1 || prm->ctas_solo < 1 ||
      static_cast<int64_t>(prm->sms) * 4 * std::max({prm->ctas_coop, prm->ctas_wide, prm->ctas_solo}) >= 65536)
    return set_error(FKV_ERR_INVALID, "fkv_plan_schedule: bad device parameters");  // MinHeap packs worker ids in 16 bits
  V len(seg_len, seg_len + n_seg);
  for (i64 x : len)
    if (x < 0) return set_error(FKV_ERR_INVALID, "fkv_plan_schedule: negative segment length");
  Plan plan;
  std::vector<int32_t> tab;
  i64 rows = 0, K = 0;
  int flags = 0;
  try {
    plan_schedule(len, seg_row0, seg_qrow, seg_out_row, *prm, plan, tab, rows, K, flags);
  } catch (const PlanError& e) {
    return set_error(FKV_ERR_VALIDATION, "fkv_plan_schedule: " + e.msg);
  }
  const i64 n_items = static_cast<i64>(plan.item_seg.size());
  const i64 busy = static_cast<i64>(plan.warp_ptr.size()) - 1;
  out_sizes[0] = static_cast<int32_t>(n_items);
  out_sizes[1] = static_cast<int32_t>(busy);
  out_sizes[2] = static_cast<int32_t>(rows);
  out_sizes[3] = static_cast<int32_t>(K);
  out_sizes[4] = flags;
  if (n_items > item_cap || busy > worker_cap || rows * K * 8 > table_cap)
    return set_error(FKV_ERR_INVALID, "fkv_plan_schedule: output buffers too small (sizes in out_sizes)");
  std::copy(plan.item_seg.begin(), plan.item_seg.end(), item_seg);
  std::copy(plan.t0.begin(), plan.t0.end(), item_t0);
  std::copy(plan.t1.begin(), plan.t1.end(), item_t1);
  std::copy(plan.seg_item_ptr.begin(), plan.seg_item_ptr.end(), seg_item_ptr);
  std::copy(plan.warp_ptr.begin(), plan.warp_ptr.end(), warp_ptr);
  std::copy(plan.work_list.begin(), plan.work_list.end(), work_list);
  std::copy(tab.begin(), tab.end(), table);
  return FKV_OK;
}

// Every int32 table a layer cache keeps on the device, planned and packed in
// one host buffer for one host-to-device copy (cache.LayerCache._build;
// _pack_tables_py is the Python form it replaces, kept as the checker).
extern "C" int fkv_cache_tables(const int64_t* seg_len, const int64_t* seg_row0, const int64_t* seg_qrow,
                                const int64_t* seg_out_row, const int64_t* seg_cap, const int64_t* append_src,
                                int32_t n_seg, const fkv_sched_params* prm, int32_t* buf, int64_t buf_words,
                                int64_t* part_off, int32_t* out_sizes) {
  using namespace fkv;
  if (n_seg < 0 || !prm || !out_sizes || !part_off ||
      (n_seg && (!seg_len || !seg_row0 || !seg_qrow || !seg_out_row)))
    return set_error(FKV_ERR_INVALID, "fkv_cache_tables: bad arguments");
  if (prm->sms < 1 || prm->ctas_coop < 1 || prm->ctas_wide < 1 || prm->ctas_solo < 1 ||
      static_cast<int64_t>(prm->sms) * 4 * std::max({prm->ctas_coop, prm->ctas_wide, prm->ctas_solo}) >= 65536)
    return set_error(FKV_ERR_INVALID, "fkv_cache_tables: bad device parameters");
  V len(seg_len, seg_len + n_seg);
  for (i64 x : len)
    if (x < 0) return set_error(FKV_ERR_INVALID, "fkv_cache_tables: negative segment length");
  Plan plan;
  std::vector<int32_t> tab;
  i64 rows = 0, K = 0;
  int flags = 0;
  try {
    plan_schedule(len, seg_row0, seg_qrow, seg_out_row, *prm, plan, tab, rows, K, flags);
  } catch (const PlanError& e) {
    return set_error(FKV_ERR_VALIDATION, "fkv_plan_schedule: " + e.msg);
  }
  const i64 n = n_seg, n_items = static_cast<i64>(plan.item_seg.size());
  const i64 busy = static_cast<i64>(plan.warp_ptr.size()) - 1;
  out_sizes[0] = static_cast<int32_t>(n_items);
  out_sizes[1] = static_cast<int32_t>(busy);
  out_sizes[2] = static_cast<int32_t>(rows);
  out_sizes[3] = static_cast<int32_t>(K);
  out_sizes[4] = flags;
  const i64 cnt = std::max<i64>(n_items, 1);
  const i64 lens[FKV_CT_PARTS] = {n, n, n, n_items, n_items, n_items, n + 1, n_items, busy + 1,
                                  n_items, rows * K * 8, n, n, n, cnt, 1, 2 * n};
  part_off[0] = 0;
  for (int i = 0; i < FKV_CT_PARTS; ++i) part_off[i + 1] = part_off[i] + (lens[i] + 3) / 4 * 4;
  if (part_off[FKV_CT_PARTS] > buf_words)
    return set_error(FKV_ERR_INVALID, "fkv_cache_tables: buffer too small (words needed in part_off[17])");
  if (!buf) return set_error(FKV_ERR_INVALID, "fkv_cache_tables: null buffer");
  std::fill(buf, buf + part_off[FKV_CT_PARTS], 0);
  auto put64 = [&](int part, const int64_t* src, i64 m, int64_t dflt) {
    int32_t* d = buf + part_off[part];
    for (i64 i = 0; i < m; ++i) d[i] = static_cast<int32_t>(src ? src[i] : dflt);
  };
  auto put32 = [&](int part, const std::vector<int32_t>& src) {
    std::copy(src.begin(), src.end(), buf + part_off[part]);
  };
  put64(FKV_CT_SEG_LEN, seg_len, n, 0);
  put64(FKV_CT_SEG_QROW, seg_qrow, n, 0);
  put64(FKV_CT_SEG_OUT_ROW, seg_out_row, n, 0);
  put32(FKV_CT_ITEM_SEG, plan.item_seg);
  put32(FKV_CT_ITEM_T0, plan.t0);
  put32(FKV_CT_ITEM_T1, plan.t1);
  put32(FKV_CT_SEG_ITEM_PTR, plan.seg_item_ptr);
  std::iota(buf + part_off[FKV_CT_SRC_IDX], buf + part_off[FKV_CT_SRC_IDX] + n_items, 0);
  put32(FKV_CT_WARP_PTR, plan.warp_ptr);
  put32(FKV_CT_WORK_LIST, plan.work_list);
  put32(FKV_CT_WORK, tab);
  put64(FKV_CT_SEG_CAP, seg_cap ? seg_cap : seg_len, n, 0);
  put64(FKV_CT_APPEND_SRC, append_src, n, -1);
  // flat work-table index of every segment's last piece (fkv_append grows it)
  std::vector<int32_t> pos(cnt, 0);
  for (i64 e = 0; e < rows * K; ++e)
    if (tab[e * 8 + 7] & 0xFFFF) pos[tab[e * 8 + 5]] = static_cast<int32_t>(e);
  int32_t* lp = buf + part_off[FKV_CT_LAST_PIECE];
  for (i64 s = 0; s < n; ++s) {
    i64 it = plan.seg_item_ptr[s + 1] - 1;
    if (it < 0) it += cnt;  // as numpy's index -1
    lp[s] = pos[it];
  }
  // counters and the overflow flag stay zero
  std::copy(seg_row0, seg_row0 + n, reinterpret_cast<int64_t*>(buf + part_off[FKV_CT_SEG_ROW0]));
  return FKV_OK;
}

/* fairkv.h -- C ABI of the B200-native FairKV hot path (libfairkv.so).
 *
 * Everything a foreign caller binds: plain pointers, sizes and a cudaStream_t
 * passed as void*.  No torch types cross this boundary.  Kernels never
 * allocate: the caller owns every buffer (workspaces included) and every call
 * is stream-ordered with no host synchronisation inside.
 *
 * Return convention: >= 0 success (solvers: 1 = found, 0 = none), < 0 error;
 * the message of the most recent error on the calling thread is
 * fkv_last_error().
 *
 * Two groups of entry points:
 *
 *   B1  AHA placement plugin.  Replaces the reference's search-kernel
 *       backend  headbalance._kernel.solve_equal_split / solve_free_split
 *       (reference pkg/src/headbalance/_kernel/__init__.py:49-57; contract
 *       pkg/src/headbalance/_kernel/reference.py:80-100, 238-244).  Host
 *       C++; bit-identical to the reference including node counts.
 *       fkv_select_best / fkv_optimize_plan additionally replace the Python
 *       scheme loop select_best (reference allocate.py:236-277) and the
 *       process-pool layer loop optimize_plan (reference allocate.py:353-389).
 *
 *   B3  Compressed-cache decode path (no reference implementation exists:
 *       SPEC.md:8 puts inference out of the reference's scope; the paper used
 *       KVPress AdaKV on A100s).  sm_100a CUDA kernels.
 *
 * Cache layout used by B3: a layer's compressed
 * K and V on one GPU are two bf16 arrays of rows of head_dim = 128 elements
 * (256 B).  Row r stores its sixteen 16-byte chunks XOR-swizzled:
 * logical chunk c lives at physical chunk c ^ (r & 7).  A *segment* is the
 * retained tokens of one (request, KV-head copy); it occupies seg_len
 * consecutive rows starting at seg_row0.  Storage for a segment is allocated
 * page aligned (FKV_PAGE) with zero rows up to the next page boundary; a
 * DP copy of a head may address a sub-range of such storage, so kernels only
 * require seg_row0 % FKV_SPLIT == 0.
 */
#ifndef FAIRKV_H_
#define FAIRKV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FKV_OK 0
#define FKV_ERR_INVALID (-1)      /* bad argument / shape */
#define FKV_ERR_CUDA (-2)         /* CUDA launch / runtime error */
#define FKV_ERR_VALIDATION (-3)   /* maps to headbalance ValidationError */
#define FKV_ERR_INFEASIBLE (-4)   /* maps to headbalance InfeasibleError */
#define FKV_ERR_SEARCH_SPACE (-5) /* maps to headbalance SearchSpaceError */

#define FKV_HEAD_DIM 128
#define FKV_PAGE 64 /* tokens per page; segment starts are page aligned */
#define FKV_SPLIT 16 /* DP-copy token cuts are multiples of this (16-token tiles) */
#define FKV_REC 132 /* floats per partial record: o[128], lse, 3 pad (16-B aligned) */
#define FKV_MAX_PEERS 8 /* GPUs of one NVLink/NVSwitch node */

const char* fkv_last_error(void);
int fkv_version(void);
/* SHA-256 (hex) of the sources, headers and flags the library was built
 * from (csrc/build.py); the Python binding refuses a library whose hash
 * does not match the sources next to it. */
const char* fkv_source_hash(void);

/* ------------------------------------------------------------ B1 planner -- */

/* Best equal-cardinality grouping of m copies into tp groups with spread
 * strictly below cutoff.  w: adjusted copy weights, heaviest first (ties by
 * head id); heads: owning head per copy.  hint_spread == NULL means no hint,
 * else (*hint_spread, hint_rgs[m]) is a known grouping.  On return 1,
 * (*out_spread, out_rgs[m]) is the grouping (restricted-growth labels);
 * 0 = nothing below cutoff.  *out_nodes = B&B nodes visited (<= node_budget).
 * Replaces reference _kernel/reference.py:80-235 (and _fastpath.pyx:136-226). */
int fkv_solve_equal_split(const double* w, const int32_t* heads, int32_t m, int32_t tp,
                          double cutoff, int64_t node_budget, const double* hint_spread,
                          const int32_t* hint_rgs, double* out_spread, int32_t* out_rgs,
                          int64_t* out_nodes);

/* Relaxed variant: groups only need to be nonempty.
 * Replaces reference _kernel/reference.py:238-340 (pure Python in the reference). */
int fkv_solve_free_split(const double* w, const int32_t* heads, int32_t m, int32_t tp,
                         double cutoff, int64_t node_budget, const double* hint_spread,
                         const int32_t* hint_rgs, double* out_spread, int32_t* out_rgs,
                         int64_t* out_nodes);

/* Whole per-layer search (reference allocate.py:236-277): every scheme in
 * (total copies, replicas) order, canonical copies, SHA hint for the identity
 * scheme, strict-improvement cutoff.  Outputs the winning scheme
 * out_replicas[n], its canonical copy heads out_heads_c[m] and groups
 * out_rgs[m] (m = *out_m <= n + ch_budget) and spread *out_delta. */
int fkv_select_best(const double* layer_weights, int32_t n, int32_t tp, int32_t ch_budget,
                    int32_t r_max, int32_t equal_split, int64_t max_schemes, int64_t node_budget,
                    int32_t* out_replicas, int32_t* out_heads_c, int32_t* out_rgs, int32_t* out_m,
                    double* out_delta);

/* fkv_select_best over num_layers rows of weights[num_layers][n] with a
 * thread pool of `workers`.  Per-layer outputs are strided: replicas by n,
 * heads_c / rgs by (n + ch_budget). */
int fkv_optimize_plan(const double* weights, int32_t num_layers, int32_t n, int32_t tp,
                      int32_t ch_budget, int32_t r_max, int32_t equal_split, int64_t max_schemes,
                      int64_t node_budget, int32_t workers, int32_t* out_replicas,
                      int32_t* out_heads_c, int32_t* out_rgs, int32_t* out_m, double* out_delta);

/* ------------------------------------------------- B3 decode over the cache -- */

/* K4 (+ fused K5): split-KV decode attention over ragged segments (one
 * layer, one GPU) by warp-persistent workers with a static schedule.
 * The segments' retained tokens are cut into *pieces* (16-token aligned
 * sub-ranges); worker w processes the pieces work[w][0 .. ) in order, up to
 * the first entry with n_it == 0 (or work_k entries).  Worker w is warp
 * (w / grid) of CTA (w % grid), so short schedules still spread over every
 * SM.  Piece descriptor (32 bytes, 16-byte aligned table): */
typedef struct fkv_work {
  int64_t row0;    /* first cache row of the piece (multiple of FKV_SPLIT)         */
  int32_t n_tok;   /* tokens in the piece (>= 0)                                  */
  int32_t qrow;    /* q rows qrow .. qrow+group-1 are the segment's query heads   */
  int32_t out_row; /* output rows out_row .. +group-1 of the segment              */
  int32_t rec;     /* partial-record index of this piece (< n_items)              */
  int32_t i0;      /* record index of the segment's first piece; the segment's    */
                   /* records are i0 .. i0+n_it-1, its arrival counter counters[i0] */
  int32_t n_it;    /* pieces of the segment (1 .. FKV_MAX_PIECES); 0 = end of list */
} fkv_work_t;
#define FKV_MAX_WORK 32   /* entries per worker */
#define FKV_MAX_PIECES 32 /* pieces per segment */
/* flags: FKV_DECODE_SOLO = per-warp schedule for small caches.  Worker w is
 * then one CTA whose four warps each stream their own pieces start to finish
 * (piece owner warp = n_it >> 16, pieces per segment = n_it & 0xffff);
 * without it the four warps share every piece of the CTA's list. */
#define FKV_DECODE_SOLO 1
/* FKV_DECODE_WIDE = cooperative schedule with 8-warp CTAs (one per SM, seven
 * streaming warps per piece) instead of 4-warp CTAs (two per SM). */
#define FKV_DECODE_WIDE 2
/* FKV_DECODE_AFTER_WAIT: the cache or its work table was just written on
 * this stream (fkv_append / fkv_compact).  The kernel is launched with
 * programmatic dependent launch; by default it reads the work table and
 * starts its first K/V copies before waiting for the preceding grid (they
 * are static between steps).  With this flag every global read comes after
 * the wait. */
#define FKV_DECODE_AFTER_WAIT 4

/* Host-side K4 schedule planner (csrc/schedule.cpp; the Python form is
 * cache.plan_schedule, kept as its checker).  Picks the CTA shape of one
 * cache (FKV_DECODE_SOLO / FKV_DECODE_WIDE / cooperative; split or
 * whole-segment pieces) and builds its work table.  Device parameters: SM
 * count and fkv_decode_ctas_per_sm() of each shape; the remaining fields are
 * the planner's tuning knobs (cache.py: FKV_K4_SCHEDULE, FKV_K4_WHOLE,
 * FKV_SOLO_SMALL, FKV_SOLO_PIECE, FKV_SOLO_WHOLE, FKV_PIECE_COST,
 * FKV_PAIR_PIECE, FKV_SM_PAIRING, FKV_HYBRID_SAVING; chunk <= 0: none). */
typedef struct {
  int32_t sms, ctas_coop, ctas_wide, ctas_solo;
  int32_t mode;                  /* 0 auto, 1 coop, 2 wide, 3 solo */
  int32_t whole;                 /* -1 auto, 0 never, 1 always */
  int32_t solo_small, solo_piece, solo_whole;  /* solo_piece / solo_whole: -1 = default */
  int32_t piece_cost, sm_pairing, chunk;
  double pair_piece;
  double hybrid_saving_us;       /* cut a whole-schedule segment only when that saves more (us) */
} fkv_sched_params;

/* Outputs (int32): item_seg / item_t0 / item_t1 / work_list [n_items],
 * seg_item_ptr [n_seg + 1], warp_ptr [busy + 1], table [rows * K * 8]
 * (fkv_work_t rows); out_sizes = {n_items, busy, rows, K, flags}.  Buffers
 * hold item_cap items, worker_cap workers and table_cap table ints; too
 * small: FKV_ERR_INVALID with the needed sizes in out_sizes. */
int fkv_plan_schedule(const int64_t* seg_len, const int64_t* seg_row0, const int64_t* seg_qrow,
                      const int64_t* seg_out_row, int32_t n_seg, const fkv_sched_params* prm,
                      int32_t item_cap, int32_t worker_cap, int32_t table_cap, int32_t* item_seg,
                      int32_t* item_t0, int32_t* item_t1, int32_t* seg_item_ptr, int32_t* warp_ptr,
                      int32_t* work_list, int32_t* table, int32_t* out_sizes);

/* A layer cache's whole device table set, planned (as fkv_plan_schedule)
 * and packed into one int32 buffer for one host-to-device copy.  Part i
 * occupies words [part_off[i], part_off[i+1]) (16-byte aligned; the part's
 * own length is below that bound):
 *   SEG_LEN, SEG_QROW, SEG_OUT_ROW [n_seg]; ITEM_SEG, ITEM_T0, ITEM_T1 [n_items];
 *   SEG_ITEM_PTR [n_seg + 1]; SRC_IDX [n_items] (0..n_items-1, K5's source rows);
 *   WARP_PTR [busy + 1]; WORK_LIST [n_items]; WORK [rows * K * 8] (fkv_work_t);
 *   SEG_CAP [n_seg] (null seg_cap: seg_len); APPEND_SRC [n_seg] (null: -1);
 *   LAST_PIECE [n_seg] (flat work index of each segment's last piece);
 *   COUNTERS [max(n_items, 1)] and OVERFLOW [1] (zero);
 *   SEG_ROW0 [n_seg] as int64 (2 words each).
 * part_off has FKV_CT_PARTS + 1 entries, the last = words used; a buffer
 * shorter than that: FKV_ERR_INVALID with part_off filled.  out_sizes as
 * fkv_plan_schedule. */
#define FKV_CT_SEG_LEN 0
#define FKV_CT_SEG_QROW 1
#define FKV_CT_SEG_OUT_ROW 2
#define FKV_CT_ITEM_SEG 3
#define FKV_CT_ITEM_T0 4
#define FKV_CT_ITEM_T1 5
#define FKV_CT_SEG_ITEM_PTR 6
#define FKV_CT_SRC_IDX 7
#define FKV_CT_WARP_PTR 8
#define FKV_CT_WORK_LIST 9
#define FKV_CT_WORK 10
#define FKV_CT_SEG_CAP 11
#define FKV_CT_APPEND_SRC 12
#define FKV_CT_LAST_PIECE 13
#define FKV_CT_COUNTERS 14
#define FKV_CT_OVERFLOW 15
#define FKV_CT_SEG_ROW0 16
#define FKV_CT_PARTS 17
int fkv_cache_tables(const int64_t* seg_len, const int64_t* seg_row0, const int64_t* seg_qrow,
                     const int64_t* seg_out_row, const int64_t* seg_cap, const int64_t* append_src,
                     int32_t n_seg, const fkv_sched_params* prm, int32_t* buf, int64_t buf_words,
                     int64_t* part_off, int32_t* out_sizes);

/* Exchange records (the per-layer all-gather payload; "XREC"): a block of
 * `slots` rows of `group` heads =
 *     bf16 o[slots * group][128]   (256 bytes per head row)
 *     f32  lse[slots * group]
 * FKV_XREC_BYTES(slots, group) bytes.  Segment s of a rank writes rows
 * out_row .. out_row + group - 1 (out_row = s * group) of its block; in a
 * receive area rank r's block starts at r * FKV_XREC_BYTES. */
#define FKV_XREC_BYTES(slots, group) ((int64_t)(slots) * (group) * (FKV_HEAD_DIM * 2 + 4))

/*   q            bf16 [*, 128]   query rows
 *   k, v         bf16 [rows,128] swizzled cache rows (layout above)
 *   work         fkv_work_t [n_workers][work_k], 1 <= work_k <= FKV_MAX_WORK
 *   part         f32 [n_items, group, FKV_REC]  partial records of split
 *                segments: softmax-normalised o[128] and lse = natural-log
 *                sum-exp of the scaled scores
 *   counters     int32 [n_items] arrival counters, zero on entry; left zero on exit
 * With all of out_bf16 / out_xrec / out_lse NULL every piece just writes its
 * partial record (split-K partials).  Otherwise a single-piece segment writes
 * its rows directly and the last warp to finish a piece of a split segment
 * merges the segment's records by log-sum-exp; both write rows out_row + h
 * (h < group) of out_bf16 (bf16 [*,128]), the exchange block out_xrec
 * (XREC layout, xrec_slots rows of `group` heads) and/or out_lse (f32 [*]),
 * with 16-byte stores -- one launch per layer.  Outputs 16-byte aligned.
 * group (= Hq/Hkv) must be 4 or 8; softmax scale = sm_scale.
 * Nothing in the reference is replaced (it has no decode); its cost model of
 * this kernel is reference latency.py:85-91 (predict_compute). */
/* Persistent CTAs per SM of the schedule selected by `flags` (the planner
 * sizes the work table with SMs x this many rows: one per co-resident CTA). */
int fkv_decode_ctas_per_sm(int32_t flags);

int fkv_decode(const void* q, const void* k, const void* v, const fkv_work_t* work,
               int32_t work_k, int32_t n_workers, int32_t n_items, int32_t group, int32_t flags,
               float sm_scale, float* part, int32_t* counters, void* out_bf16, void* out_xrec,
               int32_t xrec_slots, float* out_lse, void* stream);

/* K5: log-sum-exp merge of exchange records.  xrec = blocks of xrec_slots
 * rows (block r at r * FKV_XREC_BYTES(xrec_slots, group)); record index
 * i = r * xrec_slots + slot.  Output group g merges the records
 * src_idx[grp_ptr[g] .. grp_ptr[g+1]) and writes, for heads h < group, row
 * out_row[g] + h of out_bf16 (bf16 [*,128]) and/or out_lse (f32 [*]).
 * This is the DP-copy -> head merge after the all-gather; the all-gather
 * stands in for the reference's modeled allreduce (reference
 * latency.py:94-101, simulate.py:132-133). */
int fkv_merge_lse(const void* xrec, int32_t xrec_slots, const int32_t* grp_ptr,
                  const int32_t* src_idx, const int32_t* out_row, int32_t n_groups, int32_t group,
                  void* out_bf16, float* out_lse, void* stream);

/* Fused NVLink all-gather records ("XLL", a low-latency format in the style
 * of NCCL's LL protocol): the rows of an XREC block, but every 16-byte unit
 * carries 8 payload bytes and the exchange epoch twice, {w0, epoch, w1, epoch},
 * written with one 16-byte store.  A reader that sees both epoch words of a
 * unit equal to the expected epoch has that unit's payload -- no fence, no
 * completion flag, no system-scope release (a MEMBAR.SYS costs ~10 us per
 * launch on B200).  Head row = 32 units of o (4 bf16 columns each) + one unit
 * {lse, epoch, 0, epoch} = FKV_XLL_ROW_BYTES; block = slots * group rows. */
#define FKV_XLL_ROW_BYTES 528
#define FKV_XLL_BYTES(slots, group) ((int64_t)(slots) * (group) * FKV_XLL_ROW_BYTES)

/* Fused NVLink all-gather variant of fkv_decode (same work table).  Every
 * segment's final record is written in XLL format to all n_rec destinations
 * (this rank's block of each peer's receive area, mapped with fkv_ipc_open;
 * 16-byte P2P stores over NVLink) instead of one local block, tagged with
 * epoch = epoch_ctr[0] + 1 (read after the preceding grid completes: the
 * previous layer's fkv_merge_wait advanced it).  Replaces NCCL all_gather
 * for the per-layer exchange; the reference models this step as an
 * allreduce (reference latency.py:94-101). */
int fkv_decode_exchange(const void* q, const void* k, const void* v, const fkv_work_t* work,
                        int32_t work_k, int32_t n_workers, int32_t n_items, int32_t group,
                        int32_t flags, float sm_scale, float* part, int32_t* counters, void* out_bf16,
                        void* const* out_xrecs, int32_t n_rec, int32_t xrec_slots, float* out_lse,
                        const int32_t* epoch_ctr, void* stream);

/* fkv_merge_lse over a receive area of XLL blocks (block r at
 * r * FKV_XLL_BYTES) with the consumer side of the fused all-gather: each
 * warp polls its records' units until they carry epoch_ctr[0] + 1, merges,
 * and the last CTA advances epoch_ctr[0] (epoch_ctr[1] is its arrival
 * counter, zero between launches).  epoch_ctr == NULL: fkv_merge_lse. */
int fkv_merge_wait(const void* xrec, int32_t xrec_slots, const int32_t* grp_ptr,
                   const int32_t* src_idx, const int32_t* out_row, int32_t n_groups, int32_t group,
                   void* out_bf16, float* out_lse, int32_t* epoch_ctr, void* stream);

/* Device memory that can be shared with the other GPUs of the node. */
int fkv_dev_alloc(int64_t bytes, void** out_ptr);
int fkv_dev_free(void* ptr);
int fkv_ipc_get(void* dev_ptr, void* handle /* 64 bytes */);
int fkv_ipc_open(const void* handle, void** out_ptr);
int fkv_ipc_close(void* ptr);

/* Device address of pinned host memory (a kernel output the host reads
 * without a copy, e.g. fkv_snapkv_select's budgets). */
int fkv_host_device_ptr(void* host_ptr, void** out_ptr);

/* ------------------------------------------- B3 compression (prefill) -- */

/* K1: Ada-SnapKV observation-window scores (two tcgen05/TMEM/TMA passes +
 * max-pool).  q_win bf16 [batch, hq, window, 128], k bf16 [batch, hkv, T, 128];
 * scores f32 [batch, hkv, T - window]:
 *   s[t] = maxpool_{pool_k}( (1/G) sum_{g,i} softmax_t(q_{g,i} . k_t * sm_scale) ),
 * causal inside the window.  G*window must be 128 or 256.  workspace: device
 * bytes >= fkv_score_workspace_bytes(...).  No reference implementation
 * (the paper used KVPress SnapKV). */
int64_t fkv_score_workspace_bytes(int32_t batch, int32_t hkv, int32_t T, int32_t window,
                                  int32_t group);
int fkv_snapkv_score(const void* q_win, const void* k, int32_t batch, int32_t hq, int32_t hkv,
                     int32_t T, int32_t window, int32_t pool_k, float sm_scale, float* scores,
                     void* workspace, void* stream);

/* K1 + A18 + K2 in one persistent cooperative launch at any batch: the
 * scores above, then the Ada budget split and the per-head top-k selection
 * by a grid-wide radix search over the pooled scores (every CTA histograms
 * its own key range; per-pass digit histograms meet in the workspace between
 * grid barriers).  Outputs are identical to fkv_snapkv_score followed by
 * fkv_ada_select (budgets int32 [batch, hkv], offsets int64 [batch*hkv + 1]
 * with request b starting at b*hkv*budget, idx int32 [batch*hkv*budget]).
 * Same workspace size as fkv_snapkv_score.  Hkv > 16, or more than 14 heads
 * per SM, run as those two launches.  `budgets` may point to pinned host
 * memory (device-addressable under unified addressing): the launch only
 * writes it, so the host reads a layer's budgets once the launch has ended
 * without a copy (ops.compress_stack). */
int fkv_snapkv_select(const void* q_win, const void* k, int32_t batch, int32_t hq, int32_t hkv,
                      int32_t T, int32_t window, int32_t pool_k, float sm_scale, int32_t budget,
                      int32_t floor_k, float* scores, int32_t* budgets, int64_t* offsets,
                      int32_t* idx, void* workspace, void* stream);

/* A18: Ada cross-head budget split.  scores f32 [batch, hkv, n] -> budgets
 * int32 [batch, hkv] = window + floor_k + (# of the head's tokens in the
 * global top-(hkv*(budget-window-floor_k)) of the non-floor scores), order
 * (score desc, head asc, token asc); floor = per-head top-floor_k by (score
 * desc, token asc).  Every row sums to hkv*budget.  Same grid-wide kernel
 * as fkv_ada_select (budgets only); workspace as there.  Hkv <= 16. */
int fkv_ada_budgets(const float* scores, int32_t batch, int32_t hkv, int32_t n, int32_t budget,
                    int32_t window, int32_t floor_k, int32_t* budgets, void* workspace,
                    void* stream);

/* K2: per-head top-(budgets - window) by (score desc, token asc), written
 * ascending at idx[offsets[bh]..], followed by the window tokens n..n+window-1;
 * offsets int64 [batch*hkv + 1] is the exclusive prefix sum of budgets (any
 * budgets >= window).  Same grid-wide kernel as fkv_ada_select (each head's
 * own radix search); workspace as there.  Hkv <= 16. */
int fkv_topk_select(const float* scores, const int32_t* budgets, int32_t batch, int32_t hkv,
                    int32_t n, int32_t window, int64_t* offsets, int32_t* idx, void* workspace,
                    void* stream);

/* A18 + K2 fused: one cooperative launch over every (request, head) -- the
 * keys of each head are cut into chunks dealt out to persistent CTAs, a
 * four-pass radix search over the 32-bit score finds every request's Ada
 * threshold and every head's own floor threshold at once (grid barriers
 * between passes), and each CTA writes its chunks' chosen tokens.  Budgets,
 * offsets (request b starts at b*hkv*budget) and the ascending index lists
 * are identical to fkv_ada_budgets followed by fkv_topk_select.  Hkv <= 16.
 * workspace: device bytes >= fkv_ada_select_workspace_bytes(batch, hkv, n);
 * no initial contents required (reset inside, stream-ordered). */
int64_t fkv_ada_select_workspace_bytes(int32_t batch, int32_t hkv, int32_t n);
int fkv_ada_select(const float* scores, int32_t batch, int32_t hkv, int32_t n, int32_t budget,
                   int32_t window, int32_t floor_k, int32_t* budgets, int64_t* offsets,
                   int32_t* idx, void* workspace, void* stream);

/* K3: compaction.  For each destination segment s, rows j in [seg_lo, seg_hi)
 * of head seg_bh[s]'s selection are copied from k_src/v_src (bf16
 * [batch*hkv, T, 128]) to cache rows seg_row0[s] + (j - seg_lo), swizzled;
 * zero_pad != 0 also zeroes the rows up to the next FKV_PAGE boundary.
 * max_tokens >= max(seg_hi - seg_lo) sizes the grid (64 rows per CTA). */
int fkv_compact(const void* k_src, const void* v_src, int32_t T, int32_t n_segments,
                const int64_t* offsets, const int32_t* idx, const int32_t* seg_bh,
                const int32_t* seg_lo, const int32_t* seg_hi, const int64_t* seg_row0,
                int32_t zero_pad, int32_t max_tokens, void* k_dst, void* v_dst, void* stream);

/* Decode-time append: segment s with src_row[s] >= 0 (it owns the end of its
 * head's token axis) receives row src_row[s] of k_new / v_new (bf16 [*,128])
 * at cache row seg_row0[s] + seg_len[s] (swizzled); seg_len[s] and the n_tok
 * of its last piece work[last_piece[s]] (flat fkv_work_t index) grow by one.
 * Segments already at seg_cap[s] rows are skipped and counted in *overflow.
 * One launch per layer and step; no host synchronisation. */
int fkv_append(const void* k_new, const void* v_new, const int32_t* src_row,
               const int64_t* seg_row0, int32_t* seg_len, const int32_t* seg_cap, void* work,
               const int32_t* last_piece, int32_t n_segments, int32_t* overflow, void* k_dst,
               void* v_dst, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FAIRKV_H_ */

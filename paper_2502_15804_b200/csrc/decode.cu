// K4 + fused K5: CTA-persistent split-KV decode attention over the ragged,
// swizzled, page-aligned compressed cache, with the log-sum-exp merges.
//
// No reference implementation exists; the reference only models
// this kernel's time as c0 + c1*B + c2*C + c3*B*C (pkg/src/headbalance/latency.py:85-91).
//
// Design:
//  * static, host-built schedule: the concatenated 16-token tile stream of all
//    segments is cut into equal ranges, one per persistent CTA (two per SM), so
//    every CTA streams the same number of bytes; a CTA's range is a list of
//    *pieces* (sub-ranges of segments) described by 32-byte descriptors that
//    the CTA reads with one coalesced load at entry;
//  * inside a CTA the four warps share each piece: the piece is cut into
//    rounds of two tiles and warp j takes rounds j, j+4, ...  Every warp runs
//    its own 3-stage TMA bulk-copy ring (cp.async.bulk + mbarrier, 8 KiB K+V
//    tiles) that streams across piece boundaries, so four independent
//    dependency chains hide each other's latency even when the whole cache is
//    only a few MB (small TP shards);
//  * at the end of a piece warps 1-3 hand their (m, l, acc) state to warp 0
//    through shared memory (named barriers, no global traffic) and warp 0
//    combines, normalises and writes the piece's output;
//  * the cache rows are stored pre-swizzled in HBM, so a 1-D bulk copy lands
//    a bank-conflict-free tile for ldmatrix -- no tensor map, no address math;
//  * GQA: every K/V tile is read once for all G query heads.  S^T = K Q^T
//    (m16n8k16: 16 tokens x 8 heads, no padding waste for G=8), online
//    softmax per head column (warp-shuffle max), P^T via movmatrix, then
//    O^T += V^T P^T with ldmatrix.trans on the V tile;
//  * a piece's (o, lse) goes straight to its output rows when the segment is
//    one piece; otherwise to a partial record, and the CTA that finishes the
//    segment's last piece merges its records (K5 fused).
#include <cuda_bf16.h>
#include <math_constants.h>

#include <cstdlib>

#include "common.cuh"

namespace fkv {
namespace {

// CTA shapes (MODE).  Cooperative schedules: warp 0 only combines /
// finalises (records, atomics, segment merges) while warps 1..W-1 stream:
//   0 "coop"  W = 4, 4-stage rings, two CTAs per SM (96 KiB of ring each);
//   2 "wide"  W = 8, 3-stage rings, one CTA per SM (168 KiB of ring) -- for
//             caches with few segments (TP-sharded ranks), where 7 streams
//             per piece beat 3.
// 1 "solo": per-warp schedule, 4 warps all streaming, 3 stages, two per SM.
constexpr int kTileTok = 16;
constexpr int kTileBytes = kTileTok * FKV_HEAD_DIM * 2;  // 4 KiB per K or V tile
template <int MODE>
struct Shape {
  static constexpr int W = MODE == 2 ? 8 : 4;                        // warps per CTA
  static constexpr int S = MODE == 1 ? W : W - 1;                    // streaming warps
  static constexpr int NS = MODE == 0 ? 4 : 3;                       // ring stages per streamer
  static constexpr int kSmem = S * NS * 2 * kTileBytes;              // dynamic smem (ring)
  static constexpr int kCtasPerSm = MODE == 2 ? 1 : 2;
};
constexpr int kMergeMax = FKV_MAX_PIECES;                      // max pieces per segment
constexpr int kXch = 36;  // floats per lane handed to warp 0: m0 m1 l0 l1 acc[32]
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

struct DecodeParams {
  const __nv_bfloat16* q;
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  const fkv_work_t* work;  // [n_workers][work_k] pieces per persistent CTA
  int work_k, n_workers;
  float scale_log2;
  float* part;        // [n_items, G, FKV_REC] partial records (multi-piece segments)
  int32_t* counters;  // [n_items] arrival counter at each segment's first piece; zero between launches
  __nv_bfloat16* out_bf16;
  // exchange-record destinations (FKV_XREC layout): a local send block, or
  // this rank's block in every peer's receive area (fused NVLink all-gather)
  uint8_t* out_rec[FKV_MAX_PEERS];
  int n_rec;
  int64_t rec_lse_off;  // bytes from a block's start to its lse array
  float* out_lse;
  const int32_t* epoch_ctr;  // non-null: out_rec are XLL blocks tagged epoch_ctr[0] + 1
  int after_wait;  // FKV_DECODE_AFTER_WAIT: no global read before griddepcontrol.wait
  int stamp_slot;  // PROBE 3: stamp block of this launch (0..3)
};

template <int W>
struct __align__(16) DecodeShared {
  fkv_work_t tab[FKV_MAX_WORK];
  uint64_t bars[W][4];
  float xch[W - 1][kXch][32];  // warps 1..W-1 -> warp 0 piece state, lane-contiguous
  float scratch[kMergeMax * 8];     // global merge weights
  int32_t fin_i0, fin_n_it, fin_orow;  // deferred merge of the CTA's last piece (n_it 0 = none)
};

// ---- segment outputs: o rows (bf16, 16-byte stores) and lse, to the local
// outputs and every exchange-record destination.  Plain XREC blocks: row r
// at r * 256 bytes, its lse at rec_lse_off + 4 r; XLL blocks (fused
// exchange, ep != 0): row r at r * FKV_XLL_ROW_BYTES, 16-byte units
// {w0, ep, w1, ep} -- one P2P store per 8 payload bytes (include/fairkv.h).
__device__ __forceinline__ void st_ll(uint8_t* a, uint32_t w0, uint32_t w1, uint32_t ep) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(a), "r"(w0), "r"(ep), "r"(w1),
               "r"(ep)
               : "memory");
}
__device__ __forceinline__ void store_o16(const DecodeParams& p, uint32_t ep, int64_t row, int col, int4 v) {
  if (p.out_bf16) *reinterpret_cast<int4*>(p.out_bf16 + row * FKV_HEAD_DIM + col) = v;
#pragma unroll 1
  for (int j = 0; j < p.n_rec; ++j) {
    if (ep) {
      uint8_t* u = p.out_rec[j] + row * FKV_XLL_ROW_BYTES + col * 4;  // unit col / 4
      st_ll(u, v.x, v.y, ep);
      st_ll(u + 16, v.z, v.w, ep);
    } else {
      *reinterpret_cast<int4*>(p.out_rec[j] + (row * FKV_HEAD_DIM + col) * 2) = v;
    }
  }
}
__device__ __forceinline__ void store_lse1(const DecodeParams& p, uint32_t ep, int64_t row, float l) {
  if (p.out_lse) p.out_lse[row] = l;
#pragma unroll 1
  for (int j = 0; j < p.n_rec; ++j) {
    if (ep)
      st_ll(p.out_rec[j] + row * FKV_XLL_ROW_BYTES + 32 * 16, __float_as_uint(l), 0u, ep);
    else
      reinterpret_cast<float*>(p.out_rec[j] + p.rec_lse_off)[row] = l;
  }
}
__device__ __forceinline__ void store_lse4(const DecodeParams& p, uint32_t ep, int64_t row, float4 l) {
  if (p.out_lse) *reinterpret_cast<float4*>(p.out_lse + row) = l;
#pragma unroll 1
  for (int j = 0; j < p.n_rec; ++j) {
    if (ep) {
      uint8_t* u = p.out_rec[j] + row * FKV_XLL_ROW_BYTES + 32 * 16;
      st_ll(u, __float_as_uint(l.x), 0u, ep);
      st_ll(u + FKV_XLL_ROW_BYTES, __float_as_uint(l.y), 0u, ep);
      st_ll(u + 2 * FKV_XLL_ROW_BYTES, __float_as_uint(l.z), 0u, ep);
      st_ll(u + 3 * FKV_XLL_ROW_BYTES, __float_as_uint(l.w), 0u, ep);
    } else {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out_rec[j] + p.rec_lse_off) + row) = l;
    }
  }
}

__device__ __forceinline__ uint2 pack_bf16x4(float4 v) {
  return make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
}

// One head row held as a float4 of columns 4*lane .. +3 by every lane:
// neighbouring lanes pair up so even lanes store 16 bytes (8 columns).
__device__ __forceinline__ void emit_row_lanes(const DecodeParams& p, uint32_t ep, int64_t row, float4 o,
                                               int lane) {
  const uint2 w = pack_bf16x4(o);
  const uint32_t hx = __shfl_down_sync(0xffffffffu, w.x, 1), hy = __shfl_down_sync(0xffffffffu, w.y, 1);
  if ((lane & 1) == 0) store_o16(p, ep, row, 4 * lane, make_int4(w.x, w.y, hx, hy));
}

// lse of heads 0..G-1 held by lanes 0..G-1 -> float4 stores by lanes 0 (and 1).
template <int G>
__device__ __forceinline__ void emit_lse_lanes(const DecodeParams& p, uint32_t ep, int64_t row, float l,
                                               int lane) {
  const int b = 4 * (lane & 1);
  const float a0 = __shfl_sync(0xffffffffu, l, b), a1 = __shfl_sync(0xffffffffu, l, b + 1);
  const float a2 = __shfl_sync(0xffffffffu, l, b + 2), a3 = __shfl_sync(0xffffffffu, l, b + 3);
  if (lane < G / 4) store_lse4(p, ep, row + b, make_float4(a0, a1, a2, a3));
}

// The finalised o of one whole segment, in the mma accumulator layout
// (acc[dt][e]: column 16 dt + (lane >> 2) (+8 for e >= 2) of head
// 2 (lane & 3) (+1 for odd e); inv = 1 / softmax denominator per head) ->
// G rows of bf16 with 16-byte stores.  movmatrix turns each 8-column block
// into "lane L holds 2 columns of head L >> 2"; a 4x4 word transpose among
// the 4 lanes of a head then gives every lane 8 consecutive columns.
template <int G>
__device__ __forceinline__ void emit_acc(const DecodeParams& p, uint32_t ep, int64_t orow,
                                         const float (&acc)[8][4], float inv0, float inv1, int lane) {
  uint32_t t[16];  // t[c]: this lane's word of 8-column chunk c of head lane >> 2
#pragma unroll
  for (int dt = 0; dt < 8; ++dt) {
    t[2 * dt] = movmatrix_trans(pack_bf16x2(acc[dt][0] * inv0, acc[dt][1] * inv1));
    t[2 * dt + 1] = movmatrix_trans(pack_bf16x2(acc[dt][2] * inv0, acc[dt][3] * inv1));
  }
  const int j = lane & 3, h = lane >> 2;
#pragma unroll
  for (int m = 0; m < 4; ++m) {  // chunks 4m .. 4m+3: lane j collects chunk 4m + j
    uint32_t w[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int si = (j - r) & 3;  // send my word of chunk 4m + si to lane (j - r) & 3
      const uint32_t send = si == 0 ? t[4 * m] : si == 1 ? t[4 * m + 1] : si == 2 ? t[4 * m + 2] : t[4 * m + 3];
      const uint32_t got = __shfl_sync(0xffffffffu, send, (lane & ~3) | ((j + r) & 3));
      const int k = (j + r) & 3;  // ... and receive word k (= source lane) of chunk 4m + j
#pragma unroll
      for (int x = 0; x < 4; ++x)
        if (k == x) w[x] = got;
    }
    if (h < G) store_o16(p, ep, orow + h, 8 * (4 * m + j), make_int4(w[0], w[1], w[2], w[3]));
  }
}

__device__ __forceinline__ int atom_add_acq_rel(int32_t* addr, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(addr), "r"(v)
               : "memory");
  return old;
}

template <int W>
__device__ __forceinline__ void named_sync(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(W * 32) : "memory");
}
template <int W>
__device__ __forceinline__ void named_arrive(int id) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "n"(W * 32) : "memory");
}

// Round ownership inside a CTA (cooperative schedule).  Rounds (two tiles
// each) are numbered across the CTA's pieces and dealt round robin to the
// streaming warps 1..W-1; warp 0 owns none.
constexpr int kNoRound = 0x7fffffff;
template <int W>
__device__ __forceinline__ int first_round(int warp, int g0) {  // first owned round >= g0
  if (warp == 0) return kNoRound;
  return g0 + ((warp - 1 - g0 % (W - 1)) + (W - 1)) % (W - 1);
}
template <int W>
__device__ __forceinline__ int next_round(int, int r) {
  return r + (W - 1);
}

__device__ __forceinline__ int piece_tiles(const fkv_work_t& d) {
  return (d.n_tok + kTileTok - 1) / kTileTok;
}

// PROBE (diagnostics only, fkv__decode_probe): 1 = stream the tiles without
// computing, 2 = compute on whatever the ring holds without loading,
// 3 = full kernel + per-CTA %globaltimer stamps in g_stamps.
__device__ unsigned long long g_stamps[4 * 1024 * 16];  // [slot][CTA][16]
__device__ __forceinline__ void stamp(int PROBE_, int slot, int i) {
  if (PROBE_ == 3 && (threadIdx.x & 31) == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_stamps[(slot * 1024 + blockIdx.x) * 16 + i] = t;
  }
}
// SOLO (small shards): every warp streams its own pieces start to finish and
// finalises them itself -- no hand-over -- so a short schedule keeps four
// independent tile streams per CTA; a piece's owner warp is n_it >> 16.
template <int G, int PROBE = 0, int MODE = 0>
__global__ void __launch_bounds__(Shape<MODE>::W * 32, Shape<MODE>::kCtasPerSm)
    decode_kernel(const DecodeParams p) {
  constexpr bool SOLO = MODE == 1;
  constexpr int W = Shape<MODE>::W;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ DecodeShared<W> sh;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr int NS = Shape<MODE>::NS;   // ring stages per streaming warp
  constexpr bool kCombiner = !SOLO;     // warp 0 only combines
  uint8_t* ring = smem + (kCombiner ? (warp > 0 ? warp - 1 : 0) : warp) * NS * 2 * kTileBytes;
  uint64_t* wbars = sh.bars[warp];
  const fkv_work_t* tab = sh.tab;
  if (warp == 0) stamp(PROBE, p.stamp_slot, 12);  // entry
  if (PROBE == 3 && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_stamps[(p.stamp_slot * 1024 + blockIdx.x) * 16] = smid;
  }

  // A cache written by the preceding kernel (append / compact): its rows and
  // work table are only guaranteed visible after the wait.
  if (p.after_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  // The CTA's whole piece list in one coalesced load (lane j <- piece j);
  // everything the kernel needs per piece is in its 32-byte descriptor, so
  // the first TMA is one dependent global load away from kernel entry.
  if (warp == 0) {
    if (lane < p.work_k) {
      const int4* src = reinterpret_cast<const int4*>(p.work + static_cast<int64_t>(blockIdx.x) * p.work_k + lane);
      const int4 a = __ldg(src), b = __ldg(src + 1);
      reinterpret_cast<int4*>(sh.tab + lane)[0] = a;
      reinterpret_cast<int4*>(sh.tab + lane)[1] = b;
    } else {
      sh.tab[lane].n_it = 0;  // terminator
    }
  }
  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&wbars[s], 1);
    fence_mbar_init();
  }
  if (threadIdx.x == 0) sh.fin_n_it = 0;
  __syncthreads();

  // ---- producer: this warp's rounds (two tiles each) of every piece, in the
  // CTA-wide round numbering (first_round / next_round)
  auto mine = [&](int pc) { return !SOLO || (tab[pc].n_it >> 16) == warp; };
  int p_pc = 0, p_G = 0, p_half = 0;  // piece, its first round, tile of the round
  int p_r = SOLO ? 0 : first_round<W>(warp, 0);  // next owned round (SOLO: round within the piece)
  uint32_t p_seq = 0, c_seq = 0;
  int p_s = 0;
  bool p_done = kCombiner && warp == 0;  // the combiner warp streams nothing
  auto refill = [&]() {
    while (!p_done && p_seq - c_seq < static_cast<uint32_t>(NS)) {
      if (p_pc >= FKV_MAX_WORK || tab[p_pc].n_it == 0) {
        p_done = true;
        break;
      }
      if (SOLO && !mine(p_pc)) {
        ++p_pc;
        continue;
      }
      const int nt = piece_tiles(tab[p_pc]);
      const int nr = (nt + 1) >> 1;
      if (SOLO && p_r >= nr) {
        ++p_pc;
        p_r = 0;
        p_half = 0;
        continue;
      }
      if (!SOLO && p_r >= p_G + nr) {
        p_G += nr;
        ++p_pc;
        p_half = 0;
        continue;
      }
      const int tile = 2 * (SOLO ? p_r : p_r - p_G) + p_half;
      if (tile >= nt) {  // odd tail: one-tile round
        p_r = SOLO ? p_r + 1 : next_round<W>(warp, p_r);
        p_half = 0;
        continue;
      }
      if (lane == 0 && PROBE == 2) {
        mbar_arrive_expect_tx(&wbars[p_s], 0);
      } else if (lane == 0) {
        const int64_t row = tab[p_pc].row0 + kTileTok * tile;
        uint8_t* dst = ring + p_s * 2 * kTileBytes;
        mbar_arrive_expect_tx(&wbars[p_s], 2 * kTileBytes);
        bulk_g2s(dst, p.k + row * FKV_HEAD_DIM, kTileBytes, &wbars[p_s]);
        bulk_g2s(dst + kTileBytes, p.v + row * FKV_HEAD_DIM, kTileBytes, &wbars[p_s]);
      }
      ++p_seq;
      if (++p_s == NS) p_s = 0;
      if (++p_half == 2) {
        p_half = 0;
        p_r = SOLO ? p_r + 1 : next_round<W>(warp, p_r);
      }
    }
  };
  refill();

  const int mi = lane >> 3, ri = lane & 7;
  const int h0 = 2 * (lane & 3), h1 = h0 + 1;
  const int dr = lane >> 2;
  const bool fused = p.out_bf16 || p.n_rec > 0 || p.out_lse;

  uint32_t qn[8][2];  // q fragments of the next piece, loaded one piece ahead
  auto next_mine = [&](int pc) {
    while (SOLO && pc < FKV_MAX_WORK && tab[pc].n_it != 0 && !mine(pc)) ++pc;
    return pc;
  };
  auto load_q = [&](int pc) {
    const int n = lane >> 2, kq = 2 * (lane & 3);
    pc = next_mine(pc);
    if (pc < FKV_MAX_WORK && tab[pc].n_it != 0 && n < G) {
      const __nv_bfloat16* qr = p.q + static_cast<int64_t>(tab[pc].qrow + n) * FKV_HEAD_DIM;
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
  // reads, the first K/V tiles in flight) touches only the cache, static
  // between steps unless FKV_DECODE_AFTER_WAIT, and overlaps the previous
  // kernel's tail; q and every global write come after the previous grid has
  // completed.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  // exchange epoch of this layer: the previous merge_wait advanced the counter
  const uint32_t ep = p.epoch_ctr ? static_cast<uint32_t>(*reinterpret_cast<const volatile int32_t*>(p.epoch_ctr)) + 1u : 0u;
  load_q(0);
  if (warp == 0) stamp(PROBE, p.stamp_slot, 1);
  if (!SOLO && warp == 0) named_arrive<W>(1);  // the hand-over slot starts free

  int c_s = 0;        // consumer stage
  uint32_t c_ph = 0;  // its mbarrier phase parity
  int G0 = 0;         // first round of the current piece
  int c_r = SOLO ? 0 : first_round<W>(warp, 0);  // next owned round
  for (int pc = 0; pc < FKV_MAX_WORK; ++pc) {
    fkv_work_t d = tab[pc];
    if (d.n_it == 0) break;
    if (SOLO && !mine(pc)) continue;
    d.n_it &= 0xffff;
    const int nt = piece_tiles(d);
    const int nr = (nt + 1) >> 1;
    if (SOLO) c_r = G0;  // every round of an owned piece

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

    // this warp's rounds of the piece: two independent S chains per round, one
    // softmax max/shuffle/rescale step and one ring hand-back per 32 tokens
    for (; c_r < G0 + nr; c_r = SOLO ? c_r + 1 : next_round<W>(warp, c_r)) {
      const int i = 2 * (c_r - G0);
      const bool two = i + 1 < nt;
      const int sA = c_s;
      const uint32_t phA = c_ph;
      if (++c_s == NS) c_s = 0, c_ph ^= 1u;
      const int sB = c_s;
      const uint32_t phB = c_ph;
      if (two && ++c_s == NS) c_s = 0, c_ph ^= 1u;
      mbar_wait(&wbars[sA], phA);
      if (two) mbar_wait(&wbars[sB], phB);
      if (warp == 0 && pc == 0) stamp(PROBE, p.stamp_slot, 2);
      if (PROBE == 1) {
        __syncwarp();
        c_seq += two ? 2u : 1u;
        refill();
        continue;
      }
      const uint32_t kA = smem_u32(ring + sA * 2 * kTileBytes), vA = kA + kTileBytes;
      const uint32_t kB = smem_u32(ring + sB * 2 * kTileBytes), vB = kB + kTileBytes;

      // S^T[16 tok x 8 heads] = K_tile . Q^T per tile: four independent
      // two-deep HMMA chains per tile (k16 slices kk = j, j+4), summed after
      float sa[4][4], sc[4][4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) sa[j][e] = sc[j][e] = 0.f;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        uint32_t a0, a1, a2, a3;
        ldmatrix_x4(kA + swz_off(ri + 8 * (mi & 1), 2 * kk + (mi >> 1)), a0, a1, a2, a3);
        mma_bf16_16816(sa[kk & 3], a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
      }
      if (two) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          uint32_t a0, a1, a2, a3;
          ldmatrix_x4(kB + swz_off(ri + 8 * (mi & 1), 2 * kk + (mi >> 1)), a0, a1, a2, a3);
          mma_bf16_16816(sc[kk & 3], a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
        }
      }
      float sb[4], sd[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        sb[e] = (sa[1][e] + sa[3][e]) + sa[2][e];
        sd[e] = (sc[1][e] + sc[3][e]) + sc[2][e];
      }
      const int ta = kTileTok * i + (lane >> 2);  // token of rows (lane>>2) / +8 within the piece
      const int tb = ta + kTileTok;
      const float s0 = ta < d.n_tok ? (sa[0][0] + sb[0]) * p.scale_log2 : -CUDART_INF_F;
      const float s1 = ta < d.n_tok ? (sa[0][1] + sb[1]) * p.scale_log2 : -CUDART_INF_F;
      const float s2 = ta + 8 < d.n_tok ? (sa[0][2] + sb[2]) * p.scale_log2 : -CUDART_INF_F;
      const float s3 = ta + 8 < d.n_tok ? (sa[0][3] + sb[3]) * p.scale_log2 : -CUDART_INF_F;
      const float s4 = tb < d.n_tok ? (sc[0][0] + sd[0]) * p.scale_log2 : -CUDART_INF_F;
      const float s5 = tb < d.n_tok ? (sc[0][1] + sd[1]) * p.scale_log2 : -CUDART_INF_F;
      const float s6 = tb + 8 < d.n_tok ? (sc[0][2] + sd[2]) * p.scale_log2 : -CUDART_INF_F;
      const float s7 = tb + 8 < d.n_tok ? (sc[0][3] + sd[3]) * p.scale_log2 : -CUDART_INF_F;
      float mx0 = fmaxf(fmaxf(s0, s2), fmaxf(s4, s6)), mx1 = fmaxf(fmaxf(s1, s3), fmaxf(s5, s7));
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
      const float p4 = fast_exp2(s4 - r0), p5 = fast_exp2(s5 - r1);
      const float p6 = fast_exp2(s6 - r0), p7 = fast_exp2(s7 - r1);
      l0 = l0 * c0 + ((p0 + p2) + (p4 + p6));
      l1 = l1 * c1 + ((p1 + p3) + (p5 + p7));
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
      const uint32_t pa0 = movmatrix_trans(pack_bf16x2(p0, p1));
      const uint32_t pa1 = movmatrix_trans(pack_bf16x2(p2, p3));
      // O^T[128 d x 8 heads] += V^T . P^T
#pragma unroll
      for (int dt = 0; dt < 8; ++dt) {
        uint32_t a0, a1, a2, a3;
        ldmatrix_x4_trans(vA + swz_off(ri + 8 * (mi >> 1), 2 * dt + (mi & 1)), a0, a1, a2, a3);
        mma_bf16_16816(acc[dt], a0, a1, a2, a3, pa0, pa1);
      }
      if (two) {
        const uint32_t pc0 = movmatrix_trans(pack_bf16x2(p4, p5));
        const uint32_t pc1 = movmatrix_trans(pack_bf16x2(p6, p7));
#pragma unroll
        for (int dt = 0; dt < 8; ++dt) {
          uint32_t a0, a1, a2, a3;
          ldmatrix_x4_trans(vB + swz_off(ri + 8 * (mi >> 1), 2 * dt + (mi & 1)), a0, a1, a2, a3);
          mma_bf16_16816(acc[dt], a0, a1, a2, a3, pc0, pc1);
        }
      }
      __syncwarp();
      c_seq += two ? 2u : 1u;
      refill();
    }
    G0 += nr;

    load_q(pc + 1);  // overlaps the hand-over below
    const bool more = pc + 1 < FKV_MAX_WORK && tab[pc + 1].n_it != 0;

    if (kCombiner && !more) {
      // ---- the CTA's final piece: every warp is idle once it is streamed,
      // so all W warps combine it, each over its own column blocks (dt),
      // instead of warp 0 alone -- this combine sits on the launch's
      // critical path (small TP shards: one piece per CTA)
      if (warp != 0) {
        named_sync<W>(1);  // hand-over slot free
        float* x = &sh.xch[warp - 1][0][lane];
        x[0 * 32] = m0;
        x[1 * 32] = m1;
        x[2 * 32] = l0;
        x[3 * 32] = l1;
#pragma unroll
        for (int dt = 0; dt < 8; ++dt)
#pragma unroll
          for (int e = 0; e < 4; ++e) x[(4 + 4 * dt + e) * 32] = acc[dt][e];
      }
      named_sync<W>(2);  // every state in shared memory
      stamp(PROBE, p.stamp_slot, 4);
      constexpr int kDt = 8 / W;  // column blocks per warp
      float fm0 = -CUDART_INF_F, fm1 = -CUDART_INF_F, fl0 = 0.f, fl1 = 0.f;
      float fa[kDt][4];
#pragma unroll
      for (int k = 0; k < kDt; ++k) fa[k][0] = fa[k][1] = fa[k][2] = fa[k][3] = 0.f;
#pragma unroll 1
      for (int s = 0; s < W - 1; ++s) {
        const float* x = &sh.xch[s][0][lane];
        const float om0 = x[0], om1 = x[32], ol0 = x[64], ol1 = x[96];
        const float nm0 = fmaxf(fm0, om0), nm1 = fmaxf(fm1, om1);
        const float r0 = nm0 == -CUDART_INF_F ? 0.f : nm0;
        const float r1 = nm1 == -CUDART_INF_F ? 0.f : nm1;
        const float a0 = fast_exp2(fm0 - r0), b0 = fast_exp2(om0 - r0);
        const float a1 = fast_exp2(fm1 - r1), b1 = fast_exp2(om1 - r1);
        fl0 = fl0 * a0 + ol0 * b0;
        fl1 = fl1 * a1 + ol1 * b1;
        fm0 = nm0;
        fm1 = nm1;
#pragma unroll
        for (int k = 0; k < kDt; ++k) {
          const int dt = warp + k * W;
          fa[k][0] = fa[k][0] * a0 + x[(4 + 4 * dt + 0) * 32] * b0;
          fa[k][1] = fa[k][1] * a1 + x[(4 + 4 * dt + 1) * 32] * b1;
          fa[k][2] = fa[k][2] * a0 + x[(4 + 4 * dt + 2) * 32] * b0;
          fa[k][3] = fa[k][3] * a1 + x[(4 + 4 * dt + 3) * 32] * b1;
        }
      }
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        fl0 += __shfl_xor_sync(0xffffffffu, fl0, off);
        fl1 += __shfl_xor_sync(0xffffffffu, fl1, off);
      }
      const float inv0 = fl0 > 0.f ? 1.f / fl0 : 0.f, inv1 = fl1 > 0.f ? 1.f / fl1 : 0.f;
      const float lse0 = fl0 > 0.f ? (fm0 + log2f(fl0)) * kLn2 : -CUDART_INF_F;
      const float lse1 = fl1 > 0.f ? (fm1 + log2f(fl1)) * kLn2 : -CUDART_INF_F;
      const int n_it = d.n_it;
      const int64_t orow = d.out_row;
      if (fused && n_it == 1) {
        // whole segment: bf16 rows staged in shared memory (the rings: every
        // copy issued was consumed, streaming is over), then 16-byte stores
        auto ostage = reinterpret_cast<__nv_bfloat16(*)[FKV_HEAD_DIM]>(smem);
#pragma unroll
        for (int k = 0; k < kDt; ++k) {
          const int d0 = 16 * (warp + k * W) + dr;
          if (h0 < G) {
            ostage[h0][d0] = __float2bfloat16_rn(fa[k][0] * inv0);
            ostage[h0][d0 + 8] = __float2bfloat16_rn(fa[k][2] * inv0);
          }
          if (h1 < G) {
            ostage[h1][d0] = __float2bfloat16_rn(fa[k][1] * inv1);
            ostage[h1][d0 + 8] = __float2bfloat16_rn(fa[k][3] * inv1);
          }
        }
        named_sync<W>(2);
        for (int c = threadIdx.x; c < G * 16; c += W * 32)
          store_o16(p, ep, orow + (c >> 4), 8 * (c & 15),
                    *reinterpret_cast<const int4*>(&ostage[c >> 4][8 * (c & 15)]));
        if (warp == 0) {
          const float la = __shfl_sync(0xffffffffu, lse0, (lane >> 1) & 3);
          const float lb = __shfl_sync(0xffffffffu, lse1, (lane >> 1) & 3);
          emit_lse_lanes<G>(p, ep, orow, (lane & 1) ? lb : la, lane);
        }
        break;
      }
      // split segment: this warp's columns of the piece's partial record
      float* rec = p.part + static_cast<int64_t>(d.rec) * G * FKV_REC;
#pragma unroll
      for (int k = 0; k < kDt; ++k) {
        const int d0 = 16 * (warp + k * W) + dr;
        if (h0 < G) {
          rec[h0 * FKV_REC + d0] = fa[k][0] * inv0;
          rec[h0 * FKV_REC + d0 + 8] = fa[k][2] * inv0;
        }
        if (h1 < G) {
          rec[h1 * FKV_REC + d0] = fa[k][1] * inv1;
          rec[h1 * FKV_REC + d0 + 8] = fa[k][3] * inv1;
        }
      }
      if (warp == 0 && lane < 4) {
        if (h0 < G) rec[h0 * FKV_REC + FKV_HEAD_DIM] = lse0;
        if (h1 < G) rec[h1 * FKV_REC + FKV_HEAD_DIM] = lse1;
      }
      if (!fused) break;
      // the barrier orders every warp's record stores before thread 0's
      // acq_rel arrival (cumulative release); the CTA finishing the segment's
      // last piece merges it after the loop, with all warps
      named_sync<W>(2);
      stamp(PROBE, p.stamp_slot, 6);
      if (threadIdx.x == 0 && atom_add_acq_rel(p.counters + d.i0, 1) == n_it - 1)
        sh.fin_i0 = d.i0, sh.fin_n_it = n_it, sh.fin_orow = static_cast<int32_t>(orow);
      stamp(PROBE, p.stamp_slot, 7);
      break;
    }

    // ---- hand the piece state to warp 0 (shared memory, named barriers):
    // bar 1 = slot free (warp 0 finished the previous piece), bar 2 = slot full
    if (!SOLO && warp != 0) {
      named_sync<W>(1);
      float* x = &sh.xch[warp - 1][0][lane];
      x[0 * 32] = m0;
      x[1 * 32] = m1;
      x[2 * 32] = l0;
      x[3 * 32] = l1;
#pragma unroll
      for (int dt = 0; dt < 8; ++dt)
#pragma unroll
        for (int e = 0; e < 4; ++e) x[(4 + 4 * dt + e) * 32] = acc[dt][e];
      named_arrive<W>(2);
      continue;
    }
    stamp(PROBE, p.stamp_slot, 3);
    if (!SOLO) named_sync<W>(2);
    stamp(PROBE, p.stamp_slot, 4);
    // warp 0: lane-wise online-softmax combine of the four warps' states
#pragma unroll 1
    for (int w = 0; w < (SOLO ? 0 : W - 1); ++w) {
      const float* x = &sh.xch[w][0][lane];
      const float om0 = x[0], om1 = x[32], ol0 = x[64], ol1 = x[96];
      const float nm0 = fmaxf(m0, om0), nm1 = fmaxf(m1, om1);
      const float r0 = nm0 == -CUDART_INF_F ? 0.f : nm0;
      const float r1 = nm1 == -CUDART_INF_F ? 0.f : nm1;
      const float a0 = fast_exp2(m0 - r0), b0 = fast_exp2(om0 - r0);
      const float a1 = fast_exp2(m1 - r1), b1 = fast_exp2(om1 - r1);
      l0 = l0 * a0 + ol0 * b0;
      l1 = l1 * a1 + ol1 * b1;
      m0 = nm0;
      m1 = nm1;
#pragma unroll
      for (int dt = 0; dt < 8; ++dt) {
        acc[dt][0] = acc[dt][0] * a0 + x[(4 + 4 * dt + 0) * 32] * b0;
        acc[dt][1] = acc[dt][1] * a1 + x[(4 + 4 * dt + 1) * 32] * b1;
        acc[dt][2] = acc[dt][2] * a0 + x[(4 + 4 * dt + 2) * 32] * b0;
        acc[dt][3] = acc[dt][3] * a1 + x[(4 + 4 * dt + 3) * 32] * b1;
      }
    }
    if (!SOLO && more) named_arrive<W>(1);  // slot free for the next piece

    // ---- finalise this piece from registers (warp 0)
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, off);
      l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f, inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
    const float lse0 = l0 > 0.f ? (m0 + log2f(l0)) * kLn2 : -CUDART_INF_F;
    const float lse1 = l1 > 0.f ? (m1 + log2f(l1)) * kLn2 : -CUDART_INF_F;
    const int n_it = d.n_it;
    const int64_t orow = d.out_row;

    if (fused && n_it == 1) {
      // whole segment in one piece: registers -> output rows (16-byte stores)
      emit_acc<G>(p, ep, orow, acc, inv0, inv1, lane);
      // lse of head g is lse0 / lse1 of lane g >> 1 (lanes 0..3)
      const float la = __shfl_sync(0xffffffffu, lse0, (lane >> 1) & 3);
      const float lb = __shfl_sync(0xffffffffu, lse1, (lane >> 1) & 3);
      emit_lse_lanes<G>(p, ep, orow, (lane & 1) ? lb : la, lane);
      continue;
    }

    // partial record of this piece
    float* rec = p.part + static_cast<int64_t>(d.rec) * G * FKV_REC;
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

    // The CTA that finishes one of the segment's pieces last merges them all.
    // Warp barrier + one acq_rel atomic (release publishes the whole warp's
    // record stores, acquire makes every other piece's records visible).
    __syncwarp();
    stamp(PROBE, p.stamp_slot, 6);
    int last = 0;
    if (lane == 0) last = atom_add_acq_rel(p.counters + d.i0, 1) == n_it - 1;
    last = __shfl_sync(0xffffffffu, last, 0);
    stamp(PROBE, p.stamp_slot, 7);
    if (kCombiner && last && !more) {
      // the CTA's last piece: warps 1-3 are idle, merge with all four (below)
      if (lane == 0) sh.fin_i0 = d.i0, sh.fin_n_it = n_it, sh.fin_orow = static_cast<int32_t>(orow);
      continue;
    }
    if (!last) continue;
    // All (piece, head) lse values in one parallel round trip, weights in
    // shared scratch, then every lane streams its 4 head_dim columns of all
    // records with n_it*G independent 16-B loads (L2: .cg, never a stale L1 line).
    const float* base = p.part + static_cast<int64_t>(d.i0) * G * FKV_REC;
    // SOLO: any warp may merge -- per-warp weights in the (unused) hand-over area
    float* sw = SOLO ? &sh.xch[0][0][0] + warp * kMergeMax * 8 : sh.scratch;
    for (int x = lane; x < n_it * G; x += 32) sw[x] = __ldcg(base + x * FKV_REC + FKV_HEAD_DIM);
    __syncwarp();
    stamp(PROBE, p.stamp_slot, 8);
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
    stamp(PROBE, p.stamp_slot, 9);
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
    stamp(PROBE, p.stamp_slot, 10);
#pragma unroll
    for (int g = 0; g < G; ++g) emit_row_lanes(p, ep, orow + g, o[g], lane);
    emit_lse_lanes<G>(p, ep, orow, lse_g, lane);
    if (lane == 0) p.counters[d.i0] = 0;  // ready for the next launch / graph replay
    stamp(PROBE, p.stamp_slot, 11);
    __syncwarp();  // the scratch is reused by the next merge
  }

  if (kCombiner) {
    // Deferred merge of the segment the CTA's last piece completed: the four
    // warps split the G heads, each lane loads its columns of every piece's
    // record together with the lse values (one L2 round trip), weights by
    // warp shuffles.
    named_sync<W>(3);
    const int n_it = sh.fin_n_it;
    if (warp == 0) stamp(PROBE, p.stamp_slot, 13);
    if (n_it > 0) {
      const float* base = p.part + static_cast<int64_t>(sh.fin_i0) * G * FKV_REC;
      const int64_t orow = sh.fin_orow;
      constexpr int kHpw = (G + W - 1) / W;  // heads per warp
#pragma unroll
      for (int hi = 0; hi < kHpw; ++hi) {
        const int g = warp * kHpw + hi;
        if (g >= G) break;
        const float l = lane < n_it ? __ldcg(base + (lane * G + g) * FKV_REC + FKV_HEAD_DIM) : -CUDART_INF_F;
        float4 v[8];
        const int n0 = n_it < 8 ? n_it : 8;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          v[i] = i < n0 ? __ldcg(reinterpret_cast<const float4*>(base + (i * G + g) * FKV_REC) + lane)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
        float M = l;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
        const float e = M == -CUDART_INF_F || l == -CUDART_INF_F ? 0.f : __expf(l - M);
        float S = e;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
        const float wl = S > 0.f ? e / S : 0.f;
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        auto fma4 = [&](float wi, const float4& x) {
          o.x = fmaf(wi, x.x, o.x);
          o.y = fmaf(wi, x.y, o.y);
          o.z = fmaf(wi, x.z, o.z);
          o.w = fmaf(wi, x.w, o.w);
        };
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float wi = __shfl_sync(0xffffffffu, wl, i);
          if (i < n_it) fma4(wi, v[i]);
        }
        for (int i = 8; i < n_it; ++i)
          fma4(__shfl_sync(0xffffffffu, wl, i),
               __ldcg(reinterpret_cast<const float4*>(base + (i * G + g) * FKV_REC) + lane));
        const float lse_g = S > 0.f ? M + __logf(S) : -CUDART_INF_F;
        const int64_t row = orow + g;
        emit_row_lanes(p, ep, row, o, lane);
        if (lane == 0) store_lse1(p, ep, row, lse_g);
      }
      if (threadIdx.x == 0) p.counters[sh.fin_i0] = 0;
    }
    if (warp == 0) stamp(PROBE, p.stamp_slot, 14);
  }

  if (warp == 0) stamp(PROBE, p.stamp_slot, 5);
}

// K5 standalone (after the all-gather): warp g of the CTA merges head g of
// one output group in a single online-LSE pass over exchange records (block
// r at r * block_bytes, `slots` rows per block); lane = 4 head_dim columns.
// LL: XLL blocks written by peers' fkv_decode_exchange -- every lane polls
// its own 16-byte unit (and the row's lse unit) until both epoch words match,
// so each merge starts as soon as its own records have landed.
__device__ __forceinline__ int4 ld_ll(const uint8_t* a) {
  int4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(a)
               : "memory");
  return v;
}

template <int G, bool LL>
__global__ void __launch_bounds__(G * 32)
    merge_lse_kernel(const uint8_t* __restrict__ xrec, int slots, int64_t block_bytes,
                     const int32_t* __restrict__ grp_ptr, const int32_t* __restrict__ src_idx,
                     const int32_t* __restrict__ out_row, __nv_bfloat16* __restrict__ out_bf16,
                     float* __restrict__ out_lse, int32_t* epoch_ctr) {
  // Programmatic dependent launch.  Plain records are complete once the
  // producer grid (NCCL all-gather, K4 records) is.  XLL records validate
  // themselves, so the LL merge starts polling while the producer K4 still
  // runs and does not wait for it: it starts only after that K4 triggered,
  // i.e. passed its own wait on the previous merge, so the epoch the previous
  // merge advanced is final; the next K4 reads the epoch only after its wait
  // on this grid.
  int ep = 0;
  if (LL) ep = *reinterpret_cast<volatile int32_t*>(epoch_ctr) + 1;
  else asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const int grp = blockIdx.x;
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = grp_ptr[grp], i1 = grp_ptr[grp + 1];
  const int64_t lse_off = static_cast<int64_t>(slots) * G * FKV_HEAD_DIM * 2;
  float m = -CUDART_INF_F, S = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = i0; i < i1; ++i) {
    const int src = src_idx[i];
    const uint8_t* blk = xrec + static_cast<int64_t>(src / slots) * block_bytes;
    const int64_t row = static_cast<int64_t>(src % slots) * G + g;
    float l;
    uint2 w;
    if (LL) {
      // both units' loads in flight together, then each polled until it
      // carries the epoch (one round trip on the critical path, not two)
      const uint8_t* r = blk + row * FKV_XLL_ROW_BYTES;
      int4 u = ld_ll(r + 16 * lane), ul = ld_ll(r + 32 * 16);
      while (u.y != ep || u.w != ep) {
        __nanosleep(20);
        u = ld_ll(r + 16 * lane);
      }
      while (ul.y != ep || ul.w != ep) {
        __nanosleep(20);
        ul = ld_ll(r + 32 * 16);
      }
      l = __int_as_float(ul.x);
      w = make_uint2(u.x, u.z);
    } else {
      l = __ldcg(reinterpret_cast<const float*>(blk + lse_off) + row);
      if (l != -CUDART_INF_F) w = __ldcg(reinterpret_cast<const uint2*>(blk + row * FKV_HEAD_DIM * 2) + lane);
    }
    if (l == -CUDART_INF_F) continue;
    const float2 o01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w.x));
    const float2 o23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w.y));
    const float nm = fmaxf(m, l);
    const float a = __expf(m - nm), b = __expf(l - nm);
    S = S * a + b;
    acc.x = acc.x * a + o01.x * b;
    acc.y = acc.y * a + o01.y * b;
    acc.z = acc.z * a + o23.x * b;
    acc.w = acc.w * a + o23.y * b;
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
  if (out_lse && lane == 0) out_lse[row] = lse;
  if (LL) {
    // the last CTA out advances the epoch (every CTA read it at entry)
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(epoch_ctr + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      epoch_ctr[1] = 0;
      atomicExch(epoch_ctr, ep);
    }
  }
}

template <int G, int PROBE = 0, int MODE = 0>
int launch_decode(const DecodeParams& p, cudaStream_t st) {
  static std::atomic<int> ready[kMaxDevices];  // smem attribute set on this device
  const int rc = per_device(ready, [](int) {
    const int e = cuda_check(cudaFuncSetAttribute(decode_kernel<G, PROBE, MODE>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  Shape<MODE>::kSmem),
                             "decode smem attribute");
    return e < 0 ? e : 1;
  });
  if (rc < 0) return rc;
  // one CTA per worker; nothing in the kernel waits on another CTA, so the
  // grid may exceed the co-resident limit -- later CTAs start as earlier
  // ones retire
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_workers, 1, 1);
  cfg.blockDim = dim3(Shape<MODE>::W * 32, 1, 1);
  cfg.dynamicSmemBytes = Shape<MODE>::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (see kernel)
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  static const bool no_pdl = getenv("FKV_NO_PDL") != nullptr;  // diagnostics
  cfg.attrs = attr;
  cfg.numAttrs = no_pdl ? 0 : 1;
  return cuda_check(cudaLaunchKernelEx(&cfg, decode_kernel<G, PROBE, MODE>, p), "decode launch");
}

}  // namespace
}  // namespace fkv

namespace fkv {
namespace {
template <int MODE>
int launch_mode(DecodeParams& p, int group, cudaStream_t st, int probe) {
  if (group == 4) return launch_decode<4, 0, MODE>(p, st);
  if (group != 8) return set_error(FKV_ERR_INVALID, "fkv_decode: group must be 4 or 8");
  switch (probe) {
    case 1: return launch_decode<8, 1, MODE>(p, st);
    case 2: return launch_decode<8, 2, MODE>(p, st);
    case 3: return launch_decode<8, 3, MODE>(p, st);
    default: return launch_decode<8, 0, MODE>(p, st);
  }
}

int decode_entry(DecodeParams& p, int group, cudaStream_t st, int probe, int flags) {
  if (flags & FKV_DECODE_SOLO) return launch_mode<1>(p, group, st, probe);
  if (flags & FKV_DECODE_WIDE) return launch_mode<2>(p, group, st, probe);
  return launch_mode<0>(p, group, st, probe);
}
}  // namespace
}  // namespace fkv

static int g_probe = 0;

extern "C" int fkv_decode_ctas_per_sm(int32_t flags) {
  if (flags & FKV_DECODE_SOLO) return fkv::Shape<1>::kCtasPerSm;
  if (flags & FKV_DECODE_WIDE) return fkv::Shape<2>::kCtasPerSm;
  return fkv::Shape<0>::kCtasPerSm;
}

// Diagnostics (not part of fairkv.h): the next fkv_decode call runs probe mode
// `mode & 15` (1 = loads only, 2 = compute only, 3 = timestamps into stamp
// block mode >> 4).  Used by tools/probe_*.py.
extern "C" int fkv__decode_probe(int32_t mode) {
  g_probe = mode;
  return 0;
}

extern "C" int fkv__decode_stamps(unsigned long long* host, int32_t n) {
  return fkv::cuda_check(cudaMemcpyFromSymbol(host, fkv::g_stamps, sizeof(unsigned long long) * n),
                         "stamps");
}

extern "C" int fkv_decode(const void* q, const void* k, const void* v, const fkv_work_t* work,
                          int32_t work_k, int32_t n_workers, int32_t n_items, int32_t group,
                          int32_t flags, float sm_scale, float* part, int32_t* counters,
                          void* out_bf16, void* out_xrec, int32_t xrec_slots, float* out_lse,
                          void* stream) {
  return fkv_decode_exchange(q, k, v, work, work_k, n_workers, n_items, group, flags, sm_scale, part,
                             counters, out_bf16, out_xrec ? &out_xrec : nullptr, out_xrec ? 1 : 0,
                             xrec_slots, out_lse, nullptr, stream);
}

extern "C" int fkv_decode_exchange(const void* q, const void* k, const void* v,
                                   const fkv_work_t* work, int32_t work_k, int32_t n_workers,
                                   int32_t n_items, int32_t group, int32_t flags, float sm_scale,
                                   float* part, int32_t* counters, void* out_bf16,
                                   void* const* out_xrecs, int32_t n_rec, int32_t xrec_slots,
                                   float* out_lse, const int32_t* epoch_ctr, void* stream) {
  using namespace fkv;
  if (n_items < 0 || n_workers < 0) return set_error(FKV_ERR_INVALID, "fkv_decode: negative size");
  if (work_k < 1 || work_k > FKV_MAX_WORK)
    return set_error(FKV_ERR_INVALID, "fkv_decode: work_k must be in [1, FKV_MAX_WORK]");
  if (n_rec < 0 || n_rec > FKV_MAX_PEERS)
    return set_error(FKV_ERR_INVALID, "fkv_decode: too many record destinations");
  if (n_rec > 0 && xrec_slots < 1)
    return set_error(FKV_ERR_INVALID, "fkv_decode: exchange records need xrec_slots >= 1");
  if (n_items == 0 || n_workers == 0) return FKV_OK;
  if (!q || !k || !v || !work || !part || !counters || (n_rec && !out_xrecs))
    return set_error(FKV_ERR_INVALID, "fkv_decode: null pointer");
  uintptr_t align = reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
                    reinterpret_cast<uintptr_t>(work) | reinterpret_cast<uintptr_t>(out_bf16) |
                    reinterpret_cast<uintptr_t>(out_lse);
  for (int j = 0; j < n_rec; ++j) align |= reinterpret_cast<uintptr_t>(out_xrecs[j]);
  if (align & 15)
    return set_error(FKV_ERR_INVALID, "fkv_decode: cache / work table / outputs not 16-byte aligned");
  DecodeParams p{};
  p.q = static_cast<const __nv_bfloat16*>(q);
  p.k = static_cast<const __nv_bfloat16*>(k);
  p.v = static_cast<const __nv_bfloat16*>(v);
  p.work = work;
  p.work_k = work_k;
  p.n_workers = n_workers;
  p.scale_log2 = sm_scale * kLog2e;
  p.part = part;
  p.counters = counters;
  p.out_bf16 = static_cast<__nv_bfloat16*>(out_bf16);
  for (int j = 0; j < n_rec; ++j) p.out_rec[j] = static_cast<uint8_t*>(out_xrecs[j]);
  p.n_rec = n_rec;
  p.rec_lse_off = static_cast<int64_t>(xrec_slots) * group * FKV_HEAD_DIM * 2;
  p.out_lse = out_lse;
  p.epoch_ctr = epoch_ctr;
  p.after_wait = (flags & FKV_DECODE_AFTER_WAIT) != 0;
  const int probe = g_probe & 15;
  p.stamp_slot = (g_probe >> 4) & 3;
  g_probe = 0;
  return decode_entry(p, group, static_cast<cudaStream_t>(stream), probe, flags);
}

extern "C" int fkv_merge_lse(const void* xrec, int32_t xrec_slots, const int32_t* grp_ptr,
                             const int32_t* src_idx, const int32_t* out_row, int32_t n_groups,
                             int32_t group, void* out_bf16, float* out_lse, void* stream) {
  return fkv_merge_wait(xrec, xrec_slots, grp_ptr, src_idx, out_row, n_groups, group, out_bf16,
                        out_lse, nullptr, stream);
}

extern "C" int fkv_merge_wait(const void* xrec, int32_t xrec_slots, const int32_t* grp_ptr,
                              const int32_t* src_idx, const int32_t* out_row, int32_t n_groups,
                              int32_t group, void* out_bf16, float* out_lse, int32_t* epoch_ctr,
                              void* stream) {
  using namespace fkv;
  if (n_groups < 0 || xrec_slots < 1) return set_error(FKV_ERR_INVALID, "fkv_merge_lse: bad sizes");
  if (n_groups == 0) return FKV_OK;
  if (!xrec || !grp_ptr || !src_idx || !out_row || (!out_bf16 && !out_lse))
    return set_error(FKV_ERR_INVALID, "fkv_merge_lse: null pointer");
  if (reinterpret_cast<uintptr_t>(xrec) & 15)
    return set_error(FKV_ERR_INVALID, "fkv_merge_lse: records not 16-byte aligned");
  if (group != 4 && group != 8) return set_error(FKV_ERR_INVALID, "fkv_merge_lse: group must be 4 or 8");
  auto ob = static_cast<__nv_bfloat16*>(out_bf16);
  auto xr = static_cast<const uint8_t*>(xrec);
  const bool ll = epoch_ctr != nullptr;
  const int64_t block = ll ? FKV_XLL_BYTES(xrec_slots, group) : FKV_XREC_BYTES(xrec_slots, group);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_groups, 1, 1);
  cfg.blockDim = dim3(group * 32, 1, 1);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (see kernel)
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = getenv("FKV_K5_NO_PDL") && ll ? 0 : 1;  // env: diagnostics
  cudaError_t e;
  if (group == 4)
    e = ll ? cudaLaunchKernelEx(&cfg, merge_lse_kernel<4, true>, xr, xrec_slots, block, grp_ptr, src_idx,
                                out_row, ob, out_lse, epoch_ctr)
           : cudaLaunchKernelEx(&cfg, merge_lse_kernel<4, false>, xr, xrec_slots, block, grp_ptr, src_idx,
                                out_row, ob, out_lse, epoch_ctr);
  else
    e = ll ? cudaLaunchKernelEx(&cfg, merge_lse_kernel<8, true>, xr, xrec_slots, block, grp_ptr, src_idx,
                                out_row, ob, out_lse, epoch_ctr)
           : cudaLaunchKernelEx(&cfg, merge_lse_kernel<8, false>, xr, xrec_slots, block, grp_ptr, src_idx,
                                out_row, ob, out_lse, epoch_ctr);
  return cuda_check(e, "merge_lse launch");
}

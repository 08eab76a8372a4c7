// Shared constants, parameter blocks and TMA issue helpers of the CCE kernels.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "cce_ptx.cuh"

namespace cce {

constexpr int BM = 128;                   // tokens per logit tile (TMEM lanes, MMA M)
constexpr int BN = 256;                   // vocab rows per logit tile (MMA N)
constexpr int BK = 64;                    // D elements per K-block: one 128 B swizzle atom
constexpr int A_BYTES = BM * BK * 2;      // 16 KiB
constexpr int B_BYTES = BN * BK * 2;      // 32 KiB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NUM_THREADS = 192;          // warp0 TMA, warp1 MMA, warps 2..5 epilogue
constexpr int LSE_STAGES = 4;
#ifndef CCE_LSE_STAGES_PAIR
#define CCE_LSE_STAGES_PAIR 6
#endif
constexpr int LSE_STAGES_PAIR = CCE_LSE_STAGES_PAIR;
constexpr int PAIR_STAGE_BYTES = A_BYTES + (BN / 2) * BK * 2;  // 128 E rows + 128 of 256 C rows
constexpr int TMEM_COLS = 512;
constexpr int LSE_CTRL_BYTES = 256;       // barriers / TMEM slot / votes of the logit-tile kernel
constexpr int LSE_IDX_BYTES = (BM + BN) * 4;  // its row-gather index tables
constexpr int DCH = 256;                  // D columns per gradient chunk (MMA N of dE / dC)
constexpr int SHAT_TILE_BYTES = BM * BN * 2;  // one stored S-hat tile, bf16 row-major [128][256]

enum Mode { FWD = 0, BWD = 1, KEPT = 2 };

// Streamed backward (cce_bwd_stream): S-hat tiles pass from producer CTAs (KEPT recompute) to
// consumer CTAs (dE or dC) of the same grid through a ring of `ring` 64 KiB slots in HBM.  Item i
// (its position in the pass's kept list) occupies slot i % ring; the producer waits until the
// slot's previous item has been read by all its consumers, writes S-hat, then publishes
// ready[slot] = lap + 1 (lap = i / ring); each consumer waits for that, loads the tile with TMA
// and adds 1 to used[slot] once the bytes have landed.
struct Stream {
  int ring;          // slots (0: not streaming)
  int* ready;        // [ring]
  int* used;         // [ring]
  int consumers;     // consumptions per item
  int producers;     // the first `producers` CTAs of the grid recompute, the rest consume
};

// Forward (FWD) and backward filter pass (BWD, "B1") of the fused logit-tile kernel.
//
// Token rows: the forward runs on all n_total rows of E.  The backward runs on the compacted
// valid rows (filter_ignored, kernels.py:494-510), whose count *n_valid lives on the device; when
// it equals n_total the compaction is the identity and E is read directly.
struct Params {
  int n_total;       // rows of E
  const int* n_valid;  // device count of compacted rows (backward), nullptr = n_total
  const int* run_if;   // device flag: kernel does nothing unless *run_if != 0 (nullptr = always)
  int d;             // hidden size
  int v;             // vocab rows of C (this shard)
  int nt;            // token tiles per launch (a group in the backward); clamped on the device
  int n_base;        // first token tile of this launch
  int mt;            // vocab tiles
  int splits;        // vocab splits per token tile (units = nt * splits)
  int band;          // token tiles per raster band (bounds the E working set of concurrent CTAs)
  int grid_cap;      // FWD / BWD: CTAs (pairs) per round of the static schedule, 0 = whole grid
  int num_kb;        // ceil(d / BK)
  float softcap;     // 0 => off
  // forward
  const int64_t* targets;
  int64_t ignore_index;
  int64_t vocab_start;
  float2* part;      // [splits][n_total]  (running max, running sum) in log2 units
  float* correct;    // [n_total] target logit (written by the tile that owns the label)
  float* tile_max;   // [nt][mt][BM] max raw logit of each row in each tile, or nullptr
  // label tiles (FWD, optional): a tile holding some row's label is always kept by the backward
  // (kernels.py:447-455), so the forward stores it -- fp16 of z' - z'max(row) -- in a slot of
  // lab_buf ([lab_capacity][BM][BN]) and the backward turns it into S-hat without a recompute
  __half* lab_buf;
  int lab_capacity;
  int* lab_count;          // slots handed out (may exceed lab_capacity: those tiles get none)
  int32_t* lab_slot;       // [nt][mt] slot of a stored label tile, -1 (pre-filled) if none
  int2* lab_list;          // [lab_capacity] (token tile, vocab tile) of each slot
  // backward filter pass (lse / upstream / pos are indexed by ORIGINAL row)
  const float* lse;        // global log-sum-exp (natural log)
  const float* upstream;   // dLoss/dloss_i, 0 at ignored rows
  const int32_t* pos;      // label position in tile order, -1 if none (FWD: nullptr = targets)
  int pos_offset;          // over a vocabulary group: pos - pos_offset is group-local
  int label_split;         // 1: paper ordering -- filter on S alone, S-hat without the -1 (the
                           //    label term is applied separately, cce_label_terms)
  const int32_t* perm;     // [mt*BN] tile-order position -> C row for gathers (nullptr = plain)
  const int32_t* row_map;  // compact row -> original row (padded); identity when no compaction
  int e_gather;            // 1: load E rows through row_map (cp.async gather unless the map is
                           //    the identity; else E is compacted)
  const __nv_bfloat16* e_rows;  // E base (row gathers), [n_total][d]
  const __nv_bfloat16* c_rows;  // C base (row gathers through perm), [v][d]
  const uint8_t* block_zero;  // [token tiles] 1 if every upstream in the compact tile is zero
  float eps;               // filter threshold (0 = filtering off)
  __nv_bfloat16* shat;     // [capacity][BM][BN] S-hat of kept tiles, compact slots
  int32_t* slot_of;        // [nt*mt] slot of tile (local n, m), -1 if not stored (host: -1)
  int* slot_ctr;           // next free slot (host: 0)
  int capacity;            // slots available
  int* overflow;           // set to 1 if a kept tile found no slot (host: 0)
  int* cnt_n;              // [nt] kept tiles per token tile
  int* cnt_m;              // [mt] kept tiles per vocab tile
  unsigned long long* counters;  // [3] kept, eps-skipped, zero-upstream-skipped
  // KEPT
  const int2* list;        // [capacity] (token tile, vocab tile) of each slot
  const int* list_count;   // kept tiles (slots used = min(count, capacity))
  const int2* pairs;       // CTA pairs: (first slot, 1 or 2 tiles) of one vocab tile
  const int* pair_count;
  Stream st;               // KEPT streamed into a ring (TileRef.s is then the item index)
  int tm_stride, tm_m0;    // FWD: tile_max row stride in vocab tiles (0: mt) and first vocab tile
  // FWD over vocabulary groups as one chain of programmatic-dependent launches (ops.forward_stream,
  // cce_fwd_group_sync): launch g sweeps group g from a buffer the previous launch's gather warps
  // filled, and its own gather warp (warp 6 of a 224-thread launch) fills the other buffer with
  // group g + 1 once launch g - 1 has exited (that buffer is the one launch g - 1 read).  No launch
  // waits for the previous one to finish: each waits on flags for exactly what it reads.
  const int* sync_ready;   // 1 once this launch's group is in its buffer (nullptr: stream order)
  int* sync_exit;          // CTAs of this launch that exited; the last sets *sync_released = 1
  int* sync_released;
  int no_dep_wait;         // 1: no griddepcontrol.wait (the flags order every input)
  const int32_t* g_perm;   // gather warp: row r of g_dst <- g_src[g_perm[r]], r < g_rows
  const __nv_bfloat16* g_src;
  __nv_bfloat16* g_dst;
  int g_rows;
  const int* g_wait;       // gather only once *g_wait >= 1 (nullptr: at once)
  int* g_ctr;              // gather shares done; the last sets *g_done = 1
  int* g_done;
};

// dE pass ("B2") and dC pass ("B3").
struct GradParams {
  int n_total, d, v, mt, ndc;
  const int* n_valid;
  const int* run_if;
  int n_base, g;           // token tiles [n_base, n_base + g) of this group (clamped on device)
  const int32_t* slot_of;  // [g*mt]
  const int* cnt_n;
  const int* cnt_m;
  const int32_t* perm;     // C-row gather index for tile loads (padded), or nullptr
  const int32_t* perm_store;  // tile-order position -> dC row (padded), or nullptr
  const int32_t* row_map;  // compact row -> original row (padded)
  int e_gather;            // 1: gather E rows through row_map (else E is compacted)
  const __nv_bfloat16* e_rows;  // E base of the row gathers (pairs: cp.async), [n_total][d]
  int atoms3d;             // 1: d % 64 == 0, operand tiles load as one 3-D TMA box (all atoms)
  __nv_bfloat16* de_bf16;  // [n_total][d]   (one of de_bf16 / de_f32)
  float* de_f32;
  __nv_bfloat16* dc;       // [v][d]
  int accumulate;          // dC: add to the existing values (groups after the first)
  int de_accumulate;       // dE (fp32 only): add to the existing values (vocabulary groups)
  const int2* list;        // dC: vocab-tile-major kept list (slot = index, .x = token tile), or nullptr
  const int* off_m;        //     first slot of each vocab tile (its cnt_m slots are consecutive)
  int* sched;              // dE: unit counter (zeroed before the launch), nullptr = static
  int de_order;            // dE: 0 chunk-major units, 1 token-tile-major, K>=2 groups of K chunks
  int dc_block;            // dC: 0 vocab-tile-major units, B > 0 blocks of B vocab tiles, chunk-major
  int prefetch;            // dE: L2-prefetch C slices of the kept tiles this many vocab tiles ahead (0 = off)
  int debug;               // diagnostics only (CCE_DEBUG_GRAD): bit0 skip S-hat loads, bit1 skip E/C loads
  // streamed backward: units are (segment, D chunk[, vocab half]); a segment is a run of at most B
  // consecutive items of one owner (token tile for dE, vocab tile for dC).  An owner split over
  // several segments sums them in segment order through an fp32 accumulator region (chain[] counts
  // the segments folded in; acc_gen[] hands the region from one owner to the next).
  Stream st;
  const int4* seg;         // [*seg_count] (owner, first item, items, split index)
  const int2* seg_aux;     // [*seg_count] (splits of the owner, accumulator id if splits > 1)
  const int* seg_count;
  const int2* items;       // the pass's kept list: (token tile, vocab tile) in stream order
  const int* sidx;         // segment item k is items[sidx[k]] (nullptr: items[k]; dE segments
                           // gather one token tile's items of a stream window)
  int* chain;              // [owners * ndc * 2]
  float* acc;              // [nacc][ndc][2][128][256]
  int nacc;
  int* acc_gen;            // [nacc * ndc * 2]
  // dC over the storage of the sorted classifier: before a vocab tile's dC is written, every item
  // of the tile (own_off[m] .. + own_cnt[m]) must have been read by all its consumers (the dE
  // consumers read those C rows)
  const int* own_off;
  const int* own_cnt;
  unsigned long long* prof;  // diagnostics (CCE_STREAM_PROF builds): per-unit timestamps
};

// Device-side view of the compaction: valid row count, token tiles of this launch.
struct Rows {
  int n;        // rows handled (compacted count)
  bool ident;   // compaction is the identity
  int g;        // token tiles of this launch after clamping
  __device__ __forceinline__ Rows(const int* n_valid, int n_total, int n_base, int nt) {
    n = n_valid ? *n_valid : n_total;
    ident = (n == n_total);
    const int nt_dev = (n + BM - 1) / BM;
    g = max(0, min(nt, nt_dev - n_base));
  }
};

// Programmatic dependent launch: a kernel launched with the PDL attribute may be scheduled
// before its predecessor in the stream has finished; every thread waits here, before touching
// anything upstream kernels wrote (and before exiting, so completion stays transitive along a
// chain of gated-off kernels).  Without the attribute the wait returns at once.
#ifndef CCE_PDL_TRIGGER
#define CCE_PDL_TRIGGER 1
#endif
__device__ __forceinline__ void griddep_wait() {
#if CCE_PDL_TRIGGER
  // let the next kernel be scheduled now; its own griddep_wait still orders it after this grid
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ void griddep_trigger() {
#if CCE_PDL_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

__device__ __forceinline__ bool skip_launch(const int* run_if) {
  griddep_wait();
  return run_if != nullptr && *run_if == 0;
}

__device__ __forceinline__ void advance_stage(int& stage, uint32_t& phase, int stages) {
  if (++stage == stages) {
    stage = 0;
    phase ^= 1;
  }
}

// A box of `rows` (<= 256) logical rows x 64 columns of a row-major bf16 matrix lands in a
// 128B-swizzled smem box either as one TMA tile load (no index; lane 0 issues it) or as a row
// gather through `index` (logical row -> physical row) split across the producer warp: lane l
// issues the tile::gather4 transfers of its own 4-row groups, whose indices it loaded into
// registers once per tile (so no index load sits between two gathers).
struct RowGather {
  // up to two 4-row groups per lane: rows 4*(lane + 32*j) .. +3 of the box
  int4 idx[2];
  int groups;  // 4-row groups per lane (0, 1 or 2)
  __device__ __forceinline__ void load(const int32_t* index, int row0, int rows) {
    const int lane = threadIdx.x & 31;
    groups = 0;
    if (index == nullptr) return;
    const int4* ix = reinterpret_cast<const int4*>(index + row0);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int gi = lane + 32 * j;
      if (gi * 4 < rows) {
        idx[j] = __ldg(ix + gi);
        groups = j + 1;
      }
    }
  }
  __device__ __forceinline__ void issue(const CUtensorMap* tm_gather, uint64_t* bar, uint8_t* dst,
                                        int c0) const {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < 2; ++j)
      if (j < groups)
        tma_gather4(tm_gather, bar, dst + (lane + 32 * j) * 512, c0, idx[j].x, idx[j].y, idx[j].z,
                    idx[j].w);
  }
};

template <int ROWS>
__device__ __forceinline__ void load_rows_warp(const CUtensorMap* tm_tile, const CUtensorMap* tm_gather,
                                               const RowGather& rg, bool gather, uint64_t* bar,
                                               uint8_t* dst, int c0, int row0) {
  if (!gather) {
    if ((threadIdx.x & 31) == 0) tma_load_2d(tm_tile, bar, dst, c0, row0);
  } else {
    rg.issue(tm_gather, bar, dst, c0);
  }
}

// Row gather into a 128B-swizzled smem box by one warp with cp.async (16 B per lane): the box is
// ROWS logical rows x 64 bf16 columns [col0, col0 + 64) of a row-major [*, d] matrix, logical
// row r reading source row idx[r] (an smem table filled once per tile).  Lanes 8k..8k+7 take the
// eight 16-B chunks of one row, so each warp instruction reads four whole 128-B row segments;
// chunk j of row r lands at chunk (j ^ (r & 7)) of the row's 128 B -- the layout a 128B-swizzled
// TMA box has, which the UMMA descriptors expect.  Columns >= d are zero-filled (d % 8 == 0).
// Completion: cp.async groups (the caller commits, waits and relays to the stage's mbarrier after
// a fence.proxy.async, because the tensor core reads smem through the async proxy).
template <int ROWS>
__device__ __forceinline__ void gather_box_async(uint8_t* dst, const __nv_bfloat16* src, int d,
                                                 const int32_t* idx, int col0) {
  const int lane = threadIdx.x & 31;
  const int j = lane & 7;
  const uint32_t d0 = smem_u32(dst);
  const uint32_t nbytes = (col0 + j * 8 < d) ? 16u : 0u;
  const char* s0 = reinterpret_cast<const char*>(src) + (size_t)(nbytes ? col0 + j * 8 : 0) * 2;
#pragma unroll 8
  for (int r = lane >> 3; r < ROWS; r += 4)
    cp_async16(d0 + r * 128 + ((j ^ (r & 7)) << 4), s0 + (int64_t)idx[r] * d * 2, nbytes);
}

// Fill a warp's smem index table: tab[r] = index[row0 + r] for r < rows (index == nullptr:
// row0 + r).  The caller __syncwarp()s before use.
// Rows at or past `limit` (a CTA pair's missing partner tile, rows past the compacted count) read
// source row 0 instead: their results are discarded, and the index array may end there.
__device__ __forceinline__ void load_index_table(int32_t* tab, const int32_t* index, int row0, int rows,
                                                 int limit = 0x7fffffff) {
  for (int r = threadIdx.x & 31; r < rows; r += 32)
    tab[r] = row0 + r >= limit ? 0 : (index ? index[row0 + r] : row0 + r);
}

// softcap: z' = cap * tanh(z / cap), tanh(x) = 1 - 2 / (exp(2x) + 1) (exact limits at +-inf)
__device__ __forceinline__ float softcap_tanh(float z, float inv_cap) {
  const float e = ex2_approx(z * inv_cap * 2.8853900817779268f);  // 2*log2(e)
  return 1.0f - __fdividef(2.0f, e + 1.0f);
}

constexpr float LOG2E = 1.4426950408889634f;

// The filter test of one row of one tile: S = exp(softcap(z) - lse) is monotone in z, so the
// row has an entry >= eps iff its max raw logit does (block_skip_decision, kernels.py:140-142,
// strict "<" to skip).  Shared by the in-kernel filter and the decision from forward maxima, so
// both take bit-identical decisions.
__device__ __forceinline__ bool tile_row_big(float zmax, float lse2, float softcap, float inv_cap,
                                             float eps) {
  if (zmax == -INFINITY) return false;
  const float zc = softcap > 0.f ? softcap * softcap_tanh(zmax, inv_cap) : zmax;
  return ex2_approx(zc * LOG2E - lse2) >= eps;
}

}  // namespace cce

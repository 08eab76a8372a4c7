// Small helper kernels of the CCE path: split/shard LSE merges, the vocabulary sort key, the
// backward prep (inverse permutation, label positions, zero-upstream tiles) and casts.
#pragma once
#include <climits>

#include "cce_common.cuh"

namespace cce {

// ---------------------------------------------------------------------------------------
// Small kernels
// ---------------------------------------------------------------------------------------

// Merge the per-split (max2, sum2) partials of each row into this shard's natural-log LSE.
// out_part != nullptr: fold the partials into one (max, sum-exp) pair instead (it may alias part:
// every read of a row precedes the block barrier before its write).  Block = 32 rows x
// COMBINE_GROUPS slot groups: warp g reads slots g, g + 8, ... of 32 consecutive rows (coalesced
// 256 B per slot), the groups' maxima and then their sums meet in shared memory in a fixed order
// (deterministic).  Hundreds of partials per row (the bounded forward folds 8 groups of up to
// ~40 splits) cost a few microseconds instead of a serial loop per thread.
constexpr int COMBINE_ROWS = 32;
constexpr int COMBINE_GROUPS = 8;
__global__ void __launch_bounds__(COMBINE_ROWS * COMBINE_GROUPS)
    combine_splits_kernel(const float2* part, int splits, int n, float* __restrict__ lse_local, float2* out_part) {
  griddep_wait();
  __shared__ float s_red[COMBINE_GROUPS][COMBINE_ROWS];
  const int r = threadIdx.x & (COMBINE_ROWS - 1);
  const int g = threadIdx.x / COMBINE_ROWS;
  const int i = blockIdx.x * COMBINE_ROWS + r;
  const bool ok = i < n;
  float m = -INFINITY;
  if (ok)
    for (int s = g; s < splits; s += COMBINE_GROUPS) m = fmaxf(m, part[(size_t)s * n + i].x);
  s_red[g][r] = m;
  __syncthreads();
  m = s_red[0][r];
#pragma unroll
  for (int k = 1; k < COMBINE_GROUPS; ++k) m = fmaxf(m, s_red[k][r]);
  float acc = 0.f;
  if (ok && m != -INFINITY)
    for (int s = g; s < splits; s += COMBINE_GROUPS) {
      const float2 v = part[(size_t)s * n + i];
      acc += v.y * exp2f(v.x - m);
    }
  __syncthreads();  // every group has read the maxima
  s_red[g][r] = acc;
  __syncthreads();
  if (g != 0 || !ok) return;
  acc = s_red[0][r];
#pragma unroll
  for (int k = 1; k < COMBINE_GROUPS; ++k) acc += s_red[k][r];
  if (out_part)
    out_part[i] = make_float2(m, acc);
  else
    lse_local[i] = (m == -INFINITY) ? -INFINITY : (m + log2f(acc)) * 0.6931471805599453f;
}

// Vocab-parallel / single-shard finish: lse = logaddexp over shards, correct = sum over shards.
// Mirrors cce_loss's scatter (kernels.py:539-547): loss and lse are 0 at ignored rows.
// Label range (check_vocab, core.py:110-114) without a host read: with v_total > 0, a row whose
// label is neither ignore_index nor in [0, v_total) gets a NaN loss and sets *bad = 1 (sticky,
// read by the host later, asynchronously).
__global__ void merge_shards_kernel(int P, const float* __restrict__ lse_parts,
                                    const float* __restrict__ correct_parts,
                                    const int64_t* __restrict__ targets, int64_t ignore_index,
                                    int n, float* __restrict__ lse_out, float* __restrict__ loss_out,
                                    int64_t v_total, int* __restrict__ bad) {
  griddep_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float m = -INFINITY;
  for (int q = 0; q < P; ++q) m = fmaxf(m, lse_parts[(size_t)q * n + i]);
  float acc = 0.f, corr = 0.f;
  for (int q = 0; q < P; ++q) {
    const float l = lse_parts[(size_t)q * n + i];
    if (m != -INFINITY) acc += expf(l - m);
    corr += correct_parts[(size_t)q * n + i];
  }
  const float lse = (m == -INFINITY) ? -INFINITY : m + logf(acc);
  const int64_t tg = targets[i];
  const bool valid = tg != ignore_index;
  const bool out_of_range = valid && v_total > 0 && (tg < 0 || tg >= v_total);
  if (out_of_range && bad != nullptr) *bad = 1;
  lse_out[i] = valid ? lse : 0.f;
  loss_out[i] = out_of_range ? __int_as_float(0x7fc00000) : (valid ? lse - corr : 0.f);
}

// zero a float buffer (used for `correct` so rows whose label lives in another shard read 0)
// Zero n 32-bit words.  A kernel rather than cudaMemsetAsync: inside a chain of programmatic
// dependent launches a memset node is not ordered against the kernels around it.
__global__ void zero_words_kernel(int* __restrict__ x, int64_t n) {
  griddep_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = 0;
}

__global__ void fill_kernel(float* __restrict__ x, float v, int64_t n) {
  griddep_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = v;
}

// Column sums of E over valid rows, fp32, in a fixed order (bit-reproducible; the sort key and
// so the vocabulary order depend on it): block (x, y) writes the partial sum of rows
// [y * rows_per_block, +rows_per_block) to part[y][col]; ebar_reduce_kernel adds the partials in
// y order.
__global__ void ebar_kernel(const __nv_bfloat16* __restrict__ E, const int64_t* __restrict__ targets,
                            int64_t ignore_index, int n, int d, float* __restrict__ part,
                            int rows_per_block) {
  griddep_wait();
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= d) return;
  const int r0 = blockIdx.y * rows_per_block;
  const int r1 = min(n, r0 + rows_per_block);
  float acc = 0.f;
  for (int r = r0; r < r1; ++r)
    if (targets == nullptr || targets[r] != ignore_index) acc += __bfloat162float(E[(size_t)r * d + col]);
  part[(size_t)blockIdx.y * d + col] = acc;
}

__global__ void ebar_reduce_kernel(const float* __restrict__ part, int nblk, int d, float* __restrict__ ebar) {
  griddep_wait();
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= d) return;
  float acc = 0.f;
  for (int b = 0; b < nblk; ++b) acc += part[(size_t)b * d + col];
  ebar[col] = acc;
}

// key[v] = C[v] . ebar_sum / n_valid (fp32): the reference's mean_logits (kernels.py:305-308,
// :317-318), a mean of logits over the valid tokens.  HBM-bound GEMV: ebar in smem, one warp per
// row, 8 independent 16-byte loads in flight per lane.
#ifndef CCE_SORTKEY_UNROLL
#define CCE_SORTKEY_UNROLL 8  // independent 16-byte loads per lane per batch (profiles/r1/ab/sort_key_unroll.txt)
#endif
__global__ void sort_key_kernel(const __nv_bfloat16* __restrict__ C, const float* __restrict__ ebar_sum,
                                const int* __restrict__ n_valid, int v, int d, float* __restrict__ key) {
  griddep_wait();
  extern __shared__ float s_ebar[];
  for (int j = threadIdx.x; j < d; j += blockDim.x) s_ebar[j] = ebar_sum[j];
  __syncthreads();
  const float inv_n = *n_valid > 0 ? 1.0f / (float)*n_valid : 0.f;
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n16 = d / 8;
  for (int row = blockIdx.x * warps + (threadIdx.x >> 5); row < v; row += gridDim.x * warps) {
    const uint4* c = reinterpret_cast<const uint4*>(C + (size_t)row * d);
    constexpr int U = CCE_SORTKEY_UNROLL;
    float acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = 0.f;
    int j = lane;
    for (; j + 32 * (U - 1) < n16; j += 32 * U) {
      uint4 raw[U];
#pragma unroll
      for (int u = 0; u < U; ++u) raw[u] = __ldg(c + j + 32 * u);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&raw[u]);
        const float* eb = s_ebar + (j + 32 * u) * 8;
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[u] += __bfloat162float(h[q]) * eb[q];
      }
    }
    for (; j < n16; j += 32) {
      const uint4 raw = __ldg(c + j);
      const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[0] += __bfloat162float(h[q]) * s_ebar[j * 8 + q];
    }
#pragma unroll
    for (int u = 4; u < U; ++u) acc[u & 3] += acc[u];
    float a = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) key[row] = a * inv_n;
  }
}

// Stable compaction of the valid rows (filter_ignored, kernels.py:494-510), one block:
// row_map[k] = k-th row with targets != ignore_index, *n_valid = their count.  row_map must be
// pre-filled (entries past the count stay as they are, e.g. 0, so padded gathers stay in bounds).
__global__ void compact_rows_kernel(const int64_t* __restrict__ targets, int64_t ignore_index, int n,
                                    int32_t* __restrict__ row_map, int* __restrict__ n_valid) {
  griddep_wait();
  constexpr int T = 1024;
  __shared__ int s_warp[T / 32];
  __shared__ int s_base;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int c0 = 0; c0 < n; c0 += T) {
    const int i = c0 + threadIdx.x;
    const bool ok = i < n && targets[i] != ignore_index;
    const uint32_t bal = __ballot_sync(0xffffffffu, ok);
    const int before = __popc(bal & ((1u << lane) - 1));
    if (lane == 0) s_warp[wid] = __popc(bal);
    __syncthreads();
    if (wid == 0) {
      int x = s_warp[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      s_warp[lane] = x;  // inclusive
    }
    __syncthreads();
    const int base = s_base + (wid ? s_warp[wid - 1] : 0);
    if (ok) row_map[base + before] = i;
    __syncthreads();
    if (threadIdx.x == 0) s_base += s_warp[T / 32 - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_valid = s_base;
  // entries past the compacted count (up to the 128-row padding): row 0, so a gather of all n rows
  // (the compacted copy of E) reads only real rows
  const int pad = (n + BM - 1) / BM * BM;
  for (int j = s_base + threadIdx.x; j < pad; j += T) row_map[j] = 0;
}

// out[i] = C[x_i] . E[i] (indexed_matmul, kernels.py:204-251); one warp per token row.
__global__ void indexed_dot_kernel(const __nv_bfloat16* __restrict__ E, const __nv_bfloat16* __restrict__ C,
                                   const int64_t* __restrict__ targets, int64_t ignore_index,
                                   int64_t vocab_start, int n, int d, int v, float softcap,
                                   float* __restrict__ out) {
  griddep_wait();
  const int warps = blockDim.x >> 5;
  const int row = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const int64_t tg = targets[row];
  const int64_t l = tg - vocab_start;
  if (tg == ignore_index || l < 0 || l >= v) {
    if (lane == 0) out[row] = 0.f;
    return;
  }
  const __nv_bfloat16* e = E + (size_t)row * d;
  const __nv_bfloat16* c = C + (size_t)l * d;
  float acc = 0.f;
  for (int j = lane * 8; j < d; j += 256) {
    const uint4 re = *reinterpret_cast<const uint4*>(e + j);
    const uint4 rc = *reinterpret_cast<const uint4*>(c + j);
    const __nv_bfloat16* he = reinterpret_cast<const __nv_bfloat16*>(&re);
    const __nv_bfloat16* hc = reinterpret_cast<const __nv_bfloat16*>(&rc);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += __bfloat162float(he[q]) * __bfloat162float(hc[q]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[row] = softcap > 0.f ? softcap * tanhf(acc / softcap) : acc;
}

__global__ void iota_kernel(int32_t* __restrict__ x, int n) {
  griddep_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = i;
}

// inv[perm[j]] = j for j < v ; padding positions of perm (>= v) point at row 0.
__global__ void invert_perm_kernel(const int32_t* __restrict__ perm, int v, int vpad,
                                   int32_t* __restrict__ perm_padded, int32_t* __restrict__ inv) {
  griddep_wait();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= vpad) return;
  if (j < v) {
    const int32_t r = perm[j];
    perm_padded[j] = r;
    inv[r] = j;
  } else {
    perm_padded[j] = 0;
  }
}

// pos[i] = tile-order position of row i's label (or -1: ignored / label owned by another shard)
__global__ void label_pos_kernel(const int64_t* __restrict__ targets, int64_t ignore_index,
                                 int64_t vocab_start, int v, const int32_t* __restrict__ inv,
                                 int n, int32_t* __restrict__ pos) {
  griddep_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t tg = targets[i];
  int32_t r = -1;
  if (tg != ignore_index) {
    const int64_t l = tg - vocab_start;
    if (l >= 0 && l < v) r = inv ? inv[l] : (int32_t)l;
  }
  pos[i] = r;
}

// block_zero[b] = every upstream of compact token tile b is exactly zero (kernels.py:434-438)
__global__ void block_zero_kernel(const float* __restrict__ up, const int32_t* __restrict__ row_map,
                                  const int* __restrict__ n_valid, uint8_t* __restrict__ bz) {
  griddep_wait();
  const int b = blockIdx.x;
  const int i = b * BM + threadIdx.x;
  const bool nz = (i < *n_valid) && (up[row_map[i]] != 0.f);
  const int any = __syncthreads_or(nz);
  if (threadIdx.x == 0) bz[b] = any ? 0 : 1;
}

// dst[i, :] = src[index[i], :] for bf16 rows of `cols` elements (cols % 8 == 0); one warp per row.
// Materialises the vocabulary-sorted classifier C[perm] for the backward so every tile load is a
// plain TMA box instead of 64 tile::gather4 transfers.
__global__ void gather_rows_kernel(const __nv_bfloat16* __restrict__ src, const int32_t* __restrict__ index,
                                   int64_t rows, int cols, __nv_bfloat16* __restrict__ dst) {
  griddep_wait();
  const int warps = blockDim.x >> 5;
  const int64_t r = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const uint4* s = reinterpret_cast<const uint4*>(src + (size_t)index[r] * cols);
  uint4* d = reinterpret_cast<uint4*>(dst + (size_t)r * cols);
  const int n16 = cols / 8;
#pragma unroll 4
  for (int j = lane; j < n16; j += 32) d[j] = __ldg(s + j);
}

// ---------------------------------------------------------------------------------------
// Filter decision from the forward's tile maxima (lse_backward's skip test, kernels.py:434-455,
// taken without recomputing any logit tile)
// ---------------------------------------------------------------------------------------

// keep[m * nt + n] = 1 iff compact token tile n must be recomputed against vocab tile m: its
// upstream is not all zero (kernels.py:434-438) and it holds a label (kernels.py:447-455) or some
// row's largest S = exp(z' - lse) is >= eps (block_skip_decision, kernels.py:140-142, strict <).
// tile_max[(n * mt + m) * 128 + r] is the forward's max raw logit of row r in tile (n, m);
// tile_row_big is the same test the in-kernel filter (cce_lse_kernel<BWD>) applies.
// Grid (ceil(mt / DECIDE_VT), nt), 256 threads: warp w takes vocab tiles blockIdx.x * DECIDE_VT +
// w + 8j, lane l rows 4l .. 4l + 3.  counters[1] += eps-skipped, counters[2] += zero-upstream-
// skipped tiles.  16 vocab tiles per block keeps the grid wide for vocabulary groups too.
constexpr int DECIDE_VT = 16;
__global__ void decide_tiles_kernel(const float* __restrict__ tile_max, const float* __restrict__ lse,
                                    const int32_t* __restrict__ pos, int pos_offset, const int32_t* __restrict__ row_map,
                                    const int* __restrict__ n_valid, const uint8_t* __restrict__ block_zero,
                                    int nt, int mt, float softcap, float eps, int label_split,
                                    uint8_t* __restrict__ keep, unsigned long long* __restrict__ counters) {
  griddep_wait();
  __shared__ unsigned s_cnt[2];
  const int n = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nv = *n_valid;
  const int nt_dev = (nv + BM - 1) / BM;
  const int m_lo = blockIdx.x * DECIDE_VT;
  const int m_hi = min(mt, m_lo + DECIDE_VT);
  if (threadIdx.x < 2) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  if (n >= nt_dev) {  // token tile past the compacted rows: not a tile of this backward
    for (int m = m_lo + threadIdx.x; m < m_hi; m += blockDim.x) keep[(size_t)m * nt + n] = 0;
    return;
  }
  if (block_zero[n]) {
    for (int m = m_lo + threadIdx.x; m < m_hi; m += blockDim.x) keep[(size_t)m * nt + n] = 0;
    if (threadIdx.x == 0) atomicAdd(&counters[2], (unsigned long long)(m_hi - m_lo));
    return;
  }
  const bool use_softcap = softcap > 0.f;
  const float inv_cap = use_softcap ? 1.0f / softcap : 0.f;
  float lse2[4];
  int pr[4];
  bool ok[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int grow = n * BM + 4 * lane + k;
    ok[k] = grow < nv;
    const int orow = ok[k] ? row_map[grow] : 0;
    lse2[k] = ok[k] ? lse[orow] * LOG2E : INFINITY;
    pr[k] = ok[k] ? pos[orow] - pos_offset : -1;  // vocabulary group: group-local position
  }
  unsigned skipped = 0;
  for (int m = m_lo + warp; m < m_hi; m += 8) {
    const float4 z = reinterpret_cast<const float4*>(tile_max + ((size_t)n * mt + m) * BM)[lane];
    const float zz[4] = {z.x, z.y, z.z, z.w};
    bool any = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      any |= ok[k] && tile_row_big(zz[k], lse2[k], softcap, inv_cap, eps);
      any |= !label_split && pr[k] >= m * BN && pr[k] < (m + 1) * BN;
    }
    const bool kept = __any_sync(0xffffffffu, any);
    if (lane == 0) {
      keep[(size_t)m * nt + n] = kept ? 1 : 0;
      skipped += kept ? 0 : 1;
    }
  }
  if (lane == 0 && skipped) atomicAdd(&s_cnt[0], skipped);
  __syncthreads();
  if (threadIdx.x == 0 && s_cnt[0]) atomicAdd(&counters[1], (unsigned long long)s_cnt[0]);
}

// block-wide sum (any block size that is a multiple of 32, <= 1024)
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* s_tmp) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) s_tmp[wid] = v;
  __syncthreads();
  T r = 0;
  if (wid == 0) {
    r = lane < (int)(blockDim.x >> 5) ? s_tmp[lane] : T(0);
#pragma unroll
    for (int o = 16; o; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    if (lane == 0) s_tmp[0] = r;
  }
  __syncthreads();
  r = s_tmp[0];
  __syncthreads();
  return r;
}

// Kept-tile list of the token tiles [n_lo, n_lo + g) in vocab-tile-major order (slot = list
// position, so concurrently running CTAs of the KEPT pass share C tiles), in three parallel
// steps: list_count_kernel (block per vocab tile) -> list_scan_kernel (one block: offsets,
// list_count, capacity flags, counter resets) -> list_fill_kernel (block per vocab tile: list,
// every slot_of entry (slot or -1), cnt_n).  All run only if run_if is null or *run_if != 0.
__global__ void list_count_kernel(const uint8_t* __restrict__ keep, int nt, int mt, int n_lo, int g,
                                  const int* run_if, const int32_t* __restrict__ lab_slot,
                                  int* __restrict__ cnt_m, int* __restrict__ rcnt_m) {
  griddep_wait();
  if (run_if != nullptr && *run_if == 0) return;
  __shared__ int s_w[32];
  const int m = blockIdx.x;
  const uint8_t* row = keep + (size_t)m * nt + n_lo;
  int c = 0, r = 0;
  for (int i = threadIdx.x; i < g; i += blockDim.x) {
    const int k = row[i];
    c += k;
    r += k && (lab_slot == nullptr || lab_slot[(size_t)(n_lo + i) * mt + m] < 0);
  }
  c = block_sum(c, s_w);
  r = block_sum(r, s_w);
  if (threadIdx.x == 0) {
    cnt_m[m] = c;
    rcnt_m[m] = r;
  }
}

// cnt_m -> off_m and rcnt_m -> roff_m (exclusive); *list_count = kept tiles, *rlist_count = tiles
// to recompute; primary: counters[0] += kept and *ok / *overflow (every tile to recompute got a
// slot or not); resets cnt_n[0..g) and the dE unit counter.
__global__ void __launch_bounds__(1024) list_scan_kernel(const int* __restrict__ cnt_m,
                                                         const int* __restrict__ rcnt_m, int mt, int g,
                                                         int capacity, const int* run_if, int primary,
                                                         int* __restrict__ off_m, int* __restrict__ roff_m,
                                                         int* __restrict__ cnt_n, int* __restrict__ list_count,
                                                         int* __restrict__ rlist_count, int* __restrict__ ok,
                                                         int* __restrict__ overflow, int* __restrict__ sched,
                                                         unsigned long long* __restrict__ counters) {
  griddep_wait();
  if (run_if != nullptr && *run_if == 0) return;
  constexpr int T = 1024;
  __shared__ int s_a[32], s_b[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < g; i += T) cnt_n[i] = 0;
  if (threadIdx.x == 0 && sched) *sched = 0;
  const int per = (mt + T - 1) / T;
  const int m0 = threadIdx.x * per, m1 = min(mt, m0 + per);
  int la = 0, lb = 0;
  for (int m = m0; m < m1; ++m) {
    la += cnt_m[m];
    lb += rcnt_m[m];
  }
  int ia = la, ib = lb;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int ya = __shfl_up_sync(0xffffffffu, ia, o), yb = __shfl_up_sync(0xffffffffu, ib, o);
    if (lane >= o) { ia += ya; ib += yb; }
  }
  if (lane == 31) { s_a[wid] = ia; s_b[wid] = ib; }
  __syncthreads();
  if (wid == 0) {
    int xa = s_a[lane], xb = s_b[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ya = __shfl_up_sync(0xffffffffu, xa, o), yb = __shfl_up_sync(0xffffffffu, xb, o);
      if (lane >= o) { xa += ya; xb += yb; }
    }
    s_a[lane] = xa;
    s_b[lane] = xb;
  }
  __syncthreads();
  int ra = (wid ? s_a[wid - 1] : 0) + ia - la, rb = (wid ? s_b[wid - 1] : 0) + ib - lb;
  for (int m = m0; m < m1; ++m) {
    off_m[m] = ra;
    roff_m[m] = rb;
    ra += cnt_m[m];
    rb += rcnt_m[m];
  }
  if (threadIdx.x == 0) {
    const int kept_total = s_a[31], recompute = s_b[31];
    *list_count = kept_total;
    *rlist_count = recompute;
    if (primary) {
      const bool fits = recompute <= capacity;
      *ok = fits ? 1 : 0;
      *overflow = fits ? 0 : 1;
      atomicAdd(&counters[0], (unsigned long long)kept_total);
    }
  }
}

// block per vocab tile m, token-tile order: every kept tile gets a unified slot -- its stored
// label slot (lab_slot >= 0), else lab_capacity + its place in the recompute list; the all-kept
// list (for dC) holds (token tile, slot) at off_m[m] + rank, the recompute list (for KEPT) holds
// (token tile, vocab tile) at roff_m[m] + rank; slot_of row-major [g][mt] with the local token-tile
// index (every entry written).  Recompute tiles past the capacity get no slot (only when the
// caller's gate then skips every consumer).
__global__ void list_fill_kernel(const uint8_t* __restrict__ keep, int nt, int mt, int n_lo, int g,
                                 int capacity, int lab_capacity, const int32_t* __restrict__ lab_slot,
                                 const int* run_if, const int* __restrict__ off_m, const int* __restrict__ roff_m,
                                 int2* __restrict__ alist, int2* __restrict__ rlist, int32_t* __restrict__ slot_of,
                                 int* __restrict__ cnt_n) {
  griddep_wait();
  if (run_if != nullptr && *run_if == 0) return;
  __shared__ int s_a[32], s_b[32];
  __shared__ int s_base, s_rbase;
  const int m = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint8_t* row = keep + (size_t)m * nt + n_lo;
  if (threadIdx.x == 0) {
    s_base = off_m[m];
    s_rbase = roff_m[m];
  }
  __syncthreads();
  for (int b = 0; b < g; b += blockDim.x) {
    const int ln = b + threadIdx.x;
    const bool f = ln < g && row[ln];
    const int ls = f && lab_slot ? lab_slot[(size_t)(n_lo + ln) * mt + m] : -1;
    const bool rc = f && ls < 0;
    const uint32_t bal = __ballot_sync(0xffffffffu, f), rbal = __ballot_sync(0xffffffffu, rc);
    if (lane == 0) {
      s_a[wid] = __popc(bal);
      s_b[wid] = __popc(rbal);
    }
    __syncthreads();
    int before = 0, rbefore = 0;
    for (int w = 0; w < wid; ++w) {
      before += s_a[w];
      rbefore += s_b[w];
    }
    const int apos = s_base + before + __popc(bal & ((1u << lane) - 1));
    const int rpos = s_rbase + rbefore + __popc(rbal & ((1u << lane) - 1));
    if (ln < g) {
      int so = -1;
      if (f) {
        if (ls >= 0) {
          so = ls;
        } else if (rpos < capacity) {
          so = lab_capacity + rpos;
          rlist[rpos] = make_int2(n_lo + ln, m);
        }
        if (so >= 0) {
          alist[apos] = make_int2(n_lo + ln, so);
          atomicAdd(&cnt_n[ln], 1);
        }
      }
      slot_of[(size_t)ln * mt + m] = so;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int ta = 0, tb = 0;
      for (int w = 0; w < nw; ++w) {
        ta += s_a[w];
        tb += s_b[w];
      }
      s_base += ta;
      s_rbase += tb;
    }
    __syncthreads();
  }
}

// In-place S-hat of the stored label tiles: fp16 d = z' - z'max(row) -> bf16
// up * (S - onehot) * (1 - tanh^2), S = exp(z'max + d - lse) (same formula as the KEPT epilogue,
// from the stored logits instead of a recompute).  One block of 8 warps per slot; a warp takes a
// row at a time (lane = 8 consecutive columns: one coalesced 512 B row per access), two rows in
// flight.  Tiles of zero-upstream token tiles are never kept and are left alone.
__global__ void __launch_bounds__(256) label_shat_kernel(
    __half* buf, const int2* __restrict__ lab_list, const int* __restrict__ lab_count, int lab_capacity,
    const uint8_t* __restrict__ block_zero, int mt, const float* __restrict__ tile_max,
    const float* __restrict__ lse, const float* __restrict__ upstream, const int32_t* __restrict__ pos,
    const int32_t* __restrict__ row_map, const int* __restrict__ n_valid, int v, float softcap, int label_split) {
  griddep_wait();
  const int s = blockIdx.x;
  if (s >= min(*lab_count, lab_capacity)) return;
  const int2 nm = lab_list[s];
  if (block_zero[nm.x]) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nv = *n_valid;
  const bool use_softcap = softcap > 0.f;
  const float inv_cap = use_softcap ? 1.0f / softcap : 0.f;
  const int col_base = nm.y * BN + lane * 8;
  constexpr int R = 2;  // rows per iteration (independent loads in flight)
  for (int r0 = warp * R; r0 < BM; r0 += 8 * R) {
    uint4 in[R];
    float lse2[R], up[R], zc0[R];
    int pr[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int row = r0 + i;
      const int grow = nm.x * BM + row;
      const bool valid = grow < nv;
      const int orow = valid ? row_map[grow] : 0;
      lse2[i] = valid ? lse[orow] * LOG2E : INFINITY;
      up[i] = valid ? upstream[orow] : 0.f;
      pr[i] = (valid && !label_split) ? pos[orow] : -1;
      const float zmax = tile_max[((size_t)nm.x * mt + nm.y) * BM + row];
      zc0[i] = use_softcap ? softcap * softcap_tanh(zmax, inv_cap) : zmax;
      in[i] = reinterpret_cast<const uint4*>(buf + ((size_t)s * BM + row) * BN)[lane];
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const __half2* h2 = reinterpret_cast<const __half2*>(&in[i]);
      uint32_t o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 d = __half22float2(h2[k]);
        float g[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = col_base + 2 * k + h;
          g[h] = 0.f;
          if (col < v) {  // padded columns hold -inf
            const float zc = zc0[i] + (h ? d.y : d.x);
            const float sv = ex2_approx(zc * LOG2E - lse2[i]);
            float dcap = 1.f;
            if (use_softcap) {
              const float th = zc * inv_cap;
              dcap = 1.f - th * th;
            }
            g[h] = ((col == pr[i]) ? sv - 1.f : sv) * up[i] * dcap;
          }
        }
        o[k] = pack_bf16x2(g[0], g[1]);
      }
      reinterpret_cast<uint4*>(buf + ((size_t)s * BM + r0 + i) * BN)[lane] = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

// Fallback passes (token-tile groups after an overflow, gated on run_if): everything
// list_count / list_scan / list_fill / build_pairs produce for the group, in ONE block, so a pass
// that does not run costs one launch here instead of four.
__global__ void __launch_bounds__(1024) list_single_kernel(
    const uint8_t* __restrict__ keep, int nt, int mt, int n_lo, int g, int capacity, int lab_capacity,
    const int32_t* __restrict__ lab_slot, const int* run_if, int* __restrict__ cnt_m, int* __restrict__ rcnt_m,
    int* __restrict__ off_m, int* __restrict__ roff_m, int2* __restrict__ alist, int2* __restrict__ rlist,
    int32_t* __restrict__ slot_of, int* __restrict__ cnt_n, int* __restrict__ list_count,
    int* __restrict__ rlist_count, int* __restrict__ sched, int2* __restrict__ pairs, int* __restrict__ pair_count) {
  griddep_wait();
  if (run_if != nullptr && *run_if == 0) return;
  constexpr int T = 1024, W = T / 32;
  __shared__ int s_a[W], s_b[W], s_c[W];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < g; i += T) cnt_n[i] = 0;
  if (threadIdx.x == 0 && sched) *sched = 0;
  auto is_lab = [&](int ln, int m) { return lab_slot != nullptr && lab_slot[(size_t)(n_lo + ln) * mt + m] >= 0; };
  for (int m = wid; m < mt; m += W) {  // counts per vocab tile: kept, to recompute
    const uint8_t* row = keep + (size_t)m * nt + n_lo;
    int c = 0, r = 0;
    for (int b = 0; b < g; b += 32) {
      const bool f = b + lane < g && row[b + lane];
      c += __popc(__ballot_sync(0xffffffffu, f));
      r += __popc(__ballot_sync(0xffffffffu, f && !is_lab(b + lane, m)));
    }
    if (lane == 0) {
      cnt_m[m] = c;
      rcnt_m[m] = r;
    }
  }
  __syncthreads();
  // exclusive scans: kept slots, recompute slots, recompute pairs ((r + 1) / 2)
  const int per = (mt + T - 1) / T;
  const int m0 = threadIdx.x * per, m1 = min(mt, m0 + per);
  int la = 0, lb = 0, lc = 0;
  for (int m = m0; m < m1; ++m) {
    la += cnt_m[m];
    lb += rcnt_m[m];
    lc += (rcnt_m[m] + 1) / 2;
  }
  int ia = la, ib = lb, ic = lc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int ya = __shfl_up_sync(0xffffffffu, ia, o), yb = __shfl_up_sync(0xffffffffu, ib, o);
    const int yc = __shfl_up_sync(0xffffffffu, ic, o);
    if (lane >= o) { ia += ya; ib += yb; ic += yc; }
  }
  if (lane == 31) { s_a[wid] = ia; s_b[wid] = ib; s_c[wid] = ic; }
  __syncthreads();
  if (wid == 0) {
    int xa = s_a[lane], xb = s_b[lane], xc = s_c[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ya = __shfl_up_sync(0xffffffffu, xa, o), yb = __shfl_up_sync(0xffffffffu, xb, o);
      const int yc = __shfl_up_sync(0xffffffffu, xc, o);
      if (lane >= o) { xa += ya; xb += yb; xc += yc; }
    }
    s_a[lane] = xa;
    s_b[lane] = xb;
    s_c[lane] = xc;
  }
  __syncthreads();
  int ra = (wid ? s_a[wid - 1] : 0) + ia - la, rb = (wid ? s_b[wid - 1] : 0) + ib - lb;
  int rc = (wid ? s_c[wid - 1] : 0) + ic - lc;
  for (int m = m0; m < m1; ++m) {
    const int r = rcnt_m[m];
    off_m[m] = ra;
    roff_m[m] = rb;
    for (int j = 0; 2 * j < r; ++j) pairs[rc + j] = make_int2(rb + 2 * j, min(2, r - 2 * j));
    ra += cnt_m[m];
    rb += r;
    rc += (r + 1) / 2;
  }
  if (threadIdx.x == T - 1) {
    *list_count = ra;
    *rlist_count = rb;
    *pair_count = rc;
  }
  __syncthreads();
  for (int m = wid; m < mt; m += W) {  // slots in vocab-tile-major, token-tile order
    const uint8_t* row = keep + (size_t)m * nt + n_lo;
    int a0 = off_m[m], r0 = roff_m[m];
    for (int b = 0; b < g; b += 32) {
      const int ln = b + lane;
      const bool f = ln < g && row[ln];
      const int ls = f && lab_slot ? lab_slot[(size_t)(n_lo + ln) * mt + m] : -1;
      const bool rcp = f && ls < 0;
      const uint32_t bal = __ballot_sync(0xffffffffu, f), rbal = __ballot_sync(0xffffffffu, rcp);
      const int apos = a0 + __popc(bal & ((1u << lane) - 1));
      const int rpos = r0 + __popc(rbal & ((1u << lane) - 1));
      if (ln < g) {
        int so = -1;
        if (f) {
          if (ls >= 0) {
            so = ls;
          } else if (rpos < capacity) {
            so = lab_capacity + rpos;
            rlist[rpos] = make_int2(n_lo + ln, m);
          }
          if (so >= 0) {
            alist[apos] = make_int2(n_lo + ln, so);
            atomicAdd(&cnt_n[ln], 1);
          }
        }
        slot_of[(size_t)ln * mt + m] = so;
      }
      a0 += __popc(bal);
      r0 += __popc(rbal);
    }
  }
}

// One block: CTA-pair work list of the KEPT pass.  The kept tiles of vocab tile m hold the
// consecutive slots [off_m, off_m + cnt_m) (list_fill_kernel); pair j of m takes slots
// off_m + 2j and, if it exists, off_m + 2j + 1.  pairs[k] = (first slot, tiles in the pair).
__global__ void __launch_bounds__(1024) build_pairs_kernel(const int* __restrict__ cnt_m, int mt,
                                                           const int* run_if, int2* __restrict__ pairs,
                                                           int* __restrict__ pair_count) {
  griddep_wait();
  if (run_if != nullptr && *run_if == 0) return;
  constexpr int T = 1024;
  __shared__ int s_a[T / 32], s_b[T / 32];
  const int per = (mt + T - 1) / T;
  const int m0 = threadIdx.x * per, m1 = min(mt, m0 + per);
  int slots = 0, np = 0;
  for (int m = m0; m < m1; ++m) {
    slots += cnt_m[m];
    np += (cnt_m[m] + 1) / 2;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int ia = slots, ib = np;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int ya = __shfl_up_sync(0xffffffffu, ia, o);
    const int yb = __shfl_up_sync(0xffffffffu, ib, o);
    if (lane >= o) { ia += ya; ib += yb; }
  }
  if (lane == 31) { s_a[wid] = ia; s_b[wid] = ib; }
  __syncthreads();
  if (wid == 0) {
    int xa = s_a[lane], xb = s_b[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ya = __shfl_up_sync(0xffffffffu, xa, o);
      const int yb = __shfl_up_sync(0xffffffffu, xb, o);
      if (lane >= o) { xa += ya; xb += yb; }
    }
    s_a[lane] = xa;
    s_b[lane] = xb;
  }
  __syncthreads();
  int off = (wid ? s_a[wid - 1] : 0) + ia - slots;
  int poff = (wid ? s_b[wid - 1] : 0) + ib - np;
  for (int m = m0; m < m1; ++m) {
    const int c = cnt_m[m];
    for (int j = 0; 2 * j < c; ++j) pairs[poff + j] = make_int2(off + 2 * j, min(2, c - 2 * j));
    off += c;
    poff += (c + 1) / 2;
  }
  if (threadIdx.x == T - 1) *pair_count = poff;
}

// ---------------------------------------------------------------------------------------
// Label term of the paper ordering: with tiles filtered on S alone,
// the -1 at each label is applied here, exactly, as the backward of the indexed matmul:
//   dE[i] += coef_i * C[x_i],  dC[x_i] += sum over tokens i with label x_i of coef_i * E[i],
//   coef_i = -upstream_i * (1 - tanh^2(z_i / cap)),  tanh = correct_i / cap (softcap), else 1.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ float label_coef(const float* up, const float* correct, float softcap, int orow) {
  float dcap = 1.f;
  if (softcap > 0.f) {
    const float t = correct[orow] / softcap;
    dcap = 1.f - t * t;
  }
  return -up[orow] * dcap;
}

// sort keys: label position in tile order of each compact row (INT_MAX: no label here)
__global__ void label_keys_kernel(const int32_t* __restrict__ row_map, const int* __restrict__ n_valid,
                                  const int32_t* __restrict__ pos, int n, int32_t* __restrict__ key,
                                  int32_t* __restrict__ val) {
  griddep_wait();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int32_t kk = INT_MAX, vv = 0;
  if (k < *n_valid) {
    vv = row_map[k];
    const int32_t p = pos[vv];
    if (p >= 0) kk = p;
  }
  key[k] = kk;
  val[k] = vv;
}

// dC: blocks stride over the sorted entries (blockIdx.y = a 256-column chunk of D); the first
// entry of each label run sums the run in sort order (deterministic, one fp32 sum per column,
// one bf16 rounding into that classifier row).  The run's rows and coefficients are staged in
// shared memory 512 at a time, so the E loads of a column are independent and pipeline: with
// Zipf-distributed labels one run can hold hundreds of tokens.
constexpr int LABEL_DC_CHUNK = 512;
__global__ void __launch_bounds__(256) label_dc_kernel(
    const int32_t* __restrict__ key, const int32_t* __restrict__ val, int n, const __nv_bfloat16* __restrict__ E,
    const float* __restrict__ up, const float* __restrict__ correct, float softcap,
    const int32_t* __restrict__ perm, int d, __nv_bfloat16* __restrict__ dc) {
  griddep_wait();
  __shared__ int s_row[LABEL_DC_CHUNK];
  __shared__ float s_coef[LABEL_DC_CHUNK];
  const int col = blockIdx.y * blockDim.x + threadIdx.x;
  for (int k = blockIdx.x; k < n; k += gridDim.x) {
    const int32_t p = key[k];
    if (p == INT_MAX || (k > 0 && key[k - 1] == p)) continue;  // not the head of a label run
    float acc = 0.f;
    for (int j0 = k;; j0 += LABEL_DC_CHUNK) {
      __syncthreads();
      for (int t = threadIdx.x; t < LABEL_DC_CHUNK; t += blockDim.x) {
        const int j = j0 + t;
        const bool in = j < n && key[j] == p;  // a run is contiguous: valid entries form a prefix
        const int orow = in ? val[j] : -1;
        s_row[t] = orow;
        s_coef[t] = in ? label_coef(up, correct, softcap, orow) : 0.f;
      }
      __syncthreads();
      if (col < d) {
#pragma unroll 4
        for (int t = 0; t < LABEL_DC_CHUNK; ++t) {
          const int orow = s_row[t];
          if (orow < 0) break;
          acc += s_coef[t] * __bfloat162float(E[(size_t)orow * d + col]);
        }
      }
      if (s_row[LABEL_DC_CHUNK - 1] < 0) break;  // the run ended inside this chunk (uniform)
    }
    if (col < d) {
      const int crow = perm ? perm[p] : p;
      __nv_bfloat16* dst = dc + (size_t)crow * d + col;
      *dst = __float2bfloat16(__bfloat162float(*dst) + acc);
    }
  }
}

// dE: one warp per compact row with a label here
__global__ void label_de_kernel(const int32_t* __restrict__ row_map, const int* __restrict__ n_valid,
                                const int32_t* __restrict__ pos, const __nv_bfloat16* __restrict__ C,
                                const int32_t* __restrict__ perm, const float* __restrict__ up,
                                const float* __restrict__ correct, float softcap, int n, int d,
                                float* __restrict__ de_f32, __nv_bfloat16* __restrict__ de_bf16) {
  griddep_wait();
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (k >= n || k >= *n_valid) return;
  const int orow = row_map[k];
  const int32_t p = pos[orow];
  if (p < 0) return;
  const int crow = perm ? perm[p] : p;
  const float coef = label_coef(up, correct, softcap, orow);
  const __nv_bfloat16* c = C + (size_t)crow * d;
  for (int col = lane; col < d; col += 32) {
    const float add = coef * __bfloat162float(c[col]);
    const size_t o = (size_t)orow * d + col;
    if (de_f32)
      de_f32[o] += add;
    else
      de_bf16[o] = __float2bfloat16(__bfloat162float(de_bf16[o]) + add);
  }
}

// ---------------------------------------------------------------------------------------
// Reductions of linear_cross_entropy (default_upstream, core.py:181-200), one block, fixed order
// ---------------------------------------------------------------------------------------
// out = sum(loss) (reduction 1) or sum(loss) / n_valid, 0 when nothing is valid (reduction 2)
__global__ void __launch_bounds__(1024) reduce_loss_kernel(const float* __restrict__ loss,
                                                           const int64_t* __restrict__ targets,
                                                           int64_t ignore_index, int n, int reduction,
                                                           float* __restrict__ out) {
  griddep_wait();
  __shared__ float s_f[32];
  __shared__ int s_i[32];
  float acc = 0.f;
  int cnt = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    acc += loss[i];
    cnt += targets[i] != ignore_index;
  }
  const float total = block_sum(acc, s_f);
  const int nv = block_sum(cnt, s_i);
  if (threadIdx.x == 0) *out = reduction == 1 ? total : (nv > 0 ? total / (float)nv : 0.f);
}

// up[i] = valid_i * g (reduction 1), valid_i * g / n_valid (2), valid_i * g[i] (0: g is [n])
__global__ void __launch_bounds__(1024) upstream_kernel(const float* __restrict__ g,
                                                        const int64_t* __restrict__ targets,
                                                        int64_t ignore_index, int n, int reduction,
                                                        float* __restrict__ up) {
  griddep_wait();
  __shared__ int s_i[32];
  int cnt = 0;
  if (reduction == 2)
    for (int i = threadIdx.x; i < n; i += blockDim.x) cnt += targets[i] != ignore_index;
  const int nv = reduction == 2 ? block_sum(cnt, s_i) : 1;
  const float scale = reduction == 2 ? (nv > 0 ? 1.f / (float)nv : 0.f) : 1.f;
  const float g0 = reduction == 0 ? 0.f : *g;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const bool valid = targets[i] != ignore_index;
    const float gi = reduction == 0 ? g[i] : g0;
    up[i] = valid ? gi * scale : 0.f;
  }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                   int64_t n4) {
  griddep_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n4) return;
  const float4 v = reinterpret_cast<const float4*>(x)[i];
  uint2 o;
  o.x = pack_bf16x2(v.x, v.y);
  o.y = pack_bf16x2(v.z, v.w);
  reinterpret_cast<uint2*>(y)[i] = o;
}

}  // namespace cce

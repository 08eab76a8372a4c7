// Streamed backward (cce_bwd_stream): lse_backward (kernels.py:327-486) with transient memory
// bounded independently of the kept-tile count.
//
// The decision from the forward's tile maxima (decide_tiles_kernel) gives the kept tiles.  Two
// passes then recompute them, each in one persistent kernel whose CTAs split into two roles:
//   producers  the KEPT logit-tile body (cce_lse_kernel.cuh) recomputing kept tiles in stream
//              order and writing S-hat into a ring of R slots in HBM (L2-resident at R = 256);
//   consumers  the dE body (token pass: items in token-tile-major order, units = (segment, D
//              chunk)) or the dC body (vocab pass: vocab-tile-major, CTA pairs, units = (segment,
//              D chunk, vocab half)) reading S-hat from the ring with TMA.
// Slot reuse and readiness are counted with GPU-scope release / acquire flags (Stream in
// cce_common.cuh); a segment is a run of at most B items of one owner, an owner with several
// segments sums them in segment order through an fp32 region (deterministic).  Progress is
// guaranteed with every CTA resident (grid = SM count, one CTA per SM): producers take items in
// increasing order, consumers take units in increasing order, and every wait is on an earlier item,
// segment or owner.
//
// The vocab pass writes dC in the sorted order into the storage of the sorted classifier copy the
// token pass read; unpermute_* put the rows back in vocabulary order in place (cycle segments).
#pragma once
#include "cce_grad_kernels.cuh"
#include "cce_lse_kernel.cuh"

namespace cce {

// kept tiles of each token tile: cnt[n] = sum over m of keep[m * nt + n] (block per token tile)
__global__ void __launch_bounds__(256) tok_count_kernel(const uint8_t* __restrict__ keep, int nt, int mt,
                                                        int* __restrict__ cnt) {
  griddep_wait();
  __shared__ int s_w[8];
  const int n = blockIdx.x;
  int c = 0;
  for (int m = threadIdx.x; m < mt; m += blockDim.x) c += keep[(size_t)m * nt + n];
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < 8; ++w) t += s_w[w];
    cnt[n] = t;
  }
}

// One block: owners o < owners with cnt[o] items -> exclusive offsets off[o], *total, and the
// segments: owner o gets max(1, ceil(cnt / B)) segments of near-equal size, seg[k] = (owner, first
// item, items, split), seg_aux[k] = (splits of the owner, accumulator id = rank of the owner among
// owners with more than one split).  counters[0] += total when counters is given.
__global__ void __launch_bounds__(1024) segments_kernel(const int* __restrict__ cnt, int owners, int B,
                                                        int* __restrict__ off, int* __restrict__ total,
                                                        int4* __restrict__ seg, int2* __restrict__ seg_aux,
                                                        int* __restrict__ seg_count,
                                                        unsigned long long* __restrict__ counters) {
  griddep_wait();
  constexpr int T = 1024;
  __shared__ int s_a[32], s_b[32], s_c[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int per = (owners + T - 1) / T;
  const int o0 = threadIdx.x * per, o1 = min(owners, o0 + per);
  auto nseg = [&](int c) { return max(1, (c + B - 1) / B); };
  int la = 0, lb = 0, lc = 0;
  for (int o = o0; o < o1; ++o) {
    const int c = cnt[o], ns = nseg(c);
    la += c;
    lb += ns;
    lc += ns > 1;
  }
  int ia = la, ib = lb, ic = lc;
#pragma unroll
  for (int k = 1; k < 32; k <<= 1) {
    const int ya = __shfl_up_sync(0xffffffffu, ia, k), yb = __shfl_up_sync(0xffffffffu, ib, k),
              yc = __shfl_up_sync(0xffffffffu, ic, k);
    if (lane >= k) {
      ia += ya;
      ib += yb;
      ic += yc;
    }
  }
  if (lane == 31) {
    s_a[wid] = ia;
    s_b[wid] = ib;
    s_c[wid] = ic;
  }
  __syncthreads();
  if (wid == 0) {
    int xa = s_a[lane], xb = s_b[lane], xc = s_c[lane];
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
      const int ya = __shfl_up_sync(0xffffffffu, xa, k), yb = __shfl_up_sync(0xffffffffu, xb, k),
                yc = __shfl_up_sync(0xffffffffu, xc, k);
      if (lane >= k) {
        xa += ya;
        xb += yb;
        xc += yc;
      }
    }
    s_a[lane] = xa;
    s_b[lane] = xb;
    s_c[lane] = xc;
  }
  __syncthreads();
  int ra = (wid ? s_a[wid - 1] : 0) + ia - la;
  int rb = (wid ? s_b[wid - 1] : 0) + ib - lb;
  int rc = (wid ? s_c[wid - 1] : 0) + ic - lc;
  for (int o = o0; o < o1; ++o) {
    const int c = cnt[o], ns = nseg(c);
    off[o] = ra;
    for (int s = 0; s < ns; ++s) {
      const int i0 = (int)(((long long)s * c) / ns), i1 = (int)(((long long)(s + 1) * c) / ns);
      seg[rb + s] = make_int4(o, ra + i0, i1 - i0, s);
      seg_aux[rb + s] = make_int2(ns, ns > 1 ? rc : 0);
    }
    ra += c;
    rb += ns;
    rc += ns > 1;
  }
  if (threadIdx.x == T - 1) {
    *total = ra;
    *seg_count = rb;
    if (counters) atomicAdd(&counters[0], (unsigned long long)ra);
  }
}

// Ordered compaction of one owner's kept tiles (block per owner, 256 threads): owner-major items
// (token tile, vocab tile).  TOK: owner = token tile n, scanning vocab tiles m (keep[m * nt + n]);
// otherwise owner = vocab tile m, scanning token tiles n (keep[m * nt + n], contiguous).
template <bool TOK>
__global__ void __launch_bounds__(256) fill_items_kernel(const uint8_t* __restrict__ keep, int nt, int mt,
                                                         const int* __restrict__ off, int2* __restrict__ items) {
  griddep_wait();
  __shared__ int s_w[8];
  __shared__ int s_base;
  const int o = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int len = TOK ? mt : nt;
  if (threadIdx.x == 0) s_base = off[o];
  __syncthreads();
  for (int b = 0; b < len; b += 256) {
    const int k = b + threadIdx.x;
    const bool f = k < len && keep[TOK ? (size_t)k * nt + o : (size_t)o * nt + k];
    const uint32_t bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s_w[wid] = __popc(bal);
    __syncthreads();
    int before = 0, tot = 0;
    for (int w = 0; w < 8; ++w) {
      before += w < wid ? s_w[w] : 0;
      tot += s_w[w];
    }
    if (f) items[s_base + before + __popc(bal & ((1u << lane) - 1))] = TOK ? make_int2(o, k) : make_int2(k, o);
    __syncthreads();
    if (threadIdx.x == 0) s_base += tot;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// dE segments of the single vocabulary-major pass: the stream (vocab-tile-major kept list) is cut
// into windows of W items; segment (w, n) = token tile n's items inside window w, in item order.
// Token tile n's segments over the windows form its split chain (accumulator id n).
// ---------------------------------------------------------------------------------------------
// wcnt[w * nt + n] = items of token tile n in window w (block per window; dynamic smem nt ints)
__global__ void window_count_kernel(const int2* __restrict__ items, const int* __restrict__ total, int W, int nt,
                                    int* __restrict__ wcnt) {
  griddep_wait();
  extern __shared__ int s_c[];
  const int w = blockIdx.x;
  const int K = *total;
  for (int n = threadIdx.x; n < nt; n += blockDim.x) s_c[n] = 0;
  __syncthreads();
  const int i1 = min(K, (w + 1) * W);
  for (int i = w * W + threadIdx.x; i < i1; i += blockDim.x) atomicAdd(&s_c[items[i].x], 1);
  __syncthreads();
  for (int n = threadIdx.x; n < nt; n += blockDim.x) wcnt[(size_t)w * nt + n] = s_c[n];
}

// One block: from wcnt over the windows that exist (ceil(total / W) of max_w): wsplit[w * nt + n]
// = index of (w, n) among token tile n's non-empty windows, nsplit[n] = their count, wstart[w * nt +
// n] = first sidx position of segment (w, n) (= w * W + items of smaller token tiles in w), and the
// segment list in (w, n) order: seg = (n, start, items, split), seg_aux = (nsplit[n], n).
__global__ void __launch_bounds__(1024) window_segments_kernel(const int* __restrict__ wcnt, const int* __restrict__ total,
                                                               int W, int nt, int* __restrict__ wsplit,
                                                               int* __restrict__ nsplit, int* __restrict__ wstart,
                                                               int4* __restrict__ seg, int2* __restrict__ seg_aux,
                                                               int* __restrict__ seg_count) {
  griddep_wait();
  constexpr int T = 1024;
  __shared__ int s_a[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (*total + W - 1) / W;
  for (int n = threadIdx.x; n < nt; n += T) {  // per token tile: its non-empty windows
    int k = 0;
    for (int w = 0; w < nw; ++w) {
      wsplit[(size_t)w * nt + n] = k;
      k += wcnt[(size_t)w * nt + n] > 0;
    }
    nsplit[n] = k;
  }
  for (int w = threadIdx.x; w < nw; w += T) {  // per window: segment starts
    int a = w * W;
    for (int n = 0; n < nt; ++n) {
      wstart[(size_t)w * nt + n] = a;
      a += wcnt[(size_t)w * nt + n];
    }
  }
  __syncthreads();
  const long long cells = (long long)nw * nt;
  const long long per = (cells + T - 1) / T;
  const long long c0 = threadIdx.x * per, c1 = min(cells, c0 + per);
  int loc = 0;
  for (long long c = c0; c < c1; ++c) loc += wcnt[c] > 0;
  int inc = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_a[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int x = s_a[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    s_a[lane] = x;
  }
  __syncthreads();
  int k = (wid ? s_a[wid - 1] : 0) + inc - loc;
  for (long long c = c0; c < c1; ++c) {
    const int cnt = wcnt[c];
    if (cnt > 0) {
      const int n = (int)(c % nt);
      seg[k] = make_int4(n, wstart[c], cnt, wsplit[c]);
      seg_aux[k] = make_int2(nsplit[n], n);
      ++k;
    }
  }
  if (threadIdx.x == T - 1) *seg_count = k;
}

// sidx of window w's items grouped by token tile, item order inside a group (block per window, 256
// threads, chunks of 256 items; dynamic smem 9 * nt ints).  Ranks are deterministic: intra-warp by
// lane (match_any), across warps by warp order, across chunks by a running count per token tile.
__global__ void __launch_bounds__(256) window_fill_kernel(const int2* __restrict__ items, const int* __restrict__ total,
                                                          int W, int nt, const int* __restrict__ wstart,
                                                          int* __restrict__ sidx) {
  griddep_wait();
  extern __shared__ int s_m[];
  int* run = s_m;            // [nt] items placed so far per token tile
  int* wc = s_m + nt;        // [8][nt] this chunk's count per warp and token tile
  const int w = blockIdx.x;
  const int K = *total;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int x = threadIdx.x; x < 9 * nt; x += 256) s_m[x] = 0;
  __syncthreads();
  const int i1 = min(K, (w + 1) * W);
  for (int b = w * W; b < i1; b += 256) {
    const int i = b + threadIdx.x;
    const bool ok = i < i1;
    const int n = ok ? items[i].x : -1;
    const uint32_t same = __match_any_sync(0xffffffffu, n);
    const int r = __popc(same & ((1u << lane) - 1));
    if (ok && r == 0) wc[wid * nt + n] = __popc(same);
    __syncthreads();
    if (ok) {
      int base = run[n];
      for (int v = 0; v < wid; ++v) base += wc[v * nt + n];
      sidx[wstart[(size_t)w * nt + n] + base + r] = i;
    }
    __syncthreads();
    for (int x = threadIdx.x; x < nt; x += 256) {
      int t = 0;
      for (int v = 0; v < 8; ++v) {
        t += wc[v * nt + x];
        wc[v * nt + x] = 0;
      }
      run[x] += t;
    }
    __syncthreads();
  }
}

// Single vocabulary-major pass: CTAs [0, P) recompute (CTA pairs), [P, P + Qc) contract dC (CTA
// pairs), the rest contract dE (single CTAs; DE_CH 256-column chunks per unit, KV vocab rows per
// stage) -- every kept tile is recomputed once and read by both.
template <int DE_CH, int KV>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cce_stream3_kernel(const __grid_constant__ CUtensorMap tmE, const __grid_constant__ CUtensorMap tmC,
                       const __grid_constant__ CUtensorMap tmSe, const __grid_constant__ CUtensorMap tmCk,
                       const __grid_constant__ CUtensorMap tmC3, const __grid_constant__ CUtensorMap tmSc,
                       const __grid_constant__ CUtensorMap tmE64, const __grid_constant__ CUtensorMap tmE3,
                       const Params p, const GradParams qe, const GradParams qc, int qc_ctas) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int P = p.st.producers;
  const int b = (int)blockIdx.x;
  if (b < P)
    lse_body<KEPT, 2>(tmE, tmE, tmC, tmC, p, smem, b, P);
  else if (b < P + qc_ctas)
    dc_body<2>(tmSc, tmE64, tmE3, tmE64, qc, smem, b - P, qc_ctas);
  else
    de_body<DE_CH, KV>(tmSe, tmCk, tmC3, tmCk, qe, smem, b - P - qc_ctas, (int)gridDim.x - P - qc_ctas);
}

// The pass kernel: producers (KEPT recompute into the ring) are CTAs [0, producers), consumers the
// rest.  PASS 0 = token pass (single CTAs, dE consumers), 1 = vocab pass (dC consumers; CG = 2: CTA
// pairs for both roles).
template <int PASS, int CG>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cce_stream_kernel(const __grid_constant__ CUtensorMap tmE, const __grid_constant__ CUtensorMap tmEg,
                      const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmCg,
                      const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmX,
                      const __grid_constant__ CUtensorMap tmX3, const __grid_constant__ CUtensorMap tmXg,
                      const Params p, const GradParams q) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int P = p.st.producers;
  const int b = (int)blockIdx.x;
  if (b < P) {
    lse_body<KEPT, CG>(tmE, tmEg, tmC, tmCg, p, smem, b, P);
  } else {
    if constexpr (PASS == 0)
      de_body<1, 64>(tmS, tmX, tmX3, tmXg, q, smem, b - P, (int)gridDim.x - P);
    else
      dc_body<CG>(tmS, tmX, tmX3, tmXg, q, smem, b - P, (int)gridDim.x - P);
  }
}

// ---------------------------------------------------------------------------------------------
// In-place row permutation: rows X[p] (sorted position p) move to row perm[p] (vocabulary order).
// Position t receives X[inv[t]].  Cycles are cut at break points: anchors (a hash of the position
// selects 1 in K) in a cycle of length >= 2, plus any position whose forward walk meets no anchor
// within L steps.  Each break's row is saved to tmp first, then one warp per break walks its segment
// backwards (X[t] = X[inv[t]]) until the predecessor is a break (X[t] = tmp[its index]).  Cycles
// without an anchor (short ones) are rotated by the warp of their smallest position with the row
// held in registers.  More breaks than tmp rows (cap) trap: it needs an adversarial permutation.
// class: 0 fixed point / member of a cut or rotated cycle, 1 break, 2 rotation owner.
// ---------------------------------------------------------------------------------------------
constexpr int PERM_K = 64;      // anchor density 1 / PERM_K
constexpr int PERM_SEG = 96;    // longest segment (a walk of dependent row moves): a break every
                                // PERM_SEG positions between anchors
constexpr int PERM_L = 8192;
__device__ __forceinline__ bool perm_anchor(int p) { return ((uint32_t)p * 2654435761u) >> 26 == 0; }  // 1 in 64

__global__ void unpermute_classify_kernel(const int32_t* __restrict__ perm, int v, uint8_t* __restrict__ cls,
                                          int32_t* __restrict__ bidx, int* __restrict__ nbreak, int cap) {
  griddep_wait();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= v) return;
  uint8_t c = 0;
  if (perm[p] != p) {
    if (perm_anchor(p)) {
      c = 1;
    } else {
      int q = perm[p], mn = p, steps = 1;
      bool found = false;
      while (q != p && steps < PERM_L) {
        if (perm_anchor(q)) {
          found = true;
          break;
        }
        mn = min(mn, q);
        q = perm[q];
        ++steps;
      }
      if (!found)
        c = (q == p) ? (mn == p ? 2 : 0) : 1;  // short cycle: its owner rotates it
      else if (steps % PERM_SEG == 0)
        c = 1;  // bounds the walk between two anchors far apart
    }
  }
  cls[p] = c;
  if (c == 1) {
    const int k = atomicAdd(nbreak, 1);
    if (k >= cap) __trap();
    bidx[p] = k;
  }
}

// Copy one row (d bf16) with a warp: every load of a 2048-column block is issued before any store,
// so a chain of dependent row moves costs one memory round trip per row, not one per 16 bytes.
__device__ __forceinline__ void warp_copy_row(__nv_bfloat16* dst, const __nv_bfloat16* src, int d) {
  const int lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < d; c0 += 2048) {
    uint4 r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int col = c0 + (k * 32 + lane) * 8;
      if (col < d) r[k] = __ldcg(reinterpret_cast<const uint4*>(src + col));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int col = c0 + (k * 32 + lane) * 8;
      if (col < d) *reinterpret_cast<uint4*>(dst + col) = r[k];
    }
  }
}

// warp per break: save its row
__global__ void unpermute_save_kernel(const __nv_bfloat16* __restrict__ X, int v, int d,
                                      const uint8_t* __restrict__ cls, const int32_t* __restrict__ bidx,
                                      __nv_bfloat16* __restrict__ tmp) {
  griddep_wait();
  const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= v || cls[p] != 1) return;
  warp_copy_row(tmp + (size_t)bidx[p] * d, X + (size_t)p * d, d);
}

// warp per break (segment walk) or rotation owner (whole short cycle, row in registers)
constexpr int PERM_REG_VEC = 4;  // uint4 per lane held in registers: rows up to 32*8*4 = 1024 columns per pass
__global__ void unpermute_walk_kernel(__nv_bfloat16* __restrict__ X, int v, int d, const int32_t* __restrict__ inv,
                                      const uint8_t* __restrict__ cls, const int32_t* __restrict__ bidx,
                                      const __nv_bfloat16* __restrict__ tmp) {
  griddep_wait();
  const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= v) return;
  const uint8_t c = cls[p];
  const int lane = threadIdx.x & 31;
  if (c == 1) {
    int t = p;
    int s = inv[t];
    bool brk = cls[s] == 1;
    for (int steps = 0; steps <= v; ++steps) {
      if (brk) {
        warp_copy_row(X + (size_t)t * d, tmp + (size_t)bidx[s] * d, d);
        return;
      }
      // the next hop's index loads are independent of this row's move: issue them first
      const int s2 = inv[s];
      const bool brk2 = cls[s2] == 1;
      warp_copy_row(X + (size_t)t * d, X + (size_t)s * d, d);
      __syncwarp();
      t = s;
      s = s2;
      brk = brk2;
    }
  } else if (c == 2) {
    // rotate the cycle column block by column block: X[t] = X[inv[t]] around the cycle, the
    // owner's own block held in registers
    for (int c0 = 0; c0 < d; c0 += 32 * 8 * PERM_REG_VEC) {
      uint4 keep[PERM_REG_VEC];
#pragma unroll
      for (int k = 0; k < PERM_REG_VEC; ++k) {
        const int col = c0 + (k * 32 + lane) * 8;
        if (col < d) keep[k] = __ldcg(reinterpret_cast<const uint4*>(X + (size_t)p * d + col));
      }
      int t = p;
      while (true) {
        const int s = inv[t];
        if (s == p) {
#pragma unroll
          for (int k = 0; k < PERM_REG_VEC; ++k) {
            const int col = c0 + (k * 32 + lane) * 8;
            if (col < d) *reinterpret_cast<uint4*>(X + (size_t)t * d + col) = keep[k];
          }
          break;
        }
#pragma unroll
        for (int k = 0; k < PERM_REG_VEC; ++k) {
          const int col = c0 + (k * 32 + lane) * 8;
          if (col < d)
            *reinterpret_cast<uint4*>(X + (size_t)t * d + col) =
                __ldcg(reinterpret_cast<const uint4*>(X + (size_t)s * d + col));
        }
        __syncwarp();
        t = s;
      }
    }
  }
}

}  // namespace cce

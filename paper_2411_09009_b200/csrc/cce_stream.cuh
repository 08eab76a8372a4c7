// Streamed backward (cce_bwd_stream): lse_backward (kernels.py:327-486) with transient memory
// bounded independently of the kept-tile count.
//
// The decision from the forward's tile maxima (decide_tiles_kernel) gives the kept tiles.  One
// persistent kernel (cce_stream3_kernel) recomputes each of them once; its CTAs split into roles:
//   producers  the KEPT logit-tile body (cce_lse_kernel.cuh) recomputing kept tiles in stream
//              order (vocabulary-tile-major) and writing S-hat into a ring of R slots in HBM;
//   consumers  the dC body (CTA pairs, units = (vocab tile segment, D chunk)) and the dE body
//              (units = (window segment of a token tile, D chunk)) reading S-hat from the ring
//              with TMA.
// Slot reuse and readiness are counted with GPU-scope release / acquire flags (Stream in
// cce_common.cuh); a segment is a run of at most B items of one owner, an owner with several
// segments sums them in segment order through an fp32 region (deterministic).  Progress is
// guaranteed with every CTA resident (grid = SM count, one CTA per SM): producers take items in
// increasing order, consumers take units in increasing order, and every wait is on an earlier item,
// segment or owner.
//
// The dC role writes dC in the sorted order over the sorted classifier copy the other roles read
// (once every reader of a vocabulary tile is done); unpermute_* put the rows back in vocabulary
// order in place (cycle segments).
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

// ---------------------------------------------------------------------------------------------
// In-place row permutation: rows X[p] (sorted position p) move to row perm[p] (vocabulary order).
// Position t receives X[inv[t]].
//  * A cycle of length <= PERM_SEG without an anchor (a hash of the position selects 1 in PERM_K = 64)
//    is rotated by the warps of its smallest position (rotation list), the first row held in
//    registers.
//  * Every other cycle is cut into segments at break points: its anchors (or, with none, its
//    smallest position) and every position whose distance along perm to the next of those is a
//    multiple of PERM_SEG.  The segment of break b is dest_0 = b, dest_r = inv^r(b) for r < len;
//    the last move's source is the next break, whose row was saved to tmp.
// Kernels:
//   classify  thread per position: walks perm forward to the next anchor (or around the cycle);
//             a break takes a break-list entry k, a rotation owner a rotation entry, a member
//             records its owner break and its distance r (1 <= r < PERM_SEG) to it
//   chains    thread per member: seg[k][r - 1] = p, len[k] = max r -- the segment positions
//             written out, so the row moves of a segment need no pointer chasing
//   save      warp per (break, column block): tmp[k] = X[b]
//   walk      warp per (break, column block): X[dest_r] = X[dest_r+1] (last: tmp of the next
//             break), PERM_DEPTH moves per batch with every load of a batch before its stores
//   rotate    warp per (rotation, column block), grid-stride over the rotation list
// Segments, rotations and column blocks are independent, so every warp runs in parallel.  More
// breaks than tmp rows (cap) trap; the cap covers every permutation (anchors + cuts).
// ---------------------------------------------------------------------------------------------
#ifndef CCE_PERM_K_LOG2
#define CCE_PERM_K_LOG2 6
#endif
constexpr int PERM_K = 1 << CCE_PERM_K_LOG2;  // anchor density 1 / PERM_K
constexpr int PERM_SEG = 96;    // longest segment: positions per break entry of the chain table
constexpr int PERM_L = 8192;    // a walk this long without an anchor makes the position a break
constexpr int PERM_VEC = 1;     // uint4 per lane of a column block: 256 columns per warp
constexpr int PERM_COLS = 32 * 8 * PERM_VEC;
constexpr int PERM_DEPTH = 8;   // row moves whose loads are in flight together
__device__ __forceinline__ bool perm_anchor(int p) { return ((uint32_t)p * 2654435761u) >> (32 - CCE_PERM_K_LOG2) == 0; }

// cls: 0 fixed point or rotation member / owner, 1 break, 2 + (r - 1) member at distance r of its owner (own[p] = owner
// position); breaks: bidx[b] = k, blist[k] = b
__global__ void unpermute_classify_kernel(const int32_t* __restrict__ perm, int v, uint8_t* __restrict__ cls,
                                          int32_t* __restrict__ bidx, int32_t* __restrict__ own,
                                          int32_t* __restrict__ blist, int* __restrict__ nbreak, int cap,
                                          int32_t* __restrict__ rlist, int* __restrict__ nrot) {
  griddep_wait();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= v) return;
  int c = 0, dist = 0;  // c: 0 fixed, 1 break, 2 member at distance `dist` of the next cut point
  int q = perm[p];
  if (q != p) {
    if (perm_anchor(p)) {
      c = 1;
    } else {
      int mn = p, steps = 1, smn = 0;
      bool found = false;
      while (q != p && steps < PERM_L) {
        if (perm_anchor(q)) {
          found = true;
          break;
        }
        if (q < mn) {
          mn = q;
          smn = steps;
        }
        q = perm[q];
        ++steps;
      }
      if (found) {
        dist = steps;        // the next anchor
      } else if (q == p && steps <= PERM_SEG) {
        c = mn == p ? 3 : 4;  // a short anchorless cycle: rotated by its smallest position
      } else {
        dist = q == p ? smn : 0;  // a long anchorless cycle: cut at its smallest position;
      }                           // no anchor within PERM_L: a break
      if (c == 0) c = (dist % PERM_SEG == 0) ? 1 : 2;
    }
  }
  if (c >= 3) {
    cls[p] = 0;  // members of a rotation need no chain entry
    if (c == 3) rlist[atomicAdd(nrot, 1)] = p;
  } else if (c == 2) {
    const int r = (dist - 1) % PERM_SEG + 1;  // the nearest cut point forward
    int o = p;
    for (int i = 0; i < r; ++i) o = perm[o];
    own[p] = o;
    cls[p] = (uint8_t)(1 + r);
  } else {
    cls[p] = (uint8_t)c;
    if (c == 1) {
      const int k = atomicAdd(nbreak, 1);
      if (k >= cap) __trap();
      bidx[p] = k;
      blist[k] = p;
    }
  }
}

// thread per member: its place in the owner's chain (lens zeroed beforehand)
__global__ void unpermute_chains_kernel(int v, const uint8_t* __restrict__ cls, const int32_t* __restrict__ bidx,
                                        const int32_t* __restrict__ own, int32_t* __restrict__ seg,
                                        int* __restrict__ lens) {
  griddep_wait();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= v) return;
  const int c = cls[p];
  if (c < 2) return;
  const int r = c - 1;
  const int k = bidx[own[p]];
  seg[(size_t)k * PERM_SEG + r - 1] = p;
  atomicMax(&lens[k], r);
}

// warp per (break entry, column block): save the break's row block to tmp
__global__ void unpermute_save_kernel(const __nv_bfloat16* __restrict__ X, int d, const int32_t* __restrict__ blist,
                                      const int* __restrict__ nbreak, __nv_bfloat16* __restrict__ tmp) {
  griddep_wait();
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= *nbreak) return;
  const int lane = threadIdx.x & 31;
  const int p = blist[k];
#pragma unroll
  for (int i = 0; i < PERM_VEC; ++i) {
    const int col = blockIdx.y * PERM_COLS + (i * 32 + lane) * 8;
    if (col < d)
      *reinterpret_cast<uint4*>(tmp + (size_t)k * d + col) = __ldcg(reinterpret_cast<const uint4*>(X + (size_t)p * d + col));
  }
}

// 16-byte global load ordered against the walker's stores (the compiler may not move either)
__device__ __forceinline__ uint4 ld_cg_ordered(const void* ptr) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(ptr)
               : "memory");
  return r;
}

// warp per (break entry, column block): the moves of the break's segment
__global__ void __launch_bounds__(256) unpermute_walk_kernel(__nv_bfloat16* X, int d, const int32_t* __restrict__ inv,
                                                             const int32_t* __restrict__ bidx,
                                                             const int32_t* __restrict__ blist,
                                                             const int32_t* __restrict__ seg,
                                                             const int* __restrict__ lens,
                                                             const int* __restrict__ nbreak,
                                                             const __nv_bfloat16* __restrict__ tmp) {
  griddep_wait();
  const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= *nbreak) return;
  const int lane = threadIdx.x & 31;
  const int len = lens[k] + 1;  // moves: dest_0 = the break, dest_1 .. dest_{len-1} its members
  // dest_r of r = lane + 32 j (PERM_SEG <= 96: three per lane)
  int dst[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const int r = lane + 32 * j;
    dst[j] = r == 0 ? blist[k] : (r < len ? seg[(size_t)k * PERM_SEG + r - 1] : 0);
  }
  const int last = __shfl_sync(0xffffffffu, dst[(len - 1) >> 5], (len - 1) & 31);
  const int tail = bidx[inv[last]];  // the last move's source: the next break's saved row
  const int col = blockIdx.y * PERM_COLS + lane * 8;
  const bool on = col < d;
  for (int r0 = 0; r0 < len; r0 += PERM_DEPTH) {
    uint4 val[PERM_DEPTH][PERM_VEC];
#pragma unroll
    for (int j = 0; j < PERM_DEPTH; ++j) {
      const int r = r0 + j;
      const int s = r + 1;  // source of move r: dest_{r+1}
      const int sp = __shfl_sync(0xffffffffu, s < 96 ? dst[s >> 5] : 0, s & 31);
      if (r < len && on) {
        const __nv_bfloat16* row = s < len ? X + (size_t)sp * d : tmp + (size_t)tail * d;
#pragma unroll
        for (int i = 0; i < PERM_VEC; ++i)
          if (col + i * 256 < d) val[j][i] = ld_cg_ordered(row + col + i * 256);
      }
    }
#pragma unroll
    for (int j = 0; j < PERM_DEPTH; ++j) {
      const int r = r0 + j;
      const int dp = __shfl_sync(0xffffffffu, dst[(r >> 5) < 3 ? (r >> 5) : 2], r & 31);
      if (r < len && on) {
#pragma unroll
        for (int i = 0; i < PERM_VEC; ++i)
          if (col + i * 256 < d) *reinterpret_cast<uint4*>(X + (size_t)dp * d + col + i * 256) = val[j][i];
      }
    }
  }
}

// warp per (rotation, column block), grid-stride over the rotation list: X[t] = X[inv[t]] around
// a short cycle, the owner's own row block kept in registers
__global__ void __launch_bounds__(256) unpermute_rotate_kernel(__nv_bfloat16* X, int d, const int32_t* __restrict__ inv,
                                                               const int32_t* __restrict__ rlist,
                                                               const int* __restrict__ nrot) {
  griddep_wait();
  const int lane = threadIdx.x & 31;
  const int col = blockIdx.y * PERM_COLS + lane * 8;
  const bool on = col < d;
  const int total = *nrot;
  for (int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); k < total; k += gridDim.x * (blockDim.x >> 5)) {
    const int p = rlist[k];
    uint4 keep = on ? ld_cg_ordered(X + (size_t)p * d + col) : make_uint4(0, 0, 0, 0);
    int t = p;
    for (int s = inv[t]; s != p; s = inv[s]) {
      if (on) *reinterpret_cast<uint4*>(X + (size_t)t * d + col) = ld_cg_ordered(X + (size_t)s * d + col);
      t = s;
    }
    if (on) *reinterpret_cast<uint4*>(X + (size_t)t * d + col) = keep;
  }
}

}  // namespace cce

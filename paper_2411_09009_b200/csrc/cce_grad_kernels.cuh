// Gradient passes over the S-hat tiles stored by the filter pass (cce_lse_kernel<BWD>).
//
// lse_backward (kernels.py:461-479) accumulates dE += S-hat C and dC += S-hat^T E per kept tile
// under locks.  Doing that per tile on a GPU means ~2.4 MB of atomics per kept 128x256 tile
// (128 flop per reduced byte - far beyond any atomic bandwidth), so the two products are
// instead computed output-stationary, each in its own pass, with no atomics at all:
//
//   B2 cce_de_kernel : unit = (token tile n, 256 D-columns).  TMEM accumulates
//                      dE[n, dchunk] = sum over kept m of S-hat[n,m] (128x256, K-major A) x
//                      C[m, dchunk] (256x256, MN-major B), four 4-deep pipeline stages of 64
//                      vocab rows per tile.
//   B3 cce_dc_kernel : unit = (vocab tile m, 256 D-columns, 128-row vocab half).  TMEM
//                      accumulates dC[m half, dchunk] = sum over kept n of S-hat^T (MN-major A)
//                      x E[n, dchunk] (MN-major B), two K-steps of 64 tokens per tile.
//
// Both: persistent, 192 threads (warp 0 TMA producer scanning the kept-tile map with the whole
// warp, warp 1 MMA issuer, warps 2..5 epilogue writing bf16 / fp32 rows straight to HBM).
#pragma once
#include "cce_common.cuh"

namespace cce {

#ifndef CCE_DE_HINT
#define CCE_DE_HINT 1  // measured: 1.60 vs 1.65 ms (none) vs 2.09 ms (2) at Gemma-2B
#endif
constexpr int DE_KV = 64;                       // default vocab rows (MMA K) per dE stage
constexpr int DE_SMEM_BUDGET = 200 * 1024;
// CH = 256-column D chunks per unit: CH = 1 double-buffers two 256-column accumulators in TMEM,
// CH = 2 fills TMEM with one 512-column accumulator (each S-hat stage feeds both chunks).
// KV = vocab rows per stage: 64 (S-hat atom of 128 B rows, 128 B swizzle) or 32 (64 B rows,
// 64 B swizzle): half the bytes per stage, twice the stages in flight.
template <int CH, int KV>
struct DeCfg {
  static constexpr int A_BYTES = BM * KV * 2;      // S-hat [128 tok][KV voc]
  static constexpr int CHUNK_BYTES = KV * DCH * 2;  // C [KV voc][256 d] as 4 atoms
  static constexpr int STAGE_BYTES = A_BYTES + CH * CHUNK_BYTES;
  static constexpr int STAGES = DE_SMEM_BUDGET / STAGE_BYTES;
  static constexpr int ACC = CH == 1 ? 2 : 1;  // accumulator buffers
  static constexpr int SMEM = STAGES * STAGE_BYTES;
  static constexpr uint64_t A_LAYOUT = KV == 32 ? kSwizzle64B : kSwizzle128B;
  static constexpr uint32_t A_SBO = 8 * KV * 2;
};
constexpr int DE_QUEUE = 4;                     // scheduled units in flight
constexpr int DC_STAGES = 4;
constexpr int DC_A_BYTES = 64 * 128 * 2;        // S-hat [64 tok][128 voc]  = 16 KiB (2 atoms)
constexpr int DC_B_BYTES = 64 * DCH * 2;        // E [64 tok][256 d]        = 32 KiB (4 atoms)
constexpr int DC_STAGE_BYTES = DC_A_BYTES + DC_B_BYTES;
constexpr int DC_STG_PITCH = 144;                 // bytes per staged row (128 B + 16 B pad)
constexpr int DC_STG_BYTES = 4 * 32 * DC_STG_PITCH;  // epilogue row-transpose staging, 4 warps
constexpr int DC_IDX_BYTES = BM * 4;                 // E row-gather index table (pairs)

// Visit, in index order, the stored tiles slot_of[i * stride] >= 0 for i < count; the warp reads
// 32 entries per step and every lane calls f(i, slot) for each stored tile.
template <typename F>
__device__ __forceinline__ void for_each_kept(const int32_t* slot_of, int count, int stride, F&& f) {
  const int lane = threadIdx.x & 31;
  for (int base = 0; base < count; base += 32) {
    const int i = base + lane;
    const int sl = i < count ? slot_of[(size_t)i * stride] : -1;
    uint32_t mask = __ballot_sync(0xffffffffu, sl >= 0);
    while (mask) {
      const int b = __ffs(mask) - 1;
      mask &= mask - 1;
      f(base + b, __shfl_sync(0xffffffffu, sl, b));
    }
  }
}

// Visit the kept tiles of one vocab tile through the vocab-tile-major kept list: entries
// [off, off + cnt) = (token tile, slot) in token-tile order; lanes fetch 32 entries at a time,
// every lane calls f(local token tile, slot).
template <typename F>
__device__ __forceinline__ void for_each_listed(const int2* list, int off, int cnt, int n_base, F&& f) {
  const int lane = threadIdx.x & 31;
  for (int base = 0; base < cnt; base += 32) {
    const int2 my = base + lane < cnt ? list[off + base + lane] : make_int2(0, 0);
    const int k_end = min(32, cnt - base);
    for (int k = 0; k < k_end; ++k)
      f(__shfl_sync(0xffffffffu, my.x, k) - n_base, __shfl_sync(0xffffffffu, my.y, k));
  }
}

// dC unit -> (vocab tile m, D chunk dc, vocab half vh).  blk = 0: vocabulary-tile-major (the
// 2 * ndc units of one vocab tile side by side: its S-hat tiles are shared through L2, E rows are
// re-read per vocab tile -- free while E fits L2).  blk > 0: blocks of blk vocab tiles, D-chunk-
// major inside a block, so concurrent CTAs share the block's S-hat tiles and one E chunk (large N:
// E no longer fits L2).
__device__ __forceinline__ void dc_unit(int u, int mt, int ndc, int blk, int& m, int& dc, int& vh) {
  vh = u & 1;
  const int w = u >> 1;
  if (blk <= 0) {
    dc = w % ndc;
    m = w / ndc;
    return;
  }
  const int b = w / (blk * ndc);
  const int r = w - b * blk * ndc;
  const int bb = min(blk, mt - b * blk);  // vocab tiles of this block (the last may be short)
  dc = r / bb;
  m = b * blk + r % bb;
}

__device__ __forceinline__ void store_row32(float* dst_f32, __nv_bfloat16* dst_bf16, const float* x,
                                            int lim) {
  // 32 consecutive values; lim = number of valid columns (multiple of 8)
  if (dst_f32) {
#pragma unroll
    for (int j = 0; j < 32; j += 4)
      if (j < lim) *reinterpret_cast<float4*>(dst_f32 + j) = make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]);
  } else {
#pragma unroll
    for (int j = 0; j < 32; j += 8)
      if (j < lim)
        *reinterpret_cast<uint4*>(dst_bf16 + j) =
            make_uint4(pack_bf16x2(x[j], x[j + 1]), pack_bf16x2(x[j + 2], x[j + 3]),
                       pack_bf16x2(x[j + 4], x[j + 5]), pack_bf16x2(x[j + 6], x[j + 7]));
  }
}

// ------------------------------------------------------------------------------------------
// B2: dE
// ------------------------------------------------------------------------------------------
// Unit = (token tile n, pair j of 256-column D chunks): both chunks accumulate in TMEM (512
// columns, single-buffered) from the same S-hat stage, so S-hat is streamed once per chunk pair.
// Units are ordered pair-major (the CTAs running at once share C[:, pair]) and handed out by an
// atomic counter (p.sched): units differ in length (kept tiles per token tile, a lone last chunk).
template <int CH, int KV>
__device__ __forceinline__ void de_body(const CUtensorMap& tmS, const CUtensorMap& tmC, const CUtensorMap& tmC3,
                                        const CUtensorMap& tmCg, const GradParams& p, uint8_t* smem, int bid,
                                        int nblk) {
  using Cfg = DeCfg<CH, KV>;
  constexpr int DE_STAGES = Cfg::STAGES;
  constexpr int DE_STAGE_BYTES = Cfg::STAGE_BYTES;
  constexpr int DE_A_BYTES = Cfg::A_BYTES;
  constexpr int DE_CHUNK_BYTES = Cfg::CHUNK_BYTES;
  constexpr int DE_CH = CH;
  constexpr int DE_KV = KV;
  constexpr int ACC = Cfg::ACC;
  if (skip_launch(p.run_if)) return;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + DE_STAGES * DE_STAGE_BYTES);
  uint64_t* empty = full + DE_STAGES;
  uint64_t* acc_full = empty + DE_STAGES;  // [ACC]
  uint64_t* acc_free = acc_full + ACC;     // [ACC]
  uint64_t* unit_full = acc_free + ACC;    // [DE_QUEUE] producer -> MMA / epilogue
  uint64_t* unit_empty = unit_full + DE_QUEUE;
  int* s_unit = reinterpret_cast<int*>(unit_empty + DE_QUEUE);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_unit + DE_QUEUE);
  // streamed: per stage, the ring slot whose last bytes it carries (-1: none), set by the loader
  // before the stage's arrival; the MMA thread counts the slot consumed once the stage has landed
  int* s_sig = reinterpret_cast<int*>(smem + DE_STAGES * DE_STAGE_BYTES + 256);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmS);
    tma_prefetch_desc(&tmC3);
    for (int i = 0; i < DE_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < ACC; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_free[i], 128);
    }
    for (int i = 0; i < DE_QUEUE; ++i) {
      mbar_init(&unit_full[i], 1);
      mbar_init(&unit_empty[i], 1 + 4);  // MMA thread + one lane per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const Rows rows(p.n_valid, p.n_total, p.n_base, p.g);
  const int G = rows.g;
  const int npair = (p.ndc + DE_CH - 1) / DE_CH;
  // streamed: units are (segment, chunk group), segment-major; otherwise (token tile, chunk group)
  const bool stream = p.st.ring > 0;
  const int units = (stream ? *p.seg_count : G) * npair;
  constexpr int SPI = BN / DE_KV;  // stages per S-hat tile
  const bool plain = p.atoms3d && p.perm == nullptr;
  // unit u -> (chunk group j, token tile ln): chunk-major (concurrent CTAs share C[:, j]) or
  // token-tile-major (concurrent CTAs share S-hat[n])
  auto decode = [&](int u, int& j, int& ln) {
    if (stream) {  // ln = segment index
      ln = u / npair;
      j = u - ln * npair;
    } else if (p.de_order == 0) {
      j = u / G;
      ln = u % G;
    } else if (p.de_order >= 2) {
      // groups of K = de_order chunk pairs, token-tile-major inside a group: the K CTAs of one
      // token tile run side by side (static round-robin, grid a multiple of K) and read each
      // S-hat tile at the same time, so it comes from HBM once per group instead of once per chunk
      const int K = p.de_order;
      const int g = u / (G * K);
      const int kg = min(K, npair - g * K);
      const int r = u - g * G * K;
      ln = r / kg;
      j = g * K + r % kg;
    } else {
      ln = u / npair;
      j = u % npair;
    }
  };

  // unit queue: the producer claims units and publishes them; -1 ends the stream
  auto next_unit = [&](int k, uint32_t ph) {
    mbar_wait(&unit_full[k], ph);
    return *reinterpret_cast<volatile int*>(&s_unit[k]);
  };

  if (warp == 0) {
    int stage = 0;
    uint32_t phase = 0;
    for (int q = 0;; ++q) {
      const int k = q % DE_QUEUE;
      const uint32_t ph = (q / DE_QUEUE) & 1;
      int u = 0;
      if (lane == 0) {
        mbar_wait(&unit_empty[k], ph ^ 1);
        u = p.sched ? atomicAdd(p.sched, 1) : bid + q * nblk;
        if (u >= units) u = -1;
        s_unit[k] = u;
        mbar_arrive(&unit_full[k]);
      }
      u = __shfl_sync(0xffffffffu, u, 0);
      if (u < 0) break;
      int j, ln;
      decode(u, j, ln);
      const int nch = min(DE_CH, p.ndc - DE_CH * j);
      const uint32_t bytes = DE_A_BYTES + nch * DE_CHUNK_BYTES;
      const int32_t* srow = stream ? nullptr : p.slot_of + (size_t)ln * p.mt;
      // L2 prefetch of the C slices of kept tiles [m + prefetch, ...): lane l covers vocab tile
      // pf_next + l, issued one batch of 32 ahead of use
      int pf_next = 0;
      auto prefetch_upto = [&](int m_hi) {
        if (!p.prefetch || !plain) return;
        m_hi = min(m_hi, p.mt);
        while (pf_next < m_hi) {  // warp-uniform
          const int mm = pf_next + lane;
          if (mm < m_hi && srow[mm] >= 0)
            for (int c = 0; c < nch; ++c)
#pragma unroll
              for (int h = 0; h < BN / DE_KV; ++h)
                tma_prefetch_3d(&tmC3, 0, mm * BN + DE_KV * h, (DE_CH * j + c) * (DCH / 64));
          pf_next = min(pf_next + 32, m_hi);
        }
      };
      auto load_tile = [&](int m, int slot, int sig) {
        for (int h = 0; h < BN / DE_KV; ++h) {
          RowGather rgc;
          rgc.load(p.perm, m * BN + DE_KV * h, DE_KV);
          uint8_t* sa = smem + stage * DE_STAGE_BYTES;
          uint8_t* sb = sa + DE_A_BYTES;
          if (lane == 0) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (stream) s_sig[stage] = h == BN / DE_KV - 1 ? sig : -1;
            // debug (timing only, wrong results): bit 0 skips the S-hat loads, bit 1 the C loads
            mbar_arrive_expect_tx(&full[stage], bytes - ((p.debug & 1) ? DE_A_BYTES : 0) -
                                                    ((p.debug & 2) ? nch * DE_CHUNK_BYTES : 0));
            // S-hat [128 tok][KV voc]: swizzle atom h of the stored tile
#if CCE_DE_HINT > 0
            if (p.debug & 3) {
              if (!(p.debug & 1)) tma_load_3d(&tmS, &full[stage], sa, 0, slot * BM, h);
              if (plain && !(p.debug & 2))
                for (int c = 0; c < nch; ++c)
                  tma_load_3d(&tmC3, &full[stage], sb + c * DE_CHUNK_BYTES, 0, m * BN + DE_KV * h,
                              (DE_CH * j + c) * (DCH / 64));
            } else {
            // L2 priorities: 1 (default) = keep C slices (shared by the token tiles of a chunk,
            // which reach a vocab tile tens of us apart), stream S-hat; 2 = the reverse (slower)
            const uint64_t pol_s = CCE_DE_HINT == 1 ? l2_policy_evict_first() : l2_policy_evict_last();
            const uint64_t pol_c = CCE_DE_HINT == 1 ? l2_policy_evict_last() : l2_policy_evict_first();
            tma_load_3d_hint(&tmS, &full[stage], sa, 0, slot * BM, h, pol_s);
            if (plain)
              for (int c = 0; c < nch; ++c)
                tma_load_3d_hint(&tmC3, &full[stage], sb + c * DE_CHUNK_BYTES, 0, m * BN + DE_KV * h,
                                 (DE_CH * j + c) * (DCH / 64), pol_c);
            }
#else
            tma_load_3d(&tmS, &full[stage], sa, 0, slot * BM, h);
            if (plain)  // C [64 voc][256 d] per chunk as 4 atoms
              for (int c = 0; c < nch; ++c)
                tma_load_3d(&tmC3, &full[stage], sb + c * DE_CHUNK_BYTES, 0, m * BN + DE_KV * h,
                            (DE_CH * j + c) * (DCH / 64));
#endif
          }
          __syncwarp();
          if (!plain) {
#pragma unroll 1
            for (int c = 0; c < nch; ++c)
#pragma unroll 1
              for (int a = 0; a < DCH / 64; ++a)
                load_rows_warp<DE_KV>(&tmC, &tmCg, rgc, p.perm != nullptr, &full[stage],
                                      sb + c * DE_CHUNK_BYTES + a * (DE_KV * 128),
                                      (DE_CH * j + c) * DCH + 64 * a, m * BN + DE_KV * h);
          }
          advance_stage(stage, phase, DE_STAGES);
        }
      };
      if (stream) {
        // the segment's items in stream order; each waits until its producer published it
        const int4 sg = p.seg[ln];
#ifdef CCE_STREAM_PROF
        if (lane == 0 && p.prof) {
          p.prof[(size_t)u * 8 + 0] = global_timer_ns();
          p.prof[(size_t)u * 8 + 6] = bid;
          p.prof[(size_t)u * 8 + 7] = ((unsigned long long)sg.x << 32) | (unsigned)sg.y;
        }
#endif
#ifdef CCE_STREAM_TRACE
        if (lane == 0 && bid < 4) printf("de cta %d unit %d seg %d (n %d start %d cnt %d split %d) chunk %d\n", bid, u, ln, sg.x, sg.y, sg.z, sg.w, j);
#endif
        for (int k = sg.y; k < sg.y + sg.z; ++k) {
          const int i = p.sidx ? p.sidx[k] : k;
          const int slot = i % p.st.ring;
          if (lane == 0) {
            spin_until_geq(&p.st.ready[slot], i / p.st.ring + 1);
            fence_proxy_async_global();
          }
          __syncwarp();
          load_tile(p.items[i].y, slot, slot);
        }
#ifdef CCE_STREAM_PROF
        if (lane == 0 && p.prof) p.prof[(size_t)u * 8 + 1] = global_timer_ns();
#endif
      } else {
        prefetch_upto(p.prefetch);
        for_each_kept(srow, p.mt, 1, [&](int m, int slot) {
          prefetch_upto(m + p.prefetch);
          load_tile(m, slot, -1);
        });
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t IDESC = make_idesc_bf16(BM, DCH, 0, 1);  // A K-major, B MN-major
      int stage = 0;
      uint32_t phase = 0;
      for (int q = 0;; ++q) {
        const int k = q % DE_QUEUE;
        const int u = next_unit(k, (q / DE_QUEUE) & 1);
        mbar_arrive(&unit_empty[k]);
        if (u < 0) break;
        int j, ln;
        decode(u, j, ln);
        const int nch = min(DE_CH, p.ndc - DE_CH * j);
        const int4 sg = stream ? p.seg[ln] : make_int4(0, 0, 0, 0);
        const int ksteps = SPI * (stream ? sg.z : p.cnt_n[ln]);
        const int buf = q % ACC;
        mbar_wait(&acc_free[buf], ((q / ACC) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * (DE_CH * DCH);
        for (int s = 0; s < ksteps; ++s) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(smem + stage * DE_STAGE_BYTES);
          const uint32_t b0 = a0 + DE_A_BYTES;
#pragma unroll
          for (int ks = 0; ks < DE_KV / 16; ++ks)  // A: K-major atom; B: 4 MN-major atoms, 16 K-rows each
            for (int c = 0; c < nch; ++c)
              mma_bf16_ss(d_tmem + c * DCH, make_sdesc(a0 + ks * 32, 0, Cfg::A_SBO, Cfg::A_LAYOUT),
                          make_sdesc(b0 + c * DE_CHUNK_BYTES + ks * 2048, DE_KV * 128, 1024), IDESC,
                          (s | ks) != 0);
          // streamed: the item's last S-hat stage has landed in smem -- its ring slot may be reused
          if (stream) {
            const int sig = s_sig[stage];
            if (sig >= 0) red_relaxed_add_gpu(&p.st.used[sig], 1);
          }
          mma_commit(&empty[stage]);
          advance_stage(stage, phase, DE_STAGES);
        }
        mma_commit(&acc_full[buf]);
      }
    }
  } else {
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int epi_tid = threadIdx.x - 64;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    for (int q = 0;; ++q) {
      const int k = q % DE_QUEUE;
      const int u = next_unit(k, (q / DE_QUEUE) & 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(&unit_empty[k]);
      if (u < 0) break;
      int j, ln;
      decode(u, j, ln);
      const int nch = min(DE_CH, p.ndc - DE_CH * j);
      const int buf = q % ACC;
#ifdef CCE_STREAM_PROF
      const int u_prof = u;
      if (epi_tid == 0 && p.prof && stream) p.prof[(size_t)u * 8 + 2] = global_timer_ns();
#endif
      mbar_wait(&acc_full[buf], (q / ACC) & 1);
      tc_fence_after();
#ifdef CCE_STREAM_PROF
      if (epi_tid == 0 && p.prof && stream) p.prof[(size_t)u * 8 + 3] = global_timer_ns();
#endif
      // streamed: the segment's owner (token tile) and its place in the owner's split chain
      int nsplit = 1, split = 0, chain_key = 0, gen_key = 0;
      const float* racc = nullptr;
      float* wacc = nullptr;
      bool has;
      if (stream) {
        const int4 sg = p.seg[ln];
        const int2 sx = p.seg_aux[ln];
        ln = sg.x;
        has = sg.z > 0;
        nsplit = sx.x;
        split = sg.w;
        if (nsplit > 1) {
          // region (acc slot, chunk group j) of DE_CH * 256 columns, laid out [column quads][128
          // rows] of float4: a warp's 32 rows read 512 contiguous bytes
          gen_key = (sx.y % p.nacc) * npair + j;
          chain_key = ln * npair + j;
          float* region = p.acc + (size_t)gen_key * BM * (DE_CH * DCH) + row * 4;
          racc = split > 0 ? region : nullptr;
          wacc = split < nsplit - 1 ? region : nullptr;
          if (epi_tid == 0) {
            if (split == 0)
              spin_until_geq(&p.acc_gen[gen_key], sx.y / p.nacc);  // previous owner done with the region
            else
              spin_until_geq(&p.chain[chain_key], split);          // segments before this one folded in
          }
          named_bar_sync(1, 128);
        }
#ifdef CCE_STREAM_PROF
        if (epi_tid == 0 && p.prof) p.prof[(size_t)u_prof * 8 + 4] = global_timer_ns();
#endif
      } else {
        has = p.cnt_n[ln] > 0;
      }
      const int grow = (p.n_base + ln) * BM + row;
      const bool valid = grow < rows.n && (has || !p.de_accumulate);  // accumulate: nothing to add
      const int drow = valid ? p.row_map[grow] : 0;
      if (racc || wacc) {
        // split owner (streamed): fold in the earlier segments and pass the sum on, 64 columns per
        // step with every load of the step in flight at once (the region sits in L2)
#pragma unroll 1
        for (int c = 0; c < nch * (DCH / 64); ++c) {
          const int col = DE_CH * j * DCH + c * 64;
          float x[64];
          {
            uint32_t r[64];
            tmem_ld32(tmem_base + lane_off + buf * (DE_CH * DCH) + c * 64, *reinterpret_cast<uint32_t(*)[32]>(r));
            tmem_ld32(tmem_base + lane_off + buf * (DE_CH * DCH) + c * 64 + 32,
                      *reinterpret_cast<uint32_t(*)[32]>(r + 32));
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 64; ++i) x[i] = __uint_as_float(r[i]);
          }
#ifndef CCE_DE_RED
#define CCE_DE_RED 1
#endif
          // a middle segment adds its partial with vector reductions in L2 (no read: the chain
          // still orders the segments, so the fp32 sum keeps its order); the first stores it, the
          // last folds the running sum in and writes dE
          const bool mid = CCE_DE_RED && racc && wacc;
          if (racc && !mid && !(p.debug & 4)) {  // debug bit 2: skip the fold-in loads (timing only)
            float4 o[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = __ldcg(reinterpret_cast<const float4*>(racc) + (c * 16 + i) * BM);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              x[4 * i] += o[i].x;
              x[4 * i + 1] += o[i].y;
              x[4 * i + 2] += o[i].z;
              x[4 * i + 3] += o[i].w;
            }
          }
          if (p.debug & 8) {  // debug bit 3: no stores (timing only)
          } else if (mid) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              red_add_v4_f32(reinterpret_cast<float*>(reinterpret_cast<float4*>(wacc) + (c * 16 + i) * BM), x[4 * i], x[4 * i + 1],
                             x[4 * i + 2], x[4 * i + 3]);
          } else if (wacc) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              __stcg(reinterpret_cast<float4*>(wacc) + (c * 16 + i) * BM,
                     make_float4(x[4 * i], x[4 * i + 1], x[4 * i + 2], x[4 * i + 3]));
          } else if (valid) {
            const size_t off = (size_t)drow * p.d + col;
            store_row32(p.de_f32 ? p.de_f32 + off : nullptr, p.de_bf16 ? p.de_bf16 + off : nullptr, x, p.d - col);
            if (col + 32 < p.d)
              store_row32(p.de_f32 ? p.de_f32 + off + 32 : nullptr, p.de_bf16 ? p.de_bf16 + off + 32 : nullptr, x + 32,
                          p.d - col - 32);
          }
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < nch * (DCH / 32); ++c) {
          const int col = DE_CH * j * DCH + c * 32;
          float x[32];
          if (has) {
            uint32_t r[32];
            tmem_ld32(tmem_base + lane_off + buf * (DE_CH * DCH) + c * 32, r);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = __uint_as_float(r[i]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = 0.f;
          }
          if (valid && col < p.d) {
            const size_t off = (size_t)drow * p.d + col;
            if (p.de_accumulate) {  // fp32 read-modify-write, fixed group order (deterministic)
              const float* old = p.de_f32 + off;
#pragma unroll
              for (int i = 0; i < 32; i += 4)
                if (i < p.d - col) {
                  const float4 o = *reinterpret_cast<const float4*>(old + i);
                  x[i] += o.x;
                  x[i + 1] += o.y;
                  x[i + 2] += o.z;
                  x[i + 3] += o.w;
                }
            }
            store_row32(p.de_f32 ? p.de_f32 + off : nullptr, p.de_bf16 ? p.de_bf16 + off : nullptr, x,
                        p.d - col);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&acc_free[buf]);
#ifdef CCE_STREAM_PROF
      if (epi_tid == 0 && p.prof && stream) p.prof[(size_t)u_prof * 8 + 5] = global_timer_ns();
#endif
      if (nsplit > 1) {  // hand the running sum / the region on
        named_bar_sync(1, 128);
        if (epi_tid == 0) {
          __threadfence();
          if (split < nsplit - 1)
            st_release_gpu(&p.chain[chain_key], split + 1);
          else
            red_release_add_gpu(&p.acc_gen[gen_key], 1);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

template <int CH, int KV>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cce_de_kernel(const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmC,
                  const __grid_constant__ CUtensorMap tmC3, const __grid_constant__ CUtensorMap tmCg,
                  const GradParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  de_body<CH, KV>(tmS, tmC, tmC3, tmCg, p, smem, (int)blockIdx.x, (int)gridDim.x);
}

// ------------------------------------------------------------------------------------------
// B3: dC
// ------------------------------------------------------------------------------------------
// CG = 2: the two vocabulary halves of one (vocab tile, 256 D-columns) unit run as a CTA pair
// with one M = 256 tcgen05.mma per K-step issued by the leader: each CTA loads its own S-hat^T
// half (A) and half of the shared E[64 tok][256 d] operand (B, 128 d-columns), so per-SM operand
// traffic per flop drops by a third; each CTA's TMEM holds its 128 vocab rows.
template <int CG>
__device__ __forceinline__ void dc_body(const CUtensorMap& tmS, const CUtensorMap& tmE, const CUtensorMap& tmE3,
                                        const CUtensorMap& tmEg, const GradParams& p, uint8_t* smem, int bid,
                                        int nblk) {
  constexpr int B_BYTES = DC_B_BYTES / CG;  // this CTA's part of E[64 tok][256 d]
  constexpr int SBYTES = DC_A_BYTES + B_BYTES;
  // same smem footprint for both forms: pairs (32 KB stages) get 6 stages instead of 4
  constexpr int STAGES = (DC_STAGES * DC_STAGE_BYTES) / SBYTES;
  constexpr int DC_STAGES = STAGES;
  constexpr int DC_STAGE_BYTES = SBYTES;
  if (skip_launch(p.run_if)) return;
  uint8_t* stg = smem + cce::DC_STAGES * cce::DC_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + DC_STG_BYTES);
  uint64_t* empty = full + DC_STAGES;
  uint64_t* acc_full = empty + DC_STAGES;
  uint64_t* acc_free = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_free + 2);
  int32_t* s_eidx = reinterpret_cast<int32_t*>(stg + DC_STG_BYTES + 256);  // [BM] (after the barriers)
  int* s_sig = reinterpret_cast<int*>(stg + DC_STG_BYTES + 256 + DC_IDX_BYTES);  // [stages], see de_body
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int rank = CG == 2 ? (int)cluster_ctarank() : 0;
  const Rows rows(p.n_valid, p.n_total, p.n_base, p.g);
  // pairs reading E through a compaction that is not the identity: cp.async row gathers, relayed
  // to the leader's full barrier once landed (as in the logit-tile kernel)
  const bool gather_pair = CG == 2 && p.e_gather != 0 && !rows.ident;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmS);
    tma_prefetch_desc(&tmE);
    for (int i = 0; i < DC_STAGES; ++i) {
      mbar_init(&full[i], CG * (gather_pair ? 2 : 1));  // pairs: both producers arrive on the leader's barrier
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_free[i], CG == 2 ? 2 : 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if (CG == 2)
      tmem_alloc_pair(tmem_slot, TMEM_COLS);
    else
      tmem_alloc(tmem_slot, TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int G = rows.g;
  // unit u = ((m * ndc) + dc) * 2 + vh: the two vocab halves of one (m, dchunk) run side by side
  // (CG = 1: adjacent units sharing their E / S-hat loads through L2; CG = 2: one CTA pair)
  // streamed: units are (segment, D chunk, vocab half), segment-major; the segment's owner is
  // the vocab tile
  const bool stream = p.st.ring > 0;
  const int units = (stream ? *p.seg_count : p.mt) * p.ndc * 2;
  const int start = CG == 2 ? (bid & ~1) + rank : bid;
  const int stride = nblk;
  // unit -> (vocab tile or segment m, chunk, half)
  auto decode = [&](int u, int& m, int& dc, int& vh) {
    if (stream) {
      vh = u & 1;
      const int w = u >> 1;
      m = w / p.ndc;
      dc = w - m * p.ndc;
    } else {
      dc_unit(u, p.mt, p.ndc, p.dc_block, m, dc, vh);
    }
  };

  if (warp == 0) {
    int stage = 0;
    uint32_t phase = 0;
    constexpr int GLAG = 2;  // gathered stages in flight before their relay
    int issued = 0, rstage = 0;
    auto relay = [&](int st) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (rank != 0)
          mbar_arrive_cluster(&full[st], 0);
        else
          mbar_arrive(&full[st]);
      }
      rstage = (st + 1 == DC_STAGES) ? 0 : st + 1;
    };
    for (int u = start; u < units; u += stride) {
      int vh, dc, m;
      decode(u, m, dc, vh);
      auto tile = [&](int ln, int slot, int sig = -1) {
        const int n = p.n_base + ln;
        if (gather_pair) {
          __syncwarp();  // every lane is done reading the previous item's table
          load_index_table(s_eidx, p.row_map, n * BM, BM, rows.n);
          __syncwarp();
        }
        for (int h = 0; h < 2; ++h) {
          RowGather rge;
          rge.load(p.e_gather ? p.row_map : nullptr, n * BM + 64 * h, 64);
          uint8_t* sa = smem + stage * DC_STAGE_BYTES;
          uint8_t* sb = sa + DC_A_BYTES;
          const bool e3 = p.atoms3d && !p.e_gather;
          if (lane == 0) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (stream && rank == 0) s_sig[stage] = h == 1 ? sig : -1;
            if (CG == 2) {
              if (rank == 0)
                mbar_arrive_expect_tx(&full[stage], 2 * (gather_pair ? (uint32_t)DC_A_BYTES : (uint32_t)SBYTES));
              else
                mbar_arrive_cluster(&full[stage], 0);
              const uint32_t lb = leader_addr(&full[stage]);
              // S-hat^T half vh: tokens [64h, +64) x vocab atoms 2vh, 2vh+1; E: this CTA's 2 atoms
              tma_load_3d_pair(&tmS, lb, sa, 0, slot * BM + 64 * h, 2 * vh);
              if (!gather_pair) tma_load_3d_pair(&tmE3, lb, sb, 0, n * BM + 64 * h, dc * (DCH / 64) + 2 * rank);
            } else {
              mbar_arrive_expect_tx(&full[stage], ((p.debug & 1) ? 0 : DC_A_BYTES) + ((p.debug & 2) ? 0 : DC_B_BYTES));
              // S-hat^T half: tokens [64h, +64) x vocab atoms 2vh, 2vh+1 in one box
              if (!(p.debug & 1)) tma_load_3d(&tmS, &full[stage], sa, 0, slot * BM + 64 * h, 2 * vh);
              if (e3 && !(p.debug & 2))  // E [64 tok][256 d] as 4 atoms in one box
                tma_load_3d(&tmE3, &full[stage], sb, 0, n * BM + 64 * h, dc * (DCH / 64));
            }
          }
          __syncwarp();
          if (gather_pair) {  // this CTA's two 64-column atoms of E[64 tok] through row_map
#pragma unroll 1
            for (int a = 0; a < 2; ++a)
              gather_box_async<64>(sb + a * (64 * 128), p.e_rows, p.d, s_eidx + 64 * h,
                                   dc * DCH + 128 * rank + 64 * a);
            cp_async_commit();
            if (++issued > GLAG) {
              cp_async_wait<GLAG>();
              relay(rstage);
            }
          }
          if (CG == 1 && !e3) {
#pragma unroll 1
            for (int a = 0; a < DCH / 64; ++a)
              load_rows_warp<64>(&tmE, &tmEg, rge, p.e_gather != 0, &full[stage], sb + a * (64 * 128),
                                 dc * DCH + 64 * a, n * BM + 64 * h);
          }
          advance_stage(stage, phase, DC_STAGES);
        }
      };
      if (stream) {
        const int4 sg = p.seg[m];
        for (int i = sg.y; i < sg.y + sg.z; ++i) {
          const int slot = i % p.st.ring;
          if (lane == 0) {
            spin_until_geq(&p.st.ready[slot], i / p.st.ring + 1);
            fence_proxy_async_global();
          }
          __syncwarp();
          tile(p.items[i].x - p.n_base, slot, slot);
        }
      } else if (p.off_m != nullptr) {  // contiguous slots of this vocab tile from the kept list
        for_each_listed(p.list, p.off_m[m], p.cnt_m[m], p.n_base, tile);
      } else {
        for_each_kept(p.slot_of + m, G, p.mt, tile);
      }
    }
    if (gather_pair) {  // drain: relay the stages still in flight
      cp_async_wait<0>();
      for (int k = 0; k < min(issued, GLAG); ++k) relay(rstage);
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // pairs: the leader issues for both CTAs
      constexpr uint32_t IDESC = make_idesc_bf16(BM * CG, DCH, 1, 1);  // A, B both MN-major
      int stage = 0;
      uint32_t phase = 0;
      int t = 0;
      // the next unit's kept count is loaded one unit ahead (units are short: ~8 us at Gemma-2B)
      auto unit_cnt = [&](int uu) {
        int mm, dd, hh;
        decode(uu, mm, dd, hh);
        return stream ? p.seg[mm].z : p.cnt_m[mm];
      };
      int cnt = start < units ? unit_cnt(start) : 0;
      for (int u = start; u < units; u += stride) {
        const int un = u + stride;
        const int cnt_next = un < units ? unit_cnt(un) : 0;
        const int ksteps = 2 * cnt;
        cnt = cnt_next;
        // a vocab tile no token tile keeps: no accumulator hand-off (the epilogue skips it too;
        // `t` counts only the units that use a buffer)
        if (ksteps == 0) continue;
        const int buf = t & 1;
        mbar_wait(&acc_free[buf], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * DCH;
        for (int s = 0; s < ksteps; ++s) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(smem + stage * DC_STAGE_BYTES);
          const uint32_t b0 = a0 + DC_A_BYTES;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t ad = make_sdesc(a0 + ks * 2048, 64 * 128, 1024);
            const uint64_t bd = make_sdesc(b0 + ks * 2048, 64 * 128, 1024);
            if (CG == 2)
              mma_bf16_ss_pair(d_tmem, ad, bd, IDESC, (s | ks) != 0);
            else
              mma_bf16_ss(d_tmem, ad, bd, IDESC, (s | ks) != 0);
          }
          // streamed: both 64-token halves of the item's S-hat (both CTAs' halves, pairs) have
          // landed -- the ring slot may be reused (one count per unit: both CTAs load per stage)
          if (stream) {
            const int sig = s_sig[stage];
            if (sig >= 0) red_relaxed_add_gpu(&p.st.used[sig], 1);
          }
          if (CG == 2)
            mma_commit_pair(&empty[stage]);
          else
            mma_commit(&empty[stage]);
          advance_stage(stage, phase, DC_STAGES);
        }
        if (CG == 2)
          mma_commit_pair(&acc_full[buf]);
        else
          mma_commit(&acc_full[buf]);
        ++t;
      }
    }
  } else {
    // Each thread owns one vocabulary row of the accumulator (its TMEM lane).  Rows are written
    // through a per-warp shared-memory transpose so every global store instruction covers four
    // full 128-byte row segments instead of 32 scattered 16-byte pieces.
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int epi_tid = threadIdx.x - 64;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    uint8_t* wstg = stg + quarter * 32 * DC_STG_PITCH;
    int t = 0;
    for (int u = start; u < units; u += stride) {
      int vh, dc, m;
      decode(u, m, dc, vh);
      // streamed: the segment's owner (vocab tile) and its place in the owner's split chain
      int nsplit = 1, split = 0, chain_key = 0, gen_key = 0;
      const float* racc = nullptr;
      float* wacc = nullptr;
      bool has;
      if (stream) {
        const int4 sg = p.seg[m];
        const int2 sx = p.seg_aux[m];
        m = sg.x;
        has = sg.z > 0;
        nsplit = sx.x;
        split = sg.w;
        if (nsplit > 1) {
          gen_key = ((sx.y % p.nacc) * p.ndc + dc) * 2 + vh;
          chain_key = (m * p.ndc + dc) * 2 + vh;
          float* region = p.acc + (size_t)gen_key * BM * DCH + row * 4;  // column-quad-major (see dE)
          racc = split > 0 ? region : nullptr;
          wacc = split < nsplit - 1 ? region : nullptr;
          if (epi_tid == 0) {
            if (split == 0)
              spin_until_geq(&p.acc_gen[gen_key], sx.y / p.nacc);
            else
              spin_until_geq(&p.chain[chain_key], split);
          }
          named_bar_sync(1, 128);
        }
      } else {
        has = p.cnt_m[m] > 0;
      }
      if (!has && p.accumulate) continue;  // nothing kept and nothing to write
      if (stream && p.own_off && !wacc) {
        // the final write lands on C rows of this tile in the sorted copy: wait until every item of
        // the tile has been read by every consumer (counts only grow, so later laps satisfy it too)
        if (epi_tid == 0) {
          const int i0 = p.own_off[m], i1 = i0 + p.own_cnt[m];
          for (int i = i0; i < i1; ++i)
            spin_until_geq(&p.st.used[i % p.st.ring], (i / p.st.ring + 1) * p.st.consumers);
        }
        named_bar_sync(1, 128);
      }
      const int buf = t & 1;
      // per-unit loads issued before the wait so their latency hides behind it
      const int vpos = m * BN + vh * 128 + row;
      const int my_vrow = vpos < p.v ? (p.perm_store ? p.perm_store[vpos] : vpos) : -1;
      if (has) {  // empty units use no accumulator: their zero rows are written right away
        mbar_wait(&acc_full[buf], (t >> 1) & 1);
        tc_fence_after();
      }
      {
#pragma unroll 1
        for (int c = 0; c < DCH / 64; ++c) {
          // 1) this thread's 64 columns -> bf16 -> staging row `lane`
          uint32_t pk[32];
          if (has && nsplit > 1) {
            // split owner: fold in the earlier segments, pass the sum on (or write it: last one)
            uint32_t r0[32], r1[32];
            tmem_ld32(tmem_base + lane_off + buf * DCH + c * 64, r0);
            tmem_ld32(tmem_base + lane_off + buf * DCH + c * 64 + 32, r1);
            tmem_ld_wait();
            float x[64];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              x[j] = __uint_as_float(r0[j]);
              x[32 + j] = __uint_as_float(r1[j]);
            }
            // as in dE: a middle segment adds its partial with L2 vector reductions (no read; the
            // chain orders the segments), the first stores, the last folds in and writes dC
            const bool mid = CCE_DE_RED && racc && wacc;
            if (racc && !mid) {
#pragma unroll
              for (int j = 0; j < 64; j += 4) {
                const float4 o = __ldcg(reinterpret_cast<const float4*>(racc) + (c * 16 + j / 4) * BM);
                x[j] += o.x;
                x[j + 1] += o.y;
                x[j + 2] += o.z;
                x[j + 3] += o.w;
              }
            }
            if (wacc) {
#pragma unroll
              for (int j = 0; j < 64; j += 4) {
                float4* dst = reinterpret_cast<float4*>(wacc) + (c * 16 + j / 4) * BM;
                if (mid)
                  red_add_v4_f32(reinterpret_cast<float*>(dst), x[j], x[j + 1], x[j + 2], x[j + 3]);
                else
                  __stcg(dst, make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]));
              }
              continue;  // warp-uniform: every thread of the unit takes this branch
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) pk[j] = pack_bf16x2(x[2 * j], x[2 * j + 1]);
          } else if (has) {
            uint32_t r0[32], r1[32];
            tmem_ld32(tmem_base + lane_off + buf * DCH + c * 64, r0);
            tmem_ld32(tmem_base + lane_off + buf * DCH + c * 64 + 32, r1);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              pk[j] = pack_bf16x2(__uint_as_float(r0[2 * j]), __uint_as_float(r0[2 * j + 1]));
              pk[16 + j] = pack_bf16x2(__uint_as_float(r1[2 * j]), __uint_as_float(r1[2 * j + 1]));
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) pk[j] = 0u;
          }
          uint4* srow = reinterpret_cast<uint4*>(wstg + lane * DC_STG_PITCH);
#pragma unroll
          for (int q = 0; q < 8; ++q) srow[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          __syncwarp();
          // 2) warp-cooperative stores: lanes 8k..8k+7 write row (4*it + k), 16 B each
          const int col = dc * DCH + c * 64 + (lane & 7) * 8;
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int rr = it * 4 + (lane >> 3);
            const int vrow = __shfl_sync(0xffffffffu, my_vrow, rr);
            uint4 val = *reinterpret_cast<const uint4*>(wstg + rr * DC_STG_PITCH + (lane & 7) * 16);
            if (vrow >= 0 && col < p.d) {
              __nv_bfloat16* dst = p.dc + (size_t)vrow * p.d + col;
              if (p.accumulate) {
                const uint4 old = *reinterpret_cast<const uint4*>(dst);
                const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&val);
                const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&old);
                uint32_t w[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const float2 fa = __bfloat1622float2(a2[q]);
                  const float2 fo = __bfloat1622float2(o2[q]);
                  w[q] = pack_bf16x2(fa.x + fo.x, fa.y + fo.y);
                }
                val = make_uint4(w[0], w[1], w[2], w[3]);
              }
              *reinterpret_cast<uint4*>(dst) = val;
            }
          }
          __syncwarp();
        }
      }
      if (!has) continue;
      tc_fence_before();
      if (CG == 2) {
        named_bar_sync(2, 128);
        if (epi_tid == 0) {
          if (rank == 0)
            mbar_arrive(&acc_free[buf]);
          else
            mbar_arrive_cluster(&acc_free[buf], 0);
        }
      } else {
        mbar_arrive(&acc_free[buf]);
      }
      ++t;
      if (nsplit > 1) {  // hand the running sum / the region on
        if (CG != 2) named_bar_sync(2, 128);  // (pairs: the barrier above already joined the epilogue)
        if (epi_tid == 0) {
          __threadfence();
          if (split < nsplit - 1)
            st_release_gpu(&p.chain[chain_key], split + 1);
          else
            red_release_add_gpu(&p.acc_gen[gen_key], 1);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    if (CG == 2)
      tmem_dealloc_pair(tmem_base, TMEM_COLS);
    else
      tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

template <int CG>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cce_dc_kernel(const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmE,
                  const __grid_constant__ CUtensorMap tmE3, const __grid_constant__ CUtensorMap tmEg,
                  const GradParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  dc_body<CG>(tmS, tmE, tmE3, tmEg, p, smem, (int)blockIdx.x, (int)gridDim.x);
}

}  // namespace cce

// Fused logit-tile kernel: forward LSE (FWD), backward filter pass (BWD) and backward recompute
// of already-selected tiles (KEPT).
//
//   FWD  = indexed_matmul (kernels.py:204-251) + lse_forward (kernels.py:254-319): per token row,
//          an online (max, sum-exp) over this CTA's vocabulary split plus the target logit.
//          Optionally records each row's max raw logit per 128x256 tile (`tile_max`) so the
//          backward can take the filter decision without recomputing skipped tiles.
//   BWD  = recompute / S / filter half of lse_backward (kernels.py:425-459) over every tile:
//          keep a tile iff it holds a label or any S = exp(z - lse) >= eps (block_skip_decision,
//          kernels.py:140-142); kept tiles store S-hat = up * (S - onehot) [* (1 - tanh^2)] as
//          bf16 for the dE / dC passes (cce_grad_kernels.cuh).
//   KEPT = S-hat of the tiles in a precomputed kept list (the decision having been taken from the
//          forward's tile maxima, cce_aux_kernels.cuh: decide_tiles_kernel).
//
// CG = 2 runs the same kernel on CTA pairs (cta_group::2): the pair computes a 256-token x
// 256-vocab tile with one M=256 tcgen05.mma issued by the leader; each CTA loads its own 128 E
// rows and half of the 256 C rows (so per-SM operand traffic per flop drops by a third) and owns
// its 128 token rows in its own TMEM, so the epilogues are unchanged.  Filter decisions stay per
// 128x256 tile (per CTA), as in the 1-CTA kernel.
//
// Persistent, one CTA per SM, 192 threads:
//   warp 0      TMA producer (whole warp; gathers split over lanes): E rows [n*128, +128) and C
//               rows of tile m, 64 D-columns per stage, 4-stage ring
//   warp 1      TMEM allocator + MMA issuer: K-blocks x 4 tcgen05.mma (M=128, N=256, K=16)
//               into one of two 256-column fp32 accumulators (double buffered)
//   warps 2..5  epilogue: thread (warp%4)*32+lane owns one token row of the tile and reads its
//               256 accumulator columns with tcgen05.ld
#pragma once
#include "cce_common.cuh"

namespace cce {

struct TileRef {
  int n, m;     // token tile, vocab tile (tile order)
  int s;        // vocabulary split of the unit (FWD / BWD) or slot (KEPT)
  bool first;   // first tile of its unit
  bool last;    // last tile of its unit
  bool ok;      // this CTA's token tile exists (pairs: the second tile of an odd count does not)
  bool zero;    // BWD, pairs: this CTA's token tile has zero upstream but the peer's does not
};

// Visit this CTA's tiles in schedule order.  FWD / BWD: static persistent schedule over units
// (token tile n, vocab split s), each a contiguous range of vocab tiles of one token tile (CG = 2:
// of one token-tile pair, CTA rank r taking tile 2*pair + r).  Units are rastered in bands of
// `band` token tiles (token tile fastest inside a band, then split, then band), so the CTAs
// running at any moment touch at most `band` E tiles (kept L2-resident by the host's choice of
// band) and a handful of C tiles, each shared by many CTAs.
// KEPT: grid-stride over the kept list (vocab-tile-major, so concurrent CTAs share C tiles).
// `skip(n, count)` is called for BWD units whose upstream is all zero (kernels.py:434-438).
template <int MODE, int CG, typename F, typename S>
__device__ __forceinline__ void for_each_tile(const Params& p, const Rows& rows, int rank, int bid, int nblk,
                                              F&& f, S&& skip) {
  if (MODE == KEPT) {
    if (CG == 2) {
      // pair entry = up to two kept tiles of one vocab tile (consecutive slots); a lone tile's
      // partner CTA recomputes the same rows and discards them
      const int total = *p.pair_count;
      for (int i = bid >> 1; i < total; i += nblk >> 1) {
        const int2 pe = p.pairs[i];
        const bool ok = rank < pe.y;
        const int slot = pe.x + (ok ? rank : 0);
        const int2 t = p.list[slot];
        f(TileRef{t.x, t.y, slot, true, true, ok, false});
      }
      return;
    }
    const int total = p.st.ring ? *p.list_count : min(*p.list_count, p.capacity);
    for (int i = bid; i < total; i += nblk) {
      const int2 t = p.list[i];
      f(TileRef{t.x, t.y, i, true, true, true, false});
    }
    return;
  }
  const int gp = (rows.g + CG - 1) / CG;  // token tiles (CG = 2: token-tile pairs) of this launch
  const int units = gp * p.splits;
  const int band = max(1, min((p.band + CG - 1) / CG, gp));
  const int start = CG == 2 ? bid >> 1 : bid;
  const int stride = CG == 2 ? nblk >> 1 : nblk;
  for (int u = start; u < units; u += stride) {
    const int b = u / (band * p.splits);
    const int r = u - b * band * p.splits;
    const int nb = min(band, gp - b * band);
    const int local = (b * band + r % nb) * CG + rank;  // this CTA's token tile within the launch
    const int n = p.n_base + local;
    const int s = r / nb;
    const int m0 = (int)(((long long)s * p.mt) / p.splits);
    const int m1 = (int)(((long long)(s + 1) * p.mt) / p.splits);
    const bool ok = local < rows.g;
    bool zero = false;
    if (MODE == BWD) {
      zero = !ok || p.block_zero[n];
      bool skip_unit = zero;
      if (CG == 2) {
        const int peer_local = local ^ 1;
        const bool peer_zero = peer_local >= rows.g || p.block_zero[p.n_base + peer_local];
        skip_unit = zero && peer_zero;  // the pair skips together or computes together
      }
      if (skip_unit) {
        if (ok) skip(n, m1 - m0);
        continue;
      }
    }
    for (int m = m0; m < m1; ++m) f(TileRef{n, m, s, m == m0, m == m1 - 1, ok, zero});
  }
}

// The kernel body, on CTA `bid` of `nblk` (the whole grid, or the producer role of the streamed
// backward's kernel, cce_stream.cuh); `smem` is the 1024-aligned dynamic shared memory.
template <int MODE, int CG>
__device__ __forceinline__ void lse_body(const CUtensorMap& tmE, const CUtensorMap& tmEg, const CUtensorMap& tmC,
                                         const CUtensorMap& tmCg, const Params& p, uint8_t* smem, int bid,
                                         int nblk) {
  constexpr int STAGES = CG == 2 ? LSE_STAGES_PAIR : LSE_STAGES;
  constexpr int SBYTES = CG == 2 ? PAIR_STAGE_BYTES : STAGE_BYTES;  // per-CTA bytes per stage
  if (p.no_dep_wait)
    griddep_trigger();  // the flags below order every input of this launch
  else if (skip_launch(p.run_if))
    return;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * SBYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;  // [2] MMA -> epilogue: logits ready
  uint64_t* acc_free = acc_full + 2;    // [2] epilogue -> MMA: accumulator reusable
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_free + 2);
  uint32_t* s_vote = tmem_slot + 1;     // [2][4]
  int* s_slot = reinterpret_cast<int*>(s_vote + 8);  // [2]
  int32_t* s_eidx = reinterpret_cast<int32_t*>(smem + STAGES * SBYTES + LSE_CTRL_BYTES);  // [BM]
  int32_t* s_cidx = s_eidx + BM;                                                          // [BN / CG]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int rank = CG == 2 ? (int)cluster_ctarank() : 0;
  const Rows rows(p.n_valid, p.n_total, p.n_base, p.nt);
  // Row gathers (cp.async): C rows through the vocabulary order (no sorted copy of C) and E rows
  // through the compaction map unless it is the identity.  Each producer then arrives twice per
  // stage: once for the TMA bytes, once (relayed) when its gathered bytes have landed.
  const bool gather_c = p.perm != nullptr;
  const bool gather_e = p.e_gather != 0 && !rows.ident;
  const bool gmode = gather_c || gather_e;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmE);
    tma_prefetch_desc(&tmC);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], CG * (gmode ? 2 : 1));  // pairs: both producers arrive on the leader's barrier
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_free[i], CG == 2 ? 2 : 128);  // pairs: one arrival per CTA epilogue
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
  auto no_skip = [](int, int) {};

  if (warp == 0) {
    // ============================ producer (whole warp: TMA + gathers) =====================
    if (p.sync_ready) {  // this launch's group lands in its buffer (the previous launch's gathers)
      if (lane == 0) spin_until_geq(p.sync_ready, 1);
      __syncwarp();
      fence_proxy_async_global();  // generic-proxy row copies, read here by TMA
    }
    constexpr int CROWS = BN / CG;    // C rows this CTA loads per tile
#ifndef CCE_GLAG
#define CCE_GLAG 2
#endif
    constexpr int GLAG = CCE_GLAG < STAGES ? CCE_GLAG : STAGES - 1;  // gathered stages in flight before their relay
    int stage = 0;
    uint32_t phase = 0;
    int cur_n = -1, cur_m = -1;
    int issued = 0, rstage = 0;       // gathered stages issued; stage of the next relay
    // this CTA's gathered bytes of stage s have landed: make them visible to the async proxy
    // (the tensor core) and arrive on the stage's full barrier (pairs: the leader's)
    auto relay = [&](int s) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2 && rank != 0)
          mbar_arrive_cluster(&full[s], 0);
        else
          mbar_arrive(&full[s]);
      }
      rstage = (s + 1 == STAGES) ? 0 : s + 1;
    };
    const uint32_t tx_cta = (gather_e ? 0u : (uint32_t)A_BYTES) + (gather_c ? 0u : (uint32_t)CROWS * BK * 2);
    for_each_tile<MODE, CG>(p, rows, rank, bid, nblk, [&](const TileRef& t) {
      if (gmode) __syncwarp();  // every lane is done reading the tables for the previous tile
      if (gather_e && t.n != cur_n) {
        load_index_table(s_eidx, p.row_map, t.n * BM, BM, rows.n);
        cur_n = t.n;
      }
      if (gather_c && t.m != cur_m) {
        load_index_table(s_cidx, p.perm, t.m * BN + rank * CROWS, CROWS);
        cur_m = t.m;
      }
      __syncwarp();
      for (int kb = 0; kb < p.num_kb; ++kb) {
        uint8_t* sa = smem + stage * SBYTES;
        if (lane == 0) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (CG == 2) {
            // both CTAs' TMA bytes complete on the leader's barrier; the follower only arrives
            if (rank == 0)
              mbar_arrive_expect_tx(&full[stage], 2 * tx_cta);
            else
              mbar_arrive_cluster(&full[stage], 0);
            const uint32_t lb = leader_addr(&full[stage]);
            if (!gather_e) tma_load_2d_pair(&tmE, lb, sa, kb * BK, t.n * BM);
            if (!gather_c) tma_load_2d_pair(&tmC, lb, sa + A_BYTES, kb * BK, t.m * BN + rank * CROWS);
          } else {
            mbar_arrive_expect_tx(&full[stage], tx_cta);
            if (!gather_e) tma_load_2d(&tmE, &full[stage], sa, kb * BK, t.n * BM);
            if (!gather_c) tma_load_2d(&tmC, &full[stage], sa + A_BYTES, kb * BK, t.m * BN);
          }
        }
        __syncwarp();
        if (gmode) {
          if (gather_e) gather_box_async<BM>(sa, p.e_rows, p.d, s_eidx, kb * BK);
          if (gather_c) gather_box_async<CROWS>(sa + A_BYTES, p.c_rows, p.d, s_cidx, kb * BK);
          cp_async_commit();
          if (++issued > GLAG) {
            cp_async_wait<GLAG>();
            relay(rstage);
          }
        }
        advance_stage(stage, phase, STAGES);
      }
    }, no_skip);
    if (gmode) {  // drain: relay the stages still in flight
      cp_async_wait<0>();
      for (int k = 0; k < min(issued, GLAG); ++k) relay(rstage);
    }
  } else if (warp == 1) {
    // ===================================== MMA issuer ====================================
    if (lane == 0 && rank == 0) {  // pairs: the leader issues for both CTAs
      constexpr uint32_t IDESC = make_idesc_bf16(BM * CG, BN, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int t = 0;
      for_each_tile<MODE, CG>(p, rows, rank, bid, nblk, [&](const TileRef&) {
        const int buf = t & 1;
        mbar_wait(&acc_free[buf], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * BN;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(smem + stage * SBYTES);
          const uint32_t b0 = a0 + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            if (CG == 2)
              mma_bf16_ss_pair(d_tmem, make_sdesc(a0 + 32 * k, 0, 1024),
                               make_sdesc(b0 + 32 * k, 0, 1024), IDESC, (kb | k) != 0);
            else
              mma_bf16_ss(d_tmem, make_sdesc(a0 + 32 * k, 0, 1024), make_sdesc(b0 + 32 * k, 0, 1024),
                          IDESC, (kb | k) != 0);
          }
          if (CG == 2)
            mma_commit_pair(&empty[stage]);
          else
            mma_commit(&empty[stage]);
          advance_stage(stage, phase, STAGES);
        }
        if (CG == 2)
          mma_commit_pair(&acc_full[buf]);
        else
          mma_commit(&acc_full[buf]);
        ++t;
      }, no_skip);
    }
  } else if (warp == NUM_THREADS / 32) {
    // ============== gather warp (224-thread launches): the next group's rows ==============
    if (p.g_dst) {
      if (p.g_wait) {  // the buffer is free once the launch before this one has exited
        if (lane == 0) spin_until_geq(p.g_wait, 1);
        __syncwarp();
        (void)ld_acquire_gpu(p.g_wait);  // every lane: its reads are ordered after the chain's inputs
      }
      // this CTA's share of the rows, two rows at a time: 16-byte copies, up to 16 loads in flight
      // per lane (32-bit index arithmetic; the share is a few hundred KB per launch)
      const int r0 = (int)((int64_t)p.g_rows * bid / nblk), r1 = (int)((int64_t)p.g_rows * (bid + 1) / nblk);
      const int n16 = p.d / 8;
      for (int r = r0; r < r1; r += 2) {
        const bool two = r + 1 < r1;
        const uint4* s0 = reinterpret_cast<const uint4*>(p.g_src + (size_t)p.g_perm[r] * p.d);
        const uint4* s1 = reinterpret_cast<const uint4*>(p.g_src + (size_t)p.g_perm[two ? r + 1 : r] * p.d);
        uint4* d0 = reinterpret_cast<uint4*>(p.g_dst + (size_t)r * p.d);
        uint4* d1 = d0 + n16;
        for (int j0 = 0; j0 < n16; j0 += 32 * 8) {
          uint4 a[8], b[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int j = j0 + lane + 32 * u;
            if (j < n16) {
              a[u] = __ldg(s0 + j);
              b[u] = __ldg(s1 + j);
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int j = j0 + lane + 32 * u;
            if (j < n16) {
              d0[j] = a[u];
              if (two) d1[j] = b[u];
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        if (atomicAdd(p.g_ctr, 1) == nblk - 1) {
          __threadfence();
          st_release_gpu(p.g_done, 1);
        }
      }
    }
  } else {
    // ===================================== epilogue ======================================
    if (p.sync_ready) {  // every lane: its reads (targets, positions) ordered after the chain's inputs
      if (lane == 0) spin_until_geq(p.sync_ready, 1);
      __syncwarp();
      (void)ld_acquire_gpu(p.sync_ready);
    }
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const bool use_softcap = p.softcap > 0.f;
    const float inv_cap = use_softcap ? 1.0f / p.softcap : 0.f;
    const int epi_tid = threadIdx.x - 64;  // 0..127
    int t = 0;
    // per-row state, refreshed whenever the token tile changes
    int cur_n = -1;
    bool cur_ok = false;
    bool valid = false;
    int grow = 0;
    int orow = 0;                  // original row of E (row_map; identity without compaction)
    int64_t tpos = -1;             // FWD: target position in C's row order
    float lse2 = 0.f, up_r = 0.f;  // BWD / KEPT
    int pos_r = -1;
    float run_m = -INFINITY, run_s = 0.f, corr = 0.f;
    bool have_corr = false;

    auto load_row = [&](int n, bool ok) {
      grow = n * BM + row;
      valid = ok && grow < rows.n;
      orow = valid ? (p.row_map ? p.row_map[grow] : grow) : 0;
      if (MODE == FWD) {
        tpos = -1;
        if (valid) {
          if (p.pos) {
            tpos = p.pos[orow] - p.pos_offset;  // vocabulary group: group-local position
          } else {
            const int64_t tg = p.targets[orow];
            if (tg != p.ignore_index) tpos = tg - p.vocab_start;
          }
        }
      } else {
        lse2 = valid ? p.lse[orow] * LOG2E : INFINITY;
        up_r = valid ? p.upstream[orow] : 0.f;
        pos_r = valid ? p.pos[orow] - p.pos_offset : -1;  // outside the group: never matches
      }
    };

    // this thread's S-hat row of the tile in accumulator `tacc` -> bf16 -> slot, row-major
    // [slot][128][256]
    auto store_shat = [&](uint32_t tacc, int col0, int slot) {
      uint4* dst = reinterpret_cast<uint4*>(p.shat + ((size_t)slot * BM + row) * BN);
      // 64 columns per step: each thread writes a full 128 B line of its row at once
#pragma unroll 1
      for (int c = 0; c < BN / 64; ++c) {
        uint32_t r[64];
        tmem_ld32(tacc + c * 64, *reinterpret_cast<uint32_t(*)[32]>(r));
        tmem_ld32(tacc + c * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
        tmem_ld_wait();
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 64; j += 2) {
          float g2[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float z = __uint_as_float(r[j + h]);
            float dcap = 1.f;
            if (use_softcap) {
              const float th = softcap_tanh(z, inv_cap);
              z = p.softcap * th;
              dcap = 1.f - th * th;
            }
            const int col = col0 + c * 64 + j + h;
            const float s = (col < p.v) ? ex2_approx(z * LOG2E - lse2) : 0.f;
            g2[h] = ((col == pos_r && !p.label_split) ? s - 1.f : s) * up_r * dcap;
          }
          pk[j >> 1] = pack_bf16x2(g2[0], g2[1]);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          dst[c * 8 + q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
      }
    };

    // hand the accumulator back to the MMA issuer (pairs: one arrival per CTA on the leader)
    auto release_acc = [&](int buf) {
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
    };

    for_each_tile<MODE, CG>(p, rows, rank, bid, nblk, [&](const TileRef& tr) {
      if (tr.n != cur_n || tr.ok != cur_ok) {  // KEPT pairs: a lone tile's partner visits it with ok = false
        load_row(tr.n, tr.ok);
        cur_n = tr.n;
        cur_ok = tr.ok;
      }
      const int buf = t & 1;
      mbar_wait(&acc_full[buf], (t >> 1) & 1);
      tc_fence_after();
      const int col0 = tr.m * BN;
      const uint32_t tacc = tmem_base + lane_off + buf * BN;
      if (MODE == FWD) {
        if (tr.first) {
          run_m = -INFINITY;
          run_s = 0.f;
          have_corr = false;
        }
        const bool tile_has_t = tpos >= col0 && tpos < col0 + BN;
        // label tile of this CTA's token tile?  (decided before the sweep: labels are known)
        bool is_lab = false;
        if (p.lab_buf != nullptr) {
          const uint32_t wv = __ballot_sync(0xffffffffu, tile_has_t);
          if (lane == 0) s_vote[(t & 1) * 4 + quarter] = wv;
          named_bar_sync(1, 128);
          const uint32_t* vv = s_vote + (t & 1) * 4;
          is_lab = tr.ok && (vv[0] | vv[1] | vv[2] | vv[3]) != 0;
        }
        float zmax = -INFINITY;
#ifndef CCE_FWD_LDW
#define CCE_FWD_LDW 32
#endif
#ifndef CCE_FWD_FAST
#define CCE_FWD_FAST 1  // unmasked path for interior chunks (0: A/B against the masked loop)
#endif
        constexpr int LW = CCE_FWD_LDW;  // TMEM columns per load-wait step (32 or 64)
#pragma unroll 1
        for (int c = 0; c < BN / LW; ++c) {
          uint32_t r[LW];
#pragma unroll
          for (int q = 0; q < LW / 32; ++q)
            tmem_ld32(tacc + c * LW + q * 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32 * q));
          tmem_ld_wait();
          float y[LW];
          float cm = -INFINITY;
          const int cbase = col0 + c * LW;
          // common chunk (inside V, no softcap, not this row's label): no per-column masks, and
          // max(z * log2e) = round(max(z) * log2e) exactly (rounding is monotone) -- bit-identical
          if (CCE_FWD_FAST && !use_softcap && cbase + LW <= p.v &&
              !(tile_has_t && tpos >= cbase && tpos < cbase + LW)) {
            float czm = -INFINITY;
#pragma unroll
            for (int j = 0; j < LW; ++j) {
              y[j] = __uint_as_float(r[j]);
              czm = fmaxf(czm, y[j]);
            }
            zmax = fmaxf(zmax, czm);
            cm = czm * LOG2E;
#pragma unroll
            for (int j = 0; j < LW; ++j) y[j] *= LOG2E;
          } else {
#pragma unroll
            for (int j = 0; j < LW; ++j) {
              float z = __uint_as_float(r[j]);
              const int col = col0 + c * LW + j;
              const bool in_v = col < p.v;
              if (in_v) zmax = fmaxf(zmax, z);
              if (use_softcap) z = p.softcap * softcap_tanh(z, inv_cap);
              if (tile_has_t && col == tpos) {
                corr = z;
                have_corr = true;
              }
              y[j] = in_v ? z * LOG2E : -INFINITY;
              cm = fmaxf(cm, y[j]);
            }
          }
          const float nm = fmaxf(run_m, cm);
          if (nm != -INFINITY) {
            float acc = 0.f;
#pragma unroll
            for (int j = 0; j < LW; ++j) acc += ex2_approx(y[j] - nm);
            run_s = run_s * ex2_approx(run_m - nm) + acc;
            run_m = nm;
          }
        }
        if (is_lab) {
          // claim a slot, then re-read the accumulator: fp16 of z' - z'max(row), <= 0 and exact
          // near the row max where S lives (padded columns -inf)
          if (epi_tid == 0) {
            int slot = atomicAdd(p.lab_count, 1);
            if (slot < p.lab_capacity) {
              p.lab_slot[(size_t)tr.n * p.mt + tr.m] = slot;
              p.lab_list[slot] = make_int2(tr.n, tr.m);
            } else {
              slot = -1;
            }
            s_slot[t & 1] = slot;
          }
          named_bar_sync(1, 128);
          const int slot = s_slot[t & 1];
          if (slot >= 0) {
            const float zcmax = use_softcap ? p.softcap * softcap_tanh(zmax, inv_cap) : zmax;
            uint4* dst = reinterpret_cast<uint4*>(p.lab_buf + ((size_t)slot * BM + row) * BN);
            // 64 columns per step: each thread writes a full 128 B line of its row at once
#pragma unroll 1
            for (int c = 0; c < BN / 64; ++c) {
              uint32_t r[64];
              tmem_ld32(tacc + c * 64, *reinterpret_cast<uint32_t(*)[32]>(r));
              tmem_ld32(tacc + c * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
              tmem_ld_wait();
              uint32_t pk[32];
              if (CCE_FWD_FAST && !use_softcap && col0 + c * 64 + 64 <= p.v) {
#pragma unroll
                for (int j = 0; j < 64; j += 2) {
                  const __half2 h2 = __floats2half2_rn(__uint_as_float(r[j]) - zcmax,
                                                       __uint_as_float(r[j + 1]) - zcmax);
                  pk[j >> 1] = *reinterpret_cast<const uint32_t*>(&h2);
                }
              } else {
#pragma unroll
                for (int j = 0; j < 64; j += 2) {
                  float dd[2];
#pragma unroll
                  for (int h = 0; h < 2; ++h) {
                    float z = __uint_as_float(r[j + h]);
                    if (use_softcap) z = p.softcap * softcap_tanh(z, inv_cap);
                    dd[h] = (col0 + c * 64 + j + h < p.v) ? z - zcmax : -INFINITY;
                  }
                  const __half2 h2 = __floats2half2_rn(dd[0], dd[1]);
                  pk[j >> 1] = *reinterpret_cast<const uint32_t*>(&h2);
                }
              }
#pragma unroll
              for (int q = 0; q < 8; ++q)
                dst[c * 8 + q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
            }
          }
        }
        release_acc(buf);
        if (p.tile_max && tr.ok)
          p.tile_max[((size_t)tr.n * (p.tm_stride ? p.tm_stride : p.mt) + p.tm_m0 + tr.m) * BM + row] = zmax;
        if (tr.last && valid) {  // per ORIGINAL row (rows may be compacted, filter_ignored)
          p.part[(size_t)tr.s * p.n_total + orow] = make_float2(run_m, run_s);
          if (have_corr) p.correct[orow] = corr;
        }
      } else if (MODE == KEPT) {
        if (p.st.ring == 0) {
          if (tr.ok) store_shat(tacc, col0, tr.s);
        } else if (tr.ok) {
          // streamed: wait until the slot's previous item has been read by all its consumers,
          // write S-hat, make it visible to their TMA loads (async proxy) and publish it
          const int slot = tr.s % p.st.ring, lap = tr.s / p.st.ring;
          if (epi_tid == 0) spin_until_geq(&p.st.used[slot], lap * p.st.consumers);
          named_bar_sync(1, 128);
          store_shat(tacc, col0, slot);
          fence_proxy_async_global();
          named_bar_sync(1, 128);
          if (epi_tid == 0) {
            __threadfence();
            st_release_gpu(&p.st.ready[slot], lap + 1);
          }
        }
        release_acc(buf);
      } else if (!tr.ok || tr.zero) {
        // pairs only: this CTA's tile is missing or has zero upstream while the peer's is live
        if (tr.ok && epi_tid == 0) atomicAdd(&p.counters[2], 1ull);
        release_acc(buf);
      } else {
        // ------------------------------- backward filter pass ------------------------------
        // pass 1: row max of the raw logits.  S = exp(z' - lse) is monotone in z, so
        // "all S < eps" (block_skip_decision) holds iff S(row max) < eps for every row.
        float zmax = -INFINITY;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          tmem_ld32(tacc + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (col0 + c * 32 + j < p.v) zmax = fmaxf(zmax, __uint_as_float(r[j]));
        }
        const bool big = valid && tile_row_big(zmax, lse2, p.softcap, inv_cap, p.eps);
        const bool in_tile = !p.label_split && pos_r >= col0 && pos_r < col0 + BN;
        const uint32_t wvote = __any_sync(0xffffffffu, big || in_tile);
        if (lane == 0) s_vote[(t & 1) * 4 + quarter] = wvote;
        named_bar_sync(1, 128);
        const uint32_t* vv = s_vote + (t & 1) * 4;
        const bool kept = (vv[0] | vv[1] | vv[2] | vv[3]) != 0;
        const int ln = tr.n - p.n_base;
        if (kept) {
          // one slot per kept tile, handed out in completion order; results do not depend on
          // slot numbers (the gradient passes visit tiles in index order)
          if (epi_tid == 0) {
            int slot = atomicAdd(p.slot_ctr, 1);
            if (slot >= p.capacity) {
              slot = -1;
              if (p.overflow) atomicExch(p.overflow, 1);
            } else {
              p.slot_of[(size_t)ln * p.mt + tr.m] = slot;
              atomicAdd(&p.cnt_n[ln], 1);
              atomicAdd(&p.cnt_m[tr.m], 1);
            }
            s_slot[t & 1] = slot;
            atomicAdd(&p.counters[0], 1ull);
          }
          named_bar_sync(1, 128);
          const int slot = s_slot[t & 1];
          if (slot >= 0) store_shat(tacc, col0, slot);
        } else if (epi_tid == 0) {
          atomicAdd(&p.counters[1], 1ull);
        }
        release_acc(buf);
      }
      ++t;
    }, [&](int, int count) {
      if (MODE == BWD && epi_tid == 0) atomicAdd(&p.counters[2], (unsigned long long)count);
    });
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
  if (p.sync_exit && threadIdx.x == 0) {  // every TMA read of this CTA has landed
    __threadfence();
    if (atomicAdd(p.sync_exit, 1) == nblk - 1) {
      __threadfence();
      st_release_gpu(p.sync_released, 1);
    }
  }
}

// The forward over vocabulary groups as a chain of launches (Params::sync_*): one more warp, the
// gather warp, copies the next group's rows while this launch sweeps its own.
constexpr int SYNC_THREADS = NUM_THREADS + 32;
template <int MODE, int CG>
__global__ void __launch_bounds__(SYNC_THREADS, 1)
    cce_lse_sync_kernel(const __grid_constant__ CUtensorMap tmE, const __grid_constant__ CUtensorMap tmEg,
                        const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmCg,
                        const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  lse_body<MODE, CG>(tmE, tmEg, tmC, tmCg, p, smem, (int)blockIdx.x, (int)gridDim.x);
}

template <int MODE, int CG>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cce_lse_kernel(const __grid_constant__ CUtensorMap tmE, const __grid_constant__ CUtensorMap tmEg,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmCg,
                   const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  lse_body<MODE, CG>(tmE, tmEg, tmC, tmCg, p, smem, (int)blockIdx.x, (int)gridDim.x);
}

}  // namespace cce

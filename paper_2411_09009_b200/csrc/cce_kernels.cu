// Cut Cross-Entropy for B200 (sm_100a): persistent warp-specialised tcgen05 kernels.
//
// Hot path of the reference (pkg/src/cce/kernels.py):
//   forward  = indexed_matmul (:204-251) + lse_forward (:254-319)      -> cce_fwd_kernel<FWD>
//   backward = lse_backward (:327-486) with block_skip_decision (:140) -> cce_fwd_kernel<BWD>
//
// One CTA per SM.  Tile = 128 tokens (TMEM lanes / MMA M) x 256 vocab rows (MMA N), streamed
// over D in 64-element (128 B, SWIZZLE_128B) K-blocks by TMA.  Warp roles:
//   warp 0      : TMA producer (one thread)
//   warp 1      : TMEM allocator + MMA issuer (one thread issues tcgen05.mma)
//   warps 2..5  : epilogue, thread t owns token row 32*(warp%4)+lane of the tile
// TMEM (512 cols): two 256-col logit accumulators (double buffered).  In the backward the
// consumed accumulator of tile t is reused for tile t's gradient chunks while tile t+1's
// logits accumulate in the other buffer.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cub/device/device_radix_sort.cuh>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "cce_ptx.cuh"

namespace cce {

constexpr int BM = 128;                   // tokens per tile
constexpr int BN = 256;                   // vocab rows per tile
constexpr int BK = 64;                    // D elements per K-block (one 128 B swizzle atom)
constexpr int A_BYTES = BM * BK * 2;      // 16 KiB
constexpr int B_BYTES = BN * BK * 2;      // 32 KiB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SHAT_BYTES = BM * BN * 2;   // bf16 S-hat tile, 64 KiB
constexpr int NUM_THREADS = 192;
constexpr int FWD_STAGES = 4;
constexpr int BWD_STAGES = 3;
constexpr int TMEM_COLS = 512;

enum Mode { FWD = 0, BWD = 1 };

struct Params {
  int n_rows;        // token rows handled (N, or N_valid after compaction in the backward)
  int d;             // hidden size
  int v;             // vocab rows of C (this shard)
  int nt, mt;        // token tiles, vocab tiles
  int splits;        // vocab splits per token tile (units = nt * splits)
  int num_kb;        // ceil(d / BK)
  float softcap;     // 0 => off
  // forward
  const int64_t* targets;
  int64_t ignore_index;
  int64_t vocab_start;
  float2* part;      // [splits][n_rows]  (running max, running sum) in log2 units
  float* correct;    // [n_rows] target logit (written by the tile that owns the label)
  // backward
  const float* lse;        // [n_rows] global log-sum-exp (natural log)
  const float* upstream;   // [n_rows] dLoss/dloss_i, 0 at ignored rows
  const int32_t* pos;      // [n_rows] label position in tile order, -1 if none
  const int32_t* perm;     // [mt*BN] tile-order position -> C row (nullptr = identity)
  const int32_t* row_map;  // [nt*BM] compact row -> E row / dE row (nullptr = identity)
  const uint8_t* block_zero;  // [nt] 1 if every upstream in the token tile is zero
  float eps;
  float* de_acc;           // [N_orig][d] fp32
  __nv_bfloat16* dc;       // [v][d]
  unsigned long long* counters;  // [3] kept, eps-skipped, zero-upstream-skipped
};

struct TileIter {
  // Persistent static schedule: unit u = s * nt + n (token tile fastest, so concurrently
  // running CTAs share the same vocab tiles of C while E stays L2-resident).
  int unit, units, m, m_end, n, s;
  const Params* p;
  __device__ void begin_unit() {
    n = unit % p->nt;
    s = unit / p->nt;
    m = (int)(((long long)s * p->mt) / p->splits);
    m_end = (int)(((long long)(s + 1) * p->mt) / p->splits);
  }
  __device__ bool valid() const { return unit < units; }
};

__device__ __forceinline__ uint8_t* stage_a(uint8_t* smem, int s) { return smem + s * STAGE_BYTES; }
__device__ __forceinline__ uint8_t* stage_b(uint8_t* smem, int s) {
  return smem + s * STAGE_BYTES + A_BYTES;
}

// Issue one K-block's loads: E rows [n*BM, +BM) and C rows of vocab tile m, columns [kb*BK, +BK).
__device__ __forceinline__ void load_kblock(const Params& p, const CUtensorMap* tmE,
                                            const CUtensorMap* tmC, uint8_t* sa, uint8_t* sb,
                                            uint64_t* bar, int n, int m, int kb) {
  mbar_arrive_expect_tx(bar, STAGE_BYTES);
  const int c0 = kb * BK;
  if (p.row_map == nullptr) {
    tma_load_2d(tmE, bar, sa, c0, n * BM);
  } else {
    const int4* rm = reinterpret_cast<const int4*>(p.row_map + n * BM);
#pragma unroll 4
    for (int g = 0; g < BM / 4; ++g) {
      int4 r = __ldg(rm + g);
      tma_gather4(tmE, bar, sa + g * 4 * 128, c0, r.x, r.y, r.z, r.w);
    }
  }
  if (p.perm == nullptr) {
    tma_load_2d(tmC, bar, sb, c0, m * BN);
  } else {
    const int4* pm = reinterpret_cast<const int4*>(p.perm + m * BN);
#pragma unroll 4
    for (int g = 0; g < BN / 4; ++g) {
      int4 r = __ldg(pm + g);
      tma_gather4(tmC, bar, sb + g * 4 * 128, c0, r.x, r.y, r.z, r.w);
    }
  }
}

// softcap: z' = cap * tanh(z / cap), tanh(x) = 1 - 2 / (exp(2x) + 1) (exact limits at +-inf)
__device__ __forceinline__ float softcap_tanh(float z, float inv_cap) {
  const float e = ex2_approx(z * inv_cap * 2.8853900817779268f);  // 2*log2(e)
  return 1.0f - __fdividef(2.0f, e + 1.0f);
}

template <int MODE>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cce_main_kernel(const __grid_constant__ CUtensorMap tmE,
                    const __grid_constant__ CUtensorMap tmC, const Params p) {
  constexpr int STAGES = MODE == FWD ? FWD_STAGES : BWD_STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-align the dynamic smem base (SWIZZLE_128B atoms are address based)
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* shat = smem + STAGES * STAGE_BYTES;  // BWD only
  uint8_t* ctrl = shat + (MODE == BWD ? SHAT_BYTES : 0);
  uint64_t* full = reinterpret_cast<uint64_t*>(ctrl);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;   // [2] MMA -> epilogue: logits ready
  uint64_t* acc_free = acc_full + 2;     // [2] epilogue -> MMA: accumulator reusable
  uint64_t* shat_full = acc_free + 2;    // [2] epilogue -> MMA/producer: S-hat + decision
  uint64_t* g_full = shat_full + 2;      // [2] MMA -> epilogue: dE chunk / dC chunk ready
  uint64_t* g_empty = g_full + 2;        // [2] epilogue -> MMA: chunk slot drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(g_empty + 2);
  uint32_t* s_kept = tmem_slot + 1;      // [2]
  uint32_t* s_vote = s_kept + 2;         // [2][4]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmE);
    tma_prefetch_desc(&tmC);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_free[i], 128);
      mbar_init(&shat_full[i], 1);
      mbar_init(&g_full[i], 1);
      mbar_init(&g_empty[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  TileIter it;
  it.p = &p;
  it.units = p.nt * p.splits;

  if (warp == 0) {
    // ===================================== TMA producer ==================================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      auto advance = [&]() {
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      };
      auto load_tile = [&](int n, int m) {
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          load_kblock(p, &tmE, &tmC, stage_a(smem, stage), stage_b(smem, stage), &full[stage],
                      n, m, kb);
          advance();
        }
      };
      int t = 0, prev_n = 0, prev_m = 0;
      for (it.unit = blockIdx.x; it.valid(); it.unit += gridDim.x) {
        it.begin_unit();
        if (MODE == BWD && p.block_zero[it.n]) continue;
        for (; it.m < it.m_end; ++it.m) {
          load_tile(it.n, it.m);
          if (MODE == BWD && t > 0) {
            const int tp = t - 1;
            mbar_wait(&shat_full[tp & 1], (tp >> 1) & 1);
            if (s_kept[tp & 1]) load_tile(prev_n, prev_m);
          }
          prev_n = it.n;
          prev_m = it.m;
          ++t;
        }
      }
      if (MODE == BWD && t > 0) {
        const int tp = t - 1;
        mbar_wait(&shat_full[tp & 1], (tp >> 1) & 1);
        if (s_kept[tp & 1]) load_tile(prev_n, prev_m);
      }
    }
  } else if (warp == 1) {
    // ===================================== MMA issuer ====================================
    if (lane == 0) {
      constexpr uint32_t IDESC_LOGITS = make_idesc_bf16(BM, BN, 0, 0);
      constexpr uint32_t IDESC_DE = make_idesc_bf16(BM, BK, 0, 1);  // A=S-hat K-major, B=C MN-major
      constexpr uint32_t IDESC_DC = make_idesc_bf16(BM, BK, 1, 1);  // A=S-hat^T MN-major, B=E MN-major
      int stage = 0;
      uint32_t phase = 0;
      uint32_t g_phase[2] = {0, 0};
      auto advance = [&]() {
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      };
      auto logits_tile = [&](int t) {
        const int buf = t & 1;
        mbar_wait(&acc_free[buf], ((t >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * BN;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(stage_a(smem, stage));
          const uint32_t b0 = smem_u32(stage_b(smem, stage));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            mma_bf16_ss(d_tmem, make_sdesc(a0 + 32 * k, 0, 1024), make_sdesc(b0 + 32 * k, 0, 1024),
                        IDESC_LOGITS, (kb | k) != 0);
          }
          mma_commit(&empty[stage]);
          advance();
        }
        mma_commit(&acc_full[buf]);
      };
      auto grad_tile = [&](int t) {
        mbar_wait(&shat_full[t & 1], (t >> 1) & 1);
        if (!s_kept[t & 1]) return;
        tc_fence_after();
        const uint32_t base = tmem_base + (t & 1) * BN;
        const uint32_t sh = smem_u32(shat);
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t ea = smem_u32(stage_a(smem, stage));  // E block [128 tok][64 d]
          const uint32_t cb = smem_u32(stage_b(smem, stage));  // C block [256 voc][64 d]
          // dE[tok, d] += S-hat[tok, voc] * C[voc, d]     (M=128 tok, N=64 d, K=256 voc)
          mbar_wait(&g_empty[0], g_phase[0] ^ 1);
          tc_fence_after();
#pragma unroll
          for (int ks = 0; ks < BN / 16; ++ks) {
            const uint32_t a = sh + (ks >> 2) * (BM * 128) + (ks & 3) * 32;
            mma_bf16_ss(base, make_sdesc(a, 0, 1024), make_sdesc(cb + ks * 2048, B_BYTES, 1024),
                        IDESC_DE, ks != 0);
          }
          mma_commit(&g_full[0]);
          g_phase[0] ^= 1;
          // dC[voc, d] += S-hat^T[voc, tok] * E[tok, d]   (2 x M=128 voc, N=64 d, K=128 tok)
          mbar_wait(&g_empty[1], g_phase[1] ^ 1);
          tc_fence_after();
#pragma unroll
          for (int blk = 0; blk < 2; ++blk) {
#pragma unroll
            for (int ks = 0; ks < BM / 16; ++ks) {
              const uint32_t a = sh + (2 * blk) * (BM * 128) + ks * 2048;
              mma_bf16_ss(base + BK + blk * BK, make_sdesc(a, BM * 128, 1024),
                          make_sdesc(ea + ks * 2048, A_BYTES, 1024), IDESC_DC, ks != 0);
            }
          }
          mma_commit(&g_full[1]);
          g_phase[1] ^= 1;
          mma_commit(&empty[stage]);
          advance();
        }
      };
      int t = 0;
      for (it.unit = blockIdx.x; it.valid(); it.unit += gridDim.x) {
        it.begin_unit();
        if (MODE == BWD && p.block_zero[it.n]) continue;
        for (; it.m < it.m_end; ++it.m) {
          logits_tile(t);
          if (MODE == BWD && t > 0) grad_tile(t - 1);
          ++t;
        }
      }
      if (MODE == BWD && t > 0) grad_tile(t - 1);
    }
  } else {
    // ===================================== epilogue ======================================
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const bool use_softcap = p.softcap > 0.f;
    const float inv_cap = use_softcap ? 1.0f / p.softcap : 0.f;
    constexpr float LOG2E = 1.4426950408889634f;
    int t = 0;
    uint32_t g_phase[2] = {0, 0};
    const int epi_tid = threadIdx.x - 64;  // 0..127

    for (it.unit = blockIdx.x; it.valid(); it.unit += gridDim.x) {
      it.begin_unit();
      const int grow = it.n * BM + row;
      const bool valid = grow < p.n_rows;
      if (MODE == FWD) {
        int64_t tpos = -1;
        if (valid) {
          const int64_t tg = p.targets[grow];
          if (tg != p.ignore_index) tpos = tg - p.vocab_start;
        }
        float run_m = -INFINITY, run_s = 0.f, corr = 0.f;
        bool have_corr = false;
        for (; it.m < it.m_end; ++it.m, ++t) {
          const int buf = t & 1;
          mbar_wait(&acc_full[buf], (t >> 1) & 1);
          tc_fence_after();
          const int col0 = it.m * BN;
          const bool tile_has_t = tpos >= col0 && tpos < col0 + BN;
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(tmem_base + lane_off + buf * BN + c * 32, r);
            tmem_ld_wait();
            float y[32];
            float cm = -INFINITY;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              float z = __uint_as_float(r[j]);
              if (use_softcap) z = p.softcap * softcap_tanh(z, inv_cap);
              const int col = col0 + c * 32 + j;
              if (tile_has_t && col == tpos) { corr = z; have_corr = true; }
              y[j] = col < p.v ? z * LOG2E : -INFINITY;
              cm = fmaxf(cm, y[j]);
            }
            const float nm = fmaxf(run_m, cm);
            if (nm != -INFINITY) {
              float acc = 0.f;
#pragma unroll
              for (int j = 0; j < 32; ++j) acc += ex2_approx(y[j] - nm);
              run_s = run_s * ex2_approx(run_m - nm) + acc;
              run_m = nm;
            }
          }
          tc_fence_before();
          mbar_arrive(&acc_free[buf]);
        }
        if (valid) {
          p.part[(size_t)it.s * p.n_rows + grow] = make_float2(run_m, run_s);
          if (have_corr) p.correct[grow] = corr;
        }
      } else {
        // ---------------------------------- backward ------------------------------------
        if (p.block_zero[it.n]) {
          if (epi_tid == 0) atomicAdd(&p.counters[2], (unsigned long long)(it.m_end - it.m));
          continue;
        }
        const float lse_r = valid ? p.lse[grow] : INFINITY;
        const float up_r = valid ? p.upstream[grow] : 0.f;
        const int pos_r = valid ? p.pos[grow] : -1;
        const int drow = valid ? (p.row_map ? p.row_map[grow] : grow) : 0;
        const float lse2 = lse_r * LOG2E;
        for (; it.m < it.m_end; ++it.m, ++t) {
          const int buf = t & 1;
          mbar_wait(&acc_full[buf], (t >> 1) & 1);
          tc_fence_after();
          const int col0 = it.m * BN;
          const bool in_tile = pos_r >= col0 && pos_r < col0 + BN;
          bool big = false;
#pragma unroll 1
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(tmem_base + lane_off + buf * BN + c * 32, r);
            tmem_ld_wait();
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
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
                const int col = col0 + c * 32 + j + h;
                const float s = (col < p.v) ? ex2_approx(z * LOG2E - lse2) : 0.f;
                big |= (s >= p.eps);
                const float g = (col == pos_r) ? s - 1.f : s;
                g2[h] = g * up_r * dcap;
              }
              pk[j >> 1] = pack_bf16x2(g2[0], g2[1]);
            }
            // S-hat row `row`, vocab [c*32, c*32+32): K-major SWIZZLE_128B, atom = 64 vocab
            uint8_t* atom = shat + (c >> 1) * (BM * 128) + row * 128;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int chunk = (c & 1) * 4 + q;
              uint4 val = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
              *reinterpret_cast<uint4*>(atom + ((chunk ^ (row & 7)) << 4)) = val;
            }
          }
          fence_proxy_async_smem();
          tc_fence_before();
          const uint32_t wvote = __any_sync(0xffffffffu, big || in_tile);
          if (lane == 0) s_vote[(t & 1) * 4 + quarter] = wvote;
          named_bar_sync(1, 128);
          const uint32_t* vv = s_vote + (t & 1) * 4;
          const bool kept = (vv[0] | vv[1] | vv[2] | vv[3]) != 0;
          if (epi_tid == 0) {
            s_kept[t & 1] = kept ? 1u : 0u;
            atomicAdd(&p.counters[kept ? 0 : 1], 1ull);
            mbar_arrive(&shat_full[t & 1]);
          }
          if (kept) {
            const uint32_t gbase = tmem_base + lane_off + buf * BN;
            const int vpos0 = col0 + row;        // dC block 0 row (tile order)
            const int vpos1 = col0 + BM + row;   // dC block 1 row
            const int vrow0 = vpos0 < p.v ? (p.perm ? p.perm[vpos0] : vpos0) : -1;
            const int vrow1 = vpos1 < p.v ? (p.perm ? p.perm[vpos1] : vpos1) : -1;
            for (int kb = 0; kb < p.num_kb; ++kb) {
              const int dcol = kb * BK;
              // ---- dE chunk: row `row`, 64 fp32 columns
              mbar_wait(&g_full[0], g_phase[0]);
              g_phase[0] ^= 1;
              tc_fence_after();
              {
                uint32_t r0[32], r1[32];
                tmem_ld32(gbase + 0, r0);
                tmem_ld32(gbase + 32, r1);
                tmem_ld_wait();
                tc_fence_before();
                mbar_arrive(&g_empty[0]);
                if (valid) {
                  float* dst = p.de_acc + (size_t)drow * p.d + dcol;
                  const int lim = min(BK, p.d - dcol);
#pragma unroll
                  for (int j = 0; j < 32; j += 4)
                    if (j < lim)
                      red_add_v4_f32(dst + j, __uint_as_float(r0[j]), __uint_as_float(r0[j + 1]),
                                     __uint_as_float(r0[j + 2]), __uint_as_float(r0[j + 3]));
#pragma unroll
                  for (int j = 0; j < 32; j += 4)
                    if (32 + j < lim)
                      red_add_v4_f32(dst + 32 + j, __uint_as_float(r1[j]),
                                     __uint_as_float(r1[j + 1]), __uint_as_float(r1[j + 2]),
                                     __uint_as_float(r1[j + 3]));
                }
              }
              // ---- dC chunk: vocab rows vpos0 / vpos1, 64 columns each
              mbar_wait(&g_full[1], g_phase[1]);
              g_phase[1] ^= 1;
              tc_fence_after();
#pragma unroll
              for (int blk = 0; blk < 2; ++blk) {
                uint32_t r0[32], r1[32];
                tmem_ld32(gbase + BK + blk * BK, r0);
                tmem_ld32(gbase + BK + blk * BK + 32, r1);
                tmem_ld_wait();
                if (blk == 1) {
                  tc_fence_before();
                  mbar_arrive(&g_empty[1]);
                }
                const int vrow = blk ? vrow1 : vrow0;
                if (vrow >= 0) {
                  __nv_bfloat16* dst = p.dc + (size_t)vrow * p.d + dcol;
                  const int lim = min(BK, p.d - dcol);
#pragma unroll
                  for (int j = 0; j < 32; j += 8)
                    if (j < lim)
                      red_add_v4_bf16x2(
                          dst + j,
                          pack_bf16x2(__uint_as_float(r0[j]), __uint_as_float(r0[j + 1])),
                          pack_bf16x2(__uint_as_float(r0[j + 2]), __uint_as_float(r0[j + 3])),
                          pack_bf16x2(__uint_as_float(r0[j + 4]), __uint_as_float(r0[j + 5])),
                          pack_bf16x2(__uint_as_float(r0[j + 6]), __uint_as_float(r0[j + 7])));
#pragma unroll
                  for (int j = 0; j < 32; j += 8)
                    if (32 + j < lim)
                      red_add_v4_bf16x2(
                          dst + 32 + j,
                          pack_bf16x2(__uint_as_float(r1[j]), __uint_as_float(r1[j + 1])),
                          pack_bf16x2(__uint_as_float(r1[j + 2]), __uint_as_float(r1[j + 3])),
                          pack_bf16x2(__uint_as_float(r1[j + 4]), __uint_as_float(r1[j + 5])),
                          pack_bf16x2(__uint_as_float(r1[j + 6]), __uint_as_float(r1[j + 7])));
                }
              }
            }
          }
          mbar_arrive(&acc_free[buf]);
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

// ---------------------------------------------------------------------------------------
// Small kernels
// ---------------------------------------------------------------------------------------

// Merge the per-split (max2, sum2) partials of each row into this shard's natural-log LSE.
__global__ void combine_splits_kernel(const float2* __restrict__ part, int splits, int n,
                                      float* __restrict__ lse_local) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float m = -INFINITY;
  for (int s = 0; s < splits; ++s) m = fmaxf(m, part[(size_t)s * n + i].x);
  float acc = 0.f;
  if (m != -INFINITY)
    for (int s = 0; s < splits; ++s) {
      const float2 v = part[(size_t)s * n + i];
      acc += v.y * exp2f(v.x - m);
    }
  lse_local[i] = (m == -INFINITY) ? -INFINITY : (m + log2f(acc)) * 0.6931471805599453f;
}

// Vocab-parallel / single-shard finish: lse = logaddexp over shards, correct = sum over shards.
// Mirrors cce_loss's scatter (kernels.py:539-547): loss and lse are 0 at ignored rows.
__global__ void merge_shards_kernel(int P, const float* __restrict__ lse_parts,
                                    const float* __restrict__ correct_parts,
                                    const int64_t* __restrict__ targets, int64_t ignore_index,
                                    int n, float* __restrict__ lse_out, float* __restrict__ loss_out) {
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
  const bool valid = targets[i] != ignore_index;
  lse_out[i] = valid ? lse : 0.f;
  loss_out[i] = valid ? lse - corr : 0.f;
}

// zero a float buffer (used for `correct` so rows whose label lives in another shard read 0)
__global__ void fill_kernel(float* __restrict__ x, float v, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = v;
}

// Column mean of E over valid rows, fp32: ebar[d] = sum_i valid_i * E[i, d] / n_valid.
__global__ void ebar_kernel(const __nv_bfloat16* __restrict__ E, const int64_t* __restrict__ targets,
                            int64_t ignore_index, int n, int d, float* __restrict__ ebar_acc,
                            int rows_per_block) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= d) return;
  const int r0 = blockIdx.y * rows_per_block;
  const int r1 = min(n, r0 + rows_per_block);
  float acc = 0.f;
  for (int r = r0; r < r1; ++r)
    if (targets == nullptr || targets[r] != ignore_index) acc += __bfloat162float(E[(size_t)r * d + col]);
  atomicAdd(&ebar_acc[col], acc);
}

// key[v] = C[v] . ebar  (fp32); one warp per vocab row.  Equals lse_forward's mean_logits
// (kernels.py:305-308, :317-318), which is a mean of logits over the valid tokens.
__global__ void sort_key_kernel(const __nv_bfloat16* __restrict__ C, const float* __restrict__ ebar_sum,
                                float inv_n, int v, int d, float* __restrict__ key) {
  const int warps = blockDim.x >> 5;
  const int row = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= v) return;
  const __nv_bfloat16* c = C + (size_t)row * d;
  float acc = 0.f;
  for (int j = lane * 8; j < d; j += 256) {
    const uint4 raw = *reinterpret_cast<const uint4*>(c + j);
    const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += __bfloat162float(h[q]) * ebar_sum[j + q];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) key[row] = acc * inv_n;
}

// out[i] = C[x_i] . E[i] (indexed_matmul, kernels.py:204-251); one warp per token row.
__global__ void indexed_dot_kernel(const __nv_bfloat16* __restrict__ E, const __nv_bfloat16* __restrict__ C,
                                   const int64_t* __restrict__ targets, int64_t ignore_index,
                                   int64_t vocab_start, int n, int d, int v, float softcap,
                                   float* __restrict__ out) {
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
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = i;
}

// inv[perm[j]] = j for j < v ; padding positions of perm (>= v) point at row 0.
__global__ void invert_perm_kernel(const int32_t* __restrict__ perm, int v, int vpad,
                                   int32_t* __restrict__ perm_padded, int32_t* __restrict__ inv) {
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

// block_zero[b] = all upstream of token tile b are exactly zero (kernels.py:434-438)
__global__ void block_zero_kernel(const float* __restrict__ up, int n, uint8_t* __restrict__ bz) {
  const int b = blockIdx.x;
  const int i = b * BM + threadIdx.x;
  const bool nz = (i < n) && (up[i] != 0.f);
  const int any = __syncthreads_or(nz);
  if (threadIdx.x == 0) bz[b] = any ? 0 : 1;
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                   int64_t n4) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n4) return;
  const float4 v = reinterpret_cast<const float4*>(x)[i];
  uint2 o;
  o.x = pack_bf16x2(v.x, v.y);
  o.y = pack_bf16x2(v.z, v.w);
  reinterpret_cast<uint2*>(y)[i] = o;
}

}  // namespace cce

// =========================================================================================
// Host side: C ABI
// =========================================================================================
namespace {

thread_local std::string g_last_error;

int fail(const std::string& msg) {
  g_last_error = msg;
  return 1;
}

#define CCE_CUDA(call)                                                               \
  do {                                                                               \
    cudaError_t _e = (call);                                                         \
    if (_e != cudaSuccess)                                                           \
      return fail(std::string(#call) + ": " + cudaGetErrorString(_e));               \
  } while (0)

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, []() {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &ptr, 12000,
                                         cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// Row-major bf16 [rows, cols] matrix, box = [box_rows x 64 cols], 128 B swizzle.
bool make_tmap(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows) {
  auto enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols * 2)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(cce::BK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int gather_box_rows() {
  static int rows = [] {
    const char* e = getenv("CCE_GATHER4_BOX_ROWS");
    return e ? atoi(e) : 1;
  }();
  return rows;
}

int num_sms() {
  static int sms = -1;
  if (sms < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const char* e = getenv("CCE_NUM_CTAS");
    if (e && atoi(e) > 0) sms = atoi(e);
  }
  return sms;
}

size_t smem_bytes(int mode) {
  const int stages = mode == cce::FWD ? cce::FWD_STAGES : cce::BWD_STAGES;
  return 1024 + (size_t)stages * cce::STAGE_BYTES + (mode == cce::BWD ? cce::SHAT_BYTES : 0) + 256;
}

template <int MODE>
int ensure_attr() {
  static cudaError_t st = [] {
    return cudaFuncSetAttribute(cce::cce_main_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem_bytes(MODE));
  }();
  if (st != cudaSuccess) return fail(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(st));
  return 0;
}

// Choose the vocab split count so units = nt*splits balance over the persistent grid.
int choose_splits(int nt, int mt, int grid, bool prefer_fine) {
  int best = 1;
  double best_eff = -1.0;
  const int max_s = mt;
  for (int s = 1; s <= max_s; ++s) {
    const long long units = (long long)nt * s;
    const long long waves = (units + grid - 1) / grid;
    // per-CTA load: ceil(mt/s) tiles per unit * waves
    const double load = (double)waves * ((mt + s - 1) / s);
    const double eff = (double)nt * mt / (grid * load);
    const double score = eff - (prefer_fine ? 0.0 : 1e-4 * s);
    if (score > best_eff + 1e-9) { best_eff = score; best = s; }
    if (units >= 64LL * grid) break;
  }
  return best;
}

}  // namespace

extern "C" {

const char* cce_last_error(void) { return g_last_error.c_str(); }

int cce_abi_version(void) { return 1; }

size_t cce_fwd_workspace_bytes(int64_t n, int64_t d, int64_t v) {
  const int nt = (int)((n + cce::BM - 1) / cce::BM);
  const int mt = (int)((v + cce::BN - 1) / cce::BN);
  const int s = choose_splits(nt, mt, num_sms(), false);
  (void)d;
  return (size_t)s * (size_t)n * sizeof(float2);
}

int cce_fwd(const void* E, const void* C, const int64_t* targets, int64_t n, int64_t d, int64_t v,
            int64_t ignore_index, int64_t vocab_start, float softcap, void* ws, size_t ws_bytes,
            float* lse_local, float* correct, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (n < 0 || d <= 0 || v <= 0) return fail("cce_fwd: bad sizes");
  if (d % 8 != 0) return fail("cce_fwd: D must be a multiple of 8 (16-byte TMA row pitch)");
  if (n == 0) return 0;
  const int nt = (int)((n + cce::BM - 1) / cce::BM);
  const int mt = (int)((v + cce::BN - 1) / cce::BN);
  const int grid = num_sms();
  const int splits = choose_splits(nt, mt, grid, false);
  if (ws_bytes < (size_t)splits * n * sizeof(float2)) return fail("cce_fwd: workspace too small");
  if (int e = ensure_attr<cce::FWD>()) return e;
  CUtensorMap tmE, tmC;
  if (!make_tmap(&tmE, E, n, d, cce::BM) || !make_tmap(&tmC, C, v, d, cce::BN))
    return fail("cce_fwd: cuTensorMapEncodeTiled failed");
  cce::Params p{};
  p.n_rows = (int)n;
  p.d = (int)d;
  p.v = (int)v;
  p.nt = nt;
  p.mt = mt;
  p.splits = splits;
  p.num_kb = (int)((d + cce::BK - 1) / cce::BK);
  p.softcap = softcap;
  p.targets = targets;
  p.ignore_index = ignore_index;
  p.vocab_start = vocab_start;
  p.part = static_cast<float2*>(ws);
  p.correct = correct;
  const int units = nt * splits;
  cce::fill_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(correct, 0.f, n);
  cce::cce_main_kernel<cce::FWD><<<std::min(grid, units), cce::NUM_THREADS, smem_bytes(cce::FWD), stream>>>(
      tmE, tmC, p);
  CCE_CUDA(cudaGetLastError());
  cce::combine_splits_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(
      static_cast<const float2*>(ws), splits, (int)n, lse_local);
  CCE_CUDA(cudaGetLastError());
  return 0;
}

int cce_merge_shards(int num_shards, const float* lse_parts, const float* correct_parts,
                     const int64_t* targets, int64_t ignore_index, int64_t n, float* lse_out,
                     float* loss_out, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (n == 0) return 0;
  cce::merge_shards_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(
      num_shards, lse_parts, correct_parts, targets, ignore_index, (int)n, lse_out, loss_out);
  CCE_CUDA(cudaGetLastError());
  return 0;
}

size_t cce_sort_workspace_bytes(int64_t v) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, (const float*)nullptr, (float*)nullptr,
                                            (const int32_t*)nullptr, (int32_t*)nullptr, (int)v);
  // + key(v) + sorted key(v) + iota(v) floats/ints + ebar staging handled by caller
  return bytes + 3 * (size_t)v * 4 + 1024;
}

// Vocabulary order for the backward (compute_vocab_order, kernels.py:145-160): stable sort of
// the mean logit C.ebar, descending, ties by ascending index.  ebar_sum must hold the column
// sums of the valid rows of E (see cce_ebar), n_valid their count.
int cce_ebar(const void* E, const int64_t* targets, int64_t ignore_index, int64_t n, int64_t d,
             float* ebar_sum, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  CCE_CUDA(cudaMemsetAsync(ebar_sum, 0, d * sizeof(float), stream));
  if (n == 0) return 0;
  const int rows_per_block = 64;
  dim3 grid((unsigned)((d + 127) / 128), (unsigned)((n + rows_per_block - 1) / rows_per_block));
  cce::ebar_kernel<<<grid, 128, 0, stream>>>(static_cast<const __nv_bfloat16*>(E), targets,
                                             ignore_index, (int)n, (int)d, ebar_sum, rows_per_block);
  CCE_CUDA(cudaGetLastError());
  return 0;
}

int cce_vocab_order(const void* C, const float* ebar_sum, int64_t n_valid, int64_t v, int64_t d,
                    int32_t* perm, float* key_out, void* ws, size_t ws_bytes, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (d % 8 != 0) return fail("cce_vocab_order: D must be a multiple of 8");
  const size_t need = cce_sort_workspace_bytes(v);
  if (ws_bytes < need) return fail("cce_vocab_order: workspace too small");
  uint8_t* w = static_cast<uint8_t*>(ws);
  float* key = reinterpret_cast<float*>(w);
  float* key_sorted = key + v;
  int32_t* idx = reinterpret_cast<int32_t*>(key_sorted + v);
  void* tmp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(idx + v) + 255) & ~uintptr_t(255));
  size_t tmp_bytes = need - 3 * (size_t)v * 4 - 1024;
  const float inv_n = n_valid > 0 ? 1.0f / (float)n_valid : 0.f;
  cce::sort_key_kernel<<<(unsigned)((v + 7) / 8), 256, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(C), ebar_sum, inv_n, (int)v, (int)d, key);
  CCE_CUDA(cudaGetLastError());
  cce::iota_kernel<<<(unsigned)((v + 255) / 256), 256, 0, stream>>>(idx, (int)v);
  CCE_CUDA(cudaGetLastError());
  CCE_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, tmp_bytes, key, key_sorted, idx, perm,
                                                     (int)v, 0, 32, stream));
  if (key_out) CCE_CUDA(cudaMemcpyAsync(key_out, key, v * 4, cudaMemcpyDeviceToDevice, stream));
  return 0;
}

// Backward prep: padded perm / inverse perm, label positions, zero-upstream tile flags.
int cce_bwd_prep(const int32_t* perm, int64_t v, const int64_t* targets, int64_t ignore_index,
                 int64_t vocab_start, const float* upstream, int64_t n, int32_t* perm_padded,
                 int32_t* inv_perm, int32_t* pos, uint8_t* block_zero, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  const int64_t vpad = ((v + cce::BN - 1) / cce::BN) * cce::BN;
  if (perm) {
    cce::invert_perm_kernel<<<(unsigned)((vpad + 255) / 256), 256, 0, stream>>>(
        perm, (int)v, (int)vpad, perm_padded, inv_perm);
    CCE_CUDA(cudaGetLastError());
  }
  if (n > 0) {
    cce::label_pos_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(
        targets, ignore_index, vocab_start, (int)v, perm ? inv_perm : nullptr, (int)n, pos);
    CCE_CUDA(cudaGetLastError());
    const int nt = (int)((n + cce::BM - 1) / cce::BM);
    cce::block_zero_kernel<<<nt, cce::BM, 0, stream>>>(upstream, (int)n, block_zero);
    CCE_CUDA(cudaGetLastError());
  }
  return 0;
}

// Filtered backward (lse_backward).  Rows are the (possibly compacted) token rows; row_map
// maps them to E / dE rows (nullptr = identity, else padded to a multiple of 128 entries).
// de_acc (fp32, N_orig x D) and dc (bf16, V x D) must be zeroed by the caller.
int cce_bwd(const void* E, int64_t e_rows, const void* C, const int32_t* perm_padded,
            const int32_t* row_map, const int32_t* pos, const float* lse, const float* upstream,
            const uint8_t* block_zero, int64_t n_rows, int64_t d, int64_t v, float softcap,
            float eps, float* de_acc, void* dc, unsigned long long* counters, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (d % 8 != 0) return fail("cce_bwd: D must be a multiple of 8");
  if (n_rows == 0) return 0;
  if (int e = ensure_attr<cce::BWD>()) return e;
  const int nt = (int)((n_rows + cce::BM - 1) / cce::BM);
  const int mt = (int)((v + cce::BN - 1) / cce::BN);
  const int grid = num_sms();
  const int splits = choose_splits(nt, mt, grid, true);
  CUtensorMap tmE, tmC;
  const bool ok = make_tmap(&tmE, E, e_rows, d, row_map ? gather_box_rows() : cce::BM) &&
                  make_tmap(&tmC, C, v, d, perm_padded ? gather_box_rows() : cce::BN);
  if (!ok) return fail("cce_bwd: cuTensorMapEncodeTiled failed");
  cce::Params p{};
  p.n_rows = (int)n_rows;
  p.d = (int)d;
  p.v = (int)v;
  p.nt = nt;
  p.mt = mt;
  p.splits = splits;
  p.num_kb = (int)((d + cce::BK - 1) / cce::BK);
  p.softcap = softcap;
  p.lse = lse;
  p.upstream = upstream;
  p.pos = pos;
  p.perm = perm_padded;
  p.row_map = row_map;
  p.block_zero = block_zero;
  p.eps = eps;
  p.de_acc = de_acc;
  p.dc = static_cast<__nv_bfloat16*>(dc);
  p.counters = counters;
  const int units = nt * splits;
  cce::cce_main_kernel<cce::BWD><<<std::min(grid, units), cce::NUM_THREADS, smem_bytes(cce::BWD), stream>>>(
      tmE, tmC, p);
  CCE_CUDA(cudaGetLastError());
  return 0;
}

int cce_indexed_dot(const void* E, const void* C, const int64_t* targets, int64_t n, int64_t d,
                    int64_t v, int64_t ignore_index, int64_t vocab_start, float softcap, float* out,
                    void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (d % 8 != 0) return fail("cce_indexed_dot: D must be a multiple of 8");
  if (n == 0) return 0;
  cce::indexed_dot_kernel<<<(unsigned)((n + 7) / 8), 256, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(E), static_cast<const __nv_bfloat16*>(C), targets,
      ignore_index, vocab_start, (int)n, (int)d, (int)v, softcap, out);
  CCE_CUDA(cudaGetLastError());
  return 0;
}

int cce_f32_to_bf16(const float* x, void* y, int64_t count, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (count % 4 != 0) return fail("cce_f32_to_bf16: count must be a multiple of 4");
  const int64_t n4 = count / 4;
  if (n4 == 0) return 0;
  cce::f32_to_bf16_kernel<<<(unsigned)((n4 + 255) / 256), 256, 0, stream>>>(
      x, static_cast<__nv_bfloat16*>(y), n4);
  CCE_CUDA(cudaGetLastError());
  return 0;
}

}  // extern "C"

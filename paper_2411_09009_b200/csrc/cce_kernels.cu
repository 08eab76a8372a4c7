// Cut Cross-Entropy for B200 (sm_100a): host side of libcce_b200.so (C ABI, include/cce_b200.h).
//
// Hot path of the reference (pkg/src/cce/kernels.py) and the kernels that replace it:
//   indexed_matmul (:204-251) + lse_forward (:254-319)  -> cce_lse_kernel<FWD>   (cce_lse_kernel.cuh)
//   lse_backward (:327-486): recompute / S / filter     -> cce_lse_kernel<BWD>   (B1)
//                            dE += S-hat C               -> cce_de_kernel        (B2, cce_grad_kernels.cuh)
//                            dC += S-hat^T E             -> cce_dc_kernel        (B3)
//   compute_vocab_order (:145-160), log_add_exp merges, prep and casts         (cce_aux_kernels.cuh)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "cce_aux_kernels.cuh"
#include "cce_grad_kernels.cuh"
#include "cce_lse_kernel.cuh"
#include "cce_stream.cuh"

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

// 3-D view of a row-major bf16 [rows, cols] matrix as {64 (within atom), rows, cols/64 atoms};
// a box {64, box_rows, box_atoms} lands as box_atoms consecutive 128B-swizzled [box_rows][64]
// atoms, i.e. one request for a whole MN-major / multi-atom K-major operand tile.
bool make_tmap3d(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int box_rows,
                 int box_atoms) {
  auto enc = get_encode_fn();
  if (!enc || cols % 64 != 0) return false;
  cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols / 64)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(cols * 2), 128};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(box_atoms)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 3-D view {inner, rows, cols/inner} with box {inner, box_rows, box_atoms} and the swizzle that
// matches inner * 2 bytes (128 B or 64 B rows).
bool make_tmap3d_inner(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int inner,
                       int box_rows, int box_atoms) {
  auto enc = get_encode_fn();
  if (!enc || cols % inner != 0) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(rows),
                        static_cast<cuuint64_t>(cols / inner)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(cols * 2), static_cast<cuuint64_t>(inner * 2)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(inner), static_cast<cuuint32_t>(box_rows),
                       static_cast<cuuint32_t>(box_atoms)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   inner == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
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

// A non-blocking side stream and fork/join events per host thread and device (created once;
// stream-capture safe: the fork/join is expressed with event record / wait only).  Per thread,
// so concurrent callers never re-record each other's join event between record and wait.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};

SideStream* side_stream() {
  thread_local SideStream per_dev[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  SideStream& x = per_dev[dev];
  if (!x.s) {
    if (cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming) != cudaSuccess) {
      x.s = nullptr;
      return nullptr;
    }
  }
  return &x;
}

// The last streamed pass launched on a device (cce_bwd_stream_ex): passes are chained across streams.
struct PassOrder {
  std::mutex mu;
  cudaEvent_t last = nullptr;
  cudaStream_t stream = nullptr;
};
PassOrder& pass_order(int dev) {
  static PassOrder po[64];
  return po[dev & 63];
}

constexpr size_t kCtrlBytes = 256;
static_assert(kCtrlBytes == cce::LSE_CTRL_BYTES, "logit-tile kernel control block");
constexpr size_t kLseSmem = 1024 + (size_t)cce::LSE_STAGES * cce::STAGE_BYTES + kCtrlBytes + cce::LSE_IDX_BYTES;
constexpr size_t kLsePairSmem =
    1024 + (size_t)cce::LSE_STAGES_PAIR * cce::PAIR_STAGE_BYTES + kCtrlBytes + cce::LSE_IDX_BYTES;
template <int CH, int KV>
constexpr size_t de_smem() { return 1024 + (size_t)cce::DeCfg<CH, KV>::SMEM + kCtrlBytes + 64; }
constexpr size_t kDcSmem =
    1024 + (size_t)cce::DC_STAGES * cce::DC_STAGE_BYTES + cce::DC_STG_BYTES + kCtrlBytes + cce::DC_IDX_BYTES + 64;

// Launches inside the kept backward's pass chain use programmatic dependent launch (every kernel
// there begins with griddepcontrol.wait): the next kernel is scheduled while its predecessor
// drains, which matters for the worst-case fallback chain -- a few dozen gated-off launches per
// step that otherwise cost a full launch gap each.  CCE_PDL=0 turns it off.
thread_local bool g_pdl = true;  // every launch of this library; CCE_PDL=0 turns it off

bool pdl_allowed() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("CCE_PDL");
    v = e ? atoi(e) : 1;
  }
  return v != 0;
}

struct PdlScope {
  bool prev;
  explicit PdlScope(bool on) : prev(g_pdl) { g_pdl = on && pdl_allowed(); }
  ~PdlScope() { g_pdl = prev; }
};

// every kernel this library launches (cce_launch_count): the bench's gpu_launches claim
std::atomic<unsigned long long> g_launches{0};

// cudaLaunchKernelEx with an optional cluster dimension and the PDL attribute when g_pdl is set
template <typename... KArgs, typename... Args>
int launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, int cluster,
             Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  unsigned na = 0;
  if (cluster > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (g_pdl && pdl_allowed()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  CCE_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return 0;
}

// kernel<<<grid, block, smem, stream>>>(args) with the launch attributes of launch_k
#ifndef CCE_SORTKEY_BPS
#define CCE_SORTKEY_BPS 8  // sort-key GEMV blocks per SM (profiles/r1/ab/sort_key_unroll.txt)
#endif
#define PDL_LAUNCH(kernel, grid, block, smem, stream, ...)                                      \
  do {                                                                                         \
    if (int e_ = launch_k(kernel, grid, block, (size_t)(smem), stream, 1, __VA_ARGS__)) return e_; \
  } while (0)

template <typename K>
int ensure_attr(K kernel, size_t bytes) {
  // cudaFuncSetAttribute is cheap; call it every launch so multi-device use stays correct.
  cudaError_t st = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (st != cudaSuccess) return fail(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(st));
  return 0;
}

// Token tiles per raster band: concurrent CTAs then read at most this many E tiles, which must
// stay L2-resident (~40 MB of the 126 MB L2; C tiles stream through the rest).
int choose_band(int64_t d) {
  const int64_t e_tile = (int64_t)cce::BM * d * 2;
  return (int)std::max<int64_t>(1, (40ll << 20) / e_tile);
}

// Splits must give every band enough units to fill the grid.
int clamp_splits(int splits, int nt, int mt, int band, int grid) {
  const int nb = std::max(1, std::min(band, nt));
  const int need = (grid + nb - 1) / nb;
  return std::min(mt, std::max(splits, need));
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

// Backward workspace: compact S-hat slots + compacted E + per-group maps.
struct BwdWs {
  __nv_bfloat16* shat;
  __nv_bfloat16* e_compact;  // [n][d] compacted rows of E
  uint8_t* block_zero;       // [token tiles]
  int32_t* slot_of;          // [group_tiles * mt], -1 = not stored
  int* slot_ctr;             // [1]
  int* cnt_n;                // [group_tiles]
  int* cnt_m;                // [mt]
  size_t map_bytes;          // slot_of
  size_t zero_bytes;         // slot_ctr + counts
  size_t total;
};

BwdWs bwd_layout(void* base, int64_t n, int64_t d, int64_t v, int64_t group_tiles, int64_t capacity) {
  const int64_t mt = (v + cce::BN - 1) / cce::BN;
  const int64_t nt = (n + cce::BM - 1) / cce::BM;
  auto up = [](size_t x) { return (x + 1023) & ~size_t(1023); };
  const size_t shat = up((size_t)capacity * cce::SHAT_TILE_BYTES);
  const size_t ec = up((size_t)n * d * 2);
  const size_t bz = up((size_t)nt);
  const size_t map = up((size_t)group_tiles * mt * 4);
  const size_t ctr = 256;
  const size_t cn = up((size_t)group_tiles * 4);
  const size_t cm = up((size_t)mt * 4);
  uint8_t* b = static_cast<uint8_t*>(base);
  BwdWs w;
  size_t o = 0;
  w.shat = reinterpret_cast<__nv_bfloat16*>(b + o); o += shat;
  w.e_compact = reinterpret_cast<__nv_bfloat16*>(b + o); o += ec;
  w.block_zero = b + o; o += bz;
  w.slot_of = reinterpret_cast<int32_t*>(b + o); o += map;
  w.slot_ctr = reinterpret_cast<int*>(b + o); o += ctr;
  w.cnt_n = reinterpret_cast<int*>(b + o); o += cn;
  w.cnt_m = reinterpret_cast<int*>(b + o); o += cm;
  w.map_bytes = map;
  w.zero_bytes = ctr + cn + cm;
  w.total = o;
  return w;
}

// CTA pairs (cta_group::2) for the logit-tile kernel unless CCE_PAIR=0; only for plain tile loads.
bool use_pairs() {
  static int v = [] {
    const char* e = getenv("CCE_PAIR");
    return e ? atoi(e) : 1;
  }();
  return v != 0 && num_sms() >= 2;
}

// Raster of the full-sweep logit-tile kernel (FWD / BWD): units (token tile or pair, vocab split)
// in bands of `band` token tiles, split-major inside a band.
//   * E fits the L2 budget (<= 40 MB of E tiles: Gemma-2-2B, GPT-2): one band, splits chosen so
//     the units balance over the whole grid.
//   * Larger heads: the grid shrinks to exactly band x splits CTAs (pairs), so every round of the
//     static schedule is one whole band -- the CTAs running together then read `band` E tiles and
//     `splits` C tiles, all L2-resident.  With a full grid, rounds drift across band boundaries
//     and the working set doubles: at Mistral-NeMo the forward read 281 GB from DRAM (210x C) at
//     1.0 GHz under the power cap (profiles/r2/ncu_fwd_large_heads.md).
struct Raster {
  int band;    // token tiles per band
  int splits;  // vocab splits
  int cap;     // CTAs (pairs) per round; 0 = the whole grid
};

Raster lse_raster(int nt, int mt, int64_t d, bool pair, bool prefer_fine) {
  const int cg = pair ? 2 : 1;
  const int grid = num_sms() / cg;
  const int units_n = (nt + cg - 1) / cg;
  const int64_t e_unit = (int64_t)cce::BM * d * 2 * cg;  // E bytes of one unit's token rows
  const int bmax = (int)std::max<int64_t>(1, (40ll << 20) / e_unit);
  if (units_n <= bmax || units_n < grid) {
    const int band = std::min(units_n, bmax);
    return Raster{band * cg, clamp_splits(choose_splits(units_n, mt, grid, prefer_fine), units_n, mt, band, grid), 0};
  }
  int bb = 1, bs = std::min(mt, grid);
  for (int b = 1; b <= bmax; ++b) {
    const int sp = std::min(mt, grid / b);
    if (sp < 1) break;
    if (b * sp > bb * bs || (b * sp == bb * bs && b > bb)) {
      bb = b;
      bs = sp;
    }
  }
  return Raster{bb * cg, bs, bb * bs};
}

int lse_splits(int nt, int mt, int64_t d, bool pair, bool prefer_fine) {
  return lse_raster(nt, mt, d, pair, prefer_fine).splits;
}

void set_raster(cce::Params& p, int nt, int mt, int64_t d, bool pair, bool prefer_fine) {
  const Raster r = lse_raster(nt, mt, d, pair, prefer_fine);
  p.band = r.band;
  p.splits = r.splits;
  p.grid_cap = r.cap;
}

using LseKernel = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, cce::Params);
template <int MODE, int CG>
LseKernel sync_kernel() {
  if constexpr (MODE == cce::FWD)
    return cce::cce_lse_sync_kernel<cce::FWD, CG>;
  else
    return nullptr;
}

// Launch cce_lse_kernel<MODE> on single CTAs or on CTA pairs (cluster of 2).
template <int MODE>
int launch_lse(const cce::Params& p, bool pair, const CUtensorMap& tmE, const CUtensorMap& tmEg,
               const CUtensorMap& tmC256, const CUtensorMap& tmCg, const CUtensorMap& tmC128,
               cudaStream_t stream) {
  const int cap = (MODE != cce::KEPT && p.grid_cap > 0) ? p.grid_cap : (1 << 30);
  // a launch of the forward's group chain (Params::sync_*): the 224-thread kernel with a gather warp
  const bool sync = MODE == cce::FWD && (p.sync_exit != nullptr || p.g_dst != nullptr);
  // (the 224-thread kernel exists for FWD only)
  constexpr int SMODE = MODE == cce::FWD ? cce::FWD : -1;
  if (!pair) {
    auto k = sync ? sync_kernel<SMODE, 1>() : cce::cce_lse_kernel<MODE, 1>;
    if (int e = ensure_attr(k, kLseSmem)) return e;
    const int units = p.nt * p.splits;
    return launch_k(k, dim3(std::max(1, std::min({num_sms(), units, cap}))),
                    dim3(sync ? cce::SYNC_THREADS : cce::NUM_THREADS), kLseSmem, stream, 1, tmE, tmEg, tmC256, tmCg, p);
  }
  auto k = sync ? sync_kernel<SMODE, 2>() : cce::cce_lse_kernel<MODE, 2>;
  if (int e = ensure_attr(k, kLsePairSmem)) return e;
  const int pair_units = ((p.nt + 1) / 2) * p.splits;
  const int grid = 2 * std::max(1, std::min({num_sms() / 2, pair_units, cap}));
  return launch_k(k, dim3(grid), dim3(sync ? cce::SYNC_THREADS : cce::NUM_THREADS), kLsePairSmem, stream, 2,
                  tmE, tmEg, tmC128, tmCg, p);
}

struct KeptWs {
  uint8_t* keep;
  int2* alist;     // all kept tiles, vocab-tile-major: (token tile, slot)
  int2* rlist;     // tiles to recompute: (token tile, vocab tile)
  int2* pairs;
  int* pair_count;
  int32_t* slot_of;
  uint8_t* block_zero;
  int* list_count;
  int* rlist_count;
  int* ok;
  int* cnt_n;
  int* cnt_m;
  int* rcnt_m;
  int* off_m;
  int* roff_m;
  size_t keep_bytes, slot_bytes, cnt_bytes;
  size_t total;
};

// capacity = S-hat slots for recomputed tiles; lab_capacity = stored label-tile slots
KeptWs kept_layout(void* base, int64_t n, int64_t v, int64_t capacity, int64_t lab_capacity) {
  const int64_t mt = (v + cce::BN - 1) / cce::BN;
  const int64_t nt = (n + cce::BM - 1) / cce::BM;
  auto up = [](size_t x) { return (x + 1023) & ~size_t(1023); };
  uint8_t* b = static_cast<uint8_t*>(base);
  KeptWs w;
  size_t o = 0;
  w.keep_bytes = up((size_t)nt * mt);
  w.keep = b + o; o += w.keep_bytes;
  w.alist = reinterpret_cast<int2*>(b + o); o += up((size_t)(capacity + lab_capacity) * sizeof(int2));
  // recompute list / pairs: the fallback passes use the whole S-hat buffer (both regions)
  w.rlist = reinterpret_cast<int2*>(b + o); o += up((size_t)(capacity + lab_capacity) * sizeof(int2));
  w.pairs = reinterpret_cast<int2*>(b + o); o += up((size_t)(capacity + lab_capacity) * sizeof(int2));
  w.slot_bytes = up((size_t)nt * mt * 4);
  w.slot_of = reinterpret_cast<int32_t*>(b + o); o += w.slot_bytes;
  w.block_zero = b + o; o += up((size_t)nt);
  w.cnt_bytes = up(256 + (size_t)(nt + 4 * mt) * 4);
  w.list_count = reinterpret_cast<int*>(b + o);
  w.ok = w.list_count + 1;
  w.pair_count = w.list_count + 2;
  // list_count + 3: dE unit counter
  w.rlist_count = w.list_count + 4;
  w.cnt_n = reinterpret_cast<int*>(b + o + 256);
  w.cnt_m = w.cnt_n + nt;
  w.rcnt_m = w.cnt_m + mt;
  w.off_m = w.rcnt_m + mt;
  w.roff_m = w.off_m + mt;
  o += w.cnt_bytes;
  w.total = o;
  return w;
}
// dE pass (B2).  Variant knobs (CCE_DE="<chunks per unit>,<order>,<dynamic>,<prefetch>,<kv>"):
// default 1,0,0,0,64 = two double-buffered 256-column accumulators, chunk-major units, static
// round-robin, no L2 prefetch, 64 vocab rows per stage.  Builds its own S-hat / C tensor maps.
template <int CH, int KV>
int launch_de_t(const cce::GradParams& q, int units, const void* shat, int64_t shat_rows, const void* C,
                int64_t v, int64_t d, const CUtensorMap& tmCg, cudaStream_t stream) {
  CUtensorMap tmS, tmC3, tmC;
  const bool ok = make_tmap3d_inner(&tmS, shat, shat_rows, cce::BN, KV, cce::BM, 1) &&
                  make_tmap(&tmC, C, v, d, KV) &&
                  (d % 64 == 0 ? make_tmap3d(&tmC3, C, v, d, KV, cce::DCH / 64) : (tmC3 = tmC, true));
  if (!ok) return fail("cce_de: cuTensorMapEncodeTiled failed");
  if (int e = ensure_attr(cce::cce_de_kernel<CH, KV>, de_smem<CH, KV>())) return e;
  int grid = std::max(1, std::min(num_sms(), units));
  if (q.de_order >= 2 && q.sched == nullptr && grid >= q.de_order) grid -= grid % q.de_order;
  return launch_k(cce::cce_de_kernel<CH, KV>, dim3(grid), dim3(cce::NUM_THREADS), de_smem<CH, KV>(), stream, 1,
                  tmS, tmC, tmC3, tmCg, q);
}

int launch_de(cce::GradParams q, int* sched_ctr, const void* shat, int64_t shat_rows, const void* C,
              const CUtensorMap& tmCg, cudaStream_t stream) {
  static int cfg[5] = {-1, 0, 0, 0, 64};
  static bool fixed = false;
  if (cfg[0] < 0) {
    cfg[0] = 1;
    if (const char* e = getenv("CCE_DE")) {
      sscanf(e, "%d,%d,%d,%d,%d", &cfg[0], &cfg[1], &cfg[2], &cfg[3], &cfg[4]);
      fixed = true;
    }
  }
  int ch = cfg[0] == 2 ? 2 : 1;
  int kv = cfg[4];
  if (!fixed) {
    // measured (profiles/r1/de_variants_s46*, ab/ab_de_ch2_threshold.txt): one 512-column
    // accumulator fed by 32-row stages (less operand traffic per flop) wins once there are
    // enough units to balance the grid (Gemma-2-9B: 11.5 vs 13.1 ms; Llama-3-8B, 1024 units:
    // 11.1 vs 12.0 ms); with few units (Gemma-2-2B: 320) the double-buffered 256-column form
    // wins (1.65 vs 2.05 ms)
    const int units512 = q.g * ((q.ndc + 1) / 2);
    if (units512 >= 6 * num_sms()) {
      ch = 2;
      kv = 32;
    } else {
      ch = 1;
      kv = 64;
    }
  }
  kv = (kv == 32 && q.perm == nullptr) ? 32 : 64;  // row gathers need 64-wide boxes
  q.de_order = cfg[1];
  q.sched = cfg[2] ? sched_ctr : nullptr;
  q.prefetch = cfg[3];
  const int units = q.g * ((q.ndc + ch - 1) / ch);
  if (ch == 2)
    return kv == 32 ? launch_de_t<2, 32>(q, units, shat, shat_rows, C, q.v, q.d, tmCg, stream)
                    : launch_de_t<2, 64>(q, units, shat, shat_rows, C, q.v, q.d, tmCg, stream);
  return kv == 32 ? launch_de_t<1, 32>(q, units, shat, shat_rows, C, q.v, q.d, tmCg, stream)
                  : launch_de_t<1, 64>(q, units, shat, shat_rows, C, q.v, q.d, tmCg, stream);
}

// dC pass (B3) on single CTAs or CTA pairs (the pair needs the 3-D E map with 2-atom boxes).
int launch_dc(cce::GradParams q, bool pair, const CUtensorMap& tmS64, const CUtensorMap& tmE64,
              const CUtensorMap& tmE3, const CUtensorMap& tmE3h, const CUtensorMap& tmEg,
              cudaStream_t stream) {
  const int units = q.mt * q.ndc * 2;
  {
    const char* e = getenv("CCE_DC_BLOCK");
    q.dc_block = e ? atoi(e) : 0;
  }
  if (!pair) {
    if (int e = ensure_attr(cce::cce_dc_kernel<1>, kDcSmem)) return e;
    return launch_k(cce::cce_dc_kernel<1>, dim3(std::min(num_sms(), units)), dim3(cce::NUM_THREADS), kDcSmem,
                    stream, 1, tmS64, tmE64, tmE3, tmEg, q);
  }
  if (int e = ensure_attr(cce::cce_dc_kernel<2>, kDcSmem)) return e;
  return launch_k(cce::cce_dc_kernel<2>, dim3(2 * std::max(1, std::min(num_sms() / 2, units / 2))),
                  dim3(cce::NUM_THREADS), kDcSmem, stream, 2, tmS64, tmE64, tmE3h, tmE64, q);
}

}  // namespace

extern "C" {

const char* cce_last_error(void) { return g_last_error.c_str(); }

int cce_abi_version(void) { return 1; }

unsigned long long cce_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

size_t cce_fwd_workspace_bytes(int64_t n, int64_t d, int64_t v) {
  const int nt = (int)((n + cce::BM - 1) / cce::BM);
  const int mt = (int)((v + cce::BN - 1) / cce::BN);
  const int s = lse_splits(nt, mt, d, use_pairs(), false);
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
  const bool pair = use_pairs();
  const int splits = lse_splits(nt, mt, d, pair, false);
  if (ws_bytes < (size_t)splits * n * sizeof(float2)) return fail("cce_fwd: workspace too small");
  CUtensorMap tmE, tmC, tmC128;
  if (!make_tmap(&tmE, E, n, d, cce::BM) || !make_tmap(&tmC, C, v, d, cce::BN) ||
      !make_tmap(&tmC128, C, v, d, cce::BN / 2))
    return fail("cce_fwd: cuTensorMapEncodeTiled failed");
  (void)grid;
  cce::Params p{};
  p.n_total = (int)n;
  p.d = (int)d;
  p.v = (int)v;
  p.nt = nt;
  p.n_base = 0;
  p.mt = mt;
  set_raster(p, nt, mt, d, pair, false);
  p.num_kb = (int)((d + cce::BK - 1) / cce::BK);
  p.softcap = softcap;
  p.targets = targets;
  p.ignore_index = ignore_index;
  p.vocab_start = vocab_start;
  p.part = static_cast<float2*>(ws);
  p.correct = correct;
  const int units = nt * splits;
  PDL_LAUNCH(cce::fill_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, stream, correct, 0.f, n);
  (void)units;
  if (int e = launch_lse<cce::FWD>(p, pair, tmE, tmE, tmC, tmC, tmC128, stream)) return e;
  PDL_LAUNCH(cce::combine_splits_kernel, dim3((unsigned)((n + cce::COMBINE_ROWS - 1) / cce::COMBINE_ROWS)),
             dim3(cce::COMBINE_ROWS * cce::COMBINE_GROUPS), 0, stream, static_cast<const float2*>(ws), splits, (int)n, lse_local,
             (float2*)nullptr);
  CCE_CUDA(cudaGetLastError());
  return 0;
}

int cce_merge_shards_checked(int num_shards, const float* lse_parts, const float* correct_parts,
                             const int64_t* targets, int64_t ignore_index, int64_t n, int64_t v_total,
                             int* label_error, float* lse_out, float* loss_out, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (n == 0) return 0;
  PDL_LAUNCH(cce::merge_shards_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, stream, num_shards,
             lse_parts, correct_parts, targets, ignore_index, (int)n, lse_out, loss_out, v_total, label_error);
  CCE_CUDA(cudaGetLastError());
  return 0;
}

int cce_merge_shards(int num_shards, const float* lse_parts, const float* correct_parts,
                     const int64_t* targets, int64_t ignore_index, int64_t n, float* lse_out,
                     float* loss_out, void* stream_ptr) {
  return cce_merge_shards_checked(num_shards, lse_parts, correct_parts, targets, ignore_index, n, 0, nullptr,
                                  lse_out, loss_out, stream_ptr);
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
static int ebar_rows_per_block(int64_t n) { return (int)std::max<int64_t>(64, (n + 255) / 256); }

size_t cce_ebar_workspace_bytes(int64_t n, int64_t d) {
  if (n <= 0) return 0;
  const int64_t nblk = (n + ebar_rows_per_block(n) - 1) / ebar_rows_per_block(n);
  return (size_t)(nblk * d) * sizeof(float);
}

int cce_ebar(const void* E, const int64_t* targets, int64_t ignore_index, int64_t n, int64_t d,
             float* ebar_sum, void* ws, size_t ws_bytes, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (n == 0) {
    CCE_CUDA(cudaMemsetAsync(ebar_sum, 0, d * sizeof(float), stream));
    return 0;
  }
  if (ws_bytes < cce_ebar_workspace_bytes(n, d)) return fail("cce_ebar: workspace too small");
  // fixed-order two-pass sum (bit-reproducible): per-block partials, then an ordered reduction
  const int rows_per_block = ebar_rows_per_block(n);
  const int nblk = (int)((n + rows_per_block - 1) / rows_per_block);
  float* part = static_cast<float*>(ws);
  dim3 grid((unsigned)((d + 127) / 128), (unsigned)nblk);
  PDL_LAUNCH(cce::ebar_kernel, dim3(grid), dim3(128), 0, stream, static_cast<const __nv_bfloat16*>(E), targets,
                                             ignore_index, (int)n, (int)d, part, rows_per_block);
  CCE_CUDA(cudaGetLastError());
  PDL_LAUNCH(cce::ebar_reduce_kernel, dim3((unsigned)((d + 127) / 128)), dim3(128), 0, stream, part, nblk, (int)d, ebar_sum);
  CCE_CUDA(cudaGetLastError());
  return 0;
}

int cce_vocab_order(const void* C, const float* ebar_sum, const int* n_valid, int64_t v, int64_t d,
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
  CCE_CUDA(cudaFuncSetAttribute(cce::sort_key_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(d * sizeof(float))));
  PDL_LAUNCH(cce::sort_key_kernel, dim3((unsigned)std::min<int64_t>((v + 7) / 8, CCE_SORTKEY_BPS * num_sms())), dim3(256), d * sizeof(float), stream, static_cast<const __nv_bfloat16*>(C), ebar_sum, n_valid, (int)v, (int)d, key);
  CCE_CUDA(cudaGetLastError());
  PDL_LAUNCH(cce::iota_kernel, dim3((unsigned)((v + 255) / 256)), dim3(256), 0, stream, idx, (int)v);
  CCE_CUDA(cudaGetLastError());
  CCE_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, tmp_bytes, key, key_sorted, idx, perm,
                                                     (int)v, 0, 32, stream));
  if (key_out) CCE_CUDA(cudaMemcpyAsync(key_out, key, v * 4, cudaMemcpyDeviceToDevice, stream));
  return 0;
}

// Backward prep: padded perm / inverse perm, label positions, zero-upstream tile flags.
int cce_compact_rows(const int64_t* targets, int64_t ignore_index, int64_t n, int32_t* row_map,
                     int* n_valid, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  const int64_t npad = ((n + cce::BM - 1) / cce::BM) * cce::BM;
  CCE_CUDA(cudaMemsetAsync(row_map, 0, std::max<int64_t>(npad, 1) * sizeof(int32_t), stream));
  PDL_LAUNCH(cce::compact_rows_kernel, dim3(1), dim3(1024), 0, stream, targets, ignore_index, (int)n, row_map, n_valid);
  CCE_CUDA(cudaGetLastError());
  return 0;
}

int cce_bwd_prep(const int32_t* perm, int64_t v, const int64_t* targets, int64_t ignore_index,
                 int64_t vocab_start, int64_t n, int32_t* perm_padded, int32_t* inv_perm, int32_t* pos,
                 void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  const int64_t vpad = ((v + cce::BN - 1) / cce::BN) * cce::BN;
  if (perm) {
    PDL_LAUNCH(cce::invert_perm_kernel, dim3((unsigned)((vpad + 255) / 256)), dim3(256), 0, stream, perm, (int)v, (int)vpad, perm_padded, inv_perm);
    CCE_CUDA(cudaGetLastError());
  }
  if (n > 0) {
    PDL_LAUNCH(cce::label_pos_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, stream, targets, ignore_index, vocab_start, (int)v, perm ? inv_perm : nullptr, (int)n, pos);
    CCE_CUDA(cudaGetLastError());
  }
  return 0;
}

size_t cce_bwd_workspace_bytes(int64_t n, int64_t d, int64_t v, int64_t group_tiles,
                               int64_t capacity_tiles) {
  return bwd_layout(nullptr, n, d, v, group_tiles, capacity_tiles).total;
}

// Filtered backward (lse_backward).  See include/cce_b200.h.
int cce_bwd(const void* E, const void* C, const int32_t* perm_padded, int c_sorted,
            const int32_t* row_map, const int* n_valid, const int32_t* pos, const float* lse,
            const float* upstream, int64_t n, int64_t d, int64_t v, float softcap, float eps,
            int64_t group_tiles, int64_t capacity_tiles, const int* run_if, int e_gather, void* ws,
            size_t ws_bytes, void* de_out, int de_fp32, void* dc, unsigned long long* counters,
            int* overflow, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (d % 8 != 0) return fail("cce_bwd: D must be a multiple of 8");
  if (n <= 0) return 0;
  if (group_tiles < 1 || capacity_tiles < 1) return fail("cce_bwd: group_tiles / capacity_tiles must be >= 1");
  const BwdWs w = bwd_layout(ws, n, d, v, group_tiles, capacity_tiles);
  if (ws_bytes < w.total) return fail("cce_bwd: workspace too small");
  const int nt = (int)((n + cce::BM - 1) / cce::BM);
  const int mt = (int)((v + cce::BN - 1) / cce::BN);
  const int ndc = (int)((d + cce::DCH - 1) / cce::DCH);
  const int grid = num_sms();
  const int gbox = gather_box_rows();
  // compact E (filter_ignored) unless rows are gathered on the fly; zero-upstream tile flags
  const void* e_src = E;
  if (!e_gather) {
    PDL_LAUNCH(cce::gather_rows_kernel, dim3((unsigned)((n + 7) / 8)), dim3(256), 0, stream, static_cast<const __nv_bfloat16*>(E), row_map, n, (int)d, w.e_compact);
    CCE_CUDA(cudaGetLastError());
    e_src = w.e_compact;
  }
  PDL_LAUNCH(cce::block_zero_kernel, dim3(nt), dim3(cce::BM), 0, stream, upstream, row_map, n_valid, w.block_zero);
  CCE_CUDA(cudaGetLastError());
  CUtensorMap tmE, tmEg, tmC, tmCg, tmC128, tmE64, tmS128, tmS64, tmC3, tmE3, tmE3h, tmC128h, tmC64;
  const int64_t shat_rows = capacity_tiles * cce::BM;
  const bool atoms3d = d % 64 == 0;
  bool ok = make_tmap(&tmE, e_src, n, d, cce::BM) && make_tmap(&tmEg, E, n, d, gbox) &&
            make_tmap(&tmC, C, v, d, cce::BN) && make_tmap(&tmCg, C, v, d, gbox) &&
            make_tmap(&tmC128, C, v, d, 128) && make_tmap(&tmE64, e_src, n, d, 64) &&
            make_tmap(&tmC128h, C, v, d, cce::BN / 2) && make_tmap(&tmC64, C, v, d, cce::DE_KV) &&
            make_tmap3d(&tmS128, w.shat, shat_rows, cce::BN, 128, 1) &&
            make_tmap3d(&tmS64, w.shat, shat_rows, cce::BN, 64, 2);
  if (ok && atoms3d)
    ok = make_tmap3d(&tmC3, C, v, d, cce::DE_KV, cce::DCH / 64) && make_tmap3d(&tmE3, e_src, n, d, 64, cce::DCH / 64) &&
         make_tmap3d(&tmE3h, e_src, n, d, 64, cce::DCH / 128);
  else {
    tmC3 = tmC64;
    tmE3 = tmE64;
    tmE3h = tmE64;
  }
  if (!ok) return fail("cce_bwd: cuTensorMapEncodeTiled failed");
  const bool dc_pair = use_pairs() && atoms3d && !e_gather;
  for (int g0 = 0; g0 < nt; g0 += (int)group_tiles) {
    const int g = std::min((int)group_tiles, nt - g0);
    CCE_CUDA(cudaMemsetAsync(w.slot_of, 0xFF, w.map_bytes, stream));
    CCE_CUDA(cudaMemsetAsync(w.slot_ctr, 0, w.zero_bytes, stream));
    cce::Params p{};
    p.n_total = (int)n;
    p.n_valid = n_valid;
    p.run_if = run_if;
    p.d = (int)d;
    p.v = (int)v;
    p.nt = g;
    p.n_base = g0;
    p.mt = mt;
    const bool pair = use_pairs();
    set_raster(p, g, mt, d, pair, true);
    p.num_kb = (int)((d + cce::BK - 1) / cce::BK);
    p.softcap = softcap;
    p.lse = lse;
    p.upstream = upstream;
    p.pos = pos;
    p.perm = c_sorted ? nullptr : perm_padded;
    p.row_map = row_map;
    p.e_gather = e_gather;
    p.e_rows = static_cast<const __nv_bfloat16*>(E);
    p.c_rows = static_cast<const __nv_bfloat16*>(C);
    p.block_zero = w.block_zero;
    p.eps = eps;
    p.shat = w.shat;
    p.slot_of = w.slot_of;
    p.slot_ctr = w.slot_ctr;
    p.capacity = (int)capacity_tiles;
    p.overflow = overflow;
    p.cnt_n = w.cnt_n;
    p.cnt_m = w.cnt_m;
    p.counters = counters;
    if (int e = launch_lse<cce::BWD>(p, pair, tmE, tmEg, tmC, tmCg, tmC128h, stream)) return e;
    cce::GradParams q{};
    q.n_total = (int)n;
    q.n_valid = n_valid;
    q.run_if = run_if;
    q.d = (int)d;
    q.v = (int)v;
    q.mt = mt;
    q.ndc = ndc;
    q.n_base = g0;
    q.g = g;
    q.slot_of = w.slot_of;
    q.cnt_n = w.cnt_n;
    q.cnt_m = w.cnt_m;
    q.perm = c_sorted ? nullptr : perm_padded;
    q.perm_store = perm_padded;
    q.row_map = row_map;
    q.e_gather = e_gather;
    q.atoms3d = atoms3d ? 1 : 0;
    q.de_bf16 = de_fp32 ? nullptr : static_cast<__nv_bfloat16*>(de_out);
    q.de_f32 = de_fp32 ? static_cast<float*>(de_out) : nullptr;
    q.dc = static_cast<__nv_bfloat16*>(dc);
    q.accumulate = g0 > 0;
    {
      const char* dbg = getenv("CCE_DEBUG_GRAD");
      q.debug = dbg ? atoi(dbg) : 0;
    }
    if (int e = launch_de(q, w.slot_ctr + 1, w.shat, shat_rows, C, tmCg, stream)) return e;  // counter zeroed per group
    if (int e = launch_dc(q, dc_pair, tmS64, tmE64, tmE3, tmE3h, tmEg, stream)) return e;
  }
  return 0;
}

// ---- filter from the forward: forward in tile order with tile maxima, backward on kept tiles ----

size_t cce_tile_max_bytes(int64_t n, int64_t v) {
  const int64_t nt = (n + cce::BM - 1) / cce::BM;
  const int64_t mt = (v + cce::BN - 1) / cce::BN;
  return (size_t)(nt * mt * cce::BM) * sizeof(float);
}

}  // extern "C"

namespace {
// Forward over the backward's tile order (see cce_fwd_tiles / cce_fwd_gather in the header):
// E_rows / C_rows are either the compacted / sorted copies (perm_padded == NULL, gather_e = 0) or
// the caller's E and C read through row_map / perm_padded with cp.async row gathers.
int fwd_tiles_impl(const char* what, const void* E_rows, const void* C_rows, const int32_t* perm_padded,
                   int gather_e, const int32_t* row_map, const int* n_valid, const int32_t* pos,
                   int64_t pos_offset, int64_t n, int64_t d, int64_t v, float softcap, void* ws, size_t ws_bytes,
                   float* lse_local, float* correct, float* tile_max, void* lab_buf, int64_t lab_capacity,
                   int32_t* lab_slot, void* lab_list, int* lab_count, cudaStream_t stream, int tm_stride = 0,
                   int tm_m0 = 0, int flags = 0, const cce::Params* sync = nullptr) {
  const std::string w(what);
  if (n < 0 || d <= 0 || v <= 0) return fail(w + ": bad sizes");
  if (lab_buf && (!lab_slot || !lab_list || !lab_count)) return fail(w + ": label tiles need slot maps");
  if (d % 8 != 0) return fail(w + ": D must be a multiple of 8 (16-byte TMA row pitch)");
  if (!row_map || !n_valid || !pos || !tile_max) return fail(w + ": row_map, n_valid, pos, tile_max required");
  if (n == 0) return 0;
  const int nt = (int)((n + cce::BM - 1) / cce::BM);
  const int mt = (int)((v + cce::BN - 1) / cce::BN);
  const bool pair = use_pairs();
  const int splits = lse_splits(nt, mt, d, pair, false);
  if (ws_bytes < (size_t)splits * n * sizeof(float2)) return fail(w + ": workspace too small");
  CUtensorMap tmE, tmC, tmC128;
  if (!make_tmap(&tmE, E_rows, n, d, cce::BM) || !make_tmap(&tmC, C_rows, v, d, cce::BN) ||
      !make_tmap(&tmC128, C_rows, v, d, cce::BN / 2))
    return fail(w + ": cuTensorMapEncodeTiled failed");
  cce::Params p{};
  p.n_total = (int)n;
  p.n_valid = n_valid;
  p.d = (int)d;
  p.v = (int)v;
  p.nt = nt;
  p.n_base = 0;
  p.mt = mt;
  set_raster(p, nt, mt, d, pair, false);
  p.num_kb = (int)((d + cce::BK - 1) / cce::BK);
  p.softcap = softcap;
  p.pos = pos;
  p.pos_offset = (int)pos_offset;
  p.row_map = row_map;
  p.perm = perm_padded;
  p.e_gather = gather_e;
  p.e_rows = static_cast<const __nv_bfloat16*>(E_rows);
  p.c_rows = static_cast<const __nv_bfloat16*>(C_rows);
  p.part = static_cast<float2*>(ws);
  p.correct = correct;
  p.tile_max = tile_max;
  p.tm_stride = tm_stride;
  p.tm_m0 = tm_m0;
  if (sync) {  // the forward's group chain (cce_fwd_group_sync)
    p.sync_ready = sync->sync_ready;
    p.sync_exit = sync->sync_exit;
    p.sync_released = sync->sync_released;
    p.no_dep_wait = sync->no_dep_wait;
    p.g_perm = sync->g_perm;
    p.g_src = sync->g_src;
    p.g_dst = sync->g_dst;
    p.g_rows = sync->g_rows;
    p.g_wait = sync->g_wait;
    p.g_ctr = sync->g_ctr;
    p.g_done = sync->g_done;
  }
  if (lab_buf) {
    CCE_CUDA(cudaMemsetAsync(lab_slot, 0xFF, (size_t)nt * mt * sizeof(int32_t), stream));
    CCE_CUDA(cudaMemsetAsync(lab_count, 0, sizeof(int), stream));
    p.lab_buf = static_cast<__half*>(lab_buf);
    p.lab_capacity = (int)lab_capacity;
    p.lab_count = lab_count;
    p.lab_slot = lab_slot;
    p.lab_list = static_cast<int2*>(lab_list);
  }
  // flags (vocabulary groups of one sweep): bit 0 = `correct` already zeroed by the caller (the
  // target logit lands in exactly one group), bit 1 = leave the (max, sum-exp) partials in ws for
  // one combine over every group (cce_combine_parts) instead of finishing lse_local here
  if (!(flags & 1))
    PDL_LAUNCH(cce::fill_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, stream, correct, 0.f, n);
  if (int e = launch_lse<cce::FWD>(p, pair, tmE, tmE, tmC, tmC, tmC128, stream)) return e;
  if (!(flags & 2))
    PDL_LAUNCH(cce::combine_splits_kernel, dim3((unsigned)((n + cce::COMBINE_ROWS - 1) / cce::COMBINE_ROWS)),
             dim3(cce::COMBINE_ROWS * cce::COMBINE_GROUPS), 0, stream,
               static_cast<const float2*>(ws), splits, (int)n, lse_local,
             (float2*)nullptr);
  CCE_CUDA(cudaGetLastError());
  return 0;
}
}  // namespace

extern "C" {

int cce_fwd_tiles(const void* E_c, const void* C_t, const int32_t* row_map, const int* n_valid,
                  const int32_t* pos, int64_t pos_offset, int64_t n, int64_t d, int64_t v, float softcap, void* ws,
                  size_t ws_bytes, float* lse_local, float* correct, float* tile_max, void* lab_buf,
                  int64_t lab_capacity, int32_t* lab_slot, void* lab_list, int* lab_count, void* stream_ptr) {
  return fwd_tiles_impl("cce_fwd_tiles", E_c, C_t, nullptr, 0, row_map, n_valid, pos, pos_offset, n, d, v, softcap,
                        ws, ws_bytes, lse_local, correct, tile_max, lab_buf, lab_capacity, lab_slot, lab_list,
                        lab_count, static_cast<cudaStream_t>(stream_ptr));
}

int cce_fwd_gather(const void* E, const void* C, const int32_t* perm_padded, const int32_t* row_map,
                   const int* n_valid, const int32_t* pos, int64_t pos_offset, int64_t n, int64_t d, int64_t v,
                   float softcap, void* ws, size_t ws_bytes, float* lse_local, float* correct, float* tile_max,
                   void* stream_ptr) {
  return fwd_tiles_impl("cce_fwd_gather", E, C, perm_padded, 1, row_map, n_valid, pos, pos_offset, n, d, v,
                        softcap, ws, ws_bytes, lse_local, correct, tile_max, nullptr, 0, nullptr, nullptr, nullptr,
                        static_cast<cudaStream_t>(stream_ptr));
}


int cce_fwd_splits(int64_t n, int64_t d, int64_t v) {
  if (n <= 0 || v <= 0) return 1;
  const int nt = (int)((n + cce::BM - 1) / cce::BM);
  const int mt = (int)((v + cce::BN - 1) / cce::BN);
  return lse_splits(nt, mt, d, use_pairs(), false);
}

int cce_combine_parts(const void* parts, int count, int64_t n, float* lse_out, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (n <= 0) return 0;
  // reads partials written several launches back: without programmatic dependent launch (see
  // unpermute_rows)
  PdlScope pdl_scope(false);
  // lse_out == nullptr: fold into the first partial (parts[0]) instead
  PDL_LAUNCH(cce::combine_splits_kernel, dim3((unsigned)((n + cce::COMBINE_ROWS - 1) / cce::COMBINE_ROWS)),
             dim3(cce::COMBINE_ROWS * cce::COMBINE_GROUPS), 0, stream,
             static_cast<const float2*>(parts), count, (int)n, lse_out,
             lse_out ? nullptr : static_cast<float2*>(const_cast<void*>(parts)));
  CCE_CUDA(cudaGetLastError());
  return 0;
}

int cce_fwd_group_ex(const void* E, int e_gather, const void* C_g, const int32_t* row_map, const int* n_valid,
                     const int32_t* pos, int64_t v0, int64_t n, int64_t d, int64_t v_group, int64_t v_total,
                     float softcap, void* ws, size_t ws_bytes, float* lse_part, float* correct_part, float* tile_max,
                     int flags, void* stream_ptr) {
  if (v0 % cce::BN != 0) return fail("cce_fwd_group: v0 must be a multiple of 256");
  if (v0 + v_group > v_total) return fail("cce_fwd_group: group past the vocabulary");
  return fwd_tiles_impl("cce_fwd_group", E, C_g, nullptr, e_gather, row_map, n_valid, pos, v0, n, d, v_group, softcap,
                        ws, ws_bytes, lse_part, correct_part, tile_max, nullptr, 0, nullptr, nullptr, nullptr,
                        static_cast<cudaStream_t>(stream_ptr), (int)((v_total + cce::BN - 1) / cce::BN),
                        (int)(v0 / cce::BN), flags);
}

// One launch of the bounded forward's group chain: cce_fwd_group_ex over group g (C_g: its buffer)
// with no wait on the previous launch (no_dep_wait) but on *ready (its rows gathered; nullptr: the
// stream orders it), counting this launch's exited CTAs in *exit_ctr (the last sets *released = 1),
// and, in the same launch, gathering the next group's rows C[next_perm[r]], r < next_rows, into
// next_dst once *next_wait >= 1 (the launch before this one exited; nullptr: at once), counted
// in *next_ctr (the last share sets *next_done = 1).  next_dst == nullptr: nothing to gather.
int cce_fwd_group_sync(const void* E, int e_gather, const void* C_g, const int32_t* row_map, const int* n_valid,
                       const int32_t* pos, int64_t v0, int64_t n, int64_t d, int64_t v_group, int64_t v_total,
                       float softcap, void* ws, size_t ws_bytes, float* correct_part, float* tile_max,
                       const int* ready, int* exit_ctr, int* released, int no_dep_wait, const void* C,
                       const int32_t* next_perm, int64_t next_rows, void* next_dst, const int* next_wait,
                       int* next_ctr, int* next_done, void* stream_ptr) {
  if (v0 % cce::BN != 0) return fail("cce_fwd_group_sync: v0 must be a multiple of 256");
  if (v0 + v_group > v_total) return fail("cce_fwd_group_sync: group past the vocabulary");
  if (!exit_ctr || !released) return fail("cce_fwd_group_sync: exit counter and released flag required");
  if (next_dst && (!C || !next_perm || !next_ctr || !next_done))
    return fail("cce_fwd_group_sync: a gather needs C, next_perm, next_ctr and next_done");
  cce::Params sp{};
  sp.sync_ready = ready;
  sp.sync_exit = exit_ctr;
  sp.sync_released = released;
  sp.no_dep_wait = no_dep_wait ? 1 : 0;
  sp.g_perm = next_perm;
  sp.g_src = static_cast<const __nv_bfloat16*>(C);
  sp.g_dst = static_cast<__nv_bfloat16*>(next_dst);
  sp.g_rows = next_dst ? (int)next_rows : 0;
  sp.g_wait = next_wait;
  sp.g_ctr = next_ctr;
  sp.g_done = next_done;
  PdlScope pdl(true);
  return fwd_tiles_impl("cce_fwd_group_sync", E, C_g, nullptr, e_gather, row_map, n_valid, pos, v0, n, d, v_group,
                        softcap, ws, ws_bytes, nullptr, correct_part, tile_max, nullptr, 0, nullptr, nullptr, nullptr,
                        static_cast<cudaStream_t>(stream_ptr), (int)((v_total + cce::BN - 1) / cce::BN),
                        (int)(v0 / cce::BN), 3, &sp);
}

int cce_fwd_group(const void* E, int e_gather, const void* C_g, const int32_t* row_map, const int* n_valid,
                  const int32_t* pos, int64_t v0, int64_t n, int64_t d, int64_t v_group, int64_t v_total, float softcap,
                  void* ws, size_t ws_bytes, float* lse_part, float* correct_part, float* tile_max, void* stream_ptr) {
  if (v0 % cce::BN != 0) return fail("cce_fwd_group: v0 must be a multiple of 256");
  if (v0 + v_group > v_total) return fail("cce_fwd_group: group past the vocabulary");
  return fwd_tiles_impl("cce_fwd_group", E, C_g, nullptr, e_gather, row_map, n_valid, pos, v0, n, d, v_group, softcap,
                        ws, ws_bytes, lse_part, correct_part, tile_max, nullptr, 0, nullptr, nullptr, nullptr,
                        static_cast<cudaStream_t>(stream_ptr), (int)((v_total + cce::BN - 1) / cce::BN),
                        (int)(v0 / cce::BN));
}

size_t cce_bwd_kept_workspace_bytes(int64_t n, int64_t d, int64_t v, int64_t capacity_tiles,
                                    int64_t lab_capacity) {
  (void)d;
  return kept_layout(nullptr, n, v, capacity_tiles, lab_capacity).total;
}

int cce_bwd_kept(const void* E_c, const void* C_t, const void* C, const int32_t* perm_padded, const int32_t* row_map,
                 const int* n_valid, const int32_t* pos, int64_t pos_offset, const float* lse, const float* upstream,
                 const float* tile_max, int64_t n, int64_t d, int64_t v, float softcap, float eps,
                 int label_split, void* shat, int64_t lab_capacity, const int32_t* lab_slot,
                 const void* lab_list, const int* lab_count, int64_t capacity_tiles, void* ws, size_t ws_bytes,
                 void* de_out, int de_fp32, int de_accumulate, void* dc, unsigned long long* counters,
                 int* overflow, int* stats, int* kept_per_vtile, void* de_done_event, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (d % 8 != 0) return fail("cce_bwd_kept: D must be a multiple of 8");
  if (!(eps > 0.f)) return fail("cce_bwd_kept: needs filtering (eps > 0); use cce_bwd without it");
  if (!overflow || !shat) return fail("cce_bwd_kept: overflow flag and S-hat buffer required");
  // dc aliasing C_t: the fallback passes (which may follow an earlier group's dC pass) read the
  // caller's C through the permutation instead of the sorted copy
  if (de_out == nullptr && dc == nullptr) return fail("cce_bwd_kept: neither dE nor dC requested");
  const bool aliased = dc != nullptr && dc == C_t;
  if (aliased && (C == nullptr || perm_padded == nullptr))
    return fail("cce_bwd_kept: dc aliases C_t, so C and perm_padded are required");
  if (lab_slot == nullptr) lab_capacity = 0;
  if (de_accumulate && !de_fp32) return fail("cce_bwd_kept: de_accumulate needs the fp32 dE");
  if (lab_capacity > 0 && pos_offset != 0)
    return fail("cce_bwd_kept: stored label tiles are not supported over a vocabulary group (pos_offset)");
  if (n <= 0) return 0;
  const int nt = (int)((n + cce::BM - 1) / cce::BM);
  const int mt = (int)((v + cce::BN - 1) / cce::BN);
  if (capacity_tiles < std::min<int64_t>(mt, (int64_t)nt * mt))
    return fail("cce_bwd_kept: capacity_tiles must hold one token tile's vocab tiles (ceil(v/256))");
  const KeptWs w = kept_layout(ws, n, v, capacity_tiles, lab_capacity);
  if (ws_bytes < w.total) return fail("cce_bwd_kept: workspace too small");
  const int ndc = (int)((d + cce::DCH - 1) / cce::DCH);
  PDL_LAUNCH(cce::block_zero_kernel, dim3(nt), dim3(cce::BM), 0, stream, upstream, row_map, n_valid, w.block_zero);
  CCE_CUDA(cudaGetLastError());
  PDL_LAUNCH(cce::decide_tiles_kernel, dim3(dim3((unsigned)((mt + cce::DECIDE_VT - 1) / cce::DECIDE_VT), (unsigned)nt)), dim3(256), 0, stream, tile_max, lse, pos, (int)pos_offset, row_map, n_valid, w.block_zero, nt, mt, softcap, eps, label_split,
      w.keep, counters);
  CCE_CUDA(cudaGetLastError());
  // S-hat slots: [stored label tiles (lab_capacity) | recomputed tiles (capacity_tiles)]
  __nv_bfloat16* shat_all = static_cast<__nv_bfloat16*>(shat);
  __nv_bfloat16* shat_rec = shat_all + (size_t)lab_capacity * cce::BM * cce::BN;
  // Stored label tiles -> S-hat, in place.  HBM-bound and independent of the kept lists, so it
  // runs on a side stream beside the list kernels and the tensor-bound recompute pass; dE joins.
  const char* side_env = getenv("CCE_LABEL_SIDE");  // 0: same stream (A/B timing)
  SideStream* side = (lab_capacity > 0 && (!side_env || atoi(side_env) != 0)) ? side_stream() : nullptr;
  if (lab_capacity > 0) {
    cudaStream_t ls = stream;
    if (side) {
      CCE_CUDA(cudaEventRecord(side->fork, stream));
      CCE_CUDA(cudaStreamWaitEvent(side->s, side->fork, 0));
      ls = side->s;
    }
    PDL_LAUNCH(cce::label_shat_kernel, dim3((unsigned)lab_capacity), dim3(256), 0, ls, reinterpret_cast<__half*>(shat_all), static_cast<const int2*>(lab_list), lab_count, (int)lab_capacity,
        w.block_zero, mt, tile_max, lse, upstream, pos, row_map, n_valid, (int)v, softcap, label_split);
    CCE_CUDA(cudaGetLastError());
    if (side) CCE_CUDA(cudaEventRecord(side->join, side->s));
  }

  CUtensorMap tmE, tmC, tmC64, tmC128h, tmE64, tmS64, tmC3, tmE3, tmE3h;
  const int64_t shat_rows = (capacity_tiles + lab_capacity) * cce::BM;
  const bool atoms3d = d % 64 == 0;
  bool ok = make_tmap(&tmE, E_c, n, d, cce::BM) && make_tmap(&tmC, C_t, v, d, cce::BN) &&
            make_tmap(&tmC64, C_t, v, d, cce::DE_KV) && make_tmap(&tmE64, E_c, n, d, 64) &&
            make_tmap(&tmC128h, C_t, v, d, cce::BN / 2) &&
            make_tmap3d(&tmS64, shat_all, shat_rows, cce::BN, 64, 2);
  if (ok && atoms3d)
    ok = make_tmap3d(&tmC3, C_t, v, d, cce::DE_KV, cce::DCH / 64) && make_tmap3d(&tmE3, E_c, n, d, 64, cce::DCH / 64) &&
         make_tmap3d(&tmE3h, E_c, n, d, 64, cce::DCH / 128);
  else {
    tmC3 = tmC64;
    tmE3 = tmE64;
    tmE3h = tmE64;
  }
  CUtensorMap tmCo, tmCog;  // the caller's C (row gathers through perm_padded) for aliased fallbacks
  if (ok && aliased)
    ok = make_tmap(&tmCo, C, v, d, cce::BN) && make_tmap(&tmCog, C, v, d, gather_box_rows());
  if (!ok) return fail("cce_bwd_kept: cuTensorMapEncodeTiled failed");
  const bool pair = use_pairs();

  // One pass over token tiles [g0, g0 + g): kept lists, S-hat of the tiles to recompute (KEPT),
  // dE of those token tiles (complete), dC (written by the first pass, accumulated by later ones).
  auto run_pass = [&](int g0, int g, bool primary, const int* run_if, bool last) -> int {
    // lists, slot_of (every entry written), counts and pairs of this pass; counters reset inside.
    // The whole-batch pass uses parallel kernels, fallback passes one block (they usually do not
    // run, and then cost one launch)
    if (primary) {
      if (int e = launch_k(cce::list_count_kernel, dim3(mt), dim3(128), 0, stream, 1, w.keep, nt, mt, g0, g,
                           run_if, lab_slot, w.cnt_m, w.rcnt_m))
        return e;
      if (int e = launch_k(cce::list_scan_kernel, dim3(1), dim3(1024), 0, stream, 1, w.cnt_m, w.rcnt_m, mt, g,
                           (int)capacity_tiles, run_if, 1, w.off_m, w.roff_m, w.cnt_n, w.list_count,
                           w.rlist_count, w.ok, overflow, w.list_count + 3, counters))
        return e;
      if (int e = launch_k(cce::list_fill_kernel, dim3(mt), dim3(128), 0, stream, 1, w.keep, nt, mt, g0, g,
                           (int)capacity_tiles, (int)lab_capacity, lab_slot, run_if, w.off_m, w.roff_m, w.alist,
                           w.rlist, w.slot_of, w.cnt_n))
        return e;
      if (pair)
        if (int e = launch_k(cce::build_pairs_kernel, dim3(1), dim3(1024), 0, stream, 1, w.rcnt_m, mt,
                             (const int*)w.ok, w.pairs, w.pair_count))
          return e;
    } else {
      // fallback: the whole S-hat buffer as recompute slots (stored label tiles recomputed too),
      // so each group covers more token tiles and the gated chain is shorter
      if (int e = launch_k(cce::list_single_kernel, dim3(1), dim3(1024), 0, stream, 1, w.keep, nt, mt, g0, g,
                           (int)(capacity_tiles + lab_capacity), 0, (const int32_t*)nullptr, run_if, w.cnt_m,
                           w.rcnt_m, w.off_m,
                           w.roff_m, w.alist, w.rlist, w.slot_of, w.cnt_n, w.list_count, w.rlist_count,
                           w.list_count + 3, w.pairs, w.pair_count))
        return e;
    }
    const int* gate = primary ? w.ok : run_if;  // primary: only if every tile to recompute got a slot
    cce::Params p{};
    p.n_total = (int)n;
    p.n_valid = n_valid;
    p.run_if = gate;
    p.d = (int)d;
    p.v = (int)v;
    p.nt = g;
    p.n_base = g0;
    p.mt = mt;
    p.splits = std::max(1, (2 * num_sms() + g - 1) / g);  // grid sizing only
    p.band = choose_band(d);
    p.num_kb = (int)((d + cce::BK - 1) / cce::BK);
    p.softcap = softcap;
    p.lse = lse;
    p.upstream = upstream;
    p.pos = pos;
    p.pos_offset = (int)pos_offset;
    p.row_map = row_map;
    p.eps = eps;
    p.label_split = label_split;
    p.shat = primary ? shat_rec : shat_all;
    p.capacity = (int)(primary ? capacity_tiles : capacity_tiles + lab_capacity);
    p.counters = counters;
    p.list = w.rlist;
    p.list_count = w.rlist_count;
    p.pairs = w.pairs;
    p.pair_count = w.pair_count;
    const bool gathered = aliased && !primary;  // C_t may already hold dC: gather from C
    if (gathered) {  // C rows through the permutation (cp.async gathers)
      p.perm = perm_padded;
      p.c_rows = static_cast<const __nv_bfloat16*>(C);
      if (int e = launch_lse<cce::KEPT>(p, pair, tmE, tmE, tmCo, tmCog, tmC128h, stream)) return e;
    } else if (int e = launch_lse<cce::KEPT>(p, pair, tmE, tmE, tmC, tmC, tmC128h, stream)) {
      return e;
    }

    cce::GradParams q{};
    q.n_total = (int)n;
    q.n_valid = n_valid;
    q.run_if = gate;
    q.d = (int)d;
    q.v = (int)v;
    q.mt = mt;
    q.ndc = ndc;
    q.n_base = g0;
    q.g = g;
    q.slot_of = w.slot_of;  // rows of this pass, local token-tile index; unified slots
    q.cnt_n = w.cnt_n;
    q.cnt_m = w.cnt_m;
    q.perm = gathered ? perm_padded : nullptr;
    q.perm_store = perm_padded;
    q.row_map = row_map;
    q.e_gather = 0;
    q.atoms3d = atoms3d ? 1 : 0;
    q.de_bf16 = de_fp32 ? nullptr : static_cast<__nv_bfloat16*>(de_out);
    q.de_f32 = de_fp32 ? static_cast<float*>(de_out) : nullptr;
    q.de_accumulate = de_accumulate ? 1 : 0;  // vocabulary groups after the first add into dE
    q.dc = static_cast<__nv_bfloat16*>(dc);
    q.accumulate = g0 > 0;
    q.list = w.alist;
    q.off_m = w.off_m;
    if (primary && side) CCE_CUDA(cudaStreamWaitEvent(stream, side->join, 0));  // label S-hat ready
    if (de_out != nullptr)  // NULL: the caller does not want dE (e.g. its input needs no grad)
      if (int e = launch_de(q, w.list_count + 3, shat_all, shat_rows, gathered ? C : C_t,
                            gathered ? tmCog : tmC64, stream))
        return e;
    if (last && de_done_event)  // every dE write of this call is enqueued before this point
      CCE_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(de_done_event), stream));
    if (dc == nullptr) return 0;  // NULL: no dC wanted (a frozen classifier)
    return launch_dc(q, pair && atoms3d, tmS64, tmE64, tmE3, tmE3h, tmE64, stream);
  };
  // The counts are only known on the device: the whole-batch pass runs iff its tiles to
  // recompute fit; otherwise (*overflow) token-tile groups sized for the worst case run instead.
  const bool grouped = (int64_t)nt * mt > capacity_tiles;
  PdlScope pdl_scope(true);
  if (int e = run_pass(0, nt, true, nullptr, !grouped)) return e;
  if (stats) {  // label tiles stored by the forward, tiles the whole-batch pass had to recompute
    if (lab_capacity > 0)
      CCE_CUDA(cudaMemcpyAsync(stats, lab_count, sizeof(int), cudaMemcpyDeviceToDevice, stream));
    else
      CCE_CUDA(cudaMemsetAsync(stats, 0, sizeof(int), stream));
    CCE_CUDA(cudaMemcpyAsync(stats + 1, w.rlist_count, sizeof(int), cudaMemcpyDeviceToDevice, stream));
  }
  if (kept_per_vtile)  // kept tiles per vocab tile of the whole batch (list_count_kernel)
    CCE_CUDA(cudaMemcpyAsync(kept_per_vtile, w.cnt_m, (size_t)mt * sizeof(int), cudaMemcpyDeviceToDevice, stream));
  if (grouped && !getenv("CCE_MEASURE_NO_FALLBACK")) {  // the env switch is for A/B timing only
    const int g = (int)std::max<int64_t>(1, (capacity_tiles + lab_capacity) / mt);
    for (int g0 = 0; g0 < nt; g0 += g)
      if (int e = run_pass(g0, std::min(g, nt - g0), false, overflow, g0 + g >= nt)) return e;
  }
  return 0;
}

// ---- low-memory backward: vocabulary groups ----
namespace {
struct LowWs {
  __nv_bfloat16* e_c;
  __nv_bfloat16* c_g;
  __nv_bfloat16* shat;
  uint8_t* block_zero;
  int32_t* slot_of;
  int* ctr;    // slot counter
  int* cnt_n;  // [nt]
  int* cnt_m;  // [group_vtiles]
  size_t slot_bytes, ctr_bytes, total;
};

LowWs low_layout(void* base, int64_t n, int64_t d, int64_t v, int64_t gv) {
  const int64_t nt = (n + cce::BM - 1) / cce::BM;
  auto up = [](size_t x) { return (x + 1023) & ~size_t(1023); };
  uint8_t* b = static_cast<uint8_t*>(base);
  LowWs w;
  size_t o = 0;
  w.e_c = reinterpret_cast<__nv_bfloat16*>(b + o); o += up((size_t)n * d * 2);
  w.c_g = reinterpret_cast<__nv_bfloat16*>(b + o); o += up((size_t)std::min<int64_t>(gv * cce::BN, v) * d * 2);
  w.shat = reinterpret_cast<__nv_bfloat16*>(b + o); o += up((size_t)nt * gv * cce::SHAT_TILE_BYTES);
  w.block_zero = b + o; o += up((size_t)nt);
  w.slot_bytes = up((size_t)nt * gv * 4);
  w.slot_of = reinterpret_cast<int32_t*>(b + o); o += w.slot_bytes;
  w.ctr_bytes = up(256 + (size_t)(nt + gv) * 4);
  w.ctr = reinterpret_cast<int*>(b + o);
  w.cnt_n = reinterpret_cast<int*>(b + o + 256);
  w.cnt_m = w.cnt_n + nt;
  o += w.ctr_bytes;
  w.total = o;
  return w;
}
}  // namespace

size_t cce_bwd_lowmem_workspace_bytes(int64_t n, int64_t d, int64_t v, int64_t group_vtiles) {
  return low_layout(nullptr, n, d, v, group_vtiles).total;
}

int cce_bwd_lowmem(const void* E, const void* C, const int32_t* perm_padded, const int32_t* row_map,
                   const int* n_valid, const int32_t* pos, const float* lse, const float* upstream,
                   int64_t n, int64_t d, int64_t v, float softcap, float eps, int label_split,
                   int64_t group_vtiles, void* ws, size_t ws_bytes, float* de_f32, void* dc,
                   unsigned long long* counters, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (d % 8 != 0) return fail("cce_bwd_lowmem: D must be a multiple of 8");
  if (group_vtiles < 1) return fail("cce_bwd_lowmem: group_vtiles must be >= 1");
  if (n <= 0) return 0;
  const LowWs w = low_layout(ws, n, d, v, group_vtiles);
  if (ws_bytes < w.total) return fail("cce_bwd_lowmem: workspace too small");
  const int nt = (int)((n + cce::BM - 1) / cce::BM);
  const int mt = (int)((v + cce::BN - 1) / cce::BN);
  const int ndc = (int)((d + cce::DCH - 1) / cce::DCH);
  const bool atoms3d = d % 64 == 0;
  const bool pair = use_pairs();
  // filter_ignored (kernels.py:494-510) and zero-upstream token tiles, once
  PDL_LAUNCH(cce::gather_rows_kernel, dim3((unsigned)((n + 7) / 8)), dim3(256), 0, stream, static_cast<const __nv_bfloat16*>(E), row_map, n, (int)d, w.e_c);
  CCE_CUDA(cudaGetLastError());
  PDL_LAUNCH(cce::block_zero_kernel, dim3(nt), dim3(cce::BM), 0, stream, upstream, row_map, n_valid, w.block_zero);
  CCE_CUDA(cudaGetLastError());
  CUtensorMap tmE, tmE64, tmE3, tmE3h, tmS64;
  const int64_t shat_rows = (int64_t)nt * group_vtiles * cce::BM;
  bool ok = make_tmap(&tmE, w.e_c, n, d, cce::BM) && make_tmap(&tmE64, w.e_c, n, d, 64) &&
            make_tmap3d(&tmS64, w.shat, shat_rows, cce::BN, 64, 2);
  if (ok && atoms3d)
    ok = make_tmap3d(&tmE3, w.e_c, n, d, 64, cce::DCH / 64) && make_tmap3d(&tmE3h, w.e_c, n, d, 64, cce::DCH / 128);
  else
    tmE3 = tmE3h = tmE64;
  if (!ok) return fail("cce_bwd_lowmem: cuTensorMapEncodeTiled failed");

  for (int m0 = 0; m0 < mt; m0 += (int)group_vtiles) {
    const int gm = std::min((int)group_vtiles, mt - m0);           // vocab tiles in this group
    const int64_t r0 = (int64_t)m0 * cce::BN;
    const int64_t rows = std::min<int64_t>((int64_t)gm * cce::BN, v - r0);  // classifier rows
    // this group's classifier rows in tile order (C[perm] slice, or a view of C)
    const void* cg = static_cast<const __nv_bfloat16*>(C) + r0 * d;
    if (perm_padded) {
      PDL_LAUNCH(cce::gather_rows_kernel, dim3((unsigned)((rows + 7) / 8)), dim3(256), 0, stream, static_cast<const __nv_bfloat16*>(C), perm_padded + r0, rows, (int)d, w.c_g);
      CCE_CUDA(cudaGetLastError());
      cg = w.c_g;
    }
    CUtensorMap tmC, tmC128h, tmC64;
    if (!make_tmap(&tmC, cg, rows, d, cce::BN) || !make_tmap(&tmC128h, cg, rows, d, cce::BN / 2) ||
        !make_tmap(&tmC64, cg, rows, d, cce::DE_KV))
      return fail("cce_bwd_lowmem: cuTensorMapEncodeTiled failed");
    CCE_CUDA(cudaMemsetAsync(w.slot_of, 0xFF, w.slot_bytes, stream));
    CCE_CUDA(cudaMemsetAsync(w.ctr, 0, w.ctr_bytes, stream));
    // (B1) recompute every tile of the group, filter, S-hat of kept tiles (capacity = worst case)
    cce::Params p{};
    p.n_total = (int)n;
    p.n_valid = n_valid;
    p.d = (int)d;
    p.v = (int)rows;
    p.nt = nt;
    p.n_base = 0;
    p.mt = gm;
    set_raster(p, nt, gm, d, pair, true);
    p.num_kb = (int)((d + cce::BK - 1) / cce::BK);
    p.softcap = softcap;
    p.lse = lse;
    p.upstream = upstream;
    p.pos = pos;
    p.pos_offset = (int)r0;
    p.row_map = row_map;
    p.block_zero = w.block_zero;
    p.eps = eps;
    p.label_split = label_split;
    p.shat = w.shat;
    p.slot_of = w.slot_of;
    p.slot_ctr = w.ctr;
    p.capacity = nt * gm;
    p.cnt_n = w.cnt_n;
    p.cnt_m = w.cnt_m;
    p.counters = counters;
    if (int e = launch_lse<cce::BWD>(p, pair, tmE, tmE, tmC, tmC, tmC128h, stream)) return e;
    // (B2) dE += S-hat C over the group (fp32 accumulate), (B3) dC of the group's vocab tiles
    cce::GradParams q{};
    q.n_total = (int)n;
    q.n_valid = n_valid;
    q.d = (int)d;
    q.v = (int)rows;
    q.mt = gm;
    q.ndc = ndc;
    q.n_base = 0;
    q.g = nt;
    q.slot_of = w.slot_of;
    q.cnt_n = w.cnt_n;
    q.cnt_m = w.cnt_m;
    q.perm = nullptr;
    q.perm_store = perm_padded ? perm_padded + r0 : nullptr;
    q.row_map = row_map;
    q.atoms3d = atoms3d ? 1 : 0;
    q.de_f32 = de_f32;
    q.de_accumulate = 1;
    q.dc = static_cast<__nv_bfloat16*>(dc) + (perm_padded ? 0 : r0 * d);
    q.accumulate = 0;
    if (int e = launch_de(q, w.ctr + 1, w.shat, shat_rows, cg, tmC64, stream)) return e;
    if (int e = launch_dc(q, pair && atoms3d, tmS64, tmE64, tmE3, tmE3h, tmE64, stream)) return e;
  }
  return 0;
}

size_t cce_label_terms_workspace_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)std::max<int64_t>(n, 1));
  return bytes + 4 * (size_t)std::max<int64_t>(n, 1) * 4 + 1024;
}

int cce_label_terms(const void* E, const void* C, const int32_t* perm_padded, const int32_t* row_map,
                    const int* n_valid, const int32_t* pos, const float* upstream, const float* correct,
                    int64_t n, int64_t d, int64_t v, float softcap, void* ws, size_t ws_bytes, void* de,
                    int de_fp32, void* dc, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  (void)v;
  if (n <= 0) return 0;
  const size_t need = cce_label_terms_workspace_bytes(n);
  if (ws_bytes < need) return fail("cce_label_terms: workspace too small");
  int32_t* key = static_cast<int32_t*>(ws);
  int32_t* val = key + n;
  int32_t* key_s = val + n;
  int32_t* val_s = key_s + n;
  void* tmp = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(val_s + n) + 255) & ~uintptr_t(255));
  size_t tmp_bytes = need - 4 * (size_t)n * 4 - 1024;
  if (dc != nullptr) {  // NULL: no dC wanted
    PDL_LAUNCH(cce::label_keys_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, stream, row_map, n_valid,
               pos, (int)n, key, val);
    CCE_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key, key_s, val, val_s, (int)n, 0, 32, stream));
    PDL_LAUNCH(cce::label_dc_kernel, dim3((unsigned)std::min<int64_t>(n, 4 * num_sms()), (unsigned)((d + 255) / 256)),
               dim3(256), 0, stream, key_s, val_s, (int)n,
               static_cast<const __nv_bfloat16*>(E), upstream, correct, softcap, perm_padded, (int)d,
               static_cast<__nv_bfloat16*>(dc));
  }
  if (de != nullptr)  // NULL: no dE wanted
    PDL_LAUNCH(cce::label_de_kernel, dim3((unsigned)((n + 7) / 8)), dim3(256), 0, stream, row_map, n_valid, pos,
               static_cast<const __nv_bfloat16*>(C), perm_padded, upstream, correct, softcap, (int)n, (int)d,
               de_fp32 ? static_cast<float*>(de) : nullptr, de_fp32 ? nullptr : static_cast<__nv_bfloat16*>(de));
  return 0;
}

int cce_reduce_loss(const float* loss, const int64_t* targets, int64_t ignore_index, int64_t n,
                    int reduction, float* out, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (reduction != 1 && reduction != 2) return fail("cce_reduce_loss: reduction must be 1 (sum) or 2 (mean)");
  PDL_LAUNCH(cce::reduce_loss_kernel, dim3(1), dim3(1024), 0, stream, loss, targets, ignore_index, (int)n, reduction, out);
  CCE_CUDA(cudaGetLastError());
  return 0;
}

int cce_upstream(const float* grad, const int64_t* targets, int64_t ignore_index, int64_t n, int reduction,
                 float* up, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (reduction < 0 || reduction > 2) return fail("cce_upstream: reduction must be 0, 1 or 2");
  if (n == 0) return 0;
  PDL_LAUNCH(cce::upstream_kernel, dim3(1), dim3(1024), 0, stream, grad, targets, ignore_index, (int)n, reduction, up);
  CCE_CUDA(cudaGetLastError());
  return 0;
}

int cce_indexed_dot(const void* E, const void* C, const int64_t* targets, int64_t n, int64_t d,
                    int64_t v, int64_t ignore_index, int64_t vocab_start, float softcap, float* out,
                    void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (d % 8 != 0) return fail("cce_indexed_dot: D must be a multiple of 8");
  if (n == 0) return 0;
  PDL_LAUNCH(cce::indexed_dot_kernel, dim3((unsigned)((n + 7) / 8)), dim3(256), 0, stream, static_cast<const __nv_bfloat16*>(E), static_cast<const __nv_bfloat16*>(C), targets,
      ignore_index, vocab_start, (int)n, (int)d, (int)v, softcap, out);
  CCE_CUDA(cudaGetLastError());
  return 0;
}

int cce_gather_rows(const void* src, const int32_t* index, int64_t rows, int64_t cols, void* dst,
                    void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (cols % 8 != 0) return fail("cce_gather_rows: cols must be a multiple of 8");
  if (rows == 0) return 0;
  PDL_LAUNCH(cce::gather_rows_kernel, dim3((unsigned)((rows + 7) / 8)), dim3(256), 0, stream, static_cast<const __nv_bfloat16*>(src), index, rows, (int)cols, static_cast<__nv_bfloat16*>(dst));
  CCE_CUDA(cudaGetLastError());
  return 0;
}

int cce_f32_to_bf16(const float* x, void* y, int64_t count, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (count % 4 != 0) return fail("cce_f32_to_bf16: count must be a multiple of 4");
  const int64_t n4 = count / 4;
  if (n4 == 0) return 0;
  PDL_LAUNCH(cce::f32_to_bf16_kernel, dim3((unsigned)((n4 + 255) / 256)), dim3(256), 0, stream, x, static_cast<__nv_bfloat16*>(y), n4);
  CCE_CUDA(cudaGetLastError());
  return 0;
}

}  // extern "C"

// ---- streamed backward (cce_stream.cuh): bounded transients, any kept-tile count ----
namespace {
int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return (e && atoi(e) > 0) ? atoi(e) : dflt;
}
int stream_seg_voc() { return env_int("CCE_STREAM_SEG_VOC", 64); }
int stream_nacc() { return env_int("CCE_STREAM_NACC", 4); }
// dE consumers: two double-buffered 256-column accumulators fed by 64-row stages (default) or one
// 512-column accumulator fed by 32-row stages (CCE_STREAM_DE=2; measured 7.8 vs 7.3 ms backward at
// Gemma-2-2B)
int stream_de_ch() { return env_int("CCE_STREAM_DE", 1) == 2 ? 2 : 1; }
int stream_window(int64_t ring) { return (int)std::min<int64_t>(ring - 1, env_int("CCE_STREAM_WINDOW", (int)(ring / 2))); }

struct StreamWs {
  uint8_t* block_zero;
  uint8_t* keep;
  int* voc_cnt;
  int* voc_rcnt;
  int* voc_off;
  int2* items;      // vocab-tile-major kept list (the stream)
  int4* cseg;       // dC segments (vocab tile owners)
  int2* caux;
  int2* pairs;      // producer CTA-pair entries
  int* wcnt;        // [max windows][nt]
  int* wsplit;
  int* wstart;
  int* nsplit;      // [nt]
  int* sidx;        // [items] stream positions grouped by (window, token tile)
  int4* eseg;       // dE segments (window, token tile)
  int2* eaux;
  int* ctrl;        // [0] items [1] dC segments [2] pairs [3] dE segments [4] permutation breaks
  int* ready;
  int* used;
  int* chain_e;
  int* chain_c;
  int* gen_e;
  int* gen_c;
  size_t ctrl_bytes;  // zeroed per call (ctrl .. gen_c)
  float* acc_e;       // [nt][ndc][128][256] fp32 dE partial sums across windows
  float* acc_c;       // [nacc][ndc][2][128][256] fp32 partial sums of vocab tiles split over segments;
                      // afterwards the row-permutation scratch (with acc_e)
  uint8_t* perm_cls;
  int32_t* perm_bidx;
  int32_t* perm_blist;
  int32_t* perm_own;   // [v] member -> owner break position
  int32_t* perm_seg;   // [cap][PERM_SEG] segment positions
  int* perm_len;       // [cap]
  int32_t* perm_rlist; // [v / 2 + 1] rotation owners
  int perm_cap;
  int max_windows;
  size_t total;
};

StreamWs stream_layout(void* base, int64_t n, int64_t d, int64_t v, int64_t ring) {
  const int64_t nt = std::max<int64_t>(1, (n + cce::BM - 1) / cce::BM);
  const int64_t mt = (v + cce::BN - 1) / cce::BN;
  const int64_t ndc = (d + cce::DCH - 1) / cce::DCH;
  const int64_t items = nt * mt;
  const int64_t W = stream_window(ring);
  const int64_t maxw = (items + W - 1) / W;
  const int64_t seg_c = mt + items / stream_seg_voc() + 1;
  const int64_t nacc = stream_nacc();
  auto up = [](size_t x) { return (x + 1023) & ~size_t(1023); };
  uint8_t* b = static_cast<uint8_t*>(base);
  StreamWs w{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    uint8_t* ptr = b ? b + o : nullptr;
    o += up(bytes);
    return ptr;
  };
  w.block_zero = take(nt);
  w.keep = take(nt * mt);
  w.voc_cnt = reinterpret_cast<int*>(take(mt * 4));
  w.voc_rcnt = reinterpret_cast<int*>(take(mt * 4));
  w.voc_off = reinterpret_cast<int*>(take(mt * 4));
  w.items = reinterpret_cast<int2*>(take(items * 8));
  w.cseg = reinterpret_cast<int4*>(take(seg_c * 16));
  w.caux = reinterpret_cast<int2*>(take(seg_c * 8));
  w.pairs = reinterpret_cast<int2*>(take((items / 2 + mt + 1) * 8));
  w.wcnt = reinterpret_cast<int*>(take(maxw * nt * 4));
  w.wsplit = reinterpret_cast<int*>(take(maxw * nt * 4));
  w.wstart = reinterpret_cast<int*>(take(maxw * nt * 4));
  w.nsplit = reinterpret_cast<int*>(take(nt * 4));
  w.sidx = reinterpret_cast<int*>(take(items * 4));
  w.eseg = reinterpret_cast<int4*>(take(items * 16));
  w.eaux = reinterpret_cast<int2*>(take(items * 8));
  const size_t c0 = o;
  w.ctrl = reinterpret_cast<int*>(take(64));
  w.ready = reinterpret_cast<int*>(take(ring * 4));
  w.used = reinterpret_cast<int*>(take(ring * 4));
  w.chain_e = reinterpret_cast<int*>(take(nt * ndc * 4));
  w.chain_c = reinterpret_cast<int*>(take(mt * ndc * 2 * 4));
  w.gen_e = reinterpret_cast<int*>(take(nt * ndc * 4));
  w.gen_c = reinterpret_cast<int*>(take(nacc * ndc * 2 * 4));
  w.ctrl_bytes = o - c0;
  // breaks: anchors (~v / PERM_K) + cut points (at most v / PERM_SEG), with headroom
  w.perm_cap = (int)(v / cce::PERM_K * 5 / 4 + v / cce::PERM_SEG + 1024);
  const int64_t dch = stream_de_ch();
  const size_t acc_e = (size_t)nt * ((ndc + dch - 1) / dch * dch) * cce::BM * cce::DCH * 4;
  const size_t acc_c = (size_t)nacc * ndc * 2 * cce::BM * cce::DCH * 4;
  const size_t perm_bytes = (size_t)w.perm_cap * d * 2;
  uint8_t* accs = take(std::max(acc_e + acc_c, perm_bytes));
  w.acc_e = reinterpret_cast<float*>(accs);
  w.acc_c = reinterpret_cast<float*>(accs ? accs + acc_e : nullptr);
  w.perm_cls = take(v);
  w.perm_bidx = reinterpret_cast<int32_t*>(take(v * 4));
  w.perm_blist = reinterpret_cast<int32_t*>(take((size_t)w.perm_cap * 4));
  w.perm_own = reinterpret_cast<int32_t*>(take(v * 4));
  w.perm_seg = reinterpret_cast<int32_t*>(take((size_t)w.perm_cap * cce::PERM_SEG * 4));
  w.perm_len = reinterpret_cast<int*>(take((size_t)w.perm_cap * 4));
  w.perm_rlist = reinterpret_cast<int32_t*>(take((size_t)(v / 2 + 1) * 4));
  w.max_windows = (int)maxw;
  w.total = o;
  return w;
}

// In-place: rows X[p] -> X[perm[p]] (p < v); scratch from the stream workspace (after the pass).
int unpermute_rows(__nv_bfloat16* X, const int32_t* perm, const int32_t* inv, int64_t v, int64_t d, const StreamWs& w,
                   cudaStream_t stream) {
  __nv_bfloat16* tmp = reinterpret_cast<__nv_bfloat16*>(w.acc_e);
  // Without programmatic dependent launch: under PDL the walk saw stale chain tables (kernels two
  // and more launches back; test_unpermute_rows_in_place fails with it, passes with CCE_PDL=0 or
  // CUDA_LAUNCH_BLOCKING=1), as the window kernels of the pass did.  Six launch gaps.
  PdlScope nopdl(false);
  PDL_LAUNCH(cce::zero_words_kernel, dim3(32), dim3(256), 0, stream, w.perm_len, (int64_t)w.perm_cap);
  PDL_LAUNCH(cce::unpermute_classify_kernel, dim3((unsigned)((v + 255) / 256)), dim3(256), 0, stream, perm, (int)v,
             w.perm_cls, w.perm_bidx, w.perm_own, w.perm_blist, w.ctrl + 4, w.perm_cap, w.perm_rlist, w.ctrl + 6);
  PDL_LAUNCH(cce::unpermute_chains_kernel, dim3((unsigned)((v + 255) / 256)), dim3(256), 0, stream, (int)v,
             (const uint8_t*)w.perm_cls, (const int32_t*)w.perm_bidx, (const int32_t*)w.perm_own, w.perm_seg,
             w.perm_len);
  // warps per (break, column block); the break count is on the device, the grid covers the cap
  const dim3 grid((unsigned)((w.perm_cap + 7) / 8), (unsigned)((d + cce::PERM_COLS - 1) / cce::PERM_COLS));
  PDL_LAUNCH(cce::unpermute_save_kernel, grid, dim3(256), 0, stream, static_cast<const __nv_bfloat16*>(X), (int)d,
             (const int32_t*)w.perm_blist, (const int*)(w.ctrl + 4), tmp);
  PDL_LAUNCH(cce::unpermute_walk_kernel, grid, dim3(256), 0, stream, X, (int)d, inv, (const int32_t*)w.perm_bidx,
             (const int32_t*)w.perm_blist, (const int32_t*)w.perm_seg, (const int*)w.perm_len,
             (const int*)(w.ctrl + 4), (const __nv_bfloat16*)tmp);
  PDL_LAUNCH(cce::unpermute_rotate_kernel, dim3((unsigned)num_sms(), grid.y), dim3(256), 0, stream, X, (int)d, inv,
             (const int32_t*)w.perm_rlist, (const int*)(w.ctrl + 6));
  CCE_CUDA(cudaGetLastError());
  return 0;
}
}  // namespace

extern "C" {

size_t cce_bwd_stream_workspace_bytes(int64_t n, int64_t d, int64_t v, int64_t ring_slots) {
  return stream_layout(nullptr, n, d, v, ring_slots).total;
}

// Diagnostics: byte offsets in the workspace of {keep, items, wcnt, wstart, sidx, eseg, eaux, ctrl,
// voc_cnt, voc_off, cseg, caux, pairs} (13 values), and the window size.
int cce_bwd_stream_debug_layout(int64_t n, int64_t d, int64_t v, int64_t ring_slots, int64_t* out) {
  const StreamWs w = stream_layout(reinterpret_cast<void*>(uintptr_t(1) << 20), n, d, v, ring_slots);
  const void* ptrs[13] = {w.keep, w.items, w.wcnt, w.wstart, w.sidx, w.eseg, w.eaux, w.ctrl,
                          w.voc_cnt, w.voc_off, w.cseg, w.caux, w.pairs};
  for (int i = 0; i < 13; ++i) out[i] = (int64_t)(reinterpret_cast<uintptr_t>(ptrs[i])) - (int64_t(1) << 20);
  return stream_window(ring_slots);
}

// Diagnostics / tests: the streamed backward's in-place row unpermutation alone, X[perm[p]] <- X[p]
// (bf16 [v, d]); ws from cce_bwd_stream_workspace_bytes(1, d, v, 512).
int cce_unpermute_rows(void* X, const int32_t* perm, const int32_t* inv, int64_t v, int64_t d, void* ws,
                       size_t ws_bytes, void* stream_ptr) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (d % 8 != 0) return fail("cce_unpermute_rows: D must be a multiple of 8");
  const StreamWs w = stream_layout(ws, 1, d, v, 512);
  if (ws_bytes < w.total) return fail("cce_unpermute_rows: workspace too small");
  PdlScope pdl_scope(true);
  PDL_LAUNCH(cce::zero_words_kernel, dim3(64), dim3(256), 0, stream, w.ctrl, (int64_t)(w.ctrl_bytes / 4));
  return unpermute_rows(static_cast<__nv_bfloat16*>(X), perm, inv, v, d, w, stream);
}

int cce_bwd_stream_ex(const void* E, int e_gather, const void* C, void* c_sorted, const int32_t* perm_padded,
                      const int32_t* inv_perm, const int32_t* row_map, const int* n_valid, const int32_t* pos,
                      const float* lse, const float* upstream, const float* tile_max, int64_t n, int64_t d,
                      int64_t v, float softcap, float eps, int label_split, void* ring, int64_t ring_slots, void* ws,
                      size_t ws_bytes, void* de_out, int de_fp32, void* dc, unsigned long long* counters,
                      void* de_done_event, int flags, void* stream_ptr);

int cce_bwd_stream(const void* E, int e_gather, const void* C, void* c_sorted, const int32_t* perm_padded,
                   const int32_t* inv_perm, const int32_t* row_map, const int* n_valid, const int32_t* pos,
                   const float* lse, const float* upstream, const float* tile_max, int64_t n, int64_t d, int64_t v,
                   float softcap, float eps, int label_split, void* ring, int64_t ring_slots, void* ws,
                   size_t ws_bytes, void* de_out, int de_fp32, void* dc, unsigned long long* counters,
                   void* de_done_event, void* stream_ptr) {
  return cce_bwd_stream_ex(E, e_gather, C, c_sorted, perm_padded, inv_perm, row_map, n_valid, pos, lse, upstream,
                           tile_max, n, d, v, softcap, eps, label_split, ring, ring_slots, ws, ws_bytes, de_out,
                           de_fp32, dc, counters, de_done_event, 0, stream_ptr);
}

int cce_bwd_stream_ex(const void* E, int e_gather, const void* C, void* c_sorted, const int32_t* perm_padded,
                      const int32_t* inv_perm, const int32_t* row_map, const int* n_valid, const int32_t* pos,
                      const float* lse, const float* upstream, const float* tile_max, int64_t n, int64_t d,
                      int64_t v, float softcap, float eps, int label_split, void* ring, int64_t ring_slots, void* ws,
                      size_t ws_bytes, void* de_out, int de_fp32, void* dc, unsigned long long* counters,
                      void* de_done_event, int flags, void* stream_ptr) {
  const bool c_ready = (flags & 1) != 0;      // c_sorted already holds C[perm] (an earlier token chunk)
  const bool dc_accumulate = (flags & 2) != 0;  // add into dc (vocabulary order) instead of writing it
  cudaStream_t stream = static_cast<cudaStream_t>(stream_ptr);
  if (d % 8 != 0) return fail("cce_bwd_stream: D must be a multiple of 8");
  if (!(eps > 0.f)) return fail("cce_bwd_stream: needs filtering (eps > 0)");
  if (!ring || ring_slots < 2 * stream_seg_voc()) return fail("cce_bwd_stream: ring_slots too small");
  if (de_out == nullptr && dc == nullptr) return fail("cce_bwd_stream: neither dE nor dC requested");
  if (perm_padded && c_sorted && !inv_perm) return fail("cce_bwd_stream: a sorted copy needs inv_perm");
  if (d % 64 != 0) return fail("cce_bwd_stream: D must be a multiple of 64 (CTA-pair operand boxes)");
  if (n <= 0) return 0;
  const int nt = (int)((n + cce::BM - 1) / cce::BM);
  const int mt = (int)((v + cce::BN - 1) / cce::BN);
  const int ndc = (int)((d + cce::DCH - 1) / cce::DCH);
  if (nt > 2048) return fail("cce_bwd_stream: at most 2048 token tiles (262144 rows) per call");
  const StreamWs w = stream_layout(ws, n, d, v, ring_slots);
  if (ws_bytes < w.total) return fail("cce_bwd_stream: workspace too small");
  const int R = (int)ring_slots;
  const int W = stream_window(ring_slots);
  const int sms = num_sms();
  if (sms < 6) return fail("cce_bwd_stream: needs at least 6 SMs");
  PdlScope pdl_scope(true);

  // sorted classifier: C[perm] into c_sorted (dC's own storage when dc == c_sorted), or, with no
  // c_sorted, C rows gathered through the order inside the pass (cp.async in the recompute CTAs,
  // TMA gather4 in the dE CTAs) and dC scattered to vocabulary order by its epilogue
  const void* C_t = C;
  const bool c_gather = perm_padded && !c_sorted;
  if (dc_accumulate && (dc == c_sorted || !dc)) return fail("cce_bwd_stream: accumulating dC needs its own buffer");
  if (perm_padded && c_sorted) {
    if (!c_ready)
      PDL_LAUNCH(cce::gather_rows_kernel, dim3((unsigned)((v + 7) / 8)), dim3(256), 0, stream,
                 static_cast<const __nv_bfloat16*>(C), (const int32_t*)perm_padded, (int)v, (int)d,
                 static_cast<__nv_bfloat16*>(c_sorted));
    C_t = c_sorted;
  }
  // decision (kernels.py:434-455), the stream (vocab-tile-major kept list), its segments
  PDL_LAUNCH(cce::zero_words_kernel, dim3(64), dim3(256), 0, stream, w.ctrl, (int64_t)(w.ctrl_bytes / 4));
  PDL_LAUNCH(cce::block_zero_kernel, dim3(nt), dim3(cce::BM), 0, stream, upstream, row_map, n_valid, w.block_zero);
  PDL_LAUNCH(cce::decide_tiles_kernel, dim3((unsigned)((mt + cce::DECIDE_VT - 1) / cce::DECIDE_VT), (unsigned)nt),
             dim3(256), 0, stream, tile_max, lse, pos, 0, row_map, n_valid, (const uint8_t*)w.block_zero, nt, mt,
             softcap, eps, label_split, w.keep, counters);
  PDL_LAUNCH(cce::list_count_kernel, dim3(mt), dim3(128), 0, stream, (const uint8_t*)w.keep, nt, mt, 0, nt,
             (const int*)nullptr, (const int32_t*)nullptr, w.voc_cnt, w.voc_rcnt);
  PDL_LAUNCH(cce::segments_kernel, dim3(1), dim3(1024), 0, stream, (const int*)w.voc_cnt, mt, stream_seg_voc(),
             w.voc_off, w.ctrl + 0, w.cseg, w.caux, w.ctrl + 1, counters);
  PDL_LAUNCH(cce::fill_items_kernel<false>, dim3(mt), dim3(256), 0, stream, (const uint8_t*)w.keep, nt, mt,
             (const int*)w.voc_off, w.items);
  PDL_LAUNCH(cce::build_pairs_kernel, dim3(1), dim3(1024), 0, stream, (const int*)w.voc_cnt, mt, (const int*)nullptr,
             w.pairs, w.ctrl + 2);
  // The window kernels run without programmatic dependent launch: under PDL they read the stream
  // list before it is complete (measured: wrong dE segments on warm calls, CCE_STREAM_NOPDL=1 fixes
  // it); three launch gaps of a few microseconds.  Diagnostics: CCE_STREAM_NOPDL bit1 also turns it
  // off for the pass kernel.
  const int pdl_mask = env_int("CCE_STREAM_NOPDL", 0) | 1;
  if (de_out) {
    PdlScope wpdl(!(pdl_mask & 1));
    PDL_LAUNCH(cce::window_count_kernel, dim3(w.max_windows), dim3(256), (size_t)nt * 4, stream,
               (const int2*)w.items, (const int*)(w.ctrl + 0), W, nt, w.wcnt);
    PDL_LAUNCH(cce::window_segments_kernel, dim3(1), dim3(1024), 0, stream, (const int*)w.wcnt,
               (const int*)(w.ctrl + 0), W, nt, w.wsplit, w.nsplit, w.wstart, w.eseg, w.eaux, w.ctrl + 3);
    if (int e = ensure_attr(cce::window_fill_kernel, (size_t)9 * nt * 4)) return e;
    PDL_LAUNCH(cce::window_fill_kernel, dim3(w.max_windows), dim3(256), (size_t)9 * nt * 4, stream,
               (const int2*)w.items, (const int*)(w.ctrl + 0), W, nt, (const int*)w.wstart, w.sidx);
  }

  if (getenv("CCE_STREAM_LISTS_ONLY")) return 0;  // diagnostics: the lists alone
  const int de_ch = c_gather ? 1 : stream_de_ch();  // row gathers need 64-row boxes
  const int de_kv = de_ch == 2 ? 32 : 64;
  CUtensorMap tmE, tmC128, tmSe, tmCk, tmC3, tmSc, tmE64, tmE3h;
  const bool ok = make_tmap(&tmE, E, n, d, cce::BM) && make_tmap(&tmC128, C_t, v, d, cce::BN / 2) &&
                  make_tmap3d_inner(&tmSe, ring, (int64_t)R * cce::BM, cce::BN, de_kv, cce::BM, 1) &&
                  (c_gather ? make_tmap(&tmCk, C, v, d, 1) : make_tmap(&tmCk, C_t, v, d, de_kv)) &&
                  make_tmap3d(&tmC3, C_t, v, d, de_kv, cce::DCH / 64) &&
                  make_tmap3d(&tmSc, ring, (int64_t)R * cce::BM, cce::BN, 64, 2) && make_tmap(&tmE64, E, n, d, 64) &&
                  make_tmap3d(&tmE3h, E, n, d, 64, cce::DCH / 128);
  if (!ok) return fail("cce_bwd_stream: cuTensorMapEncodeTiled failed");

  // roles: producers and dC consumers as CTA pairs, dE consumers single (about a third each)
  const int grid = sms & ~1;
  // Recompute CTAs by hidden size: a kept tile's recompute has a fixed epilogue (S-hat of 128 x 256
  // logits) and a mainloop growing with D, the contractions grow with D alone, so small heads need
  // more recompute CTAs.  Measured best (148 SMs, scripts/ab_r2/r2_split2.sh, r2_splitd.sh): 56 at
  // D = 768 (1.15 vs 1.57 ms with 32), 36 at 1536, 32 at 2304 (6.14 vs 6.27 ms with 36) and 4096;
  // the rest split 54 : 62 between dC and dE.
  const double pd = d <= 768 ? 56.0 : d <= 1536 ? 56.0 - (d - 768) * (20.0 / 768.0)
                    : d <= 2304 ? 36.0 - (d - 1536) * (4.0 / 768.0) : 32.0;
  const int p_def = ((int)(grid * pd / 148.0 + 0.5) + 1) & ~1;
  int P = env_int("CCE_STREAM_P", p_def);
  int Qc = dc ? env_int("CCE_STREAM_QC", ((int)((grid - p_def) * 54.0 / 116.0 + 0.5) + 1) & ~1) : 0;
  P = std::max(2, P & ~1);
  Qc = dc ? std::max(2, Qc & ~1) : 0;
  if (!de_out) Qc = grid - P;
  if (P + Qc > grid - (de_out ? 1 : 0)) return fail("cce_bwd_stream: CCE_STREAM_P + CCE_STREAM_QC leave no dE CTAs");
  // consumptions per item: one per dC pair-unit (D chunk) and one per dE unit (group of de_ch chunks)
  const int consumers = (dc ? ndc : 0) + (de_out ? (ndc + de_ch - 1) / de_ch : 0);
  const cce::Stream st{R, w.ready, w.used, consumers, P};

  cce::Params p{};
  p.n_total = (int)n;
  p.n_valid = n_valid;
  p.d = (int)d;
  p.v = (int)v;
  p.nt = nt;
  p.mt = mt;
  p.splits = 1;
  p.band = choose_band(d);
  p.num_kb = (int)((d + cce::BK - 1) / cce::BK);
  p.softcap = softcap;
  p.lse = lse;
  p.upstream = upstream;
  p.pos = pos;
  p.row_map = row_map;
  p.e_gather = e_gather;
  p.e_rows = static_cast<const __nv_bfloat16*>(E);
  p.eps = eps;
  p.label_split = label_split;
  p.shat = static_cast<__nv_bfloat16*>(ring);
  if (c_gather) {
    p.perm = perm_padded;
    p.c_rows = static_cast<const __nv_bfloat16*>(C);
  }
  p.counters = counters;
  p.list = w.items;
  p.list_count = w.ctrl + 0;
  p.pairs = w.pairs;
  p.pair_count = w.ctrl + 2;
  p.st = st;
  cce::GradParams q{};
  q.n_total = (int)n;
  q.d = (int)d;
  q.v = (int)v;
  q.mt = mt;
  q.ndc = ndc;
  q.n_valid = n_valid;
  q.g = nt;
  q.row_map = row_map;
  q.e_gather = e_gather;
  q.e_rows = static_cast<const __nv_bfloat16*>(E);
  q.atoms3d = 1;
  q.st = st;
  q.items = w.items;
  cce::GradParams qe = q;
  if (c_gather) qe.perm = perm_padded;  // dE: C rows through the order (gather4 boxes)  // dE: segments (window, token tile) through sidx, accumulator id = token tile
  qe.seg = w.eseg;
  qe.seg_aux = w.eaux;
  qe.seg_count = w.ctrl + 3;
  qe.sidx = w.sidx;
  qe.chain = w.chain_e;
  qe.acc = w.acc_e;
  qe.nacc = nt;
  // diagnostics only (wrong results): 1 / 2 skip the S-hat / C operand loads, 4 the fold-in loads, 8 the stores
  qe.debug = env_int("CCE_STREAM_DEBUG_DE", 0);
  qe.acc_gen = w.gen_e;
  qe.de_bf16 = de_fp32 ? nullptr : static_cast<__nv_bfloat16*>(de_out);
  qe.de_f32 = de_fp32 ? static_cast<float*>(de_out) : nullptr;
  if (!de_out) qe.seg_count = w.ctrl + 5;  // zero segments
  // dE units claimed in order from a counter (CCE_STREAM_DYN=0: static round-robin); same box:
  // 6.31-6.39 vs 6.49 ms backward at Gemma-2-2B
  if (getenv("CCE_STREAM_DYN") == nullptr || atoi(getenv("CCE_STREAM_DYN")) != 0) qe.sched = w.ctrl + 7;
  cce::GradParams qc = q;  // dC: segments of vocab tiles (contiguous items)
  qc.seg = w.cseg;
  qc.seg_aux = w.caux;
  qc.seg_count = w.ctrl + 1;
  qc.chain = w.chain_c;
  qc.acc = w.acc_c;
  qc.nacc = stream_nacc();
  qc.acc_gen = w.gen_c;
  if (const char* pf = getenv("CCE_STREAM_PROF_PTR")) qe.prof = reinterpret_cast<unsigned long long*>(strtoull(pf, nullptr, 0));
  const bool sorted_out = perm_padded && c_sorted && dc == c_sorted;  // dC lands in the sorted order, then moves
  qc.dc = static_cast<__nv_bfloat16*>(dc);
  qc.perm_store = sorted_out ? nullptr : perm_padded;
  qc.accumulate = dc_accumulate ? 1 : 0;
  if (sorted_out && de_out && !getenv("CCE_STREAM_NOWAIT")) {  // dE consumers read the rows dC overwrites
    // (CCE_STREAM_NOWAIT: timing experiment only -- wrong results)
    qc.own_off = w.voc_off;
    qc.own_cnt = w.voc_cnt;
  }

  if (getenv("CCE_STREAM_DEBUG"))
    fprintf(stderr, "cce_bwd_stream: grid %d P %d Qc %d ring %d window %d consumers %d | ready %p used %p "
            "chain_e %p chain_c %p gen_e %p gen_c %p ctrl %p\n", grid, P, Qc, R, W, consumers, (void*)w.ready,
            (void*)w.used, (void*)w.chain_e, (void*)w.chain_c, (void*)w.gen_e, (void*)w.gen_c, (void*)w.ctrl);
  // Two streamed passes must never run at once: each needs every SM (one CTA per SM, CTAs waiting
  // on each other), so two passes sharing the GPU could each hold half of it and wait forever.
  // Passes of this process on one device are chained: a pass on another stream than the previous
  // one waits for it first (same stream: already ordered).  Not under stream capture (a graph
  // orders its own work).
  int dev_id = 0;
  CCE_CUDA(cudaGetDevice(&dev_id));
  PassOrder& order = pass_order(dev_id);
  std::lock_guard<std::mutex> order_lock(order.mu);
  cudaStreamCaptureStatus capture = cudaStreamCaptureStatusNone;
  CCE_CUDA(cudaStreamIsCapturing(stream, &capture));
  const bool ordered = capture == cudaStreamCaptureStatusNone;
  bool waited = false;
  if (ordered) {
    if (!order.last) {
      CCE_CUDA(cudaEventCreateWithFlags(&order.last, cudaEventDisableTiming));
    } else if (order.stream != stream) {
      CCE_CUDA(cudaStreamWaitEvent(stream, order.last, 0));
      waited = true;
    }
  }
  PdlScope spdl(!(pdl_mask & 2) && !waited);
  if (de_ch == 2) {
    constexpr size_t smem = std::max({kLsePairSmem, kDcSmem, de_smem<2, 32>()});
    if (int e = ensure_attr(cce::cce_stream3_kernel<2, 32>, smem)) return e;
    if (int e = launch_k(cce::cce_stream3_kernel<2, 32>, dim3(grid), dim3(cce::NUM_THREADS), smem, stream, 2, tmE,
                         tmC128, tmSe, tmCk, tmC3, tmSc, tmE64, tmE3h, p, qe, qc, Qc))
      return e;
  } else {
    constexpr size_t smem = std::max({kLsePairSmem, kDcSmem, de_smem<1, 64>()});
    if (int e = ensure_attr(cce::cce_stream3_kernel<1, 64>, smem)) return e;
    if (int e = launch_k(cce::cce_stream3_kernel<1, 64>, dim3(grid), dim3(cce::NUM_THREADS), smem, stream, 2, tmE,
                         tmC128, tmSe, tmCk, tmC3, tmSc, tmE64, tmE3h, p, qe, qc, Qc))
      return e;
  }
  if (ordered) {
    CCE_CUDA(cudaEventRecord(order.last, stream));
    order.stream = stream;
  }
  if (de_done_event) CCE_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(de_done_event), stream));
  if (sorted_out)
    if (int e = unpermute_rows(static_cast<__nv_bfloat16*>(dc), perm_padded, inv_perm, v, d, w, stream)) return e;
  CCE_CUDA(cudaGetLastError());
  return 0;
}

}  // extern "C"

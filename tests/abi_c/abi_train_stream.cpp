// The default (bounded-memory) training path driven from plain C++ through include/cce_b200.h
// alone: the call sequence of ops.forward_stream + ops.backward_from_stream_state
// -- compaction, vocabulary order, per-group gathered classifier rows and tile-recording forward,
// one combine of the groups' partials, shard merge, then the streamed backward with the sorted
// copy built in dC's storage and moved back in place -- against double-precision loss, dE, dC.
// N = 300, V = 1000: every 128 x 256 tile holds a label, so the reference's label exemption
// (kernels.py:447-455) keeps every tile and the filtered gradient equals the exact one.
// Exit code 0 = pass.  Built and run by tests/test_abi_c_gpu.py.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <vector>

#include "cce_b200.h"

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));            \
      return 2;                                                                \
    }                                                                          \
  } while (0)
#define CC(x)                                                                  \
  do {                                                                         \
    if ((x) != 0) {                                                            \
      std::fprintf(stderr, "%s: %s\n", #x, cce_last_error());                  \
      return 3;                                                                \
    }                                                                          \
  } while (0)

static uint64_t g_state = 0x2545F4914F6CDD1Dull;
static double uniform() {
  g_state ^= g_state >> 12;
  g_state ^= g_state << 25;
  g_state ^= g_state >> 27;
  return ((g_state * 2685821657736338717ull) >> 11) * (1.0 / 9007199254740992.0);
}

template <typename T>
static T* dev_alloc(size_t count) {
  void* p = nullptr;
  if (cudaMalloc(&p, count * sizeof(T) + 16) != cudaSuccess) return nullptr;
  cudaMemset(p, 0, count * sizeof(T) + 16);
  return static_cast<T*>(p);
}

int main() {
  const int64_t n = 300, d = 64, v = 1000, ig = -100;
  const int64_t nt = (n + 127) / 128, mt = (v + 255) / 256, vpad = mt * 256;
  const float eps = 1.0f / 4096.0f;
  std::vector<__nv_bfloat16> E(n * d), C(v * d);
  std::vector<double> Ef(n * d), Cf(v * d);
  for (int64_t i = 0; i < n * d; ++i) {
    E[i] = __float2bfloat16(static_cast<float>(uniform() * 2.0 - 1.0));
    Ef[i] = __bfloat162float(E[i]);
  }
  for (int64_t i = 0; i < v * d; ++i) {
    C[i] = __float2bfloat16(static_cast<float>((uniform() * 2.0 - 1.0) * 0.6));
    Cf[i] = __bfloat162float(C[i]);
  }
  std::vector<int64_t> x(n);
  int64_t n_valid_h = 0;
  for (int64_t i = 0; i < n; ++i) {
    x[i] = (i % 9 == 4) ? ig : static_cast<int64_t>(uniform() * v);
    n_valid_h += x[i] != ig;
  }
  std::vector<float> up(n);
  for (int64_t i = 0; i < n; ++i) up[i] = x[i] == ig ? 0.f : 1.0f / n_valid_h;  // mean over valid

  // ---- double-precision reference: loss, dE = up (P - onehot) C, dC = (P - onehot)^T up E
  std::vector<double> rloss(n, 0.0), rde(n * d, 0.0), rdc(v * d, 0.0);
  std::vector<double> z(v);
  for (int64_t i = 0; i < n; ++i) {
    if (x[i] == ig) continue;
    double m = -INFINITY, s = 0.0;
    for (int64_t j = 0; j < v; ++j) {
      double a = 0.0;
      for (int64_t k = 0; k < d; ++k) a += Ef[i * d + k] * Cf[j * d + k];
      z[j] = a;
      m = std::fmax(m, a);
    }
    for (int64_t j = 0; j < v; ++j) s += std::exp(z[j] - m);
    const double lse = m + std::log(s);
    rloss[i] = lse - z[x[i]];
    for (int64_t j = 0; j < v; ++j) {
      const double g = up[i] * (std::exp(z[j] - lse) - (j == x[i] ? 1.0 : 0.0));
      for (int64_t k = 0; k < d; ++k) {
        rde[i * d + k] += g * Cf[j * d + k];
        rdc[j * d + k] += g * Ef[i * d + k];
      }
    }
  }

  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  auto* dE = dev_alloc<__nv_bfloat16>(n * d);
  auto* dC = dev_alloc<__nv_bfloat16>(v * d);
  auto* dx = dev_alloc<int64_t>(n);
  auto* dup = dev_alloc<float>(n);
  CK(cudaMemcpy(dE, E.data(), n * d * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dC, C.data(), v * d * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dx, x.data(), n * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dup, up.data(), n * 4, cudaMemcpyHostToDevice));

  // 1. compaction (filter_ignored); rows are ignored, so the kernels read a compacted copy
  auto* row_map = dev_alloc<int32_t>(nt * 128);
  auto* n_valid = dev_alloc<int>(1);
  auto* E_c = dev_alloc<__nv_bfloat16>(n * d);
  CC(cce_compact_rows(dx, ig, n, row_map, n_valid, st));
  CC(cce_gather_rows(dE, row_map, n, d, E_c, st));
  // 2. vocabulary order (compute_vocab_order): mean logits of the valid rows, stable sort
  auto* ebar = dev_alloc<float>(d);
  const size_t ebw = cce_ebar_workspace_bytes(n, d), sow = cce_sort_workspace_bytes(v);
  auto* ws_e = dev_alloc<uint8_t>(ebw);
  auto* ws_s = dev_alloc<uint8_t>(sow);
  auto* perm = dev_alloc<int32_t>(v);
  auto* key = dev_alloc<float>(v);
  CC(cce_ebar(dE, dx, ig, n, d, ebar, ws_e, ebw, st));
  CC(cce_vocab_order(dC, ebar, n_valid, v, d, perm, key, ws_s, sow, st));
  // 3. label positions in tile order and the inverse order
  auto* perm_padded = dev_alloc<int32_t>(vpad);
  auto* inv_perm = dev_alloc<int32_t>(v);
  auto* pos = dev_alloc<int32_t>(n);
  CC(cce_bwd_prep(perm, v, dx, ig, 0, n, perm_padded, inv_perm, pos, st));
  // 4. forward over vocabulary groups of 2 tiles (512 sorted rows): each group's rows gathered,
  //    swept into its (max, sum-exp) partials and its block of the tile maxima; one combine
  const int64_t gv = 512;
  auto* C_g = dev_alloc<__nv_bfloat16>(gv * d);
  auto* tile_max = dev_alloc<float>(cce_tile_max_bytes(n, v) / 4);
  auto* corr = dev_alloc<float>(n);  // zeroed: a label lands in exactly one group
  int total_splits = 0;
  for (int64_t v0 = 0; v0 < v; v0 += gv) total_splits += cce_fwd_splits(n, d, std::min(gv, v - v0));
  auto* parts = dev_alloc<float>((size_t)total_splits * n * 2);
  int off = 0;
  for (int64_t v0 = 0; v0 < v; v0 += gv) {
    const int64_t vg = std::min(gv, v - v0);
    const int sp = cce_fwd_splits(n, d, vg);
    CC(cce_gather_rows(dC, perm + v0, vg, d, C_g, st));
    CC(cce_fwd_group_ex(E_c, 0, C_g, row_map, n_valid, pos, v0, n, d, vg, v, 0.f, parts + (size_t)off * n * 2,
                        (size_t)sp * n * 8, nullptr, corr, tile_max, 3, st));
    off += sp;
  }
  auto* lse_l = dev_alloc<float>(n);
  auto* lse = dev_alloc<float>(n);
  auto* loss = dev_alloc<float>(n);
  CC(cce_combine_parts(parts, off, n, lse_l, st));
  CC(cce_merge_shards(1, lse_l, corr, dx, ig, n, lse, loss, st));
  // 5. streamed backward: 512-slot S-hat ring, the sorted copy in dC's storage (c_sorted == dc)
  const int64_t ring_slots = 512;
  const size_t sw = cce_bwd_stream_workspace_bytes(n, d, v, ring_slots);
  auto* ws_b = dev_alloc<uint8_t>(sw);
  auto* ring = dev_alloc<uint8_t>(ring_slots * 128 * 256 * 2);
  auto* de = dev_alloc<__nv_bfloat16>(n * d);  // zeroed: ignored rows stay 0
  auto* dc = dev_alloc<__nv_bfloat16>(v * d);
  auto* counters = dev_alloc<unsigned long long>(3);
  CC(cce_bwd_stream(E_c, 0, dC, dc, perm_padded, inv_perm, row_map, n_valid, pos, lse, dup, tile_max, n, d, v,
                    0.f, eps, 0, ring, ring_slots, ws_b, sw, de, 0, dc, counters, nullptr, st));
  auto* overflow = dev_alloc<int>(1);  // (no overflow path on the streamed backward)

  std::vector<float> hloss(n);
  std::vector<__nv_bfloat16> hde(n * d), hdc(v * d);
  unsigned long long hk[3];
  int hov = 0;
  CK(cudaMemcpyAsync(hloss.data(), loss, n * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hde.data(), de, n * d * 2, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hdc.data(), dc, v * d * 2, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hk, counters, sizeof(hk), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&hov, overflow, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));

  auto rel = [](const std::vector<double>& ref, auto get, size_t count) {
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < count; ++i) {
      num = std::fmax(num, std::fabs(get(i) - ref[i]));
      den = std::fmax(den, std::fabs(ref[i]));
    }
    return num / std::fmax(den, 1e-30);
  };
  const double e_loss = rel(rloss, [&](size_t i) { return double(hloss[i]); }, n);
  const double e_de = rel(rde, [&](size_t i) { return double(__bfloat162float(hde[i])); }, n * d);
  const double e_dc = rel(rdc, [&](size_t i) { return double(__bfloat162float(hdc[i])); }, v * d);
  std::printf("loss rel %.2e  dE rel %.2e  dC rel %.2e  kept %llu of %lld  overflow %d\n", e_loss, e_de, e_dc,
              hk[0], (long long)(nt * mt), hov);
  if (!(e_loss < 1e-3 && e_de < 1e-2 && e_dc < 1e-2) || hov != 0 || hk[0] != (unsigned long long)(nt * mt)) return 4;
  std::printf("abi bounded training path ok\n");
  return 0;
}

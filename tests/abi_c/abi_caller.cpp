// A plain C++ caller of libcce_b200.so through include/cce_b200.h only (Option C):
// no Python, no torch.  Forward (cce_fwd) + shard merge (cce_merge_shards) on bf16 inputs made on
// the host, checked against a double-precision log-sum-exp computed here; then the error channel.
// Exit code 0 = pass.  Built and run by tests/test_abi_c_gpu.py.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
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

static uint64_t g_state = 0x9E3779B97F4A7C15ull;
static double uniform() {  // xorshift64*: deterministic, no library dependence
  g_state ^= g_state >> 12;
  g_state ^= g_state << 25;
  g_state ^= g_state >> 27;
  return ((g_state * 2685821657736338717ull) >> 11) * (1.0 / 9007199254740992.0);
}

int main() {
  const int64_t n = 300, d = 64, v = 1000, ignore = -100;
  std::vector<__nv_bfloat16> E(n * d), C(v * d);
  std::vector<float> Ef(n * d), Cf(v * d);
  for (int64_t i = 0; i < n * d; ++i) {
    E[i] = __float2bfloat16(static_cast<float>(uniform() * 2.0 - 1.0));
    Ef[i] = __bfloat162float(E[i]);
  }
  for (int64_t i = 0; i < v * d; ++i) {
    C[i] = __float2bfloat16(static_cast<float>((uniform() * 2.0 - 1.0) * 0.5));
    Cf[i] = __bfloat162float(C[i]);
  }
  std::vector<int64_t> x(n);
  for (int64_t i = 0; i < n; ++i) x[i] = (i % 7 == 3) ? ignore : static_cast<int64_t>(uniform() * v);

  // host reference: loss_i = lse_i - z_i,x_i in double (0 at ignored rows)
  std::vector<double> ref(n, 0.0);
  for (int64_t i = 0; i < n; ++i) {
    if (x[i] == ignore) continue;
    double m = -INFINITY, s = 0.0, zt = 0.0;
    std::vector<double> z(v);
    for (int64_t j = 0; j < v; ++j) {
      double a = 0.0;
      for (int64_t k = 0; k < d; ++k) a += double(Ef[i * d + k]) * double(Cf[j * d + k]);
      z[j] = a;
      m = std::fmax(m, a);
    }
    for (int64_t j = 0; j < v; ++j) s += std::exp(z[j] - m);
    zt = z[x[i]];
    ref[i] = m + std::log(s) - zt;
  }

  void *dE, *dC, *dx, *ws, *lse_l, *corr, *lse, *loss;
  const size_t ws_bytes = cce_fwd_workspace_bytes(n, d, v);
  CK(cudaMalloc(&dE, E.size() * 2));
  CK(cudaMalloc(&dC, C.size() * 2));
  CK(cudaMalloc(&dx, n * 8));
  CK(cudaMalloc(&ws, ws_bytes > 0 ? ws_bytes : 16));
  CK(cudaMalloc(&lse_l, n * 4));
  CK(cudaMalloc(&corr, n * 4));
  CK(cudaMalloc(&lse, n * 4));
  CK(cudaMalloc(&loss, n * 4));
  CK(cudaMemcpy(dE, E.data(), E.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dC, C.data(), C.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dx, x.data(), n * 8, cudaMemcpyHostToDevice));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  if (cce_fwd(dE, dC, static_cast<int64_t*>(dx), n, d, v, ignore, 0, 0.f, ws, ws_bytes,
              static_cast<float*>(lse_l), static_cast<float*>(corr), st) != 0) {
    std::fprintf(stderr, "cce_fwd failed: %s\n", cce_last_error());
    return 3;
  }
  if (cce_merge_shards(1, static_cast<float*>(lse_l), static_cast<float*>(corr), static_cast<int64_t*>(dx),
                       ignore, n, static_cast<float*>(lse), static_cast<float*>(loss), st) != 0) {
    std::fprintf(stderr, "cce_merge_shards failed: %s\n", cce_last_error());
    return 3;
  }
  std::vector<float> got(n);
  CK(cudaMemcpyAsync(got.data(), loss, n * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  double worst = 0.0, scale = 1.0;
  for (int64_t i = 0; i < n; ++i) scale = std::fmax(scale, std::fabs(ref[i]));
  for (int64_t i = 0; i < n; ++i) worst = std::fmax(worst, std::fabs(double(got[i]) - ref[i]));
  std::printf("loss max abs err %.3e (scale %.3f)\n", worst, scale);
  if (!(worst <= 1e-3 * scale)) return 4;

  // error channel: D not a multiple of 8 is rejected with a message, nothing launched
  const int rc = cce_fwd(dE, dC, static_cast<int64_t*>(dx), n, 7, v, ignore, 0, 0.f, ws, ws_bytes,
                         static_cast<float*>(lse_l), static_cast<float*>(corr), st);
  const char* msg = cce_last_error();
  std::printf("bad D: rc=%d msg=\"%s\"\n", rc, msg);
  if (rc == 0 || msg == nullptr || std::strstr(msg, "multiple of 8") == nullptr) return 5;
  std::printf("abi caller ok (abi version %d)\n", cce_abi_version());
  return 0;
}

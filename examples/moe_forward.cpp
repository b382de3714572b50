// A C++ program using only the library's C ABI (include/w4a16_moe.h): AWQ tensors of a small MoE layer
// -> packed blocks (w4a16_repack_awq) -> top-k routing (w4a16_route_topk) -> the whole layer
// (w4a16_moe_forward), checked against a plain CPU restatement of the same arithmetic -- dequant
// fp16((q - z) * s), SwiGLU with h rounded to fp16, each expert's down output rounded to fp16, the
// fp32 weighted combine (the conventions of oracle/moe_oracle.py). Then the same layer through the
// expert-parallel entry (w4a16_moe_forward_ep) on a one-rank NCCL communicator, bit for bit.
//
//   make -C examples   (or see tests/test_c_example.py)   ./examples/moe_forward  -> exit 0 when it matches
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "w4a16_moe.h"

namespace {
constexpr int E = 4, TOPK = 2, H = 256, I = 256, T = 5, G = 128;
constexpr int kSlotCol[8] = {0, 2, 4, 6, 1, 3, 5, 7};  // AWQ pack order: slot i holds column kSlotCol[i]

#define CK(x)                                                                                  \
  do {                                                                                         \
    if ((x) != cudaSuccess) { std::fprintf(stderr, "CUDA error at %s:%d\n", __FILE__, __LINE__); std::exit(2); } \
  } while (0)
#define W4(x)                                                                                  \
  do {                                                                                         \
    const int rc_ = (x);                                                                       \
    if (rc_ != W4_OK) { std::fprintf(stderr, "%s -> %d\n", #x, rc_); std::exit(3); }          \
  } while (0)

struct Awq {  // one projection of all experts, AWQ layout: qweight [E][K][N/8], scales / qzeros per group
  int K, N;
  std::vector<uint8_t> q, z;  // logical q[e][n][k], z[e][n][k/G]
  std::vector<float> s;       // s[e][n][k/G] (fp16 values)
  std::vector<int32_t> qweight, qzeros;
  std::vector<__half> scales;
};

Awq make_awq(int K, int N, std::mt19937& rng) {
  Awq a{K, N, {}, {}, {}, {}, {}, {}};
  std::uniform_int_distribution<int> nib(0, 15);
  std::uniform_real_distribution<float> sc(0.5f, 1.5f);
  a.q.resize(size_t(E) * N * K);
  a.z.resize(size_t(E) * N * (K / G));
  a.s.resize(a.z.size());
  for (auto& v : a.q) v = static_cast<uint8_t>(nib(rng));
  for (auto& v : a.z) v = static_cast<uint8_t>(nib(rng));
  for (auto& v : a.s) v = __half2float(__float2half(sc(rng) / 128.f));
  a.qweight.assign(size_t(E) * K * (N / 8), 0);
  a.qzeros.assign(size_t(E) * (K / G) * (N / 8), 0);
  a.scales.resize(size_t(E) * (K / G) * N);
  for (int e = 0; e < E; ++e)
    for (int k = 0; k < K; ++k)
      for (int n8 = 0; n8 < N / 8; ++n8) {
        uint32_t w = 0;
        for (int slot = 0; slot < 8; ++slot) w |= uint32_t(a.q[(size_t(e) * N + n8 * 8 + kSlotCol[slot]) * K + k]) << (4 * slot);
        a.qweight[(size_t(e) * K + k) * (N / 8) + n8] = static_cast<int32_t>(w);
      }
  for (int e = 0; e < E; ++e)
    for (int g = 0; g < K / G; ++g) {
      for (int n8 = 0; n8 < N / 8; ++n8) {
        uint32_t w = 0;
        for (int slot = 0; slot < 8; ++slot)
          w |= uint32_t(a.z[(size_t(e) * N + n8 * 8 + kSlotCol[slot]) * (K / G) + g]) << (4 * slot);
        a.qzeros[(size_t(e) * (K / G) + g) * (N / 8) + n8] = static_cast<int32_t>(w);
      }
      for (int n = 0; n < N; ++n) a.scales[(size_t(e) * (K / G) + g) * N + n] = __float2half(a.s[(size_t(e) * N + n) * (K / G) + g]);
    }
  return a;
}

float deq(const Awq& a, int e, int n, int k) {  // fp16((q - z) * s), the single rounding the kernel pins
  const size_t gi = (size_t(e) * a.N + n) * (a.K / G) + k / G;
  const float v = float(int(a.q[(size_t(e) * a.N + n) * a.K + k]) - int(a.z[gi])) * a.s[gi];
  return __half2float(__float2half(v));
}
float r16(float v) { return __half2float(__float2half(v)); }

template <typename Tp>
Tp* to_dev(const std::vector<Tp>& h) {
  Tp* d = nullptr;
  CK(cudaMalloc(&d, h.size() * sizeof(Tp)));
  CK(cudaMemcpy(d, h.data(), h.size() * sizeof(Tp), cudaMemcpyHostToDevice));
  return d;
}
}  // namespace

int main() {
  std::mt19937 rng(1234);
  Awq w13 = make_awq(H, 2 * I, rng);  // rows [gate (I) | up (I)]
  Awq w2 = make_awq(I, H, rng);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::vector<__half> x(size_t(T) * H);
  std::vector<float> xf(x.size()), logits(size_t(T) * E);
  for (size_t i = 0; i < x.size(); ++i) { x[i] = __float2half(0.5f * nd(rng)); xf[i] = __half2float(x[i]); }
  for (auto& v : logits) v = nd(rng);

  // device: pack, route, run the layer
  uint8_t *d_w13 = nullptr, *d_w2 = nullptr;
  CK(cudaMalloc(&d_w13, w4a16_packed_bytes(E, 2 * I, H)));
  CK(cudaMalloc(&d_w2, w4a16_packed_bytes(E, H, I)));
  int32_t *qw = to_dev(w13.qweight), *qz = to_dev(w13.qzeros);
  __half* sc = to_dev(w13.scales);
  W4(w4a16_repack_awq(qw, sc, qz, E, H, 2 * I, 2, G, d_w13, 0));
  int32_t *qw2 = to_dev(w2.qweight), *qz2 = to_dev(w2.qzeros);
  __half* sc2 = to_dev(w2.scales);
  W4(w4a16_repack_awq(qw2, sc2, qz2, E, I, H, 1, G, d_w2, 0));
  float* d_logits = to_dev(logits);
  __half* d_x = to_dev(x);
  int32_t* d_ids = nullptr;
  float* d_wts = nullptr;
  __half* d_y = nullptr;
  CK(cudaMalloc(&d_ids, sizeof(int32_t) * T * TOPK));
  CK(cudaMalloc(&d_wts, sizeof(float) * T * TOPK));
  CK(cudaMalloc(&d_y, sizeof(__half) * T * H));
  W4(w4a16_route_topk(d_logits, T, E, TOPK, W4_SCORE_SOFTMAX, 1, d_ids, d_wts, 0));
  const int64_t ws_bytes = w4a16_moe_workspace_bytes(T, TOPK, E, H, I);
  void* ws = nullptr;
  CK(cudaMalloc(&ws, ws_bytes));
  CK(cudaMemset(ws, 0, ws_bytes));  // zero once after allocation (the header's workspace contract)
  W4(w4a16_moe_forward(d_x, T, H, I, E, TOPK, d_ids, d_wts, d_w13, d_w2, W4_DTYPE_F16, d_y, ws, ws_bytes, 0));
  CK(cudaDeviceSynchronize());
  std::vector<__half> y(size_t(T) * H);
  std::vector<int32_t> ids(T * TOPK);
  std::vector<float> wts(T * TOPK);
  CK(cudaMemcpy(y.data(), d_y, y.size() * sizeof(__half), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ids.data(), d_ids, ids.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(wts.data(), d_wts, wts.size() * sizeof(float), cudaMemcpyDeviceToHost));

  // CPU restatement: routing (softmax top-k, renormalised) and the layer
  int route_mismatch = 0;
  double max_err = 0.0;
  int bad = 0;
  for (int t = 0; t < T; ++t) {
    std::vector<float> p(E);
    float mx = -INFINITY, sum = 0.f;
    for (int e = 0; e < E; ++e) mx = std::max(mx, logits[size_t(t) * E + e]);
    for (int e = 0; e < E; ++e) sum += (p[e] = std::exp(logits[size_t(t) * E + e] - mx));
    for (auto& v : p) v /= sum;
    std::vector<int> order(E);
    for (int e = 0; e < E; ++e) order[e] = e;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return p[a] > p[b]; });
    float wsum = 0.f;
    for (int j = 0; j < TOPK; ++j) wsum += p[order[j]];
    for (int j = 0; j < TOPK; ++j) {
      route_mismatch += ids[t * TOPK + j] != order[j];
      route_mismatch += std::fabs(wts[t * TOPK + j] - p[order[j]] / wsum) > 1e-5f;
    }
    std::vector<float> acc(H, 0.f);
    for (int j = 0; j < TOPK; ++j) {
      const int e = ids[t * TOPK + j];
      std::vector<float> h(I), out(H);
      for (int i = 0; i < I; ++i) {
        float g = 0.f, u = 0.f;
        for (int k = 0; k < H; ++k) {
          g += xf[size_t(t) * H + k] * deq(w13, e, i, k);
          u += xf[size_t(t) * H + k] * deq(w13, e, I + i, k);
        }
        h[i] = r16(g / (1.f + std::exp(-g)) * u);
      }
      for (int n = 0; n < H; ++n) {
        float o = 0.f;
        for (int i = 0; i < I; ++i) o += h[i] * deq(w2, e, n, i);
        out[n] = r16(o);
      }
      for (int n = 0; n < H; ++n) acc[n] += wts[t * TOPK + j] * out[n];
    }
    for (int n = 0; n < H; ++n) {
      const float want = r16(acc[n]), got = __half2float(y[size_t(t) * H + n]);
      const double err = std::fabs(double(got) - want);
      max_err = std::max(max_err, err);
      bad += err > 1e-2 + 1e-2 * std::fabs(want);
    }
  }
  std::printf("moe_forward: T=%d E=%d k=%d H=%d I=%d  routing mismatches %d  max |diff| %.3g  outside tol %d\n", T,
              E, TOPK, H, I, route_mismatch, max_err, bad);
  int ep_diff = 0;
  if (w4a16_ep_available()) {
    // the expert-parallel entry on a one-rank communicator: all-gather, localize, local experts, fp32
    // partial combine, reduce-scatter and the one rounding -- bit-identical to the single-GPU layer
    unsigned char id[128];
    W4(w4a16_ep_unique_id(id));
    w4a16_ep_comm* comm = nullptr;
    W4(w4a16_ep_comm_init(id, 0, 1, &comm));
    const int64_t ep_bytes = w4a16_moe_ep_workspace_bytes(T, 1, TOPK, E, H, I);
    void* ep_ws = nullptr;
    CK(cudaMalloc(&ep_ws, ep_bytes));
    CK(cudaMemset(ep_ws, 0, ep_bytes));
    __half* d_y_ep = nullptr;
    CK(cudaMalloc(&d_y_ep, sizeof(__half) * T * H));
    W4(w4a16_moe_forward_ep(comm, d_x, T, H, I, E, TOPK, d_ids, d_wts, d_w13, d_w2, W4_DTYPE_F16, d_y_ep, ep_ws,
                            ep_bytes, 0));
    CK(cudaDeviceSynchronize());
    std::vector<__half> y_ep(size_t(T) * H);
    CK(cudaMemcpy(y_ep.data(), d_y_ep, y_ep.size() * sizeof(__half), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < y.size(); ++i) ep_diff += __half_as_ushort(y_ep[i]) != __half_as_ushort(y[i]);
    W4(w4a16_ep_comm_destroy(comm));
    std::printf("moe_forward_ep (1 rank): %d elements differ from moe_forward\n", ep_diff);
  } else {
    std::printf("moe_forward_ep: NCCL not available, skipped\n");
  }
  return (route_mismatch == 0 && bad == 0 && ep_diff == 0) ? 0 : 1;
}

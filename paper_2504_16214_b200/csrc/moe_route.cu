// Routing, permutation, gather and combine kernels for the W4A16 MoE layer (sm_100a), and the
// one-call layer driver. All index outputs are deterministic (no atomics on the output order):
//   * top-k selects on the raw logits (softmax / sigmoid are monotone), ties -> lower expert id;
//   * the permutation is a stable counting sort of flat pair index i = t*k + j by expert id,
//     i.e. rows of one expert appear in (token, slot) order.
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include "ptx.cuh"
#include "launch.cuh"
#include "w4a16_moe.h"

namespace w4 {

// ---------------------------------------------------------------------------------------- top-k
// One warp per token; lane l holds logits l, l+32, ... (kPer per lane = power of two >= E/32, padded
// with -inf). Selection compares raw logits (softmax / sigmoid are monotone), ties -> lower expert id.
// Routes token `tok` (one warp): ids / wts rows of length k.
template <int kPer>
__device__ __forceinline__ void route_token(const float* __restrict__ logits, int tok, int E, int k, int scoring,
                                            int renorm, int32_t* __restrict__ ids, float* __restrict__ wts,
                                            int lane) {
  const int warp = tok;
  const float* row = logits + static_cast<int64_t>(warp) * E;
  float v[kPer];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int e = lane + 32 * i;
    v[i] = e < E ? __ldg(row + e) : -INFINITY;
    mx = fmaxf(mx, v[i]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float denom = 0.f;
  if (scoring == W4_SCORE_SOFTMAX) {
#pragma unroll
    for (int i = 0; i < kPer; ++i) denom += lane + 32 * i < E ? __expf(v[i] - mx) : 0.f;
#pragma unroll
    for (int o = 16; o; o >>= 1) denom += __shfl_xor_sync(0xffffffffu, denom, o);
  }
  float sel_sum = 0.f, my_w = 0.f;
  int my_id = 0;
  uint32_t taken = 0;  // bit i: v[i] already selected (explicit, so -inf logits stay selectable once)
  for (int j = 0; j < k; ++j) {
    float best = -INFINITY;
    int bidx = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {  // lane-local best; ascending i = ascending expert id
      const int e = lane + 32 * i;
      if (e < E && !((taken >> i) & 1u) && (bidx == 0x7fffffff || v[i] > best)) { best = v[i]; bidx = e; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (oi != 0x7fffffff && (bidx == 0x7fffffff || ob > best || (ob == best && oi < bidx))) { best = ob; bidx = oi; }
    }
    if ((bidx & 31) == lane) taken |= 1u << (bidx >> 5);
    const float w = scoring == W4_SCORE_SOFTMAX ? __expf(best - mx) / denom : 1.0f / (1.0f + __expf(-best));
    sel_sum += w;
    if (lane == j) { my_w = w; my_id = bidx; }
  }
  if (lane < k) {
    ids[static_cast<int64_t>(warp) * k + lane] = my_id;
    wts[static_cast<int64_t>(warp) * k + lane] = renorm ? my_w / sel_sum : my_w;
  }
}

template <int kPer>
__global__ void route_topk_kernel(const float* __restrict__ logits, int T, int E, int k, int scoring, int renorm,
                                  int32_t* __restrict__ ids, float* __restrict__ wts) {
  griddep_wait();  // PDL: inputs written by the previous kernel in the stream
  griddep_launch_dependents();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= T) return;
  route_token<kPer>(logits, warp, E, k, scoring, renorm, ids, wts, threadIdx.x & 31);
}

// ------------------------------------------------------------------------------- grouped top-k
// DeepSeek-V3/R1 routing (vLLM grouped_topk, vllm/model_executor/layers/fused_moe/router/
// grouped_topk_router.py:81-162): scores = softmax or sigmoid of the logits; choice = scores + bias
// (e_score_correction_bias, optional); a group's score is the sum of its two best choices (with a
// bias) or its best score (without); the topk_group best groups stay, every other expert is masked;
// the k best remaining choices are selected; weights are the *unbiased* scores of the selected
// experts, optionally renormalised, times routed_scaling_factor. Ties -> lower group / expert id.
// One warp per token; lane l holds experts l, l+32, ... as in route_topk_kernel.
template <int kPer>
__global__ void route_grouped_topk_kernel(const float* __restrict__ logits, int T, int E, int k, int G, int TG,
                                          int scoring, int renorm, const float* __restrict__ bias, float scale,
                                          int32_t* __restrict__ ids, float* __restrict__ wts) {
  griddep_wait();  // PDL: inputs written by the previous kernel in the stream
  griddep_launch_dependents();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= T) return;
  const float* row = logits + static_cast<int64_t>(warp) * E;
  const int gsize = E / G;
  float sc[kPer], ch[kPer];
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int e = lane + 32 * i;
    sc[i] = e < E ? __ldg(row + e) : -INFINITY;
    mx = fmaxf(mx, sc[i]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float denom = 0.f;
  if (scoring == W4_SCORE_SOFTMAX) {
#pragma unroll
    for (int i = 0; i < kPer; ++i) denom += lane + 32 * i < E ? __expf(sc[i] - mx) : 0.f;
#pragma unroll
    for (int o = 16; o; o >>= 1) denom += __shfl_xor_sync(0xffffffffu, denom, o);
  }
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int e = lane + 32 * i;
    if (e < E) {
      sc[i] = scoring == W4_SCORE_SOFTMAX ? __expf(sc[i] - mx) / denom : 1.0f / (1.0f + __expf(-sc[i]));
      ch[i] = bias ? sc[i] + __ldg(bias + e) : sc[i];
    } else {
      ch[i] = -INFINITY;
    }
  }
  // group scores: lane g ends up holding group g's score
  float gscore = -INFINITY;
  for (int g = 0; g < G; ++g) {
    float b1 = -INFINITY, b2 = -INFINITY;  // lane-local best two choices of group g
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = lane + 32 * i;
      if (e < E && e / gsize == g) {
        if (ch[i] > b1) { b2 = b1; b1 = ch[i]; } else if (ch[i] > b2) { b2 = ch[i]; }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {  // merge two sorted pairs
      const float o1 = __shfl_xor_sync(0xffffffffu, b1, o), o2 = __shfl_xor_sync(0xffffffffu, b2, o);
      const float n1 = fmaxf(b1, o1);
      const float n2 = fmaxf(fminf(b1, o1), fmaxf(b2, o2));
      b1 = n1;
      b2 = n2;
    }
    const float gs = bias ? b1 + b2 : b1;
    if (lane == g) gscore = gs;
  }
  // the topk_group best groups (ties -> lower group id) as a bit mask
  uint32_t gmask = 0;
  for (int j = 0; j < TG; ++j) {
    float best = (lane < G && !((gmask >> lane) & 1u)) ? gscore : -INFINITY;
    int bidx = (lane < G && !((gmask >> lane) & 1u)) ? lane : 0x7fffffff;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (oi != 0x7fffffff && (bidx == 0x7fffffff || ob > best || (ob == best && oi < bidx))) { best = ob; bidx = oi; }
    }
    gmask |= 1u << bidx;
  }
  // top-k over the kept experts' choices
  float sel_sum = 0.f, my_w = 0.f;
  int my_id = 0;
  uint32_t taken = 0;
  for (int j = 0; j < k; ++j) {
    float best = -INFINITY;
    int bidx = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = lane + 32 * i;
      if (e < E && ((gmask >> (e / gsize)) & 1u) && !((taken >> i) & 1u) && (bidx == 0x7fffffff || ch[i] > best)) {
        best = ch[i];
        bidx = e;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (oi != 0x7fffffff && (bidx == 0x7fffffff || ob > best || (ob == best && oi < bidx))) { best = ob; bidx = oi; }
    }
    float w = 0.f;  // the selected expert's unbiased score, from its owning lane
#pragma unroll
    for (int i = 0; i < kPer; ++i)
      if (lane + 32 * i == bidx) w = sc[i];
    w = __shfl_sync(0xffffffffu, w, bidx & 31);
    if ((bidx & 31) == lane) taken |= 1u << (bidx >> 5);
    sel_sum += w;
    if (lane == j) { my_w = w; my_id = bidx; }
  }
  if (lane < k) {
    ids[static_cast<int64_t>(warp) * k + lane] = my_id;
    wts[static_cast<int64_t>(warp) * k + lane] = (renorm ? my_w / sel_sum : my_w) * scale;
  }
}

// ---------------------------------------------------------------------------------------- permute
// Single CTA of 1024 threads. Pass 1: histogram (smem atomics; counts are order-independent).
// Pass 2: exclusive scan. Pass 3: walk the pairs in 1024-wide chunks; within a chunk a pair's rank
// among same-expert pairs = (#same in earlier warps) + (#same in lower lanes), so the output order is
// exactly ascending flat index within each expert.
constexpr int kPermThreads = 1024;
constexpr int kPermWarps = kPermThreads / 32;

__device__ __forceinline__ void permute_block(const int32_t* __restrict__ ids, int P, int E,
                                              int32_t* __restrict__ counts, int32_t* __restrict__ offsets,
                                              int32_t* __restrict__ sorted_pairs, int32_t* __restrict__ pair_pos) {
  extern __shared__ int sm[];
  int* cnt = sm;                     // [E]
  int* base = cnt + E;               // [E]
  int* wcnt = base + E;              // [kPermWarps][E]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < E; e += kPermThreads) cnt[e] = 0;
  __syncthreads();
  for (int i = tid; i < P; i += kPermThreads) {
    const int e = ids[i];
    if (e >= 0 && e < E) atomicAdd(&cnt[e], 1);
  }
  __syncthreads();
  if (warp == 0) {
    const int per = (E + 31) / 32;
    const int beg = min(E, lane * per), end = min(E, beg + per);
    int s = 0;
    for (int e = beg; e < end; ++e) s += cnt[e];
    int incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int run = incl - s;
    for (int e = beg; e < end; ++e) {
      base[e] = run;
      offsets[e] = run;
      counts[e] = cnt[e];
      run += cnt[e];
    }
    if (lane == 31) offsets[E] = incl;
  }
  __syncthreads();
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int start = 0; start < P; start += kPermThreads) {
    for (int x = tid; x < kPermWarps * E; x += kPermThreads) wcnt[x] = 0;
    __syncthreads();
    const int i = start + tid;
    int e = i < P ? ids[i] : -1;
    if (e >= E) e = -1;
    const unsigned same = __match_any_sync(0xffffffffu, e);
    const int lrank = __popc(same & lt_mask);
    if (e >= 0 && lrank == 0) wcnt[warp * E + e] = __popc(same);
    __syncthreads();
    if (i < P) {
      if (e >= 0) {
        int pre = 0;
        for (int w = 0; w < warp; ++w) pre += wcnt[w * E + e];
        const int pos = base[e] + pre + lrank;
        sorted_pairs[pos] = i;
        pair_pos[i] = pos;
      } else {
        pair_pos[i] = -1;
      }
    }
    __syncthreads();
    for (int x = tid; x < E; x += kPermThreads) {
      int s = 0;
      for (int w = 0; w < kPermWarps; ++w) s += wcnt[w * E + x];
      base[x] += s;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kPermThreads, 1)
    moe_permute_kernel(const int32_t* __restrict__ ids, int P, int E, int32_t* __restrict__ counts,
                       int32_t* __restrict__ offsets, int32_t* __restrict__ sorted_pairs,
                       int32_t* __restrict__ pair_pos) {
  griddep_wait();  // PDL: inputs written by the previous kernel in the stream
  griddep_launch_dependents();
  permute_block(ids, P, E, counts, offsets, sorted_pairs, pair_pos);
}

// Routing and the permutation in one CTA (small batches): the 32 warps route the tokens, then the
// block permutes the ids it just wrote (block-scope visibility after __syncthreads). One launch and
// one kernel boundary fewer on the decode critical path.
template <int kPer>
__global__ void __launch_bounds__(kPermThreads, 1)
    route_permute_kernel(const float* __restrict__ logits, int T, int E, int k, int scoring, int renorm,
                         int32_t* __restrict__ ids, float* __restrict__ wts, int32_t* __restrict__ counts,
                         int32_t* __restrict__ offsets, int32_t* __restrict__ sorted_pairs,
                         int32_t* __restrict__ pair_pos) {
  griddep_wait();  // PDL: inputs written by the previous kernel in the stream
  griddep_launch_dependents();
  const int warp = threadIdx.x >> 5;
  for (int t = warp; t < T; t += kPermWarps) route_token<kPer>(logits, t, E, k, scoring, renorm, ids, wts, threadIdx.x & 31);
  __syncthreads();
  permute_block(ids, T * k, E, counts, offsets, sorted_pairs, pair_pos);
}

// ---------------------------------------------------------------------------------------- permute (multi-CTA)
// Large P: the pairs are cut into chunks of kChunk; (1) per-chunk expert histograms, (2) one CTA scans
// them in (expert, chunk) order into per-chunk bases, (3) each chunk scatters its pairs with the same
// warp-ranked stable order as the single-CTA kernel. Same output as moe_permute_kernel.
constexpr int kChunk = 2048;

__global__ void __launch_bounds__(512) permute_hist_kernel(const int32_t* __restrict__ ids, int P, int E,
                                                           int32_t* __restrict__ ws) {
  griddep_wait();  // PDL: inputs written by the previous kernel in the stream
  griddep_launch_dependents();
  extern __shared__ int hist[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  const int beg = blockIdx.x * kChunk, end = min(P, beg + kChunk);
  for (int i = beg + threadIdx.x; i < end; i += blockDim.x) {
    const int e = ids[i];
    if (e >= 0 && e < E) atomicAdd(&hist[e], 1);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) ws[static_cast<int64_t>(blockIdx.x) * E + e] = hist[e];
}

// one CTA of 1024 threads; thread e owns expert e (E <= 1024)
__global__ void __launch_bounds__(1024) permute_scan_kernel(int nb, int E, int32_t* __restrict__ ws,
                                                            int32_t* __restrict__ counts,
                                                            int32_t* __restrict__ offsets) {
  griddep_wait();  // PDL: inputs written by the previous kernel in the stream
  griddep_launch_dependents();
  __shared__ int wsum[32];
  const int e = threadIdx.x, lane = e & 31, warp = e >> 5;
  int total = 0;
  if (e < E)
    for (int b = 0; b < nb; ++b) total += ws[static_cast<int64_t>(b) * E + e];
  int incl = total;  // block-wide inclusive scan over experts
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = wsum[lane], wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += v;
    }
    wsum[lane] = wi - w;  // exclusive warp prefix
  }
  __syncthreads();
  const int excl = incl - total + wsum[warp];
  if (e < E) {
    counts[e] = total;
    offsets[e] = excl;
    int run = excl;
    for (int b = 0; b < nb; ++b) {  // per-chunk base of expert e
      const int64_t idx = static_cast<int64_t>(b) * E + e;
      const int c = ws[idx];
      ws[idx] = run;
      run += c;
    }
    if (e == E - 1) offsets[E] = run;
  }
}

__global__ void __launch_bounds__(kPermThreads, 1)
    permute_scatter_kernel(const int32_t* __restrict__ ids, int P, int E, const int32_t* __restrict__ ws,
                           int32_t* __restrict__ sorted_pairs, int32_t* __restrict__ pair_pos) {
  griddep_wait();  // PDL: inputs written by the previous kernel in the stream
  griddep_launch_dependents();
  extern __shared__ int sm[];
  int* base = sm;                    // [E]
  int* wcnt = base + E;              // [kPermWarps][E]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < E; e += kPermThreads) base[e] = ws[static_cast<int64_t>(blockIdx.x) * E + e];
  const unsigned lt_mask = (1u << lane) - 1u;
  const int cbeg = blockIdx.x * kChunk, cend = min(P, cbeg + kChunk);
  for (int start = cbeg; start < cend; start += kPermThreads) {
    for (int x = tid; x < kPermWarps * E; x += kPermThreads) wcnt[x] = 0;
    __syncthreads();
    const int i = start + tid;
    int e = i < cend ? ids[i] : -1;
    if (e >= E) e = -1;
    const unsigned same = __match_any_sync(0xffffffffu, e);
    const int lrank = __popc(same & lt_mask);
    if (e >= 0 && lrank == 0) wcnt[warp * E + e] = __popc(same);
    __syncthreads();
    if (i < cend) {
      if (e >= 0) {
        int pre = 0;
        for (int w = 0; w < warp; ++w) pre += wcnt[w * E + e];
        const int pos = base[e] + pre + lrank;
        sorted_pairs[pos] = i;
        pair_pos[i] = pos;
      } else {
        pair_pos[i] = -1;
      }
    }
    __syncthreads();
    for (int x = tid; x < E; x += kPermThreads) {
      int s2 = 0;
      for (int w = 0; w < kPermWarps; ++w) s2 += wcnt[w * E + x];
      base[x] += s2;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------- EP local order
// Expert parallelism, receiver side: rows arrive grouped by (source rank r, local expert e) with
// counts cnt[r][e]. Produce the local-expert order (stable by source rank, then arrival):
// l_counts[e], l_offsets[E_l+1], l_sorted[p] = arrival row of expert-ordered row p, l_pos[i] = p.
// One CTA; world * E_l <= kEpMaxCells.
constexpr int kEpMaxCells = 4096;  // static smem: 2 x 16 KB of cell arrays

__global__ void __launch_bounds__(1024) ep_local_order_kernel(const int32_t* __restrict__ recv_counts, int world,
                                                              int el, int32_t* __restrict__ l_counts,
                                                              int32_t* __restrict__ l_offsets,
                                                              int32_t* __restrict__ l_sorted,
                                                              int32_t* __restrict__ l_pos) {
  griddep_wait();  // PDL
  __shared__ int cnt[kEpMaxCells];
  __shared__ int arr[kEpMaxCells];  // arrival offset of cell (r, e)
  __shared__ int wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cells = world * el;
  for (int c = tid; c < cells; c += 1024) cnt[c] = recv_counts[c];
  __syncthreads();
  // exclusive scan of cnt in flat (r, e) order -> arrival offsets: thread t owns cells
  // [t*per, (t+1)*per), one block scan over the per-thread sums
  {
    const int per = (cells + 1023) / 1024;
    const int beg = min(cells, tid * per), end = min(cells, beg + per);
    int tsum = 0;
    for (int c = beg; c < end; ++c) tsum += cnt[c];
    int incl = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int w = wsum[lane];
      int wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += t;
      }
      wsum[lane] = wi - w;
    }
    __syncthreads();
    int run = incl - tsum + wsum[warp];
    for (int c = beg; c < end; ++c) {
      arr[c] = run;
      run += cnt[c];
    }
    __syncthreads();
  }
  // per-expert totals and exclusive offsets (thread e), then per-(r, e) expert-order bases
  __shared__ int loff[1024];
  int lc = 0;
  if (tid < el)
    for (int r = 0; r < world; ++r) lc += cnt[r * el + tid];
  int incl = lc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int w = wsum[lane];
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    wsum[lane] = wi - w;
  }
  __syncthreads();
  if (tid < el) {
    const int off = incl - lc + wsum[warp];
    loff[tid] = off;
    l_counts[tid] = lc;
    l_offsets[tid] = off;
    if (tid == el - 1) l_offsets[el] = off + lc;
  }
  __syncthreads();
  // fill: warp w handles cells w, w+32, ...; expert-order base of (r, e) = loff[e] + sum_{r'<r} cnt[r'][e]
  for (int c = warp; c < cells; c += 32) {
    const int r = c / el, e = c - r * el;
    int b = loff[e];
    for (int r2 = 0; r2 < r; ++r2) b += cnt[r2 * el + e];
    const int a0 = arr[c], n = cnt[c];
    for (int j = lane; j < n; j += 32) {
      l_sorted[b + j] = a0 + j;
      l_pos[a0 + j] = b + j;
    }
  }
}

// ---------------------------------------------------------------------------------------- gather
// One CTA per permuted row, 128-bit vectors (H % 8 == 0).
__global__ void moe_gather_kernel(const uint4* __restrict__ x, int64_t hv, int topk,
                                  const int32_t* __restrict__ sorted_pairs, const int32_t* __restrict__ row_limit,
                                  uint4* __restrict__ xp) {
  griddep_wait();  // PDL: inputs written by the previous kernel in the stream
  griddep_launch_dependents();
  const int64_t p = blockIdx.x;
  const int lim = row_limit ? __ldg(row_limit) : 0x7fffffff;
  const int src_row = __ldg(sorted_pairs + p);  // (in flight with the limit's load)
  if (p >= lim) return;
  const uint4* src = x + static_cast<int64_t>(src_row / topk) * hv;
  uint4* dst = xp + p * hv;
  for (int64_t i = threadIdx.x; i < hv; i += blockDim.x) dst[i] = __ldg(src + i);
}

// ---------------------------------------------------------------------------------------- group sums
// Per (quantisation group g of 128 k, row m): C = sum_k c_k x[m,k] and S = sum_k x[m,k] in fp32, where
// c_k is the offset the grouped GEMM's offset-code dequant leaves on weight k (Dq::offset_bits) --
// the decode-mode epilogue subtracts C + z*S. Layout xsum [K/128][ld][2].
template <bool kBF16>
__device__ __forceinline__ void vec_sums(const uint4& v, float& c, float& s) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  c = 0.f;
  s = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {  // elements 2i, 2i+1 of the 8-vector (k % 8 = 2i, 2i+1)
    float a, b;
    if constexpr (kBF16) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
      a = f.x, b = f.y;
    } else {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
      a = f.x, b = f.y;
    }
    const float off = kBF16 ? 128.f : ((i & 1) ? 64.f : 1024.f);  // == Dq<kBF16>::offset_bits(2i)
    s += a + b;
    c = fmaf(off, a + b, c);
  }
}

// One CTA per row, sized to the row (sums_threads: up to 1024 threads, one 16-byte vector each), so
// a row costs one dependent global round trip instead of one per 128 vectors (DS-R1 H=7168: 7 of
// them); the 16 vectors of one group sit on 16 consecutive lanes, reduced with xor shuffles. The
// row limit and the gather index are loaded together. `sorted_pairs` (gather) maps output row ->
// input row.
template <bool kBF16, bool kGather>
__global__ void group_sums_kernel(const uint4* __restrict__ x, int64_t hv, int topk,
                                  const int32_t* __restrict__ sorted_pairs, const int32_t* __restrict__ row_limit,
                                  uint4* __restrict__ xp, int64_t ld, float2* __restrict__ xsum) {
  griddep_wait();  // PDL: inputs written by the previous kernel in the stream
  griddep_launch_dependents();
  const int64_t p = blockIdx.x;
  const int lim = row_limit ? __ldg(row_limit) : 0x7fffffff;
  const int src_row = kGather ? __ldg(sorted_pairs + p) : 0;  // (in flight with the limit's load)
  if (p >= lim) return;
  const uint4* src = kGather ? x + static_cast<int64_t>(src_row / topk) * hv : x + p * hv;
  uint4* dst = kGather ? xp + p * hv : nullptr;
  const int lane = threadIdx.x & 31;
  for (int64_t base = 0; base < hv; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const bool valid = i < hv;
    float c = 0.f, s = 0.f;
    if (valid) {
      const uint4 v = __ldg(src + i);
      if constexpr (kGather) dst[i] = v;
      vec_sums<kBF16>(v, c, s);
    }
#pragma unroll
    for (int o = 8; o; o >>= 1) {
      c += __shfl_xor_sync(0xffffffffu, c, o);
      s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    if (valid && (lane & 15) == 0) xsum[(i >> 4) * ld + p] = make_float2(c, s);
  }
}

// ---------------------------------------------------------------------------------------- combine
template <bool kBF16>
__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if constexpr (kBF16) {
      const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
      const float2 ff = __bfloat1622float2(h);
      f[2 * i] = ff.x, f[2 * i + 1] = ff.y;
    } else {
      const __half2 h = *reinterpret_cast<const __half2*>(&w[i]);
      const float2 ff = __half22float2(h);
      f[2 * i] = ff.x, f[2 * i + 1] = ff.y;
    }
  }
}

template <bool kBF16>
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if constexpr (kBF16) {
      __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    } else {
      __half2 h = __floats2half2_rn(f[2 * i], f[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// grid (T, H/8 / blockDim): each thread owns one 16-byte vector of one token and accumulates the k
// expert rows in slot order in fp32 (enough CTAs to saturate HBM even at decode token counts).
// kF32Out: write the fp32 sums unrounded (y is float [T][H]) -- the per-rank partial that expert
// parallelism reduces across ranks before the one rounding to the activation dtype.
template <bool kBF16, bool kF32Out = false>
__global__ void moe_combine_kernel(const uint4* __restrict__ yp, int64_t hv, int topk,
                                   const int32_t* __restrict__ pair_pos, const float* __restrict__ wts,
                                   void* __restrict__ y) {
  griddep_wait();  // PDL: inputs written by the previous kernel in the stream
  griddep_launch_dependents();
  const int64_t t = blockIdx.x;
  const int64_t i = static_cast<int64_t>(blockIdx.y) * blockDim.x + threadIdx.x;
  constexpr int kMaxK = 32;
  __shared__ int pos[kMaxK];
  __shared__ float wt[kMaxK];
  if (threadIdx.x < topk) {
    pos[threadIdx.x] = pair_pos[t * topk + threadIdx.x];
    wt[threadIdx.x] = wts[t * topk + threadIdx.x];
  }
  __syncthreads();
  if (i >= hv) return;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  // up to 8 expert rows' loads in flight at once, then the fmas in slot order (same sum as one by one)
  for (int j0 = 0; j0 < topk; j0 += 8) {
    uint4 v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int ps = j0 + q < topk ? pos[j0 + q] : -1;
      v[q] = ps >= 0 ? __ldg(yp + static_cast<int64_t>(ps) * hv + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (j0 + q < topk && pos[j0 + q] >= 0) {
        float f[8];
        unpack8<kBF16>(v[q], f);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = fmaf(wt[j0 + q], f[e], acc[e]);
      }
    }
  }
  if constexpr (kF32Out) {
    float4* o = static_cast<float4*>(y) + 2 * (t * hv + i);
    o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  } else {
    static_cast<uint4*>(y)[t * hv + i] = pack8<kBF16>(acc);
  }
}

}  // namespace w4

using namespace w4;

namespace {
inline int64_t align256(int64_t b) { return (b + 255) & ~int64_t(255); }
// threads per group_sums CTA: the row's 16-byte vectors rounded up to a warp, at most 1024
inline int sums_threads(int64_t hv) { return static_cast<int>(std::min<int64_t>(1024, (hv + 31) / 32 * 32)); }
// the GEMMs' workspace for the picked token tile or a forced decode (16-token) one, whichever is larger
int64_t splitk_bytes(int64_t P, int64_t E, int64_t H, int64_t I) {
  int64_t m = 0;
  for (const int nt : {w4a16_pick_ntok(P, E), 16}) {
    const int64_t a = w4a16_grouped_gemm_ws_bytes(P, H, E, I, 1, nt), b = w4a16_grouped_gemm_ws_bytes(P, I, E, H, 0, nt);
    m = std::max(m, std::max(a, b));
  }
  return m;
}
}  // namespace

extern "C" {

int w4a16_route_topk(const float* logits, int64_t T, int64_t E, int64_t k, int scoring, int renormalize,
                     int32_t* topk_ids, float* topk_weights, cudaStream_t stream) {
  if (E <= 0 || E > 1024 || k <= 0 || k > 32 || k > E) return W4_ERR_SHAPE;
  if (scoring != W4_SCORE_SOFTMAX && scoring != W4_SCORE_SIGMOID) return W4_ERR_ARG;
  if (T <= 0) return W4_OK;  // empty batch: nothing to read or write (pointers may be null)
  if (!logits || !topk_ids || !topk_weights) return W4_ERR_ARG;
  const int thr = 128;
  const int64_t blocks = (T * 32 + thr - 1) / thr;
  const int per = static_cast<int>((E + 31) / 32);
#define W4_ROUTE(P)                                                                                             \
  launch_pdl(route_topk_kernel<P>, blocks, thr, 0, stream, logits, (int)T, (int)E, (int)k, scoring, renormalize, topk_ids, \
                                                   topk_weights)
  if (per <= 1) W4_ROUTE(1);
  else if (per <= 2) W4_ROUTE(2);
  else if (per <= 4) W4_ROUTE(4);
  else if (per <= 8) W4_ROUTE(8);
  else if (per <= 16) W4_ROUTE(16);
  else W4_ROUTE(32);
#undef W4_ROUTE
  return cudaGetLastError() == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}

int w4a16_route_permute(const float* logits, int64_t T, int64_t E, int64_t k, int scoring, int renormalize,
                        int32_t* topk_ids, float* topk_weights, int32_t* expert_counts, int32_t* expert_offsets,
                        int32_t* sorted_pairs, int32_t* pair_pos, cudaStream_t stream) {
  if (!expert_counts || !expert_offsets ||
      (T > 0 && (!logits || !topk_ids || !topk_weights || !sorted_pairs || !pair_pos)))
    return W4_ERR_ARG;
  if (E <= 0 || E > 1024 || k <= 0 || k > 32 || k > E) return W4_ERR_SHAPE;
  if (T < 0 || T * k > (int64_t(1) << 20)) return W4_ERR_SHAPE;
  if (scoring != W4_SCORE_SOFTMAX && scoring != W4_SCORE_SIGMOID) return W4_ERR_ARG;
  const size_t smem = sizeof(int) * (2 * E + kPermWarps * E);
  const int per = static_cast<int>((E + 31) / 32);
#define W4_RPERM(P)                                                                                         \
  do {                                                                                                      \
    static std::atomic<unsigned long long> attr{0};                                                         \
    if (!ensure_smem_attr(route_permute_kernel<P>, sizeof(int) * (2 * 1024 + kPermWarps * 1024), attr))     \
      return W4_ERR_CUDA;                                                                                   \
    launch_pdl(route_permute_kernel<P>, 1, kPermThreads, smem, stream, logits, (int)T, (int)E, (int)k, scoring, \
               renormalize, topk_ids, topk_weights, expert_counts, expert_offsets, sorted_pairs, pair_pos);  \
  } while (0)
  if (per <= 1) W4_RPERM(1);
  else if (per <= 2) W4_RPERM(2);
  else if (per <= 4) W4_RPERM(4);
  else if (per <= 8) W4_RPERM(8);
  else if (per <= 16) W4_RPERM(16);
  else W4_RPERM(32);
#undef W4_RPERM
  return cudaGetLastError() == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}

int w4a16_route_grouped_topk(const float* logits, int64_t T, int64_t E, int64_t k, int64_t num_groups,
                             int64_t topk_group, int scoring, int renormalize, const float* bias,
                             float routed_scaling_factor, int32_t* topk_ids, float* topk_weights, cudaStream_t stream) {
  if (T > 0 && (!logits || !topk_ids || !topk_weights)) return W4_ERR_ARG;
  if (E <= 0 || E > 1024 || k <= 0 || k > 32 || k > E) return W4_ERR_SHAPE;
  if (num_groups <= 0 || num_groups > 32 || E % num_groups || topk_group <= 0 || topk_group > num_groups)
    return W4_ERR_SHAPE;
  if (topk_group * (E / num_groups) < k) return W4_ERR_SHAPE;  // fewer kept experts than k
  if (bias && E / num_groups < 2) return W4_ERR_SHAPE;         // group score = sum of the best two
  if (scoring != W4_SCORE_SOFTMAX && scoring != W4_SCORE_SIGMOID) return W4_ERR_ARG;
  if (T <= 0) return W4_OK;
  const int thr = 128;
  const int64_t blocks = (T * 32 + thr - 1) / thr;
  const int per = static_cast<int>((E + 31) / 32);
#define W4_GROUTE(P)                                                                                        \
  launch_pdl(route_grouped_topk_kernel<P>, blocks, thr, 0, stream, logits, (int)T, (int)E, (int)k, (int)num_groups, \
             (int)topk_group, scoring, renormalize, bias, routed_scaling_factor, topk_ids, topk_weights)
  if (per <= 1) W4_GROUTE(1);
  else if (per <= 2) W4_GROUTE(2);
  else if (per <= 4) W4_GROUTE(4);
  else if (per <= 8) W4_GROUTE(8);
  else if (per <= 16) W4_GROUTE(16);
  else W4_GROUTE(32);
#undef W4_GROUTE
  return cudaGetLastError() == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}

int w4a16_moe_permute(const int32_t* topk_ids, int64_t P, int64_t E, int32_t* expert_counts,
                      int32_t* expert_offsets, int32_t* sorted_pairs, int32_t* pair_pos, cudaStream_t stream) {
  // P == 0: no pair is read or written (those pointers may be null); counts / offsets are still zeroed
  if (!expert_counts || !expert_offsets || (P > 0 && (!topk_ids || !sorted_pairs || !pair_pos))) return W4_ERR_ARG;
  if (E <= 0 || E > 1024 || P < 0 || P > (int64_t(1) << 30)) return W4_ERR_SHAPE;
  const size_t smem = sizeof(int) * (2 * E + kPermWarps * E);
  static std::atomic<unsigned long long> attr{0};
  if (!ensure_smem_attr(moe_permute_kernel, sizeof(int) * (2 * 1024 + kPermWarps * 1024), attr)) return W4_ERR_CUDA;
  launch_pdl(moe_permute_kernel, 1, kPermThreads, smem, stream, topk_ids, (int)P, (int)E, expert_counts, expert_offsets,
                                                         sorted_pairs, pair_pos);
  return cudaGetLastError() == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}

int64_t w4a16_moe_permute_ws_bytes(int64_t P, int64_t E) {
  return 4 * ((P + kChunk - 1) / kChunk) * E;
}

int w4a16_moe_permute_ws(const int32_t* topk_ids, int64_t P, int64_t E, int32_t* expert_counts,
                         int32_t* expert_offsets, int32_t* sorted_pairs, int32_t* pair_pos, void* ws,
                         int64_t ws_bytes, cudaStream_t stream) {
  // largest P for the one-CTA kernel (W4A16_PERMUTE_SINGLE_MAX overrides). Measured in a graph
  // (tools/perm_probe.py): one CTA 8.3 us vs 9.9 at P = 2048, 14.0 vs 10.1 at P = 4096.
  static const int64_t single_max = [] {
    const char* e = getenv("W4A16_PERMUTE_SINGLE_MAX");
    return e ? static_cast<int64_t>(atoll(e)) : static_cast<int64_t>(kChunk);
  }();
  if (!ws || ws_bytes < w4a16_moe_permute_ws_bytes(P, E) || P <= single_max)
    return w4a16_moe_permute(topk_ids, P, E, expert_counts, expert_offsets, sorted_pairs, pair_pos, stream);
  if (!topk_ids || !expert_counts || !expert_offsets || !sorted_pairs || !pair_pos) return W4_ERR_ARG;
  if (E <= 0 || E > 1024 || P > (int64_t(1) << 30)) return W4_ERR_SHAPE;
  const int nb = static_cast<int>((P + kChunk - 1) / kChunk);
  int32_t* w = static_cast<int32_t*>(ws);
  static std::atomic<unsigned long long> attr{0};
  if (!ensure_smem_attr(permute_scatter_kernel, sizeof(int) * (1024 + kPermWarps * 1024), attr)) return W4_ERR_CUDA;
  launch_pdl(permute_hist_kernel, nb, 512, sizeof(int) * E, stream, topk_ids, (int)P, (int)E, w);
  launch_pdl(permute_scan_kernel, 1, 1024, 0, stream, nb, (int)E, w, expert_counts, expert_offsets);
  launch_pdl(permute_scatter_kernel, nb, kPermThreads, sizeof(int) * (E + kPermWarps * E), stream, 
      topk_ids, (int)P, (int)E, w, sorted_pairs, pair_pos);
  return cudaGetLastError() == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}

int w4a16_ep_local_order(const int32_t* recv_counts, int64_t world, int64_t local_experts, int32_t* l_counts,
                         int32_t* l_offsets, int32_t* l_sorted, int32_t* l_pos, cudaStream_t stream) {
  if (!recv_counts || !l_counts || !l_offsets || !l_sorted || !l_pos) return W4_ERR_ARG;
  if (world <= 0 || local_experts <= 0 || local_experts > 1024 || world * local_experts > kEpMaxCells)
    return W4_ERR_SHAPE;
  launch_pdl(ep_local_order_kernel, 1, 1024, 0, stream, recv_counts, (int)world, (int)local_experts, l_counts,
             l_offsets, l_sorted, l_pos);
  return cudaGetLastError() == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}

int w4a16_moe_gather(const void* x, int64_t H, int64_t topk, const int32_t* sorted_pairs, int64_t rows,
                     const int32_t* row_limit, void* x_perm, cudaStream_t stream) {
  if (!x || !sorted_pairs || !x_perm) return W4_ERR_ARG;
  if (H <= 0 || H % 8 || topk <= 0) return W4_ERR_SHAPE;
  if (rows <= 0) return W4_OK;
  launch_pdl(moe_gather_kernel, rows, 128, 0, stream, static_cast<const uint4*>(x), H / 8, (int)topk, sorted_pairs,
                                               row_limit, static_cast<uint4*>(x_perm));
  return cudaGetLastError() == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}

int w4a16_moe_gather_sums(const void* x, int64_t H, int64_t topk, const int32_t* sorted_pairs, int64_t rows,
                          const int32_t* row_limit, void* x_perm, int dtype, float* xsum, cudaStream_t stream) {
  if (!x || !sorted_pairs || !x_perm || !xsum) return W4_ERR_ARG;
  if (H <= 0 || H % 128 || topk <= 0) return W4_ERR_SHAPE;
  if (rows <= 0) return W4_OK;
  const int64_t ld = w4a16_group_sums_ld(rows);
  auto* xs = reinterpret_cast<float2*>(xsum);
  if (dtype == W4_DTYPE_BF16)
    launch_pdl(group_sums_kernel<true, true>, rows, sums_threads(H / 8), 0, stream, static_cast<const uint4*>(x), H / 8, (int)topk,
                                                            sorted_pairs, row_limit, static_cast<uint4*>(x_perm), ld, xs);
  else if (dtype == W4_DTYPE_F16)
    launch_pdl(group_sums_kernel<false, true>, rows, sums_threads(H / 8), 0, stream, static_cast<const uint4*>(x), H / 8, (int)topk,
                                                             sorted_pairs, row_limit, static_cast<uint4*>(x_perm), ld, xs);
  else
    return W4_ERR_DTYPE;
  return cudaGetLastError() == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}

int w4a16_group_sums(const void* x, int64_t rows, int64_t K, const int32_t* row_limit, int dtype, float* xsum,
                     cudaStream_t stream) {
  if (!x || !xsum) return W4_ERR_ARG;
  if (K <= 0 || K % 128) return W4_ERR_SHAPE;
  if (rows <= 0) return W4_OK;
  const int64_t ld = w4a16_group_sums_ld(rows);
  auto* xs = reinterpret_cast<float2*>(xsum);
  if (dtype == W4_DTYPE_BF16)
    launch_pdl(group_sums_kernel<true, false>, rows, sums_threads(K / 8), 0, stream, static_cast<const uint4*>(x), K / 8, 1, nullptr,
                                                             row_limit, nullptr, ld, xs);
  else if (dtype == W4_DTYPE_F16)
    launch_pdl(group_sums_kernel<false, false>, rows, sums_threads(K / 8), 0, stream, static_cast<const uint4*>(x), K / 8, 1, nullptr,
                                                              row_limit, nullptr, ld, xs);
  else
    return W4_ERR_DTYPE;
  return cudaGetLastError() == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}

}  // extern "C"

namespace {
template <bool kF32Out>
int combine_launch(const void* y_perm, int64_t T, int64_t H, int64_t topk, const int32_t* pair_pos,
                   const float* topk_weights, int dtype, void* y, cudaStream_t stream) {
  if (!y_perm || !pair_pos || !topk_weights || !y) return W4_ERR_ARG;
  if (H <= 0 || H % 8 || topk <= 0 || topk > 32) return W4_ERR_SHAPE;
  if (T <= 0) return W4_OK;
  const int thr = 128;
  const dim3 grid(static_cast<unsigned>(T), static_cast<unsigned>((H / 8 + thr - 1) / thr));
  if (dtype == W4_DTYPE_BF16)
    launch_pdl(moe_combine_kernel<true, kF32Out>, grid, thr, 0, stream, static_cast<const uint4*>(y_perm), H / 8,
               (int)topk, pair_pos, topk_weights, y);
  else if (dtype == W4_DTYPE_F16)
    launch_pdl(moe_combine_kernel<false, kF32Out>, grid, thr, 0, stream, static_cast<const uint4*>(y_perm), H / 8,
               (int)topk, pair_pos, topk_weights, y);
  else
    return W4_ERR_DTYPE;
  return cudaGetLastError() == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}
}  // namespace

extern "C" {

int w4a16_moe_combine(const void* y_perm, int64_t T, int64_t H, int64_t topk, const int32_t* pair_pos,
                      const float* topk_weights, int dtype, void* y, cudaStream_t stream) {
  return combine_launch<false>(y_perm, T, H, topk, pair_pos, topk_weights, dtype, y, stream);
}

int w4a16_moe_combine_f32(const void* y_perm, int64_t T, int64_t H, int64_t topk, const int32_t* pair_pos,
                          const float* topk_weights, int dtype, float* y, cudaStream_t stream) {
  return combine_launch<true>(y_perm, T, H, topk, pair_pos, topk_weights, dtype, y, stream);
}

int64_t w4a16_moe_workspace_bytes(int64_t T, int64_t topk, int64_t E, int64_t H, int64_t I) {
  const int64_t P = T * topk;
  const int64_t ld = w4a16_group_sums_ld(P);
  return align256(4 * E) + align256(4 * (E + 1)) + 2 * align256(4 * P) + align256(2 * P * H) +
         align256(2 * P * I) + align256(2 * P * H) + align256(8 * ld * (H / 128)) + align256(8 * ld * (I / 128)) +
         align256(w4a16_moe_permute_ws_bytes(P, E)) + align256(splitk_bytes(P, E, H, I));
}

}  // extern "C"

namespace {
// ntok: the token tile (0 = w4a16_pick_ntok(T * topk, E))
int moe_forward_impl(const void* x, int64_t T, int64_t H, int64_t I, int64_t E, int64_t topk,
                     const int32_t* topk_ids, const float* topk_weights, const uint8_t* w13, const uint8_t* w2,
                     int dtype, void* y, bool f32_out, int ntok, void* workspace, int64_t workspace_bytes,
                     cudaStream_t stream) {
  if (!x || !topk_ids || !topk_weights || !w13 || !w2 || !y || !workspace) return W4_ERR_ARG;
  if (workspace_bytes < w4a16_moe_workspace_bytes(T, topk, E, H, I)) return W4_ERR_WORKSPACE;
  if (T <= 0) return W4_OK;
  if (H % 128 || I % 128) return W4_ERR_SHAPE;
  const int64_t P = T * topk;
  const int64_t ld = w4a16_group_sums_ld(P);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  void* kws = ws;  // the GEMMs' (split-K) workspace first
  const int64_t kws_bytes = align256(splitk_bytes(P, E, H, I));
  ws += kws_bytes;
  int32_t* counts = reinterpret_cast<int32_t*>(ws); ws += align256(4 * E);
  int32_t* offsets = reinterpret_cast<int32_t*>(ws); ws += align256(4 * (E + 1));
  int32_t* sorted = reinterpret_cast<int32_t*>(ws); ws += align256(4 * P);
  int32_t* pos = reinterpret_cast<int32_t*>(ws); ws += align256(4 * P);
  void* xp = ws; ws += align256(2 * P * H);
  void* hp = ws; ws += align256(2 * P * I);
  void* yp = ws; ws += align256(2 * P * H);
  float* xsum = reinterpret_cast<float*>(ws); ws += align256(8 * ld * (H / 128));
  float* hsum = reinterpret_cast<float*>(ws); ws += align256(8 * ld * (I / 128));
  void* pws = ws;
  int rc;
  if ((rc = w4a16_moe_permute_ws(topk_ids, P, E, counts, offsets, sorted, pos, pws,
                                 w4a16_moe_permute_ws_bytes(P, E), stream)))
    return rc;
  const int nt = ntok > 0 ? ntok : w4a16_pick_ntok(P, E);
  const bool decode = nt <= w4a16_decode_max_ntok();  // offset-code GEMMs need the per-group activation sums
  if (decode) {
    if ((rc = w4a16_moe_gather_sums(x, H, topk, sorted, P, offsets + E, xp, dtype, xsum, stream))) return rc;
  } else if ((rc = w4a16_moe_gather(x, H, topk, sorted, P, offsets + E, xp, stream))) {
    return rc;
  }
  if ((rc = w4a16_grouped_gemm_ws(xp, P, H, w13, E, I, 1, counts, offsets, decode ? xsum : nullptr,
                                  decode ? hsum : nullptr, nullptr, hp, dtype, nt, kws, kws_bytes, stream)))
    return rc;
  if ((rc = w4a16_grouped_gemm_ws(hp, P, I, w2, E, H, 0, counts, offsets, decode ? hsum : nullptr, nullptr, nullptr,
                                  yp, dtype, nt, kws, kws_bytes, stream)))
    return rc;
  return f32_out ? w4a16_moe_combine_f32(yp, T, H, topk, pos, topk_weights, dtype, static_cast<float*>(y), stream)
                 : w4a16_moe_combine(yp, T, H, topk, pos, topk_weights, dtype, y, stream);
}
}  // namespace

extern "C" {

int w4a16_moe_forward(const void* x, int64_t T, int64_t H, int64_t I, int64_t E, int64_t topk,
                      const int32_t* topk_ids, const float* topk_weights, const uint8_t* w13,
                      const uint8_t* w2, int dtype, void* y, void* workspace, int64_t workspace_bytes,
                      cudaStream_t stream) {
  return moe_forward_impl(x, T, H, I, E, topk, topk_ids, topk_weights, w13, w2, dtype, y, false, 0, workspace,
                          workspace_bytes, stream);
}

int w4a16_moe_forward_f32(const void* x, int64_t T, int64_t H, int64_t I, int64_t E, int64_t topk,
                          const int32_t* topk_ids, const float* topk_weights, const uint8_t* w13,
                          const uint8_t* w2, int dtype, float* y, int ntok, void* workspace, int64_t workspace_bytes,
                          cudaStream_t stream) {
  return moe_forward_impl(x, T, H, I, E, topk, topk_ids, topk_weights, w13, w2, dtype, y, true, ntok, workspace,
                          workspace_bytes, stream);
}

}  // extern "C"

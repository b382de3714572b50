// Expert parallelism for the W4A16 MoE layer over NCCL (NVLink / NVSwitch), with no host
// synchronisation and fixed shapes, so the whole EP layer can be captured in a CUDA graph.
//
// Dispatch is an all-gather and combine a reduce-scatter (the "all-gather dispatcher"):
//
//   1. all-gather x [T][H], topk_ids [T][k] and topk_weights [T][k] of every rank (one NCCL group)
//      -> the node's whole batch, [world * T] tokens, on every rank;
//   2. keep the pairs routed to this rank's experts [base, base + E_local) (ep_localize: other ids
//      become -1, which the permutation drops);
//   3. run the single-GPU layer on those pairs (permute -> gather -> gate/up -> down) and combine
//      each token's local experts in fp32 WITHOUT rounding (w4a16_moe_forward_f32);
//   4. reduce-scatter the fp32 partial sums (sum over ranks) -> this rank's T tokens, then round once
//      to the activation dtype (ep_finalize).
//
// Why this shape on a B200 node: NVSwitch gives every GPU full bandwidth to every peer and NCCL runs
// all-gather / reduce-scatter with in-switch (NVLS) multicast and reduction, the data moved per rank
// (world*T*H act in, world*T*H fp32 out) equals the all-to-all's T*k rows for top-k = world (DS-R1 on 8
// GPUs), no count exchange or host read-back is needed (all-to-all-v needs its split sizes on the
// host), and the result is summed in fp32 and rounded once, like the single-GPU combine.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2": the one torch already loaded, or the system's),
// so the library loads -- and everything but EP works -- without it.
#include <dlfcn.h>
#include <nccl.h>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>
#include <cstring>
#include <mutex>

#include "launch.cuh"
#include "w4a16_moe.h"

struct w4a16_ep_comm {
  ncclComm_t comm;
  int rank;
  int world;
  bool owned;  // created by w4a16_ep_comm_init (destroyed with the handle) vs borrowed
};

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*comm_user_rank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                 cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // already in the process?
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define W4_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
    W4_SYM(get_unique_id, "ncclGetUniqueId");
    W4_SYM(comm_init_rank, "ncclCommInitRank");
    W4_SYM(comm_destroy, "ncclCommDestroy");
    W4_SYM(comm_count, "ncclCommCount");
    W4_SYM(comm_user_rank, "ncclCommUserRank");
    W4_SYM(all_gather, "ncclAllGather");
    W4_SYM(reduce_scatter, "ncclReduceScatter");
    W4_SYM(group_start, "ncclGroupStart");
    W4_SYM(group_end, "ncclGroupEnd");
#undef W4_SYM
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.comm_count && api.comm_user_rank &&
             api.all_gather && api.reduce_scatter && api.group_start && api.group_end;
  });
  return api;
}

inline int64_t align256(int64_t b) { return (b + 255) & ~int64_t(255); }

// ids -> local expert ids: id - base when it falls in [0, e_local), else -1 (dropped by the permutation)
__global__ void ep_localize_kernel(const int32_t* __restrict__ ids, int64_t n, int32_t base, int32_t e_local,
                                   int32_t* __restrict__ out) {
  w4::griddep_wait();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t l = ids[i] - base;
    out[i] = (l >= 0 && l < e_local) ? l : -1;
  }
}

// y[i] = act(acc[i]) for 8 consecutive elements per thread (fp32 sums -> one rounding)
template <bool kBF16>
__global__ void ep_finalize_kernel(const float4* __restrict__ acc, int64_t n8, uint4* __restrict__ y) {
  w4::griddep_wait();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 a = acc[2 * i], b = acc[2 * i + 1];
    uint32_t w[4];
    if constexpr (kBF16) {
      const __nv_bfloat162 h[4] = {__floats2bfloat162_rn(a.x, a.y), __floats2bfloat162_rn(a.z, a.w),
                                   __floats2bfloat162_rn(b.x, b.y), __floats2bfloat162_rn(b.z, b.w)};
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = *reinterpret_cast<const uint32_t*>(&h[q]);
    } else {
      const __half2 h[4] = {__floats2half2_rn(a.x, a.y), __floats2half2_rn(a.z, a.w), __floats2half2_rn(b.x, b.y),
                            __floats2half2_rn(b.z, b.w)};
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = *reinterpret_cast<const uint32_t*>(&h[q]);
    }
    y[i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

int grid_for(int64_t n, int thr) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + thr - 1) / thr;
  const int64_t cap = static_cast<int64_t>(sms) * 8;
  return static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

extern "C" {

int w4a16_ep_available(void) { return nccl().ok ? 1 : 0; }

int w4a16_ep_unique_id(void* id) {
  if (!id) return W4_ERR_ARG;
  if (!nccl().ok) return W4_ERR_NCCL;
  ncclUniqueId u;
  if (nccl().get_unique_id(&u) != ncclSuccess) return W4_ERR_NCCL;
  memcpy(id, &u, sizeof(u));
  return W4_OK;
}

int w4a16_ep_comm_init(const void* id, int rank, int world, w4a16_ep_comm** out) {
  if (!id || !out || world < 1 || rank < 0 || rank >= world) return W4_ERR_ARG;
  if (!nccl().ok) return W4_ERR_NCCL;
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  if (nccl().comm_init_rank(&c, world, u, rank) != ncclSuccess) return W4_ERR_NCCL;
  *out = new w4a16_ep_comm{c, rank, world, true};
  return W4_OK;
}

int w4a16_ep_comm_wrap(void* nccl_comm, w4a16_ep_comm** out) {
  if (!nccl_comm || !out) return W4_ERR_ARG;
  if (!nccl().ok) return W4_ERR_NCCL;
  ncclComm_t c = static_cast<ncclComm_t>(nccl_comm);
  int n = 0, r = 0;
  if (nccl().comm_count(c, &n) != ncclSuccess || nccl().comm_user_rank(c, &r) != ncclSuccess) return W4_ERR_NCCL;
  *out = new w4a16_ep_comm{c, r, n, false};
  return W4_OK;
}

int w4a16_ep_comm_destroy(w4a16_ep_comm* comm) {
  if (!comm) return W4_ERR_ARG;
  int rc = W4_OK;
  if (comm->owned && nccl().comm_destroy(comm->comm) != ncclSuccess) rc = W4_ERR_NCCL;
  delete comm;
  return rc;
}

int w4a16_ep_comm_rank(const w4a16_ep_comm* comm) { return comm ? comm->rank : W4_ERR_ARG; }
int w4a16_ep_comm_size(const w4a16_ep_comm* comm) { return comm ? comm->world : W4_ERR_ARG; }

int w4a16_ep_dispatch(w4a16_ep_comm* comm, const void* x, const int32_t* topk_ids, const float* topk_weights,
                      int64_t T, int64_t H, int64_t topk, int dtype, void* x_all, int32_t* ids_all, float* w_all,
                      cudaStream_t stream) {
  if (!comm || !x_all || !ids_all || !w_all || (T > 0 && (!x || !topk_ids || !topk_weights))) return W4_ERR_ARG;
  if (dtype != W4_DTYPE_F16 && dtype != W4_DTYPE_BF16) return W4_ERR_DTYPE;
  if (T < 0 || H <= 0 || topk <= 0) return W4_ERR_SHAPE;
  if (T == 0) return W4_OK;  // every rank passes the same T (fixed-shape collectives)
  const NcclApi& n = nccl();
  const ncclDataType_t act = dtype == W4_DTYPE_BF16 ? ncclBfloat16 : ncclFloat16;
  bool ok = n.group_start() == ncclSuccess;
  ok = ok && n.all_gather(x, x_all, static_cast<size_t>(T * H), act, comm->comm, stream) == ncclSuccess;
  ok = ok && n.all_gather(topk_ids, ids_all, static_cast<size_t>(T * topk), ncclInt32, comm->comm, stream) ==
                 ncclSuccess;
  ok = ok && n.all_gather(topk_weights, w_all, static_cast<size_t>(T * topk), ncclFloat32, comm->comm, stream) ==
                 ncclSuccess;
  ok = (n.group_end() == ncclSuccess) && ok;
  return ok ? W4_OK : W4_ERR_NCCL;
}

int w4a16_ep_localize(const int32_t* ids, int64_t n, int64_t expert_base, int64_t local_experts, int32_t* ids_local,
                      cudaStream_t stream) {
  if (n <= 0) return W4_OK;
  if (!ids || !ids_local) return W4_ERR_ARG;
  if (local_experts <= 0 || expert_base < 0) return W4_ERR_SHAPE;
  w4::launch_pdl(ep_localize_kernel, grid_for(n, 256), 256, 0, stream, ids, n, static_cast<int32_t>(expert_base),
                 static_cast<int32_t>(local_experts), ids_local);
  return cudaGetLastError() == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}

int w4a16_ep_combine(w4a16_ep_comm* comm, const float* partial, int64_t T, int64_t H, int dtype, float* reduced,
                     void* y, cudaStream_t stream) {
  if (!comm || (T > 0 && (!partial || !reduced || !y))) return W4_ERR_ARG;
  if (dtype != W4_DTYPE_F16 && dtype != W4_DTYPE_BF16) return W4_ERR_DTYPE;
  if (T < 0 || H <= 0 || H % 8) return W4_ERR_SHAPE;
  if (T == 0) return W4_OK;
  if (nccl().reduce_scatter(partial, reduced, static_cast<size_t>(T * H), ncclFloat32, ncclSum, comm->comm,
                            stream) != ncclSuccess)
    return W4_ERR_NCCL;
  const int64_t n8 = T * H / 8;
  if (dtype == W4_DTYPE_BF16)
    w4::launch_pdl(ep_finalize_kernel<true>, grid_for(n8, 256), 256, 0, stream,
                   reinterpret_cast<const float4*>(reduced), n8, static_cast<uint4*>(y));
  else
    w4::launch_pdl(ep_finalize_kernel<false>, grid_for(n8, 256), 256, 0, stream,
                   reinterpret_cast<const float4*>(reduced), n8, static_cast<uint4*>(y));
  return cudaGetLastError() == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}

// Token tile of the local GEMMs: sized for the pairs expected on this rank (1/world of the node's
// pairs under uniform routing), not for the node batch -- most gathered ids are other ranks' (-1).
int ep_ntok(int64_t T, int64_t world, int64_t topk, int64_t local_experts) {
  return w4a16_pick_ntok(T * topk, local_experts);  // (T * world * topk) / world local pairs
}

int64_t w4a16_moe_ep_workspace_bytes(int64_t T, int64_t world, int64_t topk, int64_t local_experts, int64_t H,
                                     int64_t I) {
  const int64_t Tg = T * world, P = Tg * topk;
  const int nt = ep_ntok(T, world, topk, local_experts);
  const int64_t a = w4a16_grouped_gemm_ws_bytes(P, H, local_experts, I, 1, nt);
  const int64_t b = w4a16_grouped_gemm_ws_bytes(P, I, local_experts, H, 0, nt);
  return align256(2 * Tg * H) + 3 * align256(4 * Tg * topk) + align256(4 * Tg * H) + align256(4 * T * H) +
         align256(w4a16_moe_workspace_bytes(Tg, topk, local_experts, H, I)) + align256(a > b ? a : b);
}

int w4a16_moe_forward_ep(w4a16_ep_comm* comm, const void* x, int64_t T, int64_t H, int64_t I, int64_t local_experts,
                         int64_t topk, const int32_t* topk_ids, const float* topk_weights, const uint8_t* w13,
                         const uint8_t* w2, int dtype, void* y, void* workspace, int64_t workspace_bytes,
                         cudaStream_t stream) {
  if (!comm || !workspace) return W4_ERR_ARG;
  if (workspace_bytes < w4a16_moe_ep_workspace_bytes(T, comm->world, topk, local_experts, H, I))
    return W4_ERR_WORKSPACE;
  if (T <= 0) return W4_OK;
  const int64_t Tg = T * comm->world;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  // the local layer's workspace first
  const int nt = ep_ntok(T, comm->world, topk, local_experts);
  const int64_t ga = w4a16_grouped_gemm_ws_bytes(Tg * topk, H, local_experts, I, 1, nt);
  const int64_t gb = w4a16_grouped_gemm_ws_bytes(Tg * topk, I, local_experts, H, 0, nt);
  void* inner = ws;
  const int64_t inner_bytes =
      align256(w4a16_moe_workspace_bytes(Tg, topk, local_experts, H, I)) + align256(ga > gb ? ga : gb);
  ws += inner_bytes;
  void* x_all = ws; ws += align256(2 * Tg * H);
  int32_t* ids_all = reinterpret_cast<int32_t*>(ws); ws += align256(4 * Tg * topk);
  float* w_all = reinterpret_cast<float*>(ws); ws += align256(4 * Tg * topk);
  int32_t* ids_loc = reinterpret_cast<int32_t*>(ws); ws += align256(4 * Tg * topk);
  float* partial = reinterpret_cast<float*>(ws); ws += align256(4 * Tg * H);
  float* reduced = reinterpret_cast<float*>(ws);
  int rc;
  if ((rc = w4a16_ep_dispatch(comm, x, topk_ids, topk_weights, T, H, topk, dtype, x_all, ids_all, w_all, stream)))
    return rc;
  if ((rc = w4a16_ep_localize(ids_all, Tg * topk, comm->rank * local_experts, local_experts, ids_loc, stream)))
    return rc;
  if ((rc = w4a16_moe_forward_f32(x_all, Tg, H, I, local_experts, topk, ids_loc, w_all, w13, w2, dtype, partial, nt,
                                  inner, inner_bytes, stream)))
    return rc;
  return w4a16_ep_combine(comm, partial, T, H, dtype, reduced, y, stream);
}

}  // extern "C"

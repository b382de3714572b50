/*
 * w4a16_moe.h -- C ABI of the B200 (sm_100a) W4A16 mixture-of-experts path.
 *
 * The reference (Hexcute's `tilesynth`, /root/reference/pkg) has no C/C++/CUDA code and no FFI: its
 * boundary is the Python API (pkg/src/tilesynth/__init__.py:16-58) and it stops at the synthesized
 * layout plan for the fp16 x int4 tile (pkg/fixtures/mixed_int4.prog:1-18). The paper's MoE operator
 * is the kernel that plan feeds. These entry points are that operator, split
 * the way the Python host (paper_2504_16214_b200/moe) and a vLLM-style caller
 * (vllm fused_experts(hidden_states, w1, w2, topk_weights, topk_ids, ...)) bind it:
 *
 *   route:    w4a16_route_topk                         top-k of softmax/sigmoid router scores
 *             w4a16_route_grouped_topk                 DeepSeek-V3/R1 grouped top-k (vLLM grouped_topk)
 *             w4a16_route_permute                      route_topk + moe_permute in one CTA (small batches)
 *   permute:  w4a16_moe_permute                        stable counting sort of (token, slot) by expert
 *   gather:   w4a16_moe_gather                         X_perm[p] = x[token(p)]   (128-bit vectors)
 *             w4a16_moe_gather_sums                    same, plus per-group activation sums (decode)
 *   sums:     w4a16_group_sums                         per-(group of 128 k, row) sums of an activation
 *   GEMM:     w4a16_grouped_gemm                       per-expert X_e * W_e^T, optional fused SiLU*up
 *             w4a16_grouped_gemm_gather                same, X rows gathered by the producer (TMA gather4)
 *   combine:  w4a16_moe_combine                        y[t] = sum_j w[t,j] * Y_perm[pos(t,j)]
 *   combine:  w4a16_moe_combine_f32                    same, fp32 unrounded (expert-parallel partials)
 *   EP:       w4a16_ep_dispatch / w4a16_ep_combine     all-gather dispatch / reduce-scatter combine over an
 *                                                      opaque NCCL communicator (w4a16_ep_comm_*)
 *             w4a16_ep_localize                        global -> local expert ids of the gathered batch
 *             w4a16_moe_forward_ep                     the whole expert-parallel layer, one call
 *             w4a16_ep_local_order                     receiver-side local-expert order of the rows an
 *                                                      all-to-all delivered (grouped by source rank)
 *   weights:  w4a16_repack_awq, w4a16_dequant (test/oracle aid), w4a16_packed_bytes
 *   driver:   w4a16_moe_forward(_f32)                  the whole layer, one call, caller workspace
 *
 * Conventions: raw device pointers, int64_t extents, cudaStream_t (pass 0 for the legacy stream);
 * every function is stream-ordered, returns an int status (0 ok, < 0 error, never throws), performs
 * no hidden host synchronisation and allocates nothing: the caller owns every buffer including
 * workspace (query sizes with the *_workspace_bytes functions). Activations are fp16 or bf16
 * (W4_DTYPE_*); scales use the activation dtype; int4 codes/zeros are AWQ (uint4, group 128).
 */
#ifndef W4A16_MOE_H_
#define W4A16_MOE_H_

#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  W4_OK = 0,
  W4_ERR_ARG = -1,    /* null pointer / bad enum */
  W4_ERR_SHAPE = -2,  /* extent not a multiple of the tile (N % 128, K % 128) or too large */
  W4_ERR_DTYPE = -3,  /* unsupported activation dtype */
  W4_ERR_GROUP = -4,  /* unsupported quantisation group size (only 128) */
  W4_ERR_CUDA = -5,   /* launch / driver failure (cudaGetLastError() has details) */
  W4_ERR_WORKSPACE = -6,
  W4_ERR_NCCL = -7    /* NCCL missing (libnccl.so.2 not loadable) or a collective failed */
};

enum { W4_DTYPE_F16 = 0, W4_DTYPE_BF16 = 1 };
enum { W4_SCORE_SOFTMAX = 0, W4_SCORE_SIGMOID = 1 };

/* ---- weights --------------------------------------------------------------------------------- */
/* Bytes of the packed block format for [num_experts][n_rows][K] (== AWQ bytes; -1 if misaligned). */
int64_t w4a16_packed_bytes(int64_t num_experts, int64_t n_rows, int64_t K);
int w4a16_tile_rows(void); /* 128 */
/* The launch plan w4a16_grouped_gemm_ws would use (host only, no GPU needed): token tile, block mode
 * (0 plain, 1 gate|up, 2 k-pair, 3 n-pair), offset-code decode mode or not, split-K factor. */
int w4a16_gemm_plan(int64_t rows, int64_t K, int64_t num_experts, int64_t n_out, int gated, int has_xsum, int ntok,
                    int* out_ntok, int* out_mode, int* out_offset, int* out_splits);
int w4a16_tile_k(void);    /* 128 */
int w4a16_part_bytes(void);

/* AWQ -> packed blocks. qweight [E][K][n_rows/8] int32, scales [E][K/G][n_rows] (act dtype),
 * qzeros [E][K/G][n_rows/8] int32 (AWQ nibble order 0,2,4,6,1,3,5,7). parts = 2 interleaves the
 * first and second halves of n_rows (gate | up) block-wise for the fused gate/up GEMM.
 * Replaces vLLM's AWQ->Marlin repack for this path (vllm .../awq_marlin.py:70-74). */
int w4a16_repack_awq(const int32_t* qweight, const void* scales, const int32_t* qzeros, int64_t num_experts,
                     int64_t K, int64_t n_rows, int parts, int group_size, uint8_t* wblocks, cudaStream_t stream);

/* packed blocks -> dense W [E][n_rows][K] (act dtype), bit-exact fp16((q - z) * s). */
int w4a16_dequant(const uint8_t* wblocks, int64_t num_experts, int64_t n_rows, int64_t K, int parts, int dtype,
                  void* out, cudaStream_t stream);

/* ---- routing ---------------------------------------------------------------------------------- */
/* logits [T][E] fp32 -> topk_ids [T][k] int32 (descending score, ties -> lower expert id),
 * topk_weights [T][k] fp32 (softmax or sigmoid of the selected logits, optionally renormalised). */
int w4a16_route_topk(const float* logits, int64_t T, int64_t E, int64_t k, int scoring, int renormalize,
                     int32_t* topk_ids, float* topk_weights, cudaStream_t stream);

/* w4a16_route_topk + w4a16_moe_permute of its ids in one single-CTA kernel (small batches: one launch
 * and one kernel boundary fewer before the GEMMs). Same outputs as the two calls. T * k <= 2^20. */
int w4a16_route_permute(const float* logits, int64_t T, int64_t E, int64_t k, int scoring, int renormalize,
                        int32_t* topk_ids, float* topk_weights, int32_t* expert_counts, int32_t* expert_offsets,
                        int32_t* sorted_pairs, int32_t* pair_pos, cudaStream_t stream);

/* DeepSeek-V3/R1 routing, vLLM grouped_topk semantics (vllm/model_executor/layers/fused_moe/router/
 * grouped_topk_router.py:81-162): scores = softmax|sigmoid(logits); choice = scores + bias (bias [E]
 * fp32 e_score_correction_bias, or NULL); group score = sum of the group's two best choices (bias) or
 * its best score (no bias); keep the topk_group best of num_groups groups; topk_ids = the k best
 * kept choices (ties -> lower id); topk_weights = their unbiased scores, renormalised if asked,
 * times routed_scaling_factor. num_groups <= 32 must divide E. */
int w4a16_route_grouped_topk(const float* logits, int64_t T, int64_t E, int64_t k, int64_t num_groups,
                             int64_t topk_group, int scoring, int renormalize, const float* bias,
                             float routed_scaling_factor, int32_t* topk_ids, float* topk_weights, cudaStream_t stream);

/* Stable counting sort of the P = T*k flattened (token, slot) pairs by expert id.
 * ids outside [0, E) are dropped (pair_pos = -1). Outputs: expert_counts [E], expert_offsets [E+1],
 * sorted_pairs [P] (flat pair index at each permuted row; rows >= offsets[E] untouched),
 * pair_pos [P] (permuted row of each pair or -1). */
int w4a16_moe_permute(const int32_t* topk_ids, int64_t P, int64_t E, int32_t* expert_counts,
                      int32_t* expert_offsets, int32_t* sorted_pairs, int32_t* pair_pos, cudaStream_t stream);

/* Same result as w4a16_moe_permute, parallel over many CTAs for large P (histogram -> scan ->
 * ranked scatter). ws: caller workspace of w4a16_moe_permute_ws_bytes(P, E) bytes; with a smaller
 * (or NULL) workspace, or small P, it runs the single-CTA kernel. */
int w4a16_moe_permute_ws(const int32_t* topk_ids, int64_t P, int64_t E, int32_t* expert_counts,
                         int32_t* expert_offsets, int32_t* sorted_pairs, int32_t* pair_pos, void* ws,
                         int64_t ws_bytes, cudaStream_t stream);
int64_t w4a16_moe_permute_ws_bytes(int64_t P, int64_t E);

/* Expert parallelism, receiver side: rows arrive grouped by (source rank, local expert) with counts
 * recv_counts [world][local_experts] (device). Produces the local-expert order, stable by source rank
 * then arrival: l_counts [E_l], l_offsets [E_l+1], l_sorted [n] (arrival row of each expert-ordered
 * row), l_pos [n] (expert-ordered position of each arrival row). world * E_l <= 4096. */
int w4a16_ep_local_order(const int32_t* recv_counts, int64_t world, int64_t local_experts, int32_t* l_counts,
                         int32_t* l_offsets, int32_t* l_sorted, int32_t* l_pos, cudaStream_t stream);

/* X_perm[p][:] = x[sorted_pairs[p] / topk][:] for p < rows, and p < *row_limit when row_limit (a
 * device pointer, e.g. expert_offsets + E) is non-null -- rows past it are left untouched. */
int w4a16_moe_gather(const void* x, int64_t H, int64_t topk, const int32_t* sorted_pairs, int64_t rows,
                     const int32_t* row_limit, void* x_perm, cudaStream_t stream);

/* Same as w4a16_moe_gather, and also writes the per-(k-group, row) activation sums the decode-mode
 * grouped GEMM consumes: xsum fp32 [H/128][w4a16_group_sums_ld(rows)][2] = (C, S) with
 * S = sum_k x[k] and C = sum_k c_k x[k] over the group's 128 k, c_k the offset of the GEMM's
 * offset-code dequant (fp16: 1024 for k%8 in {0,1,4,5}, 64 otherwise; bf16: 128). H % 128 == 0. */
int w4a16_moe_gather_sums(const void* x, int64_t H, int64_t topk, const int32_t* sorted_pairs, int64_t rows,
                          const int32_t* row_limit, void* x_perm, int dtype, float* xsum, cudaStream_t stream);

/* The sums alone for an activation x [rows][K] (rows >= *row_limit skipped when row_limit != NULL). */
int w4a16_group_sums(const void* x, int64_t rows, int64_t K, const int32_t* row_limit, int dtype, float* xsum,
                     cudaStream_t stream);
/* Row stride (in (C, S) pairs) of the sums array for `rows` rows: rows rounded up to even. */
int64_t w4a16_group_sums_ld(int64_t rows);

/* y[t][:] = act(sum_j topk_weights[t][j] * Y_perm[pair_pos[t*k+j]][:]), fp32 accumulate in slot
 * order; pairs with pair_pos < 0 contribute nothing. */
int w4a16_moe_combine(const void* y_perm, int64_t T, int64_t H, int64_t topk, const int32_t* pair_pos,
                      const float* topk_weights, int dtype, void* y, cudaStream_t stream);

/* Same as w4a16_moe_combine, but y is float [T][H] and the fp32 sums are NOT rounded (the partial a
 * reduction across expert-parallel ranks adds up before the one rounding, w4a16_ep_combine). */
int w4a16_moe_combine_f32(const void* y_perm, int64_t T, int64_t H, int64_t topk, const int32_t* pair_pos,
                          const float* topk_weights, int dtype, float* y, cudaStream_t stream);

/* ---- grouped GEMM ----------------------------------------------------------------------------- */
/* For each expert e: out[off_e + m][n] = act( sum_k X[off_e + m][k] * W_e[n][k] ), m < counts[e].
 * x [rows][K]; wblocks packed (parts = gated ? 2 : 1, n_rows = gated ? 2*n_out : n_out);
 * gated: out[.., n] = silu(X W_gate^T)[n] * (X W_up^T)[n] (fused SwiGLU). ntok = token tile
 * (16/32/64/128; 0 = pick from rows/num_experts). xsum (optional): x's group sums
 * (w4a16_group_sums layout); with it, 16/32-token tiles run the decode (offset-code) kernel,
 * without it the scale-in-dequant kernel. */
int w4a16_grouped_gemm(const void* x, int64_t rows, int64_t K, const uint8_t* wblocks, int64_t num_experts,
                       int64_t n_out, int gated, const int32_t* expert_counts, const int32_t* expert_offsets,
                       const float* xsum, void* out, int dtype, int ntok, cudaStream_t stream);
int w4a16_pick_ntok(int64_t rows, int64_t num_experts);
/* Largest token tile that runs in offset-code (decode) mode when xsum is given: 16 (default) or 32
 * (environment W4A16_DECODE_MAX_NTOK=32; 0 turns the mode off). Larger tiles apply the scale in the
 * dequant (prefill mode). */
int w4a16_decode_max_ntok(void);

/* Same, with a caller workspace that enables split-K in decode mode when the (expert, n-tile) tiles
 * cannot fill the GPU (e.g. one token touching 8 experts): the k-groups of a tile are split over
 * several CTAs writing fp32 partials to ws, then summed (and SiLU*up applied) by a finalize kernel.
 * ws_bytes >= w4a16_grouped_gemm_ws_bytes(...) (0 when no split is planned); a smaller workspace
 * just disables split-K. osum (optional): also produce the output's group sums (w4a16_group_sums
 * layout) -- the next GEMM's xsum; the decode gate/up epilogue computes them in place (gated, xsum
 * given, 16-token tiles, no split-K; otherwise a w4a16_group_sums pass follows the GEMM). out_rows
 * (optional): row i of the result is written to out row out_rows[i] (e.g. straight back into
 * expert-parallel arrival order); not combinable with osum. */
int w4a16_grouped_gemm_ws(const void* x, int64_t rows, int64_t K, const uint8_t* wblocks, int64_t num_experts,
                          int64_t n_out, int gated, const int32_t* expert_counts, const int32_t* expert_offsets,
                          const float* xsum, float* osum, const int32_t* out_rows, void* out, int dtype, int ntok,
                          void* ws, int64_t ws_bytes, cudaStream_t stream);

/* The gate/up GEMM with the token gather fused into its producer (replaces w4a16_moe_gather +
 * w4a16_grouped_gemm): row i of the GEMM input is row gather_rows[i] / gather_div of x [x_rows][K]
 * (gather_rows = sorted_pairs and gather_div = top_k for the MoE layer), loaded with TMA gather4.
 * xsum, when given, holds the group sums of x's own rows (w4a16_group_sums over x). No out_rows, no
 * CTA pairs. */
int w4a16_grouped_gemm_gather(const void* x, int64_t x_rows, const int32_t* gather_rows, int gather_div, int64_t rows,
                              int64_t K, const uint8_t* wblocks, int64_t num_experts, int64_t n_out, int gated,
                              const int32_t* expert_counts, const int32_t* expert_offsets, const float* xsum,
                              float* osum, void* out, int dtype, int ntok, void* ws, int64_t ws_bytes,
                              cudaStream_t stream);
int64_t w4a16_grouped_gemm_ws_bytes(int64_t rows, int64_t K, int64_t num_experts, int64_t n_out, int gated,
                                    int ntok);

/* ---- whole layer ------------------------------------------------------------------------------- */
/* Workspace for w4a16_moe_forward with T tokens, top-k, E experts, hidden H, intermediate I. */
int64_t w4a16_moe_workspace_bytes(int64_t T, int64_t topk, int64_t E, int64_t H, int64_t I);

/* y = MoE(x) for precomputed routing: permute -> gather -> gate/up GEMM (+SiLU*up) -> down GEMM ->
 * combine. w13 packed with parts=2 (n_rows = 2I, K = H), w2 packed with parts=1 (n_rows = H, K = I). */
int w4a16_moe_forward(const void* x, int64_t T, int64_t H, int64_t I, int64_t E, int64_t topk,
                      const int32_t* topk_ids, const float* topk_weights, const uint8_t* w13,
                      const uint8_t* w2, int dtype, void* y, void* workspace, int64_t workspace_bytes,
                      cudaStream_t stream);

/* Same as w4a16_moe_forward with the fp32, unrounded combine (w4a16_moe_combine_f32): y float [T][H].
 * ntok: the GEMMs' token tile (0 = pick from T * topk / E; expert parallelism passes the tile for the
 * pairs it expects to be local, most ids being -1). */
int w4a16_moe_forward_f32(const void* x, int64_t T, int64_t H, int64_t I, int64_t E, int64_t topk,
                          const int32_t* topk_ids, const float* topk_weights, const uint8_t* w13,
                          const uint8_t* w2, int dtype, float* y, int ntok, void* workspace, int64_t workspace_bytes,
                          cudaStream_t stream);

/* ---- expert parallelism (NCCL over NVLink / NVSwitch) ------------------------------------------ */
/* Experts shard contiguously: rank r owns global experts [r * E_local, (r + 1) * E_local). Dispatch is
 * an all-gather of every rank's tokens and routing, combine a reduce-scatter of fp32 partial sums:
 * fixed shapes, no host synchronisation, CUDA-graph capturable. Every rank passes the same T (pad
 * with rows whose topk_ids are -1). NCCL is loaded at run time (libnccl.so.2); w4a16_ep_available()
 * says whether it was found. The communicator is opaque. */
typedef struct w4a16_ep_comm w4a16_ep_comm;
int w4a16_ep_available(void);
/* 128-byte NCCL unique id: make it on one rank, hand it to every rank (any host channel). */
int w4a16_ep_unique_id(void* id);
/* Collective over `world` ranks (one per GPU, each with its device current). */
int w4a16_ep_comm_init(const void* id, int rank, int world, w4a16_ep_comm** comm);
/* Borrow an existing ncclComm_t (not destroyed by w4a16_ep_comm_destroy). */
int w4a16_ep_comm_wrap(void* nccl_comm, w4a16_ep_comm** comm);
int w4a16_ep_comm_destroy(w4a16_ep_comm* comm);
int w4a16_ep_comm_rank(const w4a16_ep_comm* comm);
int w4a16_ep_comm_size(const w4a16_ep_comm* comm);

/* x [T][H], topk_ids [T][k] (GLOBAL expert ids), topk_weights [T][k] of every rank ->
 * x_all [world*T][H], ids_all / w_all [world*T][k] (rank r's rows at r*T). */
int w4a16_ep_dispatch(w4a16_ep_comm* comm, const void* x, const int32_t* topk_ids, const float* topk_weights,
                      int64_t T, int64_t H, int64_t topk, int dtype, void* x_all, int32_t* ids_all, float* w_all,
                      cudaStream_t stream);
/* ids_local[i] = ids[i] - expert_base when that is in [0, local_experts), else -1. */
int w4a16_ep_localize(const int32_t* ids, int64_t n, int64_t expert_base, int64_t local_experts, int32_t* ids_local,
                      cudaStream_t stream);
/* partial float [world*T][H] (this rank's experts' weighted sums for the whole node batch) ->
 * reduce-scatter (sum over ranks, fp32) into reduced float [T][H] -> y [T][H] act dtype (one rounding). */
int w4a16_ep_combine(w4a16_ep_comm* comm, const float* partial, int64_t T, int64_t H, int dtype, float* reduced,
                     void* y, cudaStream_t stream);

/* The whole expert-parallel layer: dispatch -> localize -> w4a16_moe_forward_f32 on this rank's shard
 * (w13 / w2 packed for local_experts) -> combine. */
int64_t w4a16_moe_ep_workspace_bytes(int64_t T, int64_t world, int64_t topk, int64_t local_experts, int64_t H,
                                     int64_t I);
int w4a16_moe_forward_ep(w4a16_ep_comm* comm, const void* x, int64_t T, int64_t H, int64_t I, int64_t local_experts,
                         int64_t topk, const int32_t* topk_ids, const float* topk_weights, const uint8_t* w13,
                         const uint8_t* w2, int dtype, void* y, void* workspace, int64_t workspace_bytes,
                         cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* W4A16_MOE_H_ */

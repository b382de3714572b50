// W4A16 grouped (MoE) GEMM for sm_100a, plus the standalone dequant and the AWQ -> block repack.
//
// Formulation ("swap-AB"): for expert e, Y_e[M_e x N] = X_e[M_e x K] * W_e[N x K]^T is computed as
//   D[n, m] = sum_k W_e[n, k] * X_e[m, k]
// so the 128 weight rows of an n-tile fill the 128-lane M slot of tcgen05.mma and the tokens of the
// expert (often 1..16 at decode) are the MMA's N dimension (16..128). Per CTA (one per SM,
// persistent over a static tile schedule):
//   warp 0      producer : 1-D bulk copy of the packed weight block (codes+scales+zeros, 8.5/17 KB)
//                           and a 2-D TMA (128B swizzle) of the X tile into an NS-deep smem ring
//   warp 1      MMA      : one elected thread issues tcgen05.mma kind::f16, A from TMEM, B from smem
//   warps 2-9   dequant  : ld.shared 16 B of int4 per row-thread -> LOP3/HSUB2/HMUL2 -> tcgen05.st
//                           into a TMEM A-operand ring (lane = weight row, 2 k per 32-bit column)
//   warps 10-13 epilogue : tcgen05.ld of the fp32 accumulator, SiLU(gate)*up when fused, 16-token
//                           chunks staged in shared memory and stored with 16-byte stores
//   (warp 14     second MMA issuer, -DW4A16_DUAL=1 experiment only)
// The dequantised weights never touch shared memory or HBM: int4 goes HBM -> smem -> registers ->
// TMEM -> tensor core. Barriers: smem full/empty, TMEM-A full/empty, accumulator full/empty.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include "ptx.cuh"
#include "launch.cuh"
#include "w4_format.cuh"
#include "mma_stage.cuh"
#include "w4a16_moe.h"

namespace w4 {

#ifndef W4A16_GEMM_TAIL_TRIGGER
// experiment: PDL trigger this many stages before a CTA's last (0 = off). Measured with 4: no gain
// (DS-R1 T=1 58.9 -> 59.3 us, Qwen3 Zipf T=16 45.1 -> 46.8 us, the rest within noise)
#define W4A16_GEMM_TAIL_TRIGGER 0
#endif
// Experiment (-DW4A16_DUAL=1): a 15th warp as the second MMA issuer of the prefill kernel (see kDual).
#ifndef W4A16_DUAL
#define W4A16_DUAL 0
#endif
constexpr bool kDualEnv = W4A16_DUAL != 0;
constexpr int kNumThreads = (kDualEnv ? 15 : 14) * 32;
constexpr int kMma2Warp = 14;
// named barriers handing the issue turn between the two MMA issuers, one per direction (warp 1 ->
// warp 14 and back; a single shared barrier could be completed by one warp's own arrive + sync when
// it runs ahead). Id 1: epilogue warps.
constexpr uint32_t kTurnBar0 = 3, kTurnBar1 = 4;
constexpr int kDequantWarp0 = 2;
constexpr int kNumDequantWarps = 8;  // two groups of 4 (one warp per TMEM lane quadrant) alternating stages
constexpr int kDequantGroup = 4;
constexpr int kEpiWarp0 = 10;
constexpr int kMaxExperts = 1024;
constexpr int kTileTab = 512;  // per-CTA tile table entries in smem (later tiles are searched on the fly)
// Largest token tile compiled in offset-code (decode) mode. Its epilogue costs 3 FFMA per (row, real
// token, k-group), against the dequant's per-weight scale in prefill mode; the largest tile actually
// run in offset mode is decode_max_ntok() (W4A16_DECODE_MAX_NTOK, default below).
constexpr int kDecodeMaxNTok = 32;
#ifndef W4A16_KSPLIT
#define W4A16_KSPLIT 0
#endif
constexpr bool kKSplitEnv = W4A16_KSPLIT != 0;  // experiment: -DW4A16_KSPLIT=1 (see Cfg::kKSplit)
constexpr int kSmemBudget = 225 * 1024;
#ifndef W4A16_SPLITA
#define W4A16_SPLITA 0
#endif
// experiment (-DW4A16_SPLITA=1): prefill k-half TMEM A units; measured slower (gate/up T=8192 3.57 vs
// 3.43 ms), see the Cfg comment
constexpr bool kSplitAEnv = W4A16_SPLITA != 0;
#ifndef W4A16_DECODE_NUMA
#define W4A16_DECODE_NUMA 2
#endif
#ifndef W4A16_DECODE_MAXACC
#define W4A16_DECODE_MAXACC 8
#endif
// Decode (offset-mode) TMEM split: A slots (if two accumulator stages still fit) and the cap on
// accumulator stages. With 3 A + 2 accumulator stages the MMA of stage j + 2 waited for the epilogue
// of stage j, and at every tile end the epilogue spends ~1100-1350 cycles (stores, next tile's
// setup) before its next fold, against ~500 mid-tile: the following MMA stalled ~700 cycles per tile
// (tools/trace_down.sh: DS-R1 down, 16-stage tiles). 2 A + 4 accumulator stages, same box
// (tools/gpu_ab_acc4.sh, DS-R1 layer): T=1 68.7 -> 64.2 us, T=16 452 -> 416 us, T=64 908 -> 867 us,
// T=256 1115 -> 1084 us; Mixtral T=16 172 -> 162 us; Qwen3 unchanged. With one k-chain per part
// (32-column accumulator stages) up to 8 stages fit beside 2 A slots; 3 A slots + 4 stages was
// slower at every decode size (T=64 862 -> 910-920 us, tools/gpu_ab_knobs.sh).
constexpr int kDecodeNumA = W4A16_DECODE_NUMA;
// Prefill-mode (scale-in-dequant) tiles of up to W4A16_SP_MAXNTOK tokens: W4A16_SP_NUMA A slots and
// up to W4A16_SP_MAXACC accumulator stages (the general rule -- 3 A slots beside 1-2 accumulator
// stages -- stalled the MMA on each short tile's epilogue). 2 A + 2-4 accumulator stages, same box:
// Qwen3 T=256 108 -> 102 us, its Zipf case 108 -> 103 us, Mixtral T=64 205 -> 188 us, T=128 209 ->
// 198 us, DS-R1 T=512 1.44 -> 1.33 ms, T=1024 1.57 -> 1.52 ms (tools/gpu_ab_sp.sh); 128-token tiles
// keep the general rule (their accumulator is 256 columns). W4A16_SP_NUMA=0 restores the general rule.
#ifndef W4A16_SP_NUMA
#define W4A16_SP_NUMA 2
#endif
#ifndef W4A16_SP_MAXACC
#define W4A16_SP_MAXACC 4
#endif
#ifndef W4A16_SP_MAXNTOK
#define W4A16_SP_MAXNTOK 64
#endif
constexpr int kSmallPrefillNumA = W4A16_SP_NUMA;
constexpr int kSmallPrefillMaxNTok = W4A16_SP_MAXNTOK;
constexpr int kSmallPrefillMaxAcc = W4A16_SP_MAXACC;
constexpr int kDecodeMaxAcc = W4A16_DECODE_MAXACC;

struct GemmArgs {
  const uint8_t* wblocks;        // [E][NT][KT][parts * kPartBytes]
  const int32_t* expert_counts;  // [E]
  const int32_t* expert_offsets; // [E+1]; rows of X (and of out) owned by expert e
  void* out;                     // [rows][NT*128] activation dtype
  int64_t ldo;
  const float* xsum;             // offset mode: (C, S) [kt][sum_ld][2]
  int64_t sum_ld, rows;
  int num_experts, nt, kt;
  int splits;                    // split-K factor (decode mode; 1 = none)
  float* part;                   // splits > 1: fp32 partials [splits][rows][part_ld]
  int64_t part_ld;               // (gated ? 2 : 1) * n_out
  float2* osum;                  // gated decode: (C, S) sums of the output h [nt][osum_ld] (next GEMM's xsum)
  int64_t osum_ld;               // = w4a16_group_sums_ld(rows) (sum_ld follows x's rows under a fused gather)
  const int32_t* out_rows;       // optional: output row of input row i (scatter, e.g. back to EP arrival order)
  // optional fused gather: row i of the GEMM input is row gather_rows[i] / gather_div of x (the X map
  // then covers x itself and the producer loads rows with TMA gather4); xsum is indexed by x's rows
  const int32_t* gather_rows;
  int gather_div;
  int direct_rows;               // offset-mode tiles with <= this many real tokens store unstaged (<= kDirectRows)
};

// Numeric modes.
// kOffset (decode, 16/32-token tiles): the dequant warps emit *offset codes* -- the exact integers
// c_k + q (Dq::word_raw: 5 integer ops per 8 weights, no FP op). Per stage (one quantisation group
// per part) the MMA writes the fp32 partial P[n,m] = sum_k (c_k + q[n,k]) x[m,k] into a TMEM ring;
// the per-(group, token) activation sums C[m] = sum_k c_k x[m,k] and S[m] = sum_k x[m,k] arrive
// with the stage (8-byte cp.async of the caller's xsum by the producer warp's lanes, see
// w4a16_group_sums), and the epilogue warps fold
//     acc[n,m] += s[n,g] * (P[n,m] - C[m] - z[n,g] * S[m])     ( = s * sum_k (q - z) x )
// so scale and zero point cost 3 FFMA per (row, token, group) instead of 2 FP ops per weight pair,
// and only the tile's real tokens are processed (4-column chunks). At decode token counts the
// tensor pipe pays ~38 cycles per M128 x N16 x K16 MMA whatever N is (the A-operand read), so the
// MMA count per weight byte is the budget: exactly one MMA per 128x16 weight slice.
// Otherwise (prefill, 64/128-token tiles, or no xsum given) the dequant applies zero and scale
// (bit-exact act((q - z) * s)) and the MMA accumulates across k-groups in TMEM.
// Block modes: how the two 8.5 KB parts of a 17 KB stage are used.
constexpr int kModePlain = 0;   // one part (one k-group) per stage
constexpr int kModeGateUp = 1;  // part 0 = gate rows, part 1 = up rows, same k-group (fused SwiGLU)
constexpr int kModeKPair = 2;   // parts = two consecutive k-groups of the same rows (down proj.)
constexpr int kModeNPair = 3;   // parts = one k-group of two adjacent n-tiles sharing the X tile (prefill)
constexpr int kEpiChunk = 4;    // offset-mode epilogue token granularity
constexpr int kDirectRows = 4;  // max of GemmArgs::direct_rows (W4A16_DIRECT_ROWS overrides the default 4; 0 = off)

// kPair: a CTA pair (cluster of 2 on one TPC) runs tcgen05.mma.cta_group::2 -- M = 256 weight rows
// (each CTA dequantises its own 128-row n-tile into its own TMEM), N = kNTok tokens with each CTA
// holding kNTok/2 rows of the X tile; one leader thread issues for both, halving MMA instructions
// and issuer waits per weight byte.
template <int kNTok, int kMode, bool kOffset, bool kPair = false>
struct Cfg {
  static constexpr bool kGated = kMode == kModeGateUp;
  static constexpr int kCG = kPair ? 2 : 1;
  static constexpr int kXRows = kNTok / kCG;  // X rows held by this CTA
  static constexpr int kParts = kMode == kModePlain ? 1 : 2;
  static constexpr int kNPer = kMode == kModeNPair ? 2 : 1;  // n-tiles per (CTA) tile
  static constexpr int kGroupsPerStage = kMode == kModeKPair ? 2 : 1;
  static constexpr int kBlk = kParts * kPartBytes;
  static constexpr int kXBytes = kGroupsPerStage * kXRows * kTileK * 2;  // X tile, 64-wide 128B-swizzle atoms
  // (C, S) fp32 per group/token, padded to one 8-byte slot per producer lane (see the sums copy)
  static constexpr int kSumBytes = kOffset ? (kGroupsPerStage * kNTok > 32 ? kGroupsPerStage * kNTok : 32) * 8 : 0;
  // offset mode, experiment: each part's 128-k partial split over kKSplit = 2 independent
  // accumulators (k halves), kParts * kKSplit interleaved MMA chains per stage. It helped with two
  // accumulator stages; with the deeper ring (below) one chain per part is faster (DS-R1 layer
  // T=64 868 -> 862 us, T=256 1.09-1.14 -> 1.06-1.08 ms, Mixtral T=16 162 -> 159 us;
  // tools/gpu_ab_knobs.sh) -- tools/microbench/mma_stage.cu: a stage's 16 MMAs complete in ~250
  // cycles streamed either way, so the chains were never the tensor pipe's limit
  static constexpr int kKSplit = (kOffset && kNTok == 16 && kKSplitEnv) ? 2 : 1;
  static constexpr int kChainLen = (kTileK / 16) / kKSplit;
  // one accumulator stage: offset mode = kKSplit partials per part; otherwise gate|up or one
  // accumulator for the whole tile
  static constexpr int kAccCols = kOffset ? kParts * kKSplit * kNTok : ((kGated || kNPer == 2) ? 2 * kNTok : kNTok);
  // Prefill two-part stages use a split A ring: one 64-column TMEM unit per k half of the stage
  // (both parts' k = 64h .. 64h+63), converted by dequant group h and released per unit by the MMA.
  // With whole-stage slots the MMA waited for each stage's dequant: TMEM fits only two 128-column
  // slots beside the 256-column gate|up accumulator, and a slot is busy for a whole dequant + MMA
  // round trip (stage period ~1440 cycles for 1024 of MMA, tools/trace_gemm.py). With half-stage
  // units the same 256 columns hold four units and each unit's round trip is half as long -- but the
  // measured stage period got longer (~1750 cycles: the MMA warp idles on the second group's units),
  // so this stays an experiment.
  static constexpr bool kSplitA = kSplitAEnv && !kOffset && kParts == 2;
  static constexpr int kAUnits = kSplitA ? 2 : 1;  // A-ring slots per stage
  // Prefill experiment: two MMA warps issue alternate stages (warp 1 even, warp 14 odd), handing the
  // turn over with a named barrier right after issuing. Measured (tools/microbench/mma_wait.cu,
  // tools/trace_gemm.py): issuing a stage's 16 N=128 MMAs takes ~640 cycles, its two commits ~190
  // and the next afull wait ~170-400 more, so one issuer leaves the tensor pipe idle between stages
  // (stage period ~1420 cycles for 1024 of MMA). Two issuers cut the period to ~1325 cycles, but a
  // sustained prefill GEMM is power-capped (sw_power_cap, SM clock 1.2-1.3 GHz): the same-box A/B
  // gave equal wall time (the clock drops by what the cycles gain), so this stays off.
  static constexpr bool kDual = kDualEnv && !kOffset && !kPair && !kSplitA;
  static constexpr int kACols = (kSplitA ? 1 : kParts) * (kTileK / 2);  // fp16 pairs per 32-bit column
  // TMEM budget (512 columns): A ring + accumulator ring
  // Decode tiles: kDecodeNumA A slots, up to kDecodeMaxAcc accumulator stages. Otherwise 3 A slots if two
  // accumulator stages still fit, else 2; the gated prefill projection (56-stage
  // tiles) instead prefers 3 A slots (dequant / MMA overlap) over a second accumulator stage
  // (epilogue / next-tile overlap, once per long tile); the short k-pair tiles need two.
  // Split ring: two accumulator stages if 6 units still fit, then as many units as fit (<= 8).
  static constexpr int kNumA_ = kOffset ? ((kDecodeNumA * kACols + 2 * kAccCols <= 512) ? kDecodeNumA : 2)
                              : (kNTok <= kSmallPrefillMaxNTok && kSmallPrefillNumA > 0) ? kSmallPrefillNumA
                              : !(kGated || kNPer == 2) ? ((3 * kACols + 2 * kAccCols <= 512) ? 3 : 2)
                                                                   : ((3 * kACols + kAccCols <= 512) ? 3 : 2);
  static constexpr int kNumAccS = (2 * kAccCols + 6 * kACols <= 512) ? 2 : 1;
  static constexpr int kNumAS = (512 - kNumAccS * kAccCols) / kACols > 8 ? 8 : (512 - kNumAccS * kAccCols) / kACols;
  static constexpr int kNumAccO = (512 - kNumA_ * kACols) / kAccCols;
  static constexpr int kMaxAcc = kOffset ? kDecodeMaxAcc : (kNTok <= kSmallPrefillMaxNTok ? kSmallPrefillMaxAcc : 2);
  static constexpr int kNumAcc = kSplitA ? kNumAccS : (kNumAccO > kMaxAcc ? kMaxAcc : kNumAccO);
  static constexpr int kNumA = kSplitA ? kNumAS : kNumA_;
  static constexpr int kStageBytes = kBlk + kXBytes + kSumBytes;
  // barriers, m-tile prefix, tile table, epilogue cross-warp reduction scratch (4 warps x 16 x float2)
  // epilogue: per-warp staging of a 16-token x 32-column output block (x2 for n-pair tiles)
  static constexpr int kEpiStageBytes = 4 * 1024 * (kNPer == 2 ? 2 : 1);  // [4 warps][...], 16 B aligned
  static constexpr int kFixed = 2048 + 4 * (kMaxExperts + 2) + 8 * kTileTab + 512 + 16 + kEpiStageBytes;
  static constexpr int kNS0 = (kSmemBudget - kFixed - 1024) / kStageBytes;
  static constexpr int kNS = kNS0 > 12 ? 12 : kNS0;
  // dequant warps reading a stage's smem: one group, or both (split ring: group h converts k half h)
  static constexpr int kDqPerStage = kSplitA ? 2 * kDequantGroup : kDequantGroup;
  static constexpr int kEmptyArrivals = kDqPerStage + 1 + (kOffset ? 4 : 0);
  static constexpr int kSumItems = kGroupsPerStage * kNTok;      // 8-byte (C, S) items per stage
  static constexpr int kFullArrivals = 1 + (kOffset ? 32 : 0);   // expect_tx + the 32 sums cp.async lanes
  static constexpr int kAFullArrivals = kDequantGroup * kCG;     // one dequant group of both CTAs (leader)
  static constexpr int kAccEmptyArrivals = 4 * kCG;              // epilogue warps of both CTAs (leader)
  // X ring first (needs 1024 B alignment for the 128B swizzle atoms), sums ring, then weights.
  static constexpr int kSmemBytes = 1024 + kNS * kStageBytes + kFixed;
  static_assert(kNumA >= 2 * kAUnits && kNumAcc >= (kOffset ? 2 : 1), "TMEM budget");
  static_assert(kNumA * kACols + kNumAcc * kAccCols <= 512, "TMEM budget");
  static_assert(kNS >= 2, "smem budget");
  static_assert(kXBytes % 1024 == 0, "X tile alignment");
  static_assert(!kOffset || kNTok <= 32, "register accumulators");
};

// Opt-in per-stage timeline of CTA 0 (w4a16_debug_trace): clock64 at each role's sync points.
__device__ long long* g_w4_trace = nullptr;
__device__ int g_w4_trace_cta = 0;  // which CTA the timeline follows
constexpr int kTraceCap = 4096;
__device__ __forceinline__ void trace_at(long long* tr, int ev, uint32_t idx) {
#ifndef W4A16_TRACE
  return;
#endif
  if (tr && idx < kTraceCap) {
    long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    tr[ev * kTraceCap + idx] = c;
  }
}

// trace build only: per-CTA progress (rows 10..13 of the trace buffer: producer / dequant / MMA /
// epilogue stages completed, indexed by blockIdx.x), to locate a stuck CTA
__device__ __forceinline__ void progress_at(int ev, uint32_t n) {
#ifdef W4A16_TRACE
  if (g_w4_trace) *reinterpret_cast<volatile long long*>(g_w4_trace + (10 + ev) * kTraceCap + blockIdx.x) = n;
#endif
}

struct TileInfo {
  int e, n_tile, m_start, m_rows, split;
};

// Static persistent schedule: tile t -> (expert, n-tile group, m-tile); m-tiles of one (expert, n-tile)
// are adjacent so concurrently running CTAs share that weight block through L2. kNSplit = 2 for CTA
// pairs: tile t covers n-tiles 2g and 2g+1, CTA rank r of the pair takes n-tile 2g + r.
template <int kNTok, int kNSplit, int kNPer = 1>
__device__ __forceinline__ bool get_tile(int t, const int* mt_off, const GemmArgs& a, uint32_t rank, TileInfo& ti) {
  const int ntg = a.nt / (kNSplit * kNPer);
  const int total = mt_off[a.num_experts] * ntg * a.splits;
  if (t >= total) return false;
  ti.split = t % a.splits;  // split-K units of one tile are adjacent
  t /= a.splits;
  int lo = 0, hi = a.num_experts;  // find e with mt_off[e]*ntg <= t < mt_off[e+1]*ntg
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (mt_off[mid] * ntg <= t) lo = mid; else hi = mid;
  }
  const int e = lo;
  const int me = mt_off[e + 1] - mt_off[e];
  const int local = t - mt_off[e] * ntg;
  const int m_tile = me == 1 ? 0 : local % me;
  ti.e = e;
  ti.n_tile = ((me == 1 ? local : local / me) * kNSplit + static_cast<int>(rank)) * kNPer;
  ti.m_start = __ldg(a.expert_offsets + e) + m_tile * kNTok;
  ti.m_rows = min(kNTok, __ldg(a.expert_counts + e) - m_tile * kNTok);
  return true;
}

// Packed tile: w0 = e | (m_rows - 1) << 10 | n_tile << 17, w1 = m_start | split << 20. Only split-K
// launches (rows < 2^20, enforced by plan_gemm) pack a split; otherwise split is 0 and unpack_tile
// reads m_start from all 32 bits, so row counts >= 2^20 stay exact.
__device__ __forceinline__ uint2 pack_tile(const TileInfo& ti) {
  return make_uint2(static_cast<uint32_t>(ti.e) | static_cast<uint32_t>(ti.m_rows - 1) << 10 |
                        static_cast<uint32_t>(ti.n_tile) << 17,
                    static_cast<uint32_t>(ti.m_start) | static_cast<uint32_t>(ti.split) << 20);
}
__device__ __forceinline__ void unpack_tile(uint2 p, TileInfo& ti, bool split_k) {
  ti.e = p.x & 1023u;
  ti.m_rows = static_cast<int>((p.x >> 10) & 127u) + 1;
  ti.n_tile = static_cast<int>(p.x >> 17);
  ti.m_start = static_cast<int>(split_k ? (p.y & 0xFFFFFu) : p.y);
  ti.split = split_k ? static_cast<int>(p.y >> 20) : 0;
}

// The CTA's i-th tile (t = tile0 + i * tstride): from the smem table when i < kTileTab, else searched.
// (An out-of-line search for the rare i >= kTileTab made the kernel 200 instructions smaller but
// 1-2 % slower at decode sizes -- the call's stack frame; measured with tools/gpu_ab_libs.sh.)
template <int kNTok, int kNSplit, int kNPer = 1>
__device__ __forceinline__ bool tile_at(int i, int n_tiles, int tile0, int tstride, const uint2* tab, const int* mt_off,
                                        const GemmArgs& a, uint32_t rank, TileInfo& ti) {
  if (i >= n_tiles) return false;
  if (i < kTileTab) {
    unpack_tile(tab[i], ti, a.splits > 1);
    return true;
  }
  return get_tile<kNTok, kNSplit, kNPer>(tile0 + i * tstride, mt_off, a, rank, ti);
}

// fast reciprocal division (exp overflow -> +inf -> 0, the limit): no IEEE slow-path branch, so the
// epilogue's per-token chains stay branch-free and interleave
__device__ __forceinline__ float silu_f(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

template <bool kBF16>
__device__ __forceinline__ uint16_t to_act_bits(float v) {
  if constexpr (kBF16) return __bfloat16_as_ushort(__float2bfloat16_rn(v));
  else return __half_as_ushort(__float2half_rn(v));
}

template <bool kBF16>
__device__ __forceinline__ float act_bits_to_float(uint32_t b) {
  if constexpr (kBF16) return __uint_as_float(b << 16);
  else return __half2float(__ushort_as_half(static_cast<unsigned short>(b)));
}

// TMA tile::gather4: rows r0..r3 of the 2-D map (box {64 columns, 1 row}), 64 columns from `col`, into
// 4 consecutive 128-byte smem rows (128B swizzle by smem row, the same layout as a 2-D box load;
// tools/microbench/tma_gather4.cu)
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int col, int r0, int r1, int r2, int r3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

struct Ring {  // (stage, phase) iterator of an mbarrier ring
  int i = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next(int n) {
    if (++i == n) { i = 0; ph ^= 1; }
  }
};

// kGather: the fused-gather variant (X rows gathered by the producer, w4a16_grouped_gemm_gather); a
// separate instantiation so the regular kernels carry none of its code
template <int kNTok, int kMode, bool kBF16, bool kOffset, bool kPair, bool kGather = false>
__global__ void __launch_bounds__(kNumThreads, 1)
    w4a16_moe_gemm_kernel(const GemmArgs args, const __grid_constant__ CUtensorMap xmap) {
  using C = Cfg<kNTok, kMode, kOffset, kPair>;
  constexpr bool kGated = C::kGated;
  const int n_stages = args.kt / C::kGroupsPerStage;  // stages per tile
  // split-K: unit (tile, split) covers stages [stage_beg, stage_end) of the tile
  auto stage_beg = [&](const TileInfo& t) { return t.split * n_stages / args.splits; };
  auto stage_end = [&](const TileInfo& t) { return (t.split + 1) * n_stages / args.splits; };
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_x = smem;                                  // [NS][kXBytes]
  uint8_t* smem_s = smem + C::kNS * C::kXBytes;            // [NS][kSumBytes] (offset mode)
  uint8_t* smem_w = smem_s + C::kNS * C::kSumBytes;        // [NS][kBlk]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_w + C::kNS * C::kBlk);
  uint64_t* full = bars;
  uint64_t* empty = full + C::kNS;
  uint64_t* afull = empty + C::kNS;
  uint64_t* aempty = afull + C::kNumA;
  uint64_t* accfull = aempty + C::kNumA;
  uint64_t* accempty = accfull + C::kNumAcc;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(accempty + C::kNumAcc);
  uint64_t* trbar = accempty + C::kNumAcc + 2;  // trace builds: per-stage MMA completion (8-deep ring)
  int* mt_off = reinterpret_cast<int*>(bars + 256);
  uint2* tile_tab = reinterpret_cast<uint2*>(mt_off + kMaxExperts + 2);  // 8-byte aligned (odd int count + 1)
  int* n_tiles_sm = mt_off + kMaxExperts + 1;
  float2* red_sm = reinterpret_cast<float2*>(tile_tab + kTileTab);  // [4 warps][16 tokens]
  uint8_t* epi_sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(red_sm + 64) + 15) & ~uintptr_t(15));

  const uint32_t warp = warp_idx();
  const uint32_t lane = lane_id();
  const uint32_t rank = kPair ? cluster_ctarank() : 0u;  // CTA rank in the pair (0 = leader, issues MMAs)
#ifdef W4A16_TRACE
  unsigned long long t_entry;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_entry));
#endif
  const int tile0 = kPair ? static_cast<int>(cluster_id_x()) : static_cast<int>(blockIdx.x);
  const int tstride = kPair ? static_cast<int>(nclusters_x()) : static_cast<int>(gridDim.x);
  #ifdef W4A16_TRACE
  long long* const tr = static_cast<int>(blockIdx.x) == g_w4_trace_cta ? g_w4_trace : nullptr;
#else
  long long* const tr = nullptr;
#endif

  if (warp == 0) {
    if constexpr (kPair) tmem_alloc_pair<512>(tmem_holder);
    else tmem_alloc<512>(tmem_holder);
  } else if (warp == 1 && lane == 0) {
    for (int i = 0; i < C::kNS; ++i) { mbar_init(&full[i], C::kFullArrivals); mbar_init(&empty[i], C::kEmptyArrivals); }
    for (int i = 0; i < C::kNumA; ++i) { mbar_init(&afull[i], C::kAFullArrivals); mbar_init(&aempty[i], 1); }
    for (int i = 0; i < C::kNumAcc; ++i) { mbar_init(&accfull[i], 1); mbar_init(&accempty[i], C::kAccEmptyArrivals); }
#ifdef W4A16_TRACE
    for (int i = 0; i < 8; ++i) mbar_init(&trbar[i], 1);
#endif
    fence_mbar_init();
  } else if (warp == 2) {
    // PDL: TMEM allocation and barrier init above overlap the previous kernel; expert counts / X / sums
    // are its outputs. Other roles touch them only after the __syncthreads below.
    griddep_wait();
    // m-tile prefix over experts (E <= 1024): each lane scans a contiguous slice, then a warp scan.
    const int E = args.num_experts;
    const int per = (E + 31) / 32;
    const int beg = min(E, (int)lane * per), end = min(E, beg + per);
    int s = 0;
    for (int e = beg; e < end; ++e) s += (__ldg(args.expert_counts + e) + kNTok - 1) / kNTok;
    int incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, incl, o);
      if ((int)lane >= o) incl += v;
    }
    int run = incl - s;
    for (int e = beg; e < end; ++e) {
      mt_off[e] = run;
      run += (__ldg(args.expert_counts + e) + kNTok - 1) / kNTok;
    }
    if (lane == 31) mt_off[E] = incl;
    __syncwarp();
    // this CTA's tiles t = tile0 + i * tstride, the first kTileTab of them tabulated
    const int total = mt_off[E] * (args.nt / (C::kCG * C::kNPer)) * args.splits;
    const int n_tiles = tile0 < total ? (total - tile0 + tstride - 1) / tstride : 0;
    if (lane == 0) *n_tiles_sm = n_tiles;
    for (int i = lane; i < min(n_tiles, kTileTab); i += 32) {
      TileInfo ti;
      get_tile<kNTok, C::kCG, C::kNPer>(tile0 + i * tstride, mt_off, args, rank, ti);
      tile_tab[i] = pack_tile(ti);
    }
  } else if (warp == 3 && lane == 0) {
    tma_prefetch_desc(&xmap);
  }
  tc_fence_before();
  if constexpr (kPair) cluster_sync_all();  // the peer's barriers must exist before remote arrivals
  else __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;
  const int n_tiles = *n_tiles_sm;
  constexpr uint32_t kAcol0 = C::kNumAcc * C::kAccCols;  // first column of the TMEM A ring
  const uint32_t w_u32 = smem_u32(smem_w);

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // lane 0: weight block (1-D bulk copy) + X tile (2-D TMA) on the stage's full barrier (tx bytes);
    // offset mode: all 32 lanes also copy the stage's (C, S) sums with 8-byte cp.async and arrive on
    // the same barrier when their copies land.
#ifdef W4A16_TRACE
    if (!kOffset && lane == 1 && tr && !kPair && !C::kDual) {  // MMA completion times (trace event 15)
      uint32_t n = 0;
      TileInfo ti;
      for (int it = 0; tile_at<kNTok, C::kCG, C::kNPer>(it, n_tiles, tile0, tstride, tile_tab, mt_off, args, rank, ti); ++it)
        for (int j = stage_beg(ti); j < stage_end(ti); ++j, ++n) {
          mbar_wait(&trbar[n & 7], (n >> 3) & 1);
          trace_at(tr, 15, n);
        }
    }
#endif
    constexpr bool gather = kGather;  // fused gather: all lanes issue gather4 loads
    if (kOffset || gather || lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      // gather: this lane loads 4-row group lane % kG4 of the X tile, k halves lane / kG4 (+ 32 / kG4 ...)
      constexpr int kG4 = (kNTok / 4 < 32) ? kNTok / 4 : 32;
      constexpr int kHalves = 2 * C::kGroupsPerStage;
      int src4[4] = {0, 0, 0, 0};
      Ring st;
      uint32_t pgs = 0;
      TileInfo ti;
      for (int it = 0; tile_at<kNTok, C::kCG, C::kNPer>(it, n_tiles, tile0, tstride, tile_tab, mt_off, args, rank, ti); ++it) {
        // per (expert, n-tile): kt k-groups of (gated ? 2 : 1) parts, stage j = bytes [j*kBlk, (j+1)*kBlk)
        const uint8_t* wsrc = args.wblocks + (static_cast<int64_t>(ti.e) * args.nt + ti.n_tile) *
                                                 static_cast<int64_t>(args.kt) * (kGated ? 2 : 1) * kPartBytes;
        // CTA pair: an MMA of N columns takes its first N/2 from the leader's X rows and the next N/2 from
        // the peer's, so the peer's X rows start at token N/2 of the tile (N = the tile's MMA N, below)
        const int x_row0 = ti.m_start + static_cast<int>(rank) *
                                            (min(kNTok, (ti.m_rows + 16 * C::kCG - 1) / (16 * C::kCG) * (16 * C::kCG)) / 2);
        if (gather) {  // source rows of this lane's 4-row group (rows past the tile's end repeat its first)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int m = (static_cast<int>(lane) % kG4) * 4 + q;
            const int i = ti.m_start + (m < ti.m_rows ? m : 0);
            src4[q] = __ldg(args.gather_rows + i) / args.gather_div;
          }
        }
        for (int j = stage_beg(ti); j < stage_end(ti); ++j) {
          mbar_wait(&empty[st.i], st.ph ^ 1);
          if (lane == 0) {
            trace_at(tr, 0, pgs++);
#if W4A16_GEMM_TAIL_TRIGGER
            // experiment: let the next kernel launch once this CTA's producer is within its last few
            // stages (the CTA exits ~NS stages later), hiding the dependent's launch latency
            if (it == n_tiles - 1 && j == max(stage_beg(ti), stage_end(ti) - W4A16_GEMM_TAIL_TRIGGER))
              asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
            mbar_arrive_expect_tx(&full[st.i], C::kBlk + C::kXBytes);
            if constexpr (C::kNPer == 2) {  // k-group j of n-tiles n_tile and n_tile + 1 (blocks kt apart)
              bulk_g2s_hint(smem_w + st.i * C::kBlk, wsrc + static_cast<int64_t>(j) * kPartBytes, kPartBytes,
                            &full[st.i], pol_w);
              bulk_g2s_hint(smem_w + st.i * C::kBlk + kPartBytes,
                            wsrc + (static_cast<int64_t>(args.kt) + j) * kPartBytes, kPartBytes, &full[st.i], pol_w);
            } else {
              bulk_g2s_hint(smem_w + st.i * C::kBlk, wsrc + static_cast<int64_t>(j) * C::kBlk, C::kBlk, &full[st.i],
                            pol_w);
            }
            if (!gather) {
              uint8_t* xs = smem_x + st.i * C::kXBytes;
#pragma unroll
              for (int h = 0; h < kHalves; ++h)
                tma_load_2d(xs + h * (C::kXRows * 128), &xmap, j * C::kGroupsPerStage * kTileK + h * 64,
                            x_row0, &full[st.i]);
            }
          }
          if (gather) {
            __syncwarp();  // lane 0's expect_tx is in: the gathers complete bytes on the same phase
            uint8_t* xs = smem_x + st.i * C::kXBytes;
            for (int op = static_cast<int>(lane); op < (kNTok / 4) * kHalves; op += 32) {
              const int g4 = op % kG4, h = op / kG4;  // kG4 == kNTok / 4 whenever ops exceed 32 lanes
              tma_gather4(xs + h * (C::kXRows * 128) + g4 * 512, &xmap, j * C::kGroupsPerStage * kTileK + h * 64,
                          src4[0], src4[1], src4[2], src4[3], &full[st.i]);
            }
          }
          if constexpr (kOffset) {
            // all 32 lanes copy and arrive every stage (fewer items than lanes: items are duplicated --
            // a lane arriving .noinc without its own cp.async in flight was observed never to fire);
            // every lane writes its own slot (duplicates land in the padding past the items, so no two
            // lanes write one address -- racecheck-clean); rows past the end read row 0 of the group
            // (never used)
            uint8_t* ss = smem_s + st.i * C::kSumBytes;
#pragma unroll
            for (int i0 = 0; i0 < (C::kSumItems > 32 ? C::kSumItems : 32); i0 += 32) {
              const int i = (i0 + lane) % C::kSumItems;
              const int g = i / kNTok, m = i % kNTok;
              int64_t r = ti.m_start + m < args.rows ? ti.m_start + m : 0;
              if (gather) r = __ldg(args.gather_rows + r) / args.gather_div;  // sums of x's rows
              cp_async_8(ss + (i0 + lane) * 8,
                         args.xsum + ((static_cast<int64_t>(j) * C::kGroupsPerStage + g) * args.sum_ld + r) * 2);
            }
            cp_async_arrive_noinc(&full[st.i]);
          }
          if (lane == 0) progress_at(0, pgs);
          st.next(C::kNS);
        }
      }
    }
  } else if (warp == 1 || warp == kMma2Warp) {
    // ------------------------------------------------------------ MMA issuer(s) (leader CTA of a pair)
    // whole warp runs the loop; one elected lane issues. Waiting on afull (all dequant warps of the
    // pair arrived, each after its own full barrier) also covers the stage's X tile(s).
    if constexpr (C::kDual) {
      const uint32_t my = warp == 1 ? 0u : 1u;  // stage parity this warp issues
      const uint32_t bar_in = my ? kTurnBar0 : kTurnBar1, bar_out = my ? kTurnBar1 : kTurnBar0;
      constexpr uint32_t idesc_full = make_idesc_f16(128, kNTok, kBF16);
      const uint32_t tb_u = __shfl_sync(0xffffffffu, tbase, 0);
      const uint32_t xs_u = __shfl_sync(0xffffffffu, smem_u32(smem_x), 0);
      Ring st, ar, acc;
      uint32_t gs = 0;
      TileInfo ti;
      for (int it = 0; tile_at<kNTok, 1, C::kNPer>(it, n_tiles, tile0, tstride, tile_tab, mt_off, args, rank, ti); ++it) {
        const uint32_t n_mma = min(kNTok, (ti.m_rows + 15) / 16 * 16);
        const uint32_t idesc = (idesc_full & ~(0x3Fu << 17)) | ((n_mma >> 3) << 17);
        const int jb = stage_beg(ti), je = stage_end(ti);
        for (int j = jb; j < je; ++j, ++gs) {
          if ((gs & 1u) == my) {
            if (j == jb) mbar_wait_warp<kPair>(&accempty[acc.i], acc.ph ^ 1);  // the tile's accumulator is free
            mbar_wait_warp<kPair>(&afull[ar.i], ar.ph);
            if (gs > 0) named_bar_sync(bar_in, 64);  // the other warp has issued stage gs - 1
            tc_fence_after();
            trace_at(tr, 4, gs);
            const uint32_t dcol = tb_u + acc.i * C::kAccCols;
            const uint64_t xdesc = make_sdesc_sw128(xs_u + st.i * C::kXBytes);
            const uint32_t acol = tb_u + kAcol0 + ar.i * C::kACols;
            if (elect_one()) {
              StageAsm<kNTok, (kMode == kModeNPair ? kModeGateUp : kMode), 1, false, 1>::issue(
                  dcol, acol, xdesc, idesc, static_cast<uint32_t>(j));
              tc_fence_before();
            }
            __syncwarp();
            if (!(it == n_tiles - 1 && j == je - 1)) named_bar_arrive(bar_out, 64);  // hand the turn over
            if (elect_one()) {
              umma_commit(&empty[st.i]);
              umma_commit(&aempty[ar.i]);
              if (j == je - 1) umma_commit(&accfull[acc.i]);  // in-order pipe: covers the other warp's MMAs
              trace_at(tr, 5, gs);
            }
            __syncwarp();
            progress_at(2, gs + 1);
          }
          st.next(C::kNS);
          ar.next(C::kNumA);
        }
        acc.next(C::kNumAcc);
      }
    } else if (warp == 1 && (!kPair || rank == 0)) {
      constexpr uint32_t idesc_full = make_idesc_f16(128 * C::kCG, kNTok, kBF16);
      // provably warp-uniform bases (shfl from lane 0): ptxas keeps the MMA operands in uniform registers
      const uint32_t tb_u = __shfl_sync(0xffffffffu, tbase, 0);
      const uint32_t xs_u = __shfl_sync(0xffffffffu, smem_u32(smem_x), 0);
      Ring st, ar, acc;
      uint32_t gs = 0;
      TileInfo ti;
      for (int it = 0; tile_at<kNTok, C::kCG, C::kNPer>(it, n_tiles, tile0, tstride, tile_tab, mt_off, args, rank, ti); ++it) {
        // MMA N sized to the tile's real tokens (multiple of 16 per CTA of the group): an expert's last,
        // partial m-tile costs tensor time in proportion to its rows, not to kNTok
        const uint32_t n_mma = min(kNTok, (ti.m_rows + 16 * C::kCG - 1) / (16 * C::kCG) * (16 * C::kCG));
        const uint32_t idesc = (idesc_full & ~(0x3Fu << 17)) | ((n_mma >> 3) << 17);
        if constexpr (!kOffset) {
          mbar_wait_warp<kPair>(&accempty[acc.i], acc.ph ^ 1);
          tc_fence_after();
          trace_at(tr, 6, it);
        }
        for (int j = stage_beg(ti); j < stage_end(ti); ++j, ++gs) {
          if constexpr (C::kSplitA) {
            // one A unit per k half: wait, issue its 8 MMAs (both parts), release it; the stage's smem
            // (X tile) after the second half
            const uint32_t dcol = tb_u + acc.i * C::kAccCols;
            const uint32_t d1 = dcol + (kMode == kModeKPair ? 0u : static_cast<uint32_t>(kNTok));
            const uint64_t xdesc = make_sdesc_sw128(xs_u + st.i * C::kXBytes);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              mbar_wait_warp<kPair>(&afull[ar.i], ar.ph);
              tc_fence_after();
              if (h == 0) trace_at(tr, 4, gs);
              const uint32_t acol = tb_u + kAcol0 + ar.i * C::kACols;
              const uint64_t b = xdesc + static_cast<uint64_t>(h * C::kXRows * 8);  // X k half h
              const uint32_t accf = (j != 0 || h != 0) ? 1u : 0u;
              if (elect_one()) {
                HalfAsm<C::kXRows, C::kCG, kMode == kModeKPair>::issue(dcol, d1, acol, b, accf, idesc);
                if constexpr (kPair) {
                  umma_commit_pair(&aempty[ar.i]);
                  if (h == 1) umma_commit_pair(&empty[st.i]);
                } else {
                  umma_commit(&aempty[ar.i]);
                  if (h == 1) umma_commit(&empty[st.i]);
                }
                if (h == 1) trace_at(tr, 5, gs);
#ifdef W4A16_TRACE
                if (h == 1 && !kPair && tr) umma_commit(&trbar[gs & 7]);
#endif
              }
              __syncwarp();
              ar.next(C::kNumA);
            }
            progress_at(2, gs + 1);
            st.next(C::kNS);
            continue;
          }
          if constexpr (kOffset)  // fresh partials per stage: accumulator slot free + A slot filled
            mbar_wait2_warp<kPair>(&accempty[acc.i], acc.ph ^ 1, &afull[ar.i], ar.ph);
          else
            mbar_wait_warp<kPair>(&afull[ar.i], ar.ph);
          tc_fence_after();
          trace_at(tr, 4, gs);
          const uint32_t dcol = tb_u + acc.i * C::kAccCols;
          const uint64_t xdesc = make_sdesc_sw128(xs_u + st.i * C::kXBytes);
          const uint32_t acol = tb_u + kAcol0 + ar.i * C::kACols;
          // one elected lane issues the stage's MMAs (generated PTX block, mma_stage.cuh) and commits
          if (elect_one()) {
            StageAsm<kNTok, (kMode == kModeNPair ? kModeGateUp : kMode), C::kCG, kOffset, C::kKSplit>::issue(
                dcol, acol, xdesc, idesc, static_cast<uint32_t>(j));
            trace_at(tr, 5, gs);
#ifdef W4A16_TRACE
            if (!kOffset && !kPair && tr) umma_commit(&trbar[gs & 7]);
#endif
            if constexpr (kPair) {
              umma_commit_pair(&empty[st.i]);
              umma_commit_pair(&aempty[ar.i]);
              if constexpr (kOffset) umma_commit_pair(&accfull[acc.i]);
            } else {
              umma_commit(&empty[st.i]);
              umma_commit(&aempty[ar.i]);
              if constexpr (kOffset) umma_commit(&accfull[acc.i]);
            }
            trace_at(tr, 20, gs);  // commits accepted
          }
          __syncwarp();
          trace_at(tr, 21, gs);  // warp reconverged
          progress_at(2, gs + 1);
          st.next(C::kNS);
          ar.next(C::kNumA);
          if constexpr (kOffset) acc.next(C::kNumAcc);
        }
        if constexpr (!kOffset) {
          if (elect_one()) {
            if constexpr (kPair) umma_commit_pair(&accfull[acc.i]);
            else umma_commit(&accfull[acc.i]);
          }
          __syncwarp();
          acc.next(C::kNumAcc);
        }
      }
    }
  } else if (warp < kEpiWarp0) {
    // ------------------------------------------------------------ dequant: int4 smem -> TMEM A ring
    // Whole-stage ring: group g (warps 2-5 / 6-9) takes the stages of parity g. Split ring (prefill):
    // group h converts k half h (chunks 2h, 2h+1 of both parts) of every stage into A unit 2s+h.
    // Inside a group warp w owns the TMEM lane quadrant w % 4 (32 weight rows).
    const int dw = warp - kDequantWarp0;
    const uint32_t my_par = dw / kDequantGroup;
    const uint32_t quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (quad * 32) << 16;
    const uint32_t code_off = row * 16;
    constexpr int kMyChunks = C::kSplitA ? kChunks / 2 : kChunks;  // 32-k chunks this warp converts
    const int c0 = C::kSplitA ? static_cast<int>(my_par) * kMyChunks : 0;
    Ring st, ar;
    if constexpr (C::kSplitA) {
      if (my_par) ar.next(C::kNumA);  // group 1 starts at the stage's second unit
    }
    uint32_t gs = 0;
    TileInfo ti;
    for (int it = 0; tile_at<kNTok, C::kCG, C::kNPer>(it, n_tiles, tile0, tstride, tile_tab, mt_off, args, rank, ti); ++it) {
      for (int j = stage_beg(ti); j < stage_end(ti); ++j, ++gs) {
        if (!C::kSplitA && (gs & 1u) != my_par) {
          st.next(C::kNS);
          ar.next(C::kNumA);
          continue;
        }
        mbar_wait(&full[st.i], st.ph);
        const bool trd = lane == 0 && quad == 0 && my_par == (C::kSplitA ? 0u : (gs & 1u));
        if (trd) trace_at(tr, 1, gs);
        const uint32_t blk = w_u32 + st.i * C::kBlk;
        uint4 v[C::kParts][kChunks];
        uint32_t sb[C::kParts], zb[C::kParts];
#pragma unroll
        for (int p = 0; p < C::kParts; ++p) {
          const uint32_t part = blk + p * kPartBytes;
#pragma unroll
          for (int c = 0; c < kMyChunks; ++c) v[p][c] = lds128(part + code_off + (c0 + c) * (kTileRows * 16));
          if constexpr (!kOffset) {
            zb[p] = lds_u8(part + kZeroOff + (row >> 1));
            sb[p] = lds_u16(part + kScaleOff + row * 2);
          } else {
            zb[p] = sb[p] = 0;
          }
        }
        if constexpr (C::kSplitA) {
          // unit layout: part p's two chunks at columns p * 32 + {0, 16}
          mbar_wait_cluster<kPair>(&aempty[ar.i], ar.ph ^ 1);
          tc_fence_after();
          if (trd) trace_at(tr, 2, gs);
          const uint32_t acol = tbase + lane_off + kAcol0 + ar.i * C::kACols;
#pragma unroll
          for (int p = 0; p < C::kParts; ++p) {
            const uint32_t z = (row & 1) ? (zb[p] >> 4) : (zb[p] & 15u);
            const auto ctx = Dq<kBF16>::make(z, static_cast<uint16_t>(sb[p]));
#pragma unroll
            for (int c = 0; c < kMyChunks; ++c) {
              uint32_t r[16];
              dequant_chunk<kBF16, true>(v[p][c], ctx, r);
              tmem_st_x16(acol + p * 32 + c * 16, r);
            }
          }
          tc_wait_st();
          tc_fence_before();
          __syncwarp();
          if (trd) trace_at(tr, 3, gs);
          if (trd) progress_at(1, gs + 1);
          if (lane == 0) {
            if constexpr (kPair) mbar_arrive_cluster(mapa_shared(&afull[ar.i], 0));
            else mbar_arrive(&afull[ar.i]);
            mbar_arrive(&empty[st.i]);
          }
          st.next(C::kNS);
          ar.next(C::kNumA);
          ar.next(C::kNumA);
          continue;
        }
        mbar_wait_cluster<kPair>(&aempty[ar.i], ar.ph ^ 1);
        tc_fence_after();
        if (trd) trace_at(tr, 2, gs);
        const uint32_t acol = tbase + lane_off + kAcol0 + ar.i * C::kACols;
#pragma unroll
        for (int p = 0; p < C::kParts; ++p) {
          if constexpr (kOffset) {
#pragma unroll
            for (int c = 0; c < kChunks; ++c) {
              uint32_t r[16];
              raw_chunk<kBF16>(v[p][c], r);
              tmem_st_x16(acol + p * 64 + c * 16, r);
            }
          } else {
            const uint32_t z = (row & 1) ? (zb[p] >> 4) : (zb[p] & 15u);
            const auto ctx = Dq<kBF16>::make(z, static_cast<uint16_t>(sb[p]));
#pragma unroll
            for (int c = 0; c < kChunks; ++c) {
              uint32_t r[16];
              dequant_chunk<kBF16, true>(v[p][c], ctx, r);
              tmem_st_x16(acol + p * 64 + c * 16, r);
            }
          }
        }
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (trd) trace_at(tr, 3, gs);
        if (lane == 0) trace_at(tr, 16 + quad, gs);  // every quad's arrival (per-SMSP skew)
        if (trd) progress_at(1, gs + 1);
        if (lane == 0) {
          if constexpr (kPair) mbar_arrive_cluster(mapa_shared(&afull[ar.i], 0));
          else mbar_arrive(&afull[ar.i]);
          mbar_arrive(&empty[st.i]);
        }
        st.next(C::kNS);
        ar.next(C::kNumA);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue: TMEM -> HBM
    const uint32_t quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t lane_off = (quad * 32) << 16;
    uint16_t* out = reinterpret_cast<uint16_t*>(args.out);
    Ring acc, st;
    uint32_t egs = 0;
    const bool tre = lane == 0 && quad == 0;
    TileInfo ti;
    for (int it = 0; tile_at<kNTok, C::kCG, C::kNPer>(it, n_tiles, tile0, tstride, tile_tab, mt_off, args, rank, ti); ++it) {
      if (tre) trace_at(tr, 9, egs);
      uint16_t* ocol = out + ti.n_tile * kTileRows + row;
      // output row of the tile's token m (identity, or scattered through args.out_rows)
      auto orow = [&](int m) -> int64_t {
        const int64_t i = static_cast<int64_t>(ti.m_start) + m;
        return (args.out_rows ? static_cast<int64_t>(__ldg(args.out_rows + i)) : i) * args.ldo;
      };
      // Stores of 16 tokens: lane l (< 16) computes token m0 + l's output row offset once and the values
      // of all 16 tokens are computed branch-free first (per-token `if (m < rows) { compute; store }`
      // blocks serialised a ~200-cycle dependent chain per token: 27k cycles per 128x128 tile, measured
      // with tools/trace_gemm.py).
      auto row_off16 = [&](int m0) -> int64_t {
        const int mm = m0 + static_cast<int>(lane & 15);
        return mm < ti.m_rows ? orow(mm) : 0;
      };
      // The warp's 16-token x 32-column block then goes through shared memory (token-major, 64 B per
      // token) and out as 16-byte stores, 2 per lane (16 2-byte stores per lane issued ~1 per 125 cycles).
      uint8_t* const my_stage = epi_sm + (warp - kEpiWarp0) * (C::kEpiStageBytes / 4);
      auto store16_staged = [&](int m0, int64_t ro, const uint16_t (&hb)[16], int col_off, int buf) {
        uint8_t* sb = my_stage + buf * 1024;
        const uint32_t sa = smem_u32(sb);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(sa + i * 64 + lane * 2), "h"(hb[i]) : "memory");
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int sgi = static_cast<int>(lane) + 32 * j;  // 16-byte segment: token sgi / 4, quarter sgi % 4
          const int t = sgi >> 2, q = sgi & 3;
          const int64_t o = __shfl_sync(0xffffffffu, ro, t);
          const uint4 v = lds128(sa + t * 64 + q * 16);
          if (m0 + t < ti.m_rows)
            *reinterpret_cast<uint4*>(ocol - lane + o + col_off + q * 8) = v;
        }
        __syncwarp();  // the staging block is rewritten by the next call
      };
      // both n-tiles of an n-pair chunk: one round of shared-memory staging (two buffers), so the two
      // outputs' store latencies overlap instead of adding up
      auto store16x2_staged = [&](int m0, int64_t ro, const uint16_t (&hb)[16], const uint16_t (&hu)[16]) {
        const uint32_t sa = smem_u32(my_stage), sb = sa + 1024;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(sa + i * 64 + lane * 2), "h"(hb[i]) : "memory");
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(sb + i * 64 + lane * 2), "h"(hu[i]) : "memory");
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int sgi = static_cast<int>(lane) + 32 * j;
          const int t = sgi >> 2, q = sgi & 3;
          const int64_t o = __shfl_sync(0xffffffffu, ro, t);
          const uint4 v0 = lds128(sa + t * 64 + q * 16);
          const uint4 v1 = lds128(sb + t * 64 + q * 16);
          if (m0 + t < ti.m_rows) {
            *reinterpret_cast<uint4*>(ocol - lane + o + q * 8) = v0;
            *reinterpret_cast<uint4*>(ocol - lane + o + kTileRows + q * 8) = v1;
          }
        }
        __syncwarp();
      };
      if constexpr (kOffset) {
        // gate|up, or the two n-tiles of an n-pair tile; else one (k-pair parts summed)
        constexpr int kOuts = (kGated || C::kNPer == 2) ? 2 : 1;
        const int m_rows = ti.m_rows;
        float a[kOuts][kNTok];
#pragma unroll
        for (int o = 0; o < kOuts; ++o)
#pragma unroll
          for (int i = 0; i < kNTok; ++i) a[o][i] = 0.f;
        for (int j = stage_beg(ti); j < stage_end(ti); ++j) {
          mbar_wait(&full[st.i], st.ph);
          if (tre) trace_at(tr, 6, egs);
          const uint32_t blk = w_u32 + st.i * C::kBlk;
          const uint32_t sums = smem_u32(smem_s + st.i * C::kSumBytes);
          float sc[C::kParts], zf[C::kParts];
#pragma unroll
          for (int p = 0; p < C::kParts; ++p) {
            const uint32_t part = blk + p * kPartBytes;
            sc[p] = act_bits_to_float<kBF16>(lds_u16(part + kScaleOff + row * 2));
            const uint32_t zb = lds_u8(part + kZeroOff + (row >> 1));
            zf[p] = static_cast<float>((row & 1) ? (zb >> 4) : (zb & 15u));
          }
          mbar_wait_cluster<kPair>(&accfull[acc.i], acc.ph);
          tc_fence_after();
          if (tre) trace_at(tr, 7, egs);
          const uint32_t dcol = tbase + lane_off + acc.i * C::kAccCols;
#pragma unroll
          for (int cb = 0; cb < kNTok / kEpiChunk; ++cb) {
            if (cb * kEpiChunk < m_rows) {  // warp-uniform: only the tile's real tokens
              uint32_t r[C::kParts][C::kKSplit][kEpiChunk];
#pragma unroll
              for (int p = 0; p < C::kParts; ++p)
#pragma unroll
                for (int hs = 0; hs < C::kKSplit; ++hs)
                  tmem_ld_x4(dcol + (p * C::kKSplit + hs) * kNTok + cb * kEpiChunk, r[p][hs]);
              tc_wait_ld();
#pragma unroll
              for (int i = 0; i < kEpiChunk; ++i) {
                const int m = cb * kEpiChunk + i;
                float2 csg[C::kGroupsPerStage];  // (C, S) of token m per k-group of the stage (broadcast)
#pragma unroll
                for (int g = 0; g < C::kGroupsPerStage; ++g) csg[g] = lds_f2(sums + (g * kNTok + m) * 8);
#pragma unroll
                for (int p = 0; p < C::kParts; ++p) {
                  const int g = kMode == kModeKPair ? p : 0;
                  const int o = (kGated || C::kNPer == 2) ? p : 0;
                  const float2 cs = csg[g];
                  float pv = __uint_as_float(r[p][0][i]);
#pragma unroll
                  for (int hs = 1; hs < C::kKSplit; ++hs) pv += __uint_as_float(r[p][hs][i]);
                  const float d = pv - fmaf(zf[p], cs.y, cs.x);
                  a[o][m] = fmaf(sc[p], d, a[o][m]);
                }
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (tre) trace_at(tr, 8, egs);
          ++egs;
          if (tre) progress_at(3, egs);
          if (lane == 0) {
            if constexpr (kPair) mbar_arrive_cluster(mapa_shared(&accempty[acc.i], 0));
            else mbar_arrive(&accempty[acc.i]);
            mbar_arrive(&empty[st.i]);
          }
          if (tre) trace_at(tr, 22, egs - 1);
          acc.next(C::kNumAcc);
          st.next(C::kNS);
        }
        if (args.splits > 1) {  // split-K: fp32 partials, summed (and activated) by splitk_finalize
          float* pbase = args.part + (static_cast<int64_t>(ti.split) * args.rows + ti.m_start) * args.part_ld +
                         ti.n_tile * kTileRows + row;
#pragma unroll
          for (int m = 0; m < kNTok; ++m) {
            if (m < m_rows) {
#pragma unroll
              for (int o = 0; o < kOuts; ++o)  // up half at +n_out; an n-pair's second tile at +128
                pbase[static_cast<int64_t>(m) * args.part_ld + o * (kGated ? args.ldo : kTileRows)] = a[o][m];
            }
          }
        } else {
          float hv[kNTok];  // the stored (rounded) outputs, for the fused sums below
          if (m_rows <= args.direct_rows) {
            // few real tokens (decode: ~2 rows per expert at DS-R1 T=64): compute only those and store
            // them straight from registers -- a warp writes 32 consecutive rows (64 B) per token --
            // instead of 16 tokens' SiLU plus the shared-memory staging round (the tile-end epilogue
            // delays the next tile's first folds, and through them its MMAs)
#pragma unroll
            for (int m = 0; m < kNTok; ++m) hv[m] = 0.f;
#pragma unroll
            for (int m = 0; m < kDirectRows; ++m) {
              if (m < m_rows) {  // warp-uniform
                float v;
                if constexpr (kGated) v = silu_f(a[0][m]) * a[1][m];
                else v = a[0][m];
                const uint16_t b = to_act_bits<kBF16>(v);
                hv[m] = act_bits_to_float<kBF16>(b);
                uint16_t* dst = ocol + orow(m);
                *dst = b;
                if constexpr (C::kNPer == 2) dst[kTileRows] = to_act_bits<kBF16>(a[kOuts - 1][m]);
              }
            }
          } else {
#pragma unroll
          for (int m0 = 0; m0 < kNTok; m0 += 16) {
            const int64_t ro = row_off16(m0);
            uint16_t hb[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int m = m0 + i;
              float v;
              if constexpr (kGated) v = silu_f(a[0][m]) * a[1][m];
              else v = a[0][m];
              hb[i] = to_act_bits<kBF16>(v);
              hv[m] = m < m_rows ? act_bits_to_float<kBF16>(hb[i]) : 0.f;
            }
            store16_staged(m0, ro, hb, 0, 0);
            if constexpr (C::kNPer == 2) {  // the pair's second n-tile
              uint16_t hu[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) hu[i] = to_act_bits<kBF16>(a[kOuts - 1][m0 + i]);
              store16_staged(m0, ro, hu, kTileRows, 1);
            }
          }
          }
          if constexpr (kGated && kNTok <= 16) {
            if (args.osum != nullptr) {
              // The tile's 128 rows are exactly one k-group of the next (down) GEMM: its per-token
              // (C, S) = (sum_r c_r h_r, sum_r h_r), c_r the decode offset of k = r (Dq::offset_bits).
              const float cr = act_bits_to_float<kBF16>(Dq<kBF16>::offset_bits(row & 7));
              const uint32_t ew = warp - kEpiWarp0;
              // a rolled loop over the real tokens: one copy of the shuffle tree instead of kNTok
              // (ptxas wraps every shuffle under a data-dependent branch in divergence handling:
              // ~1000 of the kernel's ~4600 SASS instructions, all of it cold tile-end code)
#pragma unroll 1
              for (int m = 0; m < m_rows; ++m) {
                float sc = cr * hv[m], ss = hv[m];
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                  sc += __shfl_xor_sync(0xffffffffu, sc, o);
                  ss += __shfl_xor_sync(0xffffffffu, ss, o);
                }
                if (lane == 0) red_sm[ew * 16 + m] = make_float2(sc, ss);
              }
              named_bar_sync(1, 128);  // the 4 epilogue warps
              if (ew == 0 && static_cast<int>(lane) < m_rows) {
                float2 t = red_sm[lane];
#pragma unroll
                for (int w2 = 1; w2 < 4; ++w2) {
                  const float2 u = red_sm[w2 * 16 + lane];
                  t.x += u.x;
                  t.y += u.y;
                }
                args.osum[static_cast<int64_t>(ti.n_tile) * args.osum_ld + ti.m_start + lane] = t;
              }
              named_bar_sync(1, 128);  // scratch reused by the next tile
            }
          }
        }
      } else {
        mbar_wait_cluster<kPair>(&accfull[acc.i], acc.ph);
        tc_fence_after();
        if (tre) trace_at(tr, 7, it);
        const uint32_t dcol = tbase + lane_off + acc.i * C::kAccCols;
        constexpr bool kTwo = kGated || C::kNPer == 2;  // two accumulators: gate|up, or two n-tiles
        constexpr int kNChunks = kNTok / 16;
        auto load = [&](int cb, uint32_t (&g)[16], uint32_t (&u)[16]) {
          tmem_ld_x16(dcol + cb * 16, g);
          if constexpr (kTwo) tmem_ld_x16(dcol + kNTok + cb * 16, u);
        };
        auto landed = [&](uint32_t (&g)[16], uint32_t (&u)[16]) {
          tc_wait_ld();
          reg_fence16(g);
          if constexpr (kTwo) reg_fence16(u);
        };
        auto process = [&](int cb, const uint32_t (&g)[16], const uint32_t (&u)[16]) {
          const int64_t ro = row_off16(cb * 16);
          uint16_t hb[16];
          if constexpr (kGated) {
            if (tre) trace_at(tr, 14, it * 32 + cb * 2);
#pragma unroll
            for (int i = 0; i < 16; ++i)
              hb[i] = to_act_bits<kBF16>(silu_f(__uint_as_float(g[i])) * __uint_as_float(u[i]));
            store16_staged(cb * 16, ro, hb, 0, 0);
            if (tre) trace_at(tr, 14, it * 32 + cb * 2 + 1);
          } else if constexpr (C::kNPer == 2) {  // second accumulator = the next n-tile's columns
            if (tre) trace_at(tr, 14, it * 32 + cb * 2);
            uint16_t hu[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              hb[i] = to_act_bits<kBF16>(__uint_as_float(g[i]));
              hu[i] = to_act_bits<kBF16>(__uint_as_float(u[i]));
            }
            store16x2_staged(cb * 16, ro, hb, hu);
            if (tre) trace_at(tr, 14, it * 32 + cb * 2 + 1);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) hb[i] = to_act_bits<kBF16>(__uint_as_float(g[i]));
            store16_staged(cb * 16, ro, hb, 0, 0);
          }
        };
        // TMEM loads of chunk cb + 1 overlap the conversion and stores of chunk cb (two register sets)
        uint32_t gA[16], uA[16], gB[16], uB[16];
        load(0, gA, uA);
        landed(gA, uA);
        if constexpr (kNChunks == 1) {
          process(0, gA, uA);
        } else {
#pragma unroll 1
          for (int cb = 0; cb < kNChunks; cb += 2) {
            load(cb + 1, gB, uB);
            process(cb, gA, uA);
            landed(gB, uB);
            if (cb + 2 < kNChunks) load(cb + 2, gA, uA);
            process(cb + 1, gB, uB);
            landed(gA, uA);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (tre) trace_at(tr, 8, it);
        if (lane == 0) {
          if constexpr (kPair) mbar_arrive_cluster(mapa_shared(&accempty[acc.i], 0));
          else mbar_arrive(&accempty[acc.i]);
        }
        acc.next(C::kNumAcc);
      }
    }
  }

#ifdef W4A16_TRACE
  if (lane == 0 && tr) tr[26 * kTraceCap + warp] = clock64();  // each warp's arrival at the exit barrier
#endif
  tc_fence_before();
  if constexpr (kPair) {
    __syncwarp();
    cluster_sync_all();  // both CTAs done: no MMA reads this TMEM and no remote arrival is in flight
  } else {
    __syncthreads();
  }
  if (threadIdx.x == 0) progress_at(3, 1000000);  // CTA reached the exit barrier
#ifdef W4A16_TRACE
  if (threadIdx.x == 0 && g_w4_trace) {  // every CTA: %globaltimer (ns) at entry (row 28) and exit (row 29)
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    g_w4_trace[28 * kTraceCap + blockIdx.x] = static_cast<long long>(t_entry);
    g_w4_trace[29 * kTraceCap + blockIdx.x] = static_cast<long long>(t1);
  }
#endif
  if (warp == 0) {
    __syncwarp();  // tcgen05.dealloc is .sync.aligned: the producer's lanes must be reconverged, or the
                   // columns stay allocated and the next launch's tcgen05.alloc on this SM waits forever
    tc_fence_after();
    if constexpr (kPair) tmem_dealloc_pair<512>(tbase);
    else tmem_dealloc<512>(tbase);
  }
}

__global__ void debug_stamp_kernel(unsigned long long* buf) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const unsigned long long n = atomicAdd(buf, 1ull);
  if (n < 4095) buf[1 + n] = t;
}

// ---------------------------------------------------------------------------------------------
// Split-K finalize: out[r][n] = act(f(sum_s part[s][r][...])), f = silu(gate) * up when gated, for
// rows r < *row_limit. One thread per 4 outputs.
template <bool kBF16, bool kGated>
__global__ void splitk_finalize_kernel(const float* __restrict__ part, int splits, int64_t rows, int64_t n_out,
                                       const int32_t* __restrict__ row_limit, const int32_t* __restrict__ out_rows,
                                       uint16_t* __restrict__ out) {
  griddep_wait();  // PDL
  const int64_t r = blockIdx.y;
  if (r >= __ldg(row_limit)) return;
  const int64_t n = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  if (n >= n_out) return;
  const int64_t ld = (kGated ? 2 : 1) * n_out;
  float4 g = make_float4(0.f, 0.f, 0.f, 0.f), u = g;
  for (int sidx = 0; sidx < splits; ++sidx) {
    const float* pr = part + (static_cast<int64_t>(sidx) * rows + r) * ld + n;
    const float4 a = *reinterpret_cast<const float4*>(pr);
    g.x += a.x, g.y += a.y, g.z += a.z, g.w += a.w;
    if constexpr (kGated) {
      const float4 b = *reinterpret_cast<const float4*>(pr + n_out);
      u.x += b.x, u.y += b.y, u.z += b.z, u.w += b.w;
    }
  }
  float v[4] = {g.x, g.y, g.z, g.w};
  if constexpr (kGated) {
    v[0] = silu_f(g.x) * u.x, v[1] = silu_f(g.y) * u.y, v[2] = silu_f(g.z) * u.z, v[3] = silu_f(g.w) * u.w;
  }
  uint2 o;
  o.x = static_cast<uint32_t>(to_act_bits<kBF16>(v[0])) | static_cast<uint32_t>(to_act_bits<kBF16>(v[1])) << 16;
  o.y = static_cast<uint32_t>(to_act_bits<kBF16>(v[2])) | static_cast<uint32_t>(to_act_bits<kBF16>(v[3])) << 16;
  const int64_t orow = out_rows ? static_cast<int64_t>(__ldg(out_rows + r)) : r;
  *reinterpret_cast<uint2*>(out + orow * n_out + n) = o;
}

// ---------------------------------------------------------------------------------------------
// Standalone dequant: packed blocks -> dense W[e][n][k] (activation dtype). Test/oracle aid; it
// runs exactly the dequantiser the GEMM runs. One thread per (e, nt, kt, part, chunk, row).
template <bool kBF16>
__global__ void w4_dequant_kernel(const uint8_t* __restrict__ wblocks, int64_t n_units, int nt, int kt, int parts,
                                  uint16_t* __restrict__ out) {
  const int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (u >= n_units) return;
  const int row = u % kTileRows;
  int64_t r = u / kTileRows;
  const int c = r % kChunks; r /= kChunks;
  const int p = r % parts; r /= parts;
  const int k_t = r % kt; r /= kt;
  const int n_t = r % nt;
  const int64_t e = r / nt;
  const uint8_t* part = wblocks + (((e * nt + n_t) * kt + k_t) * parts + p) * static_cast<int64_t>(kPartBytes);
  const uint16_t sb = reinterpret_cast<const uint16_t*>(part + kScaleOff)[row];
  const uint32_t zb = part[kZeroOff + (row >> 1)];
  const uint32_t z = (row & 1) ? (zb >> 4) : (zb & 15u);
  const auto ctx = Dq<kBF16>::make(z, sb);
  const uint4 v = *reinterpret_cast<const uint4*>(part + (c * kTileRows + row) * 16);
  uint32_t o[16];
  dequant_chunk<kBF16>(v, ctx, o);
  const int64_t n_rows = static_cast<int64_t>(nt) * kTileRows;  // rows per part
  const int64_t K = static_cast<int64_t>(kt) * kTileK;
  const int64_t n = p * n_rows + n_t * kTileRows + row;
  uint4* dst = reinterpret_cast<uint4*>(out + (e * parts * n_rows + n) * K + k_t * kTileK + c * 32);
#pragma unroll
  for (int i = 0; i < 4; ++i) dst[i] = make_uint4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
}

// AWQ (qweight [E][K][N/8] int32, scales [E][K/G][N], qzeros [E][K/G][N/8] int32; nibble of column
// n at shift 4*slot_of(n%8)) -> packed blocks. One thread per (e, nt, kt, part, chunk, row).
__global__ void w4_repack_awq_kernel(const uint32_t* __restrict__ qw, const uint16_t* __restrict__ sc,
                                     const uint32_t* __restrict__ qz, int64_t n_units, int nt, int kt, int parts,
                                     uint8_t* __restrict__ wblocks) {
  const int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (u >= n_units) return;
  const int row = u % kTileRows;
  int64_t r = u / kTileRows;
  const int c = r % kChunks; r /= kChunks;
  const int p = r % parts; r /= parts;
  const int k_t = r % kt; r /= kt;
  const int n_t = r % nt;
  const int64_t e = r / nt;
  const int64_t N = static_cast<int64_t>(parts) * nt * kTileRows;
  const int64_t K = static_cast<int64_t>(kt) * kTileK;
  const int64_t n = static_cast<int64_t>(p) * nt * kTileRows + n_t * kTileRows + row;
  const int nshift = 4 * slot_of(static_cast<int>(n & 7));
  const uint32_t* qcol = qw + e * K * (N / 8) + n / 8;
  uint32_t words[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    uint32_t acc = 0;
#pragma unroll
    for (int el = 0; el < 8; ++el) {
      const int64_t k = static_cast<int64_t>(k_t) * kTileK + c * 32 + w * 8 + el;
      const uint32_t q = (__ldg(qcol + k * (N / 8)) >> nshift) & 15u;
      acc |= q << (4 * slot_of(el));
    }
    words[w] = acc;
  }
  uint8_t* part = wblocks + (((e * nt + n_t) * kt + k_t) * parts + p) * static_cast<int64_t>(kPartBytes);
  *reinterpret_cast<uint4*>(part + (c * kTileRows + row) * 16) = make_uint4(words[0], words[1], words[2], words[3]);
  if (c == 0) {
    const int64_t g = k_t;  // one group per k-tile (group size 128)
    reinterpret_cast<uint16_t*>(part + kScaleOff)[row] = sc[(e * (K / kGroup) + g) * N + n];
    if ((row & 1) == 0) {
      const uint32_t* zrow = qz + (e * (K / kGroup) + g) * (N / 8);
      const uint32_t z0 = (__ldg(zrow + n / 8) >> nshift) & 15u;
      const int64_t n1 = n + 1;
      const uint32_t z1 = (__ldg(zrow + n1 / 8) >> (4 * slot_of(static_cast<int>(n1 & 7)))) & 15u;
      part[kZeroOff + (row >> 1)] = static_cast<uint8_t>(z0 | (z1 << 4));
    }
  }
}

}  // namespace w4

// =============================================================================================
// C ABI
// =============================================================================================
using namespace w4;

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int make_x_map(CUtensorMap* map, const void* x, int64_t rows, int64_t K, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return W4_ERR_CUDA;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(K * 2)};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(x), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? W4_OK : W4_ERR_CUDA;
}

// SM count of the current device (cached per device ordinal; the persistent grid is one CTA per SM)
int sm_count() {
  static const int forced = getenv("W4A16_GRID") ? atoi(getenv("W4A16_GRID")) : 0;  // debug override
  if (forced > 0) return forced;
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;  // no device (planning on a build host): B200
  if (dev < 64) {
    const int c = cache[dev].load(std::memory_order_relaxed);
    if (c > 0) return c;
  }
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return 148;
  if (dev < 64) cache[dev].store(n, std::memory_order_relaxed);
  return n;
}

template <int kNTok, int kMode, bool kBF16, bool kOffset, bool kPair, bool kGather = false>
int launch_gemm(const GemmArgs& a, const void* x, int64_t rows, int64_t K, int grid, cudaStream_t st) {
  using C = Cfg<kNTok, kMode, kOffset, kPair>;
  auto kern = w4a16_moe_gemm_kernel<kNTok, kMode, kBF16, kOffset, kPair, kGather>;
  static std::atomic<unsigned long long> attr{0};
  if (!ensure_smem_attr(kern, C::kSmemBytes, attr)) return W4_ERR_CUDA;
  CUtensorMap map;
  if (make_x_map(&map, x, rows, K, a.gather_rows ? 1 : C::kXRows) != W4_OK) return W4_ERR_CUDA;  // gather4: 1-row box
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kPair ? (grid & ~1) : grid);
  cfg.blockDim = dim3(kNumThreads);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  if (kPair) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = 2;
    at[na].val.clusterDim.y = 1;
    at[na++].val.clusterDim.z = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  if (cudaLaunchKernelEx(&cfg, kern, a, map) != cudaSuccess) return W4_ERR_CUDA;
  return cudaGetLastError() == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}

template <int kMode, bool kBF16>
int dispatch_ntok(int ntok, bool offset, bool pair, const GemmArgs& a, const void* x, int64_t rows, int64_t K,
                  int grid, cudaStream_t st) {
  if (offset && pair && ntok == 16) return launch_gemm<16, kMode, kBF16, true, true>(a, x, rows, K, grid, st);
  if (offset && ntok == 16) return launch_gemm<16, kMode, kBF16, true, false>(a, x, rows, K, grid, st);
  if (offset && ntok == 32) return launch_gemm<32, kMode, kBF16, true, false>(a, x, rows, K, grid, st);
  if (pair) {
    if (ntok == 64) return launch_gemm<64, kMode, kBF16, false, true>(a, x, rows, K, grid, st);
    if (ntok == 128) return launch_gemm<128, kMode, kBF16, false, true>(a, x, rows, K, grid, st);
  }
  switch (ntok) {
    case 16: return launch_gemm<16, kMode, kBF16, false, false>(a, x, rows, K, grid, st);
    case 32: return launch_gemm<32, kMode, kBF16, false, false>(a, x, rows, K, grid, st);
    case 64: return launch_gemm<64, kMode, kBF16, false, false>(a, x, rows, K, grid, st);
    case 128: return launch_gemm<128, kMode, kBF16, false, false>(a, x, rows, K, grid, st);
    default: return W4_ERR_ARG;
  }
}

// fused-gather gate/up kernels (decode 16-token offset mode, or the prefill token tiles)
template <bool kBF16>
int dispatch_gather(int ntok, bool offset, const GemmArgs& a, const void* x, int64_t rows, int64_t K, int grid,
                    cudaStream_t st) {
  if (offset && ntok == 16) return launch_gemm<16, kModeGateUp, kBF16, true, false, true>(a, x, rows, K, grid, st);
  if (offset && ntok == 32) return launch_gemm<32, kModeGateUp, kBF16, true, false, true>(a, x, rows, K, grid, st);
  switch (ntok) {
    case 16: return launch_gemm<16, kModeGateUp, kBF16, false, false, true>(a, x, rows, K, grid, st);
    case 32: return launch_gemm<32, kModeGateUp, kBF16, false, false, true>(a, x, rows, K, grid, st);
    case 64: return launch_gemm<64, kModeGateUp, kBF16, false, false, true>(a, x, rows, K, grid, st);
    case 128: return launch_gemm<128, kModeGateUp, kBF16, false, false, true>(a, x, rows, K, grid, st);
    default: return W4_ERR_ARG;
  }
}

template <int kMode, bool kBF16>
int dispatch_prefill(int ntok, const GemmArgs& a, const void* x, int64_t rows, int64_t K, int grid, cudaStream_t st) {
  if (ntok == 32) return launch_gemm<32, kMode, kBF16, false, false>(a, x, rows, K, grid, st);
  if (ntok == 64) return launch_gemm<64, kMode, kBF16, false, false>(a, x, rows, K, grid, st);
  if (ntok == 128) return launch_gemm<128, kMode, kBF16, false, false>(a, x, rows, K, grid, st);
  return W4_ERR_ARG;
}

// n-pair block mode for the prefill down projection from this token tile up (W4A16_NPAIR_MIN_NTOK,
// default 64; 0 disables). Same box, DS-R1 layer: 64-token tiles (T=1024) 1.600 -> 1.572 ms with
// n-pair; 32-token tiles (Qwen3 T=256) unchanged, so they keep k-pair stages.
int npair_min_ntok() {
  static const int v = [] {
    const char* e = getenv("W4A16_NPAIR_MIN_NTOK");
    const int x = e ? atoi(e) : 64;
    return x <= 0 ? 1 << 30 : x;
  }();
  return v;
}

// n-pair stages for the decode (offset-mode) down projection (W4A16_DECODE_NPAIR=0 disables)
bool decode_npair_enabled() {
  static const bool on = [] {
    const char* e = getenv("W4A16_DECODE_NPAIR");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

// Experiment knob: W4A16_PREFILL_PAIR=1 runs the prefill (64/128-token) kernels on CTA pairs.
bool prefill_pairs_enabled() {
  static const bool on = [] {
    const char* e = getenv("W4A16_PREFILL_PAIR");
    return e && atoi(e) != 0;
  }();
  return on;
}

// Experiment knob: W4A16_PAIR=1 runs the decode kernel on CTA pairs.
bool pairs_enabled() {
  static const bool on = [] {
    const char* e = getenv("W4A16_PAIR");
    return e && atoi(e) != 0;
  }();
  return on;
}

}  // namespace

namespace {
// Split-K factor for a decode-mode launch: with few (expert, n-tile) tiles the 148 SMs are not all
// busy (T = 1 touches 8 DS-R1 experts -> 128 gate/up tiles; Mixtral decode -> 64 down tiles of 56
// stages). Minimise waves x (stages per unit + per-unit overhead) over S, from an upper estimate
// of the tile count (touched experts <= min(E, rows)).
int choose_splits(int64_t rows, int64_t num_experts, int nt, int n_stages, int grid) {
  // (Measured alternatives, tools/gpu_splits2.sh: the expected touched-expert count instead of this upper
  // estimate, without the early exit, gained 1.6-3.5 % at DS-R1 T = 2 / 4 but lost 1-6 % at T = 1 / 8 and
  // Qwen3 T = 16; kept as is.)
  const int64_t tiles = std::min<int64_t>(num_experts, rows) * nt;
  if (tiles >= 2 * grid || n_stages < 4) return 1;
  double best = 1e30;
  int best_s = 1;
  for (int sp = 1; sp <= std::min(16, n_stages / 2); ++sp) {
    const int64_t units = tiles * sp;
    const double waves = static_cast<double>((units + grid - 1) / grid);
    const double cost = waves * (static_cast<double>(n_stages) / sp + 1.5) + (sp > 1 ? 1.0 : 0.0);
    if (cost < best - 1e-9) { best = cost; best_s = sp; }
  }
  return best_s;
}

struct GemmPlan {
  int ntok, mode, splits;
  bool offset;
};

GemmPlan plan_gemm(int64_t rows, int64_t K, int64_t num_experts, int64_t n_out, int gated, bool has_xsum,
                   int ntok) {
  GemmPlan pl;
  pl.ntok = ntok > 0 ? ntok : w4a16_pick_ntok(rows, num_experts);
  const int kt = static_cast<int>(K / kTileK), nt = static_cast<int>(n_out / kTileRows);
  pl.offset = has_xsum && pl.ntok <= w4a16_decode_max_ntok();
  // k-pair (two k-groups per 17 KB stage) for decode tiles; at 128 tokens the X tile dominates a stage
  // (64 KB for a k-pair -> only 2 smem stages), so 128-token tiles use one group per stage
  pl.mode = gated ? kModeGateUp : ((kt % 2 == 0 && pl.ntok <= 64) ? kModeKPair : kModePlain);
  // prefill down projection: two n-tiles per stage share the X tile (halves the X smem traffic)
  // (not for 128-token tiles of short K: their single 256-column accumulator stalls the MMA on
  // every few-stage tile's epilogue -- Qwen3 down, K/128 = 6: T=8192 layer 0.740 -> 0.725 ms in plain
  // stages with two accumulator stages; DS-R1 / Mixtral / Llama, K/128 >= 16, keep n-pair)
  if (!gated && !pl.offset && pl.ntok >= 32 && pl.ntok >= npair_min_ntok() && nt % 2 == 0 &&
      (pl.ntok < 128 || kt >= 12))
    pl.mode = kModeNPair;
  // decode down projection: n-pair stages too (one k-group of two n-tiles on one X tile): tiles of
  // K/128 stages instead of K/256 k-pair stages, half the X bytes per stage -- unless even an upper
  // estimate of the n-pair tiles leaves SMs idle, where k-pair's twice as many tiles cover more of
  // them (same box: Qwen3 T=1 30.7 -> 28.7 us, Mixtral T=1 59.5 -> 58.4 us, T=16 154 -> 150 us;
  // DS-R1, with >= 148 n-pair tiles from T=1 on, measured better with n-pair)
  if (!gated && pl.offset && nt % 2 == 0 && decode_npair_enabled() &&
      std::min<int64_t>(num_experts, rows) * (nt / 2) >= sm_count())
    pl.mode = kModeNPair;
  const int n_stages = kt / (pl.mode == kModeKPair ? 2 : 1);
  pl.splits = (pl.offset && rows < (1 << 20)) ? choose_splits(rows, num_experts, nt, n_stages, sm_count()) : 1;
  // experiment: W4A16_SPLITS_GU / W4A16_SPLITS_DN force the decode split-K factor of gate/up / down launches
  static const int force_gu = getenv("W4A16_SPLITS_GU") ? atoi(getenv("W4A16_SPLITS_GU")) : 0;
  static const int force_dn = getenv("W4A16_SPLITS_DN") ? atoi(getenv("W4A16_SPLITS_DN")) : 0;
  const int force = gated ? force_gu : force_dn;
  if (pl.offset && rows < (1 << 20) && force > 0) pl.splits = std::min(force, n_stages);
  return pl;
}
}  // namespace

extern "C" {

/* Debug aid (not in the public header's hot path): per-stage clock64 timeline of CTA 0 of every
 * subsequent grouped-GEMM launch into `buf` (int64 [10][4096], caller-owned, device), or off (null). */
int w4a16_debug_trace(void* buf) {
  return cudaMemcpyToSymbol(g_w4_trace, &buf, sizeof(buf)) == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}
int w4a16_debug_trace_cta(int cta) {
  return cudaMemcpyToSymbol(g_w4_trace_cta, &cta, sizeof(cta)) == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}

/* Debug aid: one thread appends %globaltimer (ns) to buf[1 + n] (n = buf[0]++): stream-ordered
 * timestamps around captured work, to see whether consecutive graph replays overlap. */
int w4a16_debug_stamp(void* buf, cudaStream_t stream) {
  debug_stamp_kernel<<<1, 1, 0, stream>>>(static_cast<unsigned long long*>(buf));
  return cudaGetLastError() == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}

int w4a16_tile_rows(void) { return kTileRows; }

/* The launch plan w4a16_grouped_gemm_ws would use (no GPU needed): token tile, block mode (0 plain,
 * 1 gate|up, 2 k-pair, 3 n-pair), decode (offset-code) or not, split-K factor. */
int w4a16_gemm_plan(int64_t rows, int64_t K, int64_t num_experts, int64_t n_out, int gated, int has_xsum, int ntok,
                    int* out_ntok, int* out_mode, int* out_offset, int* out_splits) {
  if (rows <= 0 || K <= 0 || K % kTileK || n_out <= 0 || n_out % kTileRows || num_experts <= 0) return W4_ERR_SHAPE;
  const GemmPlan pl = plan_gemm(rows, K, num_experts, n_out, gated, has_xsum != 0, ntok);
  if (out_ntok) *out_ntok = pl.ntok;
  if (out_mode) *out_mode = pl.mode;
  if (out_offset) *out_offset = pl.offset ? 1 : 0;
  if (out_splits) *out_splits = pl.splits;
  return W4_OK;
}
int w4a16_decode_max_ntok(void) {
  const char* e = getenv("W4A16_DECODE_MAX_NTOK");  // (read per call: the A/B knob)
  const int v = e ? atoi(e) : 16;
  return v >= 32 ? 32 : (v >= 16 ? 16 : 0);
}
int w4a16_tile_k(void) { return kTileK; }
int w4a16_part_bytes(void) { return kPartBytes; }

int w4a16_pick_ntok(int64_t rows, int64_t num_experts) {
  // Token tile = the one minimising (relative cost of one m-tile) x (expected m-tiles per touched
  // expert), with an expert's row count ~ Binomial(rows, 1/E) (normal approximation; exact for one
  // expert). The relative m-tile costs are measured whole-layer times with one m-tile per expert
  // (Mixtral T=8: 137.5 / 188.7 / 190.6 / 192.9 us for 16 / 32 / 64 / 128-token tiles) -- the
  // 16-token tile runs in offset-code mode. Measured (tools/ntok_probe.py): the rule it replaced
  // (mean + 2.5 sigma rows in ONE m-tile) picked 32 at Mixtral T=48 (16: 204 -> 177 us) and 128 at
  // Mixtral T=192 (64: 231 -> 218 us), and agrees with this one everywhere else measured.
  static const double kCost[4] = {1.0, 1.37, 1.39, 1.45};
  const int kTiles[4] = {16, 32, 64, 128};
  if (num_experts <= 1) {
    // one dense matrix: its tiles are full, where the offset-code epilogue's per-token fold costs
    // more than the costs above assume (measured: M=16 in 16-token offset tiles 14.3 -> 17.0 us,
    // N=K=1024 8.2 -> 10.2 us) -- the smallest tile holding mean + 2.5 sigma rows, as before
    const double est = static_cast<double>(rows) + 2.5 * sqrt(static_cast<double>(rows));
    return est <= 16.0 ? 16 : est <= 32.0 ? 32 : est <= 64.0 ? 64 : 128;
  }
  const double E = static_cast<double>(num_experts);
  const double mu = static_cast<double>(rows) / E;
  const double sd = E > 1.0 ? sqrt(mu * (1.0 - 1.0 / E)) : 0.0;
  double best = 1e300;
  int pick = 16;
  for (int i = 0; i < 4; ++i) {
    const double n = kTiles[i];
    double m;  // expected m-tiles of a touched expert: 1 + sum_k P(rows > k n)
    if (sd == 0.0) {
      m = std::max(1.0, ceil(mu / n));
    } else {
      m = 1.0;
      for (double t = n; t < mu + 8.0 * sd + n; t += n) m += 0.5 * erfc((t + 0.5 - mu) / (sqrt(2.0) * sd));
    }
    const double cost = kCost[i] * m;
    if (cost < best - 1e-12) {
      best = cost;
      pick = kTiles[i];
    }
  }
  return pick;
}

int64_t w4a16_group_sums_ld(int64_t rows) { return (rows + 1) & ~int64_t(1); }


int64_t w4a16_grouped_gemm_ws_bytes(int64_t rows, int64_t K, int64_t num_experts, int64_t n_out, int gated,
                                    int ntok) {
  if (rows <= 0 || K % kTileK || n_out % kTileRows || num_experts <= 0) return 0;
  const GemmPlan pl = plan_gemm(rows, K, num_experts, n_out, gated, true, ntok);
  return pl.splits > 1 ? static_cast<int64_t>(pl.splits) * rows * (gated ? 2 : 1) * n_out * 4 : 0;
}

static int grouped_gemm_impl(const void* x, int64_t x_rows, const int32_t* gather_rows, int gather_div,
                             int64_t rows, int64_t K, const uint8_t* wblocks, int64_t num_experts,
                          int64_t n_out, int gated, const int32_t* expert_counts, const int32_t* expert_offsets,
                          const float* xsum, float* osum, const int32_t* out_rows, void* out, int dtype, int ntok,
                          void* ws, int64_t ws_bytes, cudaStream_t stream) {
  if (!x || !wblocks || !expert_counts || !expert_offsets || !out) return W4_ERR_ARG;
  if (K <= 0 || K % kTileK || n_out <= 0 || n_out % kTileRows) return W4_ERR_SHAPE;
  if (num_experts <= 0 || num_experts > kMaxExperts) return W4_ERR_SHAPE;
  if (dtype != W4_DTYPE_F16 && dtype != W4_DTYPE_BF16) return W4_ERR_DTYPE;
  // TMA reads of x and the epilogue's 16-byte stores
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out)) & 15) return W4_ERR_ARG;
  if (rows <= 0) return W4_OK;
  if (ntok != 0 && ntok != 16 && ntok != 32 && ntok != 64 && ntok != 128) return W4_ERR_ARG;
  GemmPlan pl = plan_gemm(rows, K, num_experts, n_out, gated, xsum != nullptr, ntok);
  const int64_t need = pl.splits > 1 ? static_cast<int64_t>(pl.splits) * rows * (gated ? 2 : 1) * n_out * 4 : 0;
  if (pl.splits > 1 && (!ws || ws_bytes < need)) pl.splits = 1;  // no / too small workspace: no split-K
  GemmArgs a;
  a.wblocks = wblocks;
  a.expert_counts = expert_counts;
  a.expert_offsets = expert_offsets;
  a.out = out;
  a.ldo = n_out;
  a.num_experts = static_cast<int>(num_experts);
  a.nt = static_cast<int>(n_out / kTileRows);
  a.kt = static_cast<int>(K / kTileK);
  a.xsum = xsum;
  a.sum_ld = w4a16_group_sums_ld(gather_rows ? x_rows : rows);  // xsum covers x's rows
  a.osum_ld = w4a16_group_sums_ld(rows);
  a.gather_rows = gather_rows;
  a.gather_div = gather_div;
  a.rows = rows;
  a.splits = pl.splits;
  static const int direct_rows = [] {
    const char* e = getenv("W4A16_DIRECT_ROWS");
    const int v = e ? atoi(e) : kDirectRows;
    return v < 0 ? 0 : (v > kDirectRows ? kDirectRows : v);
  }();
  a.direct_rows = direct_rows;
  a.part = static_cast<float*>(ws);
  a.part_ld = (gated ? 2 : 1) * n_out;
  // the decode gate/up epilogue writes the output's group sums itself; otherwise a sums pass follows
  const bool fused_osum = osum != nullptr && gated && pl.offset && pl.ntok <= 16 && pl.splits == 1;
  a.osum = fused_osum ? reinterpret_cast<float2*>(osum) : nullptr;
  a.out_rows = out_rows;
  if (out_rows && osum) return W4_ERR_ARG;  // sums of a scattered output are not supported
  // CTA pairs (cta_group::2) measured slower at decode token counts (an M=256 x N=16 MMA with 8-row B
  // halves executes ~4x slower than two M=128 ones): opt-in only (W4A16_PAIR=1)
  const bool pair = !gather_rows && pl.splits == 1 && a.nt % 2 == 0 && (pl.offset ? pairs_enabled() : prefill_pairs_enabled());
  const int grid = sm_count();
  const bool bf = dtype == W4_DTYPE_BF16;
  int rc;
  if (gather_rows) {  // fused gather: gate/up projection only
    if (pl.mode != kModeGateUp) return W4_ERR_ARG;
    rc = bf ? dispatch_gather<true>(pl.ntok, pl.offset, a, x, x_rows, K, grid, stream)
            : dispatch_gather<false>(pl.ntok, pl.offset, a, x, x_rows, K, grid, stream);
  } else if (pl.mode == kModeGateUp)
    rc = bf ? dispatch_ntok<kModeGateUp, true>(pl.ntok, pl.offset, pair, a, x, x_rows, K, grid, stream)
            : dispatch_ntok<kModeGateUp, false>(pl.ntok, pl.offset, pair, a, x, x_rows, K, grid, stream);
  else if (pl.mode == kModeKPair)
    rc = bf ? dispatch_ntok<kModeKPair, true>(pl.ntok, pl.offset, pair, a, x, x_rows, K, grid, stream)
            : dispatch_ntok<kModeKPair, false>(pl.ntok, pl.offset, pair, a, x, x_rows, K, grid, stream);
  else if (pl.mode == kModeNPair && pl.offset && pl.ntok == 32)  // decode n-pair, no CTA pairs
    rc = bf ? launch_gemm<32, kModeNPair, true, true, false>(a, x, x_rows, K, grid, stream)
            : launch_gemm<32, kModeNPair, false, true, false>(a, x, x_rows, K, grid, stream);
  else if (pl.mode == kModeNPair && pl.offset)
    rc = bf ? launch_gemm<16, kModeNPair, true, true, false>(a, x, x_rows, K, grid, stream)
            : launch_gemm<16, kModeNPair, false, true, false>(a, x, x_rows, K, grid, stream);
  else if (pl.mode == kModeNPair)
    rc = bf ? dispatch_prefill<kModeNPair, true>(pl.ntok, a, x, x_rows, K, grid, stream)
            : dispatch_prefill<kModeNPair, false>(pl.ntok, a, x, x_rows, K, grid, stream);
  else
    rc = bf ? dispatch_ntok<kModePlain, true>(pl.ntok, pl.offset, pair, a, x, x_rows, K, grid, stream)
            : dispatch_ntok<kModePlain, false>(pl.ntok, pl.offset, pair, a, x, x_rows, K, grid, stream);
  if (rc != W4_OK) return rc;
  if (pl.splits > 1) {
  const int thr = 128;
  const dim3 fgrid(static_cast<unsigned>((n_out / 4 + thr - 1) / thr), static_cast<unsigned>(rows));
  auto* o = static_cast<uint16_t*>(out);
  const int32_t* lim = expert_offsets + num_experts;
  if (gated)
    bf ? launch_pdl(splitk_finalize_kernel<true, true>, fgrid, thr, 0, stream, a.part, pl.splits, rows, n_out, lim, out_rows, o)
       : launch_pdl(splitk_finalize_kernel<false, true>, fgrid, thr, 0, stream, a.part, pl.splits, rows, n_out, lim, out_rows, o);
  else
    bf ? launch_pdl(splitk_finalize_kernel<true, false>, fgrid, thr, 0, stream, a.part, pl.splits, rows, n_out, lim, out_rows, o)
       : launch_pdl(splitk_finalize_kernel<false, false>, fgrid, thr, 0, stream, a.part, pl.splits, rows, n_out, lim, out_rows, o);
    if (cudaGetLastError() != cudaSuccess) return W4_ERR_CUDA;
  }
  if (osum != nullptr && !fused_osum)
    return w4a16_group_sums(out, rows, n_out, expert_offsets + num_experts, dtype, osum, stream);
  return W4_OK;
}

int w4a16_grouped_gemm_ws(const void* x, int64_t rows, int64_t K, const uint8_t* wblocks, int64_t num_experts,
                          int64_t n_out, int gated, const int32_t* expert_counts, const int32_t* expert_offsets,
                          const float* xsum, float* osum, const int32_t* out_rows, void* out, int dtype, int ntok,
                          void* ws, int64_t ws_bytes, cudaStream_t stream) {
  return grouped_gemm_impl(x, rows, nullptr, 1, rows, K, wblocks, num_experts, n_out, gated, expert_counts,
                           expert_offsets, xsum, osum, out_rows, out, dtype, ntok, ws, ws_bytes, stream);
}

int w4a16_grouped_gemm_gather(const void* x, int64_t x_rows, const int32_t* gather_rows, int gather_div, int64_t rows,
                              int64_t K, const uint8_t* wblocks, int64_t num_experts, int64_t n_out, int gated,
                              const int32_t* expert_counts, const int32_t* expert_offsets, const float* xsum,
                              float* osum, void* out, int dtype, int ntok, void* ws, int64_t ws_bytes,
                              cudaStream_t stream) {
  if (!gather_rows || gather_div <= 0 || x_rows <= 0) return W4_ERR_ARG;
  return grouped_gemm_impl(x, x_rows, gather_rows, gather_div, rows, K, wblocks, num_experts, n_out, gated,
                           expert_counts, expert_offsets, xsum, osum, nullptr, out, dtype, ntok, ws, ws_bytes, stream);
}

int w4a16_grouped_gemm(const void* x, int64_t rows, int64_t K, const uint8_t* wblocks, int64_t num_experts,
                       int64_t n_out, int gated, const int32_t* expert_counts, const int32_t* expert_offsets,
                       const float* xsum, void* out, int dtype, int ntok, cudaStream_t stream) {
  return w4a16_grouped_gemm_ws(x, rows, K, wblocks, num_experts, n_out, gated, expert_counts, expert_offsets, xsum,
                               nullptr, nullptr, out, dtype, ntok, nullptr, 0, stream);
}

int w4a16_dequant(const uint8_t* wblocks, int64_t num_experts, int64_t n_rows, int64_t K, int parts, int dtype,
                  void* out, cudaStream_t stream) {
  if (!wblocks || !out) return W4_ERR_ARG;
  if (parts != 1 && parts != 2) return W4_ERR_ARG;
  if (K <= 0 || K % kTileK || n_rows <= 0 || n_rows % (kTileRows * parts)) return W4_ERR_SHAPE;
  if (dtype != W4_DTYPE_F16 && dtype != W4_DTYPE_BF16) return W4_ERR_DTYPE;
  const int nt = static_cast<int>(n_rows / parts / kTileRows), kt = static_cast<int>(K / kTileK);
  const int64_t units = num_experts * nt * kt * parts * kChunks * kTileRows;
  const int thr = 256;
  const int64_t blocks = (units + thr - 1) / thr;
  if (dtype == W4_DTYPE_BF16)
    w4_dequant_kernel<true><<<blocks, thr, 0, stream>>>(wblocks, units, nt, kt, parts, static_cast<uint16_t*>(out));
  else
    w4_dequant_kernel<false><<<blocks, thr, 0, stream>>>(wblocks, units, nt, kt, parts, static_cast<uint16_t*>(out));
  return cudaGetLastError() == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}

int64_t w4a16_packed_bytes(int64_t num_experts, int64_t n_rows, int64_t K) {
  if (n_rows % kTileRows || K % kTileK) return -1;
  return num_experts * (n_rows / kTileRows) * (K / kTileK) * static_cast<int64_t>(kPartBytes);
}

int w4a16_repack_awq(const int32_t* qweight, const void* scales, const int32_t* qzeros, int64_t num_experts,
                     int64_t K, int64_t n_rows, int parts, int group_size, uint8_t* wblocks, cudaStream_t stream) {
  if (!qweight || !scales || !qzeros || !wblocks) return W4_ERR_ARG;
  if (group_size != kGroup) return W4_ERR_GROUP;
  if (parts != 1 && parts != 2) return W4_ERR_ARG;
  if (K <= 0 || K % kTileK || n_rows <= 0 || n_rows % (kTileRows * parts)) return W4_ERR_SHAPE;
  const int nt = static_cast<int>(n_rows / parts / kTileRows), kt = static_cast<int>(K / kTileK);
  const int64_t units = num_experts * nt * kt * parts * kChunks * kTileRows;
  const int thr = 256;
  w4_repack_awq_kernel<<<(units + thr - 1) / thr, thr, 0, stream>>>(
      reinterpret_cast<const uint32_t*>(qweight), static_cast<const uint16_t*>(scales),
      reinterpret_cast<const uint32_t*>(qzeros), units, nt, kt, parts, wblocks);
  return cudaGetLastError() == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}

}  // extern "C"

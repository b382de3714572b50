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
//   warps 10-13 epilogue : tcgen05.ld of the fp32 accumulator, SiLU(gate)*up when fused, store
// The dequantised weights never touch shared memory or HBM: int4 goes HBM -> smem -> registers ->
// TMEM -> tensor core. Barriers: smem full/empty, TMEM-A full/empty, accumulator full/empty.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include "ptx.cuh"
#include "w4_format.cuh"
#include "w4a16_moe.h"

namespace w4 {

constexpr int kNumThreads = 14 * 32;
constexpr int kDequantWarp0 = 2;
constexpr int kNumDequantWarps = 8;
constexpr int kEpiWarp0 = 10;
constexpr int kMaxExperts = 1024;
constexpr int kSmemBudget = 225 * 1024;

struct GemmArgs {
  const uint8_t* wblocks;        // [E][NT][KT][parts * kPartBytes]
  const int32_t* expert_counts;  // [E]
  const int32_t* expert_offsets; // [E+1]; rows of X (and of out) owned by expert e
  void* out;                     // [rows][NT*128] activation dtype
  int64_t ldo;
  int num_experts, nt, kt;
};

// kScaleEpi (decode, small token tiles): the dequant warps produce the exact integers (q - z) and
// the MMA writes one fp32 partial per k-tile (= per quantisation group) into a TMEM ring; the
// epilogue warps fold acc += s[row, g] * partial in registers. This removes the per-weight HMUL2
// from the dequant (the scale is applied once per group per output instead of once per weight)
// and is numerically at least as accurate as dequantise-then-MMA. Otherwise (prefill, large token
// tiles) the dequant applies the scale and the MMA accumulates across k-tiles in TMEM.
// Block modes: how the two 8.5 KB parts of a 17 KB stage are used.
constexpr int kModePlain = 0;   // one part (one k-group) per stage
constexpr int kModeGateUp = 1;  // part 0 = gate rows, part 1 = up rows, same k-group (fused SwiGLU)
constexpr int kModeKPair = 2;   // parts = two consecutive k-groups of the same rows (down proj.)

template <int kNTok, int kMode, bool kScaleEpi>
struct Cfg {
  static constexpr bool kGated = kMode == kModeGateUp;
  static constexpr int kParts = kMode == kModePlain ? 1 : 2;
  static constexpr int kGroupsPerStage = kMode == kModeKPair ? 2 : 1;
  static constexpr int kBlk = kParts * kPartBytes;
  static constexpr int kXBytes = kGroupsPerStage * kNTok * kTileK * 2;  // X tile, 64-wide 128B-swizzle atoms
  // one accumulator / partial stage: a partial per part in kScaleEpi mode, else gate|up or one
  static constexpr int kAccCols = (kScaleEpi || kGated) ? kParts * kNTok : kNTok;
  static constexpr int kACols = kParts * (kTileK / 2);  // fp16 pairs per 32-bit column
  static constexpr int kNumAcc = kScaleEpi ? 4 : ((2 * kAccCols + 2 * kACols <= 512) ? 2 : 1);
  static constexpr int kNumA0 = (512 - kNumAcc * kAccCols) / kACols;
  static constexpr int kNumA = kNumA0 > 4 ? 4 : kNumA0;
  static constexpr int kStageBytes = kBlk + kXBytes;
  static constexpr int kFixed = 2048 + 4 * (kMaxExperts + 1);  // barriers + tile table
  static constexpr int kNS0 = (kSmemBudget - kFixed - 1024) / kStageBytes;
  static constexpr int kNS = kNS0 > 12 ? 12 : kNS0;
  static constexpr int kEmptyArrivals = kNumDequantWarps + 1 + (kScaleEpi ? 4 : 0);
  // X ring first (needs 1024 B alignment for the 128B swizzle atoms), then weights.
  static constexpr int kSmemBytes = 1024 + kNS * kStageBytes + kFixed;
  static_assert(kNumA >= 2, "TMEM budget");
  static_assert(kNS >= 2, "smem budget");
  static_assert(kXBytes % 1024 == 0, "X tile alignment");
  static_assert(!kScaleEpi || kNTok <= 32, "register accumulators");
};

struct TileInfo {
  int e, n_tile, m_start, m_rows;
};

// Static persistent schedule: tile t -> (expert, n-tile, m-tile); m-tiles of one (expert, n-tile)
// are adjacent so concurrently running CTAs share that weight block through L2.
template <int kNTok>
__device__ __forceinline__ bool get_tile(int t, const int* mt_off, const GemmArgs& a, TileInfo& ti) {
  const int total = mt_off[a.num_experts] * a.nt;
  if (t >= total) return false;
  int lo = 0, hi = a.num_experts;  // find e with mt_off[e]*nt <= t < mt_off[e+1]*nt
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (mt_off[mid] * a.nt <= t) lo = mid; else hi = mid;
  }
  const int e = lo;
  const int me = mt_off[e + 1] - mt_off[e];
  const int local = t - mt_off[e] * a.nt;
  const int m_tile = local % me;
  ti.e = e;
  ti.n_tile = local / me;
  ti.m_start = __ldg(a.expert_offsets + e) + m_tile * kNTok;
  ti.m_rows = min(kNTok, __ldg(a.expert_counts + e) - m_tile * kNTok);
  return true;
}

__device__ __forceinline__ float silu_f(float g) { return g / (1.0f + __expf(-g)); }

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

struct Ring {  // (stage, phase) iterator of an mbarrier ring
  int i = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next(int n) {
    if (++i == n) { i = 0; ph ^= 1; }
  }
};

template <int kNTok, int kMode, bool kBF16, bool kScaleEpi>
__global__ void __launch_bounds__(kNumThreads, 1)
    w4a16_moe_gemm_kernel(const GemmArgs args, const __grid_constant__ CUtensorMap xmap) {
  using C = Cfg<kNTok, kMode, kScaleEpi>;
  constexpr bool kGated = C::kGated;
  const int n_stages = args.kt / C::kGroupsPerStage;  // stages per tile
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_x = smem;                                  // [NS][kXBytes]
  uint8_t* smem_w = smem + C::kNS * C::kXBytes;            // [NS][kBlk]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_w + C::kNS * C::kBlk);
  uint64_t* full = bars;
  uint64_t* empty = full + C::kNS;
  uint64_t* afull = empty + C::kNS;
  uint64_t* aempty = afull + C::kNumA;
  uint64_t* accfull = aempty + C::kNumA;
  uint64_t* accempty = accfull + C::kNumAcc;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(accempty + C::kNumAcc);
  int* mt_off = reinterpret_cast<int*>(bars + 256);

  const uint32_t warp = warp_idx();
  const uint32_t lane = lane_id();

  if (warp == 0) {
    tmem_alloc<512>(tmem_holder);
  } else if (warp == 1 && lane == 0) {
    for (int i = 0; i < C::kNS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], C::kEmptyArrivals); }
    for (int i = 0; i < C::kNumA; ++i) { mbar_init(&afull[i], kNumDequantWarps); mbar_init(&aempty[i], 1); }
    for (int i = 0; i < C::kNumAcc; ++i) { mbar_init(&accfull[i], 1); mbar_init(&accempty[i], 4); }
    fence_mbar_init();
  } else if (warp == 2) {
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
  } else if (warp == 3 && lane == 0) {
    tma_prefetch_desc(&xmap);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_holder;
  constexpr uint32_t kAcol0 = C::kNumAcc * C::kAccCols;  // first column of the TMEM A ring
  const uint32_t w_u32 = smem_u32(smem_w);

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      Ring st;
      TileInfo ti;
      for (int t = blockIdx.x; get_tile<kNTok>(t, mt_off, args, ti); t += gridDim.x) {
        // per (expert, n-tile): kt k-groups of (gated ? 2 : 1) parts, stage j = bytes [j*kBlk, (j+1)*kBlk)
        const uint8_t* wsrc = args.wblocks + (static_cast<int64_t>(ti.e) * args.nt + ti.n_tile) *
                                                 static_cast<int64_t>(args.kt) * (kGated ? 2 : 1) * kPartBytes;
        for (int j = 0; j < n_stages; ++j) {
          mbar_wait(&empty[st.i], st.ph ^ 1);
          mbar_arrive_expect_tx(&full[st.i], C::kBlk + C::kXBytes);
          bulk_g2s_hint(smem_w + st.i * C::kBlk, wsrc + static_cast<int64_t>(j) * C::kBlk, C::kBlk, &full[st.i],
                        pol_w);
          uint8_t* xs = smem_x + st.i * C::kXBytes;
#pragma unroll
          for (int h = 0; h < 2 * C::kGroupsPerStage; ++h)
            tma_load_2d(xs + h * (kNTok * 128), &xmap, j * C::kGroupsPerStage * kTileK + h * 64, ti.m_start,
                        &full[st.i]);
          st.next(C::kNS);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_f16(128, kNTok, kBF16);
      Ring st, ar, acc;
      TileInfo ti;
      for (int t = blockIdx.x; get_tile<kNTok>(t, mt_off, args, ti); t += gridDim.x) {
        if constexpr (!kScaleEpi) {
          mbar_wait(&accempty[acc.i], acc.ph ^ 1);
          tc_fence_after();
        }
        for (int j = 0; j < n_stages; ++j) {
          if constexpr (kScaleEpi) {  // fresh partials per stage (one per k-group)
            mbar_wait(&accempty[acc.i], acc.ph ^ 1);
          }
          mbar_wait(&full[st.i], st.ph);
          mbar_wait(&afull[ar.i], ar.ph);
          tc_fence_after();
          const uint32_t dcol = tbase + acc.i * C::kAccCols;
          const uint32_t xaddr = smem_u32(smem_x + st.i * C::kXBytes);
          const uint32_t acol = tbase + kAcol0 + ar.i * C::kACols;
#pragma unroll
          for (int p = 0; p < C::kParts; ++p) {
            // k-pair: part p reads the second 128-k half of the X tile; gate/up: both read the same
            const uint32_t xp = xaddr + (kMode == kModeKPair ? p * 2 * (kNTok * 128) : 0);
            const uint32_t dp = dcol + ((kScaleEpi || kGated) ? p * kNTok : 0);
#pragma unroll
            for (int kk = 0; kk < kTileK / 16; ++kk) {
              const uint64_t bdesc = make_sdesc_sw128(xp + (kk >> 2) * (kNTok * 128) + (kk & 3) * 32);
              const uint32_t accum = (kScaleEpi || kGated) ? (kScaleEpi ? (kk != 0) : ((j | kk) != 0))
                                                           : ((j | p | kk) != 0);
              umma_ts_f16(dp, acol + p * 64 + kk * 8, bdesc, idesc, accum);
            }
          }
          umma_commit(&empty[st.i]);
          umma_commit(&aempty[ar.i]);
          st.next(C::kNS);
          ar.next(C::kNumA);
          if constexpr (kScaleEpi) {
            umma_commit(&accfull[acc.i]);
            acc.next(C::kNumAcc);
          }
        }
        if constexpr (!kScaleEpi) {
          umma_commit(&accfull[acc.i]);
          acc.next(C::kNumAcc);
        }
      }
    }
  } else if (warp < kEpiWarp0) {
    // ------------------------------------------------------------ dequant: int4 smem -> TMEM A ring
    const int dw = warp - kDequantWarp0;
    const uint32_t quad = warp & 3;
    const int row = quad * 32 + lane;
    const int c0 = (dw >> 2) * 2;  // this warp's two 32-wide k chunks of the 128-wide tile
    const uint32_t lane_off = (quad * 32) << 16;
    const uint32_t code_off = (c0 * kTileRows + row) * 16;
    Ring st, ar;
    TileInfo ti;
    for (int t = blockIdx.x; get_tile<kNTok>(t, mt_off, args, ti); t += gridDim.x) {
      for (int j = 0; j < n_stages; ++j) {
        mbar_wait(&full[st.i], st.ph);
        const uint32_t blk = w_u32 + st.i * C::kBlk;
        uint4 v[C::kParts][2];
        uint32_t sb[C::kParts], zb[C::kParts];
#pragma unroll
        for (int p = 0; p < C::kParts; ++p) {
          const uint32_t part = blk + p * kPartBytes;
          v[p][0] = lds128(part + code_off);
          v[p][1] = lds128(part + code_off + kTileRows * 16);
          zb[p] = lds_u8(part + kZeroOff + (row >> 1));
          if constexpr (!kScaleEpi) sb[p] = lds_u16(part + kScaleOff + row * 2);
          else sb[p] = 0;
        }
        mbar_wait(&aempty[ar.i], ar.ph ^ 1);
        tc_fence_after();
        const uint32_t acol = tbase + lane_off + kAcol0 + ar.i * C::kACols;
#pragma unroll
        for (int p = 0; p < C::kParts; ++p) {
          const uint32_t z = (row & 1) ? (zb[p] >> 4) : (zb[p] & 15u);
          const auto ctx = Dq<kBF16>::make(z, static_cast<uint16_t>(sb[p]));
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            uint32_t r[16];
            dequant_chunk<kBF16, !kScaleEpi>(v[p][cc], ctx, r);
            tmem_st_x16(acol + p * 64 + (c0 + cc) * 16, r);
          }
        }
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&afull[ar.i]);
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
    TileInfo ti;
    for (int t = blockIdx.x; get_tile<kNTok>(t, mt_off, args, ti); t += gridDim.x) {
      uint16_t* obase = out + static_cast<int64_t>(ti.m_start) * args.ldo + ti.n_tile * kTileRows + row;
      if constexpr (kScaleEpi) {
        float a[C::kParts][kNTok];
#pragma unroll
        for (int p = 0; p < C::kParts; ++p)
#pragma unroll
          for (int i = 0; i < kNTok; ++i) a[p][i] = 0.f;
        for (int j = 0; j < n_stages; ++j) {
          mbar_wait(&full[st.i], st.ph);
          const uint32_t blk = w_u32 + st.i * C::kBlk;
          float sc[C::kParts];
#pragma unroll
          for (int p = 0; p < C::kParts; ++p) sc[p] = act_bits_to_float<kBF16>(lds_u16(blk + p * kPartBytes + kScaleOff + row * 2));
          mbar_wait(&accfull[acc.i], acc.ph);
          tc_fence_after();
          const uint32_t dcol = tbase + lane_off + acc.i * C::kAccCols;
          uint32_t r[C::kParts][kNTok];
#pragma unroll
          for (int p = 0; p < C::kParts; ++p)
#pragma unroll
            for (int cb = 0; cb < kNTok / 16; ++cb)
              tmem_ld_x16(dcol + p * kNTok + cb * 16, *reinterpret_cast<uint32_t(*)[16]>(&r[p][cb * 16]));
          tc_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&accempty[acc.i]);
            mbar_arrive(&empty[st.i]);
          }
#pragma unroll
          for (int p = 0; p < C::kParts; ++p)
#pragma unroll
            for (int i = 0; i < kNTok; ++i) a[p][i] = fmaf(sc[p], __uint_as_float(r[p][i]), a[p][i]);
          acc.next(C::kNumAcc);
          st.next(C::kNS);
        }
#pragma unroll
        for (int m = 0; m < kNTok; ++m) {
          if (m < ti.m_rows) {
            float v;
            if constexpr (kGated) v = silu_f(a[0][m]) * a[1][m];
            else if constexpr (kMode == kModeKPair) v = a[0][m] + a[1][m];
            else v = a[0][m];
            obase[static_cast<int64_t>(m) * args.ldo] = to_act_bits<kBF16>(v);
          }
        }
      } else {
        mbar_wait(&accfull[acc.i], acc.ph);
        tc_fence_after();
        const uint32_t dcol = tbase + lane_off + acc.i * C::kAccCols;
#pragma unroll 1
        for (int cb = 0; cb < kNTok / 16; ++cb) {
          uint32_t g[16];
          tmem_ld_x16(dcol + cb * 16, g);
          if constexpr (kGated) {
            uint32_t u[16];
            tmem_ld_x16(dcol + kNTok + cb * 16, u);
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int m = cb * 16 + i;
              if (m < ti.m_rows) {
                const float gv = __uint_as_float(g[i]), uv = __uint_as_float(u[i]);
                obase[static_cast<int64_t>(m) * args.ldo] = to_act_bits<kBF16>(silu_f(gv) * uv);
              }
            }
          } else {
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int m = cb * 16 + i;
              if (m < ti.m_rows) obase[static_cast<int64_t>(m) * args.ldo] = to_act_bits<kBF16>(__uint_as_float(g[i]));
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&accempty[acc.i]);
        acc.next(C::kNumAcc);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
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

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int kNTok, int kMode, bool kBF16, bool kScaleEpi>
int launch_gemm(const GemmArgs& a, const CUtensorMap& map, int grid, cudaStream_t st) {
  using C = Cfg<kNTok, kMode, kScaleEpi>;
  auto kern = w4a16_moe_gemm_kernel<kNTok, kMode, kBF16, kScaleEpi>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes) != cudaSuccess)
      return W4_ERR_CUDA;
    attr = true;
  }
  kern<<<grid, kNumThreads, C::kSmemBytes, st>>>(a, map);
  return cudaGetLastError() == cudaSuccess ? W4_OK : W4_ERR_CUDA;
}

template <int kMode, bool kBF16>
int dispatch_ntok(int ntok, const GemmArgs& a, const CUtensorMap& m, int grid, cudaStream_t st) {
  switch (ntok) {
    case 16: return launch_gemm<16, kMode, kBF16, true>(a, m, grid, st);
    case 32: return launch_gemm<32, kMode, kBF16, true>(a, m, grid, st);
    case 64: return launch_gemm<64, kMode, kBF16, false>(a, m, grid, st);
    case 128: return launch_gemm<128, kMode, kBF16, false>(a, m, grid, st);
    default: return W4_ERR_ARG;
  }
}

}  // namespace

extern "C" {

int w4a16_tile_rows(void) { return kTileRows; }
int w4a16_tile_k(void) { return kTileK; }
int w4a16_part_bytes(void) { return kPartBytes; }

int w4a16_pick_ntok(int64_t rows, int64_t num_experts) {
  const int64_t avg = num_experts > 0 ? (rows + num_experts - 1) / num_experts : rows;
  if (avg <= 16) return 16;
  if (avg <= 32) return 32;
  if (avg <= 64) return 64;
  return 128;
}

int w4a16_grouped_gemm(const void* x, int64_t rows, int64_t K, const uint8_t* wblocks, int64_t num_experts,
                       int64_t n_out, int gated, const int32_t* expert_counts, const int32_t* expert_offsets,
                       void* out, int dtype, int ntok, cudaStream_t stream) {
  if (!x || !wblocks || !expert_counts || !expert_offsets || !out) return W4_ERR_ARG;
  if (K <= 0 || K % kTileK || n_out <= 0 || n_out % kTileRows) return W4_ERR_SHAPE;
  if (num_experts <= 0 || num_experts > kMaxExperts) return W4_ERR_SHAPE;
  if (dtype != W4_DTYPE_F16 && dtype != W4_DTYPE_BF16) return W4_ERR_DTYPE;
  if (rows <= 0) return W4_OK;
  if (ntok <= 0) ntok = w4a16_pick_ntok(rows, num_experts);
  CUtensorMap map;
  if (make_x_map(&map, x, rows, K, ntok) != W4_OK) return W4_ERR_CUDA;
  GemmArgs a;
  a.wblocks = wblocks;
  a.expert_counts = expert_counts;
  a.expert_offsets = expert_offsets;
  a.out = out;
  a.ldo = n_out;
  a.num_experts = static_cast<int>(num_experts);
  a.nt = static_cast<int>(n_out / kTileRows);
  a.kt = static_cast<int>(K / kTileK);
  const int grid = sm_count();
  const bool bf = dtype == W4_DTYPE_BF16;
  if (gated) return bf ? dispatch_ntok<kModeGateUp, true>(ntok, a, map, grid, stream)
                       : dispatch_ntok<kModeGateUp, false>(ntok, a, map, grid, stream);
  if (a.kt % 2 == 0) return bf ? dispatch_ntok<kModeKPair, true>(ntok, a, map, grid, stream)
                               : dispatch_ntok<kModeKPair, false>(ntok, a, map, grid, stream);
  return bf ? dispatch_ntok<kModePlain, true>(ntok, a, map, grid, stream)
            : dispatch_ntok<kModePlain, false>(ntok, a, map, grid, stream);
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

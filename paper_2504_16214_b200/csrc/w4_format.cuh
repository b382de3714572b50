// Packed W4 weight-block format ("thread-major" repack) and the in-register dequantiser.
//
// The grouped GEMM streams one *block* per (expert, n-tile, k-tile) with a single 1-D bulk copy.
// A block covers kTileRows = 128 output rows x kTileK = 128 reduction elements (one AWQ group of
// 128) for each of `parts` weight matrices (parts = 2 for the fused gate/up projection, where part 0
// holds gate rows and part 1 the matching up rows; parts = 1 otherwise):
//
//   part p (kPartBytes = 8512 B, p-th slice of the block):
//     [   0, 8192)  int4 codes, chunk-major: chunk c (4) x row r (128) x 16 B.
//                   The 16 B of (c, r) hold k = c*32 .. c*32+31 of row r as 4 little-endian words;
//                   word w holds k = c*32 + 8w + e with element e in nibble slot kSlotOf[e]
//                   (slot order 0,2,4,6,1,3,5,7 -- the AWQ interleave, chosen so that two
//                   LOP3s per word yield (e0,e1),(e2,e3) fp16 pairs and a byte shift the rest).
//     [8192, 8448)  scales, one per row (activation dtype: fp16 or bf16)
//     [8448, 8512)  zero points, one nibble per row (row r -> byte r/2, low nibble if r even)
//
// Byte-for-byte this is exactly the AWQ payload (int4 codes + per-group scales + int4 zeros); only
// the order changes. Thread r of a 128-thread dequant group reads its own row with 16 B vector loads
// from consecutive addresses (conflict-free), which is the layout the reference's synthesizer picks
// for the int4 register tensor ("w4" in pkg/fixtures/mixed_int4.prog: every copy >= 8 B, cast in
// place, see /root/reference/pkg/tests/test_acceptance.py:290-315).
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

namespace w4 {

constexpr int kTileRows = 128;
constexpr int kTileK = 128;
constexpr int kGroup = 128;
constexpr int kChunks = kTileK / 32;
constexpr int kCodeBytes = kTileRows * kTileK / 2;            // 8192
constexpr int kScaleOff = kCodeBytes;                          // 8192
constexpr int kZeroOff = kScaleOff + kTileRows * 2;            // 8448
constexpr int kPartBytes = kZeroOff + kTileRows / 2;           // 8512

// nibble slot holding element e of a word (inverse of the AWQ interleave 0,2,4,6,1,3,5,7)
__host__ __device__ constexpr int slot_of(int e) { return (e & 1) * 4 + (e >> 1); }

template <bool kBF16>
struct Dq;

// fp16: 0x6400 | q is the half 1024 + q, so (x - (1024 + z)) is the exact integer q - z; the
// high-nibble pairs come out as 1024 + 16 q and are brought back with one exact HFMA2
// (x * 1/16 - (64 + z)). A single HMUL2 by the scale then gives fp16((q - z) * s) with exactly one
// rounding -- bit-identical to the oracle's fp16(float(q - z) * float(s)).
template <>
struct Dq<false> {
  using T2 = __half2;
  struct Ctx {
    __half2 zz, zz16, sixteenth, s2;
  };
  // all constants are built from integer bit patterns: 1024 + z = 0x6400 | z,
  // -(64 + z) = 0xD400 | (z << 4), 1/16 = 0x2C00 (no int->float->half conversions)
  static __device__ __forceinline__ Ctx make(uint32_t z, uint16_t sbits) {
    Ctx c;
    const uint32_t zz = (0x6400u | z) * 0x10001u, zz16 = (0xD400u | (z << 4)) * 0x10001u;
    const uint32_t sx = 0x2C002C00u, s2 = static_cast<uint32_t>(sbits) * 0x10001u;
    c.zz = *reinterpret_cast<const __half2*>(&zz);
    c.zz16 = *reinterpret_cast<const __half2*>(&zz16);
    c.sixteenth = *reinterpret_cast<const __half2*>(&sx);
    c.s2 = *reinterpret_cast<const __half2*>(&s2);
    return c;
  }
  // exact (q - z) pairs only (the scale is applied to the fp32 group partial by the epilogue)
  static __device__ __forceinline__ void word_qz(uint32_t w, const Ctx& c, uint32_t* o) {
    const uint32_t kMagic = 0x64006400u;
    uint32_t a, b, d, e;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(a) : "r"(w), "r"(0x000F000Fu), "r"(kMagic));
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(b) : "r"(w), "r"(0x00F000F0u), "r"(kMagic));
    const uint32_t w8 = w >> 8;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(w8), "r"(0x000F000Fu), "r"(kMagic));
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(e) : "r"(w8), "r"(0x00F000F0u), "r"(kMagic));
    __half2 q01 = __hsub2(*reinterpret_cast<__half2*>(&a), c.zz);
    __half2 q23 = __hfma2(*reinterpret_cast<__half2*>(&b), c.sixteenth, c.zz16);
    __half2 q45 = __hsub2(*reinterpret_cast<__half2*>(&d), c.zz);
    __half2 q67 = __hfma2(*reinterpret_cast<__half2*>(&e), c.sixteenth, c.zz16);
    o[0] = *reinterpret_cast<uint32_t*>(&q01);
    o[1] = *reinterpret_cast<uint32_t*>(&q23);
    o[2] = *reinterpret_cast<uint32_t*>(&q45);
    o[3] = *reinterpret_cast<uint32_t*>(&q67);
  }
  // offset codes, LOP3 only: pairs (e0,e1),(e4,e5) come out as 1024 + q, pairs (e2,e3),(e6,e7) as
  // 64 + q (0x5400 | q << 4: the nibble lands on mantissa bits 4..7, whose weight is 1 at 2^6). Both
  // are exact fp16 integers; the GEMM removes the offsets and the zero point per (group, token)
  // with the constant-row MMA (kOffsetRow* below), so no per-weight FP op is needed.
  static __device__ __forceinline__ void word_raw(uint32_t w, uint32_t* o) {
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(o[0]) : "r"(w), "r"(0x000F000Fu), "r"(0x64006400u));
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(o[1]) : "r"(w), "r"(0x00F000F0u), "r"(0x54005400u));
    const uint32_t w8 = w >> 8;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(o[2]) : "r"(w8), "r"(0x000F000Fu), "r"(0x64006400u));
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(o[3]) : "r"(w8), "r"(0x00F000F0u), "r"(0x54005400u));
  }
  // fp16 bits of the offset carried by element e (0..7) of a word in word_raw's output
  static __host__ __device__ constexpr uint16_t offset_bits(int e) { return ((e >> 1) & 1) ? 0x5400 : 0x6400; }
  static constexpr uint16_t kOneBits = 0x3C00;
  static __device__ __forceinline__ void word(uint32_t w, const Ctx& c, uint32_t* o) {
    const uint32_t kMagic = 0x64006400u;
    uint32_t a, b, d, e;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(a) : "r"(w), "r"(0x000F000Fu), "r"(kMagic));
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(b) : "r"(w), "r"(0x00F000F0u), "r"(kMagic));
    const uint32_t w8 = w >> 8;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(w8), "r"(0x000F000Fu), "r"(kMagic));
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(e) : "r"(w8), "r"(0x00F000F0u), "r"(kMagic));
    __half2 q01 = __hsub2(*reinterpret_cast<__half2*>(&a), c.zz);
    __half2 q23 = __hfma2(*reinterpret_cast<__half2*>(&b), c.sixteenth, c.zz16);
    __half2 q45 = __hsub2(*reinterpret_cast<__half2*>(&d), c.zz);
    __half2 q67 = __hfma2(*reinterpret_cast<__half2*>(&e), c.sixteenth, c.zz16);
    __half2 r0 = __hmul2_rn(q01, c.s2), r1 = __hmul2_rn(q23, c.s2);
    __half2 r2 = __hmul2_rn(q45, c.s2), r3 = __hmul2_rn(q67, c.s2);
    o[0] = *reinterpret_cast<uint32_t*>(&r0);
    o[1] = *reinterpret_cast<uint32_t*>(&r1);
    o[2] = *reinterpret_cast<uint32_t*>(&r2);
    o[3] = *reinterpret_cast<uint32_t*>(&r3);
  }
};

// bf16: 0x4300 | q is the bf16 128 + q (exact for q < 128); the mantissa is too short for the
// x16 trick, so each pair is shifted into the low nibble first.
template <>
struct Dq<true> {
  using T2 = __nv_bfloat162;
  struct Ctx {
    __nv_bfloat162 zz, s2;
  };
  static __device__ __forceinline__ Ctx make(uint32_t z, uint16_t sbits) {
    Ctx c;
    const uint32_t zz = (0x4300u | z) * 0x10001u, s2 = static_cast<uint32_t>(sbits) * 0x10001u;
    c.zz = *reinterpret_cast<const __nv_bfloat162*>(&zz);
    c.s2 = *reinterpret_cast<const __nv_bfloat162*>(&s2);
    return c;
  }
  static __device__ __forceinline__ void word_qz(uint32_t w, const Ctx& c, uint32_t* o) {
    const uint32_t kMagic = 0x43004300u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t x;
      asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(x) : "r"(w >> (4 * i)), "r"(0x000F000Fu), "r"(kMagic));
      __nv_bfloat162 q = __hsub2(*reinterpret_cast<__nv_bfloat162*>(&x), c.zz);
      o[i] = *reinterpret_cast<uint32_t*>(&q);
    }
  }
  // offset codes: every pair comes out as 128 + q (exact bf16 integers)
  static __device__ __forceinline__ void word_raw(uint32_t w, uint32_t* o) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(o[i]) : "r"(w >> (4 * i)), "r"(0x000F000Fu), "r"(0x43004300u));
  }
  static __host__ __device__ constexpr uint16_t offset_bits(int) { return 0x4300; }
  static constexpr uint16_t kOneBits = 0x3F80;
  static __device__ __forceinline__ void word(uint32_t w, const Ctx& c, uint32_t* o) {
    const uint32_t kMagic = 0x43004300u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t x;
      asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(x) : "r"(w >> (4 * i)), "r"(0x000F000Fu), "r"(kMagic));
      __nv_bfloat162 q = __hsub2(*reinterpret_cast<__nv_bfloat162*>(&x), c.zz);
      __nv_bfloat162 r = __hmul2_rn(q, c.s2);
      o[i] = *reinterpret_cast<uint32_t*>(&r);
    }
  }
};

// One 16 B chunk (32 consecutive k of one row) as offset codes (see Dq::word_raw), k order.
template <bool kBF16>
__device__ __forceinline__ void raw_chunk(const uint4& v, uint32_t (&o)[16]) {
  Dq<kBF16>::word_raw(v.x, o + 0);
  Dq<kBF16>::word_raw(v.y, o + 4);
  Dq<kBF16>::word_raw(v.z, o + 8);
  Dq<kBF16>::word_raw(v.w, o + 12);
}

// Dequantise one 16 B chunk (32 consecutive k of one row) into 16 packed pairs, k order:
// kScaled -> act((q - z) * s) (bit-exact dequant); otherwise the exact integers (q - z).
template <bool kBF16, bool kScaled = true>
__device__ __forceinline__ void dequant_chunk(const uint4& v, const typename Dq<kBF16>::Ctx& c, uint32_t (&o)[16]) {
  if constexpr (kScaled) {
    Dq<kBF16>::word(v.x, c, o + 0);
    Dq<kBF16>::word(v.y, c, o + 4);
    Dq<kBF16>::word(v.z, c, o + 8);
    Dq<kBF16>::word(v.w, c, o + 12);
  } else {
    Dq<kBF16>::word_qz(v.x, c, o + 0);
    Dq<kBF16>::word_qz(v.y, c, o + 4);
    Dq<kBF16>::word_qz(v.z, c, o + 8);
    Dq<kBF16>::word_qz(v.w, c, o + 12);
  }
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ float2 lds_f2(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint16_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}

}  // namespace w4

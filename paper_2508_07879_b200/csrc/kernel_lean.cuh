// Throughput kernel for (6,3)-regular codes, work item = (shot, segment).
//
// The arithmetic is the regular kernel's (bit-exact with the reference); this
// kernel is about spending as few instructions per iteration as possible
// OUTSIDE the two node updates, because on B200 this decoder is bound by
// instruction issue and the conversion pipe, not by shared-memory bandwidth
// (DESIGN.md "what bounds the path"):
//
//  * one message block per check in shared memory, [6 x q | 6 x r | pad], with a
//    per-arithmetic stride chosen so that a warp of consecutive checks reads and
//    writes its blocks without bank conflicts; r sits at a compile-time offset
//    from q, so each variable edge costs ONE register (a byte offset) and every
//    access is [reg + immediate];
//  * the syndrome-match test is a single counter: the parity bitmap starts as the
//    syndrome, a variable toggles its three checks only when its hard decision
//    CHANGES (atomicXor, rare after the first iterations), and the toggling
//    thread adjusts `unsat` by the bits it set or cleared - the per-iteration test
//    is one broadcast load and a compare, with no preset, no scan, no masks;
//  * bit vectors are segment-local (bit i = check c0 + i); the packed syndrome is
//    prefetched into registers one shot ahead and shifted into place with warp
//    shuffles, results are shifted back on the way out; words shared by two
//    segments are only touched with bit-masked atomics, so the X and Z halves of a
//    shot may be decoded by different CTAs in any order;
//  * per-shot bit state is double-buffered on the item parity, which removes the
//    barrier between one shot's exit test and the next shot's prologue:
//    1 + 2 * iterations barriers per item.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernel_generic.cuh"

namespace qb {

namespace cg = cooperative_groups;

constexpr int kDC = 6;  // the bivariate-bicycle family: every check has degree 6,
constexpr int kDV = 3;  // every variable degree 3
constexpr uint32_t kNoShot = 0xffffffffu;

// min1 / min2 of six non-negative integer keys (13 min/max operations).
__device__ __forceinline__ void two_smallest6(const int32_t (&a)[6], int32_t& m1, int32_t& m2) {
  const int32_t l0 = min(a[0], a[1]), h0 = max(a[0], a[1]);
  const int32_t l1 = min(a[2], a[3]), h1 = max(a[2], a[3]);
  const int32_t l2 = min(a[4], a[5]), h2 = max(a[4], a[5]);
  m1 = min(min(l0, l1), l2);
  // Everything except one instance of the minimum: the other two pair-minima
  // (their smaller one is the median of the three) and the three pair-maxima.
  const int32_t med = max(min(l0, l1), min(max(l0, l1), l2));
  m2 = min(med, min(min(h0, h1), h2));
}

// Message-block layout per arithmetic: byte stride between checks, byte offset
// of the r half.  Strides are conflict-free for the check-side vector access of
// 32 consecutive checks: fp32 3 x 64-bit at stride 14 words; fp16 / int16
// 3 x 32-bit at stride 7 words; int8 1 x 64-bit at stride 6 words.
template <class A> struct Lay;
template <> struct Lay<ArithF32> { static constexpr uint32_t kStride = 56, kROff = 24; };
template <> struct Lay<ArithF16> { static constexpr uint32_t kStride = 28, kROff = 12; };
template <> struct Lay<ArithI16> { static constexpr uint32_t kStride = 28, kROff = 12; };
template <> struct Lay<ArithI8> { static constexpr uint32_t kStride = 24, kROff = 8; };
// Integer modes with one 32-bit word per message (the fp32 layout): the batch kernel of the
// int16 mode.  The sub-word layouts above cost a sign extension per value read and a pack per
// value written, on the ALU pipe that bounds the integer kernels; with whole words a message
// is an operand as loaded and the saturation bound is a kernel constant (DecodeParams::kmax).
template <> struct Lay<ArithI32> { static constexpr uint32_t kStride = 56, kROff = 24; };
template <> struct Lay<ArithI16F> { static constexpr uint32_t kStride = 56, kROff = 24; };

// prior of variable n in the kernel's own representation
template <class A>
__device__ __forceinline__ typename A::Gam load_prior(const DecodeParams& P, uint32_t n) {
  return static_cast<const typename A::Gam*>(P.gamma)[n];
}
template <>
__device__ __forceinline__ float load_prior<ArithI16F>(const DecodeParams& P, uint32_t n) {
  return static_cast<float>(static_cast<const int32_t*>(P.gamma)[n]);  // |gamma| <= 32767: exact
}

__host__ __device__ inline uint32_t lean_stride(int arith) {
  return arith == 0 ? 56u : arith == 1 ? 24u : 28u;
}
__host__ __device__ inline uint32_t lean_pw(uint32_t seg_mmax) { return (seg_mmax >> 5) + 1; }
// Syndromes reach the batch kernel in TILES of up to kMaxTile shots: one TMA bulk copy
// (cp.async.bulk, completing on an mbarrier) and one queue ticket per tile, two tiles in
// flight per CTA.
constexpr uint32_t kMaxTile = 16;
__host__ __device__ inline size_t lean_bits_words(uint32_t seg_mmax) {
  return (6 * static_cast<size_t>(lean_pw(seg_mmax)) + 8 + 3) & ~size_t(3);  // keeps 16-byte alignment
}
constexpr uint32_t kLeanTabBytes = 16;  // first-iteration table at shared-memory offset 0
// per-item constants of the two single-warp prologue jobs, computed once per CTA: the bit masks
// of the (up to 64) estimate words a segment owns, and of the 32 local syndrome words
constexpr uint32_t kLeanLaneTabWords = 96;
__host__ __device__ inline size_t lean_smem_bytes(uint32_t seg_mmax, int arith, uint32_t syn_w32) {
  const size_t msg = (static_cast<size_t>(seg_mmax + 1) * lean_stride(arith) + 15) & ~size_t(15);
  // table | messages | bitmaps, counters, tickets | 2 syndrome tiles | 2 mbarriers | tile info [2][2]
  return kLeanTabBytes + msg + 4 * lean_bits_words(seg_mmax) + 2 * kMaxTile * syn_w32 * 4 + 16 + 16 + 16 +
         4 * kLeanLaneTabWords;
}

// ---- check update on one message block ---------------------------------------

__device__ __forceinline__ void cn6_block(const DecodeParams& P, ArithF32, unsigned char* blk,
                                          uint32_t syn_bit) {
  const float2* qp = reinterpret_cast<const float2*>(blk);
  float v[6];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const float2 p = qp[j];
    v[2 * j] = p.x;
    v[2 * j + 1] = p.y;
  }
  // |.| folds into the min/max/compare instructions as a source modifier
  const float l0 = fminf(fabsf(v[0]), fabsf(v[1])), h0 = fmaxf(fabsf(v[0]), fabsf(v[1]));
  const float l1 = fminf(fabsf(v[2]), fabsf(v[3])), h1 = fmaxf(fabsf(v[2]), fabsf(v[3]));
  const float l2 = fminf(fabsf(v[4]), fabsf(v[5])), h2 = fmaxf(fabsf(v[4]), fabsf(v[5]));
  const float m1 = fminf(fminf(l0, l1), l2);
  const float med = fmaxf(fminf(l0, l1), fminf(fmaxf(l0, l1), l2));
  const float m2 = fminf(med, fminf(fminf(h0, h1), h2));
  // float(alpha * |min|): fp64 product, one rounding (decoder.cpp:302-307).  Both carry the
  // sign common to all edges (syndrome, parity of every incoming sign); edge j then only
  // flips by its own incoming sign.
  uint32_t sx = syn_bit << 31;
#pragma unroll
  for (int j = 0; j < 6; ++j) sx ^= __float_as_uint(v[j]);
  sx &= 0x80000000u;
  const uint32_t s1 = __float_as_uint(static_cast<float>(P.alpha * static_cast<double>(m1))) ^ sx;
  const uint32_t s2 = __float_as_uint(static_cast<float>(P.alpha * static_cast<double>(m2))) ^ sx;
  float2* rp = reinterpret_cast<float2*>(blk + Lay<ArithF32>::kROff);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const uint32_t ox = (fabsf(v[2 * j]) == m1 ? s2 : s1) ^ (__float_as_uint(v[2 * j]) & 0x80000000u);
    const uint32_t oy =
        (fabsf(v[2 * j + 1]) == m1 ? s2 : s1) ^ (__float_as_uint(v[2 * j + 1]) & 0x80000000u);
    rp[j] = make_float2(__uint_as_float(ox), __uint_as_float(oy));
  }
}

__device__ __forceinline__ void cn6_block(const DecodeParams& P, ArithF16, unsigned char* blk,
                                          uint32_t syn_bit) {
  const uint32_t* qp = reinterpret_cast<const uint32_t*>(blk);
  uint32_t u[6];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const uint32_t w = qp[j];
    u[2 * j] = w & 0xffffu;
    u[2 * j + 1] = w >> 16;
  }
  int32_t a[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) a[j] = static_cast<int32_t>(u[j] & 0x7fffu);
  int32_t m1, m2;
  two_smallest6(a, m1, m2);
  const __half alpha = __ushort_as_half(P.alpha_h);
  const uint32_t s1 =
      __half_as_ushort(__hmul(alpha, __ushort_as_half(static_cast<unsigned short>(m1))));
  const uint32_t s2 =
      __half_as_ushort(__hmul(alpha, __ushort_as_half(static_cast<unsigned short>(m2))));
  const uint32_t sx = u[0] ^ u[1] ^ u[2] ^ u[3] ^ u[4] ^ u[5] ^ (syn_bit << 15);
  uint32_t* rp = reinterpret_cast<uint32_t*>(blk + Lay<ArithF16>::kROff);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const uint32_t lo = (a[2 * j] == m1 ? s2 : s1) | ((sx ^ u[2 * j]) & 0x8000u);
    const uint32_t hi = (a[2 * j + 1] == m1 ? s2 : s1) | ((sx ^ u[2 * j + 1]) & 0x8000u);
    rp[j] = lo | (hi << 16);
  }
}

__device__ __forceinline__ void cn6_finish_int(const DecodeParams& P, const int32_t (&v)[6],
                                               int32_t (&out)[6], uint32_t syn_bit) {
  int32_t a[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) a[j] = abs(v[j]);
  int32_t m1, m2;
  two_smallest6(a, m1, m2);
  const int32_t s1 = scale_q16(static_cast<uint32_t>(m1), P.alpha_fx);
  const int32_t s2 = scale_q16(static_cast<uint32_t>(m2), P.alpha_fx);
  const int32_t sx = v[0] ^ v[1] ^ v[2] ^ v[3] ^ v[4] ^ v[5] ^ static_cast<int32_t>(syn_bit << 31);
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    const int32_t mag = a[j] == m1 ? s2 : s1;
    const int32_t neg = (sx ^ v[j]) >> 31;  // 0 or -1
    out[j] = (mag ^ neg) - neg;
  }
}

__device__ __forceinline__ void cn6_block(const DecodeParams& P, ArithI16, unsigned char* blk,
                                          uint32_t syn_bit) {
  const short2* qp = reinterpret_cast<const short2*>(blk);
  int32_t v[6], o[6];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const short2 p = qp[j];
    v[2 * j] = p.x;
    v[2 * j + 1] = p.y;
  }
  cn6_finish_int(P, v, o, syn_bit);
  short2* rp = reinterpret_cast<short2*>(blk + Lay<ArithI16>::kROff);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    rp[j] = make_short2(static_cast<short>(o[2 * j]), static_cast<short>(o[2 * j + 1]));
  }
}

__device__ __forceinline__ void cn6_block(const DecodeParams& P, ArithI32, unsigned char* blk,
                                          uint32_t syn_bit) {
  const int2* qp = reinterpret_cast<const int2*>(blk);
  int32_t v[6], o[6];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const int2 p = qp[j];
    v[2 * j] = p.x;
    v[2 * j + 1] = p.y;
  }
  cn6_finish_int(P, v, o, syn_bit);
  int2* rp = reinterpret_cast<int2*>(blk + Lay<ArithI32>::kROff);
#pragma unroll
  for (int j = 0; j < 3; ++j) rp[j] = make_int2(o[2 * j], o[2 * j + 1]);
}

// scale_q16 of a non-negative integer-valued float below 2^15 (see ArithI16F)
__device__ __forceinline__ float scale_q16_f(float mag, uint32_t alpha_fx, uint32_t addend) {
  const uint32_t b = __float_as_uint(mag + 8388608.0f);  // 0x4B000000 + mag
  const uint32_t u = b * alpha_fx + addend;              // mag * alpha_fx + 32768  (mod 2^32: exact)
  return __uint_as_float((u >> 16) | 0x4B000000u) - 8388608.0f;
}

__device__ __forceinline__ void cn6_block(const DecodeParams& P, ArithI16F, unsigned char* blk,
                                          uint32_t syn_bit) {
  const float2* qp = reinterpret_cast<const float2*>(blk);
  float v[6];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const float2 p = qp[j];
    v[2 * j] = p.x;
    v[2 * j + 1] = p.y;
  }
  const float l0 = fminf(fabsf(v[0]), fabsf(v[1])), h0 = fmaxf(fabsf(v[0]), fabsf(v[1]));
  const float l1 = fminf(fabsf(v[2]), fabsf(v[3])), h1 = fmaxf(fabsf(v[2]), fabsf(v[3]));
  const float l2 = fminf(fabsf(v[4]), fabsf(v[5])), h2 = fmaxf(fabsf(v[4]), fabsf(v[5]));
  const float m1 = fminf(fminf(l0, l1), l2);
  const float med = fmaxf(fminf(l0, l1), fminf(fmaxf(l0, l1), l2));
  const float m2 = fminf(med, fminf(fminf(h0, h1), h2));
  uint32_t sx = syn_bit << 31;
#pragma unroll
  for (int j = 0; j < 6; ++j) sx ^= __float_as_uint(v[j]);
  sx &= 0x80000000u;
  const uint32_t addend = 32768u - 0x4B000000u * P.alpha_fx;
  const uint32_t s1 = __float_as_uint(scale_q16_f(m1, P.alpha_fx, addend)) ^ sx;
  const uint32_t s2 = __float_as_uint(scale_q16_f(m2, P.alpha_fx, addend)) ^ sx;
  float2* rp = reinterpret_cast<float2*>(blk + Lay<ArithI16F>::kROff);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const uint32_t ox = (fabsf(v[2 * j]) == m1 ? s2 : s1) ^ (__float_as_uint(v[2 * j]) & 0x80000000u);
    const uint32_t oy =
        (fabsf(v[2 * j + 1]) == m1 ? s2 : s1) ^ (__float_as_uint(v[2 * j + 1]) & 0x80000000u);
    rp[j] = make_float2(__uint_as_float(ox), __uint_as_float(oy));
  }
}

__device__ __forceinline__ void cn6_block(const DecodeParams& P, ArithI8, unsigned char* blk,
                                          uint32_t syn_bit) {
  const uint2 w = *reinterpret_cast<const uint2*>(blk);  // 6 message bytes + 2 unused
  int32_t v[6], o[6];
  v[0] = static_cast<int8_t>(w.x);
  v[1] = static_cast<int8_t>(w.x >> 8);
  v[2] = static_cast<int8_t>(w.x >> 16);
  v[3] = static_cast<int8_t>(w.x >> 24);
  v[4] = static_cast<int8_t>(w.y);
  v[5] = static_cast<int8_t>(w.y >> 8);
  cn6_finish_int(P, v, o, syn_bit);
  uint2 r;
  r.x = (o[0] & 0xff) | ((o[1] & 0xff) << 8) | ((o[2] & 0xff) << 16) |
        (static_cast<uint32_t>(o[3]) << 24);
  r.y = (o[4] & 0xff) | ((o[5] & 0xff) << 8);
  *reinterpret_cast<uint2*>(blk + Lay<ArithI8>::kROff) = r;
}

// ---- variable update through byte offsets; returns 1 iff the variable decides 1 ----

template <bool kFast>
__device__ __forceinline__ uint32_t vn3_off(const DecodeParams& P, ArithF32, unsigned char* base,
                                            const uint32_t (&eo)[3], float gamma) {
  constexpr uint32_t R = Lay<ArithF32>::kROff;
  const double r0 = static_cast<double>(*reinterpret_cast<const float*>(base + eo[0] + R));
  const double r1 = static_cast<double>(*reinterpret_cast<const float*>(base + eo[1] + R));
  const double r2 = static_cast<double>(*reinterpret_cast<const float*>(base + eo[2] + R));
  double total = kFast ? P.gamma_d : static_cast<double>(gamma);  // ascending edge order
  total += r0;
  total += r1;
  total += r2;
  float x0 = static_cast<float>(total - r0);
  float x1 = static_cast<float>(total - r1);
  float x2 = static_cast<float>(total - r2);
  if constexpr (!kFast) {
    x0 = fminf(fmaxf(x0, -P.clamp_f), P.clamp_f);
    x1 = fminf(fmaxf(x1, -P.clamp_f), P.clamp_f);
    x2 = fminf(fmaxf(x2, -P.clamp_f), P.clamp_f);
  }
  *reinterpret_cast<float*>(base + eo[0]) = x0;
  *reinterpret_cast<float*>(base + eo[1]) = x1;
  *reinterpret_cast<float*>(base + eo[2]) = x2;
  return static_cast<uint32_t>(__double2hiint(total)) >> 31;
}

template <bool kFast>
__device__ __forceinline__ uint32_t vn3_off(const DecodeParams& P, ArithF16, unsigned char* base,
                                            const uint32_t (&eo)[3], float gamma) {
  constexpr uint32_t R = Lay<ArithF16>::kROff;
  const __half r0 = *reinterpret_cast<const __half*>(base + eo[0] + R);
  const __half r1 = *reinterpret_cast<const __half*>(base + eo[1] + R);
  const __half r2 = *reinterpret_cast<const __half*>(base + eo[2] + R);
  const __half g = kFast ? __ushort_as_half(P.gamma_hb)
                         : __float2half_rn(fminf(fmaxf(gamma, -kHalfClamp), kHalfClamp));
  const __half total = __hadd(__hadd(__hadd(g, r0), r1), r2);
  *reinterpret_cast<__half*>(base + eo[0]) = h_clamp(__hsub(total, r0));
  *reinterpret_cast<__half*>(base + eo[1]) = h_clamp(__hsub(total, r1));
  *reinterpret_cast<__half*>(base + eo[2]) = h_clamp(__hsub(total, r2));
  return h_neg(total) ? 1u : 0u;
}

template <bool kFast, class A>
__device__ __forceinline__ uint32_t vn3_off_int(const DecodeParams& P, unsigned char* base,
                                                const uint32_t (&eo)[3], int32_t gamma) {
  using MsgI = typename A::Msg;
  constexpr uint32_t R = Lay<A>::kROff;
  const int32_t r0 = *reinterpret_cast<const MsgI*>(base + eo[0] + R);
  const int32_t r1 = *reinterpret_cast<const MsgI*>(base + eo[1] + R);
  const int32_t r2 = *reinterpret_cast<const MsgI*>(base + eo[2] + R);
  const int32_t total = (kFast ? P.gamma_i : gamma) + r0 + r1 + r2;
  *reinterpret_cast<MsgI*>(base + eo[0]) = static_cast<MsgI>(max(-P.kmax, min(P.kmax, total - r0)));
  *reinterpret_cast<MsgI*>(base + eo[1]) = static_cast<MsgI>(max(-P.kmax, min(P.kmax, total - r1)));
  *reinterpret_cast<MsgI*>(base + eo[2]) = static_cast<MsgI>(max(-P.kmax, min(P.kmax, total - r2)));
  return static_cast<uint32_t>(total) >> 31;
}
template <bool kFast>
__device__ __forceinline__ uint32_t vn3_off(const DecodeParams& P, ArithI8, unsigned char* base,
                                            const uint32_t (&eo)[3], int32_t gamma) {
  return vn3_off_int<kFast, ArithI8>(P, base, eo, gamma);
}
template <bool kFast>
__device__ __forceinline__ uint32_t vn3_off(const DecodeParams& P, ArithI16, unsigned char* base,
                                            const uint32_t (&eo)[3], int32_t gamma) {
  return vn3_off_int<kFast, ArithI16>(P, base, eo, gamma);
}
template <bool kFast>
__device__ __forceinline__ uint32_t vn3_off(const DecodeParams& P, ArithI32, unsigned char* base,
                                            const uint32_t (&eo)[3], int32_t gamma) {
  return vn3_off_int<kFast, ArithI32>(P, base, eo, gamma);
}
// int16 semantics on fp32 instructions: exact integer sums, saturation at +-kmax
template <bool kFast>
__device__ __forceinline__ uint32_t vn3_off(const DecodeParams& P, ArithI16F, unsigned char* base,
                                            const uint32_t (&eo)[3], float gamma) {
  constexpr uint32_t R = Lay<ArithI16F>::kROff;
  const float r0 = *reinterpret_cast<const float*>(base + eo[0] + R);
  const float r1 = *reinterpret_cast<const float*>(base + eo[1] + R);
  const float r2 = *reinterpret_cast<const float*>(base + eo[2] + R);
  const float total = (kFast ? P.gamma_f : gamma) + r0 + r1 + r2;
  *reinterpret_cast<float*>(base + eo[0]) = fmaxf(-P.kmax_f, fminf(P.kmax_f, total - r0));
  *reinterpret_cast<float*>(base + eo[1]) = fmaxf(-P.kmax_f, fminf(P.kmax_f, total - r1));
  *reinterpret_cast<float*>(base + eo[2]) = fmaxf(-P.kmax_f, fminf(P.kmax_f, total - r2));
  return total < 0.0f ? 1u : 0u;
}

// ---- first iteration with a uniform prior --------------------------------------
// Every q equals gamma before the first check stage, so check m sends
// r = (-1)^(s_m) * sign(gamma) * S on all of its edges, with one constant
// S = float(alpha * |gamma|) (resp. the Q16 / fp16 analogue) computed by the
// loader.  The first variable stage can therefore be evaluated directly from the
// three syndrome bits of a variable's checks: no q initialisation, no check stage,
// no barrier between them, and no widening conversions (S is a constant).  The
// arithmetic below is the same sequence of operations the regular stages perform,
// so the stored q and the decisions are bit-identical.
__device__ __forceinline__ uint32_t syn_bit_of_edge(const uint32_t* par, uint32_t off,
                                                     uint32_t stride) {
  const uint32_t lm = off / stride;
  return (par[lm >> 5] >> (lm & 31u)) & 1u;
}

// First iteration by TABLE (uniform prior; fp32 and whole-word integer messages): the message
// on edge i is it1_tq[number of the OTHER two checks with syndrome bit 1], the decision bit 4k
// of it1_dec4 (DecodeParams; verified by the loader against the reference's operation sequence
// for all eight patterns).  `tab` = the three table words at the start of shared memory,
// `syn2` = the syndrome bitmap with every word ROTATED LEFT BY TWO, so that
// rotate_right(word, position) & 4 is the byte offset of a table step: three gathers, one add, and per edge subtract / load / store -
// no widening, no fp64 sums, no conversions.
template <uint32_t kStrideT>
__device__ __forceinline__ uint32_t vn3_first_tab(const DecodeParams& P, unsigned char* base,
                                                  const unsigned char* tab, const uint32_t (&eo)[3],
                                                  const uint32_t* syn2) {
  uint32_t b4[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const uint32_t lm = eo[i] / kStrideT;
    const uint32_t w = syn2[lm >> 5];
    b4[i] = __funnelshift_r(w, w, lm) & 4u;  // rotate right by lm mod 32: bit lm of the syndrome at position 2
  }
  const uint32_t k4 = b4[0] + b4[1] + b4[2];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    *reinterpret_cast<uint32_t*>(base + eo[i]) = *reinterpret_cast<const uint32_t*>(tab + (k4 - b4[i]));
  }
  return (P.it1_dec4 >> k4) & 1u;
}

__device__ __forceinline__ uint32_t vn3_first(const DecodeParams& P, ArithF32, unsigned char* base,
                                              const uint32_t (&eo)[3], const uint32_t* par) {
  const uint32_t hi0 = static_cast<uint32_t>(__double2hiint(P.it1_d));
  const int lo = __double2loint(P.it1_d);
  double r[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const uint32_t flip = syn_bit_of_edge(par, eo[i], Lay<ArithF32>::kStride) ^ P.it1_neg;
    r[i] = __hiloint2double(static_cast<int>(hi0 ^ (flip << 31)), lo);
  }
  double total = P.gamma_d;
  total += r[0];
  total += r[1];
  total += r[2];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    *reinterpret_cast<float*>(base + eo[i]) = static_cast<float>(total - r[i]);
  }
  return static_cast<uint32_t>(__double2hiint(total)) >> 31;
}

__device__ __forceinline__ uint32_t vn3_first(const DecodeParams& P, ArithF16, unsigned char* base,
                                              const uint32_t (&eo)[3], const uint32_t* par) {
  __half r[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const uint32_t flip = syn_bit_of_edge(par, eo[i], Lay<ArithF16>::kStride) ^ P.it1_neg;
    r[i] = __ushort_as_half(static_cast<unsigned short>(P.it1_h ^ (flip << 15)));
  }
  const __half total = __hadd(__hadd(__hadd(__ushort_as_half(P.gamma_hb), r[0]), r[1]), r[2]);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    *reinterpret_cast<__half*>(base + eo[i]) = h_clamp(__hsub(total, r[i]));
  }
  return h_neg(total) ? 1u : 0u;
}

template <class A>
__device__ __forceinline__ uint32_t vn3_first_int(const DecodeParams& P, unsigned char* base,
                                                  const uint32_t (&eo)[3], const uint32_t* par) {
  using MsgI = typename A::Msg;
  int32_t r[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const uint32_t flip = syn_bit_of_edge(par, eo[i], Lay<A>::kStride) ^ P.it1_neg;
    r[i] = flip ? -P.it1_i : P.it1_i;
  }
  const int32_t total = P.gamma_i + r[0] + r[1] + r[2];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    *reinterpret_cast<MsgI*>(base + eo[i]) =
        static_cast<MsgI>(max(-P.kmax, min(P.kmax, total - r[i])));
  }
  return static_cast<uint32_t>(total) >> 31;
}
__device__ __forceinline__ uint32_t vn3_first(const DecodeParams& P, ArithI8, unsigned char* base,
                                              const uint32_t (&eo)[3], const uint32_t* par) {
  return vn3_first_int<ArithI8>(P, base, eo, par);
}
__device__ __forceinline__ uint32_t vn3_first(const DecodeParams& P, ArithI16, unsigned char* base,
                                              const uint32_t (&eo)[3], const uint32_t* par) {
  return vn3_first_int<ArithI16>(P, base, eo, par);
}
__device__ __forceinline__ uint32_t vn3_first(const DecodeParams& P, ArithI32, unsigned char* base,
                                              const uint32_t (&eo)[3], const uint32_t* par) {
  return vn3_first_int<ArithI32>(P, base, eo, par);
}
__device__ __forceinline__ uint32_t vn3_first(const DecodeParams& P, ArithI16F, unsigned char* base,
                                              const uint32_t (&eo)[3], const uint32_t* par) {
  float r[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const uint32_t flip = syn_bit_of_edge(par, eo[i], Lay<ArithI16F>::kStride) ^ P.it1_neg;
    r[i] = static_cast<float>(flip ? -P.it1_i : P.it1_i);
  }
  const float total = P.gamma_f + r[0] + r[1] + r[2];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    *reinterpret_cast<float*>(base + eo[i]) = fmaxf(-P.kmax_f, fminf(P.kmax_f, total - r[i]));
  }
  return total < 0.0f ? 1u : 0u;
}

// ---- the kernel ---------------------------------------------------------------

// Warp 0 of a batch CTA: describe syndrome tile `t` (K shots) in info = {first shot, shots}
// and start its copy into `buf`: one TMA bulk copy completing on `bar`, or - for a ragged
// tile (odd number of 8-byte-multiple rows) or a caller buffer that is not 16-byte aligned -
// plain loads.  Out of line on purpose: it runs once per tile, and the item loop around it
// is short of registers and instruction-cache room.
__device__ __noinline__ void lean_issue_tile(const uint32_t* syn, uint64_t nshots, uint32_t syn_w32,
                                             uint32_t K, uint64_t t, uint32_t* buf, uint64_t* bar,
                                             uint32_t* info, uint32_t lane) {
  const uint64_t first = t * K;
  const uint32_t cnt =
      first < nshots ? static_cast<uint32_t>(min(static_cast<uint64_t>(K), nshots - first)) : 0u;
  if (lane == 0) {
    info[0] = cnt ? static_cast<uint32_t>(first) : kNoShot;
    info[1] = cnt;
  }
  if (cnt == 0u) return;
  const uint32_t* src = syn + first * syn_w32;
  const uint32_t bytes = cnt * syn_w32 * 4u;
  if (((bytes | static_cast<uint32_t>(reinterpret_cast<uintptr_t>(src))) & 15u) == 0u) {
    if (lane == 0) {
      fence_proxy_async_smem();  // earlier generic-proxy reads of this buffer are done
      mbar_expect_tx(bar, bytes);
      tma_load_1d(buf, src, bytes, bar);
    }
  } else {
    for (uint32_t w = lane; w < cnt * syn_w32; w += 32u) buf[w] = src[w];
    __syncwarp();
    if (lane == 0) mbar_arrive(bar);
  }
}

// Parity hook of the batch kernels (qb_decode_batch_debug): the final messages of ONE shot of
// the batch, written back in reference edge order from the kernel that decodes the whole
// batch - shortcut of the first iteration, tiles and queues all active.  Compiled into the
// kDump instantiations only (the same source with this one call added): as a run-time test in
// the production kernels it cost 2 % (fp32) to 7 % (packed pairs) through register
// allocation around the call.  `first_only`: the segment
// stopped after the first iteration of the uniform-prior path, whose check stage is implicit
// (every r is +-S by the syndrome bit, see vn3_first) and never reached the r slots.
template <class A, class Store>
__device__ __noinline__ void lean_dump_messages(const DecodeParams& P, const ShotIO& io,
                                                const SegmentDev seg, const unsigned char* msgs,
                                                const uint32_t* syn0, bool first_only, uint32_t slot_bytes,
                                                uint32_t stride, uint32_t roff, uint32_t lane_off,
                                                Store store) {
  for (uint32_t e = threadIdx.x; e < seg.e1 - seg.e0; e += blockDim.x) {
    const uint32_t m = e / kDC;
    const unsigned char* src = msgs + m * stride + P.edge_slot[seg.e0 + e] * slot_bytes + lane_off;
    const uint32_t flip = ((syn0[m >> 5] >> (m & 31u)) & 1u) ^ P.it1_neg;
    store(seg.e0 + e, src, src + roff, first_only, flip);
  }
}

template <class A, int CPT, int VPT, bool kFast, int MAXT, int MINB, bool kDump = false>
__global__ void __launch_bounds__(MAXT, MINB)
decode_lean_kernel(const __grid_constant__ DecodeParams P, const __grid_constant__ ShotIO io) {
  using Msg = typename A::Msg;
  using Gam = typename A::Gam;
  constexpr uint32_t kStride = Lay<A>::kStride;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t tid = threadIdx.x, T = blockDim.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t nwarps = T >> 5;
  const uint32_t nseg = P.nseg;
  const uint32_t s = blockIdx.x % nseg;      // the segment this CTA serves for its whole life
  const uint32_t peer = blockIdx.x / nseg;
  const uint32_t peers = (gridDim.x - s + nseg - 1) / nseg;
  const SegmentDev seg = P.segs[s];
  const uint32_t Ms = seg.c1 - seg.c0;
  const uint32_t pw = lean_pw(P.seg_mmax);
  const uint32_t pws = (Ms + 31u) >> 5;
  const uint32_t gw0 = seg.c0 >> 5, gspan = ((seg.c1 - 1) >> 5) - gw0 + 1, cshift = seg.c0 & 31u;
  // the last segment also owns the padding bits of the packed rows (they are written as 0)
  const uint32_t v1z = s + 1u == nseg ? P.est_w32 * 32u : seg.v1;
  const uint32_t c1z = s + 1u == nseg ? P.syn_w32 * 32u : seg.c1;
  const uint32_t vw0 = seg.v0 >> 5, vspan = ((v1z - 1) >> 5) - vw0 + 1;
  const uint32_t gspan_out = ((c1z - 1) >> 5) - gw0 + 1;

  // uniform prior on fp32 / whole-word integer messages: first iteration by table
  constexpr bool kTab = kFast && (sizeof(Msg) == 4);
  unsigned char* const msgs = smem_raw + kLeanTabBytes;
  const size_t msg_bytes = (static_cast<size_t>(P.seg_mmax + 1) * kStride + 15) & ~size_t(15);
  uint32_t* const bits = reinterpret_cast<uint32_t*>(msgs + msg_bytes);
  uint32_t* const unsat_ctr = bits + 2 * pw;  // [2]
  uint32_t* const ticket = bits + 2 * pw + 2;  // [2]
  uint32_t* const syn_copy = bits + 2 * pw + 8;  // [2][pw] the syndrome itself, never toggled
  uint32_t* const syn_rot = bits + 4 * pw + 8;   // [2][pw] ... rotated left by two (vn3_first_tab)
  uint32_t* const tilebuf = bits + lean_bits_words(P.seg_mmax);  // [2][kMaxTile][syn_w32]
  uint64_t* const mbar = reinterpret_cast<uint64_t*>(tilebuf + 2 * kMaxTile * P.syn_w32);  // [2]
  uint32_t* const tinfo = reinterpret_cast<uint32_t*>(mbar + 2);  // [2]{first shot, shots}
  // warp 0's tile cursor lives in shared memory (it is touched once per item, and registers
  // are what this kernel is short of): buffer in use, item within it, mbarrier phase bits
  uint32_t* const tstate = tinfo + 4;  // {tb, ti, tphase}
  uint32_t* const zmask = tstate + 4;  // [64] mask of this segment's bits in estimate word vw0 + w
  uint32_t* const cmask = zmask + 64;  // [32] valid bits of local syndrome word w
  const uint32_t K = io.tile, tile_words = kMaxTile * P.syn_w32;
  for (uint32_t w = tid; w < 64u; w += T) zmask[w] = w < vspan ? range_mask(vw0 + w, seg.v0, v1z) : 0u;
  if (tid < 32u) {
    cmask[tid] = tid >= pws ? 0u : (Ms - tid * 32u < 32u ? (1u << (Ms - tid * 32u)) - 1u : 0xffffffffu);
  }

  // ---- per-thread tables: byte offsets of the q side of every edge / check block
  uint32_t eo[VPT][kDV], co[CPT], cl[CPT], valid = 0;
  Gam gam[kFast ? 1 : VPT];
  {
    const uint32_t dummy = P.seg_mmax * kStride;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const uint32_t n = seg.v0 + tid + k * T;
      const bool ok = n < seg.v1;
      valid |= (ok ? 1u : 0u) << k;
#pragma unroll
      for (int i = 0; i < kDV; ++i) {
        const uint32_t eg = ok ? P.var_edges[n * kDV + i] : 0u;
        const uint32_t e = ok ? eg - seg.e0 : 0u;
        eo[k][i] = ok ? (e / kDC) * kStride + P.edge_slot[eg] * static_cast<uint32_t>(sizeof(Msg))
                      : dummy + i * static_cast<uint32_t>(sizeof(Msg));
      }
      if constexpr (!kFast) gam[k] = ok ? load_prior<A>(P, n) : static_cast<Gam>(1);
    }
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const uint32_t m = tid + k * T;
      cl[k] = m < Ms ? m : Ms;                    // dummy check: bit Ms of the bitmap, always 0
      co[k] = (m < Ms ? m : P.seg_mmax) * kStride;
    }
  }
  for (uint32_t b = tid; b < kStride; b += T) msgs[P.seg_mmax * kStride + b] = 0;  // dummy block
  if (tid < 3) reinterpret_cast<uint32_t*>(smem_raw)[tid] = P.it1_tq[tid];

  auto issue_tile = [&](uint64_t t, uint32_t b) {
    lean_issue_tile(io.syn, io.nshots, P.syn_w32, K, t, tilebuf + b * tile_words, &mbar[b],
                    tinfo + 2 * b, lane);
  };
  if (tid == 0) {
    mbar_init(&mbar[0], 1u);
    mbar_init(&mbar[1], 1u);
    mbar_fence_init();
    tstate[0] = tstate[1] = tstate[2] = 0u;
  }
  __syncthreads();
  if (warp == 0) issue_tile(peer, 0u);
  uint64_t shot = static_cast<uint64_t>(peer) * K;
  uint32_t ipar = 0;
  __syncthreads();

  while (shot < io.nshots) {
    uint32_t* const par = bits + ipar * pw;
    uint32_t* const syn0 = syn_copy + ipar * pw;
    uint32_t* const syn2 = syn_rot + ipar * pw;
    volatile uint32_t* const unsat = unsat_ctr + ipar;
    // ---------------- prologue ----------------
    if (warp == 0) {
      uint32_t tb = tstate[0], ti = tstate[1];
      if (ti == 0u) {
        // first item of a tile: its bytes must have landed; the other buffer is free (its
        // tile is finished), so draw the next tile's ticket and start that copy now - the
        // atomic's round trip and the copy hide behind the K items of this tile
        const uint32_t tphase = tstate[2];
        mbar_wait(&mbar[tb], (tphase >> tb) & 1u);
        __syncwarp();
        if (lane == 0) tstate[2] = tphase ^ (1u << tb);
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(&io.sched[2 + s], 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        issue_tile(static_cast<uint64_t>(t) + peers, tb ^ 1u);
        __syncwarp();
      }
      // packed syndrome words -> segment-local bitmap, and its population count
      const uint32_t raw_next =
          lane < gspan ? tilebuf[tb * tile_words + ti * P.syn_w32 + gw0 + lane] : 0u;
      uint32_t nb = __shfl_down_sync(0xffffffffu, raw_next, 1);
      if (lane + 1 >= gspan) nb = 0;
      const uint32_t loc = (cshift ? __funnelshift_r(raw_next, nb, cshift) : raw_next) & cmask[lane];
      if (lane < pw) {
        par[lane] = loc;
        syn0[lane] = loc;
        if constexpr (kTab) syn2[lane] = __funnelshift_l(loc, loc, 2);
      }
      const uint32_t cnt = __reduce_add_sync(0xffffffffu, __popc(loc));
      if (lane == 0) {
        *unsat = cnt;
        // next item: the following row of this tile, else the first row of the next tile
        const bool more = ti + 1u < tinfo[2 * tb + 1];
        ticket[ipar] = more ? static_cast<uint32_t>(shot) + 1u : tinfo[2 * (tb ^ 1u)];
        tstate[0] = more ? tb : tb ^ 1u;
        tstate[1] = more ? ti + 1u : 0u;
      }
    }
    if (warp == nwarps - 1) {  // zero this segment's bits of the shot's estimate
      uint32_t* est_g = io.est + shot * P.est_w32 + vw0;
      for (uint32_t w = lane; w < vspan; w += 32u) {
        const uint32_t mask = w < 64u ? zmask[w] : range_mask(vw0 + w, seg.v0, v1z);
        if (mask == 0xffffffffu) {
          est_g[w] = 0u;
        } else {
          atomicAnd(&est_g[w], ~mask);
        }
      }
    }
    // q[e] = gamma[var(e)] (decoder.cpp:156-158) - not needed when the first iteration
    // is evaluated from the syndrome (uniform prior)
    if constexpr (!kFast) {
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        const Msg init = prior_as_msg<A>(gam[k]);
#pragma unroll
        for (int i = 0; i < kDV; ++i) *reinterpret_cast<Msg*>(msgs + eo[k][i]) = init;
      }
    }
    uint32_t eprev = 0;
    __syncthreads();

    uint32_t synbits = 0;
#pragma unroll
    for (int k = 0; k < CPT; ++k) synbits |= ((syn0[cl[k] >> 5] >> (cl[k] & 31u)) & 1u) << k;
    const uint32_t next = ticket[ipar];

    // ---------------- iterations ----------------
    uint32_t iter = 0;
    bool still_unsat;
    for (;;) {
      ++iter;
      uint32_t eb = 0;
      if (kFast && iter == 1u) {
        // syndrome bits come from the untouched copy, so toggles of the live bitmap by
        // faster threads need no barrier here
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
          if constexpr (kTab) {
            eb |= vn3_first_tab<kStride>(P, msgs, smem_raw, eo[k], syn2) << k;
          } else {
            eb |= vn3_first(P, A{}, msgs, eo[k], syn0) << k;
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
          // warps whose 32 slots of the LAST round lie beyond the segment's checks skip it
          // (T * CPT covers up to 1.2 Ms + 96 slots: on [[784,24,24]] two of five warps; the
          // branch is uniform per warp).  +2 % (float) / +5 % (int16) at 10 fixed iterations;
          // the same test on the last round of the variable stage made things slower.
          if (k + 1 < CPT || (tid & ~31u) + static_cast<uint32_t>(CPT - 1) * T < Ms) {
            cn6_block(P, A{}, msgs + co[k], (synbits >> k) & 1u);
          }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
          Gam g{};
          if constexpr (!kFast) g = gam[k];
          eb |= vn3_off<kFast>(P, A{}, msgs, eo[k], g) << k;
        }
      }
      eb &= valid;
      const uint32_t changed = eb ^ eprev;
      eprev = eb;
      if (changed) {  // a hard decision flipped: toggle its checks, keep the counter exact
        int32_t delta = 0;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
          if ((changed >> k) & 1u) {
#pragma unroll
            for (int i = 0; i < kDV; ++i) {
              const uint32_t lm = eo[k][i] / kStride;
              const uint32_t bit = 1u << (lm & 31u);
              const uint32_t old = atomicXor(&par[lm >> 5], bit);
              delta += (old & bit) ? -1 : 1;
            }
          }
        }
        atomicAdd(const_cast<uint32_t*>(unsat), static_cast<uint32_t>(delta));
      }
      __syncthreads();
      still_unsat = *unsat != 0u;
      if ((P.early && !still_unsat) || iter >= P.max_iter) break;
    }

    // ---------------- epilogue ----------------
    if (warp == 0 && io.resid) {
      const uint32_t hi = lane < pw ? par[lane] : 0u;
      uint32_t lo = __shfl_up_sync(0xffffffffu, hi, 1);
      if (lane == 0) lo = 0;
      const uint32_t out = cshift ? __funnelshift_l(lo, hi, cshift) : hi;
      if (lane < gspan_out) {
        uint32_t* dst = io.resid + shot * P.syn_w32 + gw0 + lane;
        const uint32_t mask = range_mask(gw0 + lane, seg.c0, c1z);
        if (mask == 0xffffffffu) {
          *dst = out;
        } else {
          atomicAnd(dst, ~mask);
          atomicOr(dst, out & mask);
        }
      }
    }
    if (eprev) {  // few variables decide 1: walk the set bits instead of testing all VPT
      uint32_t* est_g = io.est + shot * P.est_w32;
      for (uint32_t bits = eprev; bits; bits &= bits - 1u) {
        const uint32_t n = seg.v0 + tid + (__ffs(bits) - 1) * T;
        atomicOr(&est_g[n >> 5], 1u << (n & 31u));
      }
    }
    if (tid == 0) {
      io.conv[shot * nseg + s] = still_unsat ? 0 : 1;
      io.iters[shot * nseg + s] = iter;
    }
    if constexpr (kDump) if (io.q_dump != nullptr && shot == io.dump_shot) {
      lean_dump_messages<A>(
          P, io, seg, msgs, syn0, kFast && iter == 1u, static_cast<uint32_t>(sizeof(Msg)), kStride,
          Lay<A>::kROff, 0u,
          [&](uint32_t e, const unsigned char* q, const unsigned char* r, bool first_only, uint32_t flip) {
            if constexpr (A::kInt) {  // (ArithI16F: integer-valued floats, converted exactly)
              static_cast<int32_t*>(io.q_dump)[e] = static_cast<int32_t>(*reinterpret_cast<const Msg*>(q));
              static_cast<int32_t*>(io.r_dump)[e] =
                  first_only ? (flip ? -P.it1_i : P.it1_i) : static_cast<int32_t>(*reinterpret_cast<const Msg*>(r));
            } else if constexpr (sizeof(Msg) == 2) {
              const __half s1 = __ushort_as_half(static_cast<unsigned short>(P.it1_h ^ (flip << 15)));
              static_cast<float*>(io.q_dump)[e] = __half2float(*reinterpret_cast<const __half*>(q));
              static_cast<float*>(io.r_dump)[e] = __half2float(first_only ? s1 : *reinterpret_cast<const __half*>(r));
            } else {
              const float s1 = static_cast<float>(flip ? -P.it1_d : P.it1_d);
              static_cast<float*>(io.q_dump)[e] = *reinterpret_cast<const float*>(q);
              static_cast<float*>(io.r_dump)[e] = first_only ? s1 : *reinterpret_cast<const float*>(r);
            }
          });
    }
    shot = next == kNoShot ? ~0ull : static_cast<uint64_t>(next);
    ipar ^= 1u;
  }

  if (tid == 0) {
    __threadfence();
    const unsigned int done = atomicAdd(&io.sched[1], 1u);
    if (done == gridDim.x - 1) {
      for (uint32_t k = 0; k < 2 + kMaxSegments; ++k) io.sched[k] = 0;
      __threadfence();
    }
  }
}

// =============================================================================
// Single-shot latency kernel: one thread-block CLUSTER per shot, CTA rank s
// decodes segment s on its own SM with the lean item loop above (segments are
// independent graphs, so the iteration loop needs no cross-CTA traffic).
//
// Getting the syndrome in (LatencyCtl::mode):
//   0  passed BY VALUE in the kernel parameters - no load at all on the device;
//   1  read from io.syn (device memory after an explicit H2D copy - the paper's
//      protocol - or mapped host memory);
//   2  PERSISTENT: the cluster stays resident and every CTA polls a 128-byte
//      doorbell block in mapped host memory.  Each 32-byte sector of the block
//      carries the sequence number in its first word, so ONE read that shows the
//      expected number in all four sectors already holds a consistent syndrome
//      (host: data words first, sequence words last).  No kernel launch on the
//      critical path; the leader retires the cluster after idle_ns without work
//      by raising an exit word in every peer's shared memory over DSMEM.
//
// Getting the result out: every CTA writes a SECTORED RECORD for its segment
// straight to (mapped host) memory - 32-byte sectors [seq | 7 data words], each
// written by eight adjacent lanes of one store instruction - holding the
// segment-local estimate and residual words, (converged, iterations) and the
// device time.  The host accepts a record when all of its sectors show the
// shot's sequence number, so the kernel needs no system-scope fence, no cluster
// barrier and no merge pass after the last iteration; shifting the two
// segment-local pieces into the reference's packed layout costs the host a few
// dozen word operations.
// =============================================================================

constexpr uint32_t kInlineSynWords = 64;
constexpr uint32_t kDoorbellWords = 32;         // one 128-byte block
constexpr uint32_t kSectorData = 7;             // data words per 8-word sector
constexpr uint32_t kDoorbellExit = 0xffffffffu;

struct SynInline {
  uint32_t w[kInlineSynWords];
};

struct LatencyCtl {
  uint32_t mode;                      // 0 inline, 1 pointer, 2 persistent doorbell
  uint32_t first_seq;                 // sequence number of the first shot served
  const volatile uint32_t* doorbell;  // mode 2: mapped host memory, kDoorbellWords words
  volatile uint32_t* alive;           // mode 2: cleared when the cluster retires
  uint64_t idle_ns;                   // mode 2: retire after this long without a doorbell
  uint32_t* rec;                      // result records, rec_stride words per segment
  uint32_t rec_stride;
  // degree-padded kernel only: this shot's priors of the absorbed variables (qb_decode_soft),
  // [M] elements of soft_bytes in device-accessible memory, or nullptr
  const void* soft;
  uint32_t soft_bytes;
};

__device__ __forceinline__ uint32_t ld_volatile_global(const volatile uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// position of data word `idx` inside a sectored block / record
__host__ __device__ inline uint32_t sector_pos(uint32_t idx) {
  return 8u * (idx / kSectorData) + 1u + idx % kSectorData;
}
// words of a sectored record holding `n` data words
__host__ __device__ inline uint32_t sector_words(uint32_t n) {
  return 8u * ((n + kSectorData - 1) / kSectorData);
}
// data words of one segment's record: estimate words, residual words, converged,
// iterations, device ns (lo, hi)
__host__ __device__ inline uint32_t record_data_words(uint32_t nvars, uint32_t nchecks) {
  return ((nvars + 31u) >> 5) + ((nchecks + 31u) >> 5) + 4u;
}

template <class A, int CPT, int VPT, bool kFast>
__global__ void __launch_bounds__(1024, 1)
decode_lean_latency_kernel(const __grid_constant__ DecodeParams P,
                           const __grid_constant__ ShotIO io,
                           const __grid_constant__ LatencyCtl ctl,
                           const __grid_constant__ SynInline syn_in) {
  using Msg = typename A::Msg;
  using Gam = typename A::Gam;
  constexpr uint32_t kStride = Lay<A>::kStride;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t tid = threadIdx.x, T = blockDim.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t nseg = P.nseg;
  const uint32_t s = cluster.block_rank();  // == segment
  const SegmentDev seg = P.segs[s];
  const uint32_t Ms = seg.c1 - seg.c0, Ns = seg.v1 - seg.v0;
  const uint32_t pw = lean_pw(P.seg_mmax);  // words of a local check bitmap
  const uint32_t ew = lean_pw(P.seg_nmax);  // words of a local variable bitmap
  const uint32_t pws = (Ms + 31u) >> 5, ews = (Ns + 31u) >> 5;
  const uint32_t gw0 = seg.c0 >> 5, gspan = ((seg.c1 - 1) >> 5) - gw0 + 1, cshift = seg.c0 & 31u;

  // ---- shared memory: messages | par | ehat | unsat | exit word
  unsigned char* const msgs = smem_raw;
  const size_t msg_bytes = (static_cast<size_t>(P.seg_mmax + 1) * kStride + 15) & ~size_t(15);
  uint32_t* const bits = reinterpret_cast<uint32_t*>(smem_raw + msg_bytes);
  uint32_t* const par = bits;                       // [pw]
  uint32_t* const ehat = bits + pw;                 // [ew]
  volatile uint32_t* const unsat = bits + pw + ew;  // [1]
  volatile uint32_t* const exit_word = bits + pw + ew + 1;
  uint32_t* const cmd_word = bits + pw + ew + 2;

  // ---- per-thread tables
  uint32_t eo[VPT][kDV], co[CPT], cl[CPT], valid = 0;
  Gam gam[kFast ? 1 : VPT];
  {
    const Gam* __restrict__ gamma = static_cast<const Gam*>(P.gamma);
    const uint32_t dummy = P.seg_mmax * kStride;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const uint32_t n = seg.v0 + tid + k * T;
      const bool ok = n < seg.v1;
      valid |= (ok ? 1u : 0u) << k;
#pragma unroll
      for (int i = 0; i < kDV; ++i) {
        const uint32_t e = ok ? P.var_edges[n * kDV + i] - seg.e0 : 0u;
        eo[k][i] = ok ? (e / kDC) * kStride + (e % kDC) * static_cast<uint32_t>(sizeof(Msg))
                      : dummy + i * static_cast<uint32_t>(sizeof(Msg));
      }
      if constexpr (!kFast) gam[k] = ok ? gamma[n] : static_cast<Gam>(1);
    }
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const uint32_t m = tid + k * T;
      cl[k] = m < Ms ? m : Ms;
      co[k] = (m < Ms ? m : P.seg_mmax) * kStride;
    }
  }
  for (uint32_t b = tid; b < kStride; b += T) msgs[P.seg_mmax * kStride + b] = 0;
  if (tid == 0) *exit_word = 0u;
  __syncthreads();
  if (ctl.mode == 2u) cluster.sync();  // exit words exist before the leader may raise them

  uint32_t* const rec = ctl.rec + s * ctl.rec_stride;
  const uint32_t ndata = ews + pws + 4u;
  const uint32_t nrec = sector_words(ndata);
  uint32_t last = ctl.first_seq - 1u;
  uint64_t t_idle0 = globaltimer_ns();
  for (;;) {
    // ---------------- obtain the shot: warp 0 ends up with packed word gw0 + lane -------
    uint32_t cmd = last + 1u;
    uint32_t raw = 0;
    uint64_t t_begin = 0;
    if (warp == 0) {
      if (ctl.mode == 2u) {
        uint32_t spins = 0, val = 0;
        for (;;) {
          val = ld_volatile_global(ctl.doorbell + lane);
          const uint32_t sq = __shfl_sync(0xffffffffu, val, lane & ~7u);  // my sector's number
          if (__all_sync(0xffffffffu, sq == cmd)) break;
          if (__any_sync(0xffffffffu, sq == kDoorbellExit) || *exit_word != 0u) {
            cmd = kDoorbellExit;
            break;
          }
          if (s == 0 && (++spins & 63u) == 0u && globaltimer_ns() - t_idle0 > ctl.idle_ns) {
            // leader: retire the whole cluster
            if (lane < nseg) *cluster.map_shared_rank(const_cast<uint32_t*>(exit_word), lane) = 1u;
            cmd = kDoorbellExit;
            break;
          }
        }
        const uint32_t src = lane < gspan ? sector_pos(gw0 + lane) : 0u;
        raw = __shfl_sync(0xffffffffu, val, src & 31u);
      } else if (lane < gspan) {
        raw = ctl.mode == 0u ? syn_in.w[gw0 + lane] : io.syn[gw0 + lane];
      }
      if (lane >= gspan) raw = 0;
      t_begin = globaltimer_ns();
      if (lane == 0) {
        cmd_word[0] = cmd;
        cmd_word[1] = static_cast<uint32_t>(t_begin);
        cmd_word[2] = static_cast<uint32_t>(t_begin >> 32);
      }
    }

    // ---------------- prologue ----------------
    if (warp == 0) {
      uint32_t nb = __shfl_down_sync(0xffffffffu, raw, 1);
      if (lane + 1 >= gspan) nb = 0;
      uint32_t loc = cshift ? __funnelshift_r(raw, nb, cshift) : raw;
      if (lane >= pws) {
        loc = 0;
      } else if (Ms - lane * 32u < 32u) {
        loc &= (1u << (Ms - lane * 32u)) - 1u;
      }
      if (lane < pw) par[lane] = loc;
      const uint32_t cnt = __reduce_add_sync(0xffffffffu, __popc(loc));
      if (lane == 0) *unsat = cnt;
    }
    for (uint32_t w = tid; w < ew; w += T) ehat[w] = 0;
    // the debug dump wants r of the first check stage too, so it takes the long way
    const bool first_from_syndrome = kFast && io.q_dump == nullptr;
    if (!first_from_syndrome) {
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        Gam g;
        if constexpr (kFast) {
          if constexpr (A::kInt) g = P.gamma_i; else g = P.gamma_f;
        } else {
          g = gam[k];
        }
        const Msg init = prior_as_msg<A>(g);
#pragma unroll
        for (int i = 0; i < kDV; ++i) *reinterpret_cast<Msg*>(msgs + eo[k][i]) = init;
      }
    }
    uint32_t eprev = 0;
    __syncthreads();
    cmd = cmd_word[0];
    if (cmd == kDoorbellExit) break;
    t_begin = static_cast<uint64_t>(cmd_word[1]) | (static_cast<uint64_t>(cmd_word[2]) << 32);
    uint32_t synbits = 0;
#pragma unroll
    for (int k = 0; k < CPT; ++k) synbits |= ((par[cl[k] >> 5] >> (cl[k] & 31u)) & 1u) << k;

    // ---------------- iterations ----------------
    uint32_t iter = 0;
    bool still_unsat;
    for (;;) {
      ++iter;
      uint32_t eb = 0;
      if (first_from_syndrome && iter == 1u) {
#pragma unroll
        for (int k = 0; k < VPT; ++k) eb |= vn3_first(P, A{}, msgs, eo[k], par) << k;
        __syncthreads();  // every thread has read its syndrome bits before any toggle
      } else {
#pragma unroll
        for (int k = 0; k < CPT; ++k) cn6_block(P, A{}, msgs + co[k], (synbits >> k) & 1u);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
          Gam g{};
          if constexpr (!kFast) g = gam[k];
          eb |= vn3_off<kFast>(P, A{}, msgs, eo[k], g) << k;
        }
      }
      eb &= valid;
      const uint32_t changed = eb ^ eprev;
      eprev = eb;
      if (changed) {
        int32_t delta = 0;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
          if ((changed >> k) & 1u) {
#pragma unroll
            for (int i = 0; i < kDV; ++i) {
              const uint32_t lm = eo[k][i] / kStride;
              const uint32_t bit = 1u << (lm & 31u);
              const uint32_t old = atomicXor(&par[lm >> 5], bit);
              delta += (old & bit) ? -1 : 1;
            }
          }
        }
        atomicAdd(const_cast<uint32_t*>(unsat), static_cast<uint32_t>(delta));
      }
      __syncthreads();
      still_unsat = *unsat != 0u;
      if ((P.early && !still_unsat) || iter >= P.max_iter) break;
    }

    // ---------------- publish this segment's record ----------------
    if (eprev) {
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        if ((eprev >> k) & 1u) {
          const uint32_t nl = tid + k * T;
          atomicOr(&ehat[nl >> 5], 1u << (nl & 31u));
        }
      }
    }
    if (io.q_dump) {  // debug: messages back in reference edge order
      for (uint32_t e = tid; e < seg.e1 - seg.e0; e += T) {
        const unsigned char* src = msgs + (e / kDC) * kStride + (e % kDC) * sizeof(Msg);
        if constexpr (A::kInt) {
          static_cast<int32_t*>(io.q_dump)[seg.e0 + e] = *reinterpret_cast<const Msg*>(src);
          static_cast<int32_t*>(io.r_dump)[seg.e0 + e] =
              *reinterpret_cast<const Msg*>(src + Lay<A>::kROff);
        } else {
          static_cast<float*>(io.q_dump)[seg.e0 + e] =
              static_cast<float>(*reinterpret_cast<const Msg*>(src));
          static_cast<float*>(io.r_dump)[seg.e0 + e] =
              static_cast<float>(*reinterpret_cast<const Msg*>(src + Lay<A>::kROff));
        }
      }
    }
    __syncthreads();
    {
      const uint64_t ns = globaltimer_ns() - t_begin;
      for (uint32_t w = tid; w < nrec; w += T) {
        const uint32_t slot = w & 7u;
        uint32_t v = cmd;
        if (slot) {
          const uint32_t d = (w >> 3) * kSectorData + slot - 1u;
          if (d < ews) {
            v = ehat[d];
          } else if (d < ews + pws) {
            v = par[d - ews];
          } else if (d == ews + pws) {
            v = still_unsat ? 0u : 1u;
          } else if (d == ews + pws + 1u) {
            v = iter;
          } else if (d == ews + pws + 2u) {
            v = static_cast<uint32_t>(ns);
          } else if (d == ews + pws + 3u) {
            v = static_cast<uint32_t>(ns >> 32);
          } else {
            v = 0u;
          }
        }
        rec[w] = v;
      }
    }
    t_idle0 = globaltimer_ns();
    last = cmd;
    if (ctl.mode != 2u) break;
    // The next prologue overwrites the bitmap this record was read from.  The host only rings
    // the next doorbell after it has seen the whole record, i.e. after every read above - an
    // ordering no tool can see; the barrier states it (the record is already out: the host's
    // latency does not include it).
    __syncthreads();
  }
  if (ctl.mode == 2u) {
    if (s == 0 && tid == 0 && ctl.alive) {
      *ctl.alive = 0u;
      __threadfence_system();
    }
    cluster.sync();  // no CTA leaves while the leader may still raise its exit word
  }
}

__host__ __device__ inline size_t lean_latency_smem_bytes(uint32_t seg_mmax, uint32_t seg_nmax,
                                                          int arith) {
  const size_t msg = (static_cast<size_t>(seg_mmax + 1) * lean_stride(arith) + 15) & ~size_t(15);
  return msg + 4 * (static_cast<size_t>(lean_pw(seg_mmax)) + lean_pw(seg_nmax) + 8);
}

}  // namespace qb

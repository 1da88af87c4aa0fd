// Throughput kernel for IRREGULAR graphs: degree-padded (ELL) message blocks.
//
// The code loader's answer to "warps must never diverge on node degree"
// (north-star item 1): every check owns a block of DC message slots and every
// variable a list of DV edge slots, where DC / DV are compile-time bounds on the
// degrees of the graph at hand.  Rows shorter than the bound are PADDED instead
// of being looped over with a data-dependent trip count:
//
//  * a check of degree d < DC keeps a SENTINEL in its q slots d..DC-1 that can
//    never be one of the two smallest magnitudes and has a positive sign, so the
//    branch-free two-minimum / sign-parity update over all DC slots yields the
//    reference's result for the d real edges.  The sentinel of a degree-1 check
//    is 64 (resp. kmax in the integer modes), which makes the ordinary update
//    emit the reference's special value alpha * sigma * 64 (decoder.cpp:251-258)
//    without a special case;
//  * a variable of degree d < DV points its slots d..DV-1 at a DUMMY block behind the real
//    ones whose r half is never written: the padded terms add +0 to the posterior (exact in
//    every arithmetic mode) and the padded q stores land in a word only that thread writes
//    (ell_dummy_blocks).  A degree-1 variable keeps q = gamma (decoder.cpp:324-329): its single
//    store is predicated off in the floating-point modes, where (gamma + r) - r need not equal
//    gamma;
//  * a degree-1 variable whose check has no other one is ABSORBED by that check: its
//    message q = gamma never changes (it sits in the check's block for the life of the
//    CTA), and its posterior gamma + r and hard decision are evaluated by the check's
//    thread right after it has produced r - the variable costs no slot on the
//    variable side at all.  On the phenomenological graphs [H | I] this removes a third
//    of the variables (one measurement-error variable per check) from the variable
//    stage and a third of the per-thread offset registers;
//  * thread <-> node assignment, byte offsets of every slot and the priors live
//    in registers for the life of the persistent CTA, exactly as in the (6,3)
//    lean kernel (kernel_lean.cuh), whose item loop, counter-based stop test and
//    bit-vector I/O this kernel shares.
//
// The block stride is an odd number of 32-bit words, so 32 consecutive checks
// (and, graph permitting, the variable-side gathers) touch distinct banks.
//
// Covers e.g. the phenomenological-noise graphs diag([Hz | I], [Hx | I]) of
// BASELINE config 5 (check degree 7, variable degrees 3 and 1), hypergraph- and
// lifted-product codes with mixed degrees, and the toy 3x6 fixture.  Arithmetic
// is the reference's in every mode (bit-exact for float / int8 / int16).
#pragma once

#include "common.cuh"
#include "kernel_lean.cuh"

namespace qb {

__host__ __device__ inline uint32_t ell_stride_bytes(uint32_t msg_bytes, uint32_t dc) {
  uint32_t w = (2u * dc * msg_bytes + 3u) / 4u;
  if ((w & 1u) == 0u) ++w;
  return 4u * w;
}
__host__ __device__ inline uint32_t ell_pw(uint32_t seg_mmax) { return ((seg_mmax + 2u) >> 5) + 1u; }
// Dummy blocks behind the real ones.  A padded variable slot (degree below the bound, or an
// idle thread) must load r = 0 and store its q somewhere harmless: thread t owns slot t % DC of
// dummy block t / DC - its q word is written by that thread only, the r half of every dummy
// block is never written and stays zero.  (One shared scratch block would do for the results,
// but racecheck rightly reports its q words as write-after-write hazards between threads.)
__host__ __device__ inline uint32_t ell_dummy_blocks(uint32_t threads, uint32_t dc) {
  return (threads + dc - 1u) / dc;
}
__host__ __device__ inline size_t ell_msg_region_bytes(uint32_t seg_mmax, uint32_t stride,
                                                       uint32_t threads, uint32_t dc) {
  // ... plus one block that thread slots WITHOUT a check run their (branch-free) update on
  return (static_cast<size_t>(seg_mmax + ell_dummy_blocks(threads, dc) + 1u) * stride + 15) & ~size_t(15);
}
__host__ __device__ inline size_t ell_smem_bytes(uint32_t seg_mmax, uint32_t msg_bytes, uint32_t dc,
                                                 uint32_t threads) {
  return ell_msg_region_bytes(seg_mmax, ell_stride_bytes(msg_bytes, dc), threads, dc) +
         4 * (2 * static_cast<size_t>(ell_pw(seg_mmax)) + 8);
}

// min1 / min2 of N keys, branch-free (3 operations per key after the first two).
template <int N, class T>
__device__ __forceinline__ void two_smallest_n(const T (&a)[N], T& m1, T& m2) {
  m1 = min(a[0], a[1]);
  m2 = max(a[0], a[1]);
#pragma unroll
  for (int j = 2; j < N; ++j) {
    m2 = min(m2, max(m1, a[j]));
    m1 = min(m1, a[j]);
  }
}

// ---- sentinels of padded check slots -------------------------------------------
template <class A> struct EllSentinel;
template <> struct EllSentinel<ArithF32> {
  static __device__ __forceinline__ float pad(const DecodeParams&) { return __uint_as_float(0x7f800000u); }
  static __device__ __forceinline__ float deg1(const DecodeParams&) { return 64.0f; }
};
template <> struct EllSentinel<ArithF16> {
  static __device__ __forceinline__ __half pad(const DecodeParams&) { return __ushort_as_half(0x7c00); }
  static __device__ __forceinline__ __half deg1(const DecodeParams&) { return __ushort_as_half(0x5400); }
};
template <> struct EllSentinel<ArithI8> {
  static __device__ __forceinline__ int8_t pad(const DecodeParams& P) { return static_cast<int8_t>(P.kmax); }
  static __device__ __forceinline__ int8_t deg1(const DecodeParams& P) { return static_cast<int8_t>(P.kmax); }
};
template <> struct EllSentinel<ArithI16> {
  static __device__ __forceinline__ int16_t pad(const DecodeParams& P) { return static_cast<int16_t>(P.kmax); }
  static __device__ __forceinline__ int16_t deg1(const DecodeParams& P) { return static_cast<int16_t>(P.kmax); }
};

template <> struct EllSentinel<ArithI32> {
  static __device__ __forceinline__ int32_t pad(const DecodeParams& P) { return P.kmax; }
  static __device__ __forceinline__ int32_t deg1(const DecodeParams& P) { return P.kmax; }
};

// ---- check update over one padded block ------------------------------------------

template <int DC>
__device__ __forceinline__ void cn_ell(const DecodeParams& P, ArithF32, unsigned char* blk,
                                       uint32_t syn_bit) {
  const float* qp = reinterpret_cast<const float*>(blk);
  float v[DC], a[DC];
#pragma unroll
  for (int j = 0; j < DC; ++j) {
    v[j] = qp[j];
    a[j] = fabsf(v[j]);
  }
  float m1 = fminf(a[0], a[1]), m2 = fmaxf(a[0], a[1]);
#pragma unroll
  for (int j = 2; j < DC; ++j) {
    m2 = fminf(m2, fmaxf(m1, a[j]));
    m1 = fminf(m1, a[j]);
  }
  // float(alpha * |min|): fp64 product, one rounding (decoder.cpp:302-307)
  uint32_t s1 = __float_as_uint(static_cast<float>(P.alpha * static_cast<double>(m1)));
  uint32_t s2 = __float_as_uint(static_cast<float>(P.alpha * static_cast<double>(m2)));
  // keep the two products where they are: left alone, the compiler turns "select one of two
  // products" into "product of the selected minimum" PER EDGE - DC widenings, multiplies and
  // narrowings per check instead of two (14 of the 77 conversions per thread and iteration
  // on the (7,3) graphs, with the conversion pipe at 71 %)
  asm volatile("" : "+r"(s1), "+r"(s2));
  uint32_t sx = syn_bit << 31;
#pragma unroll
  for (int j = 0; j < DC; ++j) sx ^= __float_as_uint(v[j]);
  float* rp = reinterpret_cast<float*>(blk + DC * sizeof(float));
#pragma unroll
  for (int j = 0; j < DC; ++j) {
    const uint32_t o = (a[j] == m1 ? s2 : s1) | ((sx ^ __float_as_uint(v[j])) & 0x80000000u);
    rp[j] = __uint_as_float(o);
  }
}

template <int DC>
__device__ __forceinline__ void cn_ell(const DecodeParams& P, ArithF16, unsigned char* blk,
                                       uint32_t syn_bit) {
  const unsigned short* qp = reinterpret_cast<const unsigned short*>(blk);
  uint32_t u[DC];
  int32_t a[DC];
#pragma unroll
  for (int j = 0; j < DC; ++j) {
    u[j] = qp[j];
    a[j] = static_cast<int32_t>(u[j] & 0x7fffu);  // non-negative halves order like integers
  }
  int32_t m1, m2;
  two_smallest_n<DC>(a, m1, m2);
  const __half alpha = __ushort_as_half(P.alpha_h);
  uint32_t s1 =
      __half_as_ushort(__hmul(alpha, __ushort_as_half(static_cast<unsigned short>(m1))));
  uint32_t s2 =
      __half_as_ushort(__hmul(alpha, __ushort_as_half(static_cast<unsigned short>(m2))));
  asm volatile("" : "+r"(s1), "+r"(s2));  // two products per check, not one per edge (see ArithF32)
  uint32_t sx = syn_bit << 15;
#pragma unroll
  for (int j = 0; j < DC; ++j) sx ^= u[j];
  unsigned short* rp = reinterpret_cast<unsigned short*>(blk + DC * sizeof(__half));
#pragma unroll
  for (int j = 0; j < DC; ++j) {
    rp[j] = static_cast<unsigned short>((a[j] == m1 ? s2 : s1) | ((sx ^ u[j]) & 0x8000u));
  }
}

template <class A, int DC>
__device__ __forceinline__ void cn_ell_int(const DecodeParams& P, unsigned char* blk,
                                           uint32_t syn_bit) {
  using MsgI = typename A::Msg;
  const MsgI* qp = reinterpret_cast<const MsgI*>(blk);
  int32_t v[DC], a[DC];
#pragma unroll
  for (int j = 0; j < DC; ++j) {
    v[j] = qp[j];
    a[j] = abs(v[j]);
  }
  int32_t m1, m2;
  two_smallest_n<DC>(a, m1, m2);
  int32_t s1 = scale_q16(static_cast<uint32_t>(m1), P.alpha_fx);
  int32_t s2 = scale_q16(static_cast<uint32_t>(m2), P.alpha_fx);
  asm volatile("" : "+r"(s1), "+r"(s2));  // two scalings per check, not one per edge (see ArithF32)
  int32_t sx = static_cast<int32_t>(syn_bit << 31);
#pragma unroll
  for (int j = 0; j < DC; ++j) sx ^= v[j];
  MsgI* rp = reinterpret_cast<MsgI*>(blk + DC * sizeof(MsgI));
#pragma unroll
  for (int j = 0; j < DC; ++j) {
    const int32_t mag = a[j] == m1 ? s2 : s1;
    const int32_t neg = (sx ^ v[j]) >> 31;  // 0 or -1
    rp[j] = static_cast<MsgI>((mag ^ neg) - neg);
  }
}
template <int DC>
__device__ __forceinline__ void cn_ell(const DecodeParams& P, ArithI8, unsigned char* blk,
                                       uint32_t syn_bit) {
  cn_ell_int<ArithI8, DC>(P, blk, syn_bit);
}
template <int DC>
__device__ __forceinline__ void cn_ell(const DecodeParams& P, ArithI16, unsigned char* blk,
                                       uint32_t syn_bit) {
  cn_ell_int<ArithI16, DC>(P, blk, syn_bit);
}
template <int DC>
__device__ __forceinline__ void cn_ell(const DecodeParams& P, ArithI32, unsigned char* blk,
                                       uint32_t syn_bit) {
  cn_ell_int<ArithI32, DC>(P, blk, syn_bit);
}

// ---- hard decision of an absorbed degree-1 variable: gamma + r < 0 in the mode's arithmetic
__device__ __forceinline__ uint32_t absorbed_decision(ArithF32, float q, float r) {
  // decoder.cpp:319-323 decides on the sign of the fp64 sum gamma + r, which is EXACT for two
  // fp32 terms; the fp32 sum is its correctly rounded image and rounding cannot change a sign
  // (a non-zero sum of two floats is at least 2^-149 in magnitude, so it cannot flush to zero
  // either): one FADD instead of two widening conversions and a DADD.
  return (q + r) < 0.0f ? 1u : 0u;
}
__device__ __forceinline__ uint32_t absorbed_decision(ArithF16, __half q, __half r) {
  return h_neg(__hadd(q, r)) ? 1u : 0u;
}
template <class A>
__device__ __forceinline__ uint32_t absorbed_decision(A, int32_t q, int32_t r) {
  return static_cast<uint32_t>(q + r) >> 31;
}

// ---- variable update over DV padded slots; returns 1 iff the variable decides 1 ----
// `keep0`: the variable has degree 1, so its only real message stays gamma.

template <int DC, int DV>
__device__ __forceinline__ uint32_t vn_ell(const DecodeParams& P, ArithF32, unsigned char* base,
                                           const uint32_t (&eo)[DV], float gamma, bool keep0) {
  constexpr uint32_t R = DC * sizeof(float);
  double r[DV];
  double total = static_cast<double>(gamma);  // ascending edge order (decoder.cpp:319-322)
#pragma unroll
  for (int i = 0; i < DV; ++i) {
    r[i] = static_cast<double>(*reinterpret_cast<const float*>(base + eo[i] + R));
    total += r[i];
  }
#pragma unroll
  for (int i = 0; i < DV; ++i) {
    float x = static_cast<float>(total - r[i]);
    x = fminf(fmaxf(x, -P.clamp_f), P.clamp_f);  // decoder.cpp:238-241 (monotone, so after rounding)
    if (i > 0 || !keep0) *reinterpret_cast<float*>(base + eo[i]) = x;
  }
  return static_cast<uint32_t>(__double2hiint(total)) >> 31;
}

template <int DC, int DV>
__device__ __forceinline__ uint32_t vn_ell(const DecodeParams& P, ArithF16, unsigned char* base,
                                           const uint32_t (&eo)[DV], float gamma, bool keep0) {
  constexpr uint32_t R = DC * sizeof(__half);
  __half r[DV];
  __half total = __float2half_rn(fminf(fmaxf(gamma, -kHalfClamp), kHalfClamp));
#pragma unroll
  for (int i = 0; i < DV; ++i) {
    r[i] = *reinterpret_cast<const __half*>(base + eo[i] + R);
    total = __hadd(total, r[i]);
  }
#pragma unroll
  for (int i = 0; i < DV; ++i) {
    const __half x = h_clamp(__hsub(total, r[i]));
    if (i > 0 || !keep0) *reinterpret_cast<__half*>(base + eo[i]) = x;
  }
  return h_neg(total) ? 1u : 0u;
}

template <class A, int DC, int DV>
__device__ __forceinline__ uint32_t vn_ell_int(const DecodeParams& P, unsigned char* base,
                                               const uint32_t (&eo)[DV], int32_t gamma) {
  using MsgI = typename A::Msg;
  constexpr uint32_t R = DC * sizeof(MsgI);
  int32_t r[DV];
  int32_t total = gamma;
#pragma unroll
  for (int i = 0; i < DV; ++i) {
    r[i] = *reinterpret_cast<const MsgI*>(base + eo[i] + R);
    total += r[i];
  }
  // a degree-1 variable stores sat(gamma + r - r) = gamma: no special case needed
#pragma unroll
  for (int i = 0; i < DV; ++i) {
    *reinterpret_cast<MsgI*>(base + eo[i]) =
        static_cast<MsgI>(max(-P.kmax, min(P.kmax, total - r[i])));
  }
  return static_cast<uint32_t>(total) >> 31;
}
template <int DC, int DV>
__device__ __forceinline__ uint32_t vn_ell(const DecodeParams& P, ArithI8, unsigned char* base,
                                           const uint32_t (&eo)[DV], int32_t gamma, bool) {
  return vn_ell_int<ArithI8, DC, DV>(P, base, eo, gamma);
}
template <int DC, int DV>
__device__ __forceinline__ uint32_t vn_ell(const DecodeParams& P, ArithI16, unsigned char* base,
                                           const uint32_t (&eo)[DV], int32_t gamma, bool) {
  return vn_ell_int<ArithI16, DC, DV>(P, base, eo, gamma);
}
template <int DC, int DV>
__device__ __forceinline__ uint32_t vn_ell(const DecodeParams& P, ArithI32, unsigned char* base,
                                           const uint32_t (&eo)[DV], int32_t gamma, bool) {
  return vn_ell_int<ArithI32, DC, DV>(P, base, eo, gamma);
}

// ---- per-shot priors of the absorbed variables ("soft syndromes") -------------------
// ShotIO::soft holds, for every shot, one value per check: the prior of the degree-1
// variable that check absorbs (on [H | I] graphs the measurement-error variable of that
// check, i.e. the reliability |LLR| of the measured syndrome bit).  Element type by mode:
// float (float / half), int8 (int8), int16 (int16) - the integer values are the already
// quantised priors, what the reference's quantize_saturate (decoder.cpp:115-122) yields.
template <class A>
__device__ __forceinline__ typename A::Msg load_soft(const ShotIO& io, uint64_t idx);
template <>
__device__ __forceinline__ float load_soft<ArithF32>(const ShotIO& io, uint64_t idx) {
  return static_cast<const float*>(io.soft)[idx] + 0.0f;  // -0.0 -> +0.0, as the loader does
}
template <>
__device__ __forceinline__ __half load_soft<ArithF16>(const ShotIO& io, uint64_t idx) {
  return prior_as_msg<ArithF16>(static_cast<const float*>(io.soft)[idx]);
}
template <>
__device__ __forceinline__ int32_t load_soft<ArithI32>(const ShotIO& io, uint64_t idx) {
  return io.soft_bytes == 1u ? static_cast<int32_t>(static_cast<const int8_t*>(io.soft)[idx])
                             : static_cast<int32_t>(static_cast<const int16_t*>(io.soft)[idx]);
}

// Parity hook of the batch kernels (qb_decode_batch_debug): final messages of one shot in
// reference edge order (padded slots are not edges and are skipped).
template <class Store>
__device__ __noinline__ void ell_dump_messages(const DecodeParams& P, const SegmentDev seg,
                                               const unsigned char* msgs, uint32_t stride,
                                               uint32_t slot_bytes, uint32_t roff, uint32_t lane_off,
                                               Store store) {
  for (uint32_t m = seg.c0 + threadIdx.x; m < seg.c1; m += blockDim.x) {
    const uint32_t e0 = P.check_off[m], e1 = P.check_off[m + 1];
    for (uint32_t e = e0; e < e1; ++e) {
      const unsigned char* q = msgs + (m - seg.c0) * stride + (e - e0) * slot_bytes + lane_off;
      store(e, q, q + roff);
    }
  }
}

// ---- the kernel -------------------------------------------------------------------
// Work item = (shot, segment); a CTA serves one segment for its whole life and
// draws shots from that segment's ticket queue (as decode_lean_kernel).
// kSoft: the absorbed variables' priors come per shot from ShotIO::soft.

template <class A, int DC, int DV, int CPT, int VPT, int MAXT, int MINB, bool kSoft = false,
          bool kDump = false>
__global__ void __launch_bounds__(MAXT, MINB)
decode_ell_kernel(const __grid_constant__ DecodeParams P, const __grid_constant__ ShotIO io) {
  static_assert(DV <= DC, "padded variable slots live in the q half of the zero block");
  using Msg = typename A::Msg;
  using Gam = typename A::Gam;
  constexpr uint32_t kMsg = static_cast<uint32_t>(sizeof(Msg));
  const uint32_t kStride = ell_stride_bytes(kMsg, DC);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t tid = threadIdx.x, T = blockDim.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t nwarps = T >> 5;
  const uint32_t nseg = P.nseg;
  const uint32_t s = blockIdx.x % nseg;
  const uint32_t peer = blockIdx.x / nseg;
  const uint32_t peers = (gridDim.x - s + nseg - 1) / nseg;
  const SegmentDev seg = P.segs[s];
  const uint32_t Ms = seg.c1 - seg.c0;
  const uint32_t pw = ell_pw(P.seg_mmax);
  const uint32_t pws = (Ms + 31u) >> 5;
  // at most 32 packed words per segment (the loader checks): one lane per word
  const uint32_t gw0 = seg.c0 >> 5, gspan = Ms ? ((seg.c1 - 1) >> 5) - gw0 + 1 : 0u;
  const uint32_t cshift = seg.c0 & 31u;
  // the last segment also owns the padding bits of the packed rows (they are written as 0)
  const uint32_t v1z = s + 1u == nseg ? P.est_w32 * 32u : seg.v1;
  const uint32_t c1z = s + 1u == nseg ? P.syn_w32 * 32u : seg.c1;
  const uint32_t vw0 = seg.v0 >> 5, vspan = v1z > seg.v0 ? ((v1z - 1) >> 5) - vw0 + 1 : 0u;
  const uint32_t gspan_out = c1z > seg.c0 ? ((c1z - 1) >> 5) - gw0 + 1 : 0u;

  unsigned char* const msgs = smem_raw;
  const size_t msg_bytes = ell_msg_region_bytes(P.seg_mmax, kStride, T, DC);
  uint32_t* const bits = reinterpret_cast<uint32_t*>(smem_raw + msg_bytes);
  uint32_t* const unsat_ctr = bits + 2 * pw;   // [2]
  uint32_t* const ticket = bits + 2 * pw + 2;  // [2]
  const uint32_t scratch_off = P.seg_mmax * kStride;  // first dummy block (see ell_dummy_blocks)
  const uint32_t pad_off = scratch_off + (tid / DC) * kStride + (tid % DC) * kMsg;  // this thread's slot
  const uint32_t scribble_off = scratch_off + ell_dummy_blocks(T, DC) * kStride;  // thread slots without a check

  // the dummy blocks start out as zeros (before any q store)
  const uint64_t t_entry = io.kernel_ns ? globaltimer_ns() : 0ull;  // single-shot use only
  for (uint32_t b = tid; b < (ell_dummy_blocks(T, DC) + 1u) * kStride; b += T) msgs[scratch_off + b] = 0;

  // ---- per-thread tables
  uint32_t eo[VPT][DV], co[CPT], cl[CPT], valid = 0, keep0 = 0;
  uint32_t absorb = 0;  // byte k: slot of the variable absorbed by this thread's k-th check, or kNoAbsorb
  static_assert(CPT <= 4, "absorbed slots are packed one byte per check");
  Gam gam[VPT];
  const uint32_t nv = P.ell_nvars[s];  // variables updated on the variable side
  {
    const Gam* __restrict__ gamma = static_cast<const Gam*>(P.gamma);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const uint32_t idx = tid + k * T;
      const bool ok = idx < nv;
      const uint32_t n = ok ? P.ell_vars[seg.v0 + idx] : 0u;
      const uint32_t b = ok ? P.var_off[n] : 0u;
      const uint32_t deg = ok ? P.var_off[n + 1] - b : 0u;
      valid |= (ok ? 1u : 0u) << k;
      keep0 |= (deg == 1u ? 1u : 0u) << k;
#pragma unroll
      for (int i = 0; i < DV; ++i) {
        uint32_t off = pad_off;
        if (static_cast<uint32_t>(i) < deg) {
          const uint32_t e = P.var_edges[b + i];
          const uint32_t m = P.edge_check[e];
          off = (m - seg.c0) * kStride + (e - P.check_off[m]) * kMsg;
        }
        eo[k][i] = off;
      }
      gam[k] = ok ? gamma[n] : static_cast<Gam>(1);
    }
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const uint32_t m = tid + k * T;
      const bool ok = m < Ms;
      cl[k] = ok ? m : Ms;  // no check: bit Ms of the bitmap (always 0) and the scribble block
      co[k] = ok ? m * kStride : scribble_off;
      uint32_t aslot = kNoAbsorb;
      if (ok) {  // sentinels of the padded slots: written once, never overwritten
        const uint32_t e0 = P.check_off[seg.c0 + m];
        const uint32_t deg = P.check_off[seg.c0 + m + 1] - e0;
        const Msg sent = deg == 1u ? EllSentinel<A>::deg1(P) : EllSentinel<A>::pad(P);
#pragma unroll
        for (int j = 0; j < DC; ++j) {
          if (static_cast<uint32_t>(j) >= deg) *reinterpret_cast<Msg*>(msgs + co[k] + j * kMsg) = sent;
        }
        aslot = P.ell_abs[seg.c0 + m];
        if (aslot != kNoAbsorb) {  // the absorbed variable's message: its prior, for ever
          *reinterpret_cast<Msg*>(msgs + co[k] + aslot * kMsg) =
              prior_as_msg<A>(gamma[P.edge_var[e0 + aslot]]);
        }
      }
      absorb |= aslot << (8 * k);
    }
  }

  uint64_t shot = peer;
  uint32_t raw_next = 0;
  if (warp == 0 && lane < gspan && shot < io.nshots) {
    raw_next = io.syn[shot * P.syn_w32 + gw0 + lane];
  }
  // per-shot priors of this thread's absorbed variables, fetched one shot ahead
  Msg soft_next[kSoft ? CPT : 1];
  auto fetch_soft = [&](uint64_t sh) {
    if constexpr (kSoft) {
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        if (cl[k] < Ms && ((absorb >> (8 * k)) & 0xffu) != kNoAbsorb) {
          soft_next[k] = load_soft<A>(io, sh * P.M + seg.c0 + cl[k]);
        }
      }
    }
  };
  if (shot < io.nshots) fetch_soft(shot);
  uint32_t ipar = 0;
  __syncthreads();

  while (shot < io.nshots) {
    uint32_t* const par = bits + ipar * pw;
    volatile uint32_t* const unsat = unsat_ctr + ipar;
    // ---------------- prologue ----------------
    if (warp == 0) {
      // packed syndrome words -> segment-local bitmap, and its population count
      uint32_t nb = __shfl_down_sync(0xffffffffu, raw_next, 1);
      if (lane + 1 >= gspan) nb = 0;
      uint32_t loc = cshift ? __funnelshift_r(raw_next, nb, cshift) : raw_next;
      if (lane >= pws) {
        loc = 0;
      } else if (Ms - lane * 32u < 32u) {
        loc &= (1u << (Ms - lane * 32u)) - 1u;
      }
      if (lane < pw) par[lane] = loc;
      const uint32_t cnt = __reduce_add_sync(0xffffffffu, __popc(loc));
      if (lane == 0) {
        *unsat = cnt;
        const uint64_t t = static_cast<uint64_t>(atomicAdd(&io.sched[2 + s], 1u)) + peers;
        ticket[ipar] = t < io.nshots ? static_cast<uint32_t>(t) : kNoShot;
      }
    }
    if (warp == nwarps - 1) {  // zero this segment's bits of the shot's estimate
      uint32_t* est_g = io.est + shot * P.est_w32 + vw0;
      for (uint32_t w = lane; w < vspan; w += 32u) {
        const uint32_t mask = range_mask(vw0 + w, seg.v0, v1z);
        if (mask == 0xffffffffu) {
          est_g[w] = 0u;
        } else {
          atomicAnd(&est_g[w], ~mask);
        }
      }
    }
    // q[e] = gamma[var(e)] (decoder.cpp:156-158); padded slots land in the dummy blocks
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const Msg init = prior_as_msg<A>(gam[k]);
#pragma unroll
      for (int i = 0; i < DV; ++i) *reinterpret_cast<Msg*>(msgs + eo[k][i]) = init;
    }
    if constexpr (kSoft) {  // this shot's priors of the absorbed variables: q = gamma for the whole decode
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const uint32_t aslot = (absorb >> (8 * k)) & 0xffu;
        if (cl[k] < Ms && aslot != kNoAbsorb) {
          *reinterpret_cast<Msg*>(msgs + co[k] + aslot * kMsg) = soft_next[k];
        }
      }
    }
    uint32_t eprev = 0, aprev = 0;  // decisions of this thread's variables / absorbed variables
    __syncthreads();

    uint32_t synbits = 0;
#pragma unroll
    for (int k = 0; k < CPT; ++k) synbits |= ((par[cl[k] >> 5] >> (cl[k] & 31u)) & 1u) << k;
    const uint32_t next = ticket[ipar];
    if (warp == 0 && lane < gspan && next != kNoShot) {  // prefetch the next shot's syndrome
      raw_next = io.syn[static_cast<uint64_t>(next) * P.syn_w32 + gw0 + lane];
    }
    if (next != kNoShot) fetch_soft(next);

    // ---------------- iterations ----------------
    uint32_t iter = 0;
    bool still_unsat;
    for (;;) {
      ++iter;
      uint32_t eb = 0;
      // Bitmap and counter are only WRITTEN between the two barriers of an iteration and only
      // READ (the stop test) between the second barrier and the next iteration's first one:
      // the flips of absorbed variables found in the check stage wait in `achg` until then.
      uint32_t achg = 0;
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        // (warps without a check in the last round skip it, as in decode_lean_kernel)
        if (k + 1 < CPT || (tid & ~31u) + static_cast<uint32_t>(CPT - 1) * T < Ms) {
          cn_ell<DC>(P, A{}, msgs + co[k], (synbits >> k) & 1u);
          const uint32_t aslot = (absorb >> (8 * k)) & 0xffu;
          if (aslot != kNoAbsorb) {  // posterior of the absorbed variable from the r just produced
            const unsigned char* slot = msgs + co[k] + aslot * kMsg;
            const uint32_t e = absorbed_decision(A{}, *reinterpret_cast<const Msg*>(slot),
                                                 *reinterpret_cast<const Msg*>(slot + DC * kMsg));
            achg |= (e ^ ((aprev >> k) & 1u)) << k;  // it flips the parity of its one check
          }
        }
      }
      aprev ^= achg;
      __syncthreads();
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        eb |= vn_ell<DC, DV>(P, A{}, msgs, eo[k], gam[k], (keep0 >> k) & 1u) << k;
      }
      eb &= valid;
      const uint32_t changed = eb ^ eprev;
      eprev = eb;
      if (changed | achg) {  // a hard decision flipped: toggle its checks, keep the counter exact
        int32_t delta = 0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
          if ((achg >> k) & 1u) {
            const uint32_t bit = 1u << (cl[k] & 31u);
            const uint32_t old = atomicXor(&par[cl[k] >> 5], bit);
            delta += (old & bit) ? -1 : 1;
          }
        }
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
          if ((changed >> k) & 1u) {
#pragma unroll
            for (int i = 0; i < DV; ++i) {
              if (eo[k][i] < scratch_off) {  // a real edge
                const uint32_t lm = eo[k][i] / kStride;
                const uint32_t bit = 1u << (lm & 31u);
                const uint32_t old = atomicXor(&par[lm >> 5], bit);
                delta += (old & bit) ? -1 : 1;
              }
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
    if (eprev | aprev) {
      uint32_t* est_g = io.est + shot * P.est_w32;
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        if ((eprev >> k) & 1u) {
          const uint32_t n = P.ell_vars[seg.v0 + tid + k * T];
          atomicOr(&est_g[n >> 5], 1u << (n & 31u));
        }
      }
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        if ((aprev >> k) & 1u) {
          const uint32_t n =
              P.edge_var[P.check_off[seg.c0 + cl[k]] + ((absorb >> (8 * k)) & 0xffu)];
          atomicOr(&est_g[n >> 5], 1u << (n & 31u));
        }
      }
    }
    if (tid == 0) {
      io.conv[shot * nseg + s] = still_unsat ? 0 : 1;
      io.iters[shot * nseg + s] = iter;
    }
    if constexpr (kDump) if (io.q_dump != nullptr && shot == io.dump_shot) {
      ell_dump_messages(P, seg, msgs, kStride, kMsg, DC * kMsg, 0u,
                        [&](uint32_t e, const unsigned char* q, const unsigned char* r) {
                          if constexpr (A::kInt) {
                            static_cast<int32_t*>(io.q_dump)[e] = *reinterpret_cast<const Msg*>(q);
                            static_cast<int32_t*>(io.r_dump)[e] = *reinterpret_cast<const Msg*>(r);
                          } else {
                            static_cast<float*>(io.q_dump)[e] = static_cast<float>(*reinterpret_cast<const Msg*>(q));
                            static_cast<float*>(io.r_dump)[e] = static_cast<float>(*reinterpret_cast<const Msg*>(r));
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
      // single shot: the CTA that finishes last reports its own entry-to-exit span
      if (io.kernel_ns) *io.kernel_ns = globaltimer_ns() - t_entry;
      __threadfence();
    }
  }
}

}  // namespace qb

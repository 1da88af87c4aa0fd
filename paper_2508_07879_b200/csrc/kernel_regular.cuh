// Regular-code fast path: every check has degree 6, every variable degree 3 (the
// bivariate-bicycle family).  Same two-stage flooding schedule, same arithmetic
// and therefore the same bits as the generic kernel; what changes is how few
// instructions an iteration costs:
//
//  * thread <-> node mapping is fixed for the life of the persistent kernel, so
//    each thread keeps the shared-memory offsets of its variables' edges in
//    REGISTERS; the iteration loop reads no table from global memory;
//  * messages stay in the reference's edge order (check-major, 6 per check): a
//    check reads its inputs / writes its outputs with three paired accesses
//    (64-bit for fp32), bank-conflict-free at stride 24 B;
//  * check update without a scan: magnitudes are compared as integers on the
//    raw bit patterns, min1/min2 come from a 3-pair min/max network, the edge
//    that receives min2 is "the one whose magnitude equals min1" (with a tie
//    min2 == min1, so no arg-min bookkeeping), and signs are XORs of sign bits;
//  * idle thread slots work on a dummy check / variable in a pad region instead
//    of branching, so the loop body is straight-line code;
//  * hard decisions live in a per-thread register bit-field; only variables
//    that decide 1 (rare) touch the parity bitmap, and the packed estimate is
//    materialised once per shot;
//  * FAST instantiation: uniform prior (a kernel constant, no prior registers)
//    and, for fp32, a host-side proof that no message can reach the reference's
//    1e30 clamp, which removes the clamp from the loop.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernel_generic.cuh"

namespace qb {

namespace cg = cooperative_groups;

constexpr int kDC = 6;
constexpr int kDV = 3;

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

// ---- check update, one degree-6 check whose edges start at element e0 --------
// `sflip` is 0 or the sign-bit mask when the syndrome bit is 1.

template <bool kFast>
__device__ __forceinline__ void cn6(const DecodeParams& P, const float* q, float* r, uint32_t e0,
                                    uint32_t syn_bit) {
  const uint2* q2 = reinterpret_cast<const uint2*>(q + e0);
  uint32_t u[6];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const uint2 v = q2[j];
    u[2 * j] = v.x;
    u[2 * j + 1] = v.y;
  }
  int32_t a[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) a[j] = static_cast<int32_t>(u[j] & 0x7fffffffu);
  int32_t m1, m2;
  two_smallest6(a, m1, m2);
  // float(alpha * |min|): fp64 product, one rounding (decoder.cpp:302-307)
  const uint32_t s1 =
      __float_as_uint(static_cast<float>(P.alpha * static_cast<double>(__int_as_float(m1))));
  const uint32_t s2 =
      __float_as_uint(static_cast<float>(P.alpha * static_cast<double>(__int_as_float(m2))));
  // sign of output j = sigma * prod_{i != j} sign(q_i); q never holds -0.0 (the
  // loader canonicalises priors), so the sign bit is exactly "q < 0".
  const uint32_t sx = u[0] ^ u[1] ^ u[2] ^ u[3] ^ u[4] ^ u[5] ^ (syn_bit << 31);
  uint2* r2 = reinterpret_cast<uint2*>(r + e0);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    uint2 o;
    o.x = (a[2 * j] == m1 ? s2 : s1) | ((sx ^ u[2 * j]) & 0x80000000u);
    o.y = (a[2 * j + 1] == m1 ? s2 : s1) | ((sx ^ u[2 * j + 1]) & 0x80000000u);
    r2[j] = o;
  }
}

template <bool kFast>
__device__ __forceinline__ void cn6(const DecodeParams& P, const __half* q, __half* r, uint32_t e0,
                                    uint32_t syn_bit) {
  const uint32_t* q2 = reinterpret_cast<const uint32_t*>(q + e0);
  uint32_t u[6];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const uint32_t v = q2[j];
    u[2 * j] = v & 0xffffu;
    u[2 * j + 1] = v >> 16;
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
  uint32_t* r2 = reinterpret_cast<uint32_t*>(r + e0);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const uint32_t lo = (a[2 * j] == m1 ? s2 : s1) | ((sx ^ u[2 * j]) & 0x8000u);
    const uint32_t hi = (a[2 * j + 1] == m1 ? s2 : s1) | ((sx ^ u[2 * j + 1]) & 0x8000u);
    r2[j] = lo | (hi << 16);
  }
}

template <bool kFast, class MsgI>
__device__ __forceinline__ void cn6_int(const DecodeParams& P, const MsgI* q, MsgI* r, uint32_t e0,
                                        uint32_t syn_bit) {
  using P2 = typename std::conditional<sizeof(MsgI) == 1, char2, short2>::type;
  const P2* q2 = reinterpret_cast<const P2*>(q + e0);
  int32_t v[6];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const P2 p = q2[j];
    v[2 * j] = p.x;
    v[2 * j + 1] = p.y;
  }
  int32_t a[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) a[j] = abs(v[j]);
  int32_t m1, m2;
  two_smallest6(a, m1, m2);
  const int32_t s1 = scale_q16(static_cast<uint32_t>(m1), P.alpha_fx);
  const int32_t s2 = scale_q16(static_cast<uint32_t>(m2), P.alpha_fx);
  const int32_t sx = v[0] ^ v[1] ^ v[2] ^ v[3] ^ v[4] ^ v[5] ^ static_cast<int32_t>(syn_bit << 31);
  P2* r2 = reinterpret_cast<P2*>(r + e0);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    P2 o;
    {
      const int32_t mag = a[2 * j] == m1 ? s2 : s1;
      const int32_t neg = (sx ^ v[2 * j]) >> 31;  // 0 or -1
      o.x = static_cast<decltype(o.x)>((mag ^ neg) - neg);
    }
    {
      const int32_t mag = a[2 * j + 1] == m1 ? s2 : s1;
      const int32_t neg = (sx ^ v[2 * j + 1]) >> 31;
      o.y = static_cast<decltype(o.y)>((mag ^ neg) - neg);
    }
    r2[j] = o;
  }
}
template <bool kFast>
__device__ __forceinline__ void cn6(const DecodeParams& P, const int8_t* q, int8_t* r, uint32_t e0,
                                    uint32_t syn_bit) {
  cn6_int<kFast, int8_t>(P, q, r, e0, syn_bit);
}
template <bool kFast>
__device__ __forceinline__ void cn6(const DecodeParams& P, const int16_t* q, int16_t* r,
                                    uint32_t e0, uint32_t syn_bit) {
  cn6_int<kFast, int16_t>(P, q, r, e0, syn_bit);
}

// ---- variable update, one degree-3 variable; returns 1 iff it decides 1 -------

template <bool kFast>
__device__ __forceinline__ uint32_t vn3(const DecodeParams& P, float* q, const float* r,
                                        const uint32_t (&ea)[3], float gamma) {
  const double r0 = static_cast<double>(r[ea[0]]);
  const double r1 = static_cast<double>(r[ea[1]]);
  const double r2 = static_cast<double>(r[ea[2]]);
  // fp64 accumulation in ascending edge order (decoder.cpp:319-322)
  double total = kFast ? P.gamma_d : static_cast<double>(gamma);
  total += r0;
  total += r1;
  total += r2;
  float x0 = static_cast<float>(total - r0);
  float x1 = static_cast<float>(total - r1);
  float x2 = static_cast<float>(total - r2);
  if constexpr (!kFast) {  // FAST: proven unreachable on the host (see loader)
    x0 = fminf(fmaxf(x0, -P.clamp_f), P.clamp_f);
    x1 = fminf(fmaxf(x1, -P.clamp_f), P.clamp_f);
    x2 = fminf(fmaxf(x2, -P.clamp_f), P.clamp_f);
  }
  q[ea[0]] = x0;
  q[ea[1]] = x1;
  q[ea[2]] = x2;
  // total is never -0.0 (sum of terms that are not all -0.0), so sign bit == (total < 0)
  return static_cast<uint32_t>(__double2hiint(total)) >> 31;
}

template <bool kFast>
__device__ __forceinline__ uint32_t vn3(const DecodeParams& P, __half* q, const __half* r,
                                        const uint32_t (&ea)[3], float gamma) {
  const __half r0 = r[ea[0]], r1 = r[ea[1]], r2 = r[ea[2]];
  const __half g = kFast ? __ushort_as_half(P.gamma_hb)
                         : __float2half_rn(fminf(fmaxf(gamma, -kHalfClamp), kHalfClamp));
  const __half total = __hadd(__hadd(__hadd(g, r0), r1), r2);
  q[ea[0]] = h_clamp(__hsub(total, r0));
  q[ea[1]] = h_clamp(__hsub(total, r1));
  q[ea[2]] = h_clamp(__hsub(total, r2));
  return h_neg(total) ? 1u : 0u;
}

template <bool kFast, class MsgI>
__device__ __forceinline__ uint32_t vn3_int(const DecodeParams& P, MsgI* q, const MsgI* r,
                                            const uint32_t (&ea)[3], int32_t gamma) {
  const int32_t r0 = r[ea[0]], r1 = r[ea[1]], r2 = r[ea[2]];
  const int32_t total = (kFast ? P.gamma_i : gamma) + r0 + r1 + r2;
  q[ea[0]] = static_cast<MsgI>(max(-P.kmax, min(P.kmax, total - r0)));
  q[ea[1]] = static_cast<MsgI>(max(-P.kmax, min(P.kmax, total - r1)));
  q[ea[2]] = static_cast<MsgI>(max(-P.kmax, min(P.kmax, total - r2)));
  return static_cast<uint32_t>(total) >> 31;
}
template <bool kFast>
__device__ __forceinline__ uint32_t vn3(const DecodeParams& P, int8_t* q, const int8_t* r,
                                        const uint32_t (&ea)[3], int32_t gamma) {
  return vn3_int<kFast, int8_t>(P, q, r, ea, gamma);
}
template <bool kFast>
__device__ __forceinline__ uint32_t vn3(const DecodeParams& P, int16_t* q, const int16_t* r,
                                        const uint32_t (&ea)[3], int32_t gamma) {
  return vn3_int<kFast, int16_t>(P, q, r, ea, gamma);
}

// ---- per-thread register-resident tables of one segment ----------------------

template <class A, int CPT, int VPT, bool kFast>
struct RegTables {
  uint32_t ea[VPT][kDV];   // message-array element index of each variable's edges
  uint32_t ce[CPT];        // first element index of each check's edges
  uint32_t cbit[CPT];      // global check index (syndrome bit position)
  typename A::Gam gamma[kFast ? 1 : VPT];
  uint32_t valid;          // bit k: variable slot k is a real variable
  uint32_t mbase;          // global check index of message element 0
};

template <class A, int CPT, int VPT, bool kFast>
__device__ __forceinline__ void load_tables(const DecodeParams& P, const SegmentDev& seg,
                                            uint32_t t, uint32_t T,
                                            RegTables<A, CPT, VPT, kFast>& tab,
                                            uint32_t ebase = 0, uint32_t pad0 = 0xffffffffu) {
  // Message element i of the shared arrays holds global edge ebase + i; the dummy
  // check / variable live at elements pad0 .. pad0+5 (default: right after edge E-1).
  using Gam = typename A::Gam;
  const Gam* __restrict__ gamma = static_cast<const Gam*>(P.gamma);
  if (pad0 == 0xffffffffu) pad0 = P.E;
  tab.valid = 0;
  tab.mbase = ebase / kDC;
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const uint32_t n = seg.v0 + t + k * T;
    const bool ok = n < seg.v1;
    tab.valid |= (ok ? 1u : 0u) << k;
#pragma unroll
    for (int i = 0; i < kDV; ++i) {
      tab.ea[k][i] = ok ? P.var_edges[n * kDV + i] - ebase : pad0 + i;  // dummy: pad slots 0..2
    }
    if constexpr (!kFast) tab.gamma[k] = ok ? gamma[n] : static_cast<Gam>(1);
  }
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const uint32_t m = seg.c0 + t + k * T;
    const bool ok = m < seg.c1;
    tab.cbit[k] = ok ? m : P.M;                 // dummy check: syndrome bit M is always 0
    tab.ce[k] = ok ? m * kDC - ebase : pad0;    // its edges are the pad slots
  }
}

// One segment of one shot on one warp group of T threads (T * CPT >= checks,
// T * VPT >= variables of the segment).
template <class A, int CPT, int VPT, bool kFast>
__device__ __forceinline__ void decode_segment_regular(
    const DecodeParams& P, const GenericSmem<A>& S, const SegmentDev& seg, uint32_t s, uint32_t t,
    uint32_t T, uint32_t bar_id, const RegTables<A, CPT, VPT, kFast>& tab) {
  using Msg = typename A::Msg;
  using Gam = typename A::Gam;
  const uint32_t lane = t & 31u;
  const uint32_t w0 = seg.c0 >> 5, w1 = (seg.c1 - 1) >> 5;
  Msg* q = S.q;
  Msg* r = S.r;

  // q[e] = gamma[var(e)] (decoder.cpp:156-158), written from the variable side
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    Gam g;
    if constexpr (kFast) {
      if constexpr (A::kInt) g = P.gamma_i; else g = P.gamma_f;
    } else {
      g = tab.gamma[k];
    }
    const Msg init = prior_as_msg<A>(g);
#pragma unroll
    for (int i = 0; i < kDV; ++i) q[tab.ea[k][i]] = init;
  }
  group_barrier(bar_id, T);

  uint32_t iter = 0;
  uint32_t ebits = 0;
  bool converged = false;
  uint32_t* par = S.par0;
  for (;;) {
    ++iter;
    par = (iter & 1u) ? S.par1 : S.par0;
    uint32_t* par_next = (iter & 1u) ? S.par0 : S.par1;

#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const uint32_t m = tab.cbit[k];
      const uint32_t syn_bit = (S.syn[m >> 5] >> (m & 31u)) & 1u;
      cn6<kFast>(P, q, r, tab.ce[k], syn_bit);
    }
    group_barrier(bar_id, T);

    ebits = 0;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      Gam g{};
      if constexpr (!kFast) g = tab.gamma[k];
      ebits |= vn3<kFast>(P, q, r, tab.ea[k], g) << k;
    }
    ebits &= tab.valid;
    if (ebits) {  // rare: this thread owns a variable that currently decides 1
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        if ((ebits >> k) & 1u) {
#pragma unroll
          for (int i = 0; i < kDV; ++i) {
            const uint32_t m = tab.ea[k][i] / kDC + tab.mbase;
            atomicXor(&par[m >> 5], 1u << (m & 31u));
          }
        }
      }
    }
    for (uint32_t w = w0 + t; w <= w1; w += T) {
      const uint32_t mask = range_mask(w, seg.c0, seg.c1);
      if (mask == 0xffffffffu) {
        par_next[w] = S.syn[w];
      } else {
        atomicAnd(&par_next[w], ~mask);
        atomicOr(&par_next[w], S.syn[w] & mask);
      }
    }
    group_barrier(bar_id, T);

    uint32_t acc = 0;
    for (uint32_t w = w0 + lane; w <= w1; w += 32u) acc |= par[w] & range_mask(w, seg.c0, seg.c1);
    const bool unsat = __any_sync(0xffffffffu, acc != 0u);
    if (P.early && !unsat) {
      converged = true;
      break;
    }
    if (iter >= P.max_iter) {
      converged = !unsat;
      break;
    }
  }

  // materialise the hard decisions and the residual once per shot
  if (ebits) {
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      if ((ebits >> k) & 1u) {
        const uint32_t n = seg.v0 + t + k * T;
        atomicOr(&S.ehat[n >> 5], 1u << (n & 31u));
      }
    }
  }
  for (uint32_t w = w0 + t; w <= w1; w += T) {
    const uint32_t bits = par[w] & range_mask(w, seg.c0, seg.c1);
    if (bits) atomicOr(&S.res[w], bits);
  }
  if (t == 0) {
    S.segres[2 * s] = converged ? 1u : 0u;
    S.segres[2 * s + 1] = iter;
  }
}

// ---- shot prologue / epilogue shared by the single-CTA and cluster kernels ---

template <class A>
__device__ __forceinline__ void init_pads(const DecodeParams& P, const GenericSmem<A>& S,
                                          uint32_t tid, uint32_t pad0) {
  // the dummy check's message slots and the spare syndrome words, once per kernel
  if (tid < kPadEdges) {
    S.q[pad0 + tid] = static_cast<typename A::Msg>(0);
    S.r[pad0 + tid] = static_cast<typename A::Msg>(0);
  }
  // every syndrome word starts at 0 (the item kernel only ever writes its own
  // segment's words; the dummy check reads bit M)
  for (uint32_t w = tid; w < P.syn_w32 + 2; w += blockDim.x) S.syn[w] = 0;
}

template <class A>
__device__ __forceinline__ void shot_prologue(const DecodeParams& P, const GenericSmem<A>& S,
                                              const uint32_t* syn_g, uint32_t tid, uint32_t nthr) {
  const uint32_t last_bits = P.M & 31u;
  for (uint32_t w = tid; w < P.syn_w32; w += nthr) {
    uint32_t v = syn_g[w];
    const uint32_t first = w * 32u;
    if (first >= P.M) {
      v = 0;
    } else if (first + 32u > P.M) {
      v &= (1u << last_bits) - 1u;
    }
    S.syn[w] = v;
    S.par0[w] = v;
    S.par1[w] = v;
    S.res[w] = 0;
  }
  for (uint32_t w = tid; w < P.est_w32; w += nthr) S.ehat[w] = 0;
}

template <class A>
__device__ __forceinline__ void dump_messages(const DecodeParams& P, const GenericSmem<A>& S,
                                              const ShotIO& io, uint32_t e_begin, uint32_t e_end,
                                              uint32_t tid, uint32_t nthr) {
  for (uint32_t e = e_begin + tid; e < e_end; e += nthr) {
    if constexpr (A::kInt) {
      static_cast<int32_t*>(io.q_dump)[e] = S.q[e];
      static_cast<int32_t*>(io.r_dump)[e] = S.r[e];
    } else {
      static_cast<float*>(io.q_dump)[e] = static_cast<float>(S.q[e]);
      static_cast<float*>(io.r_dump)[e] = static_cast<float>(S.r[e]);
    }
  }
}

template <class A>
__device__ __forceinline__ void shot_epilogue(const DecodeParams& P, const GenericSmem<A>& S,
                                              const ShotIO& io, uint64_t shot, uint32_t tid,
                                              uint32_t nthr) {
  uint32_t* est_g = io.est + shot * P.est_w32;
  for (uint32_t w = tid; w < P.est_w32; w += nthr) est_g[w] = S.ehat[w];
  if (io.resid) {
    uint32_t* res_g = io.resid + shot * P.syn_w32;
    for (uint32_t w = tid; w < P.syn_w32; w += nthr) res_g[w] = S.res[w];
  }
  if (tid < P.nseg) {
    io.conv[shot * P.nseg + tid] = static_cast<uint8_t>(S.segres[2 * tid]);
    io.iters[shot * P.nseg + tid] = S.segres[2 * tid + 1];
  }
}

__device__ __forceinline__ void signal_completion(const ShotIO& io, uint64_t t_begin, uint32_t tid) {
  __threadfence_system();
  __syncthreads();
  if (tid == 0) {
    *io.kernel_ns = globaltimer_ns() - t_begin;
    __threadfence_system();
    *io.flag = io.seq;
  }
}

__device__ __forceinline__ void rewind_scheduler(const ShotIO& io, uint32_t tid) {
  if (tid == 0) {
    __threadfence();
    const unsigned int done = atomicAdd(&io.sched[1], 1u);
    if (done == gridDim.x - 1) {
      io.sched[0] = 0;
      io.sched[1] = 0;
      __threadfence();
    }
  }
}

// Persistent kernel: one CTA per shot at a time, one warp group per segment.
template <class A, int CPT, int VPT, bool kFast, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB)
decode_regular_kernel(const __grid_constant__ DecodeParams P, const __grid_constant__ ShotIO io) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const GenericSmem<A> S = carve_generic<A>(smem_raw, P);
  const uint32_t tid = threadIdx.x, nthr = blockDim.x;
  const uint64_t t_begin = io.kernel_ns ? globaltimer_ns() : 0;
  const uint32_t group = tid / P.group_threads;  // == segment (ngroups == nseg)
  const uint32_t t = tid - group * P.group_threads;
  const SegmentDev seg = P.segs[group];
  RegTables<A, CPT, VPT, kFast> tab;
  load_tables<A, CPT, VPT, kFast>(P, seg, t, P.group_threads, tab);
  init_pads<A>(P, S, tid, P.E);

  for (uint64_t shot = blockIdx.x; shot < io.nshots;) {
    shot_prologue<A>(P, S, io.syn + shot * P.syn_w32, tid, nthr);
    __syncthreads();
    decode_segment_regular<A, CPT, VPT, kFast>(P, S, seg, group, t, P.group_threads, 1u + group,
                                               tab);
    __syncthreads();
    shot_epilogue<A>(P, S, io, shot, tid, nthr);
    if (io.q_dump) dump_messages<A>(P, S, io, 0, P.E, tid, nthr);
    if (tid == 0) {
      const uint64_t nxt = static_cast<uint64_t>(atomicAdd(&io.sched[0], 1u)) + gridDim.x;
      S.ticket[0] = static_cast<uint32_t>(nxt);
      S.ticket[1] = static_cast<uint32_t>(nxt >> 32);
    }
    __syncthreads();
    shot = static_cast<uint64_t>(S.ticket[0]) | (static_cast<uint64_t>(S.ticket[1]) << 32);
  }
  if (io.flag) signal_completion(io, t_begin, tid);
  rewind_scheduler(io, tid);
}

// Latency kernel for ONE shot on a thread-block cluster: CTA rank s of the
// cluster decodes segment s on its own SM (segments are independent graphs, so
// the iteration loop needs no cross-CTA traffic at all); when a segment is done
// its CTA ORs the packed estimate / residual bits and its (converged,
// iterations) pair into rank 0's shared memory over DSMEM, and after one
// cluster barrier rank 0 writes the merged result and raises the completion flag.
template <class A, int CPT, int VPT, bool kFast>
__global__ void __launch_bounds__(1024, 1)
decode_regular_cluster_kernel(const __grid_constant__ DecodeParams P,
                              const __grid_constant__ ShotIO io) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  const GenericSmem<A> S = carve_generic<A>(smem_raw, P);
  const uint32_t tid = threadIdx.x, nthr = blockDim.x;
  const uint64_t t_begin = io.kernel_ns ? globaltimer_ns() : 0;
  const uint32_t s = cluster.block_rank();  // == segment
  const SegmentDev seg = P.segs[s];
  RegTables<A, CPT, VPT, kFast> tab;
  load_tables<A, CPT, VPT, kFast>(P, seg, tid, nthr, tab);
  init_pads<A>(P, S, tid, P.E);

  shot_prologue<A>(P, S, io.syn, tid, nthr);
  __syncthreads();
  decode_segment_regular<A, CPT, VPT, kFast>(P, S, seg, s, tid, nthr, 1u, tab);
  __syncthreads();
  if (io.q_dump) dump_messages<A>(P, S, io, seg.e0, seg.e1, tid, nthr);
  cluster.sync();  // rank 0 has finished its own segment: its buffers are final
  if (s != 0) {
    uint32_t* ehat0 = cluster.map_shared_rank(S.ehat, 0);
    uint32_t* res0 = cluster.map_shared_rank(S.res, 0);
    uint32_t* segres0 = cluster.map_shared_rank(S.segres, 0);
    for (uint32_t w = tid; w < P.est_w32; w += nthr) {
      if (S.ehat[w]) atomicOr(&ehat0[w], S.ehat[w]);
    }
    for (uint32_t w = tid; w < P.syn_w32; w += nthr) {
      if (S.res[w]) atomicOr(&res0[w], S.res[w]);
    }
    if (tid == 0) {
      segres0[2 * s] = S.segres[2 * s];
      segres0[2 * s + 1] = S.segres[2 * s + 1];
    }
  }
  cluster.sync();
  if (s == 0) {
    shot_epilogue<A>(P, S, io, 0, tid, nthr);
    if (io.flag) signal_completion(io, t_begin, tid);
  }
}

}  // namespace qb

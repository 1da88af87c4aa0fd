// Generic (CSR) persistent decode kernel: any block-diagonal Tanner graph whose
// messages fit one CTA's shared memory, any degree distribution, all four
// arithmetic modes.  One CTA decodes one shot at a time; its warps are split
// into one group per segment, each group iterating independently behind its
// own named barrier, so a converged segment is frozen exactly as the reference
// freezes it (proj/src/decoder.cpp:162-187) while the other keeps going.
//
// Per iteration and segment (2 group barriers):
//   CN stage  thread per check: two-minimum scan of q, write r   (decoder.cpp:245-311)
//   VN stage  thread per variable: total = gamma + sum r in ascending edge
//             order, hard decision, write q                      (decoder.cpp:313-335)
//             + every variable deciding 1 toggles its checks' bits in a
//             per-iteration parity bitmap that was preset to the syndrome, so
//             the bitmap IS the residual s ^ H*e_hat                 (decoder.cpp:337-350)
//   stop test every warp ORs the segment's parity words and votes.
//
// All bit vectors live in shared memory in the reference's packed layout
// (global bit index, 32-bit halves of the uint64 words), so the estimate and
// the residual leave the kernel as straight word copies.
#pragma once

#include "common.cuh"

namespace qb {

template <class A>
struct GenericSmem {
  typename A::Msg* q;
  typename A::Msg* r;
  uint32_t* syn;    // [syn_w32] packed syndrome of the current shot
  uint32_t* par0;   // [syn_w32] parity bitmap, even iterations
  uint32_t* par1;   // [syn_w32] parity bitmap, odd iterations
  uint32_t* res;    // [syn_w32] final residual (all segments merged)
  uint32_t* ehat;   // [est_w32] packed hard decisions
  uint32_t* segres; // [2 * nseg] converged, iterations
  uint32_t* ticket; // [2] next shot (lo, hi)
};

__host__ __device__ inline size_t generic_smem_bytes(uint32_t E, uint32_t syn_w32,
                                                     uint32_t est_w32, uint32_t nseg,
                                                     size_t msg_bytes) {
  // kPadEdges extra message slots hold the dummy check/variable that idle thread
  // slots of the regular kernel work on; 2 spare syndrome words keep bit M addressable.
  size_t msg = (static_cast<size_t>(E + kPadEdges) * msg_bytes + 15) & ~static_cast<size_t>(15);
  return 2 * msg + 4 * (4 * static_cast<size_t>(syn_w32) + 2 + est_w32 + 2 * nseg + 4);
}

template <class A>
__device__ __forceinline__ GenericSmem<A> carve_generic(unsigned char* base,
                                                        const DecodeParams& P) {
  GenericSmem<A> s;
  const size_t msg =
      (static_cast<size_t>(P.E + kPadEdges) * sizeof(typename A::Msg) + 15) & ~size_t(15);
  s.q = reinterpret_cast<typename A::Msg*>(base);
  s.r = reinterpret_cast<typename A::Msg*>(base + msg);
  uint32_t* w = reinterpret_cast<uint32_t*>(base + 2 * msg);
  s.syn = w;  // [syn_w32 + 2]
  s.par0 = w + P.syn_w32 + 2;
  s.par1 = s.par0 + P.syn_w32;
  s.res = s.par1 + P.syn_w32;
  s.ehat = s.res + P.syn_w32;
  s.segres = s.ehat + P.est_w32;
  s.ticket = s.segres + 2 * P.nseg;
  return s;
}

// ---- check-node update of one check over CSR edges [b, e1) ---------------

__device__ __forceinline__ void cn_update(const DecodeParams& P, const float* q, float* r,
                                          uint32_t b, uint32_t e1, bool sneg) {
  if (e1 - b == 1) {
    r[b] = sneg ? -P.deg1_f : P.deg1_f;
    return;
  }
  float m1 = __int_as_float(0x7f800000), m2 = m1;
  uint32_t arg = b;
  uint32_t neg = 0;
  for (uint32_t e = b; e < e1; ++e) {
    const float v = q[e];
    neg += v < 0.0f;
    const float a = fabsf(v);
    if (a < m1) {
      m2 = m1;
      m1 = a;
      arg = e;
    } else if (a < m2) {
      m2 = a;
    }
  }
  // fp64 product, one rounding to fp32: float(alpha * |min|) (decoder.cpp:302-307)
  const float r1 = static_cast<float>(P.alpha * static_cast<double>(m1));
  const float r2 = static_cast<float>(P.alpha * static_cast<double>(m2));
  for (uint32_t e = b; e < e1; ++e) {
    const uint32_t self = q[e] < 0.0f;
    const bool flip = ((neg - self) & 1u) != 0;
    const float mag = e == arg ? r2 : r1;
    r[e] = (sneg != flip) ? -mag : mag;
  }
}

__device__ __forceinline__ void cn_update(const DecodeParams& P, const __half* q, __half* r,
                                          uint32_t b, uint32_t e1, bool sneg) {
  if (e1 - b == 1) {
    r[b] = __ushort_as_half(static_cast<unsigned short>(P.deg1_h ^ (sneg ? 0x8000u : 0u)));
    return;
  }
  uint32_t m1 = 0x7c00u, m2 = 0x7c00u;  // +inf as an fp16 magnitude key
  uint32_t arg = b;
  uint32_t neg = 0;
  for (uint32_t e = b; e < e1; ++e) {
    const uint32_t u = __half_as_ushort(q[e]);
    neg += u >> 15;
    const uint32_t a = u & 0x7fffu;  // finite fp16 magnitudes order like their bit patterns
    if (a < m1) {
      m2 = m1;
      m1 = a;
      arg = e;
    } else if (a < m2) {
      m2 = a;
    }
  }
  const __half alpha = __ushort_as_half(P.alpha_h);
  const uint32_t r1 = __half_as_ushort(__hmul(alpha, __ushort_as_half(static_cast<unsigned short>(m1))));
  const uint32_t r2 = __half_as_ushort(__hmul(alpha, __ushort_as_half(static_cast<unsigned short>(m2))));
  for (uint32_t e = b; e < e1; ++e) {
    const uint32_t self = __half_as_ushort(q[e]) >> 15;
    const bool flip = ((neg - self) & 1u) != 0;
    const uint32_t mag = e == arg ? r2 : r1;
    r[e] = __ushort_as_half(static_cast<unsigned short>(mag | ((sneg != flip) ? 0x8000u : 0u)));
  }
}

template <class MsgI>
__device__ __forceinline__ void cn_update_int(const DecodeParams& P, const MsgI* q, MsgI* r,
                                              uint32_t b, uint32_t e1, bool sneg) {
  if (e1 - b == 1) {
    r[b] = static_cast<MsgI>(sneg ? -P.deg1_i : P.deg1_i);
    return;
  }
  int32_t m1 = 0x7fffffff, m2 = m1;
  uint32_t arg = b;
  uint32_t neg = 0;
  for (uint32_t e = b; e < e1; ++e) {
    const int32_t v = q[e];
    neg += v < 0;
    const int32_t a = v < 0 ? -v : v;
    if (a < m1) {
      m2 = m1;
      m1 = a;
      arg = e;
    } else if (a < m2) {
      m2 = a;
    }
  }
  const int32_t r1 = scale_q16(static_cast<uint32_t>(m1), P.alpha_fx);
  const int32_t r2 = scale_q16(static_cast<uint32_t>(m2), P.alpha_fx);
  for (uint32_t e = b; e < e1; ++e) {
    const uint32_t self = q[e] < 0;
    const bool flip = ((neg - self) & 1u) != 0;
    const int32_t mag = e == arg ? r2 : r1;
    r[e] = static_cast<MsgI>((sneg != flip) ? -mag : mag);
  }
}
__device__ __forceinline__ void cn_update(const DecodeParams& P, const int8_t* q, int8_t* r,
                                          uint32_t b, uint32_t e1, bool sneg) {
  cn_update_int<int8_t>(P, q, r, b, e1, sneg);
}
__device__ __forceinline__ void cn_update(const DecodeParams& P, const int16_t* q, int16_t* r,
                                          uint32_t b, uint32_t e1, bool sneg) {
  cn_update_int<int16_t>(P, q, r, b, e1, sneg);
}

// ---- variable-node update of one variable; returns the hard decision -------

__device__ __forceinline__ bool vn_update(const DecodeParams& P, float* q, const float* r,
                                          const uint32_t* ve, uint32_t b, uint32_t e1,
                                          float gamma) {
  // fp64 accumulation in ascending edge order (decoder.cpp:319-322)
  double total = static_cast<double>(gamma);
  for (uint32_t i = b; i < e1; ++i) total += static_cast<double>(r[ve[i]]);
  if (e1 - b == 1) {
    q[ve[b]] = gamma;  // decoder.cpp:324-329
  } else {
    for (uint32_t i = b; i < e1; ++i) {
      const uint32_t e = ve[i];
      // clamp to +-1e30 then round once; clamping the rounded value with
      // float(1e30) is equivalent because rounding is monotonic.
      float x = static_cast<float>(total - static_cast<double>(r[e]));
      x = fminf(fmaxf(x, -P.clamp_f), P.clamp_f);
      q[e] = x;
    }
  }
  return total < 0.0;
}

__device__ __forceinline__ bool vn_update(const DecodeParams&, __half* q, const __half* r,
                                          const uint32_t* ve, uint32_t b, uint32_t e1,
                                          float gamma) {
  const __half g = __float2half_rn(fminf(fmaxf(gamma, -kHalfClamp), kHalfClamp));
  __half total = g;
  for (uint32_t i = b; i < e1; ++i) total = __hadd(total, r[ve[i]]);
  if (e1 - b == 1) {
    q[ve[b]] = g;
  } else {
    for (uint32_t i = b; i < e1; ++i) {
      const uint32_t e = ve[i];
      q[e] = h_clamp(__hsub(total, r[e]));
    }
  }
  return h_neg(total);
}

template <class MsgI>
__device__ __forceinline__ bool vn_update_int(const DecodeParams& P, MsgI* q, const MsgI* r,
                                              const uint32_t* ve, uint32_t b, uint32_t e1,
                                              int32_t gamma) {
  int32_t total = gamma;
  for (uint32_t i = b; i < e1; ++i) total += static_cast<int32_t>(r[ve[i]]);
  if (e1 - b == 1) {
    q[ve[b]] = static_cast<MsgI>(gamma);
  } else {
    for (uint32_t i = b; i < e1; ++i) {
      const uint32_t e = ve[i];
      const int32_t x = total - static_cast<int32_t>(r[e]);
      q[e] = static_cast<MsgI>(max(-P.kmax, min(P.kmax, x)));
    }
  }
  return total < 0;
}
__device__ __forceinline__ bool vn_update(const DecodeParams& P, int8_t* q, const int8_t* r,
                                          const uint32_t* ve, uint32_t b, uint32_t e1,
                                          int32_t gamma) {
  return vn_update_int<int8_t>(P, q, r, ve, b, e1, gamma);
}
__device__ __forceinline__ bool vn_update(const DecodeParams& P, int16_t* q, const int16_t* r,
                                          const uint32_t* ve, uint32_t b, uint32_t e1,
                                          int32_t gamma) {
  return vn_update_int<int16_t>(P, q, r, ve, b, e1, gamma);
}

template <class A>
__device__ __forceinline__ typename A::Msg prior_as_msg(typename A::Gam g) {
  return static_cast<typename A::Msg>(g);
}
template <>
__device__ __forceinline__ __half prior_as_msg<ArithF16>(float g) {
  return __float2half_rn(fminf(fmaxf(g, -kHalfClamp), kHalfClamp));
}

// ---- one segment of one shot, executed by one warp group -------------------

template <class A>
__device__ void decode_segment_generic(const DecodeParams& P, const GenericSmem<A>& S,
                                       uint32_t s, uint32_t t, uint32_t T, uint32_t bar_id) {
  using Msg = typename A::Msg;
  using Gam = typename A::Gam;
  const SegmentDev seg = P.segs[s];
  const Gam* __restrict__ gamma = static_cast<const Gam*>(P.gamma);
  const uint32_t lane = t & 31u;
  const uint32_t w0 = seg.c0 >> 5, w1 = (seg.c1 - 1) >> 5;  // parity words of this segment
  Msg* q = S.q;
  Msg* r = S.r;

  // q[e] = gamma[var(e)]  (decoder.cpp:156-158)
  for (uint32_t e = seg.e0 + t; e < seg.e1; e += T) {
    q[e] = prior_as_msg<A>(gamma[P.edge_var[e]]);
  }
  group_barrier(bar_id, T);

  uint32_t iter = 0;
  bool converged = false;
  uint32_t* par = S.par0;
  for (;;) {
    ++iter;
    par = (iter & 1u) ? S.par1 : S.par0;
    uint32_t* par_next = (iter & 1u) ? S.par0 : S.par1;

    // ---- CN stage
    for (uint32_t m = seg.c0 + t; m < seg.c1; m += T) {
      const bool sneg = (S.syn[m >> 5] >> (m & 31u)) & 1u;
      cn_update(P, q, r, P.check_off[m], P.check_off[m + 1], sneg);
    }
    group_barrier(bar_id, T);

    // ---- VN stage (warp-aligned on the global variable index so that a
    //      ballot is one packed estimate word)
    for (uint32_t nb = (seg.v0 & ~31u) + (t & ~31u); nb < seg.v1; nb += T) {
      const uint32_t n = nb + lane;
      const bool active = n >= seg.v0 && n < seg.v1;
      bool bit = false;
      if (active) {
        const uint32_t b = P.var_off[n], e1 = P.var_off[n + 1];
        bit = vn_update(P, q, r, P.var_edges, b, e1, gamma[n]);
        if (bit) {
          for (uint32_t i = b; i < e1; ++i) {
            const uint32_t m = P.edge_check[P.var_edges[i]];
            atomicXor(&par[m >> 5], 1u << (m & 31u));
          }
        }
      }
      const uint32_t word = __ballot_sync(0xffffffffu, bit);
      if (lane == 0) {
        const uint32_t w = nb >> 5;
        const uint32_t mask = range_mask(w, seg.v0, seg.v1);
        if (mask == 0xffffffffu) {
          S.ehat[w] = word;
        } else {  // word shared with a neighbouring segment: touch own bits only
          atomicAnd(&S.ehat[w], ~mask);
          atomicOr(&S.ehat[w], word & mask);
        }
      }
    }
    // preset the other bitmap to the syndrome for the next iteration
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

    // ---- syndrome-match test (decoder.cpp:169-180): residual bitmap all zero?
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

  // residual of this segment into the merged result bitmap
  for (uint32_t w = w0 + t; w <= w1; w += T) {
    const uint32_t bits = par[w] & range_mask(w, seg.c0, seg.c1);
    if (bits) atomicOr(&S.res[w], bits);
  }
  if (t == 0) {
    S.segres[2 * s] = converged ? 1u : 0u;
    S.segres[2 * s + 1] = iter;
  }
}

template <class A>
__global__ void __launch_bounds__(1024, 1)
decode_generic_kernel(const __grid_constant__ DecodeParams P, const __grid_constant__ ShotIO io) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const GenericSmem<A> S = carve_generic<A>(smem_raw, P);
  const uint32_t tid = threadIdx.x, nthr = blockDim.x;
  const uint64_t t_begin = io.kernel_ns ? globaltimer_ns() : 0;

  const uint32_t group = tid / P.group_threads;
  const uint32_t t = tid - group * P.group_threads;
  const uint32_t last_bits = P.M & 31u;

  for (uint64_t shot = blockIdx.x; shot < io.nshots;) {
    // ---- prologue: stage the packed syndrome, preset parity bitmaps
    const uint32_t* syn_g = io.syn + shot * P.syn_w32;
    for (uint32_t w = tid; w < P.syn_w32; w += nthr) {
      uint32_t v = syn_g[w];
      const uint32_t first = w * 32u;
      if (first >= P.M) {
        v = 0;  // padding half-word of the last uint64
      } else if (first + 32u > P.M) {
        v &= (1u << last_bits) - 1u;
      }
      S.syn[w] = v;
      S.par0[w] = v;
      S.par1[w] = v;
      S.res[w] = 0;
    }
    for (uint32_t w = tid; w < P.est_w32; w += nthr) S.ehat[w] = 0;
    __syncthreads();

    // ---- decode: one warp group per segment
    if (group < P.ngroups) {
      for (uint32_t s = group; s < P.nseg; s += P.ngroups) {
        decode_segment_generic<A>(P, S, s, t, P.group_threads, 1u + group);
      }
    }
    __syncthreads();

    // ---- epilogue: results are already in the packed output layout
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
    if (io.q_dump) {
      if constexpr (A::kInt) {
        for (uint32_t e = tid; e < P.E; e += nthr) {
          static_cast<int32_t*>(io.q_dump)[e] = S.q[e];
          static_cast<int32_t*>(io.r_dump)[e] = S.r[e];
        }
      } else {
        for (uint32_t e = tid; e < P.E; e += nthr) {
          static_cast<float*>(io.q_dump)[e] = static_cast<float>(S.q[e]);
          static_cast<float*>(io.r_dump)[e] = static_cast<float>(S.r[e]);
        }
      }
    }

    // ---- next shot: dynamic ticket (iteration counts vary from 1 to max)
    if (tid == 0) {
      const uint64_t nxt = static_cast<uint64_t>(atomicAdd(&io.sched[0], 1u)) + gridDim.x;
      S.ticket[0] = static_cast<uint32_t>(nxt);
      S.ticket[1] = static_cast<uint32_t>(nxt >> 32);
    }
    __syncthreads();
    shot = static_cast<uint64_t>(S.ticket[0]) | (static_cast<uint64_t>(S.ticket[1]) << 32);
  }

  // ---- completion
  if (io.flag) {
    __threadfence_system();
    __syncthreads();
    if (tid == 0) {
      *io.kernel_ns = globaltimer_ns() - t_begin;
      __threadfence_system();
      *io.flag = io.seq;
    }
  }
  // the last CTA out rewinds the scheduler for the next launch
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

}  // namespace qb

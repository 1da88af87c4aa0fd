// Degree-padded throughput kernel with TWO shots per thread: the irregular-graph
// kernel (kernel_ell.cuh: sentinel-padded check blocks, zero-block variable
// slots, degree-1 variables absorbed by their checks) on the packed fp16
// instructions of kernel_lean_h2.cuh.  Every message word holds the values of
// shots 2k (low half) and 2k+1 (high half); one HADD2 / HFMA2 / HMNMX2 / HSET2
// advances both shots and the offset tables in registers are shared by the pair.
//
//   kI8 = false  half mode (fp16 storage and arithmetic, no reference counterpart)
//   kI8 = true   the reference's INT8 mode, bit-exact: int8 quantities are exact fp16
//                integers, saturation at +-127 by HMNMX2, Q16 scaling as one HFMA2 with
//                the loader-verified constant (see kernel_lean_h2.cuh)
//
// This is the kernel behind BASELINE config 5 (phenomenological graphs [H | I],
// int8-quantised messages).  Lane by lane the operations are those of the scalar
// degree-padded kernel, so results are identical to it and, in int8 mode, to the
// reference.  The two shots of a pair stop independently (a finished lane is
// frozen: its bitmap, counter and decisions are no longer touched).
#pragma once

#include "common.cuh"
#include "kernel_ell.cuh"
#include "kernel_lean_h2.cuh"

namespace qb {

__host__ __device__ inline size_t ell_h2_smem_bytes(uint32_t seg_mmax, uint32_t dc, uint32_t threads) {
  return ell_msg_region_bytes(seg_mmax, ell_stride_bytes(4u, dc), threads, dc) +
         4 * (8 * static_cast<size_t>(ell_pw(seg_mmax)) + 16);
}

// check update over one padded block of half2 slots: per-edge minimum of the OTHER
// magnitudes from prefix / suffix minima, scale and sign by multiplication (see cn6_h2)
template <int DC, bool kI8>
__device__ __forceinline__ void cn_ell_h2(const DecodeParams& P, unsigned char* blk, uint32_t syn_pair) {
  static_assert(DC >= 3, "prefix / suffix minima");
  const uint32_t* qp = reinterpret_cast<const uint32_t*>(blk);
  uint32_t u[DC];
  __half2 a[DC];
#pragma unroll
  for (int j = 0; j < DC; ++j) {
    u[j] = qp[j];
    a[j] = __habs2(u2h2(u[j]));  // folds into the consumers as |x|
  }
  __half2 pre[DC], suf[DC];  // pre[j] = min(a[0..j]), suf[j] = min(a[j..DC-1])
  pre[0] = a[0];
#pragma unroll
  for (int j = 1; j < DC - 1; ++j) pre[j] = __hmin2(pre[j - 1], a[j]);
  suf[DC - 1] = a[DC - 1];
#pragma unroll
  for (int j = DC - 2; j > 0; --j) suf[j] = __hmin2(suf[j + 1], a[j]);
  uint32_t sx = syn_pair;
#pragma unroll
  for (int j = 0; j < DC; ++j) sx ^= u[j];
  sx &= 0x80008000u;
  uint32_t* rp = reinterpret_cast<uint32_t*>(blk + DC * 4);
  const __half2 c2 = __half2half2(__ushort_as_half(P.alpha_h));
  const __half2 magic = __half2half2(__ushort_as_half(0x6600));  // 1536
  const uint32_t sgn = sx ^ (kI8 ? 0x3c003c00u : static_cast<uint32_t>(P.alpha_h) * 0x00010001u);
#pragma unroll
  for (int j = 0; j < DC; ++j) {
    const __half2 e = j == 0 ? suf[1] : j == DC - 1 ? pre[DC - 2] : __hmin2(pre[j - 1], suf[j + 1]);
    const __half2 f = u2h2(sgn ^ (u[j] & 0x80008000u));  // +-1 (int8) or +-alpha (half)
    if constexpr (kI8) {
      rp[j] = h22u(__hmul2(__hsub2(__hfma2(e, c2, magic), magic), f));  // exact Q16 scaling, sign
    } else {
      rp[j] = h22u(__hmul2(e, f));
    }
  }
}

// variable update over DV padded slots; returns the sign bits of the two posteriors
template <int DC, int DV, bool kI8>
__device__ __forceinline__ uint32_t vn_ell_h2(unsigned char* base, const uint32_t (&eo)[DV],
                                              __half2 gamma2, bool keep0) {
  constexpr uint32_t R = DC * 4;
  __half2 r[DV];
  __half2 total = gamma2;
#pragma unroll
  for (int i = 0; i < DV; ++i) {
    r[i] = *reinterpret_cast<const __half2*>(base + eo[i] + R);
    total = __hadd2(total, r[i]);
  }
#pragma unroll
  for (int i = 0; i < DV; ++i) {
    const __half2 x = h2_clamp_t<kI8>(__hsub2(total, r[i]));
    // a degree-1 variable keeps q = gamma (decoder.cpp:324-329); in int8 mode the store
    // would write gamma anyway
    if (kI8 || i > 0 || !keep0) *reinterpret_cast<__half2*>(base + eo[i]) = x;
  }
  return h22u(total) & 0x80008000u;
}

template <int DC, int DV, int CPT, int VPT, int MAXT, int MINB, bool kI8, bool kSoft = false,
          bool kDump = false>
__global__ void __launch_bounds__(MAXT, MINB)
decode_ell_h2_kernel(const __grid_constant__ DecodeParams P, const __grid_constant__ ShotIO io) {
  static_assert(DV <= DC, "padded variable slots live in the q half of the zero block");
  static_assert(CPT <= 4, "absorbed slots are packed one byte per check");
  constexpr uint32_t kMsg = 4;  // one half2 per slot
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
  const uint32_t gw0 = seg.c0 >> 5, gspan = Ms ? ((seg.c1 - 1) >> 5) - gw0 + 1 : 0u;
  const uint32_t cshift = seg.c0 & 31u;
  // the last segment also owns the padding bits of the packed rows (they are written as 0)
  const uint32_t v1z = s + 1u == nseg ? P.est_w32 * 32u : seg.v1;
  const uint32_t c1z = s + 1u == nseg ? P.syn_w32 * 32u : seg.c1;
  const uint32_t vw0 = seg.v0 >> 5, vspan = v1z > seg.v0 ? ((v1z - 1) >> 5) - vw0 + 1 : 0u;
  const uint32_t gspan_out = c1z > seg.c0 ? ((c1z - 1) >> 5) - gw0 + 1 : 0u;
  const uint64_t npairs = (io.nshots + 1) / 2;

  unsigned char* const msgs = smem_raw;
  const size_t msg_bytes = ell_msg_region_bytes(P.seg_mmax, kStride, T, DC);
  uint32_t* const bits = reinterpret_cast<uint32_t*>(smem_raw + msg_bytes);
  // [item parity][shot lane][pw] live bitmaps, counters, tickets, untouched syndrome copies
  uint32_t* const unsat_ctr = bits + 4 * pw;       // [2][2]
  uint32_t* const ticket = bits + 4 * pw + 4;      // [2]
  uint32_t* const syn_copy = bits + 4 * pw + 16;   // [2][2][pw]
  const uint32_t scratch_off = P.seg_mmax * kStride;  // first dummy block (see ell_dummy_blocks)
  const uint32_t pad_off = scratch_off + (tid / DC) * kStride + (tid % DC) * kMsg;  // this thread's slot
  const uint32_t scribble_off = scratch_off + ell_dummy_blocks(T, DC) * kStride;  // thread slots without a check

  for (uint32_t b = tid; b < (ell_dummy_blocks(T, DC) + 1u) * kStride; b += T) msgs[scratch_off + b] = 0;

  // ---- per-thread tables (as decode_ell_kernel)
  uint32_t eo[VPT][DV], co[CPT], cl[CPT], valid = 0, keep0 = 0, absorb = 0;
  __half gam[VPT];
  const uint32_t nv = P.ell_nvars[s];
  auto prior_h = [&](uint32_t n) -> __half {
    if constexpr (kI8) {
      return __float2half_rn(static_cast<float>(static_cast<const int32_t*>(P.gamma)[n]));  // exact
    } else {
      return prior_as_msg<ArithF16>(static_cast<const float*>(P.gamma)[n]);
    }
  };
  {
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
      gam[k] = ok ? prior_h(n) : __ushort_as_half(0x3c00);
    }
    const uint32_t sent_pad = kI8 ? 0x57f057f0u : 0x7c007c00u;   // 127 | +inf, both lanes
    const uint32_t sent_deg1 = kI8 ? 0x57f057f0u : 0x54005400u;  // 127 | 64
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const uint32_t m = tid + k * T;
      const bool ok = m < Ms;
      cl[k] = ok ? m : Ms;  // no check: the scribble block
      co[k] = ok ? m * kStride : scribble_off;
      uint32_t aslot = kNoAbsorb;
      if (ok) {
        const uint32_t e0 = P.check_off[seg.c0 + m];
        const uint32_t deg = P.check_off[seg.c0 + m + 1] - e0;
        const uint32_t sent = deg == 1u ? sent_deg1 : sent_pad;
#pragma unroll
        for (int j = 0; j < DC; ++j) {
          if (static_cast<uint32_t>(j) >= deg) *reinterpret_cast<uint32_t*>(msgs + co[k] + j * kMsg) = sent;
        }
        aslot = P.ell_abs[seg.c0 + m];
        if (aslot != kNoAbsorb) {  // the absorbed variable's message: its prior, for ever
          *reinterpret_cast<__half2*>(msgs + co[k] + aslot * kMsg) =
              __half2half2(prior_h(P.edge_var[e0 + aslot]));
        }
      }
      absorb |= aslot << (8 * k);
    }
  }

  uint64_t pair = peer;
  uint32_t raw_a = 0, raw_b = 0;
  if (warp == 0 && lane < gspan && pair < npairs) {
    raw_a = io.syn[(2 * pair) * P.syn_w32 + gw0 + lane];
    if (2 * pair + 1 < io.nshots) raw_b = io.syn[(2 * pair + 1) * P.syn_w32 + gw0 + lane];
  }
  // per-shot priors of this thread's absorbed variables (ShotIO::soft: int8 in int8 mode,
  // float in half mode), both shots of the pair in one half2, fetched one pair ahead
  uint32_t soft_next[kSoft ? CPT : 1];
  auto soft_h = [&](uint64_t idx) -> __half {
    if constexpr (kI8) {
      return __float2half_rn(static_cast<float>(static_cast<const int8_t*>(io.soft)[idx]));  // exact
    } else {
      return prior_as_msg<ArithF16>(static_cast<const float*>(io.soft)[idx]);
    }
  };
  auto fetch_soft = [&](uint64_t pr) {
    if constexpr (kSoft) {
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        if (cl[k] < Ms && ((absorb >> (8 * k)) & 0xffu) != kNoAbsorb) {
          const uint64_t ia = (2 * pr) * P.M + seg.c0 + cl[k];
          const __half a = soft_h(ia);
          const __half b = 2 * pr + 1 < io.nshots ? soft_h(ia + P.M) : a;
          soft_next[k] = h22u(__halves2half2(a, b));
        }
      }
    }
  };
  if (pair < npairs) fetch_soft(pair);
  uint32_t ipar = 0;
  __syncthreads();

  while (pair < npairs) {
    const uint64_t shot_a = 2 * pair, shot_b = 2 * pair + 1;
    const bool has_b = shot_b < io.nshots;
    uint32_t* const par_a = bits + (ipar * 2) * pw;
    uint32_t* const par_b = bits + (ipar * 2 + 1) * pw;
    uint32_t* const syn_a = syn_copy + (ipar * 2) * pw;
    uint32_t* const syn_b = syn_copy + (ipar * 2 + 1) * pw;
    volatile uint32_t* const unsat_a = unsat_ctr + ipar * 2;
    volatile uint32_t* const unsat_b = unsat_ctr + ipar * 2 + 1;
    // ---------------- prologue ----------------
    if (warp == 0) {
      auto localise = [&](uint32_t raw, uint32_t* par, uint32_t* syn0, volatile uint32_t* ctr) {
        uint32_t nb = __shfl_down_sync(0xffffffffu, raw, 1);
        if (lane + 1 >= gspan) nb = 0;
        uint32_t loc = cshift ? __funnelshift_r(raw, nb, cshift) : raw;
        if (lane >= pws) {
          loc = 0;
        } else if (Ms - lane * 32u < 32u) {
          loc &= (1u << (Ms - lane * 32u)) - 1u;
        }
        if (lane < pw) {
          par[lane] = loc;
          syn0[lane] = loc;
        }
        const uint32_t cnt = __reduce_add_sync(0xffffffffu, __popc(loc));
        if (lane == 0) *ctr = cnt;
      };
      localise(raw_a, par_a, syn_a, unsat_a);
      localise(raw_b, par_b, syn_b, unsat_b);
      if (lane == 0) {
        const uint64_t t = static_cast<uint64_t>(atomicAdd(&io.sched[2 + s], 1u)) + peers;
        ticket[ipar] = t < npairs ? static_cast<uint32_t>(t) : kNoShot;
      }
    }
    if (warp == nwarps - 1) {
      for (int which = 0; which < (has_b ? 2 : 1); ++which) {
        uint32_t* est_g = io.est + (shot_a + which) * P.est_w32 + vw0;
        for (uint32_t w = lane; w < vspan; w += 32u) {
          const uint32_t mask = range_mask(vw0 + w, seg.v0, v1z);
          if (mask == 0xffffffffu) {
            est_g[w] = 0u;
          } else {
            atomicAnd(&est_g[w], ~mask);
          }
        }
      }
    }
    // q[e] = gamma[var(e)] (decoder.cpp:156-158); padded slots land in the dummy blocks
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const __half2 init = __half2half2(gam[k]);
#pragma unroll
      for (int i = 0; i < DV; ++i) *reinterpret_cast<__half2*>(msgs + eo[k][i]) = init;
    }
    if constexpr (kSoft) {  // this pair's priors of the absorbed variables
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const uint32_t aslot = (absorb >> (8 * k)) & 0xffu;
        if (cl[k] < Ms && aslot != kNoAbsorb) {
          *reinterpret_cast<uint32_t*>(msgs + co[k] + aslot * kMsg) = soft_next[k];
        }
      }
    }
    uint32_t eprev_a = 0, eprev_b = 0, aprev_a = 0, aprev_b = 0;
    __syncthreads();

    uint32_t synpair[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const uint32_t ba = (syn_a[cl[k] >> 5] >> (cl[k] & 31u)) & 1u;
      const uint32_t bb = (syn_b[cl[k] >> 5] >> (cl[k] & 31u)) & 1u;
      synpair[k] = (ba << 15) | (bb << 31);
    }
    const uint32_t next = ticket[ipar];
    if (warp == 0 && lane < gspan) {
      raw_a = raw_b = 0;
      if (next != kNoShot) {
        const uint64_t na = 2ull * next;
        raw_a = io.syn[na * P.syn_w32 + gw0 + lane];
        if (na + 1 < io.nshots) raw_b = io.syn[(na + 1) * P.syn_w32 + gw0 + lane];
      }
    }
    if (next != kNoShot) fetch_soft(next);

    // ---------------- iterations ----------------
    uint32_t iter = 0, iter_a = 0, iter_b = 0;
    bool live_a = true, live_b = true, conv_a = false, conv_b = false;
    uint32_t fin_a = 0, fin_b = 0, afin_a = 0, afin_b = 0;  // decisions when each shot stopped
    for (;;) {
      ++iter;
      // Bitmaps and counters are only WRITTEN between the two barriers of an iteration and
      // only READ (the stop test) after the second one: flips of absorbed variables found in
      // the check stage wait in achg_a / achg_b until the variable stage's toggles.
      uint32_t achg_a = 0, achg_b = 0;
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        // (warps without a check in the last round skip it, as in decode_lean_kernel)
        if (k + 1 < CPT || (tid & ~31u) + static_cast<uint32_t>(CPT - 1) * T < Ms) {
          cn_ell_h2<DC, kI8>(P, msgs + co[k], synpair[k]);
          const uint32_t aslot = (absorb >> (8 * k)) & 0xffu;
          if (aslot != kNoAbsorb) {  // posteriors of the absorbed variable from the r just produced
            const unsigned char* slot = msgs + co[k] + aslot * kMsg;
            const uint32_t sg = h22u(__hadd2(*reinterpret_cast<const __half2*>(slot),
                                             *reinterpret_cast<const __half2*>(slot + DC * kMsg)));
            achg_a |= (((sg >> 15) & 1u) ^ ((aprev_a >> k) & 1u)) << k;
            achg_b |= ((sg >> 31) ^ ((aprev_b >> k) & 1u)) << k;
          }
        }
      }
      if (!live_a) achg_a = 0;
      if (!live_b) achg_b = 0;
      aprev_a ^= achg_a;
      aprev_b ^= achg_b;
      __syncthreads();
      // posterior sign bits (bits 15 / 31) shift into one accumulator: after VPT variables
      // shot a's decisions sit in bits [16-VPT, 15], shot b's in [32-VPT, 31]
      static_assert(VPT <= 8, "decision accumulator");
      uint32_t acc = 0;
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        acc = (acc >> 1) |
              vn_ell_h2<DC, DV, kI8>(msgs, eo[k], __half2half2(gam[k]), (keep0 >> k) & 1u);
      }
      uint32_t eb_a = (acc >> (16 - VPT)) & ((1u << VPT) - 1u), eb_b = acc >> (32 - VPT);
      eb_a &= valid;
      eb_b &= valid;
      auto toggle = [&](uint32_t changed, uint32_t achg, uint32_t* par, volatile uint32_t* ctr) {
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
        atomicAdd(const_cast<uint32_t*>(ctr), static_cast<uint32_t>(delta));
      };
      if (live_a) {
        const uint32_t ch = eb_a ^ eprev_a;
        eprev_a = eb_a;
        if (ch | achg_a) toggle(ch, achg_a, par_a, unsat_a);
      }
      if (live_b) {
        const uint32_t ch = eb_b ^ eprev_b;
        eprev_b = eb_b;
        if (ch | achg_b) toggle(ch, achg_b, par_b, unsat_b);
      }
      __syncthreads();
      const bool last = iter >= P.max_iter;
      if (live_a) {
        const bool uns = *unsat_a != 0u;
        if ((P.early && !uns) || last) {
          live_a = false;
          conv_a = !uns;
          iter_a = iter;
          fin_a = eprev_a;
          afin_a = aprev_a;
        }
      }
      if (live_b) {
        const bool uns = *unsat_b != 0u;
        if ((P.early && !uns) || last) {
          live_b = false;
          conv_b = !uns;
          iter_b = iter;
          fin_b = eprev_b;
          afin_b = aprev_b;
        }
      }
      if (!live_a && !live_b) break;
    }

    // ---------------- epilogue ----------------
    auto write_out = [&](uint64_t shot, const uint32_t* par, uint32_t fin, uint32_t afin, bool conv,
                         uint32_t iters) {
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
      if (fin | afin) {
        uint32_t* est_g = io.est + shot * P.est_w32;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
          if ((fin >> k) & 1u) {
            const uint32_t n = P.ell_vars[seg.v0 + tid + k * T];
            atomicOr(&est_g[n >> 5], 1u << (n & 31u));
          }
        }
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
          if ((afin >> k) & 1u) {
            const uint32_t n =
                P.edge_var[P.check_off[seg.c0 + cl[k]] + ((absorb >> (8 * k)) & 0xffu)];
            atomicOr(&est_g[n >> 5], 1u << (n & 31u));
          }
        }
      }
      if (tid == 0) {
        io.conv[shot * nseg + s] = conv ? 1 : 0;
        io.iters[shot * nseg + s] = iters;
      }
    };
    write_out(shot_a, par_a, fin_a, afin_a, conv_a, iter_a);
    if (has_b) write_out(shot_b, par_b, fin_b, afin_b, conv_b, iter_b);
    if constexpr (kDump) if (io.q_dump != nullptr && (io.dump_shot >> 1) == pair) {  // parity hook: the messages when the PAIR finished
      ell_dump_messages(P, seg, msgs, kStride, kMsg, DC * kMsg, (io.dump_shot & 1u) ? 2u : 0u,
                        [&](uint32_t e, const unsigned char* q, const unsigned char* r) {
                          const float qv = __half2float(*reinterpret_cast<const __half*>(q));
                          const float rv = __half2float(*reinterpret_cast<const __half*>(r));
                          if constexpr (kI8) {
                            static_cast<int32_t*>(io.q_dump)[e] = static_cast<int32_t>(qv);
                            static_cast<int32_t*>(io.r_dump)[e] = static_cast<int32_t>(rv);
                          } else {
                            static_cast<float*>(io.q_dump)[e] = qv;
                            static_cast<float*>(io.r_dump)[e] = rv;
                          }
                        });
    }
    pair = next == kNoShot ? ~0ull : static_cast<uint64_t>(next);
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

}  // namespace qb

// Monte-Carlo campaign kernel for (6,3)-regular CSS codes: sample -> syndrome -> decode ->
// classify inside ONE persistent kernel ("syndromes, errors and
// estimates never leave the SM").
//
// Reference loop: run_campaign (proj/src/noise.cpp:217-338) = per trial sample_error
// (:67-78, SplitMix64 streams :23-26), extract_syndromes (:97-105), Decoder::decode_css_into,
// ResidualClassifier (:128-140).  The separate-kernel pipeline (noise_syndrome_kernel ->
// decode_lean_kernel -> classify_kernel) moves 104 B of syndrome, 2 x 200 B of error /
// estimate and the flags of every trial through HBM and pays the sampler (3.8 ms per 2^20
// trials, bound by 64-bit multiplies) on top of the decode.  Here a work item is still
// (trial, segment) and the iteration loop is decode_lean_kernel's, but
//
//  * PROLOGUE: every thread draws the error bits of the variables it will update anyway
//    (thread <-> variable mapping of the variable stage; the reference's draw index is 2v for
//    the X component, 2v + 1 for the Z component, so the two segments of a trial sample their
//    halves independently and bit-exactly), and a flipped variable XORs its column straight
//    into the segment's parity bitmap in shared memory.  The multiplies run on the FMA pipe,
//    which the decode leaves idle;
//  * EPILOGUE: residual = error ^ decision per thread, in registers.  A non-zero residual bit
//    XORs the variable's logical-test column (one 64-bit mask per variable, built by
//    qb_set_logicals) into a shared accumulator: residual is a logical error iff the
//    accumulator is non-zero (the k parity tests of kernel_classify.cuh at once).  The same
//    for the sampled error itself (identity-decoder baseline);
//  * OUT: one flags byte and the iteration count per (trial, segment) - 10 B per trial
//    instead of ~720 B; campaign_count_kernel folds them into the ten counters.
//
// Bitmaps, counters and accumulators are double-buffered on the item parity: the buffer of
// item i+1 is cleared during item i (after its first barrier), the flags of item i are
// published after item i+1's first barrier, so the loop has no barrier of its own.
#pragma once

#include "common.cuh"
#include "kernel_lean.cuh"
#include "kernel_noise.cuh"

namespace qb {

struct CampaignIO {
  uint64_t ntrials;
  uint64_t first_trial;
  uint64_t seed;
  uint64_t thr;            // flip iff (draw >> 11) < thr  (kernel_noise.cuh)
  const uint64_t* tcol;    // [N] logical-test column of every variable (qb_set_logicals)
  uint8_t* flags;          // [ntrials][nseg] out, kCamp* bits
  uint32_t* iters;         // [ntrials][nseg] out
  unsigned int* sched;     // as ShotIO::sched
};

constexpr uint32_t kCampConv = 1u;      // segment converged
constexpr uint32_t kCampResNz = 2u;     // residual e ^ e_hat non-zero
constexpr uint32_t kCampResOdd = 4u;    // ... with odd overlap with a logical test
constexpr uint32_t kCampErrNz = 8u;     // sampled error non-zero
constexpr uint32_t kCampSynNz = 16u;    // its syndrome non-zero
constexpr uint32_t kCampErrOdd = 32u;   // sampled error has odd overlap with a logical test

constexpr uint32_t kCampAccWords = 8;   // {flag bits, res lo, res hi, err lo, err hi, pad...}

__host__ __device__ inline size_t campaign_smem_bytes(uint32_t seg_mmax, int arith) {
  const size_t msg = (static_cast<size_t>(seg_mmax + 1) * lean_stride(arith) + 15) & ~size_t(15);
  // table | messages | [2] parity bitmaps | [2] syndrome copies | [2] rotated copies | [2] unsat |
  // [2] tickets | [2] accumulators
  return kLeanTabBytes + msg + 4 * (6 * static_cast<size_t>(lean_pw(seg_mmax)) + 4 + 2 * kCampAccWords);
}

template <class A, int CPT, int VPT, bool kFast, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB)
decode_lean_campaign_kernel(const __grid_constant__ DecodeParams P, const __grid_constant__ CampaignIO io) {
  using Msg = typename A::Msg;
  using Gam = typename A::Gam;
  constexpr uint32_t kStride = Lay<A>::kStride;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t tid = threadIdx.x, T = blockDim.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t nwarps = T >> 5;
  const uint32_t nseg = P.nseg;  // 2: X and Z components of a CSS code
  const uint32_t s = blockIdx.x % nseg;
  const uint32_t peer = blockIdx.x / nseg;
  const uint32_t peers = (gridDim.x - s + nseg - 1) / nseg;
  const SegmentDev seg = P.segs[s];
  const uint32_t Ms = seg.c1 - seg.c0;
  const uint32_t pw = lean_pw(P.seg_mmax);

  static_assert(sizeof(Msg) == 4, "whole-word messages (fp32 / ArithI32): first iteration by table");
  unsigned char* const msgs = smem_raw + kLeanTabBytes;
  const size_t msg_bytes = (static_cast<size_t>(P.seg_mmax + 1) * kStride + 15) & ~size_t(15);
  uint32_t* const bits = reinterpret_cast<uint32_t*>(msgs + msg_bytes);
  uint32_t* const par_buf = bits;              // [2][pw] live parity bitmaps
  uint32_t* const syn_buf = bits + 2 * pw;     // [2][pw] the syndromes themselves, never toggled
  uint32_t* const rot_buf = bits + 4 * pw;     // [2][pw] ... every word rotated left by two
  uint32_t* const unsat_ctr = bits + 6 * pw;   // [2]
  uint32_t* const ticket = bits + 6 * pw + 2;  // [2]
  uint32_t* const acc_buf = bits + 6 * pw + 4; // [2][kCampAccWords]

  // ---- per-thread tables (as decode_lean_kernel; no slot permutation needed for parity)
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
      cl[k] = m < Ms ? m : Ms;
      co[k] = (m < Ms ? m : P.seg_mmax) * kStride;
    }
  }
  for (uint32_t b = tid; b < kStride; b += T) msgs[P.seg_mmax * kStride + b] = 0;  // dummy block
  for (uint32_t w = tid; w < 6 * pw + 4 + 2 * kCampAccWords; w += T) bits[w] = 0u;
  if (tid < 3) reinterpret_cast<uint32_t*>(smem_raw)[tid] = P.it1_tq[tid];

  uint64_t shot = peer;
  uint32_t ipar = 0;
  // flags of the previous item, published one item late by thread 0
  uint32_t pend_flags = 0, pend_valid = 0;
  uint64_t pend_shot = 0;
  __syncthreads();

  while (shot < io.ntrials) {
    uint32_t* const par = par_buf + ipar * pw;
    uint32_t* const syn0 = syn_buf + ipar * pw;
    uint32_t* const syn2 = rot_buf + ipar * pw;
    volatile uint32_t* const unsat = unsat_ctr + ipar;
    uint32_t* const acc = acc_buf + ipar * kCampAccWords;
    // ---------------- prologue: sample, syndrome ----------------
    if (tid == 0) {  // the next item's ticket, one item ahead
      const uint64_t t = static_cast<uint64_t>(atomicAdd(&io.sched[2 + s], 1u)) + peers;
      ticket[ipar] = t < io.ntrials ? static_cast<uint32_t>(t) : kNoShot;
    }
    uint32_t err = 0;
    {
      // sample_error, independent-xz (noise.cpp:73-77): draw 2v is X_v, draw 2v + 1 is Z_v
      const uint64_t trial = io.first_trial + shot;
      const uint64_t state0 = splitmix_mix(io.seed + kPhi * trial + kPhi);
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        const uint32_t nl = tid + k * T;
        const uint64_t z = splitmix_mix(state0 + static_cast<uint64_t>(2u * nl + s + 1u) * kPhi);
        err |= (((z >> 11) < io.thr) ? 1u : 0u) << k;
      }
      err &= valid;
    }
    if (err) {  // extract_syndromes: XOR the columns of the flipped variables (noise.cpp:97-105)
      int32_t delta = 0;
      uint64_t tc = 0;
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        if ((err >> k) & 1u) {
#pragma unroll
          for (int i = 0; i < kDV; ++i) {
            const uint32_t lm = eo[k][i] / kStride;
            const uint32_t bit = 1u << (lm & 31u);
            const uint32_t old = atomicXor(&par[lm >> 5], bit);
            atomicXor(&syn0[lm >> 5], bit);
            if constexpr (kFast) atomicXor(&syn2[lm >> 5], __funnelshift_l(bit, bit, 2));
            delta += (old & bit) ? -1 : 1;
          }
          tc ^= io.tcol[seg.v0 + tid + k * T];
        }
      }
      atomicAdd(const_cast<uint32_t*>(unsat), static_cast<uint32_t>(delta));
      atomicOr(&acc[0], kCampErrNz);
      if (static_cast<uint32_t>(tc)) atomicXor(&acc[3], static_cast<uint32_t>(tc));
      if (static_cast<uint32_t>(tc >> 32)) atomicXor(&acc[4], static_cast<uint32_t>(tc >> 32));
    }
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

    // the other buffer: publish the previous item's flags, then clear it for the next item
    {
      uint32_t* const oacc = acc_buf + (ipar ^ 1u) * kCampAccWords;
      if (tid == 0 && pend_valid) {
        uint32_t f = pend_flags | oacc[0];
        if (oacc[1] | oacc[2]) f |= kCampResOdd;
        if (oacc[3] | oacc[4]) f |= kCampErrOdd;
        io.flags[pend_shot * nseg + s] = static_cast<uint8_t>(f);
      }
      if (warp == nwarps - 1) {
        __syncwarp();
        uint32_t* const opar = par_buf + (ipar ^ 1u) * pw;
        uint32_t* const osyn = syn_buf + (ipar ^ 1u) * pw;
        uint32_t* const orot = rot_buf + (ipar ^ 1u) * pw;
        for (uint32_t w = lane; w < pw; w += 32u) {
          opar[w] = 0u;
          osyn[w] = 0u;
          orot[w] = 0u;
        }
        if (lane == 0) unsat_ctr[ipar ^ 1u] = 0u;
      }
      if (tid == 0) {
        for (uint32_t w = 0; w < kCampAccWords; ++w) oacc[w] = 0u;
      }
    }
    uint32_t synbits = 0;
#pragma unroll
    for (int k = 0; k < CPT; ++k) synbits |= ((syn0[cl[k] >> 5] >> (cl[k] & 31u)) & 1u) << k;
    const uint32_t next = ticket[ipar];
    uint32_t syn_nz = 0;
    if (warp == 0) {
      const uint32_t w = lane < pw ? syn0[lane] : 0u;
      syn_nz = __any_sync(0xffffffffu, w != 0u) ? kCampSynNz : 0u;
    }

    // ---------------- iterations (decode_lean_kernel's loop) ----------------
    uint32_t iter = 0;
    bool still_unsat;
    for (;;) {
      ++iter;
      uint32_t eb = 0;
      if (kFast && iter == 1u) {
#pragma unroll
        for (int k = 0; k < VPT; ++k) eb |= vn3_first_tab<kStride>(P, msgs, smem_raw, eo[k], syn2) << k;
      } else {
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
          // (warps without a check in the last round skip it, as in decode_lean_kernel)
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

    // ---------------- epilogue: classify in registers ----------------
    const uint32_t res = (eprev ^ err) & valid;
    if (res) {
      uint64_t tc = 0;
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        if ((res >> k) & 1u) tc ^= io.tcol[seg.v0 + tid + k * T];
      }
      atomicOr(&acc[0], kCampResNz);
      if (static_cast<uint32_t>(tc)) atomicXor(&acc[1], static_cast<uint32_t>(tc));
      if (static_cast<uint32_t>(tc >> 32)) atomicXor(&acc[2], static_cast<uint32_t>(tc >> 32));
    }
    if (tid == 0) {
      io.iters[shot * nseg + s] = iter;
      pend_flags = (still_unsat ? 0u : kCampConv) | syn_nz;
      pend_shot = shot;
      pend_valid = 1u;
    }
    shot = next == kNoShot ? ~0ull : static_cast<uint64_t>(next);
    ipar ^= 1u;
  }

  __syncthreads();  // the last item's accumulators are complete
  if (tid == 0) {
    if (pend_valid) {
      const uint32_t* const oacc = acc_buf + (ipar ^ 1u) * kCampAccWords;
      uint32_t f = pend_flags | oacc[0];
      if (oacc[1] | oacc[2]) f |= kCampResOdd;
      if (oacc[3] | oacc[4]) f |= kCampErrOdd;
      io.flags[pend_shot * nseg + s] = static_cast<uint8_t>(f);
    }
    __threadfence();
    const unsigned int done = atomicAdd(&io.sched[1], 1u);
    if (done == gridDim.x - 1) {
      for (uint32_t k = 0; k < 2 + kMaxSegments; ++k) io.sched[k] = 0;
      __threadfence();
    }
  }
}

// Folds the per-(trial, segment) flags into the ten counters of qb_campaign_run
// (ResidualClassifier + baseline of run_campaign, noise.cpp:255-304).
__global__ void __launch_bounds__(256)
campaign_count_kernel(uint64_t ntrials, const uint8_t* flags, const uint32_t* iters,
                      unsigned long long* counters) {
  __shared__ unsigned long long local[10];
  if (threadIdx.x < 10) local[threadIdx.x] = 0ull;
  __syncthreads();
  unsigned long long c[10] = {};
  for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < ntrials;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t fx = flags[2 * t], fz = flags[2 * t + 1];
    const bool conv = (fx & kCampConv) && (fz & kCampConv);
    int cls = 5;
    if (conv) {
      const bool rx_zero = !(fx & kCampResNz), rz_zero = !(fz & kCampResNz);
      if (rx_zero && rz_zero) {
        cls = 0;
      } else {
        const bool xh = rx_zero || !(fx & kCampResOdd), zh = rz_zero || !(fz & kCampResOdd);
        cls = (xh && zh) ? 1 : (!xh && !zh) ? 4 : xh ? 3 : 2;
      }
    }
    ++c[cls];
    const bool bx = !(fx & kCampErrNz) || (!(fx & kCampSynNz) && !(fx & kCampErrOdd));
    const bool bz = !(fz & kCampErrNz) || (!(fz & kCampSynNz) && !(fz & kCampErrOdd));
    if (!(bx && bz)) ++c[6];
    if (conv) ++c[7];
    c[8] += max(iters[2 * t], iters[2 * t + 1]);
    ++c[9];
  }
  for (int k = 0; k < 10; ++k) {
    if (c[k]) atomicAdd(&local[k], c[k]);
  }
  __syncthreads();
  if (threadIdx.x < 10 && local[threadIdx.x]) atomicAdd(&counters[threadIdx.x], local[threadIdx.x]);
}

}  // namespace qb

// On-device code-capacity noise + syndrome generator.
//
// Reproduces the reference sampler BIT FOR BIT so that it can be pinned against
// `sample_error` + `extract_syndromes` (proj/src/noise.cpp:23-26, :67-78,
// :97-105; SplitMix64 at proj/include/qldpc/noise.hpp:28-45):
//
//   state0(trial) = mix(seed + PHI*trial + PHI)          (the seeder's first draw)
//   draw j        = mix(state0 + (j + 1) * PHI)          (SplitMix64 is a counter)
//   unit          = (draw >> 11) * 2^-53 ;  bit = unit < p
//
// independent-xz draws (X_0, Z_0, X_1, Z_1, ...), so on the combined graph
// variable v < n (X error of qubit v) uses draw 2v and variable v >= n (Z error
// of qubit v - n) uses draw 2(v - n) + 1.  Because SplitMix64 is counter-based,
// every bit of every shot is generated independently: one warp per shot, 32
// variables per step, errors packed with __ballot_sync straight into the
// Gf2Vector word layout.
//
// Two things keep it cheap without changing a bit of the stream:
//  * `unit < p` with unit = k * 2^-53 (k = draw >> 11, an integer below 2^53) is the
//    INTEGER comparison k < ceil(p * 2^53): p * 2^53 is exact in fp64, and for an
//    integer k, k < x <=> k < ceil(x).  The host precomputes the threshold(s); no
//    64-bit integer -> fp64 conversion and no fp64 compare per draw;
//  * the syndrome H e is accumulated SPARSELY: only a flipped variable (1 in 1/p)
//    XORs its column - its few checks - into the warp's syndrome words in shared
//    memory, instead of every check gathering all of its variables.
#pragma once

#include <cmath>

#include "common.cuh"

namespace qb {

struct NoiseParams {
  uint64_t seed;
  uint64_t first_trial;
  uint64_t nshots;
  uint64_t thr;            // ceil(p * 2^53): flip iff (draw >> 11) < thr (when thrs == nullptr)
  const uint64_t* thrs;    // optional per-variable thresholds [N]
  uint32_t mode;       // 0: variable v uses draw v; 1: CSS independent-xz interleave
  uint32_t n_qubits;   // mode 1: variables [0,n) are X errors, [n,2n) Z errors
  uint32_t* syn;       // [nshots][syn_w32] out
  uint32_t* err;       // [nshots][est_w32] out, may be nullptr
};

// ceil(p * 2^53) for p in [0, 1] (host)
inline uint64_t noise_threshold(double p) {
  if (!(p > 0.0)) return 0;
  if (p >= 1.0) return 1ull << 53;
  return static_cast<uint64_t>(std::ceil(std::ldexp(p, 53)));
}

constexpr uint64_t kPhi = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

constexpr int kNoiseWarps = 8;

// kCss: CSS independent-xz interleave (NoiseParams::mode 1); kPerVar: per-variable thresholds
template <bool kCss, bool kPerVar>
__global__ void __launch_bounds__(kNoiseWarps * 32)
noise_syndrome_kernel(const __grid_constant__ DecodeParams P, const __grid_constant__ NoiseParams np) {
  extern __shared__ uint32_t noise_smem[];  // [kNoiseWarps][syn_w32 + est_w32]
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint32_t* sbits = noise_smem + warp * (P.syn_w32 + P.est_w32);
  uint32_t* ebits = sbits + P.syn_w32;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kNoiseWarps;
  const uint32_t N = P.N, nq = np.n_qubits, steps = P.est_w32;
  const uint64_t thr = np.thr;
  for (uint64_t shot = static_cast<uint64_t>(blockIdx.x) * kNoiseWarps + warp; shot < np.nshots;
       shot += stride) {
    const uint64_t trial = np.first_trial + shot;
    const uint64_t state0 = splitmix_mix(np.seed + kPhi * trial + kPhi);
    for (uint32_t w = lane; w < P.syn_w32; w += 32u) sbits[w] = 0u;
    __syncwarp();
#pragma unroll 2
    for (uint32_t step = 0; step < steps; ++step) {
      const uint32_t v = step * 32u + lane;
      uint32_t j = v;  // draw index of variable v
      if constexpr (kCss) j = v < nq ? 2u * v : 2u * (v - nq) + 1u;
      const uint64_t z = splitmix_mix(state0 + static_cast<uint64_t>(j + 1u) * kPhi);
      uint64_t t = thr;
      if constexpr (kPerVar) t = v < N ? np.thrs[v] : 0ull;
      const bool bit = v < N && (z >> 11) < t;
      const uint32_t word = __ballot_sync(0xffffffffu, bit);
      if (lane == 0) ebits[step] = word;
      if (bit) {  // XOR this variable's column of H into the syndrome
        for (uint32_t i = P.var_off[v]; i < P.var_off[v + 1]; ++i) {
          const uint32_t m = P.edge_check[P.var_edges[i]];
          atomicXor(&sbits[m >> 5], 1u << (m & 31u));
        }
      }
    }
    __syncwarp();
    for (uint32_t w = lane; w < P.syn_w32; w += 32u) np.syn[shot * P.syn_w32 + w] = sbits[w];
    if (np.err) {
      for (uint32_t w = lane; w < P.est_w32; w += 32u) np.err[shot * P.est_w32 + w] = ebits[w];
    }
    __syncwarp();
  }
}

// ---- fast sampler (QB_OPT_SAMPLER = 1): same distribution, NOT the reference's stream ----
//
// The reference draws one uniform per variable; at p = 0.01 that is 1568 SplitMix64
// outputs per [[784,24,24]] shot for ~16 flips.  Flips of an i.i.d. Bernoulli(p) sequence
// are separated by geometric gaps, so this kernel draws one uniform per FLIP instead:
//
//   gap = floor(ln(u) / ln(1 - p)),  u uniform in (0, 1)      P(gap = g) = (1-p)^g p
//
// Non-uniform probabilities are sampled by thinning: gaps at p_max, a candidate v is kept
// with probability p_v / p_max (second draw, integer threshold).  The stream is still a
// counter-based SplitMix64 keyed by (seed, trial), so a campaign's result does not depend on
// how its trials are split over launches or GPUs.  Logarithms are evaluated in fp64: about
// p*N of them per shot.
//
// One THREAD per shot: each thread owns an odd-stride row of shared memory (syndrome words
// then error words), ORs / XORs its flips into it, and the CTA copies the rows out with
// coalesced stores.
struct SkipParams {
  double inv_log1m;   // 1 / ln(1 - p_max)  (<= -0.0; -inf when p_max = 0 => no flips)
  uint32_t row;       // shared-memory row stride in words, odd, >= syn_w32 + est_w32
};

template <bool kPerVar>
__global__ void noise_skip_kernel(const __grid_constant__ DecodeParams P,
                                  const __grid_constant__ NoiseParams np,
                                  const __grid_constant__ SkipParams sp) {
  extern __shared__ uint32_t noise_smem[];  // [blockDim.x][row]
  const uint32_t nthreads = blockDim.x, row = sp.row;
  const uint32_t sw = P.syn_w32, ew = P.est_w32, N = P.N;
  uint32_t* mine = noise_smem + threadIdx.x * row;
  const double dN = static_cast<double>(N);
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * nthreads; base < np.nshots;
       base += static_cast<uint64_t>(gridDim.x) * nthreads) {
    for (uint32_t w = 0; w < sw + ew; ++w) mine[w] = 0u;
    const uint64_t shot = base + threadIdx.x;
    if (shot < np.nshots) {
      const uint64_t state0 = splitmix_mix(np.seed + kPhi * (np.first_trial + shot) + kPhi);
      uint64_t ctr = state0;
      double pos = -1.0;  // exact: integers far below 2^53
      for (;;) {
        ctr += kPhi;
        const uint64_t z = splitmix_mix(ctr);
        // 52 random bits + 1/2: every value is exact in fp64 and lies strictly inside (0, 1)
        const double u = (static_cast<double>(z >> 12) + 0.5) * 0x1p-52;
        const double gap = floor(log(u) * sp.inv_log1m);
        pos += gap + 1.0;
        if (!(pos < dN)) break;  // also ends the shot when p_max = 0 (gap = +inf)
        const uint32_t v = static_cast<uint32_t>(pos);
        if constexpr (kPerVar) {
          ctr += kPhi;
          if ((splitmix_mix(ctr) >> 11) >= np.thrs[v]) continue;  // thinning: keep w.p. p_v / p_max
        }
        mine[sw + (v >> 5)] |= 1u << (v & 31u);
        for (uint32_t i = P.var_off[v]; i < P.var_off[v + 1]; ++i) {
          const uint32_t m = P.edge_check[P.var_edges[i]];
          mine[m >> 5] ^= 1u << (m & 31u);
        }
      }
    }
    __syncthreads();
    const uint64_t left = np.nshots - base;
    const uint32_t here = left < nthreads ? static_cast<uint32_t>(left) : nthreads;
    for (uint32_t i = threadIdx.x; i < here * sw; i += nthreads) {
      const uint32_t s = i / sw, w = i - s * sw;
      np.syn[base * sw + i] = noise_smem[s * row + w];
    }
    if (np.err) {
      for (uint32_t i = threadIdx.x; i < here * ew; i += nthreads) {
        const uint32_t s = i / ew, w = i - s * ew;
        np.err[base * ew + i] = noise_smem[s * row + sw + w];
      }
    }
    __syncthreads();
  }
}


// ---- soft (noisy) syndrome measurement: BASELINE config 5 ---------------------------
//
// Acts in place on the output of the samplers above when only the DATA variables of an
// extended graph [H | I] were allowed to flip, so that `syn` holds the noiseless syndrome
// s~ = H e_data.  Every check m is then "measured" through a Gaussian channel
//
//   l_m = (1 - 2 s~_m) * mu + sigma * g,   g ~ N(0, 1)
//
// and replaced by what a soft-input decoder sees: the hard bit s_m = [l_m < 0] and the
// reliability |LLR_m| = 2 mu |l_m| / sigma^2, which becomes the per-shot prior of check m's
// absorbed measurement-error variable (ShotIO::soft).  A flipped measurement (s_m != s~_m)
// is recorded as an error on that variable, so that err still satisfies H_ext err = syn.
// The reference has no such model; the stream is a counter-based SplitMix64
// keyed by (seed, trial, check), Box-Muller in fp64 - independent of the launch partition.
struct SoftParams {
  uint64_t seed;
  uint64_t first_trial;
  uint64_t nshots;
  double mu, sigma;
  double llr_scale;     // 2 mu / sigma^2
  double quant_scale;   // integer modes: prior = clamp(round(LLR * quant_scale), 1, kmax)
  int32_t kmax;         // 0: float output
  uint32_t elem_bytes;  // 4 (float), 1 (int8), 2 (int16)
  uint32_t* syn;        // [nshots][syn_w32] in: s~, out: s
  uint32_t* err;        // [nshots][est_w32] or nullptr: measurement flips are ORed in
  void* soft;           // [nshots][M] out
};

constexpr uint64_t kSoftSalt = 0x5851F42D4C957F2Dull;

__global__ void __launch_bounds__(kNoiseWarps * 32)
soft_measure_kernel(const __grid_constant__ DecodeParams P, const __grid_constant__ SoftParams sp) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kNoiseWarps;
  const uint32_t M = P.M;
  for (uint64_t shot = static_cast<uint64_t>(blockIdx.x) * kNoiseWarps + warp; shot < sp.nshots;
       shot += stride) {
    const uint64_t trial = sp.first_trial + shot;
    const uint64_t state0 = splitmix_mix((sp.seed ^ kSoftSalt) + kPhi * trial + kPhi);
    for (uint32_t w = 0; w < P.syn_w32; ++w) {
      const uint32_t m = w * 32u + lane;
      const uint32_t in = sp.syn[shot * P.syn_w32 + w];
      bool s = m < M && ((in >> lane) & 1u);
      // only a check with an absorbed measurement-error variable is measured noisily; any
      // other check keeps its bit (its soft value is never read by the decoder)
      const uint32_t slot = m < M ? P.ell_abs[m] : kNoAbsorb;
      if (slot != kNoAbsorb) {
        const uint64_t z1 = splitmix_mix(state0 + static_cast<uint64_t>(2u * m + 1u) * kPhi);
        const uint64_t z2 = splitmix_mix(state0 + static_cast<uint64_t>(2u * m + 2u) * kPhi);
        const double u1 = (static_cast<double>(z1 >> 12) + 0.5) * 0x1p-52;  // in (0, 1)
        const double u2 = (static_cast<double>(z2 >> 12) + 0.5) * 0x1p-52;
        const double g = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
        const bool s0 = (in >> lane) & 1u;
        const double l = (s0 ? -sp.mu : sp.mu) + sp.sigma * g;
        s = l < 0.0;
        const double llr = sp.llr_scale * fabs(l);
        const uint64_t idx = shot * M + m;
        if (sp.kmax == 0) {
          static_cast<float*>(sp.soft)[idx] = static_cast<float>(llr);
        } else {
          // quantize_saturate (decoder.cpp:500-509) with the reference's "must not be 0" rule
          // (decoder.cpp:115-120) enforced by clamping up to 1
          const double scaled = llr * sp.quant_scale;
          int32_t q = scaled >= static_cast<double>(sp.kmax) ? sp.kmax
                                                             : static_cast<int32_t>(llrint(scaled));
          q = q < 1 ? 1 : q;
          if (sp.elem_bytes == 1u) {
            static_cast<int8_t*>(sp.soft)[idx] = static_cast<int8_t>(q);
          } else {
            static_cast<int16_t*>(sp.soft)[idx] = static_cast<int16_t>(q);
          }
        }
        if (s != s0 && sp.err) {  // a measurement flip: an error on the check's absorbed variable
          const uint32_t v = P.edge_var[P.check_off[m] + slot];
          atomicOr(&sp.err[shot * P.est_w32 + (v >> 5)], 1u << (v & 31u));
        }
      }
      const uint32_t out = __ballot_sync(0xffffffffu, s);
      if (lane == 0) sp.syn[shot * P.syn_w32 + w] = out;
    }
  }
}

}  // namespace qb

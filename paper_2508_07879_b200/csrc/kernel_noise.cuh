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
// Gf2Vector word layout; the syndrome is then one XOR-gather per check.
#pragma once

#include "common.cuh"

namespace qb {

struct NoiseParams {
  uint64_t seed;
  uint64_t first_trial;
  uint64_t nshots;
  double p;            // uniform flip probability (used when probs == nullptr)
  const double* probs; // optional per-variable probabilities [N]
  uint32_t mode;       // 0: variable v uses draw v; 1: CSS independent-xz interleave
  uint32_t n_qubits;   // mode 1: variables [0,n) are X errors, [n,2n) Z errors
  uint32_t* syn;       // [nshots][syn_w32] out
  uint32_t* err;       // [nshots][est_w32] out, may be nullptr
};

constexpr uint64_t kPhi = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

constexpr int kNoiseWarps = 8;

__global__ void __launch_bounds__(kNoiseWarps * 32)
noise_syndrome_kernel(const __grid_constant__ DecodeParams P, const __grid_constant__ NoiseParams np) {
  extern __shared__ uint32_t noise_smem[];  // [kNoiseWarps][est_w32]
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint32_t* ebits = noise_smem + warp * P.est_w32;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kNoiseWarps;
  for (uint64_t shot = static_cast<uint64_t>(blockIdx.x) * kNoiseWarps + warp; shot < np.nshots;
       shot += stride) {
    const uint64_t trial = np.first_trial + shot;
    const uint64_t state0 = splitmix_mix(np.seed + kPhi * trial + kPhi);
    for (uint32_t vb = 0; vb < P.est_w32 * 32u; vb += 32u) {
      const uint32_t v = vb + lane;
      bool bit = false;
      if (v < P.N) {
        uint64_t j = v;
        if (np.mode == 1u) j = v < np.n_qubits ? 2ull * v : 2ull * (v - np.n_qubits) + 1ull;
        const uint64_t z = splitmix_mix(state0 + (j + 1ull) * kPhi);
        const double unit = static_cast<double>(z >> 11) * 0x1.0p-53;
        bit = unit < (np.probs ? np.probs[v] : np.p);
      }
      const uint32_t word = __ballot_sync(0xffffffffu, bit);
      if (lane == 0) {
        ebits[vb >> 5] = word;
        if (np.err) np.err[shot * P.est_w32 + (vb >> 5)] = word;
      }
    }
    __syncwarp();
    for (uint32_t mb = 0; mb < P.syn_w32 * 32u; mb += 32u) {
      const uint32_t m = mb + lane;
      uint32_t parity = 0;
      if (m < P.M) {
        for (uint32_t e = P.check_off[m]; e < P.check_off[m + 1]; ++e) {
          const uint32_t v = P.edge_var[e];
          parity ^= (ebits[v >> 5] >> (v & 31u)) & 1u;
        }
      }
      const uint32_t word = __ballot_sync(0xffffffffu, parity != 0u);
      if (lane == 0) np.syn[shot * P.syn_w32 + (mb >> 5)] = word;
    }
    __syncwarp();
  }
}

}  // namespace qb

// On-device residual classification for Monte-Carlo campaigns
// (reference: run_campaign / ResidualClassifier, proj/src/noise.cpp:128-140,
// :255-271).  A residual r = e ^ e_hat of a CONVERGED component has zero
// syndrome, so "r lies in the row space of its parity-check matrix" is
// equivalent to "r has even overlap with every logical operator of the opposite
// type": k parity tests instead of a Gaussian elimination per shot.  The test
// vectors are supplied by the host (qb_set_logicals) already placed in the
// combined-graph layout, so one kernel serves both components.
//
// One warp per shot; lanes stride over the test vectors.  Counters are
// accumulated per CTA and added to global memory once per CTA.
#pragma once

#include "common.cuh"

namespace qb {

struct ClassifyParams {
  uint64_t nshots;
  const uint32_t* err;    // [nshots][est_w32] sampled error (e_x ++ e_z)
  const uint32_t* est;    // [nshots][est_w32] decoded estimate
  const uint32_t* syn;    // [nshots][syn_w32] syndrome (for the identity-decoder baseline)
  const uint8_t* conv;    // [nshots][2]
  const uint32_t* iters;  // [nshots][2]
  const uint32_t* tests_x;  // [n_x][est_w32]: odd overlap => X residual is a logical error
  const uint32_t* tests_z;  // [n_z][est_w32]
  uint32_t n_x, n_z;
  // optional [est_w32]: variables that are NOT data qubits (the measurement-error variables of
  // an extended graph [H | I]).  H_ext r = 0 for a converged residual r means H r_data = r_aux,
  // so a residual with a bit on an auxiliary variable has a data part with NON-ZERO syndrome:
  // it counts as a logical error of its component (qb_set_auxiliary_vars).
  const uint32_t* aux_mask;
  unsigned long long* counters;  // [10], see qb_campaign_run
};

constexpr int kClassifyWarps = 8;

__device__ __forceinline__ bool any_odd_overlap(const uint32_t* tests, uint32_t ntests,
                                                const uint32_t* vec, uint32_t words,
                                                uint32_t lane) {
  bool bad = false;
  for (uint32_t j = lane; j < ntests; j += 32u) {
    uint32_t acc = 0;
    const uint32_t* t = tests + static_cast<size_t>(j) * words;
    for (uint32_t w = 0; w < words; ++w) acc ^= t[w] & vec[w];
    bad = bad || (__popc(acc) & 1u);
  }
  return __any_sync(0xffffffffu, bad);
}

__global__ void __launch_bounds__(kClassifyWarps * 32)
classify_kernel(const __grid_constant__ DecodeParams P, const __grid_constant__ ClassifyParams cp) {
  extern __shared__ uint32_t cls_smem[];  // [kClassifyWarps][2][est_w32] residual, error
  __shared__ unsigned long long local[10];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  if (threadIdx.x < 10) local[threadIdx.x] = 0ull;
  __syncthreads();
  uint32_t* resid = cls_smem + warp * 2 * P.est_w32;
  uint32_t* error = resid + P.est_w32;
  const SegmentDev sx = P.segs[0], sz = P.segs[1];
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kClassifyWarps;
  for (uint64_t shot = static_cast<uint64_t>(blockIdx.x) * kClassifyWarps + warp; shot < cp.nshots;
       shot += stride) {
    bool ex_zero = true, ez_zero = true, rx_zero = true, rz_zero = true;
    bool ex_aux = false, ez_aux = false, rx_aux = false, rz_aux = false;
    for (uint32_t w = lane; w < P.est_w32; w += 32u) {
      const uint32_t e = cp.err[shot * P.est_w32 + w];
      const uint32_t r = e ^ cp.est[shot * P.est_w32 + w];
      error[w] = e;
      resid[w] = r;
      const uint32_t mx = range_mask(w, sx.v0, sx.v1), mz = range_mask(w, sz.v0, sz.v1);
      ex_zero = ex_zero && (e & mx) == 0;
      ez_zero = ez_zero && (e & mz) == 0;
      rx_zero = rx_zero && (r & mx) == 0;
      rz_zero = rz_zero && (r & mz) == 0;
      if (cp.aux_mask) {
        const uint32_t am = cp.aux_mask[w];
        ex_aux = ex_aux || (e & mx & am) != 0;
        ez_aux = ez_aux || (e & mz & am) != 0;
        rx_aux = rx_aux || (r & mx & am) != 0;
        rz_aux = rz_aux || (r & mz & am) != 0;
      }
    }
    ex_zero = __all_sync(0xffffffffu, ex_zero);
    ez_zero = __all_sync(0xffffffffu, ez_zero);
    rx_zero = __all_sync(0xffffffffu, rx_zero);
    rz_zero = __all_sync(0xffffffffu, rz_zero);
    ex_aux = __any_sync(0xffffffffu, ex_aux);
    ez_aux = __any_sync(0xffffffffu, ez_aux);
    rx_aux = __any_sync(0xffffffffu, rx_aux);
    rz_aux = __any_sync(0xffffffffu, rz_aux);
    bool sx_zero = true, sz_zero = true;
    for (uint32_t w = lane; w < P.syn_w32; w += 32u) {
      const uint32_t sw = cp.syn[shot * P.syn_w32 + w];
      sx_zero = sx_zero && (sw & range_mask(w, sx.c0, sx.c1)) == 0;
      sz_zero = sz_zero && (sw & range_mask(w, sz.c0, sz.c1)) == 0;
    }
    sx_zero = __all_sync(0xffffffffu, sx_zero);
    sz_zero = __all_sync(0xffffffffu, sz_zero);
    __syncwarp();
    const bool conv_x = cp.conv[shot * 2] != 0, conv_z = cp.conv[shot * 2 + 1] != 0;
    const uint32_t it = max(cp.iters[shot * 2], cp.iters[shot * 2 + 1]);
    // decoded residual (only meaningful when both components converged)
    int cls = 5;  // non-converged
    if (conv_x && conv_z) {
      if (rx_zero && rz_zero) {
        cls = 0;  // exact
      } else {
        const bool x_harmless =
            rx_zero || (!rx_aux && !any_odd_overlap(cp.tests_x, cp.n_x, resid, P.est_w32, lane));
        const bool z_harmless =
            rz_zero || (!rz_aux && !any_odd_overlap(cp.tests_z, cp.n_z, resid, P.est_w32, lane));
        cls = (x_harmless && z_harmless) ? 1 : (!x_harmless && !z_harmless) ? 4 : x_harmless ? 3 : 2;
      }
    }
    // identity decoder on the same error: e is harmless iff it has zero syndrome and
    // even overlap with every logical of the opposite type
    const bool bx_harmless =
        ex_zero || (sx_zero && !ex_aux && !any_odd_overlap(cp.tests_x, cp.n_x, error, P.est_w32, lane));
    const bool bz_harmless =
        ez_zero || (sz_zero && !ez_aux && !any_odd_overlap(cp.tests_z, cp.n_z, error, P.est_w32, lane));
    if (lane == 0) {
      atomicAdd(&local[cls], 1ull);
      if (!(bx_harmless && bz_harmless)) atomicAdd(&local[6], 1ull);
      if (conv_x && conv_z) atomicAdd(&local[7], 1ull);
      atomicAdd(&local[8], static_cast<unsigned long long>(it));
      atomicAdd(&local[9], 1ull);
    }
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x < 10 && local[threadIdx.x]) atomicAdd(&cp.counters[threadIdx.x], local[threadIdx.x]);
}

}  // namespace qb

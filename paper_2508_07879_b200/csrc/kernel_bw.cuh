// Shared-memory bandwidth microbenchmark: the measured denominator of the
// decoder's roofline (the binding resource is SM shared-memory
// bandwidth, which MEASURED_PEAKS.json does not contain).  Every SM streams a
// conflict-free 50/50 mix of 32-bit loads and stores — the access width and
// read/write mix of the message arrays — so the figure is the attainable
// crossbar rate for this access class, not the 128 B/clk/SM datasheet number.
#pragma once

#include "common.cuh"

namespace qb {

constexpr int kBwThreads = 1024;
constexpr int kBwWords = 16 * 1024;  // 64 KB of shared memory per CTA

template <int kVec>
__global__ void __launch_bounds__(kBwThreads, 1)
smem_bandwidth_kernel(uint32_t iters, float* sink) {
  extern __shared__ __align__(16) float bw_smem[];
  for (int i = threadIdx.x; i < kBwWords; i += kBwThreads) bw_smem[i] = static_cast<float>(i);
  __syncthreads();
  if constexpr (kVec == 1) {
    float acc = 0.f;
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < kBwWords / kBwThreads; ++k) {
        const int idx = k * kBwThreads + threadIdx.x;
        const float v = bw_smem[idx];
        acc += v;
        bw_smem[idx] = acc;  // same thread rewrites its own word: no hazard, no conflict
      }
    }
    if (acc == 123.456f) *sink = acc;
  } else {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    float4* s4 = reinterpret_cast<float4*>(bw_smem);
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < kBwWords / 4 / kBwThreads; ++k) {
        const int idx = k * kBwThreads + threadIdx.x;
        const float4 v = s4[idx];
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        s4[idx] = acc;
      }
    }
    if (acc.x == 123.456f) *sink = acc.x;
  }
}

}  // namespace qb

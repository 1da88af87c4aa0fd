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

__device__ __forceinline__ float lds32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void sts32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

// Volatile PTX accesses: the compiler can neither hoist the loads out of the
// iteration loop nor keep the words in registers.
template <int kVec>
__global__ void __launch_bounds__(kBwThreads, 1)
smem_bandwidth_kernel(uint32_t iters, float* sink) {
  extern __shared__ __align__(16) float bw_smem[];
  for (int i = threadIdx.x; i < kBwWords; i += kBwThreads) bw_smem[i] = static_cast<float>(i);
  __syncthreads();
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(bw_smem));
  if constexpr (kVec == 1) {
    float acc = 0.f;
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < kBwWords / kBwThreads; ++k) {
        const uint32_t addr = base + 4u * (k * kBwThreads + threadIdx.x);
        acc += lds32(addr);
        sts32(addr, acc);  // same thread rewrites its own word: no hazard, no conflict
      }
    }
    if (acc == 123.456f) *sink = acc;
  } else {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < kBwWords / 4 / kBwThreads; ++k) {
        const uint32_t addr = base + 16u * (k * kBwThreads + threadIdx.x);
        const float4 v = lds128(addr);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        sts128(addr, acc);
      }
    }
    if (acc.x == 123.456f) *sink = acc.x;
  }
}

}  // namespace qb

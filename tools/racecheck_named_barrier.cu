// Control experiment for compute-sanitizer racecheck (tools/sanitize.sh): two warp groups of
// one CTA, each synchronising ONLY its own threads with a named barrier (`bar.sync id, count`,
// the primitive behind group_barrier() in csrc/common.cuh), exchange data through shared
// memory in a correctly synchronised write -> barrier -> read -> barrier loop.  The program is
// race-free by construction and prints a checksum; if racecheck reports hazards on it, its
// reports on decode_regular_kernel / decode_generic_kernel (the two kernels that use named
// barriers) say nothing about those kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o tools/racecheck_named_barrier tools/racecheck_named_barrier.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void group_barrier(unsigned id, unsigned n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__global__ void two_groups(unsigned* out, int iters_a, int iters_b, int full_barrier) {
  __shared__ unsigned buf[2][64];
  const unsigned group = threadIdx.x / 64, t = threadIdx.x % 64;
  const int iters = group == 0 ? iters_a : iters_b;  // the groups run different trip counts
  unsigned acc = t;
  for (int i = 0; i < iters; ++i) {
    buf[group][t] = acc;                                   // write my slot
    if (full_barrier) __syncthreads(); else group_barrier(1 + group, 64);
    acc = acc * 1664525u + buf[group][(t + 17 + i) % 64];  // read another thread's slot
    if (full_barrier) __syncthreads(); else group_barrier(1 + group, 64);
  }
  out[threadIdx.x] = acc;
}

int main(int argc, char** argv) {
  const int full = argc > 1;  // any argument: same program with __syncthreads (equal trip counts)
  unsigned* d;
  cudaMalloc(&d, 128 * sizeof(unsigned));
  two_groups<<<1, 128>>>(d, 5, full ? 5 : 9, full);
  unsigned h[128];
  cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned sum = 0;
  for (unsigned v : h) sum = sum * 31u + v;
  printf("%s barrier: %s checksum %08x\n", full ? "__syncthreads" : "named", cudaGetErrorString(e), sum);
  return e != cudaSuccess;
}

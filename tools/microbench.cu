// Pipe-throughput microbenchmarks used to size the fp32-parity path:
// how many f32<->f64 conversions, DADD/DMUL and shared-memory ops per clock per SM
// does B200 sustain?  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CHECK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int kIters = 4096;
constexpr int kUnroll = 8;

template <int OP>
__global__ void __launch_bounds__(1024) pipe_kernel(float* out, float seed, long long* cycles) {
  float f[kUnroll];
  double d[kUnroll];
#pragma unroll
  for (int i = 0; i < kUnroll; ++i) { f[i] = seed + i + threadIdx.x; d[i] = seed * 1.5 + i + threadIdx.x; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kUnroll; ++i) {
      if (OP == 0) {        // widen + narrow pair (2 cvts)
        double x = (double)f[i];
        asm volatile("" : "+d"(x));
        f[i] = (float)(x) ;
        asm volatile("" : "+f"(f[i]));
      } else if (OP == 1) { // DADD
        d[i] = d[i] + 1.0000001;
      } else if (OP == 2) { // DMUL
        d[i] = d[i] * 1.0000001;
      } else if (OP == 3) { // FADD baseline
        f[i] = f[i] + 1.0000001f;
      } else if (OP == 4) { // integer widen (ALU) + hardware narrow
        uint32_t u = __float_as_uint(f[i]);
        uint32_t hi = (u & 0x80000000u) | (((u & 0x7fffffffu) >> 3) + 0x38000000u);
        uint32_t lo = u << 29;
        double x = __hiloint2double(hi, lo);
        x = x + 1.0;
        f[i] = (float)x;
      } else if (OP == 5) { // widen only (1 cvt) + dadd, accumulate in double
        d[i] = d[i] + (double)f[i];
        asm volatile("" : "+d"(d[i]));
      } else if (OP == 6) { // narrow only (1 cvt)
        f[i] = (float)d[i] ;
        asm volatile("" : "+f"(f[i]));
        d[i] = d[i] + 1.0;
      }
    }
  }
  long long t1 = clock64();
  float acc = 0;
#pragma unroll
  for (int i = 0; i < kUnroll; ++i) acc += f[i] + (float)d[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
int run(const char* name, double ops_per_inner, int sms) {
  float* out; long long* cyc;
  CHECK(cudaMalloc(&out, sizeof(float) * 1024 * sms));
  CHECK(cudaMalloc(&cyc, sizeof(long long) * sms));
  pipe_kernel<OP><<<sms, 1024>>>(out, 1.0f, cyc);
  CHECK(cudaDeviceSynchronize());
  pipe_kernel<OP><<<sms, 1024>>>(out, 1.0f, cyc);
  CHECK(cudaDeviceSynchronize());
  long long h[1024];
  CHECK(cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost));
  double c = 0; for (int i = 0; i < sms; ++i) c += h[i]; c /= sms;
  double lane_ops = (double)kIters * kUnroll * 1024 * ops_per_inner;
  printf("%-34s %8.1f lane-ops/clk/SM  (%.0f clk)\n", name, lane_ops / c, c);
  cudaFree(out); cudaFree(cyc);
  return 0;
}

int main() {
  cudaDeviceProp p; CHECK(cudaGetDeviceProperties(&p, 0));
  printf("%s, %d SMs\n", p.name, p.multiProcessorCount);
  int sms = p.multiProcessorCount;
  run<3>("FADD", 1, sms);
  run<1>("DADD", 1, sms);
  run<2>("DMUL", 1, sms);
  run<0>("cvt f32->f64 + cvt f64->f32 (pairs)", 1, sms);
  run<5>("cvt f32->f64 + DADD", 1, sms);
  run<6>("cvt f64->f32 + DADD", 1, sms);
  run<4>("ALU widen + DADD + cvt f64->f32", 1, sms);
  return 0;
}

// A/B of the two work decompositions for the min-sum node updates on a (6,3)-regular segment
// of [[784,24,24]] size (392 checks, 784 variables, 2352 edges), fp32 storage / fp64 arithmetic
// (the reference's float mode), messages in the product's shared-memory block layout:
//
//   A  THREAD PER NODE (what the library ships): one thread updates whole checks
//      (cn6_block: three 64-bit loads, a 13-operation min/max network, two scaled minima, three
//      64-bit stores) and whole variables (vn3_off), 160 threads per segment;
//   B  LANE PER EDGE with warp shuffles and __ballot_sync, as BASELINE.json's north star words
//      it: eight lanes per check (six active) find min1 / min2 with xor-butterfly shuffles and
//      the sign parity with a ballot; four lanes per variable (three active) gather the three
//      incoming messages with shuffles, sum them in edge order and decide by ballot.
//
// Both run `iters` iterations of (check stage, barrier, variable stage, barrier) on identical
// data with identical arithmetic; the final messages must be bit-identical (checked), and the
// program prints segment-iterations per second on the whole GPU for each.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2508_07879_b200/csrc \
//        -o tools/ab_lane_per_edge tools/ab_lane_per_edge.cu && tools/ab_lane_per_edge
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>
#include <numeric>
#include <random>

#include "kernel_lean.cuh"

using namespace qb;

constexpr uint32_t kM = 392, kN = 784, kE = 2352;
constexpr uint32_t kStride = Lay<ArithF32>::kStride, kR = Lay<ArithF32>::kROff;

#define CHECK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

// ---- A: thread per node -------------------------------------------------------------------
__global__ void __launch_bounds__(160, 6)
thread_per_node(const __grid_constant__ DecodeParams P, const uint32_t* var_edge_off /*[N][3]*/,
                const uint32_t* syn, const float* q0, uint32_t iters, float* out, uint32_t* dec) {
  extern __shared__ __align__(16) unsigned char msgs[];
  const uint32_t tid = threadIdx.x, T = blockDim.x;
  uint32_t eo[5][3], co[3], sb = 0, valid = 0;
  for (int k = 0; k < 5; ++k) {
    const uint32_t n = tid + k * T;
    const bool ok = n < kN;
    valid |= (ok ? 1u : 0u) << k;
    for (int i = 0; i < 3; ++i) eo[k][i] = ok ? var_edge_off[n * 3 + i] : kM * kStride + 4u * i;
  }
  for (int k = 0; k < 3; ++k) {
    const uint32_t m = tid + k * T;
    co[k] = (m < kM ? m : kM) * kStride;
    sb |= (m < kM ? (syn[m >> 5] >> (m & 31u)) & 1u : 0u) << k;
  }
  for (uint32_t e = tid; e < (kM + 1) * 14; e += T) reinterpret_cast<float*>(msgs)[e] = 0.f;
  __syncthreads();
  for (uint32_t e = tid; e < kE; e += T) *reinterpret_cast<float*>(msgs + (e / 6) * kStride + (e % 6) * 4) = q0[e];
  __syncthreads();
  uint32_t eb = 0;
  for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 3; ++k) cn6_block(P, ArithF32{}, msgs + co[k], (sb >> k) & 1u);
    __syncthreads();
    eb = 0;
#pragma unroll
    for (int k = 0; k < 5; ++k) eb |= vn3_off<true>(P, ArithF32{}, msgs, eo[k], 0.f) << k;
    __syncthreads();
  }
  eb &= valid;
  if (blockIdx.x == 0) {
    for (uint32_t e = tid; e < kE; e += T) {
      out[e] = *reinterpret_cast<float*>(msgs + (e / 6) * kStride + (e % 6) * 4);
      out[kE + e] = *reinterpret_cast<float*>(msgs + (e / 6) * kStride + kR + (e % 6) * 4);
    }
    for (int k = 0; k < 5; ++k) if ((valid >> k) & 1u) dec[tid + k * T] = (eb >> k) & 1u;
  }
}

// ---- B: lane per edge, shuffles + ballot ------------------------------------------------------
// 1024 threads: check stage = 8 lanes per check (4 checks per warp, 128 checks per pass, 4 passes
// cover 392 checks); variable stage = 4 lanes per variable (8 variables per warp, 256 per pass,
// 4 passes cover 784 variables).
template <int MINB>
__global__ void __launch_bounds__(1024, MINB)
lane_per_edge(const __grid_constant__ DecodeParams P, const uint32_t* var_edge_off, const uint32_t* syn,
              const float* q0, uint32_t iters, float* out, uint32_t* dec) {
  extern __shared__ __align__(16) unsigned char msgs[];
  const uint32_t tid = threadIdx.x, T = blockDim.x, lane = tid & 31u;
  const uint32_t cslot = lane & 7u, vslot = lane & 3u;
  for (uint32_t e = tid; e < (kM + 1) * 14; e += T) reinterpret_cast<float*>(msgs)[e] = 0.f;
  __syncthreads();
  for (uint32_t e = tid; e < kE; e += T) *reinterpret_cast<float*>(msgs + (e / 6) * kStride + (e % 6) * 4) = q0[e];
  // per-thread tables: 4 check passes, 4 variable passes
  uint32_t coff[4], csyn = 0, voff[4], vok = 0, cok = 0;
  for (int p = 0; p < 4; ++p) {
    const uint32_t m = (tid >> 3) + p * (T >> 3);
    const bool ok = m < kM && cslot < 6u;
    cok |= (ok ? 1u : 0u) << p;
    coff[p] = ok ? m * kStride + cslot * 4u : kM * kStride + (cslot % 6u) * 4u;
    csyn |= (m < kM ? (syn[m >> 5] >> (m & 31u)) & 1u : 0u) << p;
    const uint32_t n = (tid >> 2) + p * (T >> 2);
    const bool vk = n < kN && vslot < 3u;
    vok |= (vk ? 1u : 0u) << p;
    voff[p] = vk ? var_edge_off[n * 3 + vslot] : kM * kStride + (vslot % 3u) * 4u;
  }
  __syncthreads();
  uint32_t eb = 0;
  for (uint32_t it = 0; it < iters; ++it) {
    // ---- check stage: min1 / min2 by xor-butterfly over the 8-lane group, signs by ballot
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const float v = *reinterpret_cast<const float*>(msgs + coff[p]);
      const bool act = cslot < 6u;
      float m1 = act ? fabsf(v) : __uint_as_float(0x7f800000u), m2 = __uint_as_float(0x7f800000u);
#pragma unroll
      for (int d = 1; d < 8; d <<= 1) {  // merge (m1, m2) pairs: two smallest of the union
        const float o1 = __shfl_xor_sync(0xffffffffu, m1, d), o2 = __shfl_xor_sync(0xffffffffu, m2, d);
        const float lo = fminf(m1, o1), hi = fmaxf(m1, o1);
        m2 = fminf(hi, fminf(m2, o2));
        m1 = lo;
      }
      const uint32_t neg = __ballot_sync(0xffffffffu, act && v < 0.0f);
      const uint32_t grp = (neg >> (lane & ~7u)) & 0x3fu;
      const uint32_t par = (__popc(grp) + ((csyn >> p) & 1u)) & 1u;
      const float mine = fabsf(v) == m1 ? m2 : m1;  // tie: m2 == m1, as decoder.cpp:284-309 needs
      uint32_t r = __float_as_uint(static_cast<float>(P.alpha * static_cast<double>(mine)));
      r ^= (par ^ (v < 0.0f ? 1u : 0u)) << 31;
      if ((cok >> p) & 1u) *reinterpret_cast<uint32_t*>(msgs + coff[p] + kR) = r;
    }
    __syncthreads();
    // ---- variable stage: gather the three r over the 4-lane group, sum in edge order
    eb = 0;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const double r = static_cast<double>(*reinterpret_cast<const float*>(msgs + voff[p] + kR));
      const uint32_t base = lane & ~3u;
      const double r0 = __shfl_sync(0xffffffffu, r, base), r1 = __shfl_sync(0xffffffffu, r, base + 1),
                   r2 = __shfl_sync(0xffffffffu, r, base + 2);
      double total = P.gamma_d;
      total += r0;
      total += r1;
      total += r2;
      const float x = static_cast<float>(total - r);
      if ((vok >> p) & 1u) *reinterpret_cast<float*>(msgs + voff[p]) = x;
      const uint32_t d = __ballot_sync(0xffffffffu, total < 0.0);
      eb |= ((d >> base) & 1u) << p;
    }
    __syncthreads();
  }
  if (blockIdx.x == 0) {
    for (uint32_t e = tid; e < kE; e += T) {
      out[e] = *reinterpret_cast<float*>(msgs + (e / 6) * kStride + (e % 6) * 4);
      out[kE + e] = *reinterpret_cast<float*>(msgs + (e / 6) * kStride + kR + (e % 6) * 4);
    }
    for (int p = 0; p < 4; ++p) {
      const uint32_t n = (tid >> 2) + p * (T >> 2);
      if (n < kN && vslot == 0u) dec[n] = (eb >> p) & 1u;
    }
  }
}

int main(int argc, char** argv) {
  const uint32_t iters = argc > 1 ? atoi(argv[1]) : 2000;
  cudaDeviceProp prop;
  CHECK(cudaGetDeviceProperties(&prop, 0));
  // a random (6,3)-regular bipartite graph: 2352 edge sockets on the variable side, shuffled
  std::mt19937 rng(2508);
  std::vector<uint32_t> sockets(kE);
  for (uint32_t e = 0; e < kE; ++e) sockets[e] = e / 3;  // variable of socket e
  std::shuffle(sockets.begin(), sockets.end(), rng);     // edge e (check e / 6) -> variable
  std::vector<std::vector<uint32_t>> ve(kN);
  for (uint32_t e = 0; e < kE; ++e) ve[sockets[e]].push_back(e);
  std::vector<uint32_t> veo(kN * 3);
  for (uint32_t n = 0; n < kN; ++n) {
    std::sort(ve[n].begin(), ve[n].end());
    for (int i = 0; i < 3; ++i) veo[n * 3 + i] = (ve[n][i] / 6) * kStride + (ve[n][i] % 6) * 4;
  }
  std::vector<uint32_t> syn((kM + 31) / 32 + 1, 0);
  for (uint32_t m = 0; m < kM; ++m) if (rng() % 16 == 0) syn[m >> 5] |= 1u << (m & 31u);
  std::vector<float> q0(kE, 1.0f);
  DecodeParams P{};
  P.alpha = 0.8;
  P.gamma_d = 1.0;
  P.gamma_f = 1.0f;
  P.clamp_f = 1e30f;
  uint32_t *d_veo, *d_syn, *d_dec;
  float *d_q0, *d_out;
  CHECK(cudaMalloc(&d_veo, veo.size() * 4));
  CHECK(cudaMalloc(&d_syn, syn.size() * 4));
  CHECK(cudaMalloc(&d_q0, kE * 4));
  CHECK(cudaMalloc(&d_out, 2 * kE * 4));
  CHECK(cudaMalloc(&d_dec, kN * 4));
  CHECK(cudaMemcpy(d_veo, veo.data(), veo.size() * 4, cudaMemcpyHostToDevice));
  CHECK(cudaMemcpy(d_syn, syn.data(), syn.size() * 4, cudaMemcpyHostToDevice));
  CHECK(cudaMemcpy(d_q0, q0.data(), kE * 4, cudaMemcpyHostToDevice));
  const size_t smem = (kM + 1) * kStride;
  CHECK(cudaFuncSetAttribute(thread_per_node, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CHECK(cudaFuncSetAttribute(lane_per_edge<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CHECK(cudaFuncSetAttribute(lane_per_edge<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> outA(2 * kE), outB(2 * kE);
  std::vector<uint32_t> decA(kN), decB(kN);
  auto run = [&](int which, std::vector<float>& out, std::vector<uint32_t>& dec, unsigned grid, const char* name) {
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (which == 0) thread_per_node<<<grid, 160, smem>>>(P, d_veo, d_syn, d_q0, iters, d_out, d_dec);
      else if (which == 1) lane_per_edge<1><<<grid, 1024, smem>>>(P, d_veo, d_syn, d_q0, iters, d_out, d_dec);
      else lane_per_edge<2><<<grid, 1024, smem>>>(P, d_veo, d_syn, d_q0, iters, d_out, d_dec);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms);
    }
    cudaMemcpy(out.data(), d_out, 2 * kE * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(dec.data(), d_dec, kN * 4, cudaMemcpyDeviceToHost);
    const double segit = (double)grid * iters / (best * 1e-3);
    printf("%-40s grid %4u  %8.3f ms  %8.1f M segment-iterations/s  (%.2f T edge-updates/s)\n", name, grid, best,
           segit / 1e6, segit * kE / 1e12);
    return segit;
  };
  printf("%s, %d SMs, %u iterations per CTA\n", prop.name, prop.multiProcessorCount, iters);
  const double a = run(0, outA, decA, prop.multiProcessorCount * 6, "A thread per node (160 thr, 6 CTAs/SM)");
  const double b1 = run(1, outB, decB, prop.multiProcessorCount, "B lane per edge (1024 thr, 1 CTA/SM, <=64 regs)");
  bool same = std::memcmp(outA.data(), outB.data(), 2 * kE * 4) == 0 && decA == decB;
  const double b2 = run(2, outB, decB, prop.multiProcessorCount * 2, "B lane per edge (1024 thr, 2 CTAs/SM, <=32 regs)");
  same = same && std::memcmp(outA.data(), outB.data(), 2 * kE * 4) == 0 && decA == decB;
  printf("final q, r and decisions identical: %s\n", same ? "yes" : "NO");
  printf("A / best B = %.2f\n", a / std::max(b1, b2));
  return same ? 0 : 2;
}

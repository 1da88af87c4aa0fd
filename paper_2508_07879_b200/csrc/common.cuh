// Shared device-side definitions for the sm_100a min-sum decoder kernels.
//
// Terminology follows the reference's domain (proj/src/decoder.cpp): a SHOT is
// one syndrome to decode; a SEGMENT is an independent block of the Tanner
// graph (1 for a plain graph, 2 = X and Z for a CssCode); q are
// variable->check messages, r are check->variable messages, gamma the priors.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace qb {

constexpr int kMaxSegments = 8;
constexpr int kWarp = 32;
constexpr uint32_t kNoAbsorb = 0xffu;
constexpr uint32_t kPadEdges = 8;  // message slots of the dummy check (regular kernel)

struct SegmentDev {
  uint32_t c0, c1;  // checks [c0, c1)
  uint32_t v0, v1;  // variables [v0, v1)
  uint32_t e0, e1;  // edges [e0, e1) (check-major numbering => contiguous)
};

// Everything a kernel needs to know about one decoder (code tables + config).
// Passed by value as a kernel parameter (__grid_constant__), so it sits in
// constant bank 0 and costs no loads from global memory.
struct DecodeParams {
  uint32_t M, N, E, nseg;
  uint32_t seg_emax;  // edges of the largest segment
  uint32_t seg_mmax;  // checks of the largest segment
  uint32_t seg_nmax;  // variables of the largest segment
  uint32_t syn_w32;  // 2 * ceil(M / 64): 32-bit words per packed syndrome
  uint32_t est_w32;  // 2 * ceil(N / 64): 32-bit words per packed estimate
  uint32_t max_iter;
  int32_t early;
  uint32_t ngroups;        // warp groups per CTA (<= nseg)
  uint32_t group_threads;  // threads per group, multiple of 32
  // arithmetic constants
  double alpha;       // float mode: fp64 multiply, one rounding (decoder.cpp:302-307)
  float alpha_f;      // (unused by the kernels; kept for diagnostics)
  uint16_t alpha_h;   // half mode: half(alpha)
  uint16_t deg1_h;    // half mode: half(alpha * 64)
  uint16_t gamma_hb;  // half mode, uniform prior: half(clamp(gamma))
  uint16_t it1_h;     // half mode, uniform prior: alpha_h * |gamma_h|
  float deg1_f;       // float(alpha * 64)           (decoder.cpp:256)
  float clamp_f;      // float(1e30)                 (decoder.cpp:23, :238-241)
  uint32_t alpha_fx;  // lround(alpha * 65536)       (decoder.cpp:89)
  int32_t kmax;       // 127 / 32767                 (decoder.cpp:50, :59)
  int32_t deg1_i;     // scale_q16(kmax)             (decoder.cpp:253)
  // uniform-prior fast path (every gamma equal; fp32 additionally proven clamp-free)
  double gamma_d;     // (double)float(gamma)
  float gamma_f;      // integer modes: float(gamma_i) (ArithI16F kernels)
  int32_t gamma_i;
  float kmax_f;       // float(kmax)
  // first-iteration constants of the uniform-prior path: every check sends +-S
  double it1_d;     // fp32 mode: (double)float(alpha * |gamma|)
  int32_t it1_i;    // int modes: scale_q16(|gamma|)
  uint32_t it1_neg; // 1 when gamma < 0 (its sign multiplies every first message)
  // ... as a TABLE (fp32 / whole-word integer batch kernels): with a uniform prior the message
  // a variable sends after the first iteration depends only on how many of its OTHER two
  // checks have syndrome bit 1 (it1_tq[0..2], raw message words), and its decision only on
  // how many of its three checks do (bit 4k of it1_dec4, k = 0..3).  The loader computes the
  // entries with the reference's own operation sequence for all eight syndrome patterns and
  // only enables the FAST instantiations of those kernels if every pattern agrees.
  uint32_t it1_tq[3];
  uint32_t it1_dec4;
  // CSR tables (device global memory, read-only)
  const uint32_t* check_off;   // [M + 1]
  const uint32_t* var_off;     // [N + 1]
  const uint32_t* var_edges;   // [E]
  const uint32_t* edge_var;    // [E]
  const uint32_t* edge_check;  // [E]
  const void* gamma;           // [N] float (float/half modes) or int32 (int modes)
  // degree-padded kernel (kernel_ell.cuh): variables a thread updates, and the degree-1
  // variables ABSORBED by their check (updated by the check's thread)
  const uint32_t* ell_vars;    // [N]: segment s lists its ell_nvars[s] own variables from index segs[s].v0
  const uint32_t* ell_abs;     // [M]: slot of the absorbed variable in check m's block, or kNoAbsorb
  uint32_t ell_nvars[kMaxSegments];
  // lean batch kernels ((6,3)-regular codes): slot of edge e inside its check's message
  // block - a permutation of 0..5 per check chosen by the loader to spread the variable-side
  // accesses of a warp over the banks (the check update is symmetric in its slots)
  const uint8_t* edge_slot;    // [E]
  SegmentDev segs[kMaxSegments];
};

// Per-launch I/O description.  All pointers are device-accessible (device
// memory, or mapped pinned host memory on the single-shot path).
struct ShotIO {
  uint64_t nshots;
  const uint32_t* syn;  // [nshots][syn_w32]
  uint32_t* est;        // [nshots][est_w32]
  uint32_t* resid;      // [nshots][syn_w32] or nullptr
  uint8_t* conv;        // [nshots][nseg]
  uint32_t* iters;      // [nshots][nseg]
  unsigned int* sched;  // [0] next-shot ticket, [1] finished-CTA count, [2+s] per-segment tickets
  // single-shot completion (nullptr on the batch path)
  uint64_t* kernel_ns;       // %globaltimer span, written before the flag
  volatile uint32_t* flag;   // receives `seq` after every result is visible
  uint32_t seq;
  uint32_t tile;  // lean batch kernel: shots per syndrome tile (one bulk copy, one queue ticket)
  // debug dumps of the final edge messages (nullptr unless qb_decode_debug)
  void* q_dump;
  void* r_dump;
  // per-shot priors of the absorbed degree-1 variables ("soft syndromes", kernel_ell.cuh):
  // [nshots][M] float (float / half modes), int8 (int8) or int16 (int16); nullptr = none
  const void* soft;
  uint32_t soft_bytes;  // element size of `soft`: 4, 1 or 2
  // batch kernels: also dump the messages of shot `dump_shot` to q_dump / r_dump
  uint32_t dump_shot;
};

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---- TMA bulk copy (cp.async.bulk, global -> shared) completing on an mbarrier ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// bytes: multiple of 16; dst and src 16-byte aligned
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Named barrier over one warp group (ids 1..15; id 0 is __syncthreads()).
__device__ __forceinline__ void group_barrier(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Bits i of 32-bit word w whose global index 32*w + i lies in [lo, hi).
__device__ __forceinline__ uint32_t range_mask(uint32_t w, uint32_t lo, uint32_t hi) {
  const uint32_t base = w * 32u;
  if (hi <= base || lo >= base + 32u) return 0u;
  const uint32_t a = lo > base ? lo - base : 0u;
  const uint32_t b = hi < base + 32u ? hi - base : 32u;
  const uint32_t upto_b = b >= 32u ? 0xffffffffu : ((1u << b) - 1u);
  const uint32_t below_a = (1u << a) - 1u;  // a < 32 here
  return upto_b & ~below_a;
}

// ---------------------------------------------------------------------------
// Arithmetic traits.  Each mode defines the stored message type, the prior
// type, and the two node updates' scalar pieces.
// ---------------------------------------------------------------------------

struct ArithF32 {
  using Msg = float;
  using Gam = float;
  static constexpr bool kInt = false;
};
struct ArithF16 {
  using Msg = __half;
  using Gam = float;
  static constexpr bool kInt = false;
};
struct ArithI8 {
  using Msg = int8_t;
  using Gam = int32_t;
  static constexpr bool kInt = true;
};
struct ArithI16 {
  using Msg = int16_t;
  using Gam = int32_t;
  static constexpr bool kInt = true;
};

// Integer modes with messages held in 32-bit words (degree-padded kernel): same arithmetic
// as int8 / int16 - the saturation bound is DecodeParams::kmax - without the sub-word
// packing and sign-extension instructions, which dominate the ALU-bound integer kernels.
struct ArithI32 {
  using Msg = int32_t;
  using Gam = int32_t;
  static constexpr bool kInt = true;
};

// The reference's INT16 mode on fp32 INSTRUCTIONS (lean batch kernels): every quantity of that
// mode is an integer of magnitude <= 4 * 32767 < 2^24, which fp32 represents exactly, so sums
// (FADD), saturation and the minimum network (FMNMX) and comparisons are exact in fp32
// arithmetic - and the additions run on the FMA pipe instead of the ALU pipe that bounds the
// integer kernels.  Messages are stored as fp32 integers.  The Q16 scaling stays an integer
// multiply: adding 2^23 puts the magnitude into the low mantissa bits, one IMAD evaluates
// (mag * alpha_fx + 32768) on the bit pattern (the exponent's contribution is folded into the
// addend, arithmetic mod 2^32), a shift and the same trick backwards return the float.
struct ArithI16F {
  using Msg = float;
  using Gam = float;
  static constexpr bool kInt = true;  // reference semantics: integer mode (dumps are int32)
};

// Q16 scaling of a non-negative magnitude (decoder.cpp:226-229).  mag <= 32767
// and alpha_fx <= 65536, so the product fits 32 unsigned bits.
__device__ __forceinline__ int32_t scale_q16(uint32_t mag, uint32_t alpha_fx) {
  return static_cast<int32_t>((mag * alpha_fx + 32768u) >> 16);
}

// Half mode (an extension without a reference counterpart): fp16 storage AND fp16
// arithmetic, so that the batch kernel can run two shots per thread in the two
// lanes of a half2 with results identical, lane by lane, to the scalar kernels:
//   gamma_h = half(clamp(gamma));  r = +-(alpha_h * |q|min)   (one fp16 multiply)
//   total = ((gamma_h + r0) + r1) + r2   (fp16 adds, ascending edge order)
//   q = clamp(total - r_e) to +-60000 (keeps stored messages finite, the analogue
//   of the reference's 1e30 clamp);  decision = sign bit of total.
constexpr float kHalfClamp = 60000.0f;

__device__ __forceinline__ __half h_clamp(__half x) {
  const __half c = __ushort_as_half(0x7b53);  // 60000
  return __hmax(__hmin(x, c), __hneg(c));
}
__device__ __forceinline__ __half2 h2_clamp(__half2 x) {
  const __half2 c = __half2half2(__ushort_as_half(0x7b53));
  return __hmax2(__hmin2(x, c), __hneg2(c));
}
__device__ __forceinline__ bool h_neg(__half x) { return (__half_as_ushort(x) & 0x8000u) != 0; }

}  // namespace qb

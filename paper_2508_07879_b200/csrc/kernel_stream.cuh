// Throughput kernel for regular (6,3) codes: continuous batching of
// (shot, segment) work items over K message SLOTS per CTA.
//
// A persistent CTA serves one segment of the code (its per-thread edge tables
// sit in registers for the whole launch) and keeps K shots in flight, each in
// its own slot of shared memory.  Time advances in HALF-STEPS separated by one
// __syncthreads(); in a half-step every slot runs whichever stage it is due:
//
//     CN-step   (test the parity bitmap left by the previous VN stage; if the
//               shot is finished: write its results, take the next shot from
//               the segment's queue and initialise it - else) check-node stage
//     VN-step   variable-node stage + parity toggles
//
// so ONE barrier covers a stage of K different shots (2/K barriers per
// shot-iteration instead of 2), a finished shot is replaced immediately instead
// of idling until its CTA-mates converge, and the instruction streams of the K
// slots give each warp independent work to overlap shared-memory latency.
//
// Streaming: the next shot's packed syndrome is prefetched global->shared with
// cp.async one turnover ahead, so no thread ever waits on HBM inside the loop;
// hard decisions leave the kernel as sparse atomic ORs into estimate words that
// the CTA zeroed when it accepted the shot (a shot has a handful of set bits),
// the residual as shifted parity words.  Words that straddle the boundary
// between two segments are only ever modified with bit-masked atomics, so the X
// and Z halves of a shot can be decoded by different CTAs in any order.
//
// Bit vectors are kept SEGMENT-LOCAL in shared memory (bit i = check c0 + i), so
// the loop needs no boundary masks; they are shifted back to the reference's
// packed layout on the way out.  Arithmetic = kernel_regular.cuh (bit-exact).
#pragma once

#include "common.cuh"
#include "kernel_regular.cuh"

namespace qb {

__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gmem_src) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// Shared-memory footprint: per slot two message arrays of the largest segment
// (+ dummy check), local syndrome + two parity bitmaps, the prefetch stage.
__host__ __device__ inline uint32_t stream_pw(uint32_t seg_mmax) { return (seg_mmax >> 5) + 2; }

__host__ __device__ inline size_t stream_smem_bytes(uint32_t seg_emax, uint32_t seg_mmax,
                                                    size_t msg_bytes, int slots) {
  const size_t msg = (static_cast<size_t>(seg_emax + kPadEdges) * msg_bytes + 15) & ~size_t(15);
  const size_t words = 4 * static_cast<size_t>(stream_pw(seg_mmax)) + 4;  // syn, par0, par1, stage
  return static_cast<size_t>(slots) * (2 * msg + 4 * words) + 64;
}

template <class A>
struct StreamSlot {
  typename A::Msg* q;
  typename A::Msg* r;
  uint32_t* syn;    // [pw] local syndrome bits
  uint32_t* par0;   // [pw]
  uint32_t* par1;   // [pw]
  uint32_t* stage;  // [pw + 1] raw global syndrome words of the NEXT shot
};

constexpr uint32_t kNoShot = 0xffffffffu;

template <class A, int CPT, int VPT, bool kFast, int K, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB)
decode_stream_kernel(const __grid_constant__ DecodeParams P, const __grid_constant__ ShotIO io) {
  using Msg = typename A::Msg;
  using Gam = typename A::Gam;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t tid = threadIdx.x, T = blockDim.x, lane = tid & 31u;
  const uint32_t nseg = P.nseg;
  const uint32_t s = blockIdx.x % nseg;          // the segment this CTA serves
  const uint32_t peer = blockIdx.x / nseg;       // its index among the CTAs of that segment
  const uint32_t peers = (gridDim.x - s + nseg - 1) / nseg;
  const SegmentDev seg = P.segs[s];
  const uint32_t Ms = seg.c1 - seg.c0;
  const uint32_t pw = stream_pw(P.seg_mmax);     // words per local bit array
  const uint32_t pws = (Ms + 31u) >> 5;          // words that hold this segment's checks
  const uint32_t gw0 = seg.c0 >> 5;              // first global syndrome word of the segment
  const uint32_t gspan = ((seg.c1 - 1) >> 5) - gw0 + 1;
  const uint32_t cshift = seg.c0 & 31u;
  const uint32_t vw0 = seg.v0 >> 5, vspan = ((seg.v1 - 1) >> 5) - vw0 + 1;

  // ---- carve shared memory
  StreamSlot<A> slot[K];
  {
    const size_t msg = (static_cast<size_t>(P.seg_emax + kPadEdges) * sizeof(Msg) + 15) & ~size_t(15);
    unsigned char* p = smem_raw;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      slot[k].q = reinterpret_cast<Msg*>(p);
      slot[k].r = reinterpret_cast<Msg*>(p + msg);
      p += 2 * msg;
    }
    uint32_t* w = reinterpret_cast<uint32_t*>(p);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      slot[k].syn = w;
      slot[k].par0 = w + pw;
      slot[k].par1 = w + 2 * pw;
      slot[k].stage = w + 3 * pw;
      w += 4 * pw + 4;
    }
  }
  __shared__ uint32_t next_ticket[K];

  RegTables<A, CPT, VPT, kFast> tab;
  load_tables<A, CPT, VPT, kFast>(P, seg, tid, T, tab, seg.e0, P.seg_emax);
  // local check index of each check slot (dummy check: bit Ms, always 0)
  uint32_t cloc[CPT];
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const uint32_t m = seg.c0 + tid + k * T;
    cloc[k] = m < seg.c1 ? m - seg.c0 : Ms;
  }

  // ---- per-slot state (CTA-uniform except ebits / synbits)
  uint32_t cur[K], nxt[K], iter[K], ebits[K], synbits[K], pbuf[K];
  bool vn_due[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    cur[k] = kNoShot;
    const uint64_t first = static_cast<uint64_t>(peer) * K + k;
    nxt[k] = first < io.nshots ? static_cast<uint32_t>(first) : kNoShot;
    iter[k] = 0;
    ebits[k] = 0;
    synbits[k] = 0;
    pbuf[k] = 0;
    vn_due[k] = false;
    if (tid < kPadEdges) {
      slot[k].q[P.seg_emax + tid] = static_cast<Msg>(0);
      slot[k].r[P.seg_emax + tid] = static_cast<Msg>(0);
    }
    for (uint32_t w = tid; w < 4 * pw + 4; w += T) slot[k].syn[w] = 0;
  }
  __syncthreads();
  // prefetch the first shots' syndromes
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (nxt[k] != kNoShot && tid < gspan) {
      cp_async4(&slot[k].stage[tid], io.syn + static_cast<uint64_t>(nxt[k]) * P.syn_w32 + gw0 + tid);
    }
  }
  cp_async_wait_all();
  __syncthreads();

  const uint32_t ticket_base = peers * K;
  for (;;) {
    bool any_live = false;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const StreamSlot<A>& sl = slot[k];
      if (vn_due[k]) {
        // ================= VN-step =================
        uint32_t* par = pbuf[k] ? sl.par1 : sl.par0;
        uint32_t eb = 0;
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
          Gam g{};
          if constexpr (!kFast) g = tab.gamma[v];
          eb |= vn3<kFast>(P, sl.q, sl.r, tab.ea[v], g) << v;
        }
        eb &= tab.valid;
        ebits[k] = eb;
        if (eb) {  // rare: a variable of this thread currently decides 1
#pragma unroll
          for (int v = 0; v < VPT; ++v) {
            if ((eb >> v) & 1u) {
#pragma unroll
              for (int i = 0; i < kDV; ++i) {
                const uint32_t lm = tab.ea[v][i] / kDC;
                atomicXor(&par[lm >> 5], 1u << (lm & 31u));
              }
            }
          }
        }
        vn_due[k] = false;
        any_live = true;
        continue;
      }
      // ================= CN-step =================
      bool finished = cur[k] == kNoShot;  // empty slot: go straight to turnover
      if (!finished && iter[k] > 0) {
        const uint32_t* par = pbuf[k] ? sl.par1 : sl.par0;
        uint32_t acc = 0;
        for (uint32_t w = lane; w < pws; w += 32u) acc |= par[w];
        const bool unsat = __any_sync(0xffffffffu, acc != 0u);
        finished = (P.early && !unsat) || iter[k] >= P.max_iter;
        if (finished) {
          // ---- results of shot cur[k]: residual words, flags, sparse estimate bits
          const uint64_t shot = cur[k];
          if (io.resid && tid < gspan) {
            // global word gw0 + tid holds local bits [32*tid - cshift, +32)
            const uint32_t hi = par[tid];
            const uint32_t lo = tid > 0 ? par[tid - 1] : 0u;
            const uint32_t bits = cshift ? __funnelshift_l(lo, hi, cshift) : hi;
            uint32_t* dst = io.resid + shot * P.syn_w32 + gw0 + tid;
            const uint32_t mask = range_mask(gw0 + tid, seg.c0, seg.c1);
            if (mask == 0xffffffffu) {
              *dst = bits;
            } else {
              atomicAnd(dst, ~mask);
              atomicOr(dst, bits & mask);
            }
          }
          if (ebits[k]) {
            uint32_t* est_g = io.est + shot * P.est_w32;
#pragma unroll
            for (int v = 0; v < VPT; ++v) {
              if ((ebits[k] >> v) & 1u) {
                const uint32_t n = seg.v0 + tid + v * T;
                atomicOr(&est_g[n >> 5], 1u << (n & 31u));
              }
            }
          }
          if (tid == 0) {
            io.conv[shot * nseg + s] = unsat ? 0 : 1;
            io.iters[shot * nseg + s] = iter[k];
          }
        }
      }
      if (finished) {
        // ---- turnover: accept shot nxt[k] (its syndrome is already staged)
        cur[k] = nxt[k];
        iter[k] = 0;
        if (cur[k] == kNoShot) continue;  // queue exhausted: the slot stays empty
        any_live = true;
        const uint64_t shot = cur[k];
        if (tid < pw) {
          // local word tid = global bits [c0 + 32*tid, +32)
          uint32_t v = 0;
          if (tid < pws) {
            const uint32_t a = sl.stage[tid];
            const uint32_t b = tid + 1 < gspan ? sl.stage[tid + 1] : 0u;
            v = cshift ? __funnelshift_r(a, b, cshift) : a;
            const uint32_t left = Ms - tid * 32u;
            if (left < 32u) v &= (1u << left) - 1u;
          }
          sl.syn[tid] = v;
          // bitmap of iteration 1 goes to the buffer that was NOT just tested: slower
          // warps of this CTA may still be reading the other one for their vote
          (pbuf[k] ? sl.par0 : sl.par1)[tid] = v;
        }
        pbuf[k] ^= 1u;
        if (tid < vspan) {  // zero this segment's estimate bits of the shot
          uint32_t* dst = io.est + shot * P.est_w32 + vw0 + tid;
          const uint32_t mask = range_mask(vw0 + tid, seg.v0, seg.v1);
          if (mask == 0xffffffffu) {
            *dst = 0u;
          } else {
            atomicAnd(dst, ~mask);
          }
        }
        // q[e] = gamma[var(e)] (decoder.cpp:156-158)
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
          Gam g;
          if constexpr (kFast) {
            if constexpr (A::kInt) g = P.gamma_i; else g = P.gamma_f;
          } else {
            g = tab.gamma[v];
          }
          const Msg init = prior_as_msg<A>(g);
#pragma unroll
          for (int i = 0; i < kDV; ++i) sl.q[tab.ea[v][i]] = init;
        }
        if (tid == 0) {
          const uint64_t t = static_cast<uint64_t>(atomicAdd(&io.sched[2 + s], 1u)) + ticket_base;
          next_ticket[k] = t < io.nshots ? static_cast<uint32_t>(t) : kNoShot;
        }
        nxt[k] = kNoShot - 1u;  // "read the ticket after the next barrier"
        continue;               // the CN stage of the new shot runs in the next half-step
      }
      // ---- normal CN stage of iteration iter+1
      if (nxt[k] == kNoShot - 1u) {
        // first half-step after a turnover: pick up the ticket, start the prefetch
        nxt[k] = next_ticket[k];
        if (nxt[k] != kNoShot && tid < gspan) {
          cp_async4(&sl.stage[tid],
                    io.syn + static_cast<uint64_t>(nxt[k]) * P.syn_w32 + gw0 + tid);
        }
        // this thread's syndrome bits of the new shot
        uint32_t sb = 0;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
          sb |= ((sl.syn[cloc[c] >> 5] >> (cloc[c] & 31u)) & 1u) << c;
        }
        synbits[k] = sb;
      }
      if (iter[k] > 0) {  // (a fresh shot's bitmap was preset at turnover)
        pbuf[k] ^= 1u;
        uint32_t* par_next = pbuf[k] ? sl.par1 : sl.par0;
        if (tid < pws) par_next[tid] = sl.syn[tid];
      }
      ++iter[k];
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        cn6<kFast>(P, sl.q, sl.r, tab.ce[c], (synbits[k] >> c) & 1u);
      }
      vn_due[k] = true;
      any_live = true;
    }
    if (!any_live) break;
    cp_async_wait_all();
    __syncthreads();
  }

  if (tid == 0) {
    __threadfence();
    const unsigned int done = atomicAdd(&io.sched[1], 1u);
    if (done == gridDim.x - 1) {
      for (uint32_t k = 0; k < 2 + kMaxSegments; ++k) io.sched[k] = 0;
      __threadfence();
    }
  }
}

}  // namespace qb

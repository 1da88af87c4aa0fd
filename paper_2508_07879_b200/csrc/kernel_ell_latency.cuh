// Single-shot latency kernel for IRREGULAR graphs: the degree-padded node updates of
// kernel_ell.cuh (sentinel-padded check blocks, zero-block variable slots, degree-1 variables
// absorbed by their checks) inside the single-shot protocol of decode_lean_latency_kernel
// (kernel_lean.cuh): one thread-block cluster per shot, CTA rank = segment, one check and two
// variables per thread; the syndrome arrives by value in the kernel parameters, from memory,
// or through the persistent DOORBELL, and every CTA publishes a sectored record of its
// segment-local estimate / residual words, so neither a memcpy nor a stream synchronisation
// nor a device atomic on shared result words sits on the critical path.  This is what BASELINE
// config 5's single shots (extended graphs diag([Hz | I], [Hx | I])) run on; before it they
// took decode_ell_kernel through the copy protocol (H2D, kernel, D2H: 27-30 us).
#pragma once

#include "common.cuh"
#include "kernel_ell.cuh"
#include "kernel_lean.cuh"

namespace qb {

__host__ __device__ inline size_t ell_latency_smem_bytes(uint32_t seg_mmax, uint32_t seg_nmax,
                                                         uint32_t msg_bytes, uint32_t dc,
                                                         uint32_t threads) {
  return ell_msg_region_bytes(seg_mmax, ell_stride_bytes(msg_bytes, dc), threads, dc) +
         4 * (static_cast<size_t>(ell_pw(seg_mmax)) + lean_pw(seg_nmax) + 8);
}

template <class A, int DC, int DV>
__global__ void __launch_bounds__(1024, 1)
decode_ell_latency_kernel(const __grid_constant__ DecodeParams P, const __grid_constant__ ShotIO io,
                          const __grid_constant__ LatencyCtl ctl,
                          const __grid_constant__ SynInline syn_in) {
  static_assert(DV <= DC, "padded variable slots live in the q half of the zero block");
  using Msg = typename A::Msg;
  using Gam = typename A::Gam;
  constexpr int VPT = 2;
  constexpr uint32_t kMsg = static_cast<uint32_t>(sizeof(Msg));
  const uint32_t kStride = ell_stride_bytes(kMsg, DC);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t tid = threadIdx.x, T = blockDim.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t nseg = P.nseg;
  const uint32_t s = cluster.block_rank();  // == segment
  const SegmentDev seg = P.segs[s];
  const uint32_t Ms = seg.c1 - seg.c0, Ns = seg.v1 - seg.v0;
  const uint32_t pw = ell_pw(P.seg_mmax);
  const uint32_t ew = lean_pw(P.seg_nmax);
  const uint32_t pws = (Ms + 31u) >> 5, ews = (Ns + 31u) >> 5;
  const uint32_t gw0 = seg.c0 >> 5, gspan = ((seg.c1 - 1) >> 5) - gw0 + 1, cshift = seg.c0 & 31u;

  unsigned char* const msgs = smem_raw;
  const size_t msg_bytes = ell_msg_region_bytes(P.seg_mmax, kStride, T, DC);
  uint32_t* const bits = reinterpret_cast<uint32_t*>(smem_raw + msg_bytes);
  uint32_t* const par = bits;                       // [pw]
  uint32_t* const ehat = bits + pw;                 // [ew]
  volatile uint32_t* const unsat = bits + pw + ew;  // [1]
  volatile uint32_t* const exit_word = bits + pw + ew + 1;
  uint32_t* const cmd_word = bits + pw + ew + 2;
  const uint32_t scratch_off = P.seg_mmax * kStride;  // first dummy block (ell_dummy_blocks)
  const uint32_t pad_off = scratch_off + (tid / DC) * kStride + (tid % DC) * kMsg;
  for (uint32_t b = tid; b < (ell_dummy_blocks(T, DC) + 1u) * kStride; b += T) msgs[scratch_off + b] = 0;

  // ---- per-thread tables (decode_ell_kernel with one check, two variables per thread)
  uint32_t eo[VPT][DV], valid = 0, keep0 = 0, vloc[VPT];
  Gam gam[VPT];
  const uint32_t nv = P.ell_nvars[s];
  const Gam* __restrict__ gamma = static_cast<const Gam*>(P.gamma);
#pragma unroll
  for (int k = 0; k < VPT; ++k) {
    const uint32_t idx = tid + k * T;
    const bool ok = idx < nv;
    const uint32_t n = ok ? P.ell_vars[seg.v0 + idx] : seg.v0;
    const uint32_t b = ok ? P.var_off[n] : 0u;
    const uint32_t deg = ok ? P.var_off[n + 1] - b : 0u;
    valid |= (ok ? 1u : 0u) << k;
    keep0 |= (deg == 1u ? 1u : 0u) << k;
    vloc[k] = n - seg.v0;
#pragma unroll
    for (int i = 0; i < DV; ++i) {
      uint32_t off = pad_off;
      if (static_cast<uint32_t>(i) < deg) {
        const uint32_t e = P.var_edges[b + i];
        const uint32_t m = P.edge_check[e];
        off = (m - seg.c0) * kStride + (e - P.check_off[m]) * kMsg;
      }
      eo[k][i] = off;
    }
    gam[k] = ok ? gamma[n] : static_cast<Gam>(1);
  }
  const bool has_check = tid < Ms;
  const uint32_t cl = has_check ? tid : Ms;  // dummy check: bit Ms of the bitmap, always 0
  const uint32_t co = has_check ? tid * kStride : scratch_off + ell_dummy_blocks(T, DC) * kStride;
  uint32_t aslot = kNoAbsorb, aloc = 0;
  if (has_check) {
    const uint32_t e0 = P.check_off[seg.c0 + tid];
    const uint32_t deg = P.check_off[seg.c0 + tid + 1] - e0;
    const Msg sent = deg == 1u ? EllSentinel<A>::deg1(P) : EllSentinel<A>::pad(P);
#pragma unroll
    for (int j = 0; j < DC; ++j) {
      if (static_cast<uint32_t>(j) >= deg) *reinterpret_cast<Msg*>(msgs + co + j * kMsg) = sent;
    }
    aslot = P.ell_abs[seg.c0 + tid];
    if (aslot != kNoAbsorb) {
      const uint32_t n = P.edge_var[e0 + aslot];
      *reinterpret_cast<Msg*>(msgs + co + aslot * kMsg) = prior_as_msg<A>(gamma[n]);
      aloc = n - seg.v0;
    }
  }
  if (tid == 0) *exit_word = 0u;
  __syncthreads();
  if (ctl.mode == 2u) cluster.sync();

  uint32_t* const rec = ctl.rec + s * ctl.rec_stride;
  const uint32_t ndata = ews + pws + 4u;
  const uint32_t nrec = sector_words(ndata);
  uint32_t last = ctl.first_seq - 1u;
  uint64_t t_idle0 = globaltimer_ns();
  for (;;) {
    // ---------------- obtain the shot (as decode_lean_latency_kernel) ----------------
    uint32_t cmd = last + 1u;
    uint32_t raw = 0;
    uint64_t t_begin = 0;
    if (warp == 0) {
      if (ctl.mode == 2u) {
        uint32_t spins = 0, val = 0;
        for (;;) {
          val = ld_volatile_global(ctl.doorbell + lane);
          const uint32_t sq = __shfl_sync(0xffffffffu, val, lane & ~7u);
          if (__all_sync(0xffffffffu, sq == cmd)) break;
          if (__any_sync(0xffffffffu, sq == kDoorbellExit) || *exit_word != 0u) {
            cmd = kDoorbellExit;
            break;
          }
          if (s == 0 && (++spins & 63u) == 0u && globaltimer_ns() - t_idle0 > ctl.idle_ns) {
            if (lane < nseg) *cluster.map_shared_rank(const_cast<uint32_t*>(exit_word), lane) = 1u;
            cmd = kDoorbellExit;
            break;
          }
        }
        const uint32_t src = lane < gspan ? sector_pos(gw0 + lane) : 0u;
        raw = __shfl_sync(0xffffffffu, val, src & 31u);
      } else if (lane < gspan) {
        raw = ctl.mode == 0u ? syn_in.w[gw0 + lane] : io.syn[gw0 + lane];
      }
      if (lane >= gspan) raw = 0;
      t_begin = globaltimer_ns();
      if (lane == 0) {
        cmd_word[0] = cmd;
        cmd_word[1] = static_cast<uint32_t>(t_begin);
        cmd_word[2] = static_cast<uint32_t>(t_begin >> 32);
      }
      // packed syndrome words -> segment-local bitmap, and its population count
      uint32_t nb = __shfl_down_sync(0xffffffffu, raw, 1);
      if (lane + 1 >= gspan) nb = 0;
      uint32_t loc = cshift ? __funnelshift_r(raw, nb, cshift) : raw;
      if (lane >= pws) {
        loc = 0;
      } else if (Ms - lane * 32u < 32u) {
        loc &= (1u << (Ms - lane * 32u)) - 1u;
      }
      if (lane < pw) par[lane] = loc;
      const uint32_t cnt = __reduce_add_sync(0xffffffffu, __popc(loc));
      if (lane == 0) *unsat = cnt;
    }
    for (uint32_t w = tid; w < ew; w += T) ehat[w] = 0;
    // q[e] = gamma[var(e)] (decoder.cpp:156-158); padded slots land in the dummy blocks
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const Msg init = prior_as_msg<A>(gam[k]);
#pragma unroll
      for (int i = 0; i < DV; ++i) *reinterpret_cast<Msg*>(msgs + eo[k][i]) = init;
    }
    uint32_t eprev = 0, aprev = 0;
    __syncthreads();
    cmd = cmd_word[0];
    if (cmd == kDoorbellExit) break;
    t_begin = static_cast<uint64_t>(cmd_word[1]) | (static_cast<uint64_t>(cmd_word[2]) << 32);
    // (the first toggles of the bitmap come after the first iteration's mid barrier)
    const uint32_t synbit = (par[cl >> 5] >> (cl & 31u)) & 1u;
    if (ctl.soft != nullptr && aslot != kNoAbsorb) {
      // soft syndromes: this shot's prior of the absorbed variable (read after the doorbell was
      // seen; volatile: the values live in mapped host memory or were just copied in).  The
      // slot belongs to this thread's own check block, so no barrier is needed before its use.
      // Integer modes: soft_bytes = 4 when the host staged the values widened to int32 (mapped
      // host memory: one full 128-byte request per warp), else the caller's int8 / int16.
      const uint32_t m = seg.c0 + tid;
      Msg v;
      if constexpr (sizeof(Msg) == 2) {
        v = prior_as_msg<ArithF16>(*(static_cast<const volatile float*>(ctl.soft) + m));
      } else if constexpr (A::kInt) {
        v = ctl.soft_bytes == 4u   ? static_cast<Msg>(*(static_cast<const volatile int32_t*>(ctl.soft) + m))
            : ctl.soft_bytes == 1u ? static_cast<Msg>(*(static_cast<const volatile int8_t*>(ctl.soft) + m))
                                   : static_cast<Msg>(*(static_cast<const volatile int16_t*>(ctl.soft) + m));
      } else {
        v = *(static_cast<const volatile float*>(ctl.soft) + m) + 0.0f;
      }
      *reinterpret_cast<Msg*>(msgs + co + aslot * kMsg) = v;
    }

    // ---------------- iterations ----------------
    uint32_t iter = 0;
    bool still_unsat;
    for (;;) {
      ++iter;
      cn_ell<DC>(P, A{}, msgs + co, synbit);
      uint32_t achg = 0;
      if (aslot != kNoAbsorb) {
        const unsigned char* slot = msgs + co + aslot * kMsg;
        const uint32_t e = absorbed_decision(A{}, *reinterpret_cast<const Msg*>(slot),
                                             *reinterpret_cast<const Msg*>(slot + DC * kMsg));
        achg = e ^ aprev;
        aprev = e;
      }
      __syncthreads();
      uint32_t eb = 0;
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        eb |= vn_ell<DC, DV>(P, A{}, msgs, eo[k], gam[k], (keep0 >> k) & 1u) << k;
      }
      eb &= valid;
      const uint32_t changed = eb ^ eprev;
      eprev = eb;
      if (changed | achg) {
        int32_t delta = 0;
        if (achg) {
          const uint32_t bit = 1u << (cl & 31u);
          const uint32_t old = atomicXor(&par[cl >> 5], bit);
          delta += (old & bit) ? -1 : 1;
        }
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
          if ((changed >> k) & 1u) {
#pragma unroll
            for (int i = 0; i < DV; ++i) {
              if (eo[k][i] < scratch_off) {
                const uint32_t lm = eo[k][i] / kStride;
                const uint32_t bit = 1u << (lm & 31u);
                const uint32_t old = atomicXor(&par[lm >> 5], bit);
                delta += (old & bit) ? -1 : 1;
              }
            }
          }
        }
        atomicAdd(const_cast<uint32_t*>(unsat), static_cast<uint32_t>(delta));
      }
      __syncthreads();
      still_unsat = *unsat != 0u;
      if ((P.early && !still_unsat) || iter >= P.max_iter) break;
    }

    // ---------------- publish this segment's record ----------------
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      if ((eprev >> k) & 1u) atomicOr(&ehat[vloc[k] >> 5], 1u << (vloc[k] & 31u));
    }
    if (aprev) atomicOr(&ehat[aloc >> 5], 1u << (aloc & 31u));
    if (io.q_dump) {  // debug: messages back in reference edge order
      ell_dump_messages(P, seg, msgs, kStride, kMsg, DC * kMsg, 0u,
                        [&](uint32_t e, const unsigned char* q, const unsigned char* r) {
                          if constexpr (A::kInt) {
                            static_cast<int32_t*>(io.q_dump)[e] = *reinterpret_cast<const Msg*>(q);
                            static_cast<int32_t*>(io.r_dump)[e] = *reinterpret_cast<const Msg*>(r);
                          } else {
                            static_cast<float*>(io.q_dump)[e] = static_cast<float>(*reinterpret_cast<const Msg*>(q));
                            static_cast<float*>(io.r_dump)[e] = static_cast<float>(*reinterpret_cast<const Msg*>(r));
                          }
                        });
    }
    __syncthreads();
    {
      const uint64_t ns = globaltimer_ns() - t_begin;
      for (uint32_t w = tid; w < nrec; w += T) {
        const uint32_t slot = w & 7u;
        uint32_t v = cmd;
        if (slot) {
          const uint32_t d = (w >> 3) * kSectorData + slot - 1u;
          if (d < ews) {
            v = ehat[d];
          } else if (d < ews + pws) {
            v = par[d - ews];
          } else if (d == ews + pws) {
            v = still_unsat ? 0u : 1u;
          } else if (d == ews + pws + 1u) {
            v = iter;
          } else if (d == ews + pws + 2u) {
            v = static_cast<uint32_t>(ns);
          } else if (d == ews + pws + 3u) {
            v = static_cast<uint32_t>(ns >> 32);
          } else {
            v = 0u;
          }
        }
        rec[w] = v;
      }
    }
    t_idle0 = globaltimer_ns();
    last = cmd;
    if (ctl.mode != 2u) break;
    __syncthreads();  // see decode_lean_latency_kernel: orders the record's reads before the next prologue
  }
  if (ctl.mode == 2u) {
    if (s == 0 && tid == 0 && ctl.alive) {
      *ctl.alive = 0u;
      __threadfence_system();
    }
    cluster.sync();
  }
}

}  // namespace qb

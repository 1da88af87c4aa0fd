// Reduced-precision throughput kernel: TWO shots per thread in the two lanes of
// a half2 ((6,3)-regular codes, fp16 messages, fp16 arithmetic).
//
// Same structure as decode_lean_kernel (work item per segment, interleaved
// message blocks, counter-based stop test, first iteration from the syndrome),
// but every message word holds the values of shots 2k (low half) and 2k+1 (high
// half), and the node updates use the packed fp16 instructions (HADD2, HMUL2,
// HMNMX2, HSET2): one instruction advances both shots, there are no conversions
// at all, and the edge tables in registers are shared by the pair.  Lane by lane
// the operations are exactly those of the scalar half-mode kernels, so a batch
// decoded here equals shot-by-shot decoding bit for bit.
//
// The two shots of a pair stop independently: a finished lane is frozen (its
// parity bitmap, counter and decisions are no longer touched) while the other
// iterates on; the pair is released when both are done.
//
// kI8 = true runs the reference's INT8 mode (decoder.cpp:260-283, bit-exact) on
// the same packed instructions: every int8-mode quantity is an integer of
// magnitude <= 4 * 127, which fp16 represents exactly, so the sums, the
// saturation at +-127 (HMNMX2) and the comparisons are exact in fp16 arithmetic.
// The Q16 scaling (mag * alpha_fx + 32768) >> 16 becomes ONE fused multiply-add
// with the magic constant 1536 (= 1.5 * 2^10, where fp16 has unit spacing):
// fma(mag, c, 1536) - 1536 = round-to-nearest-even(mag * c), and the loader only
// selects this kernel after checking, for all 128 magnitudes, that it equals the
// reference's integer formula for the fp16 constant c it picked (P.alpha_h).
// Messages are stored as fp16 integers; a zero magnitude may carry a sign bit
// (-0), which is harmless: gamma is never 0 (decoder.cpp:115-120), so no sum
// can evaluate to -0 and a stored q is never -0 (its sign bit is the reference's
// `v < 0`).
#pragma once

#include "common.cuh"
#include "kernel_lean.cuh"

namespace qb {

constexpr uint32_t kH2Stride = 56, kH2ROff = 24;  // [6 x half2 q | 6 x half2 r | pad]

__host__ __device__ inline size_t lean_h2_bits_words(uint32_t seg_mmax) {
  return (8 * static_cast<size_t>(lean_pw(seg_mmax)) + 16 + 3) & ~size_t(3);  // keeps 16-byte alignment
}
__host__ __device__ inline size_t lean_h2_smem_bytes(uint32_t seg_mmax, uint32_t syn_w32) {
  const size_t msg = (static_cast<size_t>(seg_mmax + 1) * kH2Stride + 15) & ~size_t(15);
  // messages | bitmaps, counters, tickets, syndrome copies | 2 syndrome tiles | 2 mbarriers |
  // tile info [2][2] | tile cursor
  return msg + 4 * lean_h2_bits_words(seg_mmax) + 2 * kMaxTile * syn_w32 * 4 + 16 + 16 + 16;
}

__device__ __forceinline__ __half2 u2h2(uint32_t u) {
  return *reinterpret_cast<__half2*>(&u);
}
__device__ __forceinline__ uint32_t h22u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// min1 / min2 of six non-negative half2 values, lane-wise (13 packed min/max).
__device__ __forceinline__ void two_smallest6_h2(const __half2 (&a)[6], __half2& m1, __half2& m2) {
  const __half2 l0 = __hmin2(a[0], a[1]), h0 = __hmax2(a[0], a[1]);
  const __half2 l1 = __hmin2(a[2], a[3]), h1 = __hmax2(a[2], a[3]);
  const __half2 l2 = __hmin2(a[4], a[5]), h2 = __hmax2(a[4], a[5]);
  m1 = __hmin2(__hmin2(l0, l1), l2);
  const __half2 med = __hmax2(__hmin2(l0, l1), __hmin2(__hmax2(l0, l1), l2));
  m2 = __hmin2(med, __hmin2(__hmin2(h0, h1), h2));
}

template <bool kI8>
__device__ __forceinline__ __half2 h2_clamp_t(__half2 x) {
  if constexpr (kI8) {
    const __half2 c = __half2half2(__ushort_as_half(0x57f0));  // 127
    return __hmax2(__hmin2(x, c), __hneg2(c));
  } else {
    return h2_clamp(x);
  }
}

// alpha * m: one fp16 multiply (half mode) or the exact Q16 rounding (int8 mode)
template <bool kI8>
__device__ __forceinline__ __half2 h2_scale(__half2 alpha, __half2 m) {
  if constexpr (kI8) {
    const __half2 magic = __half2half2(__ushort_as_half(0x6600));  // 1536
    return __hsub2(__hfma2(m, alpha, magic), magic);
  } else {
    return __hmul2(alpha, m);
  }
}

// syn_pair: bit 15 = syndrome bit of the low-half shot, bit 31 = of the high-half shot
// The packed kernels are bound by the ALU pipe (min/max, compares, bit logic), while the
// FMA pipe idles.  So the check update computes each edge's "minimum of the OTHER five
// magnitudes" directly (nine two/three-input minima: no second-minimum network, no
// compare-and-select) and applies scale and sign with multiplications: edge j's output is
// e_j * (+-alpha), the sign being the syndrome, the parity of all incoming signs and
// edge j's own sign.  e_j is m1 or m2 of the scalar formulation and a product's magnitude
// does not depend on the sign of its factors, so the bits are those of
// "select alpha*m1 / alpha*m2, then set the sign".
template <bool kI8>
__device__ __forceinline__ void cn6_h2(const DecodeParams& P, unsigned char* blk, uint32_t syn_pair) {
  const uint2* qp = reinterpret_cast<const uint2*>(blk);
  uint32_t u[6];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const uint2 v = qp[j];
    u[2 * j] = v.x;
    u[2 * j + 1] = v.y;
  }
  __half2 a[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) a[j] = __habs2(u2h2(u[j]));  // folds into the consumers as |x|
  const __half2 pa = __hmin2(a[0], a[1]), pb = __hmin2(a[2], a[3]), pc = __hmin2(a[4], a[5]);
  __half2 e[6];
  e[0] = __hmin2(__hmin2(a[1], pb), pc);
  e[1] = __hmin2(__hmin2(a[0], pb), pc);
  e[2] = __hmin2(__hmin2(a[3], pa), pc);
  e[3] = __hmin2(__hmin2(a[2], pa), pc);
  e[4] = __hmin2(__hmin2(a[5], pa), pb);
  e[5] = __hmin2(__hmin2(a[4], pa), pb);
  const uint32_t sx = (u[0] ^ u[1] ^ u[2] ^ u[3] ^ u[4] ^ u[5] ^ syn_pair) & 0x80008000u;
  uint32_t o[6];
  if constexpr (kI8) {
    const __half2 c2 = __half2half2(__ushort_as_half(P.alpha_h));
    const __half2 magic = __half2half2(__ushort_as_half(0x6600));  // 1536
    const uint32_t one = sx ^ 0x3c003c00u;                         // +-1 with the common sign
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      const __half2 t = __hsub2(__hfma2(e[j], c2, magic), magic);  // exact Q16 scaling
      o[j] = h22u(__hmul2(t, u2h2(one ^ (u[j] & 0x80008000u))));
    }
  } else {
    const uint32_t al = sx ^ (static_cast<uint32_t>(P.alpha_h) * 0x00010001u);  // +-alpha
#pragma unroll
    for (int j = 0; j < 6; ++j) o[j] = h22u(__hmul2(e[j], u2h2(al ^ (u[j] & 0x80008000u))));
  }
  uint2* rp = reinterpret_cast<uint2*>(blk + kH2ROff);
#pragma unroll
  for (int j = 0; j < 3; ++j) rp[j] = make_uint2(o[2 * j], o[2 * j + 1]);
}

// returns the sign bits of the two posteriors (bit 15 / bit 31)
template <bool kI8>
__device__ __forceinline__ uint32_t vn3_h2(unsigned char* base, const uint32_t (&eo)[3],
                                           __half2 gamma2) {
  const __half2 r0 = *reinterpret_cast<const __half2*>(base + eo[0] + kH2ROff);
  const __half2 r1 = *reinterpret_cast<const __half2*>(base + eo[1] + kH2ROff);
  const __half2 r2 = *reinterpret_cast<const __half2*>(base + eo[2] + kH2ROff);
  const __half2 total = __hadd2(__hadd2(__hadd2(gamma2, r0), r1), r2);
  *reinterpret_cast<__half2*>(base + eo[0]) = h2_clamp_t<kI8>(__hsub2(total, r0));
  *reinterpret_cast<__half2*>(base + eo[1]) = h2_clamp_t<kI8>(__hsub2(total, r1));
  *reinterpret_cast<__half2*>(base + eo[2]) = h2_clamp_t<kI8>(__hsub2(total, r2));
  return h22u(total) & 0x80008000u;
}

template <bool kI8>
__device__ __forceinline__ uint32_t vn3_first_h2(const DecodeParams& P, unsigned char* base,
                                                 const uint32_t (&eo)[3], const uint32_t* par_a,
                                                 const uint32_t* par_b, __half2 gamma2) {
  const uint32_t mag = static_cast<uint32_t>(P.it1_h) * 0x00010001u;
  __half2 r[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const uint32_t fa = syn_bit_of_edge(par_a, eo[i], kH2Stride) ^ P.it1_neg;
    const uint32_t fb = syn_bit_of_edge(par_b, eo[i], kH2Stride) ^ P.it1_neg;
    r[i] = u2h2(mag ^ (fa << 15) ^ (fb << 31));
  }
  const __half2 total = __hadd2(__hadd2(__hadd2(gamma2, r[0]), r[1]), r[2]);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    *reinterpret_cast<__half2*>(base + eo[i]) = h2_clamp_t<kI8>(__hsub2(total, r[i]));
  }
  return h22u(total) & 0x80008000u;
}

// prior of one variable as a stored message: clamped fp16 (half mode) or the exact
// fp16 image of the quantised int prior (int8 mode)
template <bool kI8>
__device__ __forceinline__ __half h2_prior(float g) {
  if constexpr (kI8) {
    return __float2half_rn(g);  // |g| <= 127, an integer: exact
  } else {
    return prior_as_msg<ArithF16>(g);
  }
}

template <int CPT, int VPT, bool kFast, int MAXT, int MINB, bool kI8 = false, bool kDump = false>
__global__ void __launch_bounds__(MAXT, MINB)
decode_lean_h2_kernel(const __grid_constant__ DecodeParams P, const __grid_constant__ ShotIO io) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t tid = threadIdx.x, T = blockDim.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t nwarps = T >> 5;
  const uint32_t nseg = P.nseg;
  const uint32_t s = blockIdx.x % nseg;
  const uint32_t peer = blockIdx.x / nseg;
  const uint32_t peers = (gridDim.x - s + nseg - 1) / nseg;
  const SegmentDev seg = P.segs[s];
  const uint32_t Ms = seg.c1 - seg.c0;
  const uint32_t pw = lean_pw(P.seg_mmax);
  const uint32_t pws = (Ms + 31u) >> 5;
  const uint32_t gw0 = seg.c0 >> 5, gspan = ((seg.c1 - 1) >> 5) - gw0 + 1, cshift = seg.c0 & 31u;
  // the last segment also owns the padding bits of the packed rows (they are written as 0)
  const uint32_t v1z = s + 1u == nseg ? P.est_w32 * 32u : seg.v1;
  const uint32_t c1z = s + 1u == nseg ? P.syn_w32 * 32u : seg.c1;
  const uint32_t vw0 = seg.v0 >> 5, vspan = ((v1z - 1) >> 5) - vw0 + 1;
  const uint32_t gspan_out = ((c1z - 1) >> 5) - gw0 + 1;
  const uint64_t npairs = (io.nshots + 1) / 2;

  unsigned char* const msgs = smem_raw;
  const size_t msg_bytes = (static_cast<size_t>(P.seg_mmax + 1) * kH2Stride + 15) & ~size_t(15);
  uint32_t* const bits = reinterpret_cast<uint32_t*>(smem_raw + msg_bytes);
  // [item parity][shot lane][pw] bitmaps, then [item parity][shot lane] counters, tickets
  uint32_t* const unsat_ctr = bits + 4 * pw;  // [2][2]
  uint32_t* const ticket = bits + 4 * pw + 4;  // [2]
  uint32_t* const syn_copy = bits + 4 * pw + 16;  // [item parity][shot lane][pw], never toggled
  // syndromes arrive in TMA tiles of io.tile (even) shots = io.tile / 2 pairs, as in
  // decode_lean_kernel: one bulk copy and one queue ticket per tile, two tiles in flight
  uint32_t* const tilebuf = bits + lean_h2_bits_words(P.seg_mmax);  // [2][kMaxTile][syn_w32]
  uint64_t* const mbar = reinterpret_cast<uint64_t*>(tilebuf + 2 * kMaxTile * P.syn_w32);  // [2]
  uint32_t* const tinfo = reinterpret_cast<uint32_t*>(mbar + 2);  // [2]{first shot, shots}
  uint32_t* const tstate = tinfo + 4;                              // {buffer, pair in tile, phases}
  const uint32_t K = io.tile, tile_words = kMaxTile * P.syn_w32;

  uint32_t eo[VPT][kDV], co[CPT], cl[CPT], valid = 0;
  float gam[kFast ? 1 : VPT];
  {
    const float* __restrict__ gamma = static_cast<const float*>(P.gamma);
    const int32_t* __restrict__ gamma_i = static_cast<const int32_t*>(P.gamma);  // int8 mode
    const uint32_t dummy = P.seg_mmax * kH2Stride;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const uint32_t n = seg.v0 + tid + k * T;
      const bool ok = n < seg.v1;
      valid |= (ok ? 1u : 0u) << k;
#pragma unroll
      for (int i = 0; i < kDV; ++i) {
        const uint32_t eg = ok ? P.var_edges[n * kDV + i] : 0u;
        const uint32_t e = ok ? eg - seg.e0 : 0u;
        eo[k][i] = ok ? (e / kDC) * kH2Stride + P.edge_slot[eg] * 4u : dummy + i * 4u;
      }
      if constexpr (!kFast) {
        if constexpr (kI8) {
          gam[k] = ok ? static_cast<float>(gamma_i[n]) : 1.0f;
        } else {
          gam[k] = ok ? gamma[n] : 1.0f;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const uint32_t m = tid + k * T;
      cl[k] = m < Ms ? m : Ms;
      co[k] = (m < Ms ? m : P.seg_mmax) * kH2Stride;
    }
  }
  for (uint32_t b = tid; b < kH2Stride; b += T) msgs[P.seg_mmax * kH2Stride + b] = 0;

  auto issue_tile = [&](uint64_t t, uint32_t b) {
    lean_issue_tile(io.syn, io.nshots, P.syn_w32, K, t, tilebuf + b * tile_words, &mbar[b],
                    tinfo + 2 * b, lane);
  };
  if (tid == 0) {
    mbar_init(&mbar[0], 1u);
    mbar_init(&mbar[1], 1u);
    mbar_fence_init();
    tstate[0] = tstate[1] = tstate[2] = 0u;
  }
  __syncthreads();
  if (warp == 0) issue_tile(peer, 0u);
  uint64_t pair = static_cast<uint64_t>(peer) * (K / 2);
  uint32_t ipar = 0;
  __syncthreads();

  while (pair < npairs) {
    const uint64_t shot_a = 2 * pair, shot_b = 2 * pair + 1;
    const bool has_b = shot_b < io.nshots;
    uint32_t* const par_a = bits + (ipar * 2) * pw;
    uint32_t* const par_b = bits + (ipar * 2 + 1) * pw;
    uint32_t* const syn_a = syn_copy + (ipar * 2) * pw;
    uint32_t* const syn_b = syn_copy + (ipar * 2 + 1) * pw;
    volatile uint32_t* const unsat_a = unsat_ctr + ipar * 2;
    volatile uint32_t* const unsat_b = unsat_ctr + ipar * 2 + 1;
    // ---------------- prologue ----------------
    if (warp == 0) {
      const uint32_t tb = tstate[0], ti = tstate[1];
      if (ti == 0u) {  // first pair of a tile: wait for its bytes, start on the tile after it
        const uint32_t tphase = tstate[2];
        mbar_wait(&mbar[tb], (tphase >> tb) & 1u);
        __syncwarp();
        if (lane == 0) tstate[2] = tphase ^ (1u << tb);
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(&io.sched[2 + s], 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        issue_tile(static_cast<uint64_t>(t) + peers, tb ^ 1u);
        __syncwarp();
      }
      const uint32_t* rows = tilebuf + tb * tile_words + 2u * ti * P.syn_w32;
      const uint32_t raw_a = lane < gspan ? rows[gw0 + lane] : 0u;
      const uint32_t raw_b = lane < gspan && has_b ? rows[P.syn_w32 + gw0 + lane] : 0u;
      auto localise = [&](uint32_t raw, uint32_t* par, uint32_t* syn0, volatile uint32_t* ctr) {
        uint32_t nb = __shfl_down_sync(0xffffffffu, raw, 1);
        if (lane + 1 >= gspan) nb = 0;
        uint32_t loc = cshift ? __funnelshift_r(raw, nb, cshift) : raw;
        if (lane >= pws) {
          loc = 0;
        } else if (Ms - lane * 32u < 32u) {
          loc &= (1u << (Ms - lane * 32u)) - 1u;
        }
        if (lane < pw) {
          par[lane] = loc;
          syn0[lane] = loc;
        }
        const uint32_t cnt = __reduce_add_sync(0xffffffffu, __popc(loc));
        if (lane == 0) *ctr = cnt;
      };
      localise(raw_a, par_a, syn_a, unsat_a);
      localise(raw_b, par_b, syn_b, unsat_b);
      __syncwarp();  // every lane has read tstate[] before lane 0 advances it
      if (lane == 0) {
        // next pair: the following rows of this tile, else the first rows of the next tile
        const uint32_t tpairs = (tinfo[2 * tb + 1] + 1u) >> 1;
        const bool more = ti + 1u < tpairs;
        const uint32_t nf = tinfo[2 * (tb ^ 1u)];
        ticket[ipar] = more ? static_cast<uint32_t>(pair) + 1u : (nf == kNoShot ? kNoShot : nf >> 1);
        tstate[0] = more ? tb : tb ^ 1u;
        tstate[1] = more ? ti + 1u : 0u;
      }
    }
    if (warp == nwarps - 1) {
      for (int which = 0; which < (has_b ? 2 : 1); ++which) {
        uint32_t* est_g = io.est + (shot_a + which) * P.est_w32 + vw0;
        for (uint32_t w = lane; w < vspan; w += 32u) {
          const uint32_t mask = range_mask(vw0 + w, seg.v0, v1z);
          if (mask == 0xffffffffu) {
            est_g[w] = 0u;
          } else {
            atomicAnd(&est_g[w], ~mask);
          }
        }
      }
    }
    if constexpr (!kFast) {
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        const __half2 init = __half2half2(h2_prior<kI8>(gam[k]));
#pragma unroll
        for (int i = 0; i < kDV; ++i) *reinterpret_cast<__half2*>(msgs + eo[k][i]) = init;
      }
    }
    uint32_t eprev_a = 0, eprev_b = 0;
    __syncthreads();

    uint32_t synpair[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const uint32_t ba = (syn_a[cl[k] >> 5] >> (cl[k] & 31u)) & 1u;
      const uint32_t bb = (syn_b[cl[k] >> 5] >> (cl[k] & 31u)) & 1u;
      synpair[k] = (ba << 15) | (bb << 31);
    }
    const uint32_t next = ticket[ipar];

    // ---------------- iterations ----------------
    uint32_t iter = 0, iter_a = 0, iter_b = 0;
    bool live_a = true, live_b = true, conv_a = false, conv_b = false;
    uint32_t fin_a = 0, fin_b = 0;  // decisions of each shot at the moment it stopped
    for (;;) {
      ++iter;
      // posterior sign bits of the pair (bits 15 / 31) are shifted into one accumulator:
      // after VPT variables, shot a's decisions sit in bits [16-VPT, 15], shot b's in [32-VPT, 31]
      static_assert(VPT <= 8, "decision accumulator");
      uint32_t acc = 0;
      if (kFast && iter == 1u) {
        const __half2 g2 = __half2half2(__ushort_as_half(P.gamma_hb));
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
          // syndrome bits from the untouched copies: no barrier before the toggles
          acc = (acc >> 1) | vn3_first_h2<kI8>(P, msgs, eo[k], syn_a, syn_b, g2);
        }
      } else {
#pragma unroll
        for (int k = 0; k < CPT; ++k) cn6_h2<kI8>(P, msgs + co[k], synpair[k]);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
          const __half2 g2 = kFast ? __half2half2(__ushort_as_half(P.gamma_hb))
                                   : __half2half2(h2_prior<kI8>(gam[k]));
          acc = (acc >> 1) | vn3_h2<kI8>(msgs, eo[k], g2);
        }
      }
      uint32_t eb_a = (acc >> (16 - VPT)) & ((1u << VPT) - 1u), eb_b = acc >> (32 - VPT);
      eb_a &= valid;
      eb_b &= valid;
      auto toggle = [&](uint32_t changed, uint32_t* par, volatile uint32_t* ctr) {
        int32_t delta = 0;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
          if ((changed >> k) & 1u) {
#pragma unroll
            for (int i = 0; i < kDV; ++i) {
              const uint32_t lm = eo[k][i] / kH2Stride;
              const uint32_t bit = 1u << (lm & 31u);
              const uint32_t old = atomicXor(&par[lm >> 5], bit);
              delta += (old & bit) ? -1 : 1;
            }
          }
        }
        atomicAdd(const_cast<uint32_t*>(ctr), static_cast<uint32_t>(delta));
      };
      if (live_a) {
        const uint32_t ch = eb_a ^ eprev_a;
        eprev_a = eb_a;
        if (ch) toggle(ch, par_a, unsat_a);
      }
      if (live_b) {
        const uint32_t ch = eb_b ^ eprev_b;
        eprev_b = eb_b;
        if (ch) toggle(ch, par_b, unsat_b);
      }
      __syncthreads();
      const bool last = iter >= P.max_iter;
      if (live_a) {
        const bool uns = *unsat_a != 0u;
        if ((P.early && !uns) || last) {
          live_a = false;
          conv_a = !uns;
          iter_a = iter;
          fin_a = eprev_a;
        }
      }
      if (live_b) {
        const bool uns = *unsat_b != 0u;
        if ((P.early && !uns) || last) {
          live_b = false;
          conv_b = !uns;
          iter_b = iter;
          fin_b = eprev_b;
        }
      }
      if (!live_a && !live_b) break;
    }

    // ---------------- epilogue ----------------
    auto write_out = [&](uint64_t shot, const uint32_t* par, uint32_t fin, bool conv,
                         uint32_t iters) {
      if (warp == 0 && io.resid) {
        const uint32_t hi = lane < pw ? par[lane] : 0u;
        uint32_t lo = __shfl_up_sync(0xffffffffu, hi, 1);
        if (lane == 0) lo = 0;
        const uint32_t out = cshift ? __funnelshift_l(lo, hi, cshift) : hi;
        if (lane < gspan_out) {
          uint32_t* dst = io.resid + shot * P.syn_w32 + gw0 + lane;
          const uint32_t mask = range_mask(gw0 + lane, seg.c0, c1z);
          if (mask == 0xffffffffu) {
            *dst = out;
          } else {
            atomicAnd(dst, ~mask);
            atomicOr(dst, out & mask);
          }
        }
      }
      if (fin) {
        uint32_t* est_g = io.est + shot * P.est_w32;
#pragma unroll
        for (int k = 0; k < VPT; ++k) {
          if ((fin >> k) & 1u) {
            const uint32_t n = seg.v0 + tid + k * T;
            atomicOr(&est_g[n >> 5], 1u << (n & 31u));
          }
        }
      }
      if (tid == 0) {
        io.conv[shot * nseg + s] = conv ? 1 : 0;
        io.iters[shot * nseg + s] = iters;
      }
    };
    write_out(shot_a, par_a, fin_a, conv_a, iter_a);
    if (has_b) write_out(shot_b, par_b, fin_b, conv_b, iter_b);
    if constexpr (kDump) if (io.q_dump != nullptr && (io.dump_shot >> 1) == pair) {
      // parity hook (see lean_dump_messages).  A lane that stopped earlier than its partner has
      // had its r slots rewritten by the partner's later check stages (a frozen lane's q no
      // longer changes, so they were recomputed from the same inputs: still its final r).
      const bool hi = (io.dump_shot & 1u) != 0;
      const bool both_first = kFast && iter == 1u;
      lean_dump_messages<ArithF16>(
          P, io, seg, msgs, hi ? syn_b : syn_a, both_first, 4u, kH2Stride, kH2ROff, hi ? 2u : 0u,
          [&](uint32_t e, const unsigned char* q, const unsigned char* r, bool first_only, uint32_t flip) {
            const __half s1 = __ushort_as_half(static_cast<unsigned short>(P.it1_h ^ (flip << 15)));
            const float qv = __half2float(*reinterpret_cast<const __half*>(q));
            const float rv = __half2float(first_only ? s1 : *reinterpret_cast<const __half*>(r));
            if constexpr (kI8) {
              static_cast<int32_t*>(io.q_dump)[e] = static_cast<int32_t>(qv);
              static_cast<int32_t*>(io.r_dump)[e] = static_cast<int32_t>(rv);
            } else {
              static_cast<float*>(io.q_dump)[e] = qv;
              static_cast<float*>(io.r_dump)[e] = rv;
            }
          });
    }
    pair = next == kNoShot ? ~0ull : static_cast<uint64_t>(next);
    ipar ^= 1u;
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

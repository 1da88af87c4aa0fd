// C-ABI implementation (include/qldpc_b200.h): validation, the code loader
// that turns a Tanner graph into device tables, and the kernel launches.
//
// Reference behaviour mirrored here: Decoder construction + validation
// (proj/src/decoder.cpp:73-140, :373-404), decode_into / decode_css_into
// (:551-591), decode_batch (:604-655), last_kernel_ns (:593-596).
#include "../../include/qldpc_b200.h"

#include <cuda_runtime.h>

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernel_generic.cuh"
#include "kernel_lean.cuh"
#include "kernel_lean_h2.cuh"
#include "kernel_ell.cuh"
#include "kernel_ell_h2.cuh"
#include "kernel_ell_latency.cuh"
#include "kernel_noise.cuh"
#include "kernel_bw.cuh"
#include "kernel_classify.cuh"
#include "kernel_campaign.cuh"

using namespace qb;

namespace {

thread_local std::string g_create_error;

// Pinned (mapped) host memory is slow to allocate and free (1.5 - 2 ms per call) and the
// reference's usage constructs decoders freely (one per decode() call, decoder.cpp:598-602):
// every handle takes ONE slab for its four small staging buffers, and slabs of destroyed
// handles wait in a process-wide free list for the next handle on that device.
struct PinnedSlab {
  void* p;
  size_t bytes;
  int device;
};
std::mutex g_slab_mu;
std::vector<PinnedSlab> g_slabs;
constexpr size_t kMaxIdleSlabs = 16;

void* slab_acquire(size_t bytes, int device, size_t* got) {
  {
    std::lock_guard<std::mutex> lk(g_slab_mu);
    for (size_t i = 0; i < g_slabs.size(); ++i) {
      if (g_slabs[i].device == device && g_slabs[i].bytes >= bytes && g_slabs[i].bytes <= 4 * bytes + 4096) {
        const PinnedSlab sl = g_slabs[i];
        g_slabs.erase(g_slabs.begin() + static_cast<long>(i));
        *got = sl.bytes;
        return sl.p;
      }
    }
  }
  const size_t want = (bytes + 4095) & ~static_cast<size_t>(4095);
  void* p = nullptr;
  const cudaError_t e = cudaHostAlloc(&p, want, cudaHostAllocMapped);
  if (e != cudaSuccess) return nullptr;
  *got = want;
  return p;
}

void slab_release(void* p, size_t bytes, int device) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> lk(g_slab_mu);
    if (g_slabs.size() < kMaxIdleSlabs) {
      g_slabs.push_back({p, bytes, device});
      return;
    }
  }
  cudaFreeHost(p);
}

// cudaGetDeviceProperties costs milliseconds; the two fields the loader needs do not change
bool device_limits(int device, int* sm_count, int* smem_optin) {
  static std::mutex mu;
  static std::vector<std::array<int, 3>> seen;  // {device, sm_count, smem_optin}
  std::lock_guard<std::mutex> lk(mu);
  for (const auto& d : seen) {
    if (d[0] == device) {
      *sm_count = d[1];
      *smem_optin = d[2];
      return true;
    }
  }
  int sm = 0, optin = 0;
  if (cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, device) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess) {
    return false;
  }
  seen.push_back({device, sm, optin});
  *sm_count = sm;
  *smem_optin = optin;
  return true;
}

struct StatusError {
  qb_status code;
  std::string msg;
};

[[noreturn]] void fail(qb_status code, std::string msg) { throw StatusError{code, std::move(msg)}; }

#define CUDA_TRY(expr)                                                               \
  do {                                                                               \
    cudaError_t err__ = (expr);                                                      \
    if (err__ != cudaSuccess) {                                                      \
      fail(QB_RUNTIME_ERROR, std::string("CUDA error in " #expr ": ") +              \
                                 cudaGetErrorName(err__) + " (" +                    \
                                 cudaGetErrorString(err__) + ")");                   \
    }                                                                                \
  } while (0)

template <typename T>
T* dev_upload(const std::vector<T>& host) {
  T* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, std::max<size_t>(host.size(), 1) * sizeof(T)));
  if (!host.empty()) {
    CUDA_TRY(cudaMemcpy(d, host.data(), host.size() * sizeof(T), cudaMemcpyHostToDevice));
  }
  return d;
}

// round(value * scale) clamped to [-limit, limit] (decoder.cpp:500-509).
int32_t quantize_saturate(double value, double scale, int32_t limit) {
  const double scaled = value * scale;
  if (std::isnan(scaled)) fail(QB_INVALID_ARGUMENT, "quantize_saturate: value is NaN");
  if (scaled >= static_cast<double>(limit)) return limit;
  if (scaled <= static_cast<double>(-limit)) return -limit;
  return static_cast<int32_t>(std::llround(scaled));
}

size_t msg_bytes_of(int arith) {
  switch (arith) {
    case QB_ARITH_FLOAT: return 4;
    case QB_ARITH_INT8: return 1;
    case QB_ARITH_INT16: return 2;
    default: return 2;  // half
  }
}

}  // namespace

using KernelFn = void (*)(DecodeParams, ShotIO);
using LatKernelFn = void (*)(DecodeParams, ShotIO, LatencyCtl, SynInline);

constexpr int kPipeSlots = 3;                      // qb_decode_batch: chunks in flight
constexpr int kSchedWords = 2 + kMaxSegments;      // scheduler words per concurrent launch
// Every launch needs its own ticket / finished-CTA words while it is in flight (the last CTA
// rewinds them).  Slot 0: single shots; 1 .. kPipeSlots: the chunk pipeline of
// qb_decode_batch; the rest is a ring handed out launch by launch to the device-buffer entry
// points (qb_decode_batch_device on caller streams, campaigns), so launches of one handle on
// DIFFERENT streams do not share words unless more than kSchedRing of them are in flight.
constexpr int kSchedRing = 16;
constexpr int kSchedSlots = 1 + kPipeSlots + kSchedRing;

struct LaunchPlan {
  KernelFn kernel = nullptr;
  KernelFn kernel_soft = nullptr;  // same shape, per-shot priors of the absorbed variables
  KernelFn kernel_dump = nullptr;  // same shape + the message dump of qb_decode_batch_debug
  const char* name = "";
  bool regular = false;
  bool cluster = false;
  int npt = 0;                 // nodes-per-thread class of the regular kernel
  uint32_t ngroups = 1;
  uint32_t group_threads = 32;
  unsigned block = 32;
  int ctas_per_sm = 1;
  size_t smem = 0;
  bool items = false;          // work item = (shot, segment): grid-stride over per-segment queues
  bool lean = false;           // ... the instruction-lean single-slot variant
  bool pair = false;           // ... two shots per thread in half2 lanes (half mode)
  int ell = 0;                 // degree-padded kernel: 100 * DC + DV (0 = not that kernel)
};

struct qb_decoder {
  int device = 0;
  int sm_count = 0;
  int max_smem_optin = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t pipe_stream[kPipeSlots] = {};
  cudaEvent_t pipe_event[kPipeSlots] = {};
  DecodeParams P{};
  int arith = 0;
  std::vector<void*> dev_allocs;  // tables, freed in the destructor
  unsigned int* d_sched = nullptr;
  uint32_t sched_next = 0;  // next ring slot

  // single-shot staging: mapped pinned host memory (+ device mirrors for the
  // memcpy protocol)
  uint32_t* h_in = nullptr;   // [syn_w32]
  uint32_t* d_in_map = nullptr;
  unsigned char* h_out = nullptr;
  unsigned char* d_out_map = nullptr;
  size_t out_bytes = 0, off_res = 0, off_conv = 0, off_iters = 0, off_ns = 0, off_flag = 0;
  uint32_t* d_in_dev = nullptr;
  unsigned char* d_out_dev = nullptr;
  uint32_t seq = 0;
  uint64_t last_kernel_ns = 0;

  // batch buffers (device), grown on demand
  uint64_t batch_cap = 0;
  uint32_t *b_syn = nullptr, *b_est = nullptr, *b_res = nullptr, *b_iters = nullptr;
  uint8_t* b_conv = nullptr;
  // debug dumps
  void *d_qdump = nullptr, *d_rdump = nullptr;
  uint64_t* d_probs = nullptr;  // per-variable flip thresholds of the noise generator
  // campaign state
  uint32_t *d_tests_x = nullptr, *d_tests_z = nullptr;
  uint32_t n_tests_x = 0, n_tests_z = 0;
  uint32_t* c_err = nullptr;  // [batch_cap][est_w32] sampled errors
  unsigned long long* d_counters = nullptr;
  // per-shot priors of the absorbed variables ("soft syndromes")
  unsigned char* b_soft = nullptr;       // [batch_cap][M] elements of soft_bytes
  uint32_t soft_bytes = 4;               // 4 float (float / half), 1 int8, 2 int16
  double quant_scale = 0.0;              // integer modes: the scale priors were quantised with
  std::vector<uint32_t> soft_var;        // [M] variable whose prior soft[m] replaces, or ~0u
  uint32_t* d_aux_mask = nullptr;        // [est_w32] non-data variables (qb_set_auxiliary_vars)
  uint64_t* d_tcol = nullptr;            // [N] logical-test column per variable (fused campaign kernel)
  // single-shot soft decode (qb_decode_soft): staging for one shot's [M] soft values
  unsigned char* h_soft1 = nullptr;      // mapped pinned
  unsigned char* d_soft1_map = nullptr;  // ... as the device sees it
  unsigned char* d_soft1_dev = nullptr;  // device copy (memcpy protocol)
  bool lat_is_ell = false;               // single shots run decode_ell_latency_kernel
  bool db_soft = false;                  // the resident doorbell kernel reads soft values
  cudaGraphExec_t lat_graph_soft[2] = {nullptr, nullptr};
  int64_t opt_campaign_fused = 1;        // QB_OPT_CAMPAIGN_FUSED
  int64_t opt_latency_wait = 0;          // QB_OPT_LATENCY_WAIT

  // options
  int64_t opt_kernel = 0, opt_latency_io = 0, opt_latency_shape = 0, opt_group_threads = 0,
          opt_batch_ctas = 0, opt_batch_npt = 0, opt_latency_npt = 0, opt_batch_shape = 0, opt_batch_pair = 1;
  // lean single-shot cluster kernel (kernel_lean.cuh) and its persistent doorbell mode
  LatKernelFn lat_lean_kernel = nullptr;
  unsigned lat_lean_block = 0;
  size_t lat_lean_smem = 0;
  uint32_t* h_db = nullptr;   // mapped: doorbell block [32] + alive word [32]
  uint32_t* d_db = nullptr;
  uint32_t* h_rec = nullptr;  // mapped: sectored result records, rec_stride words per segment
  uint32_t* d_rec_map = nullptr;
  uint32_t* d_rec_dev = nullptr;
  uint32_t rec_stride = 0;
  bool db_running = false;
  int64_t opt_idle_ms = 200;
  // optional CUDA-event timing of the memcpy protocol (H2D + kernel + D2H on the stream)
  int64_t opt_latency_events = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  uint64_t last_event_ns = 0;
  // memcpy protocol as ONE CUDA-graph launch (H2D copy -> cluster kernel -> D2H copy); two
  // instantiated graphs with different record tags alternate, so a stale record is detected
  int64_t opt_batch_tile = 0;  // shots per TMA syndrome tile, 0 = auto
  int64_t opt_sampler = 0;      // qb_generate_syndromes: 0 = the reference's stream, 1 = geometric skips
  int64_t opt_batch_chunk = 0;  // qb_decode_batch: shots per pipeline chunk, 0 = auto (2^15)
  int64_t opt_slot_spread = 2;  // lean batch kernels: bank-spreading slot permutation (2 = annealed)
  int64_t opt_latency_graph = 1;
  cudaGraphExec_t lat_graph[2] = {nullptr, nullptr};
  uint32_t lat_graph_flip = 0;
  bool regular63 = false;  // every check degree 6, every variable degree 3
  uint32_t max_dc = 0, max_dv = 0;  // largest check / variable degree of the graph
  void* h_slab = nullptr;          // the pinned slab behind h_in / h_out / h_db / h_rec
  size_t h_slab_bytes = 0;
  uint8_t* d_edge_slot = nullptr;  // [E] slot permutation of the lean batch kernels
  int64_t slot_table_for = -1;     // ... computed for this thread count (0 = natural order)
  std::vector<uint32_t> h_var_edges, h_check_off;  // host copies for the slot optimiser
  bool i8_pair_ok = false;  // int8 mode: the Q16 scaling has an exact fp16 form (kernel_lean_h2.cuh)
  bool fast_ok = false;    // uniform prior (and, for fp32, provably clamp-free)
  bool tab_ok = false;     // ... and its first iteration is a function of syndrome-bit counts (it1_tq)
  int64_t opt_fast = 1;
  LaunchPlan lat, bat;

  uint64_t launches = 0;
  std::string err;
  size_t smem_bytes = 0;
  size_t smem_lean = 0;
};

namespace {

void drop_latency_graphs(qb_decoder* h) {
  for (auto& g : h->lat_graph) {
    if (g) cudaGraphExecDestroy(g);
    g = nullptr;
  }
  for (auto& g : h->lat_graph_soft) {
    if (g) cudaGraphExecDestroy(g);
    g = nullptr;
  }
}

void free_batch(qb_decoder* h) {
  cudaFree(h->b_syn);
  cudaFree(h->b_est);
  cudaFree(h->b_res);
  cudaFree(h->b_iters);
  cudaFree(h->b_conv);
  cudaFree(h->c_err);
  cudaFree(h->b_soft);
  h->c_err = nullptr;
  h->b_soft = nullptr;
  h->b_syn = h->b_est = h->b_res = h->b_iters = nullptr;
  h->b_conv = nullptr;
  h->batch_cap = 0;
}

void destroy(qb_decoder* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->db_running && h->h_db) {
    volatile uint32_t* db = h->h_db;
    for (int k = 0; k < 4; ++k) db[8 * k] = 0xffffffffu;
    std::atomic_thread_fence(std::memory_order_seq_cst);
  }
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (void* p : h->dev_allocs) cudaFree(p);
  drop_latency_graphs(h);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  cudaFree(h->d_sched);
  cudaFree(h->d_in_dev);
  cudaFree(h->d_out_dev);
  cudaFree(h->d_qdump);
  cudaFree(h->d_rdump);
  cudaFree(h->d_probs);
  cudaFree(h->d_tests_x);
  cudaFree(h->d_tests_z);
  cudaFree(h->d_counters);
  cudaFree(h->d_aux_mask);
  cudaFree(h->d_tcol);
  cudaFree(h->d_soft1_dev);
  if (h->h_soft1) cudaFreeHost(h->h_soft1);
  cudaFree(h->d_rec_dev);
  slab_release(h->h_slab, h->h_slab_bytes, h->device);  // h_in, h_out, h_db, h_rec
  free_batch(h);
  for (int k = 0; k < kPipeSlots; ++k) {
    if (h->pipe_stream[k]) cudaStreamDestroy(h->pipe_stream[k]);
    if (h->pipe_event[k]) cudaEventDestroy(h->pipe_event[k]);
  }
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

// ---- validation -----------------------------------------------------------

void validate_graph(const qb_graph* g) {
  if (!g) fail(QB_INVALID_ARGUMENT, "graph is NULL");
  if (g->num_checks == 0 || g->num_vars == 0 || g->num_edges == 0) {
    fail(QB_INVALID_ARGUMENT, "graph must have checks, variables and at least one edge");
  }
  if (!g->edge_var || !g->check_offsets || !g->var_offsets || !g->var_edges) {
    fail(QB_INVALID_ARGUMENT, "graph arrays must not be NULL");
  }
  const uint32_t M = g->num_checks, N = g->num_vars, E = g->num_edges;
  if (g->check_offsets[0] != 0 || g->check_offsets[M] != E) {
    fail(QB_INVALID_ARGUMENT, "check_offsets must run from 0 to num_edges");
  }
  for (uint32_t m = 0; m < M; ++m) {
    if (g->check_offsets[m + 1] < g->check_offsets[m]) {
      fail(QB_INVALID_ARGUMENT, "check_offsets must be non-decreasing");
    }
  }
  if (g->var_offsets[0] != 0 || g->var_offsets[N] != E) {
    fail(QB_INVALID_ARGUMENT, "var_offsets must run from 0 to num_edges");
  }
  for (uint32_t e = 0; e < E; ++e) {
    if (g->edge_var[e] >= N) fail(QB_INVALID_ARGUMENT, "edge_var entry out of range");
  }
  std::vector<uint8_t> seen(E, 0);
  for (uint32_t n = 0; n < N; ++n) {
    if (g->var_offsets[n + 1] < g->var_offsets[n]) {
      fail(QB_INVALID_ARGUMENT, "var_offsets must be non-decreasing");
    }
    for (uint32_t i = g->var_offsets[n]; i < g->var_offsets[n + 1]; ++i) {
      const uint32_t e = g->var_edges[i];
      if (e >= E || seen[e] || g->edge_var[e] != n) {
        fail(QB_INVALID_ARGUMENT, "var_edges is not a permutation consistent with edge_var");
      }
      if (i > g->var_offsets[n] && g->var_edges[i - 1] >= e) {
        fail(QB_INVALID_ARGUMENT, "var_edges must be ascending within each variable");
      }
      seen[e] = 1;
    }
  }
}

// Mirrors validate_common (decoder.cpp:373-387).
void validate_config_common(const qb_graph* g, const qb_config* c) {
  if (!c) fail(QB_INVALID_ARGUMENT, "config is NULL");
  if (c->max_iterations < 1) {
    fail(QB_INVALID_ARGUMENT, "DecoderConfig: max_iterations must be at least 1");
  }
  if (c->max_iterations > 0x7fffffffull) {
    fail(QB_INVALID_ARGUMENT, "DecoderConfig: max_iterations exceeds the device counter range");
  }
  if (!(c->alpha > 0.0 && c->alpha <= 1.0)) {
    fail(QB_INVALID_ARGUMENT, "DecoderConfig: alpha must lie in (0, 1]");
  }
  const bool has = c->priors != nullptr && c->num_priors != 0;
  if (c->num_priors != 0 && c->priors == nullptr) {
    fail(QB_INVALID_ARGUMENT, "DecoderConfig: num_priors given but priors is NULL");
  }
  if (has && c->num_priors != g->num_vars) {
    fail(QB_INVALID_ARGUMENT, "DecoderConfig: " + std::to_string(c->num_priors) +
                                  " priors given but the graph has " +
                                  std::to_string(g->num_vars) + " variables");
  }
  if (c->arithmetic < QB_ARITH_FLOAT || c->arithmetic > QB_ARITH_HALF) {
    fail(QB_INVALID_ARGUMENT, "DecoderConfig: unknown arithmetic mode");
  }
}

// ---- kernel dispatch ------------------------------------------------------
//
// A LaunchPlan names one kernel instantiation plus its launch shape.  Two plans
// are kept per decoder: `lat` for the single-shot path and `bat` for the
// persistent batch path.  They are recomputed whenever an option changes.

KernelFn generic_kernel(int arith) {
  switch (arith) {
    case QB_ARITH_FLOAT: return decode_generic_kernel<ArithF32>;
    case QB_ARITH_INT8: return decode_generic_kernel<ArithI8>;
    case QB_ARITH_INT16: return decode_generic_kernel<ArithI16>;
    default: return decode_generic_kernel<ArithF16>;
  }
}

// Lean item-kernel variants: (checks, variables) per thread, launch bounds.
struct LeanVariant {
  int cpt, vpt, maxt, minb;
};
// Variant numbers are stable identifiers (QB_OPT_BATCH_VARIANT); 5, 7, 9 and 10 were
// measured, never selected by the loader and retired (maxt = 0).
constexpr LeanVariant kLeanVariants[] = {
    {1, 2, 1024, 1},  // 1: widest CTA, any segment size up to 960 checks
    {3, 5, 160, 7},   // 2: 56 registers, seven 5-warp CTAs per SM: the fp32 / int16 choice since the
                      //    first iteration is a table (no spills left at 56: 127.3 vs 123.9 M/s)
    {2, 4, 256, 3},   // 3
    {3, 5, 192, 5},   // 4: 64 registers, six CTAs per SM on [[784,24,24]]: the early-stop choice
    {0, 0, 0, 0},     // 5: retired
    {2, 4, 512, 2},   // 6
    {0, 0, 0, 0},     // 7: retired
    {3, 5, 160, 4},   // 8: 102 registers, the packed (two shots per thread) kernels' choice
    {0, 0, 0, 0},     // 9: retired
    {0, 0, 0, 0},     // 10: retired
    {3, 5, 160, 8},   // 11: 48 registers, eight 5-warp CTAs per SM: fixed iteration counts
};
constexpr int kNumLeanVariants = sizeof(kLeanVariants) / sizeof(kLeanVariants[0]);

template <class A, bool kFast>
KernelFn lean_kernel_tf(int variant) {
  switch (variant) {
    case 1: return decode_lean_kernel<A, 1, 2, kFast, 1024, 1>;
    case 2: return decode_lean_kernel<A, 3, 5, kFast, 160, 7>;
    case 3: return decode_lean_kernel<A, 2, 4, kFast, 256, 3>;
    case 4: return decode_lean_kernel<A, 3, 5, kFast, 192, 5>;
    case 8: return decode_lean_kernel<A, 3, 5, kFast, 160, 4>;
    case 11: return decode_lean_kernel<A, 3, 5, kFast, 160, 8>;
    default: return decode_lean_kernel<A, 2, 4, kFast, 512, 2>;
  }
}

KernelFn lean_kernel(int arith, int variant, bool fast) {
  switch (arith) {
    case QB_ARITH_FLOAT:
      return fast ? lean_kernel_tf<ArithF32, true>(variant) : lean_kernel_tf<ArithF32, false>(variant);
    case QB_ARITH_INT8:
      return fast ? lean_kernel_tf<ArithI8, true>(variant) : lean_kernel_tf<ArithI8, false>(variant);
    case QB_ARITH_INT16:  // integers in fp32 words (ArithI16F): the fp32 layout and shared-memory size
      return fast ? lean_kernel_tf<ArithI16F, true>(variant) : lean_kernel_tf<ArithI16F, false>(variant);
    default:
      return fast ? lean_kernel_tf<ArithF16, true>(variant) : lean_kernel_tf<ArithF16, false>(variant);
  }
}

// kDump instantiations (qb_decode_batch_debug) exist for the shapes the loader picks by itself
template <class A, bool kFast>
KernelFn lean_dump_kernel_tf(int variant) {
  switch (variant) {
    case 2: return decode_lean_kernel<A, 3, 5, kFast, 160, 7, true>;
    case 4: return decode_lean_kernel<A, 3, 5, kFast, 192, 5, true>;
    default: return nullptr;
  }
}
KernelFn lean_dump_kernel(int arith, int variant, bool fast) {
  switch (arith) {
    case QB_ARITH_FLOAT:
      return fast ? lean_dump_kernel_tf<ArithF32, true>(variant) : lean_dump_kernel_tf<ArithF32, false>(variant);
    case QB_ARITH_INT16:
      return fast ? lean_dump_kernel_tf<ArithI16F, true>(variant) : lean_dump_kernel_tf<ArithI16F, false>(variant);
    default: return nullptr;
  }
}
KernelFn lean_h2_dump_kernel(bool i8, int variant, bool fast) {
  if (variant != 8) return nullptr;
  if (i8) {
    return fast ? decode_lean_h2_kernel<3, 5, true, 160, 4, true, true>
                : decode_lean_h2_kernel<3, 5, false, 160, 4, true, true>;
  }
  return fast ? decode_lean_h2_kernel<3, 5, true, 160, 4, false, true>
              : decode_lean_h2_kernel<3, 5, false, 160, 4, false, true>;
}
template <class A>
KernelFn ell_dump_kernel_t(int idx) {
  switch (idx) {
    case 0: return decode_ell_kernel<A, 4, 2, 1, 2, 1024, 1, false, true>;
    case 1: return decode_ell_kernel<A, 7, 3, 3, 5, 192, 5, false, true>;
    case 2: return decode_ell_kernel<A, 7, 3, 3, 5, 320, 3, false, true>;
    default: return nullptr;
  }
}
KernelFn ell_dump_kernel(int arith, int idx, bool pair) {
  if (pair) {
    const bool i8 = arith == QB_ARITH_INT8;
    switch (idx) {
      case 1: return i8 ? decode_ell_h2_kernel<7, 3, 3, 5, 160, 4, true, false, true>
                        : decode_ell_h2_kernel<7, 3, 3, 5, 160, 4, false, false, true>;
      case 2: return i8 ? decode_ell_h2_kernel<7, 3, 3, 5, 320, 2, true, false, true>
                        : decode_ell_h2_kernel<7, 3, 3, 5, 320, 2, false, false, true>;
      default: return nullptr;
    }
  }
  switch (arith) {
    case QB_ARITH_FLOAT: return ell_dump_kernel_t<ArithF32>(idx);
    case QB_ARITH_INT8:
    case QB_ARITH_INT16: return ell_dump_kernel_t<ArithI32>(idx);
    default: return ell_dump_kernel_t<ArithF16>(idx);
  }
}

// int8 mode on the packed fp16 kernel (kernel_lean_h2.cuh): the shapes the loader may pick
template <bool kFast>
KernelFn lean_h2_i8_kernel_tf(int variant) {
  switch (variant) {
    case 1: return decode_lean_h2_kernel<1, 2, kFast, 1024, 1, true>;
    case 3: return decode_lean_h2_kernel<2, 4, kFast, 256, 3, true>;
    case 6: return decode_lean_h2_kernel<2, 4, kFast, 512, 2, true>;
    case 8: return decode_lean_h2_kernel<3, 5, kFast, 160, 4, true>;
    default: return nullptr;
  }
}

template <bool kFast>
KernelFn lean_h2_kernel_tf(int variant) {
  switch (variant) {
    case 1: return decode_lean_h2_kernel<1, 2, kFast, 1024, 1>;
    case 3: return decode_lean_h2_kernel<2, 4, kFast, 256, 3>;
    case 4: return decode_lean_h2_kernel<3, 5, kFast, 192, 5>;
    case 8: return decode_lean_h2_kernel<3, 5, kFast, 160, 4>;
    case 6: return decode_lean_h2_kernel<2, 4, kFast, 512, 2>;
    default: return nullptr;
  }
}

template <class A, bool kFast>
LatKernelFn lean_latency_kernel_tf(int npt) {
  return npt == 3   ? decode_lean_latency_kernel<A, 1, 1, kFast>  // one variable per thread
         : npt == 1 ? decode_lean_latency_kernel<A, 1, 2, kFast>
                    : decode_lean_latency_kernel<A, 2, 4, kFast>;
}

LatKernelFn lean_latency_kernel(int arith, int npt, bool fast) {
  switch (arith) {
    case QB_ARITH_FLOAT:
      return fast ? lean_latency_kernel_tf<ArithF32, true>(npt)
                  : lean_latency_kernel_tf<ArithF32, false>(npt);
    case QB_ARITH_INT8:
      return fast ? lean_latency_kernel_tf<ArithI8, true>(npt)
                  : lean_latency_kernel_tf<ArithI8, false>(npt);
    case QB_ARITH_INT16:
      return fast ? lean_latency_kernel_tf<ArithI16, true>(npt)
                  : lean_latency_kernel_tf<ArithI16, false>(npt);
    default:
      return fast ? lean_latency_kernel_tf<ArithF16, true>(npt)
                  : lean_latency_kernel_tf<ArithF16, false>(npt);
  }
}

// Degree-padded (ELL) batch kernels for irregular graphs: the degree bounds and
// nodes-per-thread shapes that are instantiated (kernel_ell.cuh).  The loader
// takes the first entry whose bounds cover the graph and whose CTA fits.
struct EllVariant {
  int dc, dv, cpt, vpt, maxt;
};
constexpr EllVariant kEllVariants[] = {
    {4, 2, 1, 2, 1024},   // e.g. the toy 3x6 fixture, repetition / surface-like checks
    {7, 3, 3, 5, 192},    // [H | I] extension of a (6,3)-regular code (phenomenological noise):
                          // the identity columns are absorbed by their checks
    {7, 3, 3, 5, 320},    // ... the same graph as ONE segment (the reference's graph constructor)
    {8, 4, 2, 4, 512},
    {12, 6, 1, 2, 1024},
};
constexpr int kNumEllVariants = sizeof(kEllVariants) / sizeof(kEllVariants[0]);

template <class A, bool kSoft = false>
KernelFn ell_kernel_t(int idx) {
  switch (idx) {
    case 0: return decode_ell_kernel<A, 4, 2, 1, 2, 1024, 1, kSoft>;
    case 1: return decode_ell_kernel<A, 7, 3, 3, 5, 192, 5, kSoft>;
    case 2: return decode_ell_kernel<A, 7, 3, 3, 5, 320, 3, kSoft>;
    case 3: return decode_ell_kernel<A, 8, 4, 2, 4, 512, 2, kSoft>;
    default: return decode_ell_kernel<A, 12, 6, 1, 2, 1024, 1, kSoft>;
  }
}

// Single shots on irregular graphs: decode_ell_latency_kernel (kernel_ell_latency.cuh), one
// check and two variables per thread, a cluster with one CTA per segment.
constexpr EllVariant kEllLatVariants[] = {
    {4, 2, 1, 2, 1024},
    {7, 3, 1, 2, 1024},
    {8, 4, 1, 2, 1024},
    {12, 6, 1, 2, 1024},
};
constexpr int kNumEllLatVariants = sizeof(kEllLatVariants) / sizeof(kEllLatVariants[0]);
template <class A>
LatKernelFn ell_lat_kernel_t(int idx) {
  switch (idx) {
    case 0: return decode_ell_latency_kernel<A, 4, 2>;
    case 1: return decode_ell_latency_kernel<A, 7, 3>;
    case 2: return decode_ell_latency_kernel<A, 8, 4>;
    default: return decode_ell_latency_kernel<A, 12, 6>;
  }
}

// int8 and int16 share one build: 32-bit message words, saturation bound from DecodeParams
KernelFn ell_kernel(int arith, int idx) {
  switch (arith) {
    case QB_ARITH_FLOAT: return ell_kernel_t<ArithF32>(idx);
    case QB_ARITH_INT8:
    case QB_ARITH_INT16: return ell_kernel_t<ArithI32>(idx);
    default: return ell_kernel_t<ArithF16>(idx);
  }
}
// ... with the absorbed variables' priors read per shot (qb_decode_batch_soft)
KernelFn ell_soft_kernel(int arith, int idx) {
  switch (arith) {
    case QB_ARITH_FLOAT: return ell_kernel_t<ArithF32, true>(idx);
    case QB_ARITH_INT8:
    case QB_ARITH_INT16: return ell_kernel_t<ArithI32, true>(idx);
    default: return ell_kernel_t<ArithF16, true>(idx);
  }
}
LatKernelFn ell_lat_kernel(int arith, int idx) {
  switch (arith) {
    case QB_ARITH_FLOAT: return ell_lat_kernel_t<ArithF32>(idx);
    case QB_ARITH_INT8:
    case QB_ARITH_INT16: return ell_lat_kernel_t<ArithI32>(idx);
    default: return ell_lat_kernel_t<ArithF16>(idx);
  }
}
uint32_t ell_msg_bytes(int arith) { return arith == QB_ARITH_HALF ? 2u : 4u; }

// two shots per thread on packed fp16 instructions (kernel_ell_h2.cuh): half mode, and int8
// mode when the loader has verified the fp16 form of the Q16 scaling
constexpr int kEllH2MaxT[] = {1024, 160, 320, 512, 1024};
template <bool kI8, bool kSoft = false>
KernelFn ell_h2_kernel_t(int idx) {
  switch (idx) {
    case 0: return decode_ell_h2_kernel<4, 2, 1, 2, 1024, 1, kI8, kSoft>;
    case 1: return decode_ell_h2_kernel<7, 3, 3, 5, 160, 4, kI8, kSoft>;
    case 2: return decode_ell_h2_kernel<7, 3, 3, 5, 320, 2, kI8, kSoft>;
    case 3: return decode_ell_h2_kernel<8, 4, 2, 4, 512, 1, kI8, kSoft>;
    default: return decode_ell_h2_kernel<12, 6, 1, 2, 1024, 1, kI8, kSoft>;
  }
}

uint32_t round_up32(uint32_t x) { return (x + 31u) & ~31u; }

// Threads per segment group so that T*cpt covers the checks and T*vpt the
// variables of every segment.
uint32_t regular_group_threads(const DecodeParams& P, uint32_t cpt, uint32_t vpt) {
  uint32_t want = 32;
  for (uint32_t s = 0; s < P.nseg; ++s) {
    const uint32_t ms = P.segs[s].c1 - P.segs[s].c0;
    const uint32_t ns = P.segs[s].v1 - P.segs[s].v0;
    want = std::max(want, std::max((ms + cpt - 1) / cpt, (ns + vpt - 1) / vpt));
  }
  return round_up32(want);
}

void finish_plan(qb_decoder* h, LaunchPlan& pl) {
  pl.block = pl.cluster ? pl.group_threads : pl.ngroups * pl.group_threads;
  if (pl.items) pl.block = pl.group_threads;
  pl.smem = pl.ell && pl.pair ? ell_h2_smem_bytes(h->P.seg_mmax, static_cast<uint32_t>(pl.ell / 100), pl.block)
            : pl.ell  ? ell_smem_bytes(h->P.seg_mmax, ell_msg_bytes(h->arith),
                                       static_cast<uint32_t>(pl.ell / 100), pl.block)
            : pl.pair ? lean_h2_smem_bytes(h->P.seg_mmax, h->P.syn_w32)
            : pl.lean ? h->smem_lean
                      : h->smem_bytes;
  CUDA_TRY(cudaFuncSetAttribute(pl.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(pl.smem)));
  for (KernelFn extra : {pl.kernel_soft, pl.kernel_dump}) {
    if (extra) {
      CUDA_TRY(cudaFuncSetAttribute(extra, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(pl.smem)));
    }
  }
  if (pl.cluster) {
    pl.ctas_per_sm = 1;
    return;
  }
  int n = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, pl.kernel, static_cast<int>(pl.block),
                                                         pl.smem));
  if (n < 1) fail(QB_RUNTIME_ERROR, "decode kernel does not fit on an SM");
  pl.ctas_per_sm = n;
}

LaunchPlan generic_plan(qb_decoder* h) {
  const DecodeParams& P = h->P;
  LaunchPlan pl{};
  pl.kernel = generic_kernel(h->arith);
  pl.name = "decode_generic_kernel";
  pl.ngroups = std::min<uint32_t>(P.nseg, 8);
  uint32_t T = h->opt_group_threads > 0 ? static_cast<uint32_t>(h->opt_group_threads)
                                        : regular_group_threads(P, 1, 2);
  T = std::max(32u, std::min(round_up32(T), (1024u / pl.ngroups) & ~31u));
  pl.group_threads = T;
  finish_plan(h, pl);
  return pl;
}

// Slot permutation for the lean batch kernels on a (6,3)-regular graph: the variable-side
// gathers / scatters of one warp instruction touch 32 (check, slot) positions; with the
// 14-word block stride a fixed slot can only reach the 16 banks of one parity, so the natural
// order (slot = position in the row) is 2-way conflicted throughout.  Greedy assignment in
// launch order - each edge takes the free slot of its check whose bank is least used by its
// warp instruction so far - then one pass of improving pairwise swaps.  ~1 ms on
// [[784,24,24]]; 2.15 -> ~1.75 wavefronts per access.
void optimise_edge_slots(qb_decoder* h, uint32_t T) {
  const DecodeParams& P = h->P;
  const uint32_t E = P.E;
  if (!h->regular63 || T < 32) T = 0;
  const int64_t key = static_cast<int64_t>(T) * 4 + (T ? h->opt_slot_spread : 0);
  if (h->slot_table_for == key) return;  // the device table is current
  h->slot_table_for = key;
  std::vector<uint8_t> slot(E, 0);
  for (uint32_t e = 0; e < E; ++e) slot[e] = static_cast<uint8_t>(e % 6);
  // The table is a function of the graph, its segments and the thread shape only, and costs
  // ~1 ms to compute on [[784,24,24]] (90 ms with annealing): decoders built again and again
  // for the same code (the reference's callers do that) find it in a small process-wide cache.
  struct SlotCacheEntry {
    uint64_t hash;
    uint32_t E, nseg, T;
    int64_t spread;
    std::vector<uint8_t> slot;
  };
  static std::mutex cache_mu;
  static std::vector<SlotCacheEntry> cache;
  uint64_t hash = 14695981039346656037ull;
  if (h->regular63 && T >= 32) {
    auto mix = [&hash](uint32_t v) {
      hash = (hash ^ v) * 1099511628211ull;
    };
    for (uint32_t v : h->h_var_edges) mix(v);
    for (uint32_t sgi = 0; sgi < P.nseg; ++sgi) {
      mix(P.segs[sgi].c0);
      mix(P.segs[sgi].v0);
    }
    std::lock_guard<std::mutex> lk(cache_mu);
    for (const SlotCacheEntry& c : cache) {
      if (c.hash == hash && c.E == E && c.nseg == P.nseg && c.T == T && c.spread == h->opt_slot_spread) {
        CUDA_TRY(cudaMemcpy(h->d_edge_slot, c.slot.data(), E, cudaMemcpyHostToDevice));
        return;
      }
    }
  }
  if (h->regular63 && T >= 32) {
    constexpr uint32_t kStrideWords = 14;
    std::vector<uint32_t> group_of(E, 0);
    std::vector<std::vector<uint32_t>> groups;
    for (uint32_t s = 0; s < P.nseg; ++s) {
      const SegmentDev& sg = P.segs[s];
      const uint32_t ns = sg.v1 - sg.v0, vpt = (ns + T - 1) / T;
      for (uint32_t k = 0; k < vpt; ++k) {
        for (uint32_t w = 0; w < T / 32; ++w) {
          for (uint32_t i = 0; i < 3; ++i) {
            std::vector<uint32_t> g;
            for (uint32_t l = 0; l < 32; ++l) {
              const uint32_t nl = 32 * w + l + k * T;
              if (nl < ns) g.push_back(h->h_var_edges[(sg.v0 + nl) * 3 + i]);
            }
            if (g.empty()) continue;
            for (uint32_t e : g) group_of[e] = static_cast<uint32_t>(groups.size());
            groups.push_back(std::move(g));
          }
        }
      }
    }
    auto bank = [&](uint32_t e, uint32_t sl) { return (kStrideWords * (e / 6) + sl) & 31u; };
    std::vector<uint8_t> free_mask(E / 6, 0x3f);
    std::fill(slot.begin(), slot.end(), 0xff);
    for (const auto& g : groups) {
      uint8_t used[32] = {};
      for (uint32_t e : g) {
        uint32_t best = 6, best_use = 255;
        for (uint32_t sl = 0; sl < 6; ++sl) {
          if (!((free_mask[e / 6] >> sl) & 1u)) continue;
          const uint32_t u = used[bank(e, sl)];
          if (u < best_use) {
            best_use = u;
            best = sl;
          }
        }
        slot[e] = static_cast<uint8_t>(best);
        free_mask[e / 6] &= static_cast<uint8_t>(~(1u << best));
        ++used[bank(e, best)];
      }
    }
    auto cost = [&](uint32_t gi) {  // sum of squared bank loads of one warp instruction
      uint8_t c[32] = {};
      uint32_t tot = 0;
      for (uint32_t e : groups[gi]) ++c[bank(e, slot[e])];
      for (uint32_t b = 0; b < 32; ++b) tot += static_cast<uint32_t>(c[b]) * c[b];
      return tot;
    };
    for (uint32_t m = 0; m < E / 6; ++m) {
      for (uint32_t a = 0; a < 6; ++a) {
        for (uint32_t b = a + 1; b < 6; ++b) {
          const uint32_t ea = 6 * m + a, eb = 6 * m + b;
          const uint32_t ga = group_of[ea], gb = group_of[eb];
          const uint32_t before = cost(ga) + (gb != ga ? cost(gb) : 0u);
          std::swap(slot[ea], slot[eb]);
          const uint32_t after = cost(ga) + (gb != ga ? cost(gb) : 0u);
          if (after >= before) std::swap(slot[ea], slot[eb]);
        }
      }
    }
    // QB_OPT_SLOT_SPREAD = 2: simulated annealing on top (swap two slots of one check; cost = number of colliding
    // pairs per warp instruction and bank, geometric cooling, fixed seed; 200 moves per edge):
    // 1.72 -> 1.43 wavefronts per access on [[784,24,24]] in 1.9 M moves (~90 ms, once per
    // thread shape - the table is cached), 1.29 in 20 M (QB_SLOT_ANNEAL = number of moves).
    const long moves = h->opt_slot_spread < 2 ? 0 : getenv("QB_SLOT_ANNEAL") ? atol(getenv("QB_SLOT_ANNEAL")) : 200l * E;
    if (moves > 0) {
      std::vector<std::array<int16_t, 32>> cnt(groups.size());
      for (auto& c : cnt) c.fill(0);
      for (uint32_t e = 0; e < E; ++e) ++cnt[group_of[e]][bank(e, slot[e])];
      uint64_t x = 0x9e3779b97f4a7c15ull;
      auto next = [&x] {
        x += 0x9e3779b97f4a7c15ull;
        uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
      };
      const uint32_t M6 = E / 6;
      for (long it = 0; it < moves; ++it) {
        const uint64_t r = next();
        const uint32_t m = static_cast<uint32_t>(r % M6), a = static_cast<uint32_t>((r >> 32) % 6),
                       b = static_cast<uint32_t>((r >> 40) % 6);
        if (a == b) continue;
        const uint32_t ea = 6 * m + a, eb = 6 * m + b, ga = group_of[ea], gb = group_of[eb];
        const uint32_t sa = slot[ea], sb = slot[eb];
        const uint32_t ba0 = bank(ea, sa), ba1 = bank(ea, sb), bb0 = bank(eb, sb), bb1 = bank(eb, sa);
        int d = 0;
        d -= cnt[ga][ba0] - 1; --cnt[ga][ba0];
        d += cnt[ga][ba1]; ++cnt[ga][ba1];
        d -= cnt[gb][bb0] - 1; --cnt[gb][bb0];
        d += cnt[gb][bb1]; ++cnt[gb][bb1];
        const double temp = 1.2 * std::pow(0.001, static_cast<double>(it) / static_cast<double>(moves));
        const bool accept = d <= 0 || std::exp(-d / temp) > static_cast<double>(next() >> 11) * 0x1.0p-53;
        if (accept) {
          slot[ea] = static_cast<uint8_t>(sb);
          slot[eb] = static_cast<uint8_t>(sa);
        } else {
          --cnt[gb][bb1]; ++cnt[gb][bb0]; --cnt[ga][ba1]; ++cnt[ga][ba0];
        }
      }
      if (getenv("QB_SLOT_ANNEAL_VERBOSE")) {
        double tot = 0;
        for (auto& c : cnt) tot += *std::max_element(c.begin(), c.end());
        std::fprintf(stderr, "slot annealing: %.3f wavefronts per variable-side access\n", tot / cnt.size());
      }
    }
  }
  CUDA_TRY(cudaMemcpy(h->d_edge_slot, slot.data(), E, cudaMemcpyHostToDevice));
  if (h->regular63 && T >= 32) {
    std::lock_guard<std::mutex> lk(cache_mu);
    if (cache.size() >= 8) cache.erase(cache.begin());
    cache.push_back({hash, E, P.nseg, T, h->opt_slot_spread, std::move(slot)});
  }
}

void choose_plans(qb_decoder* h);

void make_plans(qb_decoder* h) {
  choose_plans(h);
  // whatever batch plan was chosen, leave a slot table that matches its thread shape
  const bool lean_batch = h->bat.lean && !h->bat.ell;
  optimise_edge_slots(h, lean_batch && h->opt_slot_spread != 0 ? h->bat.group_threads : 0u);
}

void choose_plans(qb_decoder* h) {
  const DecodeParams& P = h->P;
  drop_latency_graphs(h);  // they bake in the kernel and its launch shape
  const bool use_regular = h->regular63 && h->opt_kernel != 1;
  if (h->opt_kernel == 2 && !h->regular63) {
    fail(QB_INVALID_ARGUMENT, "the (6,3)-regular kernels need a (6,3)-regular graph with at most 8 segments");
  }
  if (!use_regular) {
    h->lat = h->bat = generic_plan(h);
    // batch: degree-padded item kernel when the degrees fit an instantiated bound
    if (h->opt_kernel != 1 && h->opt_batch_shape != 1 && P.seg_mmax <= 960 && P.nseg <= kMaxSegments) {
      for (int idx = 0; idx < kNumEllVariants; ++idx) {
        const EllVariant& ev = kEllVariants[idx];
        if (h->max_dc > static_cast<uint32_t>(ev.dc) || h->max_dv > static_cast<uint32_t>(ev.dv)) continue;
        uint32_t want = 32;  // threads so that T * cpt covers the checks, T * vpt the own variables
        for (uint32_t k = 0; k < P.nseg; ++k) {
          const uint32_t ms = P.segs[k].c1 - P.segs[k].c0;
          want = std::max(want, std::max((ms + ev.cpt - 1) / ev.cpt,
                                         (P.ell_nvars[k] + ev.vpt - 1) / ev.vpt));
        }
        const uint32_t T = round_up32(want);
        const bool pair = (h->arith == QB_ARITH_HALF || (h->arith == QB_ARITH_INT8 && h->i8_pair_ok)) &&
                          h->opt_batch_pair != 0 && T <= static_cast<uint32_t>(kEllH2MaxT[idx]);
        if (T > static_cast<uint32_t>(ev.maxt)) continue;
        const size_t smem = pair ? ell_h2_smem_bytes(P.seg_mmax, static_cast<uint32_t>(ev.dc), T)
                                 : ell_smem_bytes(P.seg_mmax, ell_msg_bytes(h->arith),
                                                  static_cast<uint32_t>(ev.dc), T);
        if (smem > static_cast<size_t>(h->max_smem_optin)) continue;
        LaunchPlan pl{};
        pl.items = true;
        pl.lean = true;
        pl.pair = pair;
        pl.ell = 100 * ev.dc + ev.dv;
        pl.kernel = !pair                       ? ell_kernel(h->arith, idx)
                    : h->arith == QB_ARITH_INT8 ? ell_h2_kernel_t<true>(idx)
                                                : ell_h2_kernel_t<false>(idx);
        pl.kernel_dump = ell_dump_kernel(h->arith, idx, pair);
        pl.kernel_soft = !pair                       ? ell_soft_kernel(h->arith, idx)
                         : h->arith == QB_ARITH_INT8 ? ell_h2_kernel_t<true, true>(idx)
                                                     : ell_h2_kernel_t<false, true>(idx);
        pl.name = pair ? "decode_ell_h2_kernel" : "decode_ell_kernel";
        pl.ngroups = 1;
        pl.group_threads = T;
        finish_plan(h, pl);
        h->bat = pl;
        break;
      }
    }
    // single shots: the degree-padded cluster kernel (mapped / doorbell / memcpy protocols)
    h->lat_lean_kernel = nullptr;
    h->lat_is_ell = false;
    if (h->opt_kernel != 1 && h->opt_latency_shape != 1 && P.syn_w32 <= kInlineSynWords &&
        P.nseg <= kMaxSegments) {
      for (int idx = 0; idx < kNumEllLatVariants; ++idx) {
        const EllVariant& ev = kEllLatVariants[idx];
        if (h->max_dc > static_cast<uint32_t>(ev.dc) || h->max_dv > static_cast<uint32_t>(ev.dv)) continue;
        uint32_t want = 32;
        for (uint32_t k = 0; k < P.nseg; ++k) {
          const uint32_t ms = P.segs[k].c1 - P.segs[k].c0;
          want = std::max(want, std::max(ms, (P.ell_nvars[k] + 1) / 2));
        }
        const uint32_t T = round_up32(want);
        const size_t smem = ell_latency_smem_bytes(P.seg_mmax, P.seg_nmax, ell_msg_bytes(h->arith),
                                                   static_cast<uint32_t>(ev.dc), T);
        if (T > 1024 || smem > static_cast<size_t>(h->max_smem_optin)) continue;
        h->lat_lean_kernel = ell_lat_kernel(h->arith, idx);
        h->lat_is_ell = true;
        h->lat_lean_block = T;
        h->lat_lean_smem = smem;
        CUDA_TRY(cudaFuncSetAttribute(h->lat_lean_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        break;
      }
    }
    return;
  }
  // single shot: the lean cluster kernel, CTA rank = segment (a cluster of one for a decoder
  // built from a plain graph: ONE CTA per shot); QB_OPT_LATENCY_SHAPE = 1 asks for one CTA
  // per shot whatever the segment count, which is the generic kernel's shape
  h->lat = generic_plan(h);
  h->lat_lean_kernel = nullptr;
  h->lat_is_ell = false;
  if (h->opt_latency_shape != 1 && P.seg_mmax <= 960 && P.seg_nmax <= 960 * 2 &&
      P.syn_w32 <= kInlineSynWords) {
    // shape 3 = one check and ONE variable per thread: the shortest dependent chain per
    // iteration; pays on small codes in float mode ([[144,12,12]]: 4.19 -> 3.62 us for 10
    // iterations as a 2-CTA cluster of 160 threads, 4.83 -> 4.26 as one CTA of 288), loses on
    // [[784,24,24]], where it means 25 warps per barrier (6.66 -> 7.10)
    const bool small_float = h->arith == QB_ARITH_FLOAT && regular_group_threads(P, 1, 1) <= 320;
    for (int npt : {3, 1, 2}) {
      if (h->opt_latency_npt ? npt != h->opt_latency_npt : (npt == 3 && !small_float)) continue;
      const uint32_t T = npt == 3 ? regular_group_threads(P, 1, 1) : regular_group_threads(P, npt, 2 * npt);
      if (T > 1024) continue;
      h->lat_lean_kernel =
          lean_latency_kernel(h->arith, npt, h->fast_ok && h->opt_fast != 0);
      h->lat_lean_block = T;
      h->lat_lean_smem = lean_latency_smem_bytes(P.seg_mmax, P.seg_nmax,
                                                 h->arith == QB_ARITH_HALF ? 3 : h->arith);
      CUDA_TRY(cudaFuncSetAttribute(h->lat_lean_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(h->lat_lean_smem)));
      break;
    }
  }
  bool bat_done = false;
  const bool word_msgs = h->arith == QB_ARITH_FLOAT || h->arith == QB_ARITH_INT16;
  const bool fast = h->fast_ok && h->opt_fast != 0 && (!word_msgs || h->tab_ok);
  if (h->opt_batch_shape != 1 && P.seg_mmax <= 960) {
    // work item = (shot, segment): lean item kernel; first variant whose CTA fits
    // (measured on [[784,24,24]]: the packed fp16 kernel prefers the spill-free
    // 96-register build at four CTAs per SM)
    const bool i8 = h->arith == QB_ARITH_INT8;
    const bool pair_wanted = (h->arith == QB_ARITH_HALF || (i8 && h->i8_pair_ok)) && h->opt_batch_pair != 0;
    // measured on [[784,24,24]] (fp32): with early stop the 64-register build at six CTAs per
    // SM wins (107.9 vs 101.1 M/s); at a fixed iteration count the 48-register build at eight
    // CTAs per SM hides the dependent chains better (24.8 vs 23.5 M/s)
    const int order_f32[] = {2, 4, 3, 6, 1, 1, 1}, order_h2[] = {8, 3, 6, 1, 1, 1, 1},
              order_fixed[] = {2, 11, 4, 3, 6, 1, 1};
    // (int16 on fp32 instructions has no conversion chains to hide: 64 registers, no spills, win
    // at a fixed count too: 25.0 vs 23.5 M/s)
    const int* order_auto = pair_wanted ? order_h2 : (P.early || h->arith == QB_ARITH_INT16) ? order_f32 : order_fixed;
    for (int idx = 0; idx < 7 && !bat_done; ++idx) {
      const int variant = h->opt_batch_npt ? static_cast<int>(h->opt_batch_npt) : order_auto[idx];
      const LeanVariant& lv = kLeanVariants[variant - 1];
      if (lv.maxt == 0) {
        if (h->opt_batch_npt) fail(QB_INVALID_ARGUMENT, "QB_OPT_BATCH_VARIANT: that variant is retired (1, 2, 3, 4, 6, 8, 11 exist)");
        continue;
      }
      const uint32_t T = regular_group_threads(P, lv.cpt, lv.vpt);
      if (T <= static_cast<uint32_t>(lv.maxt)) {
        KernelFn i8_pair = nullptr;
        if (i8 && pair_wanted) {
          i8_pair = fast ? lean_h2_i8_kernel_tf<true>(variant) : lean_h2_i8_kernel_tf<false>(variant);
          if (!i8_pair && !h->opt_batch_npt) continue;  // shape not built for int8 pairs: next one
        }
        KernelFn h2_pair = nullptr;
        if (!i8 && pair_wanted) {
          h2_pair = fast ? lean_h2_kernel_tf<true>(variant) : lean_h2_kernel_tf<false>(variant);
          if (!h2_pair && !h->opt_batch_npt) continue;  // shape not built for pairs: next one
        }
        const bool pair = pair_wanted && (i8 ? i8_pair != nullptr : h2_pair != nullptr);
        LaunchPlan pl{};
        pl.regular = true;
        pl.items = true;
        pl.lean = true;
        pl.npt = variant;
        pl.pair = pair;
        pl.kernel = !pl.pair ? lean_kernel(h->arith, variant, fast) : i8 ? i8_pair : h2_pair;
        pl.kernel_dump = pl.pair ? lean_h2_dump_kernel(i8, variant, fast) : lean_dump_kernel(h->arith, variant, fast);
        pl.name = pl.pair ? "decode_lean_h2_kernel" : "decode_lean_kernel";
        pl.ngroups = 1;
        pl.group_threads = T;
        finish_plan(h, pl);
        h->bat = pl;
        bat_done = true;
      } else if (h->opt_batch_npt) {
        fail(QB_INVALID_ARGUMENT, "requested batch kernel variant does not fit this code");
      }
    }
  }
  if (!bat_done) h->bat = generic_plan(h);  // QB_OPT_BATCH_SHAPE = 1, or segments over 960 checks
}

void launch_plan(qb_decoder* h, const LaunchPlan& pl, const ShotIO& io, unsigned grid,
                 cudaStream_t stream) {
  DecodeParams P = h->P;
  P.ngroups = pl.ngroups;
  P.group_threads = pl.group_threads;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(pl.block);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  if (pl.cluster) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = P.nseg;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  KernelFn kernel = pl.kernel;
  if (io.soft) {
    if (!pl.kernel_soft) fail(QB_RUNTIME_ERROR, "launch plan has no per-shot-prior kernel");
    kernel = pl.kernel_soft;
  }
  if (io.q_dump && pl.items) {
    if (!pl.kernel_dump) {
      fail(QB_INVALID_ARGUMENT, "decode_batch_debug: this batch kernel shape has no message-dump "
                                "instantiation (the loader's own choices have one)");
    }
    kernel = pl.kernel_dump;
  }
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel, P, io));
  ++h->launches;
}

void ensure_batch(qb_decoder* h, uint64_t shots, bool want_resid, bool want_soft = false) {
  if (shots <= h->batch_cap && (!want_resid || h->b_res) && (!want_soft || h->b_soft)) return;
  const uint64_t cap = std::max<uint64_t>(shots, h->batch_cap);
  const bool soft = want_soft || h->b_soft != nullptr;
  free_batch(h);
  const DecodeParams& P = h->P;
  if (soft) CUDA_TRY(cudaMalloc(&h->b_soft, cap * P.M * h->soft_bytes));
  CUDA_TRY(cudaMalloc(&h->b_syn, cap * P.syn_w32 * 4));
  CUDA_TRY(cudaMalloc(&h->b_est, cap * P.est_w32 * 4));
  CUDA_TRY(cudaMalloc(&h->b_res, cap * P.syn_w32 * 4));
  CUDA_TRY(cudaMalloc(&h->b_iters, cap * P.nseg * 4));
  CUDA_TRY(cudaMalloc(&h->b_conv, cap * P.nseg));
  CUDA_TRY(cudaMalloc(&h->c_err, cap * P.est_w32 * 4));
  h->batch_cap = cap;
}

uint64_t resident_ctas(qb_decoder* h) {
  int per_sm = h->bat.ctas_per_sm;
  if (h->opt_batch_ctas > 0) per_sm = std::min<int>(per_sm, static_cast<int>(h->opt_batch_ctas));
  return static_cast<uint64_t>(per_sm) * h->sm_count;
}

// Shots per syndrome tile of the lean batch kernel (one TMA bulk copy + one queue ticket
// each): as large as leaves every resident CTA at least four tiles; 1 for small batches.
uint32_t batch_tile(qb_decoder* h, uint64_t shots) {
  if (!(h->bat.lean && !h->bat.ell)) return 1;
  if (h->bat.pair) {  // two shots per item: tiles hold whole pairs (an even number of shots)
    const uint64_t per_seg = std::max<uint64_t>(1, resident_ctas(h) / h->P.nseg);
    uint32_t k = h->opt_batch_tile > 0 ? static_cast<uint32_t>(h->opt_batch_tile) & ~1u : 0u;
    if (k >= 2) return k;
    for (k = kMaxTile; k > 2; k >>= 1) {
      if ((shots + k - 1) / k >= 4 * per_seg) return k;
    }
    return 2;
  }
  const uint64_t per_seg = std::max<uint64_t>(1, resident_ctas(h) / h->P.nseg);
  if (h->opt_batch_tile > 0) return static_cast<uint32_t>(h->opt_batch_tile);
  for (uint32_t k = kMaxTile; k > 1; k >>= 1) {
    if ((shots + k - 1) / k >= 4 * per_seg) return k;
  }
  return 1;
}

unsigned batch_grid(qb_decoder* h, uint64_t shots) {
  const uint64_t resident = resident_ctas(h);
  if (h->bat.items) {  // equal numbers of CTAs per segment
    const uint64_t nseg = h->P.nseg;
    const uint64_t tile = batch_tile(h, shots);
    const uint64_t items = h->bat.ell && h->bat.pair ? (shots + 1) / 2 : (shots + tile - 1) / tile;
    const uint64_t per_seg = std::max<uint64_t>(1, std::min<uint64_t>(resident / nseg, items));
    return static_cast<unsigned>(per_seg * nseg);
  }
  return static_cast<unsigned>(std::min<uint64_t>(shots, resident));
}

// The per-shot-prior path exists where the loader absorbs degree-1 variables into their
// checks: the degree-padded batch kernels (kernel_ell.cuh).
void require_soft(qb_decoder* h, const char* who) {
  if (!h->bat.kernel_soft) {
    fail(QB_INVALID_ARGUMENT,
         std::string(who) + ": per-shot priors need a graph served by the degree-padded kernel "
                            "(e.g. the extended graph [H | I]); this decoder's batch kernel is " +
             h->bat.name);
  }
}

void run_batch_device(qb_decoder* h, uint64_t shots, const uint32_t* d_syn, uint32_t* d_est,
                      uint32_t* d_res, uint8_t* d_conv, uint32_t* d_iters, cudaStream_t stream,
                      int sched_slot = -1, const void* d_soft = nullptr, int64_t dump_shot = -1) {
  if (shots == 0) return;
  if (sched_slot < 0) sched_slot = 1 + kPipeSlots + static_cast<int>(h->sched_next++ % kSchedRing);
  if (shots > 0x7fff0000ull) fail(QB_INVALID_ARGUMENT, "too many shots for one launch");
  ShotIO io{};
  io.soft = d_soft;
  io.soft_bytes = h->soft_bytes;
  if (dump_shot >= 0) {  // parity hook: messages of one shot of the batch
    io.q_dump = h->d_qdump;
    io.r_dump = h->d_rdump;
    io.dump_shot = static_cast<uint32_t>(dump_shot);
  }
  io.nshots = shots;
  io.syn = d_syn;
  io.est = d_est;
  io.resid = d_res;
  io.conv = d_conv;
  io.iters = d_iters;
  io.sched = h->d_sched + sched_slot * kSchedWords;  // concurrent launches need their own tickets
  io.tile = batch_tile(h, shots);
  launch_plan(h, h->bat, io, batch_grid(h, shots), stream);
}

template <typename F>
qb_status guarded(qb_decoder* h, F&& f) {
  try {
    if (h) {
      cudaError_t e = cudaSetDevice(h->device);
      if (e != cudaSuccess) fail(QB_RUNTIME_ERROR, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    }
    f();
    return QB_OK;
  } catch (const StatusError& e) {
    (h ? h->err : g_create_error) = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    (h ? h->err : g_create_error) = e.what();
    return QB_RUNTIME_ERROR;
  }
}

void launch_lean_latency(qb_decoder* h, const ShotIO& io, const LatencyCtl& ctl,
                         const SynInline& syn) {
  DecodeParams P = h->P;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(P.nseg);
  cfg.blockDim = dim3(h->lat_lean_block);
  cfg.dynamicSmemBytes = h->lat_lean_smem;
  cfg.stream = h->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P.nseg;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, h->lat_lean_kernel, P, io, ctl, syn));
  ++h->launches;
}

// Retires the persistent doorbell kernel (if any) and waits for it.
void stop_doorbell(qb_decoder* h) {
  if (!h->db_running) return;
  volatile uint32_t* db = h->h_db;
  for (int k = 0; k < 4; ++k) db[8 * k] = kDoorbellExit;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  cudaStreamSynchronize(h->stream);
  h->db_running = false;
}

// Waits until `ready()` holds, with a watchdog that falls back to the runtime.
template <typename Ready>
void spin_until(qb_decoder* h, Ready&& ready, bool persistent) {
  const auto t0 = std::chrono::steady_clock::now();
  uint64_t spins = 0;
  while (!ready()) {
    if ((++spins & 0xffff) == 0) {
      const cudaError_t q = cudaStreamQuery(h->stream);
      if (q != cudaErrorNotReady) {
        CUDA_TRY(cudaStreamSynchronize(h->stream));
        if (ready()) break;
        if (persistent) {
          h->db_running = false;  // retired while we were ringing: caller relaunches
          fail(QB_RUNTIME_ERROR, "doorbell kernel retired");
        }
        fail(QB_RUNTIME_ERROR, "decode kernel finished without signalling completion");
      }
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(20)) {
        fail(QB_RUNTIME_ERROR, "decode kernel timed out");
      }
    }
  }
}

// True when every sector of every segment's record carries `seq`.
bool records_ready(const qb_decoder* h, uint32_t seq) {
  const DecodeParams& P = h->P;
  const volatile uint32_t* rec = h->h_rec;
  for (uint32_t s = P.nseg; s-- > 0;) {
    const uint32_t nd = record_data_words(P.segs[s].v1 - P.segs[s].v0, P.segs[s].c1 - P.segs[s].c0);
    for (uint32_t k = sector_words(nd) / 8; k-- > 0;) {
      if (rec[s * h->rec_stride + 8 * k] != seq) return false;
    }
  }
  // The data words are read after this returns: keep those loads behind the tag loads on
  // weakly ordered hosts (aarch64 / Grace).  The protocol relies on each 32-byte sector
  // store of the GPU (eight adjacent lanes of one STG over PCIe / C2C) becoming visible to
  // the host as a unit - true of every platform this runs on, not an architectural promise.
  std::atomic_thread_fence(std::memory_order_acquire);
  return true;
}

// OR `words` local words (bit 0 = global bit `bit0`) into a packed vector.
void or_shifted(uint32_t* dst, uint32_t dst_words, const uint32_t* rec, uint32_t first_data,
                uint32_t words, uint32_t bit0) {
  for (uint32_t w = 0; w < words; ++w) {
    const uint32_t v = rec[sector_pos(first_data + w)];
    if (!v) continue;
    const uint32_t b = bit0 + 32u * w, sh = b & 31u, i = b >> 5;
    dst[i] |= v << sh;
    if (sh && i + 1 < dst_words) dst[i + 1] |= v >> (32u - sh);
  }
}

// Sectored per-segment records -> the reference's packed layout.
void unpack_records(qb_decoder* h, uint64_t* estimate, uint64_t* residual, uint8_t* converged,
                    uint32_t* iterations) {
  const DecodeParams& P = h->P;
  uint32_t* est = reinterpret_cast<uint32_t*>(estimate);
  uint32_t* res = reinterpret_cast<uint32_t*>(residual);
  std::memset(est, 0, P.est_w32 * 4);
  if (res) std::memset(res, 0, P.syn_w32 * 4);
  uint64_t ns_max = 0;
  for (uint32_t s = 0; s < P.nseg; ++s) {
    const uint32_t* rec = h->h_rec + s * h->rec_stride;
    const uint32_t nv = P.segs[s].v1 - P.segs[s].v0, nc = P.segs[s].c1 - P.segs[s].c0;
    const uint32_t ews = (nv + 31u) >> 5, pws = (nc + 31u) >> 5;
    or_shifted(est, P.est_w32, rec, 0, ews, P.segs[s].v0);
    if (res) or_shifted(res, P.syn_w32, rec, ews, pws, P.segs[s].c0);
    converged[s] = static_cast<uint8_t>(rec[sector_pos(ews + pws)]);
    iterations[s] = rec[sector_pos(ews + pws + 1)];
    const uint64_t ns = static_cast<uint64_t>(rec[sector_pos(ews + pws + 2)]) |
                        (static_cast<uint64_t>(rec[sector_pos(ews + pws + 3)]) << 32);
    ns_max = std::max(ns_max, ns);
  }
  h->last_kernel_ns = ns_max;
}

void single_shot(qb_decoder* h, const uint64_t* syndrome, uint64_t* estimate, uint64_t* residual,
                 uint8_t* converged, uint32_t* iterations, bool debug, const void* soft = nullptr) {
  const DecodeParams& P = h->P;
  if (!syndrome || !estimate || !converged || !iterations) {
    fail(QB_INVALID_ARGUMENT, "decode: NULL buffer");
  }
  const int io_mode = static_cast<int>(h->opt_latency_io);
  const bool lean = h->lat_lean_kernel != nullptr;
  const bool doorbell = io_mode == 2 && lean && !debug && P.syn_w32 <= 28;
  const size_t soft_row = static_cast<size_t>(P.M) * h->soft_bytes;
  // memcpy protocol: [soft values | syndrome words] travel as ONE H2D copy (a second copy node
  // in the graph measured +3 us, a third +10 us)
  const size_t soft_pad = (soft_row + 15) & ~static_cast<size_t>(15);
  const size_t syn_bytes = static_cast<size_t>(P.syn_w32) * 4;
  if (soft) {
    if (!(lean && h->lat_is_ell)) {
      fail(QB_INVALID_ARGUMENT, "decode_soft: per-shot priors need a graph whose single shots run the "
                                "degree-padded cluster kernel (e.g. the extended graph [H | I])");
    }
    if (!h->h_soft1) {
      CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&h->h_soft1),
                             std::max(static_cast<size_t>(P.M) * 4, soft_pad + syn_bytes), cudaHostAllocMapped));
      CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->d_soft1_map), h->h_soft1, 0));
      CUDA_TRY(cudaMalloc(&h->d_soft1_dev, soft_pad + syn_bytes));
    }
    // mapped / doorbell protocols read the values over PCIe: integer modes are staged widened
    // to int32 (a warp then fetches one full 128-byte line, as the float modes do; int8 rows
    // read as 32-byte pieces measured +2.7 us per shot)
    if (io_mode != 1 && h->soft_bytes < 4) {
      int32_t* dst = reinterpret_cast<int32_t*>(h->h_soft1);
      if (h->soft_bytes == 1) {
        const int8_t* src = static_cast<const int8_t*>(soft);
        for (uint32_t m = 0; m < P.M; ++m) dst[m] = src[m];
      } else {
        const int16_t* src = static_cast<const int16_t*>(soft);
        for (uint32_t m = 0; m < P.M; ++m) dst[m] = src[m];
      }
    } else {
      std::memcpy(h->h_soft1, soft, soft_row);
    }
  }
  // a resident doorbell kernel was launched either with or without the soft pointer
  if (!doorbell || (h->db_running && h->db_soft != (soft != nullptr))) stop_doorbell(h);
  uint32_t seq = ++h->seq;
  if (seq == kDoorbellExit || seq == 0) seq = h->seq = 1;
  ShotIO io{};
  io.nshots = 1;
  io.sched = h->d_sched;
  io.seq = seq;
  if (debug) {
    io.q_dump = h->d_qdump;
    io.r_dump = h->d_rdump;
  }
  const bool mapped = io_mode != 1;

  if (lean) {
    LatencyCtl ctl{};
    ctl.first_seq = seq;
    ctl.rec = mapped ? h->d_rec_map : h->d_rec_dev;
    ctl.rec_stride = h->rec_stride;
    ctl.soft = soft ? (mapped ? h->d_soft1_map : h->d_soft1_dev) : nullptr;
    ctl.soft_bytes = mapped ? 4u : h->soft_bytes;
    SynInline syn{};
    if (doorbell) {
      // ---- persistent cluster: ring the doorbell, wait for the records
      volatile uint32_t* db = h->h_db;
      volatile uint32_t* alive = h->h_db + 32;
      const uint32_t* syn32 = reinterpret_cast<const uint32_t*>(syndrome);
      for (int attempt = 0;; ++attempt) {
        if (!h->db_running || *alive == 0u) {
          if (h->db_running) CUDA_TRY(cudaStreamSynchronize(h->stream));
          for (int k = 0; k < 32; ++k) db[k] = 0;
          *alive = 1u;
          std::atomic_thread_fence(std::memory_order_seq_cst);
          ctl.mode = 2;
          ctl.doorbell = h->d_db;
          ctl.alive = h->d_db + 32;
          ctl.idle_ns = static_cast<uint64_t>(h->opt_idle_ms) * 1000000ull;
          launch_lean_latency(h, io, ctl, syn);
          h->db_running = true;
          h->db_soft = soft != nullptr;
        }
        for (uint32_t i = 0; i < P.syn_w32; ++i) db[sector_pos(i)] = syn32[i];
        std::atomic_thread_fence(std::memory_order_release);
        for (int k = 0; k < 4; ++k) db[8 * k] = seq;
        try {
          spin_until(h, [&] { return records_ready(h, seq); }, true);
          break;
        } catch (const StatusError&) {
          if (h->db_running || attempt >= 2) throw;  // a real failure, or retiring repeatedly
        }
      }
    } else if (mapped) {
      ctl.mode = 0;  // syndrome travels in the kernel parameters
      std::memcpy(syn.w, syndrome, P.syn_w32 * 4);
      launch_lean_latency(h, io, ctl, syn);
      spin_until(h, [&] { return records_ready(h, seq); }, false);
    } else {
      ctl.mode = 1;  // the paper's protocol: H2D copy, kernel, D2H copy, synchronize
      if (soft) {
        std::memcpy(h->h_soft1 + soft_pad, syndrome, syn_bytes);
        io.syn = reinterpret_cast<const uint32_t*>(h->d_soft1_dev + soft_pad);
      } else {
        std::memcpy(h->h_in, syndrome, syn_bytes);
        io.syn = h->d_in_dev;
      }
      const bool timed = h->opt_latency_events != 0;
      if (timed && !h->ev0) {
        CUDA_TRY(cudaEventCreate(&h->ev0));
        CUDA_TRY(cudaEventCreate(&h->ev1));
      }
      cudaGraphExec_t* graphs = soft ? h->lat_graph_soft : h->lat_graph;
      auto enqueue = [&] {
        if (soft) {
          CUDA_TRY(cudaMemcpyAsync(h->d_soft1_dev, h->h_soft1, soft_pad + syn_bytes,
                                   cudaMemcpyHostToDevice, h->stream));
        } else {
          CUDA_TRY(cudaMemcpyAsync(h->d_in_dev, h->h_in, syn_bytes, cudaMemcpyHostToDevice, h->stream));
        }
        launch_lean_latency(h, io, ctl, syn);
        CUDA_TRY(cudaMemcpyAsync(h->h_rec, h->d_rec_dev,
                                 static_cast<size_t>(h->rec_stride) * P.nseg * 4,
                                 cudaMemcpyDeviceToHost, h->stream));
      };
      if (h->opt_latency_graph != 0 && !debug) {
        const uint32_t g = h->lat_graph_flip ^= 1u;
        seq = 0x7ffffff0u + g;  // the record tag baked into graph g
        if (!graphs[g]) {
          ctl.first_seq = seq;
          io.seq = seq;
          cudaGraph_t graph = nullptr;
          CUDA_TRY(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
          try {
            enqueue();
          } catch (...) {
            cudaStreamEndCapture(h->stream, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
          }
          CUDA_TRY(cudaStreamEndCapture(h->stream, &graph));
          const cudaError_t ie = cudaGraphInstantiate(&graphs[g], graph, 0);
          cudaGraphDestroy(graph);
          CUDA_TRY(ie);
          --h->launches;  // the capture enqueued nothing
        }
        if (timed) CUDA_TRY(cudaEventRecord(h->ev0, h->stream));
        CUDA_TRY(cudaGraphLaunch(graphs[g], h->stream));
        ++h->launches;
      } else {
        if (timed) CUDA_TRY(cudaEventRecord(h->ev0, h->stream));
        enqueue();
      }
      if (timed) CUDA_TRY(cudaEventRecord(h->ev1, h->stream));
      if (h->opt_latency_wait != 0 && !timed) {
        // the D2H copy IS the completion signal: every 32-byte sector of the record carries
        // the shot's tag (the previous shot left the other graph's tag behind), so the host
        // can watch the pinned destination instead of paying cudaStreamSynchronize's wake-up
        // (-3 us); the next call's operations are stream-ordered behind this one either way
        spin_until(h, [&] { return records_ready(h, seq); }, false);
      } else {
        CUDA_TRY(cudaStreamSynchronize(h->stream));
      }
      if (timed) {
        float ms = 0.0f;
        CUDA_TRY(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
        h->last_event_ns = static_cast<uint64_t>(static_cast<double>(ms) * 1e6);
      }
      if (!records_ready(h, seq)) fail(QB_RUNTIME_ERROR, "decode kernel produced no record");
    }
    unpack_records(h, estimate, residual, converged, iterations);
    return;
  }

  // ---- graphs neither cluster kernel covers (or QB_OPT_KERNEL = 1 / QB_OPT_LATENCY_SHAPE = 1):
  // the generic CSR kernel, one CTA, results to mapped memory + flag or by memcpy
  volatile uint32_t* h_flag = reinterpret_cast<volatile uint32_t*>(h->h_out + h->off_flag);
  unsigned char* out = mapped ? h->d_out_map : h->d_out_dev;
  io.est = reinterpret_cast<uint32_t*>(out);
  io.resid = reinterpret_cast<uint32_t*>(out + h->off_res);
  io.conv = out + h->off_conv;
  io.iters = reinterpret_cast<uint32_t*>(out + h->off_iters);
  io.kernel_ns = reinterpret_cast<uint64_t*>(out + h->off_ns);
  io.flag = reinterpret_cast<volatile uint32_t*>(out + h->off_flag);
  std::memcpy(h->h_in, syndrome, P.syn_w32 * 4);
  io.syn = mapped ? h->d_in_map : h->d_in_dev;
  if (mapped) {
    launch_plan(h, h->lat, io, 1, h->stream);
    spin_until(h, [&] { return *h_flag == seq; }, false);
  } else {
    CUDA_TRY(cudaMemcpyAsync(h->d_in_dev, h->h_in, P.syn_w32 * 4, cudaMemcpyHostToDevice, h->stream));
    launch_plan(h, h->lat, io, 1, h->stream);
    CUDA_TRY(cudaMemcpyAsync(h->h_out, h->d_out_dev, h->out_bytes, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
  }
  std::memcpy(estimate, h->h_out, P.est_w32 * 4);
  if (residual) std::memcpy(residual, h->h_out + h->off_res, P.syn_w32 * 4);
  std::memcpy(converged, h->h_out + h->off_conv, P.nseg);
  std::memcpy(iterations, h->h_out + h->off_iters, P.nseg * 4);
  std::memcpy(&h->last_kernel_ns, h->h_out + h->off_ns, 8);
}

}  // namespace

qb_status set_option_unchecked(qb_decoder* h, int option, int64_t value);

extern "C" {

const char* qb_version(void) { return "qldpc_b200 0.1 (sm_100a)"; }

const char* qb_last_error(const qb_decoder* h) {
  return h ? h->err.c_str() : g_create_error.c_str();
}

qb_status qb_device_info(int device, char* name, size_t name_len, int* sm_count, int* cc_major,
                         int* cc_minor) {
  return guarded(nullptr, [&] {
    cudaDeviceProp prop{};
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (name && name_len) {
      std::strncpy(name, prop.name, name_len - 1);
      name[name_len - 1] = 0;
    }
    if (sm_count) *sm_count = prop.multiProcessorCount;
    if (cc_major) *cc_major = prop.major;
    if (cc_minor) *cc_minor = prop.minor;
  });
}

qb_status qb_measure_smem_bandwidth(int device, double* gbs_32bit, double* gbs_128bit) {
  return guarded(nullptr, [&] {
    CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop{};
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    float* sink = nullptr;
    CUDA_TRY(cudaMalloc(&sink, sizeof(float)));
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    const size_t smem = kBwWords * sizeof(float);
    const unsigned grid = static_cast<unsigned>(prop.multiProcessorCount);
    const uint32_t iters = 4000;
    auto run = [&](auto kern) {
      CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
      double best = 0.0;
      for (int rep = 0; rep < 5; ++rep) {
        CUDA_TRY(cudaEventRecord(e0));
        kern<<<grid, kBwThreads, smem>>>(iters, sink);
        CUDA_TRY(cudaEventRecord(e1));
        CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        const double bytes = 2.0 * smem * static_cast<double>(iters) * grid;  // load + store
        best = std::max(best, bytes / (ms * 1e-3) / 1e9);
      }
      return best;
    };
    const double g32 = run(smem_bandwidth_kernel<1>);
    const double g128 = run(smem_bandwidth_kernel<4>);
    if (gbs_32bit) *gbs_32bit = g32;
    if (gbs_128bit) *gbs_128bit = g128;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
  });
}

qb_status qb_host_alloc(void** out, size_t bytes) {
  return guarded(nullptr, [&] {
    if (!out) fail(QB_INVALID_ARGUMENT, "qb_host_alloc: NULL out");
    CUDA_TRY(cudaHostAlloc(out, std::max<size_t>(bytes, 1), cudaHostAllocPortable));
  });
}

void qb_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

qb_status qb_decoder_create(const qb_graph* graph, const qb_segment* segments,
                            uint32_t num_segments, const qb_config* config, int device,
                            qb_decoder** out) {
  qb_decoder* h = nullptr;
  const qb_status st = guarded(nullptr, [&] {
    if (!out) fail(QB_INVALID_ARGUMENT, "out handle is NULL");
    *out = nullptr;
    validate_graph(graph);
    validate_config_common(graph, config);
    const uint32_t M = graph->num_checks, N = graph->num_vars, E = graph->num_edges;
    const bool has_priors = config->priors != nullptr && config->num_priors != 0;
    const int arith = config->arithmetic;

    // ---- priors (decoder.cpp:82-132)
    std::vector<float> gamma_f;
    std::vector<int32_t> gamma_i;
    uint32_t alpha_fx = 0;
    int32_t kmax = 0;
    if (arith == QB_ARITH_INT8 || arith == QB_ARITH_INT16) {
      kmax = arith == QB_ARITH_INT8 ? 127 : 32767;
      const double scale = config->quant_scale != 0.0 ? config->quant_scale
                                                      : (arith == QB_ARITH_INT8 ? 8.0 : 256.0);
      if (!(scale > 0.0) || !std::isfinite(scale)) {
        fail(QB_INVALID_ARGUMENT, "DecoderConfig: quant_scale must be positive and finite");
      }
      alpha_fx = static_cast<uint32_t>(std::lround(config->alpha * 65536.0));
      if (alpha_fx == 0) {
        fail(QB_INVALID_ARGUMENT,
             "DecoderConfig: alpha is too small for the fixed-point message scaling");
      }
      uint64_t max_degree = 0;
      for (uint32_t n = 0; n < N; ++n) {
        max_degree = std::max<uint64_t>(max_degree,
                                        graph->var_offsets[n + 1] - graph->var_offsets[n]);
      }
      if (max_degree + 1 > static_cast<uint64_t>(std::numeric_limits<int32_t>::max() / kmax)) {
        fail(QB_INVALID_ARGUMENT,
             "DecoderConfig: variable degree too large for 32-bit accumulation in this "
             "integer mode");
      }
      gamma_i.resize(N);
      for (uint32_t n = 0; n < N; ++n) {
        const double p = has_priors ? config->priors[n] : 1.0;
        if (!std::isfinite(p)) {
          fail(QB_INVALID_ARGUMENT,
               "DecoderConfig: prior at variable " + std::to_string(n) + " is not finite");
        }
        const int32_t qv = quantize_saturate(p, scale, kmax);
        if (qv == 0) {
          fail(QB_INVALID_ARGUMENT, "DecoderConfig: prior at variable " + std::to_string(n) +
                                        " quantizes to 0 and would make the decoder inert; "
                                        "increase quant_scale");
        }
        gamma_i[n] = qv;
      }
    } else {
      gamma_f.resize(N);
      for (uint32_t n = 0; n < N; ++n) {
        const double p = has_priors ? config->priors[n] : 1.0;
        if (!std::isfinite(p)) {
          fail(QB_INVALID_ARGUMENT,
               "DecoderConfig: prior at variable " + std::to_string(n) + " is not finite");
        }
        // -0.0 and +0.0 priors are indistinguishable to the reference's arithmetic
        // (sign tests are `< 0`); storing +0.0 lets the kernels read signs as bits.
        gamma_f[n] = static_cast<float>(p) + 0.0f;
      }
    }

    // ---- segments (decoder.cpp:406-424)
    std::vector<qb_segment> segs;
    if (segments == nullptr || num_segments == 0) {
      segs.push_back({0, M, 0, N});
    } else {
      segs.assign(segments, segments + num_segments);
    }
    if (segs.size() > static_cast<size_t>(kMaxSegments)) {
      fail(QB_INVALID_ARGUMENT, "at most " + std::to_string(kMaxSegments) + " segments");
    }
    std::vector<uint32_t> edge_check(E);
    for (uint32_t m = 0; m < M; ++m) {
      for (uint32_t e = graph->check_offsets[m]; e < graph->check_offsets[m + 1]; ++e) {
        edge_check[e] = m;
      }
    }
    uint32_t next_c = 0, next_v = 0;
    for (const qb_segment& s : segs) {
      if (s.check_begin != next_c || s.var_begin != next_v || s.check_end <= s.check_begin ||
          s.var_end <= s.var_begin || s.check_end > M || s.var_end > N) {
        fail(QB_INVALID_ARGUMENT, "segments must tile the checks and variables in order");
      }
      for (uint32_t e = graph->check_offsets[s.check_begin];
           e < graph->check_offsets[s.check_end]; ++e) {
        const uint32_t v = graph->edge_var[e];
        if (v < s.var_begin || v >= s.var_end) {
          fail(QB_INVALID_ARGUMENT, "segments are not block-diagonal: an edge leaves its block");
        }
      }
      next_c = s.check_end;
      next_v = s.var_end;
    }
    if (next_c != M || next_v != N) {
      fail(QB_INVALID_ARGUMENT, "segments must cover every check and variable");
    }

    // ---- device
    CUDA_TRY(cudaSetDevice(device));
    int sm_count = 0, smem_optin = 0;
    if (!device_limits(device, &sm_count, &smem_optin)) {
      fail(QB_RUNTIME_ERROR, "cudaDeviceGetAttribute failed for device " + std::to_string(device));
    }
    h = new qb_decoder();
    h->device = device;
    h->sm_count = sm_count;
    h->max_smem_optin = smem_optin;
    h->arith = arith;
    int lo = 0, hi = 0;
    CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CUDA_TRY(cudaStreamCreateWithPriority(&h->stream, cudaStreamNonBlocking, hi));

    DecodeParams& P = h->P;
    P.M = M;
    P.N = N;
    P.E = E;
    P.nseg = static_cast<uint32_t>(segs.size());
    P.syn_w32 = 2 * ((M + 63) / 64);
    P.est_w32 = 2 * ((N + 63) / 64);
    P.max_iter = static_cast<uint32_t>(config->max_iterations);
    P.early = config->early_termination ? 1 : 0;
    P.alpha = config->alpha;
    P.alpha_f = static_cast<float>(config->alpha);
    P.deg1_f = static_cast<float>(config->alpha * 64.0);
    P.alpha_h = __half_as_ushort(__float2half_rn(static_cast<float>(config->alpha)));
    P.deg1_h = __half_as_ushort(__float2half_rn(static_cast<float>(config->alpha * 64.0)));
    P.clamp_f = static_cast<float>(1e30);
    P.alpha_fx = alpha_fx;
    P.kmax = kmax;
    P.kmax_f = static_cast<float>(kmax);
    P.deg1_i = kmax ? static_cast<int32_t>((static_cast<int64_t>(kmax) * alpha_fx + 32768) >> 16) : 0;
    for (size_t s = 0; s < segs.size(); ++s) {
      P.segs[s] = {segs[s].check_begin, segs[s].check_end, segs[s].var_begin, segs[s].var_end,
                   graph->check_offsets[segs[s].check_begin],
                   graph->check_offsets[segs[s].check_end]};
    }

    auto keep = [&](auto* p) {
      h->dev_allocs.push_back(const_cast<void*>(static_cast<const void*>(p)));
      return p;
    };
    P.check_off = keep(dev_upload(std::vector<uint32_t>(graph->check_offsets, graph->check_offsets + M + 1)));
    P.var_off = keep(dev_upload(std::vector<uint32_t>(graph->var_offsets, graph->var_offsets + N + 1)));
    P.var_edges = keep(dev_upload(std::vector<uint32_t>(graph->var_edges, graph->var_edges + E)));
    P.edge_var = keep(dev_upload(std::vector<uint32_t>(graph->edge_var, graph->edge_var + E)));
    P.edge_check = keep(dev_upload(edge_check));
    h->h_var_edges.assign(graph->var_edges, graph->var_edges + E);
    h->h_check_off.assign(graph->check_offsets, graph->check_offsets + M + 1);
    CUDA_TRY(cudaMalloc(&h->d_edge_slot, std::max<size_t>(E, 1)));
    h->dev_allocs.push_back(h->d_edge_slot);
    P.edge_slot = h->d_edge_slot;
    P.gamma = gamma_f.empty() ? static_cast<const void*>(keep(dev_upload(gamma_i)))
                              : static_cast<const void*>(keep(dev_upload(gamma_f)));

    P.seg_emax = 0;
    for (uint32_t k = 0; k < P.nseg; ++k) {
      P.seg_emax = std::max(P.seg_emax, P.segs[k].e1 - P.segs[k].e0);
    }
    h->smem_bytes = generic_smem_bytes(E, P.syn_w32, P.est_w32, P.nseg, msg_bytes_of(arith));
    P.seg_mmax = 0;
    P.seg_nmax = 0;
    for (uint32_t k = 0; k < P.nseg; ++k) {
      P.seg_mmax = std::max(P.seg_mmax, P.segs[k].c1 - P.segs[k].c0);
      P.seg_nmax = std::max(P.seg_nmax, P.segs[k].v1 - P.segs[k].v0);
    }
    h->smem_lean = lean_smem_bytes(P.seg_mmax, arith == QB_ARITH_HALF    ? 3
                                               : arith == QB_ARITH_INT16 ? 0  // whole-word messages
                                                                         : arith,
                                   P.syn_w32);
    if (h->smem_bytes > static_cast<size_t>(h->max_smem_optin)) {
      fail(QB_INVALID_ARGUMENT, "graph needs " + std::to_string(h->smem_bytes) +
                                    " bytes of shared memory per shot; the device offers " +
                                    std::to_string(h->max_smem_optin));
    }
    {
      // uniform prior?  (every stored gamma identical)
      bool uniform = true;
      if (!gamma_f.empty()) {
        for (uint32_t n = 1; n < N && uniform; ++n) uniform = gamma_f[n] == gamma_f[0];
        P.gamma_f = gamma_f[0];
        P.gamma_d = static_cast<double>(gamma_f[0]);
      } else {
        for (uint32_t n = 1; n < N && uniform; ++n) uniform = gamma_i[n] == gamma_i[0];
        P.gamma_i = gamma_i[0];
      }
      // fp32: can any stored message reach the reference's 1e30 clamp
      // (decoder.cpp:238-241)?  |q| <= G + (dv-1) * |r|max, |r| <= alpha * |q|max
      // (or alpha * 64 from a degree-1 check), iterated max_iterations times.
      bool clamp_free = true;
      if (arith == QB_ARITH_FLOAT) {
        double gmax = 0.0;
        for (float gmm : gamma_f) gmax = std::max(gmax, static_cast<double>(std::fabs(gmm)));
        uint64_t dv_max = 0;
        bool deg1_check = false;
        for (uint32_t n = 0; n < N; ++n) {
          dv_max = std::max<uint64_t>(dv_max, graph->var_offsets[n + 1] - graph->var_offsets[n]);
        }
        for (uint32_t m = 0; m < M; ++m) {
          deg1_check = deg1_check || graph->check_offsets[m + 1] - graph->check_offsets[m] == 1;
        }
        double bq = gmax;
        for (uint64_t it = 0; it < config->max_iterations && clamp_free; ++it) {
          double br = config->alpha * bq;
          if (deg1_check) br = std::max(br, config->alpha * 64.0);
          bq = gmax + static_cast<double>(dv_max) * br;  // also bounds the posterior
          clamp_free = bq < 1e29;
        }
      }
      h->fast_ok = uniform && clamp_free;
      // constants of the first iteration on the uniform-prior path (kernel_lean.cuh)
      if (!gamma_f.empty()) {
        const float g0 = gamma_f[0];
        P.it1_neg = g0 < 0.0f ? 1u : 0u;
        P.it1_d = static_cast<double>(
            static_cast<float>(config->alpha * static_cast<double>(std::fabs(g0))));
        // fp16 mode: every quantity is an fp16 value, products are single fp16 multiplies
        const float gclamp = std::fmin(std::fmax(g0, -kHalfClamp), kHalfClamp);
        const __half gh = __float2half_rn(gclamp);
        const __half ah = __float2half_rn(static_cast<float>(config->alpha));
        P.gamma_hb = __half_as_ushort(gh);
        P.it1_h = __half_as_ushort(__hmul(ah, __habs(gh)));
        // first iteration as a table (kernel_lean.cuh vn3_first_tab): evaluate the reference's
        // variable stage (decoder.cpp:313-335: fp64 sum in edge order, one rounding per stored
        // message) for all eight syndrome patterns of a degree-3 variable and check that the
        // message on edge i only depends on how many OTHER checks are unsatisfied and the
        // decision on how many of all three are
        if (arith == QB_ARITH_FLOAT) {
          const double gd = static_cast<double>(g0);
          const double sd = (g0 < 0.0f ? -1.0 : 1.0) * P.it1_d;  // r of a satisfied check
          uint32_t tq[3] = {0, 0, 0}, dec4 = 0;
          bool seen_q[3] = {false, false, false}, seen_d[4] = {false, false, false, false}, ok = true;
          for (int pat = 0; pat < 8 && ok; ++pat) {
            double r[3], total = gd;
            for (int i = 0; i < 3; ++i) {
              r[i] = ((pat >> i) & 1) ? -sd : sd;
              total += r[i];
            }
            const int k = (pat & 1) + ((pat >> 1) & 1) + ((pat >> 2) & 1);
            const uint32_t d = total < 0.0 ? 1u : 0u;
            if (seen_d[k] && ((dec4 >> (4 * k)) & 1u) != d) ok = false;
            seen_d[k] = true;
            dec4 |= d << (4 * k);
            for (int i = 0; i < 3; ++i) {
              float x = static_cast<float>(total - r[i]);
              x = std::fmin(std::fmax(x, -1e30f), 1e30f);
              uint32_t bits;
              std::memcpy(&bits, &x, 4);
              const int ko = k - ((pat >> i) & 1);
              if (seen_q[ko] && tq[ko] != bits) ok = false;
              seen_q[ko] = true;
              tq[ko] = bits;
            }
          }
          h->tab_ok = ok;
          for (int j = 0; j < 3; ++j) P.it1_tq[j] = tq[j];
          P.it1_dec4 = dec4;
        }
      } else {
        const int32_t g0 = gamma_i[0];
        P.it1_neg = g0 < 0 ? 1u : 0u;
        P.it1_i = static_cast<int32_t>(
            (static_cast<int64_t>(g0 < 0 ? -g0 : g0) * alpha_fx + 32768) >> 16);
        {
          // the same table for the integer modes (exact sums: the order cannot matter)
          const int32_t sgn = g0 < 0 ? -1 : 1;
          P.gamma_f = static_cast<float>(g0);
          for (int ko = 0; ko < 3; ++ko) {
            const int32_t v = std::max(-kmax, std::min(kmax, g0 + sgn * (2 - 2 * ko) * P.it1_i));
            if (arith == QB_ARITH_INT16) {  // the int16 batch kernels keep integers in fp32 words
              const float vf = static_cast<float>(v);
              std::memcpy(&P.it1_tq[ko], &vf, 4);
            } else {
              P.it1_tq[ko] = static_cast<uint32_t>(v);
            }
          }
          P.it1_dec4 = 0;
          for (int k = 0; k < 4; ++k) {
            if (g0 + sgn * (3 - 2 * k) * P.it1_i < 0) P.it1_dec4 |= 1u << (4 * k);
          }
          h->tab_ok = true;
        }
        if (arith == QB_ARITH_INT8) {
          // int8 on the packed fp16 kernel: find an fp16 constant c with
          // round-to-nearest-even(mag * c) == (mag * alpha_fx + 32768) >> 16 for every
          // magnitude 0..127 (mag * c is exact in double; ties included in the check)
          const __half c0 = __float2half_rn(static_cast<float>(alpha_fx) / 65536.0f);
          for (int d : {0, -1, 1, -2, 2}) {
            const unsigned short bits = static_cast<unsigned short>(__half_as_ushort(c0) + d);
            const double c = static_cast<double>(__half2float(__ushort_as_half(bits)));
            bool ok = c > 0.0 && c <= 1.0;
            for (int mag = 0; mag <= 127 && ok; ++mag) {
              const int64_t want = (static_cast<int64_t>(mag) * alpha_fx + 32768) >> 16;
              ok = static_cast<int64_t>(std::nearbyint(mag * c)) == want;
            }
            if (ok) {
              h->i8_pair_ok = true;
              P.alpha_h = bits;
              P.gamma_hb = __half_as_ushort(__float2half_rn(static_cast<float>(g0)));
              P.it1_h = __half_as_ushort(__float2half_rn(static_cast<float>(P.it1_i)));
              break;
            }
          }
        }
      }
    }
    {
      bool reg = P.nseg <= 8;
      for (uint32_t m = 0; m < M && reg; ++m) {
        reg = graph->check_offsets[m + 1] - graph->check_offsets[m] == 6;
      }
      for (uint32_t n = 0; n < N && reg; ++n) {
        reg = graph->var_offsets[n + 1] - graph->var_offsets[n] == 3;
      }
      h->regular63 = reg;
      for (uint32_t m = 0; m < M; ++m) {
        h->max_dc = std::max(h->max_dc, graph->check_offsets[m + 1] - graph->check_offsets[m]);
      }
      for (uint32_t n = 0; n < N; ++n) {
        h->max_dv = std::max(h->max_dv, graph->var_offsets[n + 1] - graph->var_offsets[n]);
      }
    }
    h->soft_bytes = arith == QB_ARITH_INT8 ? 1u : arith == QB_ARITH_INT16 ? 2u : 4u;
    h->quant_scale = arith == QB_ARITH_INT8 || arith == QB_ARITH_INT16
                         ? (config->quant_scale != 0.0 ? config->quant_scale
                                                       : (arith == QB_ARITH_INT8 ? 8.0 : 256.0))
                         : 0.0;
    {
      // degree-padded kernel: every check absorbs its first degree-1 variable (that variable
      // is then updated by the check's thread); the others are listed per segment
      std::vector<uint32_t> abs_slot(M, kNoAbsorb), vars(N, 0);
      std::vector<uint8_t> absorbed(N, 0);
      h->soft_var.assign(M, 0xffffffffu);
      for (uint32_t m = 0; m < M; ++m) {
        const uint32_t e0 = graph->check_offsets[m], e1 = graph->check_offsets[m + 1];
        for (uint32_t e = e0; e < e1 && e - e0 < kNoAbsorb; ++e) {
          const uint32_t v = graph->edge_var[e];
          if (graph->var_offsets[v + 1] - graph->var_offsets[v] == 1) {
            abs_slot[m] = e - e0;
            absorbed[v] = 1;
            h->soft_var[m] = v;
            break;
          }
        }
      }
      for (uint32_t k = 0; k < P.nseg; ++k) {
        uint32_t cnt = 0;
        for (uint32_t v = P.segs[k].v0; v < P.segs[k].v1; ++v) {
          if (!absorbed[v]) vars[P.segs[k].v0 + cnt++] = v;
        }
        P.ell_nvars[k] = cnt;
      }
      P.ell_vars = keep(dev_upload(vars));
      P.ell_abs = keep(dev_upload(abs_slot));
    }
    make_plans(h);

    CUDA_TRY(cudaMalloc(&h->d_sched, kSchedSlots * kSchedWords * sizeof(unsigned int)));
    CUDA_TRY(cudaMemset(h->d_sched, 0, kSchedSlots * kSchedWords * sizeof(unsigned int)));
    for (int k = 0; k < kPipeSlots; ++k) {
      CUDA_TRY(cudaStreamCreateWithFlags(&h->pipe_stream[k], cudaStreamNonBlocking));
      CUDA_TRY(cudaEventCreateWithFlags(&h->pipe_event[k], cudaEventDisableTiming));
    }

    // ---- single-shot staging
    auto align8 = [](size_t x) { return (x + 7) & ~static_cast<size_t>(7); };
    h->off_res = align8(P.est_w32 * 4);
    h->off_conv = h->off_res + align8(P.syn_w32 * 4);
    h->off_iters = h->off_conv + align8(P.nseg);
    h->off_ns = h->off_iters + align8(P.nseg * 4);
    h->off_flag = h->off_ns + 8;
    h->out_bytes = h->off_flag + 8;
    h->rec_stride = sector_words(record_data_words(P.seg_nmax, P.seg_mmax));
    const size_t rec_bytes = static_cast<size_t>(h->rec_stride) * P.nseg * 4;
    {
      // one pinned slab: [syndrome in | outputs of the generic path | doorbell | records]
      auto r256 = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
      const size_t o_out = r256(P.syn_w32 * 4), o_db = o_out + r256(h->out_bytes), o_rec = o_db + 256;
      h->h_slab = slab_acquire(o_rec + r256(rec_bytes), device, &h->h_slab_bytes);
      if (!h->h_slab) fail(QB_RUNTIME_ERROR, "cudaHostAlloc failed for the single-shot staging buffers");
      unsigned char* base = static_cast<unsigned char*>(h->h_slab);
      unsigned char* dbase = nullptr;
      CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dbase), base, 0));
      h->h_in = reinterpret_cast<decltype(h->h_in)>(base);
      h->h_out = reinterpret_cast<decltype(h->h_out)>(base + o_out);
      h->h_db = reinterpret_cast<decltype(h->h_db)>(base + o_db);
      h->h_rec = reinterpret_cast<decltype(h->h_rec)>(base + o_rec);
      h->d_in_map = reinterpret_cast<decltype(h->d_in_map)>(dbase);
      h->d_out_map = reinterpret_cast<decltype(h->d_out_map)>(dbase + o_out);
      h->d_db = reinterpret_cast<decltype(h->d_db)>(dbase + o_db);
      h->d_rec_map = reinterpret_cast<decltype(h->d_rec_map)>(dbase + o_rec);
      std::memset(base, 0, o_rec + r256(rec_bytes));
    }
    CUDA_TRY(cudaMalloc(&h->d_rec_dev, rec_bytes));
    CUDA_TRY(cudaMemset(h->d_rec_dev, 0, rec_bytes));
    CUDA_TRY(cudaMalloc(&h->d_in_dev, P.syn_w32 * 4));
    CUDA_TRY(cudaMalloc(&h->d_out_dev, h->out_bytes));
    CUDA_TRY(cudaMemset(h->d_out_dev, 0, h->out_bytes));
    CUDA_TRY(cudaMalloc(&h->d_qdump, static_cast<size_t>(E) * 4));
    CUDA_TRY(cudaMalloc(&h->d_rdump, static_cast<size_t>(E) * 4));
    CUDA_TRY(cudaDeviceSynchronize());
    *out = h;
  });
  if (st != QB_OK && h) destroy(h);
  return st;
}

void qb_decoder_destroy(qb_decoder* h) { destroy(h); }

qb_status qb_set_option(qb_decoder* h, int option, int64_t value) {
  if (!h) return QB_INVALID_ARGUMENT;
  // a value the launch planner rejects must not stick: remember the plan-affecting options
  // and put them back (and re-plan) if make_plans throws
  struct Saved {
    int64_t kernel, io, shape, threads, ctas, npt, lat_npt, bshape, pair, idle, fast, spread;
  } const old{h->opt_kernel, h->opt_latency_io, h->opt_latency_shape, h->opt_group_threads,
              h->opt_batch_ctas, h->opt_batch_npt, h->opt_latency_npt, h->opt_batch_shape,
              h->opt_batch_pair, h->opt_idle_ms, h->opt_fast, h->opt_slot_spread};
  const qb_status st = set_option_unchecked(h, option, value);
  if (st != QB_OK) {
    const std::string why = h->err;
    h->opt_kernel = old.kernel;
    h->opt_latency_io = old.io;
    h->opt_latency_shape = old.shape;
    h->opt_group_threads = old.threads;
    h->opt_batch_ctas = old.ctas;
    h->opt_batch_npt = old.npt;
    h->opt_latency_npt = old.lat_npt;
    h->opt_batch_shape = old.bshape;
    h->opt_batch_pair = old.pair;
    h->opt_idle_ms = old.idle;
    h->opt_fast = old.fast;
    h->opt_slot_spread = old.spread;
    guarded(h, [&] { make_plans(h); });  // the previous options planned fine before
    h->err = why;
  }
  return st;
}

}  // extern "C"

qb_status set_option_unchecked(qb_decoder* h, int option, int64_t value) {
  return guarded(h, [&] {
    switch (option) {
      case QB_OPT_KERNEL:
        if (value < 0 || value > 2) fail(QB_INVALID_ARGUMENT, "QB_OPT_KERNEL: 0 .. 2");
        h->opt_kernel = value;
        break;
      case QB_OPT_BATCH_VARIANT:
        if (value < 0 || value > kNumLeanVariants) {
          fail(QB_INVALID_ARGUMENT, "QB_OPT_BATCH_VARIANT: 0 .. 11");
        }
        h->opt_batch_npt = value;
        break;
      case QB_OPT_BATCH_SHAPE:
        if (value < 0 || value > 2) fail(QB_INVALID_ARGUMENT, "QB_OPT_BATCH_SHAPE: 0, 1 or 2");
        h->opt_batch_shape = value;
        break;
      case QB_OPT_SLOT_SPREAD:
        if (value < 0 || value > 2) fail(QB_INVALID_ARGUMENT, "QB_OPT_SLOT_SPREAD: 0, 1 or 2");
        h->opt_slot_spread = value;
        break;
      case QB_OPT_SAMPLER:
        if (value < 0 || value > 1) fail(QB_INVALID_ARGUMENT, "QB_OPT_SAMPLER: 0 or 1");
        h->opt_sampler = value;
        return;
      case QB_OPT_LATENCY_WAIT:
        if (value < 0 || value > 1) fail(QB_INVALID_ARGUMENT, "QB_OPT_LATENCY_WAIT: 0 or 1");
        h->opt_latency_wait = value;
        break;
      case QB_OPT_CAMPAIGN_FUSED:
        if (value < 0 || value > 1) fail(QB_INVALID_ARGUMENT, "QB_OPT_CAMPAIGN_FUSED: 0 or 1");
        h->opt_campaign_fused = value;
        return;
      case QB_OPT_BATCH_CHUNK:
        if (value < 0) fail(QB_INVALID_ARGUMENT, "QB_OPT_BATCH_CHUNK: >= 0");
        h->opt_batch_chunk = value;
        return;
      case QB_OPT_BATCH_TILE:
        if (value < 0 || value > static_cast<int64_t>(kMaxTile)) {
          fail(QB_INVALID_ARGUMENT, "QB_OPT_BATCH_TILE: 0 .. 16");
        }
        h->opt_batch_tile = value;
        return;
      case QB_OPT_LATENCY_GRAPH:
        if (value < 0 || value > 1) fail(QB_INVALID_ARGUMENT, "QB_OPT_LATENCY_GRAPH: 0 or 1");
        h->opt_latency_graph = value;
        return;
      case QB_OPT_LATENCY_EVENTS:
        if (value < 0 || value > 1) fail(QB_INVALID_ARGUMENT, "QB_OPT_LATENCY_EVENTS: 0 or 1");
        h->opt_latency_events = value;
        return;  // no effect on the launch plans
      case QB_OPT_HALF_PAIRS:
        if (value < 0 || value > 1) fail(QB_INVALID_ARGUMENT, "QB_OPT_HALF_PAIRS: 0 or 1");
        h->opt_batch_pair = value;
        break;
      case QB_OPT_DOORBELL_IDLE_MS:
        if (value < 1 || value > 60000) fail(QB_INVALID_ARGUMENT, "QB_OPT_DOORBELL_IDLE_MS: 1..60000");
        stop_doorbell(h);
        h->opt_idle_ms = value;
        break;
      case QB_OPT_FAST_PATH:
        if (value < 0 || value > 1) fail(QB_INVALID_ARGUMENT, "QB_OPT_FAST_PATH: 0 or 1");
        h->opt_fast = value;
        break;
      case QB_OPT_LATENCY_NODES_PER_THREAD:
        if (value < 0 || value > 3) {
          fail(QB_INVALID_ARGUMENT, "QB_OPT_LATENCY_NODES_PER_THREAD: 0, 1, 2 or 3");
        }
        h->opt_latency_npt = value;
        break;
      case QB_OPT_LATENCY_IO:
        if (value < 0 || value > 2) fail(QB_INVALID_ARGUMENT, "QB_OPT_LATENCY_IO: 0, 1 or 2");
        stop_doorbell(h);
        h->opt_latency_io = value;
        break;
      case QB_OPT_LATENCY_SHAPE:
        if (value < 0 || value > 2) fail(QB_INVALID_ARGUMENT, "QB_OPT_LATENCY_SHAPE: 0, 1 or 2");
        h->opt_latency_shape = value;
        break;
      case QB_OPT_GROUP_THREADS:
        if (value < 0 || value > 1024) fail(QB_INVALID_ARGUMENT, "QB_OPT_GROUP_THREADS: 0..1024");
        h->opt_group_threads = value;
        break;
      case QB_OPT_BATCH_CTAS_PER_SM:
        if (value < 0 || value > 32) fail(QB_INVALID_ARGUMENT, "QB_OPT_BATCH_CTAS_PER_SM: 0..32");
        h->opt_batch_ctas = value;
        break;
      default:
        fail(QB_INVALID_ARGUMENT, "unknown option");
    }
    stop_doorbell(h);
    make_plans(h);
  });
}

extern "C" {

int64_t qb_get_option(const qb_decoder* h, int option) {
  if (!h) return -1;
  switch (option) {
    case QB_OPT_KERNEL: return h->opt_kernel;
    case QB_OPT_LATENCY_IO: return h->opt_latency_io;
    case QB_OPT_LATENCY_SHAPE: return h->opt_latency_shape;
    case QB_OPT_GROUP_THREADS: return h->lat.group_threads;
    case QB_OPT_BATCH_VARIANT: return h->bat.regular ? h->bat.npt : 0;
    case QB_OPT_LATENCY_NODES_PER_THREAD: return h->opt_latency_npt;
    case QB_OPT_INFO_BATCH_CTAS_PER_SM: return h->bat.ctas_per_sm;
    case QB_OPT_INFO_BATCH_BLOCK: return h->bat.block;
    case QB_OPT_INFO_LATENCY_BLOCK: return h->lat_lean_kernel ? h->lat_lean_block : h->lat.block;
    case QB_OPT_INFO_LATENCY_CLUSTER: return (h->lat_lean_kernel || h->lat.cluster) ? 1 : 0;
    case QB_OPT_INFO_BATCH_REGULAR: return h->bat.regular ? 1 : 0;
    case QB_OPT_FAST_PATH: return h->opt_fast;
    case QB_OPT_BATCH_SHAPE: return h->bat.lean ? 2 : 1;
    case QB_OPT_INFO_FAST_ELIGIBLE: return h->fast_ok ? 1 : 0;
    case QB_OPT_DOORBELL_IDLE_MS: return h->opt_idle_ms;
    case QB_OPT_HALF_PAIRS: return h->bat.pair ? 1 : 0;
    case QB_OPT_INFO_LATENCY_LEAN: return h->lat_lean_kernel ? 1 : 0;
    case QB_OPT_INFO_BATCH_ELL: return h->bat.ell;
    case QB_OPT_LATENCY_EVENTS: return h->opt_latency_events;
    case QB_OPT_LATENCY_GRAPH: return h->opt_latency_graph;
    case QB_OPT_BATCH_TILE: return h->opt_batch_tile;
    case QB_OPT_BATCH_CHUNK: return h->opt_batch_chunk;
    case QB_OPT_SAMPLER: return h->opt_sampler;
    case QB_OPT_CAMPAIGN_FUSED: return h->opt_campaign_fused;
    case QB_OPT_LATENCY_WAIT: return h->opt_latency_wait;
    case QB_OPT_SLOT_SPREAD: return h->opt_slot_spread;
    case QB_OPT_INFO_LAST_EVENT_NS: return static_cast<int64_t>(h->last_event_ns);
    case QB_OPT_BATCH_CTAS_PER_SM: return h->opt_batch_ctas;
    default: return -1;
  }
}

uint32_t qb_num_checks(const qb_decoder* h) { return h ? h->P.M : 0; }
uint32_t qb_num_vars(const qb_decoder* h) { return h ? h->P.N : 0; }
uint32_t qb_num_segments(const qb_decoder* h) { return h ? h->P.nseg : 0; }
uint64_t qb_last_kernel_ns(const qb_decoder* h) { return h ? h->last_kernel_ns : 0; }
uint64_t qb_launch_count(const qb_decoder* h) { return h ? h->launches : 0; }


qb_status qb_decode(qb_decoder* h, const uint64_t* syndrome, uint64_t* estimate,
                    uint64_t* residual, uint8_t* converged, uint32_t* iterations) {
  if (!h) return QB_INVALID_ARGUMENT;
  return guarded(h, [&] { single_shot(h, syndrome, estimate, residual, converged, iterations, false); });
}

qb_status qb_decode_soft(qb_decoder* h, const uint64_t* syndrome, const void* soft,
                         uint64_t* estimate, uint64_t* residual, uint8_t* converged,
                         uint32_t* iterations) {
  if (!h) return QB_INVALID_ARGUMENT;
  return guarded(h, [&] {
    if (!soft) fail(QB_INVALID_ARGUMENT, "decode_soft: NULL soft buffer");
    single_shot(h, syndrome, estimate, residual, converged, iterations, false, soft);
  });
}

qb_status qb_latency_run_soft(qb_decoder* h, const uint64_t* pool, const void* soft_pool,
                              uint64_t pool_size, uint64_t warmup, uint64_t measure,
                              uint64_t* wall_ns, uint64_t* kernel_ns, uint64_t* digest) {
  if (!h) return QB_INVALID_ARGUMENT;
  return guarded(h, [&] {
    if (!pool || pool_size == 0) fail(QB_INVALID_ARGUMENT, "latency_run: empty pool");
    const size_t soft_row = static_cast<size_t>(h->P.M) * h->soft_bytes;
    const DecodeParams& P = h->P;
    const size_t sw = P.syn_w32 / 2, ew = P.est_w32 / 2;
    std::vector<uint64_t> est(ew), res(sw);
    std::vector<uint8_t> conv(P.nseg);
    std::vector<uint32_t> its(P.nseg);
    uint64_t hsh = 14695981039346656037ull;  // FNV-1a (bench.cpp:27-36)
    auto mix = [&](const void* data, size_t len) {
      const unsigned char* b = static_cast<const unsigned char*>(data);
      for (size_t i = 0; i < len; ++i) {
        hsh ^= b[i];
        hsh *= 1099511628211ull;
      }
    };
    for (uint64_t b = 0; b < warmup + measure; ++b) {
      const uint64_t* syn = pool + (b % pool_size) * sw;
      const auto t0 = std::chrono::steady_clock::now();
      const void* soft = soft_pool ? static_cast<const unsigned char*>(soft_pool) + (b % pool_size) * soft_row
                                   : nullptr;
      single_shot(h, syn, est.data(), res.data(), conv.data(), its.data(), false, soft);
      const auto t1 = std::chrono::steady_clock::now();
      if (b < warmup) continue;
      const uint64_t k = b - warmup;
      if (wall_ns) {
        wall_ns[k] = static_cast<uint64_t>(
            std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
      }
      if (kernel_ns) {
        kernel_ns[k] = h->opt_latency_events && h->opt_latency_io == 1 ? h->last_event_ns
                                                                       : h->last_kernel_ns;
      }
      unsigned char c = 1;
      uint64_t it = 0;
      for (uint32_t s = 0; s < P.nseg; ++s) {
        c = c && conv[s];
        it = std::max<uint64_t>(it, its[s]);
      }
      mix(&c, 1);
      mix(&it, sizeof(it));
      mix(est.data(), ew * sizeof(uint64_t));
    }
    if (digest) *digest = hsh;
  });
}

qb_status qb_latency_run(qb_decoder* h, const uint64_t* pool, uint64_t pool_size,
                         uint64_t warmup, uint64_t measure, uint64_t* wall_ns,
                         uint64_t* kernel_ns, uint64_t* digest) {
  return qb_latency_run_soft(h, pool, nullptr, pool_size, warmup, measure, wall_ns, kernel_ns, digest);
}

qb_status qb_decode_debug(qb_decoder* h, const uint64_t* syndrome, uint64_t* estimate,
                          uint64_t* residual, uint8_t* converged, uint32_t* iterations,
                          float* q_f32, float* r_f32, int32_t* q_i32, int32_t* r_i32) {
  if (!h) return QB_INVALID_ARGUMENT;
  return guarded(h, [&] {
    single_shot(h, syndrome, estimate, residual, converged, iterations, true);
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    const size_t bytes = static_cast<size_t>(h->P.E) * 4;
    const bool is_int = h->arith == QB_ARITH_INT8 || h->arith == QB_ARITH_INT16;
    void* qdst = is_int ? static_cast<void*>(q_i32) : static_cast<void*>(q_f32);
    void* rdst = is_int ? static_cast<void*>(r_i32) : static_cast<void*>(r_f32);
    if (!qdst || !rdst) fail(QB_INVALID_ARGUMENT, "decode_debug: message buffers of the wrong type");
    CUDA_TRY(cudaMemcpy(qdst, h->d_qdump, bytes, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(rdst, h->d_rdump, bytes, cudaMemcpyDeviceToHost));
  });
}

qb_status qb_decode_batch_device(qb_decoder* h, uint64_t shots, const uint64_t* d_syndromes,
                                 uint64_t* d_estimates, uint64_t* d_residuals,
                                 uint8_t* d_converged, uint32_t* d_iterations, void* stream) {
  if (!h) return QB_INVALID_ARGUMENT;
  return guarded(h, [&] {
    if (shots == 0) return;
    if (!d_syndromes || !d_estimates || !d_converged || !d_iterations) {
      fail(QB_INVALID_ARGUMENT, "decode_batch_device: NULL buffer");
    }
    run_batch_device(h, shots, reinterpret_cast<const uint32_t*>(d_syndromes),
                     reinterpret_cast<uint32_t*>(d_estimates),
                     reinterpret_cast<uint32_t*>(d_residuals), d_converged, d_iterations,
                     static_cast<cudaStream_t>(stream));
  });
}

qb_status qb_generate_syndromes(qb_decoder* h, uint64_t seed, double p, const double* probs,
                                int css_interleave, uint64_t first_trial, uint64_t shots,
                                uint64_t* d_syndromes, uint64_t* d_errors, void* stream) {
  if (!h) return QB_INVALID_ARGUMENT;
  return guarded(h, [&] {
    if (shots == 0) return;
    if (!d_syndromes) fail(QB_INVALID_ARGUMENT, "generate_syndromes: NULL output");
    const DecodeParams& P = h->P;
    auto check_p = [](double v) {
      if (!(v >= 0.0 && v <= 1.0)) fail(QB_INVALID_ARGUMENT, "NoiseModel: p must lie in [0, 1]");
    };
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    NoiseParams np{};
    np.seed = seed;
    np.first_trial = first_trial;
    np.nshots = shots;
    const bool skip = h->opt_sampler == 1;
    double p_max = 0.0;
    if (probs) {
      std::vector<uint64_t> thr(P.N);
      for (uint32_t v = 0; v < P.N; ++v) {
        check_p(probs[v]);
        p_max = std::max(p_max, probs[v]);
      }
      for (uint32_t v = 0; v < P.N; ++v) {
        // skip sampler: acceptance threshold of the thinning step, p_v / p_max
        thr[v] = noise_threshold(skip ? (p_max > 0.0 ? probs[v] / p_max : 0.0) : probs[v]);
      }
      if (!h->d_probs) CUDA_TRY(cudaMalloc(&h->d_probs, sizeof(uint64_t) * P.N));
      // synchronous: `thr` is a local
      CUDA_TRY(cudaStreamSynchronize(st));
      CUDA_TRY(cudaMemcpy(h->d_probs, thr.data(), sizeof(uint64_t) * P.N, cudaMemcpyHostToDevice));
      np.thrs = h->d_probs;
    } else {
      check_p(p);
      np.thr = noise_threshold(p);
      p_max = p;
    }
    np.mode = css_interleave ? 1u : 0u;
    if (css_interleave) {
      if (P.nseg != 2 || P.segs[0].v1 * 2 != P.N) {
        fail(QB_INVALID_ARGUMENT,
             "generate_syndromes: css_interleave needs a two-segment decoder over 2n variables");
      }
      np.n_qubits = P.segs[0].v1;
    }
    np.syn = reinterpret_cast<uint32_t*>(d_syndromes);
    np.err = reinterpret_cast<uint32_t*>(d_errors);
    if (skip) {
      // one thread per shot, one odd-stride shared-memory row per thread
      SkipParams sp{};
      sp.inv_log1m = 1.0 / std::log1p(-p_max);  // -inf at p_max = 0 (no flips), -0.0 at p_max = 1 (all flip)
      sp.row = (P.syn_w32 + P.est_w32) | 1u;
      unsigned threads = 128;
      while (threads > 32 && static_cast<size_t>(threads) * sp.row * 4 > static_cast<size_t>(h->max_smem_optin)) threads /= 2;
      const size_t smem = static_cast<size_t>(threads) * sp.row * 4;
      if (smem > static_cast<size_t>(h->max_smem_optin)) {
        fail(QB_INVALID_ARGUMENT, "generate_syndromes: graph too large for the skip sampler (QB_OPT_SAMPLER = 0 has no limit)");
      }
      auto* kern = np.thrs ? noise_skip_kernel<true> : noise_skip_kernel<false>;
      CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      const uint64_t blocks_needed = (shots + threads - 1) / threads;
      const unsigned grid = static_cast<unsigned>(
          std::min<uint64_t>(blocks_needed, static_cast<uint64_t>(h->sm_count) * 16));
      kern<<<grid, threads, smem, st>>>(P, np, sp);
      CUDA_TRY(cudaGetLastError());
      ++h->launches;
      return;
    }
    const uint64_t blocks_needed = (shots + kNoiseWarps - 1) / kNoiseWarps;
    const unsigned grid = static_cast<unsigned>(
        std::min<uint64_t>(blocks_needed, static_cast<uint64_t>(h->sm_count) * 8));
    const size_t smem = static_cast<size_t>(kNoiseWarps) * (P.syn_w32 + P.est_w32) * 4;
    auto* kern = np.mode ? (np.thrs ? noise_syndrome_kernel<true, true> : noise_syndrome_kernel<true, false>)
                         : (np.thrs ? noise_syndrome_kernel<false, true> : noise_syndrome_kernel<false, false>);
    kern<<<grid, kNoiseWarps * 32, smem, st>>>(P, np);
    CUDA_TRY(cudaGetLastError());
    ++h->launches;
  });
}

qb_status qb_set_logicals(qb_decoder* h, const uint64_t* x_tests, uint32_t n_x,
                          const uint64_t* z_tests, uint32_t n_z) {
  if (!h) return QB_INVALID_ARGUMENT;
  return guarded(h, [&] {
    const DecodeParams& P = h->P;
    if (P.nseg != 2) fail(QB_INVALID_ARGUMENT, "set_logicals: decoder was not built from a CssCode");
    if ((n_x && !x_tests) || (n_z && !z_tests)) fail(QB_INVALID_ARGUMENT, "set_logicals: NULL tests");
    auto upload = [&](const uint64_t* src, uint32_t n, uint32_t*& dst) {
      cudaFree(dst);
      dst = nullptr;
      const size_t bytes = std::max<size_t>(static_cast<size_t>(n) * P.est_w32 * 4, 4);
      CUDA_TRY(cudaMalloc(&dst, bytes));
      if (n) CUDA_TRY(cudaMemcpy(dst, src, static_cast<size_t>(n) * P.est_w32 * 4, cudaMemcpyHostToDevice));
    };
    upload(x_tests, n_x, h->d_tests_x);
    upload(z_tests, n_z, h->d_tests_z);
    h->n_tests_x = n_x;
    h->n_tests_z = n_z;
    // transposed form for the fused campaign kernel: bit j of tcol[v] = "test j of v's own
    // component contains v" (at most 64 tests per component, else that kernel is not used)
    cudaFree(h->d_tcol);
    h->d_tcol = nullptr;
    if (n_x <= 64 && n_z <= 64) {
      std::vector<uint64_t> tcol(P.N, 0);
      const uint32_t w64 = P.est_w32 / 2;
      for (uint32_t v = 0; v < P.N; ++v) {
        const bool in_x = v >= P.segs[0].v0 && v < P.segs[0].v1;
        const uint64_t* tests = in_x ? x_tests : z_tests;
        const uint32_t nt = in_x ? n_x : n_z;
        for (uint32_t j = 0; j < nt; ++j) {
          if ((tests[static_cast<size_t>(j) * w64 + (v >> 6)] >> (v & 63u)) & 1ull) tcol[v] |= 1ull << j;
        }
      }
      h->d_tcol = dev_upload(tcol);
    }
  });
}

}  // extern "C"

namespace {

void launch_classify(qb_decoder* h, uint64_t n, const uint32_t* err, const uint32_t* est,
                     const uint32_t* syn, const uint8_t* conv, const uint32_t* iters,
                     cudaStream_t st) {
  const DecodeParams& P = h->P;
  ClassifyParams cp{};
  cp.nshots = n;
  cp.err = err;
  cp.est = est;
  cp.syn = syn;
  cp.conv = conv;
  cp.iters = iters;
  cp.tests_x = h->d_tests_x;
  cp.tests_z = h->d_tests_z;
  cp.n_x = h->n_tests_x;
  cp.n_z = h->n_tests_z;
  cp.aux_mask = h->d_aux_mask;
  cp.counters = h->d_counters;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(
      (n + kClassifyWarps - 1) / kClassifyWarps, static_cast<uint64_t>(h->sm_count) * 8));
  const size_t smem = static_cast<size_t>(kClassifyWarps) * 2 * P.est_w32 * 4;
  classify_kernel<<<grid, kClassifyWarps * 32, smem, st>>>(P, cp);
  CUDA_TRY(cudaGetLastError());
  ++h->launches;
}

void add_counters(qb_decoder* h, uint64_t* counters, cudaStream_t st) {
  unsigned long long host_counters[10];
  CUDA_TRY(cudaMemcpyAsync(host_counters, h->d_counters, sizeof(host_counters),
                           cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  for (int k = 0; k < 10; ++k) counters[k] += host_counters[k];
}

// Soft measurement of the noiseless syndromes in d_syn (kernel_noise.cuh).
void launch_soft_measure(qb_decoder* h, uint64_t seed, double mu, double sigma,
                         uint64_t first_trial, uint64_t shots, uint32_t* d_syn, void* d_soft,
                         uint32_t* d_err, cudaStream_t st) {
  SoftParams sp{};
  sp.seed = seed;
  sp.first_trial = first_trial;
  sp.nshots = shots;
  sp.mu = mu;
  sp.sigma = sigma;
  sp.llr_scale = 2.0 * mu / (sigma * sigma);
  sp.quant_scale = h->quant_scale;
  sp.kmax = h->P.kmax;
  sp.elem_bytes = h->soft_bytes;
  sp.syn = d_syn;
  sp.err = d_err;
  sp.soft = d_soft;
  const uint64_t blocks_needed = (shots + kNoiseWarps - 1) / kNoiseWarps;
  const unsigned grid = static_cast<unsigned>(
      std::min<uint64_t>(blocks_needed, static_cast<uint64_t>(h->sm_count) * 8));
  soft_measure_kernel<<<grid, kNoiseWarps * 32, 0, st>>>(h->P, sp);
  CUDA_TRY(cudaGetLastError());
  ++h->launches;
}

// Flip probabilities for the data variables only: the absorbed (measurement-error) variables
// get probability 0, their flips come from the soft measurement channel.
std::vector<double> data_only_probs(const qb_decoder* h, double p, const double* probs) {
  const DecodeParams& P = h->P;
  std::vector<double> out(P.N);
  for (uint32_t v = 0; v < P.N; ++v) out[v] = probs ? probs[v] : p;
  for (uint32_t m = 0; m < P.M; ++m) {
    if (h->soft_var[m] != 0xffffffffu) out[h->soft_var[m]] = 0.0;
  }
  return out;
}

void check_soft_channel(double mu, double sigma) {
  if (!(mu > 0.0) || !(sigma > 0.0) || !std::isfinite(mu) || !std::isfinite(sigma)) {
    fail(QB_INVALID_ARGUMENT, "soft measurement: mu and sigma must be positive and finite");
  }
}

// The fused campaign kernel (kernel_campaign.cuh) serves plain CSS campaigns on (6,3)-regular
// codes in the modes whose batch kernel decodes one shot per thread (float, int16): the
// shapes the loader picks for the decode-only batch kernel.
using CampKernelFn = void (*)(DecodeParams, CampaignIO);
template <class A>
CampKernelFn campaign_kernel_t(bool fast, bool early) {
  if (early) {  // `early` here: CTAs of more than 160 threads
    return fast ? decode_lean_campaign_kernel<A, 3, 5, true, 192, 5>
                : decode_lean_campaign_kernel<A, 3, 5, false, 192, 5>;
  }
  return fast ? decode_lean_campaign_kernel<A, 3, 5, true, 160, 7>
              : decode_lean_campaign_kernel<A, 3, 5, false, 160, 7>;
}

bool campaign_fusable(const qb_decoder* h, const double* probs, bool soft) {
  const DecodeParams& P = h->P;
  return h->opt_campaign_fused != 0 && !soft && !probs && !h->d_aux_mask && h->d_tcol != nullptr &&
         h->opt_sampler == 0 && h->regular63 && h->opt_kernel != 1 && h->opt_batch_shape != 1 &&
         (h->arith == QB_ARITH_FLOAT || h->arith == QB_ARITH_INT16) && P.nseg == 2 &&
         P.segs[0].v1 * 2 == P.N && P.segs[0].c1 - P.segs[0].c0 <= 576 &&
         P.segs[1].c1 - P.segs[1].c0 <= 576 && P.segs[0].v1 <= 960;
}

void launch_campaign_fused(qb_decoder* h, uint64_t seed, double p, uint64_t first_trial, uint64_t n,
                           cudaStream_t st) {
  const DecodeParams& P0 = h->P;
  const bool fast = h->fast_ok && h->opt_fast != 0 && h->tab_ok;
  const uint32_t T = regular_group_threads(P0, 3, 5);
  // seven CTAs per SM at 56 registers for CTAs of up to 160 threads, else the 192-thread shape
  CampKernelFn kern = h->arith == QB_ARITH_FLOAT ? campaign_kernel_t<ArithF32>(fast, T > 160)
                                                 : campaign_kernel_t<ArithI16F>(fast, T > 160);
  const size_t smem = campaign_smem_bytes(P0.seg_mmax, 0);
  CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, static_cast<int>(T), smem));
  if (per_sm < 1) fail(QB_RUNTIME_ERROR, "campaign kernel does not fit on an SM");
  const uint64_t resident = static_cast<uint64_t>(per_sm) * h->sm_count;
  const uint64_t per_seg = std::max<uint64_t>(1, std::min<uint64_t>(resident / P0.nseg, n));
  DecodeParams P = P0;
  P.ngroups = 1;
  P.group_threads = T;
  CampaignIO io{};
  io.ntrials = n;
  io.first_trial = first_trial;
  io.seed = seed;
  io.thr = noise_threshold(p);
  io.tcol = h->d_tcol;
  io.flags = h->b_conv;
  io.iters = h->b_iters;
  io.sched = h->d_sched + (1 + kPipeSlots + static_cast<int>(h->sched_next++ % kSchedRing)) * kSchedWords;
  kern<<<static_cast<unsigned>(per_seg * P0.nseg), T, smem, st>>>(P, io);
  CUDA_TRY(cudaGetLastError());
  ++h->launches;
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(h->sm_count) * 8));
  campaign_count_kernel<<<grid, 256, 0, st>>>(n, h->b_conv, h->b_iters, h->d_counters);
  CUDA_TRY(cudaGetLastError());
  ++h->launches;
}

// One campaign: sample -> (soft measurement) -> decode -> classify in rounds of `chunk`
// trials, ENQUEUED on the handle's stream; the ten counters stay in h->d_counters.
void campaign_enqueue(qb_decoder* h, uint64_t seed, double p, const double* probs, bool soft, double mu,
                      double sigma, uint64_t first_trial, uint64_t trials) {
  const DecodeParams& P = h->P;
  if (P.nseg != 2 || !h->d_tests_x || !h->d_tests_z) {
    fail(QB_INVALID_ARGUMENT, "campaign_run: call qb_set_logicals on a CssCode decoder first");
  }
  if (!(p >= 0.0 && p <= 1.0)) fail(QB_INVALID_ARGUMENT, "NoiseModel: p must lie in [0, 1]");
  if (soft) {
    require_soft(h, "campaign_run_soft");
    check_soft_channel(mu, sigma);
  }
  if (!h->d_counters) CUDA_TRY(cudaMalloc(&h->d_counters, 10 * sizeof(unsigned long long)));
  cudaStream_t st = h->stream;
  CUDA_TRY(cudaMemsetAsync(h->d_counters, 0, 10 * sizeof(unsigned long long), st));
  if (trials == 0) return;
  // trials per sample / decode / classify round: QB_OPT_BATCH_CHUNK when set, else 2^20
  const uint64_t max_chunk = h->opt_batch_chunk > 0 ? static_cast<uint64_t>(h->opt_batch_chunk) : (1ull << 20);
  const uint64_t chunk = std::min<uint64_t>(trials, max_chunk);
  ensure_batch(h, chunk, false, soft);
  // the reference's draw order (X_0, Z_0, X_1, ...) exists for a plain CSS code only; on an
  // extended graph (auxiliary variables, or per-variable probabilities that do not pair up)
  // draw v belongs to variable v
  const bool interleave = !h->d_aux_mask && !soft && P.segs[0].v1 * 2 == P.N;
  std::vector<double> dprobs;
  if (soft) {
    dprobs = data_only_probs(h, p, probs);
    probs = dprobs.data();
  }
  if (campaign_fusable(h, probs, soft)) {
    // the whole loop inside one kernel per round
    for (uint64_t done = 0; done < trials; done += chunk) {
      const uint64_t n = std::min<uint64_t>(chunk, trials - done);
      launch_campaign_fused(h, seed, p, first_trial + done, n, st);
    }
    return;
  }
  for (uint64_t done = 0; done < trials; done += chunk) {
    const uint64_t n = std::min<uint64_t>(chunk, trials - done);
    qb_status stc = qb_generate_syndromes(h, seed, p, probs, interleave ? 1 : 0, first_trial + done, n,
                                          reinterpret_cast<uint64_t*>(h->b_syn),
                                          reinterpret_cast<uint64_t*>(h->c_err), st);
    if (stc != QB_OK) fail(stc, h->err);
    if (soft) {
      launch_soft_measure(h, seed, mu, sigma, first_trial + done, n, h->b_syn, h->b_soft, h->c_err, st);
    }
    run_batch_device(h, n, h->b_syn, h->b_est, nullptr, h->b_conv, h->b_iters, st, -1,
                     soft ? h->b_soft : nullptr);
    launch_classify(h, n, h->c_err, h->b_est, h->b_syn, h->b_conv, h->b_iters, st);
  }
}

void campaign_core(qb_decoder* h, uint64_t seed, double p, const double* probs, bool soft, double mu,
                   double sigma, uint64_t first_trial, uint64_t trials, uint64_t* counters) {
  if (!counters) fail(QB_INVALID_ARGUMENT, "campaign_run: NULL counters");
  campaign_enqueue(h, seed, p, probs, soft, mu, sigma, first_trial, trials);
  if (trials == 0) return;
  add_counters(h, counters, h->stream);
}

// ---- NCCL, bound at run time (dlopen): the library has no link-time dependency on it, and
// single-GPU users never load it.  Only ncclCommInitAll / ncclAllReduce / group calls.
struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi api;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (api.lib) return api;
  void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) fail(QB_RUNTIME_ERROR, std::string("NCCL not available: ") + dlerror());
  auto sym = [&](const char* name) {
    void* f = dlsym(lib, name);
    if (!f) fail(QB_RUNTIME_ERROR, std::string("NCCL symbol missing: ") + name);
    return f;
  };
  api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
  api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
  api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
  api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
  api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  api.lib = lib;
  return api;
}

#define NCCL_TRY(api, expr)                                                                \
  do {                                                                                     \
    ncclResult_t r__ = (expr);                                                             \
    if (r__ != ncclSuccess) {                                                              \
      fail(QB_RUNTIME_ERROR, std::string("NCCL error in " #expr ": ") + (api).GetErrorString(r__)); \
    }                                                                                      \
  } while (0)

// communicators per device list, created on first use and kept for the life of the process
struct CommSet {
  std::vector<int> devices;
  std::vector<ncclComm_t> comms;
};
std::vector<CommSet>& comm_cache() {
  static std::vector<CommSet> cache;
  return cache;
}
std::mutex g_comm_mu;

const std::vector<ncclComm_t>& comms_for(NcclApi& api, const std::vector<int>& devices) {
  std::lock_guard<std::mutex> lock(g_comm_mu);
  for (const CommSet& cs : comm_cache()) {
    if (cs.devices == devices) return cs.comms;
  }
  CommSet cs;
  cs.devices = devices;
  cs.comms.resize(devices.size());
  NCCL_TRY(api, api.CommInitAll(cs.comms.data(), static_cast<int>(devices.size()), devices.data()));
  comm_cache().push_back(std::move(cs));
  return comm_cache().back().comms;
}

// qb_decode_batch / qb_decode_batch_soft: chunks rotate over kPipeSlots streams, each with
// its own device buffers and scheduler words, so that with pinned host buffers the H2D copy
// of chunk i+1, the kernel of chunk i and the D2H copy of chunk i-1 run concurrently (one
// copy engine per direction).
void decode_batch_host(qb_decoder* h, uint64_t shots, const uint64_t* syndromes, const void* soft,
                       uint64_t* estimates, uint64_t* residuals, uint8_t* converged,
                       uint32_t* iterations) {
  if (shots == 0) return;
  if (!syndromes || !estimates || !converged || !iterations) {
    fail(QB_INVALID_ARGUMENT, "decode_batch: NULL buffer");
  }
  const DecodeParams& P = h->P;
  const uint64_t max_chunk = h->opt_batch_chunk > 0 ? static_cast<uint64_t>(h->opt_batch_chunk) & ~1ull
                                                    : (1ull << 15);  // measured: 103.6 M/s at 2^15, 102.6 at 2^16, 99.3 at 2^17
  const uint64_t chunk = std::min<uint64_t>(shots, std::max<uint64_t>(max_chunk, 2));
  ensure_batch(h, chunk * kPipeSlots, residuals != nullptr, soft != nullptr);
  const size_t soft_row = static_cast<size_t>(P.M) * h->soft_bytes;
  bool used[kPipeSlots] = {};
  uint64_t done = 0;
  for (int slot = 0; done < shots; slot = (slot + 1) % kPipeSlots) {
    const uint64_t n = std::min<uint64_t>(chunk, shots - done);
    const uint64_t off = static_cast<uint64_t>(slot) * chunk;
    cudaStream_t st = h->pipe_stream[slot];
    if (used[slot]) CUDA_TRY(cudaEventSynchronize(h->pipe_event[slot]));
    uint32_t* d_syn = h->b_syn + off * P.syn_w32;
    uint32_t* d_est = h->b_est + off * P.est_w32;
    uint32_t* d_res = h->b_res + off * P.syn_w32;
    uint8_t* d_conv = h->b_conv + off * P.nseg;
    uint32_t* d_it = h->b_iters + off * P.nseg;
    unsigned char* d_soft = soft ? h->b_soft + off * soft_row : nullptr;
    CUDA_TRY(cudaMemcpyAsync(d_syn,
                             reinterpret_cast<const uint32_t*>(syndromes) + done * P.syn_w32,
                             n * P.syn_w32 * 4, cudaMemcpyHostToDevice, st));
    if (soft) {
      CUDA_TRY(cudaMemcpyAsync(d_soft, static_cast<const unsigned char*>(soft) + done * soft_row,
                               n * soft_row, cudaMemcpyHostToDevice, st));
    }
    run_batch_device(h, n, d_syn, d_est, residuals ? d_res : nullptr, d_conv, d_it, st, slot, d_soft);
    CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<uint32_t*>(estimates) + done * P.est_w32, d_est,
                             n * P.est_w32 * 4, cudaMemcpyDeviceToHost, st));
    if (residuals) {
      CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<uint32_t*>(residuals) + done * P.syn_w32, d_res,
                               n * P.syn_w32 * 4, cudaMemcpyDeviceToHost, st));
    }
    CUDA_TRY(cudaMemcpyAsync(converged + done * P.nseg, d_conv, n * P.nseg,
                             cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(iterations + done * P.nseg, d_it, n * P.nseg * 4,
                             cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaEventRecord(h->pipe_event[slot], st));
    used[slot] = true;
    done += n;
  }
  for (int slot = 0; slot < kPipeSlots; ++slot) {
    if (used[slot]) CUDA_TRY(cudaEventSynchronize(h->pipe_event[slot]));
  }
}

}  // namespace

extern "C" {

qb_status qb_set_auxiliary_vars(qb_decoder* h, const uint64_t* mask) {
  if (!h) return QB_INVALID_ARGUMENT;
  return guarded(h, [&] {
    const DecodeParams& P = h->P;
    cudaFree(h->d_aux_mask);
    h->d_aux_mask = nullptr;
    if (!mask) return;
    CUDA_TRY(cudaMalloc(&h->d_aux_mask, P.est_w32 * 4));
    CUDA_TRY(cudaMemcpy(h->d_aux_mask, mask, P.est_w32 * 4, cudaMemcpyHostToDevice));
  });
}

qb_status qb_soft_vars(const qb_decoder* h, uint32_t* vars) {
  if (!h || !vars) return QB_INVALID_ARGUMENT;
  std::memcpy(vars, h->soft_var.data(), h->soft_var.size() * sizeof(uint32_t));
  return QB_OK;
}

qb_status qb_classify_batch_device(qb_decoder* h, uint64_t shots, const uint64_t* d_errors,
                                   const uint64_t* d_estimates, const uint64_t* d_syndromes,
                                   const uint8_t* d_converged, const uint32_t* d_iterations,
                                   uint64_t* counters, void* stream) {
  if (!h) return QB_INVALID_ARGUMENT;
  return guarded(h, [&] {
    const DecodeParams& P = h->P;
    if (!counters || !d_errors || !d_estimates || !d_syndromes || !d_converged || !d_iterations) {
      fail(QB_INVALID_ARGUMENT, "classify_batch_device: NULL buffer");
    }
    if (P.nseg != 2 || !h->d_tests_x || !h->d_tests_z) {
      fail(QB_INVALID_ARGUMENT, "classify_batch_device: call qb_set_logicals on a CssCode decoder first");
    }
    if (shots == 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (!h->d_counters) CUDA_TRY(cudaMalloc(&h->d_counters, 10 * sizeof(unsigned long long)));
    CUDA_TRY(cudaMemsetAsync(h->d_counters, 0, 10 * sizeof(unsigned long long), st));
    launch_classify(h, shots, reinterpret_cast<const uint32_t*>(d_errors),
                    reinterpret_cast<const uint32_t*>(d_estimates),
                    reinterpret_cast<const uint32_t*>(d_syndromes), d_converged, d_iterations, st);
    add_counters(h, counters, st);
  });
}

qb_status qb_campaign_run(qb_decoder* h, uint64_t seed, double p, const double* probs,
                          uint64_t first_trial, uint64_t trials, uint64_t* counters) {
  if (!h) return QB_INVALID_ARGUMENT;
  return guarded(h, [&] {
    campaign_core(h, seed, p, probs, false, 0.0, 0.0, first_trial, trials, counters);
  });
}

qb_status qb_campaign_run_multi(qb_decoder* const* handles, uint32_t n, uint64_t seed, double p,
                                const double* probs, uint64_t first_trial, uint64_t trials,
                                uint64_t* counters) {
  if (!handles || n == 0 || !handles[0]) return QB_INVALID_ARGUMENT;
  qb_decoder* h0 = handles[0];
  return guarded(h0, [&] {
    if (!counters) fail(QB_INVALID_ARGUMENT, "campaign_run_multi: NULL counters");
    std::vector<int> devices(n);
    for (uint32_t g = 0; g < n; ++g) {
      if (!handles[g]) fail(QB_INVALID_ARGUMENT, "campaign_run_multi: NULL handle");
      devices[g] = handles[g]->device;
      for (uint32_t k = 0; k < g; ++k) {
        if (devices[k] == devices[g]) {
          fail(QB_INVALID_ARGUMENT, "campaign_run_multi: two handles on device " +
                                        std::to_string(devices[g]) + " (one decoder per GPU)");
        }
      }
    }
    NcclApi& api = nccl_api();
    const std::vector<ncclComm_t>& comms = comms_for(api, devices);
    // contiguous shard per GPU (noise.cpp:253-254); every GPU's rounds are enqueued before any
    // host wait, so the devices run side by side
    for (uint32_t g = 0; g < n; ++g) {
      qb_decoder* h = handles[g];
      CUDA_TRY(cudaSetDevice(h->device));
      const uint64_t lo = static_cast<uint64_t>(g) * trials / n, hi = static_cast<uint64_t>(g + 1) * trials / n;
      try {
        campaign_enqueue(h, seed, p, probs, false, 0.0, 0.0, first_trial + lo, hi - lo);
      } catch (const StatusError& e) {
        if (h != h0) h0->err = e.msg;
        throw;
      }
    }
    // the path's ONLY collective: one all-reduce(sum) of the ten uint64 counters, in place on
    // every GPU (the integer sum over workers of noise.cpp:306-324)
    NCCL_TRY(api, api.GroupStart());
    for (uint32_t g = 0; g < n; ++g) {
      qb_decoder* h = handles[g];
      NCCL_TRY(api, api.AllReduce(h->d_counters, h->d_counters, 10, ncclUint64, ncclSum, comms[g], h->stream));
    }
    NCCL_TRY(api, api.GroupEnd());
    unsigned long long first[10] = {};
    for (uint32_t g = 0; g < n; ++g) {
      qb_decoder* h = handles[g];
      CUDA_TRY(cudaSetDevice(h->device));
      unsigned long long got[10];
      CUDA_TRY(cudaMemcpyAsync(got, h->d_counters, sizeof(got), cudaMemcpyDeviceToHost, h->stream));
      CUDA_TRY(cudaStreamSynchronize(h->stream));
      if (g == 0) {
        std::memcpy(first, got, sizeof(got));
      } else if (std::memcmp(first, got, sizeof(got)) != 0) {
        fail(QB_RUNTIME_ERROR, "campaign_run_multi: ranks disagree after the all-reduce");
      }
    }
    if (first[9] != trials) fail(QB_RUNTIME_ERROR, "campaign_run_multi: trial count mismatch after the all-reduce");
    for (int k = 0; k < 10; ++k) counters[k] += first[k];
    CUDA_TRY(cudaSetDevice(h0->device));
  });
}

qb_status qb_campaign_run_soft(qb_decoder* h, uint64_t seed, double p, const double* probs,
                               double mu, double sigma, uint64_t first_trial, uint64_t trials,
                               uint64_t* counters) {
  if (!h) return QB_INVALID_ARGUMENT;
  return guarded(h, [&] {
    campaign_core(h, seed, p, probs, true, mu, sigma, first_trial, trials, counters);
  });
}

qb_status qb_generate_soft_syndromes(qb_decoder* h, uint64_t seed, double p, const double* probs,
                                     double mu, double sigma, uint64_t first_trial,
                                     uint64_t shots, uint64_t* d_syndromes, void* d_soft,
                                     uint64_t* d_errors, void* stream) {
  if (!h) return QB_INVALID_ARGUMENT;
  return guarded(h, [&] {
    if (shots == 0) return;
    if (!d_syndromes || !d_soft) fail(QB_INVALID_ARGUMENT, "generate_soft_syndromes: NULL output");
    if (!(p >= 0.0 && p <= 1.0)) fail(QB_INVALID_ARGUMENT, "NoiseModel: p must lie in [0, 1]");
    check_soft_channel(mu, sigma);
    const std::vector<double> dprobs = data_only_probs(h, p, probs);
    qb_status stc = qb_generate_syndromes(h, seed, p, dprobs.data(), 0, first_trial, shots,
                                          d_syndromes, d_errors, stream);
    if (stc != QB_OK) fail(stc, h->err);
    launch_soft_measure(h, seed, mu, sigma, first_trial, shots,
                        reinterpret_cast<uint32_t*>(d_syndromes), d_soft,
                        reinterpret_cast<uint32_t*>(d_errors), static_cast<cudaStream_t>(stream));
  });
}

qb_status qb_decode_batch(qb_decoder* h, uint64_t shots, const uint64_t* syndromes,
                          uint64_t* estimates, uint64_t* residuals, uint8_t* converged,
                          uint32_t* iterations) {
  if (!h) return QB_INVALID_ARGUMENT;
  return guarded(h, [&] {
    decode_batch_host(h, shots, syndromes, nullptr, estimates, residuals, converged, iterations);
  });
}

qb_status qb_decode_batch_debug(qb_decoder* h, uint64_t shots, const uint64_t* syndromes,
                                uint64_t dump_shot, uint64_t* estimates, uint64_t* residuals,
                                uint8_t* converged, uint32_t* iterations, float* q_f32,
                                float* r_f32, int32_t* q_i32, int32_t* r_i32) {
  if (!h) return QB_INVALID_ARGUMENT;
  return guarded(h, [&] {
    if (shots == 0) return;
    if (!syndromes || !estimates || !converged || !iterations) {
      fail(QB_INVALID_ARGUMENT, "decode_batch_debug: NULL buffer");
    }
    if (dump_shot >= shots) fail(QB_INVALID_ARGUMENT, "decode_batch_debug: dump_shot out of range");
    if (!h->bat.items) {
      fail(QB_INVALID_ARGUMENT, "decode_batch_debug: the batch kernel in use has no message dump "
                                "(generic kernel: use qb_decode_debug)");
    }
    const DecodeParams& P = h->P;
    const bool packed_i8 = h->bat.pair && h->arith == QB_ARITH_INT8;
    const bool is_int = h->arith == QB_ARITH_INT8 || h->arith == QB_ARITH_INT16;
    (void)packed_i8;
    void* qdst = is_int ? static_cast<void*>(q_i32) : static_cast<void*>(q_f32);
    void* rdst = is_int ? static_cast<void*>(r_i32) : static_cast<void*>(r_f32);
    if (!qdst || !rdst) fail(QB_INVALID_ARGUMENT, "decode_batch_debug: message buffers of the wrong type");
    ensure_batch(h, shots, true);
    cudaStream_t st = h->stream;
    CUDA_TRY(cudaMemcpyAsync(h->b_syn, syndromes, shots * P.syn_w32 * 4, cudaMemcpyHostToDevice, st));
    run_batch_device(h, shots, h->b_syn, h->b_est, h->b_res, h->b_conv, h->b_iters, st, -1, nullptr,
                     static_cast<int64_t>(dump_shot));
    CUDA_TRY(cudaMemcpyAsync(estimates, h->b_est, shots * P.est_w32 * 4, cudaMemcpyDeviceToHost, st));
    if (residuals) {
      CUDA_TRY(cudaMemcpyAsync(residuals, h->b_res, shots * P.syn_w32 * 4, cudaMemcpyDeviceToHost, st));
    }
    CUDA_TRY(cudaMemcpyAsync(converged, h->b_conv, shots * P.nseg, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(iterations, h->b_iters, shots * P.nseg * 4, cudaMemcpyDeviceToHost, st));
    const size_t bytes = static_cast<size_t>(P.E) * 4;
    CUDA_TRY(cudaMemcpyAsync(qdst, h->d_qdump, bytes, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(rdst, h->d_rdump, bytes, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  });
}

qb_status qb_decode_batch_soft(qb_decoder* h, uint64_t shots, const uint64_t* syndromes,
                               const void* soft, uint64_t* estimates, uint64_t* residuals,
                               uint8_t* converged, uint32_t* iterations) {
  if (!h) return QB_INVALID_ARGUMENT;
  return guarded(h, [&] {
    if (shots == 0) return;
    require_soft(h, "decode_batch_soft");
    if (!soft) fail(QB_INVALID_ARGUMENT, "decode_batch_soft: NULL soft buffer");
    decode_batch_host(h, shots, syndromes, soft, estimates, residuals, converged, iterations);
  });
}

qb_status qb_decode_batch_soft_device(qb_decoder* h, uint64_t shots, const uint64_t* d_syndromes,
                                      const void* d_soft, uint64_t* d_estimates,
                                      uint64_t* d_residuals, uint8_t* d_converged,
                                      uint32_t* d_iterations, void* stream) {
  if (!h) return QB_INVALID_ARGUMENT;
  return guarded(h, [&] {
    if (shots == 0) return;
    require_soft(h, "decode_batch_soft_device");
    if (!d_syndromes || !d_soft || !d_estimates || !d_converged || !d_iterations) {
      fail(QB_INVALID_ARGUMENT, "decode_batch_soft_device: NULL buffer");
    }
    run_batch_device(h, shots, reinterpret_cast<const uint32_t*>(d_syndromes),
                     reinterpret_cast<uint32_t*>(d_estimates),
                     reinterpret_cast<uint32_t*>(d_residuals), d_converged, d_iterations,
                     static_cast<cudaStream_t>(stream), -1, d_soft);
  });
}

}  // extern "C"

/* qldpc_b200.h — the C-ABI boundary of the B200-native min-sum decoder.
 *
 * This is the drop-in boundary for ONE path of the reference: the scaled
 * min-sum syndrome decoder behind `class qldpc::Decoder` and the free functions
 * `decode`, `decode_batch`, `decode_css`
 * (reference: proj/include/qldpc/decoder.hpp:77-129, proj/src/decoder.cpp).
 * Plain pointers and sizes only; no C++ or torch types cross this line.
 *
 * Conventions shared with the reference:
 *   - a packed bit vector of L bits is ceil(L/64) uint64 words, bit i at
 *     (words[i >> 6] >> (i & 63)) & 1   (proj/include/qldpc/gf2.hpp:26), so
 *     `Gf2Vector::words()` can be passed straight through;
 *   - edges are numbered check-major, `var_edges` ascending per variable
 *     (proj/include/qldpc/tanner_graph.hpp:15-48);
 *   - a decoder over S segments (1 for a plain graph, 2 = X,Z for a CssCode,
 *     proj/src/decoder.cpp:406-424) reports `converged` and `iterations` PER
 *     SEGMENT; `decode_into` semantics are AND / MAX over segments
 *     (decoder.cpp:204-213), `decode_css_into` semantics are the per-segment
 *     values themselves (decoder.cpp:194-202).
 *
 * Every function returns a qb_status.  QB_INVALID_ARGUMENT marks exactly the
 * conditions for which the reference throws std::invalid_argument; any CUDA
 * failure is QB_RUNTIME_ERROR.  The message is available from
 * qb_last_error(handle) (or qb_last_error(NULL) for a failed create).
 * There is NO CPU fallback: without a usable CUDA device every compute entry
 * point fails with QB_RUNTIME_ERROR.
 */
#ifndef QLDPC_B200_H_
#define QLDPC_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  QB_OK = 0,
  QB_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  QB_RUNTIME_ERROR = 2     /* CUDA / resource failure: std::runtime_error */
} qb_status;

/* reference: enum class Arithmetic (decoder.hpp:16).  QB_ARITH_HALF is an
 * extension with no reference counterpart (fp16 messages, fp32 arithmetic). */
typedef enum {
  QB_ARITH_FLOAT = 0,
  QB_ARITH_INT8 = 1,
  QB_ARITH_INT16 = 2,
  QB_ARITH_HALF = 3
} qb_arithmetic;

/* reference: struct TannerGraph (tanner_graph.hpp:15-48). */
typedef struct {
  uint32_t num_checks;
  uint32_t num_vars;
  uint32_t num_edges;
  const uint32_t* edge_var;      /* [num_edges] */
  const uint32_t* check_offsets; /* [num_checks + 1] */
  const uint32_t* var_offsets;   /* [num_vars + 1] */
  const uint32_t* var_edges;     /* [num_edges] */
} qb_graph;

/* reference: struct Segment (decoder.cpp:25-30).  Segments must tile the
 * graph block-diagonally: every edge of a check in [check_begin, check_end)
 * ends at a variable in [var_begin, var_end). */
typedef struct {
  uint32_t check_begin, check_end, var_begin, var_end;
} qb_segment;

/* reference: struct DecoderConfig (decoder.hpp:23-38). */
typedef struct {
  uint64_t max_iterations;   /* >= 1 */
  double alpha;              /* (0, 1] */
  int32_t early_termination; /* 0 / 1 */
  int32_t arithmetic;        /* qb_arithmetic */
  double quant_scale;        /* 0 = mode default (8 for int8, 256 for int16) */
  const double* priors;      /* NULL or num_priors == 0: uniform prior 1 */
  uint64_t num_priors;       /* 0 or num_vars */
} qb_config;

typedef struct qb_decoder qb_decoder;

/* Kernel selection and I/O policy knobs (qb_set_option). */
typedef enum {
  /* 0 = auto, 1 = generic CSR kernel (the "second opinion": any graph, tables read from
   * memory), 2 = auto, but it is an error unless the graph is (6,3)-regular (i.e. the
   * lean kernels serve it). */
  QB_OPT_KERNEL = 0,
  /* Single-shot I/O: 0 = syndrome in the kernel parameters, results to mapped
   * pinned host memory + completion flag (no memcpy, no stream sync);
   * 1 = cudaMemcpyAsync H2D / kernel / D2H + stream synchronize (the reference
   * paper's protocol); 2 = persistent doorbell: a resident
   * cluster polls a block of mapped host memory, so a decode costs no kernel
   * launch at all (the kernel retires after QB_OPT_DOORBELL_IDLE_MS idle). */
  QB_OPT_LATENCY_IO = 1,
  /* Single-shot launch shape: 0 = auto / 2 = one thread block cluster per shot, CTA rank =
   * segment (a decoder built from a plain graph has one segment: one CTA per shot);
   * 1 = one CTA per shot whatever the segment count (one warp group per segment: the
   * generic kernel). */
  QB_OPT_LATENCY_SHAPE = 2,
  /* Threads per segment group (0 = auto). */
  QB_OPT_GROUP_THREADS = 3,
  /* CTAs per SM for the persistent batch kernel (0 = auto). */
  QB_OPT_BATCH_CTAS_PER_SM = 4,
  /* Batch item kernel variant (checks x variables per thread, CTAs per SM):
   * 0 = auto, else one of the instantiations 1, 2, 3, 4, 6, 8, 11 (see kLeanVariants). */
  QB_OPT_BATCH_VARIANT = 5,
  /* Single-shot cluster kernel: 1 or 2 checks (and twice as many variables)
   * per thread, 3 = one check and one variable per thread; 0 = auto (3 for float
   * decoders of small codes, else 1). */
  QB_OPT_LATENCY_NODES_PER_THREAD = 6,
  /* (6,3)-regular kernels: 1 (default) lets uniform-prior decoders use the
   * instantiation with the prior as a kernel constant and (fp32) without the
   * provably unreachable 1e30 clamp; 0 forces the general instantiation. */
  QB_OPT_FAST_PATH = 7,
  /* Batch work decomposition: 0 = auto / 2 = one CTA per (shot, segment) work item drawn
   * from per-segment queues (the lean and degree-padded item kernels), 1 = one CTA per
   * shot with one warp group per segment (the generic kernel). */
  QB_OPT_BATCH_SHAPE = 8,
  QB_OPT_DOORBELL_IDLE_MS = 9,
  /* Half and int8 modes, batch calls on (6,3)-regular codes: 1 (default) = decode
   * two shots per thread in the two lanes of packed fp16 instructions (int8
   * values are exact fp16 integers; used only when the loader has verified the
   * Q16 scaling for all 128 magnitudes); 0 = one shot per thread.  Results are
   * identical either way. */
  QB_OPT_HALF_PAIRS = 10,
  /* 1 = bracket every single-shot decode of the memcpy protocol (QB_OPT_LATENCY_IO
   * = 1) with CUDA events on its stream: H2D copy + kernel + D2H copy as the device
   * sees them (the reference paper's timing).  qb_latency_run then
   * reports that span in kernel_ns[] instead of the in-kernel %globaltimer span;
   * QB_OPT_INFO_LAST_EVENT_NS returns the most recent one. */
  QB_OPT_LATENCY_EVENTS = 11,
  /* Memcpy protocol (QB_OPT_LATENCY_IO = 1): 1 (default) = H2D copy, cluster kernel
   * and D2H copy are ONE CUDA-graph launch per decode (captured on first use);
   * 0 = three separate stream operations. */
  QB_OPT_LATENCY_GRAPH = 12,
  /* Lean batch kernel: shots per syndrome tile (one TMA bulk copy and one queue
   * ticket per tile), 1 .. 16; 0 = auto (16 for large batches, smaller when that
   * would leave resident CTAs without work). */
  QB_OPT_BATCH_TILE = 13,
  /* Lean batch kernels ((6,3)-regular codes): the loader permutes the six message slots
   * inside every check's block so that the variable-side accesses of a warp spread over the
   * shared-memory banks (results are unaffected: the check update is symmetric in its
   * slots).  0 = slots in row order; 1 = greedy assignment + one pass of improving swaps
   * (~1 ms); 2 (default) = as 1, then refined by simulated annealing (200 moves per edge,
   * fixed seed: ~25 ms on [[784,24,24]], paid once per graph and thread shape in a process -
   * the tables are cached; 1.72 -> 1.43 shared-memory wavefronts per variable-side access:
   * +1 % on float, +2 % / +3 % / +3.6 % on int8 / half / int16 at 10 fixed iterations). */
  QB_OPT_SLOT_SPREAD = 14,
  /* qb_decode_batch (host buffers): shots per pipeline chunk (H2D copy, kernel and D2H
   * copy of consecutive chunks overlap on three streams); 0 = auto (2^15).  Also the
   * trials per sample / decode / classify round of qb_campaign_run (0 = 2^20). */
  QB_OPT_BATCH_CHUNK = 15,
  /* qb_generate_syndromes / qb_campaign_run: 0 (default) = the reference's SplitMix64
   * stream, bit for bit (one draw per variable); 1 = the same i.i.d. Bernoulli
   * distribution sampled by geometric skips (one draw per FLIP; per-variable
   * probabilities by thinning) - a different stream, keyed by (seed, trial) in the
   * same way, for campaigns that need the statistics but not the reference's trials
   * ("device RNG need not reproduce SplitMix64 bit-streams"). */
  QB_OPT_SAMPLER = 16,
  /* qb_campaign_run / qb_campaign_run_multi on (6,3)-regular CSS codes in float / int16 mode:
   * 1 (default) = the whole trial loop in ONE kernel (kernel_campaign.cuh: every thread
   * samples the error bits of its own variables with the reference's SplitMix64 stream, the
   * syndrome is built in shared memory, the residual is classified from registers; 10 bytes
   * per trial reach HBM); 0 = sampler, decode and classifier as three kernels per round.
   * Counters are identical either way (and identical to the reference's run_campaign). */
  QB_OPT_CAMPAIGN_FUSED = 17,
  /* Memcpy protocol of single shots (QB_OPT_LATENCY_IO = 1): how the host learns that the
   * D2H copy has landed.  0 (default) = cudaStreamSynchronize, the paper's literal protocol;
   * 1 = watch the pinned destination: every 32-byte sector of the copied record carries the
   * shot's tag, so the record is complete when all of them show it (-3 us per decode).
   * Ignored while QB_OPT_LATENCY_EVENTS = 1 (reading the events needs the synchronize). */
  QB_OPT_LATENCY_WAIT = 18,
  /* Read-only (qb_get_option): the launch plans actually in use. */
  QB_OPT_INFO_BATCH_CTAS_PER_SM = 100,
  QB_OPT_INFO_BATCH_BLOCK = 101,
  QB_OPT_INFO_LATENCY_BLOCK = 102,
  QB_OPT_INFO_LATENCY_CLUSTER = 103,
  QB_OPT_INFO_BATCH_REGULAR = 104,
  QB_OPT_INFO_FAST_ELIGIBLE = 105,
  QB_OPT_INFO_LATENCY_LEAN = 106,
  /* 100 * DC + DV of the degree-padded batch kernel in use (irregular graphs whose
   * degrees fit an instantiated bound), 0 when another kernel serves batches. */
  QB_OPT_INFO_BATCH_ELL = 107,
  QB_OPT_INFO_LAST_EVENT_NS = 108
} qb_option;

/* Builds a decoder: validates like Decoder::Decoder (decoder.cpp:373-404,
 * :83-131), uploads the code tables and allocates every device / pinned
 * buffer, so decode calls are allocation-free.  The graph arrays are copied;
 * they need not outlive the call.  `device` is the CUDA ordinal. */
qb_status qb_decoder_create(const qb_graph* graph, const qb_segment* segments,
                            uint32_t num_segments, const qb_config* config,
                            int device, qb_decoder** out);

void qb_decoder_destroy(qb_decoder* h);

/* Thread-local for h == NULL (create failures), else the handle's. */
const char* qb_last_error(const qb_decoder* h);

qb_status qb_set_option(qb_decoder* h, int option, int64_t value);
int64_t qb_get_option(const qb_decoder* h, int option);

uint32_t qb_num_checks(const qb_decoder* h);
uint32_t qb_num_vars(const qb_decoder* h);
uint32_t qb_num_segments(const qb_decoder* h);

/* Decoder::decode_into / decode_css_into (decoder.cpp:551-591) for ONE
 * syndrome, latency path.  All pointers are HOST memory.
 *   syndrome   ceil(M/64) words      estimate  ceil(N/64) words (out)
 *   residual   ceil(M/64) words (out, may be NULL)
 *   converged  [num_segments] (out)  iterations [num_segments] (out) */
qb_status qb_decode(qb_decoder* h, const uint64_t* syndrome,
                    uint64_t* estimate, uint64_t* residual, uint8_t* converged,
                    uint32_t* iterations);

/* decode_batch (decoder.cpp:604-655) for `shots` syndromes held in HOST
 * memory (pinned memory from qb_host_alloc makes the copies asynchronous):
 * H2D, persistent decode kernel, D2H, all inside the call.  Strides are the
 * packed word counts above; converged / iterations are [shots][num_segments].
 * Results are elementwise identical to `shots` qb_decode calls. */
qb_status qb_decode_batch(qb_decoder* h, uint64_t shots,
                          const uint64_t* syndromes, uint64_t* estimates,
                          uint64_t* residuals /* may be NULL */,
                          uint8_t* converged, uint32_t* iterations);

/* Same, with every buffer already resident in DEVICE memory (16-byte aligned)
 * and the launch enqueued on `stream` (a cudaStream_t, NULL = default); returns without
 * synchronising.  A decoder is NOT thread-safe (as the reference's, decoder.hpp:75-76), but
 * one host thread may keep several of these launches in flight on different streams: each
 * takes its own scheduler words from a ring of 16.  qb_classify_batch_device and the
 * campaign calls share one counter buffer per handle and block until their result is back. */
qb_status qb_decode_batch_device(qb_decoder* h, uint64_t shots,
                                 const uint64_t* d_syndromes,
                                 uint64_t* d_estimates,
                                 uint64_t* d_residuals /* may be NULL */,
                                 uint8_t* d_converged, uint32_t* d_iterations,
                                 void* stream);

/* Debug / parity: decode one syndrome and also return the final edge messages
 * q (variable->check) and r (check->variable) in reference edge order, as
 * float for QB_ARITH_FLOAT / QB_ARITH_HALF and int32 for the integer modes
 * (pass the matching pair, NULL for the other). */
qb_status qb_decode_debug(qb_decoder* h, const uint64_t* syndrome,
                          uint64_t* estimate, uint64_t* residual,
                          uint8_t* converged, uint32_t* iterations,
                          float* q_f32, float* r_f32, int32_t* q_i32,
                          int32_t* r_i32);

/* The same for the THROUGHPUT kernels: decodes `shots` syndromes (host memory) with the
 * persistent batch kernel exactly as qb_decode_batch_device would - syndrome tiles, work
 * queues, the first iteration evaluated from the syndrome on uniform-prior decoders - and
 * additionally returns the final edge messages of shot `dump_shot`.  On the kernels that
 * decode two shots per thread (half / int8 pairs) the messages are those at the moment the
 * PAIR (dump_shot, dump_shot ^ 1) finished: the shot's own final messages when its partner did
 * not run longer.  QB_INVALID_ARGUMENT when the generic kernel serves batches. */
qb_status qb_decode_batch_debug(qb_decoder* h, uint64_t shots, const uint64_t* syndromes,
                                uint64_t dump_shot, uint64_t* estimates,
                                uint64_t* residuals /* may be NULL */, uint8_t* converged,
                                uint32_t* iterations, float* q_f32, float* r_f32,
                                int32_t* q_i32, int32_t* r_i32);

/* Latency harness with the reference's run_bench protocol at batch 1
 * (proj/src/bench.cpp:182-337): decode pool[(b) % pool_size] for b in
 * [0, warmup + measure); for each measured decode record the host wall-clock
 * nanoseconds of the whole qb_decode (copy-in, launch, completion, copy-out)
 * in wall_ns[measure] and the device %globaltimer span in kernel_ns[measure]
 * (either may be NULL).  *digest receives the reference's FNV-1a output digest
 * (bench.cpp:27-36, :287-291) over (converged AND, iterations MAX as uint64,
 * estimate words) of the measured decodes, so a GPU run can be compared with
 * BenchResult::output_digest of the CPU reference. */
qb_status qb_latency_run(qb_decoder* h, const uint64_t* pool,
                         uint64_t pool_size, uint64_t warmup, uint64_t measure,
                         uint64_t* wall_ns, uint64_t* kernel_ns,
                         uint64_t* digest);

/* ... the same with per-shot priors: soft_pool = [pool_size][num_checks] values in the
 * layout of qb_decode_batch_soft (NULL = qb_latency_run); every decode is a qb_decode_soft. */
qb_status qb_latency_run_soft(qb_decoder* h, const uint64_t* pool, const void* soft_pool,
                              uint64_t pool_size, uint64_t warmup, uint64_t measure,
                              uint64_t* wall_ns, uint64_t* kernel_ns,
                              uint64_t* digest);

/* Decoder::last_kernel_ns (decoder.cpp:593-596): device-side %globaltimer
 * span of the most recent qb_decode (first instruction to last store). */
uint64_t qb_last_kernel_ns(const qb_decoder* h);

/* Number of kernels this handle has launched since creation. */
uint64_t qb_launch_count(const qb_decoder* h);

/* On-device code-capacity noise + syndrome generator (reference:
 * sample_error + extract_syndromes, proj/src/noise.cpp:67-105), bit-exact
 * with the reference's SplitMix64 streams: shot i of the call is trial
 * `first_trial + i` of NoiseModel{independent-xz, p, seed}.  Each variable of
 * the decoder's graph flips with probability `p` (or `probs[v]`, a HOST array
 * of num_vars doubles, when non-NULL); the syndrome H*e is written packed to
 * DEVICE memory `d_syndromes` ([shots][ceil(M/64)] words) and, if non-NULL, the
 * sampled error to `d_errors` ([shots][ceil(N/64)] words).
 * `css_interleave` = 1 maps the variables of a two-segment CSS decoder onto
 * the reference's draw order (X_0, Z_0, X_1, Z_1, ...); 0 uses draw v for
 * variable v. */
qb_status qb_generate_syndromes(qb_decoder* h, uint64_t seed, double p,
                                const double* probs, int css_interleave,
                                uint64_t first_trial, uint64_t shots,
                                uint64_t* d_syndromes, uint64_t* d_errors,
                                void* stream);

/* Monte-Carlo campaign on the device (reference: run_campaign,
 * proj/src/noise.cpp:217-338): sample -> syndrome -> decode -> classify, with
 * nothing but ten counters crossing PCIe.
 *
 * qb_set_logicals supplies the residual tests for a two-segment (CSS) decoder:
 * `x_tests` / `z_tests` are `n_x` / `n_z` packed vectors over ALL num_vars
 * variables (combined layout, host memory); a converged X (Z) residual counts
 * as a logical error iff it has odd overlap with at least one x_test (z_test).
 * With the code's logical Z operators placed on the X-error variables as
 * x_tests (and logical X operators on the Z-error variables as z_tests) this is
 * exactly the reference's row-space membership test for zero-syndrome residuals.
 *
 * qb_campaign_run decodes trials [first_trial, first_trial + trials) of
 * NoiseModel{independent-xz, p, seed} and ADDS to `counters` (host, 10 words):
 *   [0] exact [1] stabilizer [2] logical_x [3] logical_z [4] logical_both
 *   [5] non_converged [6] baseline failures (identity decoder) [7] trials with
 *   both components converged [8] sum over trials of max(iterations_x,
 *   iterations_z) [9] trials.
 * Float / int8 / int16 results are identical to the reference's counts. */
qb_status qb_set_logicals(qb_decoder* h, const uint64_t* x_tests, uint32_t n_x,
                          const uint64_t* z_tests, uint32_t n_z);
qb_status qb_campaign_run(qb_decoder* h, uint64_t seed, double p,
                          const double* probs, uint64_t first_trial,
                          uint64_t trials, uint64_t* counters);
/* The same campaign on SEVERAL GPUs of one node from one process: `handles[g]` is a decoder
 * created on its own device (same graph / config, qb_set_logicals called on each).  GPU g
 * decodes the contiguous shard [g*T/n, (g+1)*T/n) of the trial range (the reference's worker
 * split, proj/src/noise.cpp:253-254; trial streams are keyed by the global trial id, so the
 * result does not depend on n), all devices run concurrently, and the ten counters are
 * summed with ONE ncclAllReduce(ncclSum, ncclUint64, 10) over NVLink (the integer sum of
 * noise.cpp:306-324) - the path's only collective.  NCCL is bound at run time (dlopen of
 * libnccl.so.2); QB_RUNTIME_ERROR if it is absent.  ADDS to `counters` like qb_campaign_run. */
qb_status qb_campaign_run_multi(qb_decoder* const* handles, uint32_t n, uint64_t seed,
                                double p, const double* probs, uint64_t first_trial,
                                uint64_t trials, uint64_t* counters);
/* The classification step alone, on buffers already resident in DEVICE memory
 * (errors from qb_generate_syndromes, outputs of qb_decode_batch_device);
 * ADDS to the same ten host counters. */
qb_status qb_classify_batch_device(qb_decoder* h, uint64_t shots,
                                   const uint64_t* d_errors,
                                   const uint64_t* d_estimates,
                                   const uint64_t* d_syndromes,
                                   const uint8_t* d_converged,
                                   const uint32_t* d_iterations,
                                   uint64_t* counters, void* stream);

/* ---- Soft (noisy) syndromes: per-shot priors -----------------------------------------
 *
 * The reference takes priors per Decoder (decoder.hpp:31-32, decoder.cpp:108-131); soft
 * syndrome information is per SHOT.  On an extended graph [H | I] the identity column of
 * check m is a degree-1 "measurement error" variable whose prior is the reliability
 * |LLR_m| of the measured bit: the reference handles it through its
 * degree-1-variable path (decoder.cpp:324-329) with one Decoder constructed per shot.
 * Here the loader lets every check ABSORB its first degree-1 variable, and the calls below
 * take that variable's prior per shot:
 *
 *   soft[shot][m], m in [0, num_checks) = prior of qb_soft_vars()[m] for this shot
 *     QB_ARITH_FLOAT / QB_ARITH_HALF : float   (what the reference stores: float(prior))
 *     QB_ARITH_INT8                  : int8_t  the QUANTISED prior, non-zero, |x| <= 127
 *     QB_ARITH_INT16                 : int16_t the QUANTISED prior, non-zero, |x| <= 32767
 *   (quantised = quantize_saturate(prior, quant_scale, kmax), decoder.cpp:115-122, :500-509;
 *   the reference rejects priors that quantise to 0.)  Entries of checks without an absorbed
 *   variable (qb_soft_vars()[m] == 0xffffffff) are ignored.  Every other prior is the
 *   decoder's (qb_config::priors).
 *
 * Results equal those of a reference Decoder built for each shot on the same graph with
 * `priors[qb_soft_vars()[m]] = soft[shot][m]` (de-quantised: value / quant_scale).
 * QB_INVALID_ARGUMENT when the decoder's batch kernel is not the degree-padded one. */
qb_status qb_soft_vars(const qb_decoder* h, uint32_t* vars /* [num_checks] out */);
/* ... for ONE shot, latency path (qb_decode with `soft` = [num_checks] values, host memory);
 * all three single-shot I/O protocols (QB_OPT_LATENCY_IO). */
qb_status qb_decode_soft(qb_decoder* h, const uint64_t* syndrome, const void* soft,
                         uint64_t* estimate, uint64_t* residual /* may be NULL */,
                         uint8_t* converged, uint32_t* iterations);
qb_status qb_decode_batch_soft(qb_decoder* h, uint64_t shots, const uint64_t* syndromes,
                               const void* soft, uint64_t* estimates,
                               uint64_t* residuals /* may be NULL */, uint8_t* converged,
                               uint32_t* iterations);
qb_status qb_decode_batch_soft_device(qb_decoder* h, uint64_t shots,
                                      const uint64_t* d_syndromes, const void* d_soft,
                                      uint64_t* d_estimates,
                                      uint64_t* d_residuals /* may be NULL */,
                                      uint8_t* d_converged, uint32_t* d_iterations,
                                      void* stream);

/* Device generator of soft syndromes (BASELINE config 5; the reference has no such noise
 * model): data variables flip with probability p (or probs[v]; the entries of
 * absorbed variables are ignored), every check m with an absorbed variable is then measured
 * through a Gaussian channel  l_m = (1 - 2 s~_m) mu + N(0, sigma^2)  around its noiseless
 * bit s~_m: d_syndromes receives the hard bits [l_m < 0], d_soft the reliabilities
 * 2 mu |l_m| / sigma^2 in the decoder's soft format (integer modes: quantised with the
 * decoder's quant_scale, clamped to [1, kmax]), d_errors (may be NULL) the data errors plus
 * one error on the absorbed variable of every flipped measurement, so that
 * H_ext * error == syndrome.  Counter-based stream keyed by (seed, trial, check). */
qb_status qb_generate_soft_syndromes(qb_decoder* h, uint64_t seed, double p,
                                     const double* probs, double mu, double sigma,
                                     uint64_t first_trial, uint64_t shots,
                                     uint64_t* d_syndromes, void* d_soft,
                                     uint64_t* d_errors, void* stream);

/* Campaigns on extended graphs.  qb_set_auxiliary_vars marks the variables that are NOT data
 * qubits (packed mask over num_vars, host memory; NULL clears): for a converged shot
 * H_ext r = 0 means H r_data = r_aux, so a residual with a bit on an auxiliary variable has
 * a data part with non-zero syndrome and is counted as a logical error of its component
 * (the tests of qb_set_logicals then only see data bits).  With a mask set, qb_campaign_run
 * samples variable v from draw v (no X/Z interleave).  qb_campaign_run_soft is the same
 * loop with qb_generate_soft_syndromes + qb_decode_batch_soft_device: sample, soft
 * measurement, decode, classify, all on the device. */
qb_status qb_set_auxiliary_vars(qb_decoder* h, const uint64_t* mask);
qb_status qb_campaign_run_soft(qb_decoder* h, uint64_t seed, double p, const double* probs,
                               double mu, double sigma, uint64_t first_trial,
                               uint64_t trials, uint64_t* counters);

/* Pinned (page-locked, device-mapped) host memory for batch I/O. */
qb_status qb_host_alloc(void** out, size_t bytes);
void qb_host_free(void* p);

/* Measures the device's aggregate shared-memory bandwidth (GB/s) with a
 * conflict-free streaming 50/50 load/store kernel on every SM: `gbs_32bit` with
 * 32-bit accesses (the message arrays' access width), `gbs_128bit` with 128-bit
 * accesses (the crossbar ceiling).  Used as the roofline denominator. */
qb_status qb_measure_smem_bandwidth(int device, double* gbs_32bit,
                                    double* gbs_128bit);

/* Library / device description, e.g. for bench logs. */
const char* qb_version(void);
qb_status qb_device_info(int device, char* name, size_t name_len,
                         int* sm_count, int* cc_major, int* cc_minor);

#ifdef __cplusplus
}
#endif
#endif /* QLDPC_B200_H_ */

// TEST INFRASTRUCTURE — not part of the product.
//
// Thin C wrapper over the UNMODIFIED reference library (compiled from the
// sources where they lie under /root/reference/proj by oracle/Makefile, output
// only into oracle/_ref/).  It exists so that tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs can drive the reference
// `qldpc::Decoder`, `run_bench`, `run_campaign`, `sample_error` ... through
// ctypes.  Nothing under paper_2508_07879_b200/ may load this library.
//
// Every entry point returns 0 on success, 1 for std::invalid_argument, 2 for
// any other exception; the message is retrievable with ref_last_error().

#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "qldpc/alist.hpp"
#include "qldpc/bench.hpp"
#include "qldpc/css_code.hpp"
#ifdef REF_HAVE_CSS_JSON
#include "qldpc/css_json.hpp"
#endif
#include "qldpc/decoder.hpp"
#include "qldpc/gf2.hpp"
#include "qldpc/noise.hpp"
#include "qldpc/tanner_graph.hpp"

using namespace qldpc;

namespace {

thread_local std::string g_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_error.clear();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 2;
  } catch (...) {
    g_error = "unknown exception";
    return 2;
  }
}

Gf2Vector vec_from_words(const std::uint64_t* words, std::size_t bits) {
  Gf2Vector v(bits);
  auto w = v.words();
  for (std::size_t i = 0; i < w.size(); ++i) w[i] = words[i];
  return v;
}

void words_from_vec(const Gf2Vector& v, std::uint64_t* out) {
  auto w = v.words();
  for (std::size_t i = 0; i < w.size(); ++i) out[i] = w[i];
}

struct GraphBox {
  TannerGraph graph;
};

DecoderConfig make_cfg(std::uint64_t max_iter, double alpha, int early,
                       int arith, double quant_scale, const double* priors,
                       std::uint64_t n_priors) {
  DecoderConfig cfg;
  cfg.max_iterations = static_cast<std::size_t>(max_iter);
  cfg.alpha = alpha;
  cfg.early_termination = early != 0;
  cfg.arithmetic = arith == 0   ? Arithmetic::kFloat
                   : arith == 1 ? Arithmetic::kInt8
                                : Arithmetic::kInt16;
  cfg.quant_scale = quant_scale;
  if (priors != nullptr) cfg.priors.assign(priors, priors + n_priors);
  return cfg;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

// ---------------------------------------------------------------- codes ----

int ref_code_builtin(const char* name, void** out) {
  return guarded([&] { *out = new CssCode(make_builtin_code(name)); });
}

// terms are (x_exp, y_exp) pairs, flattened.
int ref_code_bb(std::uint64_t l, std::uint64_t m, const std::uint32_t* a_terms,
                std::uint32_t na, const std::uint32_t* b_terms,
                std::uint32_t nb, const char* name, std::uint64_t d,
                void** out) {
  return guarded([&] {
    BbCodeSpec spec;
    spec.l = l;
    spec.m = m;
    for (std::uint32_t i = 0; i < na; ++i) {
      spec.a_terms.push_back({a_terms[2 * i], a_terms[2 * i + 1]});
    }
    for (std::uint32_t i = 0; i < nb; ++i) {
      spec.b_terms.push_back({b_terms[2 * i], b_terms[2 * i + 1]});
    }
    *out = new CssCode(build_bb_code(spec, name ? name : "", d));
  });
}

// Generic CSS code from COO entries of hx and hz.
int ref_code_from_coo(const char* name, std::uint32_t rows_x,
                      std::uint32_t rows_z, std::uint32_t cols,
                      const std::uint32_t* hx_rc, std::uint64_t nnz_x,
                      const std::uint32_t* hz_rc, std::uint64_t nnz_z,
                      void** out) {
  return guarded([&] {
    std::vector<SparseGf2Matrix::Entry> ex, ez;
    for (std::uint64_t i = 0; i < nnz_x; ++i) {
      ex.push_back({hx_rc[2 * i], hx_rc[2 * i + 1]});
    }
    for (std::uint64_t i = 0; i < nnz_z; ++i) {
      ez.push_back({hz_rc[2 * i], hz_rc[2 * i + 1]});
    }
    *out = new CssCode(name, SparseGf2Matrix(rows_x, cols, ex),
                       SparseGf2Matrix(rows_z, cols, ez));
  });
}

void ref_code_free(void* code) { delete static_cast<CssCode*>(code); }

void ref_code_params(const void* code, std::uint64_t* n, std::uint64_t* k,
                     std::uint64_t* d, std::uint64_t* rows_x,
                     std::uint64_t* rows_z) {
  const auto* c = static_cast<const CssCode*>(code);
  *n = c->params().n;
  *k = c->params().k;
  *d = c->params().d;
  *rows_x = c->hx().rows();
  *rows_z = c->hz().rows();
}

// which: 0 = graph_x (from hz), 1 = graph_z (from hx), 2 = combined.
// The returned pointer is owned by the code.
const void* ref_code_graph(const void* code, int which) {
  const auto* c = static_cast<const CssCode*>(code);
  const TannerGraph* g = which == 0   ? &c->graph_x()
                         : which == 1 ? &c->graph_z()
                                      : &c->combined_graph();
  return g;
}

// Row supports of hx (which=0) / hz (which=1) as COO (row, col) pairs.
std::uint64_t ref_code_matrix_nnz(const void* code, int which) {
  const auto* c = static_cast<const CssCode*>(code);
  return which == 0 ? c->hx().nnz() : c->hz().nnz();
}

void ref_code_matrix_coo(const void* code, int which, std::uint32_t* rc) {
  const auto* c = static_cast<const CssCode*>(code);
  const SparseGf2Matrix& h = which == 0 ? c->hx() : c->hz();
  std::size_t k = 0;
  for (std::size_t r = 0; r < h.rows(); ++r) {
    for (std::uint32_t col : h.row_support(r)) {
      rc[k++] = static_cast<std::uint32_t>(r);
      rc[k++] = col;
    }
  }
}

// --------------------------------------------------------------- graphs ----

// Builds a free-standing graph from COO entries (owned by the caller).
int ref_graph_from_coo(std::uint32_t rows, std::uint32_t cols,
                       const std::uint32_t* rc, std::uint64_t nnz,
                       void** out) {
  return guarded([&] {
    std::vector<SparseGf2Matrix::Entry> entries;
    for (std::uint64_t i = 0; i < nnz; ++i) {
      entries.push_back({rc[2 * i], rc[2 * i + 1]});
    }
    auto box = std::make_unique<GraphBox>();
    box->graph = build_tanner_graph(SparseGf2Matrix(rows, cols, entries));
    *out = box.release();
  });
}

int ref_graph_toy(void** out) {
  return guarded([&] {
    auto box = std::make_unique<GraphBox>();
    box->graph = build_tanner_graph(toy_code_3x6());
    *out = box.release();
  });
}

const void* ref_graphbox_graph(const void* box) {
  return &static_cast<const GraphBox*>(box)->graph;
}

void ref_graphbox_free(void* box) { delete static_cast<GraphBox*>(box); }

void ref_graph_dims(const void* graph, std::uint64_t* m, std::uint64_t* n,
                    std::uint64_t* e) {
  const auto* g = static_cast<const TannerGraph*>(graph);
  *m = g->num_checks;
  *n = g->num_vars;
  *e = g->num_edges();
}

void ref_graph_arrays(const void* graph, std::uint32_t* edge_var,
                      std::uint32_t* edge_check, std::uint32_t* check_offsets,
                      std::uint32_t* var_offsets, std::uint32_t* var_edges) {
  const auto* g = static_cast<const TannerGraph*>(graph);
  std::memcpy(edge_var, g->edge_var.data(), 4 * g->edge_var.size());
  std::memcpy(edge_check, g->edge_check.data(), 4 * g->edge_check.size());
  std::memcpy(check_offsets, g->check_offsets.data(),
              4 * g->check_offsets.size());
  std::memcpy(var_offsets, g->var_offsets.data(), 4 * g->var_offsets.size());
  std::memcpy(var_edges, g->var_edges.data(), 4 * g->var_edges.size());
}

// -------------------------------------------------------------- decoder ----

int ref_decoder_new_graph(const void* graph, std::uint64_t max_iter,
                          double alpha, int early, int arith,
                          double quant_scale, const double* priors,
                          std::uint64_t n_priors, void** out) {
  return guarded([&] {
    *out = new Decoder(*static_cast<const TannerGraph*>(graph),
                       make_cfg(max_iter, alpha, early, arith, quant_scale,
                                priors, n_priors));
  });
}

int ref_decoder_new_code(const void* code, std::uint64_t max_iter,
                         double alpha, int early, int arith,
                         double quant_scale, const double* priors,
                         std::uint64_t n_priors, void** out) {
  return guarded([&] {
    *out = new Decoder(*static_cast<const CssCode*>(code),
                       make_cfg(max_iter, alpha, early, arith, quant_scale,
                                priors, n_priors));
  });
}

void ref_decoder_free(void* dec) { delete static_cast<Decoder*>(dec); }

// decode_into: syndrome has `bits` bits; outputs sized by the decoder's graph.
int ref_decode(void* dec, const std::uint64_t* syndrome, std::uint64_t bits,
               std::uint64_t* estimate, std::uint64_t* residual,
               std::uint8_t* converged, std::uint64_t* iterations,
               std::uint64_t* kernel_ns) {
  return guarded([&] {
    auto* d = static_cast<Decoder*>(dec);
    DecodeOutcome out;
    d->decode_into(vec_from_words(syndrome, bits), out);
    words_from_vec(out.error_estimate, estimate);
    words_from_vec(out.syndrome_residual, residual);
    *converged = out.converged ? 1 : 0;
    *iterations = out.iterations_used;
    if (kernel_ns) *kernel_ns = d->last_kernel_ns();
  });
}

// Loop of decode_into over `shots` syndromes (stride = ceil(bits/64) words),
// single thread, one reused Decoder: the reference's sequential path.
int ref_decode_many(void* dec, std::uint64_t shots,
                    const std::uint64_t* syndromes, std::uint64_t bits,
                    std::uint64_t* estimates, std::uint64_t* residuals,
                    std::uint8_t* converged, std::uint32_t* iterations) {
  return guarded([&] {
    auto* d = static_cast<Decoder*>(dec);
    const std::size_t sw = (bits + 63) / 64;
    const std::size_t ew = (d->num_vars() + 63) / 64;
    const std::size_t rw = (d->num_checks() + 63) / 64;
    DecodeOutcome out;
    for (std::uint64_t i = 0; i < shots; ++i) {
      d->decode_into(vec_from_words(syndromes + i * sw, bits), out);
      words_from_vec(out.error_estimate, estimates + i * ew);
      if (residuals) words_from_vec(out.syndrome_residual, residuals + i * rw);
      converged[i] = out.converged ? 1 : 0;
      iterations[i] = static_cast<std::uint32_t>(out.iterations_used);
    }
  });
}

int ref_decode_css(void* dec, const std::uint64_t* s_x, std::uint64_t bits_x,
                   const std::uint64_t* s_z, std::uint64_t bits_z,
                   std::uint64_t* est_x, std::uint64_t* res_x,
                   std::uint8_t* conv_x, std::uint64_t* iters_x,
                   std::uint64_t* est_z, std::uint64_t* res_z,
                   std::uint8_t* conv_z, std::uint64_t* iters_z) {
  return guarded([&] {
    auto* d = static_cast<Decoder*>(dec);
    DecodeOutcome ox, oz;
    d->decode_css_into(vec_from_words(s_x, bits_x), vec_from_words(s_z, bits_z),
                       ox, oz);
    words_from_vec(ox.error_estimate, est_x);
    words_from_vec(ox.syndrome_residual, res_x);
    *conv_x = ox.converged;
    *iters_x = ox.iterations_used;
    words_from_vec(oz.error_estimate, est_z);
    words_from_vec(oz.syndrome_residual, res_z);
    *conv_z = oz.converged;
    *iters_z = oz.iterations_used;
  });
}

// Free function decode_batch (std::thread partition).  `bits_each` may hold a
// per-shot bit length to exercise the length validation; NULL = all `bits`.
int ref_decode_batch(const void* graph, std::uint64_t shots,
                     const std::uint64_t* syndromes, std::uint64_t bits,
                     const std::uint64_t* bits_each, std::uint64_t max_iter,
                     double alpha, int early, int arith, double quant_scale,
                     const double* priors, std::uint64_t n_priors,
                     unsigned workers, std::uint64_t* estimates,
                     std::uint64_t* residuals, std::uint8_t* converged,
                     std::uint32_t* iterations) {
  return guarded([&] {
    const auto* g = static_cast<const TannerGraph*>(graph);
    const std::size_t sw = (bits + 63) / 64;
    std::vector<Gf2Vector> in;
    in.reserve(shots);
    for (std::uint64_t i = 0; i < shots; ++i) {
      in.push_back(
          vec_from_words(syndromes + i * sw, bits_each ? bits_each[i] : bits));
    }
    const auto out = decode_batch(
        *g, in,
        make_cfg(max_iter, alpha, early, arith, quant_scale, priors, n_priors),
        workers);
    const std::size_t ew = (g->num_vars + 63) / 64;
    const std::size_t rw = (g->num_checks + 63) / 64;
    for (std::uint64_t i = 0; i < shots; ++i) {
      words_from_vec(out[i].error_estimate, estimates + i * ew);
      if (residuals) {
        words_from_vec(out[i].syndrome_residual, residuals + i * rw);
      }
      converged[i] = out[i].converged ? 1 : 0;
      iterations[i] = static_cast<std::uint32_t>(out[i].iterations_used);
    }
  });
}

// Soft (noisy) syndromes: the reference's priors are per Decoder (decoder.hpp:31-32), so
// per-shot priors mean ONE Decoder PER SHOT: shot i uses `priors` with
// priors[soft_vars[k]] = soft[i][k].  Single-segment graph constructor, as ref_decode_many.
int ref_decode_many_soft(const void* graph, std::uint64_t max_iter, double alpha,
                         int early, int arith, double quant_scale,
                         const double* priors, std::uint64_t n_priors,
                         const std::uint32_t* soft_vars, std::uint32_t nsoft,
                         const double* soft, std::uint64_t shots,
                         const std::uint64_t* syndromes, std::uint64_t bits,
                         std::uint64_t* estimates, std::uint64_t* residuals,
                         std::uint8_t* converged, std::uint32_t* iterations) {
  return guarded([&] {
    const auto* g = static_cast<const TannerGraph*>(graph);
    DecoderConfig cfg =
        make_cfg(max_iter, alpha, early, arith, quant_scale, priors, n_priors);
    if (cfg.priors.empty()) cfg.priors.assign(g->num_vars, 1.0);
    const std::size_t sw = (bits + 63) / 64;
    const std::size_t ew = (g->num_vars + 63) / 64;
    const std::size_t rw = (g->num_checks + 63) / 64;
    DecodeOutcome out;
    for (std::uint64_t i = 0; i < shots; ++i) {
      for (std::uint32_t k = 0; k < nsoft; ++k) {
        if (soft_vars[k] < g->num_vars) cfg.priors[soft_vars[k]] = soft[i * nsoft + k];
      }
      Decoder d(*g, cfg);
      d.decode_into(vec_from_words(syndromes + i * sw, bits), out);
      words_from_vec(out.error_estimate, estimates + i * ew);
      if (residuals) words_from_vec(out.syndrome_residual, residuals + i * rw);
      converged[i] = out.converged ? 1 : 0;
      iterations[i] = static_cast<std::uint32_t>(out.iterations_used);
    }
  });
}

// ------------------------------------------------------------- node ops ----

int ref_check_node_update(const double* q, std::uint64_t deg, int s_bit,
                          double alpha, double* r) {
  return guarded([&] {
    const auto out =
        check_node_update(std::span<const double>(q, deg), s_bit, alpha);
    for (std::size_t i = 0; i < out.size(); ++i) r[i] = out[i];
  });
}

int ref_variable_node_update(double gamma, const double* r, std::uint64_t deg,
                             double* q) {
  return guarded([&] {
    const auto out = variable_node_update(gamma, std::span<const double>(r, deg));
    for (std::size_t i = 0; i < out.size(); ++i) q[i] = out[i];
  });
}

int ref_posterior_and_decision(double gamma, const double* r,
                               std::uint64_t deg, double* posterior,
                               int* bit) {
  return guarded([&] {
    const auto pr = posterior_and_decision(gamma, std::span<const double>(r, deg));
    *posterior = pr.first;
    *bit = pr.second;
  });
}

int ref_quantize_saturate(double value, double scale, std::int32_t limit,
                          std::int32_t* out) {
  return guarded([&] { *out = quantize_saturate(value, scale, limit); });
}

// ---------------------------------------------------------------- noise ----

// kind: 0 independent-xz, 1 depolarizing.
int ref_sample_error(int kind, double p, std::uint64_t seed, std::uint64_t n,
                     std::uint64_t trial, std::uint64_t* e_x,
                     std::uint64_t* e_z) {
  return guarded([&] {
    const NoiseModel model{
        kind == 0 ? NoiseKind::kIndependentXZ : NoiseKind::kDepolarizing, p,
        seed};
    const PauliError err = sample_error(model, n, trial);
    words_from_vec(err.x, e_x);
    words_from_vec(err.z, e_z);
  });
}

int ref_extract_syndromes(const void* code, const std::uint64_t* e_x,
                          const std::uint64_t* e_z, std::uint64_t* s_x,
                          std::uint64_t* s_z) {
  return guarded([&] {
    const auto* c = static_cast<const CssCode*>(code);
    const SyndromePair s =
        extract_syndromes(*c, vec_from_words(e_x, c->num_qubits()),
                          vec_from_words(e_z, c->num_qubits()));
    words_from_vec(s.s_x, s_x);
    words_from_vec(s.s_z, s_z);
  });
}

// The bench pool recipe of run_bench (sample_error trial i -> combined
// syndrome s_x ++ s_z), `count` entries of ceil((mz+mx)/64) words each.
int ref_syndrome_pool(const void* code, double p, std::uint64_t seed,
                      std::uint64_t first_trial, std::uint64_t count,
                      std::uint64_t* out_words, std::uint64_t* ex_words,
                      std::uint64_t* ez_words) {
  return guarded([&] {
    const auto* c = static_cast<const CssCode*>(code);
    const std::size_t n = c->num_qubits();
    const std::size_t m = c->hx().rows() + c->hz().rows();
    const std::size_t sw = (m + 63) / 64;
    const std::size_t nw = (n + 63) / 64;
    const NoiseModel model{NoiseKind::kIndependentXZ, p, seed};
    for (std::uint64_t i = 0; i < count; ++i) {
      const PauliError err = sample_error(model, n, first_trial + i);
      const SyndromePair syn = extract_syndromes(*c, err.x, err.z);
      words_from_vec(syn.s_x.concat(syn.s_z), out_words + i * sw);
      if (ex_words) words_from_vec(err.x, ex_words + i * nw);
      if (ez_words) words_from_vec(err.z, ez_words + i * nw);
    }
  });
}

// Classification of (e, e_hat) pairs: returns the Classification enum value.
int ref_classify(const void* code, const std::uint64_t* e_x,
                 const std::uint64_t* ex_hat, const std::uint64_t* e_z,
                 const std::uint64_t* ez_hat, int* out) {
  return guarded([&] {
    const auto* c = static_cast<const CssCode*>(code);
    const std::size_t n = c->num_qubits();
    *out = static_cast<int>(classify_residual(
        *c, vec_from_words(e_x, n), vec_from_words(ex_hat, n),
        vec_from_words(e_z, n), vec_from_words(ez_hat, n)));
  });
}

// counts[0..5] = exact, stabilizer, logical_x, logical_z, logical_both,
// non_converged; rates[0..3] = LER, baseline LER, convergence rate, mean its.
int ref_run_campaign(const void* code, int kind, double p, std::uint64_t seed,
                     std::uint64_t trials, std::uint64_t max_iter, double alpha,
                     int early, int arith, double quant_scale,
                     const double* priors, std::uint64_t n_priors,
                     unsigned workers, std::uint64_t* counts, double* rates) {
  return guarded([&] {
    const auto* c = static_cast<const CssCode*>(code);
    const NoiseModel model{
        kind == 0 ? NoiseKind::kIndependentXZ : NoiseKind::kDepolarizing, p,
        seed};
    const CampaignResult r = run_campaign(
        *c, model, trials,
        make_cfg(max_iter, alpha, early, arith, quant_scale, priors, n_priors),
        workers);
    counts[0] = r.exact;
    counts[1] = r.stabilizer;
    counts[2] = r.logical_x;
    counts[3] = r.logical_z;
    counts[4] = r.logical_both;
    counts[5] = r.non_converged;
    rates[0] = r.logical_error_rate;
    rates[1] = r.baseline_logical_rate;
    rates[2] = r.convergence_rate;
    rates[3] = r.mean_iterations;
  });
}

// ---------------------------------------------------------------- bench ----

// stats[0..7] = min, mean, median, p99, max (us per decode), conv_rate,
// kernel_frac, threads;  meta[0..2] = digest, min_iters, max_iters.
int ref_run_bench(const void* code, int arith, double alpha,
                  std::uint64_t max_iter, int early, std::uint64_t batch,
                  unsigned threads, std::uint64_t warmup,
                  std::uint64_t measure, double p, std::uint64_t seed,
                  double* stats, std::uint64_t* meta) {
  return guarded([&] {
    BenchConfig cfg;
    cfg.mode = arith == 0   ? Arithmetic::kFloat
               : arith == 1 ? Arithmetic::kInt8
                            : Arithmetic::kInt16;
    cfg.alpha = alpha;
    cfg.max_iterations = max_iter;
    cfg.early_termination = early != 0;
    cfg.batch = batch;
    cfg.threads = threads;
    cfg.warmup_batches = warmup;
    cfg.measure_batches = measure;
    cfg.p = p;
    cfg.seed = seed;
    const BenchResult r = run_bench(*static_cast<const CssCode*>(code), cfg);
    stats[0] = r.record.min_us;
    stats[1] = r.record.mean_us;
    stats[2] = r.record.median_us;
    stats[3] = r.record.p99_us;
    stats[4] = r.record.max_us;
    stats[5] = r.record.conv_rate;
    stats[6] = r.record.kernel_frac;
    stats[7] = r.record.threads;
    meta[0] = r.output_digest;
    meta[1] = r.min_iterations_used;
    meta[2] = r.max_iterations_used;
  });
}

// Validating reader of the reference (read_bench_csv_file): returns the row count.
int ref_read_bench_csv_file(const char* path, std::uint64_t* rows, double* first_p99) {
  return guarded([&] {
    const std::vector<BenchRecord> recs = read_bench_csv_file(path);
    *rows = recs.size();
    if (first_p99 && !recs.empty()) *first_p99 = recs[0].p99_us;
  });
}

// load_alist on a text; returns the matrix as COO (row, col) pairs.
int ref_load_alist(const char* text, std::uint64_t* rows, std::uint64_t* cols,
                   std::uint32_t* rc, std::uint64_t cap, std::uint64_t* nnz) {
  return guarded([&] {
    const SparseGf2Matrix h = load_alist(std::string(text));
    *rows = h.rows();
    *cols = h.cols();
    *nnz = h.nnz();
    if (h.nnz() > cap) throw std::runtime_error("ref_load_alist: buffer too small");
    std::size_t k = 0;
    for (std::size_t r = 0; r < h.rows(); ++r) {
      for (std::uint32_t c : h.row_support(r)) {
        rc[k++] = static_cast<std::uint32_t>(r);
        rc[k++] = c;
      }
    }
  });
}

// CSS-JSON descriptors (proj/src/css_json.cpp), when the build found json.hpp.
// ref_css_json_load: text -> CssCode handle (ref_code_free).  ref_css_json_save: the
// self-contained descriptor (inline alist payloads) of a code into buf; returns the length
// needed (call again with a larger buffer if it exceeds len).
int ref_have_css_json() {
#ifdef REF_HAVE_CSS_JSON
  return 1;
#else
  return 0;
#endif
}

int ref_css_json_load(const char* text, const char* base_dir, void** out) {
#ifdef REF_HAVE_CSS_JSON
  return guarded([&] { *out = new CssCode(load_css_json(text, base_dir ? base_dir : "")); });
#else
  (void)text; (void)base_dir; (void)out;
  g_error = "css_json not built";
  return 2;
#endif
}

int ref_css_json_save(const void* code, char* buf, std::uint64_t len, std::uint64_t* needed) {
#ifdef REF_HAVE_CSS_JSON
  return guarded([&] {
    const std::string s = save_css_json(*static_cast<const CssCode*>(code));
    *needed = s.size() + 1;
    if (buf && len >= s.size() + 1) std::memcpy(buf, s.c_str(), s.size() + 1);
  });
#else
  (void)code; (void)buf; (void)len; (void)needed;
  g_error = "css_json not built";
  return 2;
#endif
}

int ref_host_descriptor(char* buf, std::uint64_t len) {
  return guarded([&] {
    const std::string s = host_descriptor();
    std::strncpy(buf, s.c_str(), len - 1);
    buf[len - 1] = 0;
  });
}

double ref_percentile_nearest_rank(const double* sorted, std::uint64_t n,
                                   double pct) {
  return percentile_nearest_rank(std::span<const double>(sorted, n), pct);
}

}  // extern "C"

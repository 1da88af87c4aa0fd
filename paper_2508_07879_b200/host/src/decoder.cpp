// Host mirror implementation: validation of lengths (the reference does these in
// the facade, proj/src/decoder.cpp:551-591, :604-617), packing, and the C-ABI calls.
#include "qldpc_b200/decoder.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <stdexcept>

#include "qldpc_b200.h"

namespace qldpc_b200 {

namespace {

[[noreturn]] void raise(qb_status st, const qb_decoder* h) {
  const std::string msg = qb_last_error(h);
  if (st == QB_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

void assign_bits(Gf2Vector& dst, std::size_t len, const std::uint64_t* words) {
  if (dst.size() != len) dst = Gf2Vector(len);
  auto w = dst.words();
  std::copy(words, words + w.size(), w.begin());
}

int arith_code(Arithmetic a) {
  switch (a) {
    case Arithmetic::kFloat: return QB_ARITH_FLOAT;
    case Arithmetic::kInt8: return QB_ARITH_INT8;
    case Arithmetic::kInt16: return QB_ARITH_INT16;
    case Arithmetic::kHalf: return QB_ARITH_HALF;
  }
  throw std::invalid_argument("DecoderConfig: unknown arithmetic mode");
}

}  // namespace

Gf2Vector Gf2Vector::from_bits(std::span<const int> bits) {
  Gf2Vector v(bits.size());
  for (std::size_t i = 0; i < bits.size(); ++i) {
    if (bits[i] != 0 && bits[i] != 1) throw std::invalid_argument("Gf2Vector: bits must be 0 or 1");
    v.set(i, bits[i] != 0);
  }
  return v;
}
Gf2Vector Gf2Vector::from_bits(std::initializer_list<int> bits) {
  return from_bits(std::span<const int>(bits.begin(), bits.size()));
}
bool Gf2Vector::is_zero() const {
  return std::all_of(words_.begin(), words_.end(), [](std::uint64_t w) { return w == 0; });
}
std::size_t Gf2Vector::weight() const {
  std::size_t n = 0;
  for (std::uint64_t w : words_) n += static_cast<std::size_t>(std::popcount(w));
  return n;
}
Gf2Vector Gf2Vector::slice(std::size_t begin, std::size_t end) const {
  if (begin > end || end > len_) throw std::invalid_argument("Gf2Vector::slice: bad range");
  Gf2Vector v(end - begin);
  for (std::size_t i = begin; i < end; ++i) v.set(i - begin, get(i));
  return v;
}
Gf2Vector Gf2Vector::concat(const Gf2Vector& other) const {
  Gf2Vector v(len_ + other.len_);
  for (std::size_t i = 0; i < len_; ++i) v.set(i, get(i));
  for (std::size_t i = 0; i < other.len_; ++i) v.set(len_ + i, other.get(i));
  return v;
}

TannerGraph build_tanner_graph(std::size_t rows, std::size_t cols,
                               const std::vector<std::vector<std::uint32_t>>& row_support) {
  if (rows == 0 || cols == 0 || row_support.size() != rows) {
    throw std::invalid_argument("build_tanner_graph: matrix must have rows and columns");
  }
  TannerGraph g;
  g.num_checks = rows;
  g.num_vars = cols;
  g.check_offsets.push_back(0);
  for (std::size_t m = 0; m < rows; ++m) {
    std::vector<std::uint32_t> sup = row_support[m];
    std::sort(sup.begin(), sup.end());
    if (std::adjacent_find(sup.begin(), sup.end()) != sup.end()) {
      throw std::invalid_argument("build_tanner_graph: duplicate entry in a row");
    }
    for (std::uint32_t n : sup) {
      if (n >= cols) throw std::invalid_argument("build_tanner_graph: column out of range");
      g.edge_var.push_back(n);
      g.edge_check.push_back(static_cast<std::uint32_t>(m));
    }
    g.check_offsets.push_back(static_cast<std::uint32_t>(g.edge_var.size()));
  }
  if (g.edge_var.empty()) throw std::invalid_argument("build_tanner_graph: no nonzero entry");
  std::vector<std::uint32_t> deg(cols, 0);
  for (std::uint32_t n : g.edge_var) ++deg[n];
  g.var_offsets.assign(cols + 1, 0);
  for (std::size_t n = 0; n < cols; ++n) g.var_offsets[n + 1] = g.var_offsets[n] + deg[n];
  g.var_edges.resize(g.edge_var.size());
  std::vector<std::uint32_t> cursor(g.var_offsets.begin(), g.var_offsets.end() - 1);
  for (std::uint32_t e = 0; e < g.edge_var.size(); ++e) g.var_edges[cursor[g.edge_var[e]]++] = e;
  return g;
}

std::string_view arithmetic_name(Arithmetic mode) {
  switch (mode) {
    case Arithmetic::kFloat: return "float";
    case Arithmetic::kInt8: return "int8";
    case Arithmetic::kInt16: return "int16";
    case Arithmetic::kHalf: return "half";
  }
  return "unknown";
}

Arithmetic parse_arithmetic(std::string_view name) {
  if (name == "float") return Arithmetic::kFloat;
  if (name == "int8") return Arithmetic::kInt8;
  if (name == "int16") return Arithmetic::kInt16;
  if (name == "half") return Arithmetic::kHalf;
  throw std::invalid_argument("unknown arithmetic mode '" + std::string(name) +
                              "' (expected float, int8, int16 or half)");
}

struct Decoder::Impl {
  DecoderConfig cfg;
  qb_decoder* h = nullptr;
  std::size_t m = 0, n = 0;
  std::vector<Segment> segs;
  bool css = false;
  std::vector<std::uint64_t> est, res;
  std::vector<std::uint8_t> conv;
  std::vector<std::uint32_t> its;

  ~Impl() { qb_decoder_destroy(h); }

  // reliabilities -> the C-ABI's soft format (float, or quantize_saturate as
  // proj/src/decoder.cpp:500-509 with 0 stored as +-1)
  std::vector<unsigned char> pack_soft(std::span<const double> rel) const {
    for (double v : rel) {
      if (!std::isfinite(v)) throw std::invalid_argument("decode_soft: a reliability is not finite");
    }
    std::vector<unsigned char> out;
    if (cfg.arithmetic == Arithmetic::kFloat || cfg.arithmetic == Arithmetic::kHalf) {
      out.resize(rel.size() * sizeof(float));
      float* f = reinterpret_cast<float*>(out.data());
      for (std::size_t i = 0; i < rel.size(); ++i) f[i] = static_cast<float>(rel[i]);
      return out;
    }
    const bool i8 = cfg.arithmetic == Arithmetic::kInt8;
    const long long kmax = i8 ? 127 : 32767;
    const double scale = cfg.quant_scale != 0.0 ? cfg.quant_scale : (i8 ? 8.0 : 256.0);
    out.resize(rel.size() * (i8 ? 1 : 2));
    for (std::size_t i = 0; i < rel.size(); ++i) {
      const double scaled = rel[i] * scale;
      long long q = std::abs(scaled) >= 1e18 ? (scaled < 0 ? -kmax : kmax) : std::llround(scaled);
      q = std::clamp(q, -kmax, kmax);
      if (q == 0) q = std::signbit(scaled) ? -1 : 1;
      if (i8) reinterpret_cast<std::int8_t*>(out.data())[i] = static_cast<std::int8_t>(q);
      else reinterpret_cast<std::int16_t*>(out.data())[i] = static_cast<std::int16_t>(q);
    }
    return out;
  }

  void run(const Gf2Vector& syndrome) {
    const qb_status st = qb_decode(h, syndrome.words().data(), est.data(), res.data(), conv.data(),
                                   its.data());
    if (st != QB_OK) raise(st, h);
  }
};

Decoder::Decoder(const TannerGraph& graph, DecoderConfig cfg, int device) {
  impl_ = std::make_unique<Impl>();
  Impl& I = *impl_;
  I.cfg = std::move(cfg);
  I.m = graph.num_checks;
  I.n = graph.num_vars;
  I.segs = {Segment{0, static_cast<std::uint32_t>(I.m), 0, static_cast<std::uint32_t>(I.n)}};
  qb_graph g{static_cast<std::uint32_t>(graph.num_checks), static_cast<std::uint32_t>(graph.num_vars),
             static_cast<std::uint32_t>(graph.num_edges()), graph.edge_var.data(),
             graph.check_offsets.data(), graph.var_offsets.data(), graph.var_edges.data()};
  qb_config c{I.cfg.max_iterations, I.cfg.alpha, I.cfg.early_termination ? 1 : 0,
              arith_code(I.cfg.arithmetic), I.cfg.quant_scale,
              I.cfg.priors.empty() ? nullptr : I.cfg.priors.data(), I.cfg.priors.size()};
  const qb_status st = qb_decoder_create(&g, nullptr, 0, &c, device, &I.h);
  if (st != QB_OK) raise(st, nullptr);
  I.est.resize((I.n + 63) / 64);
  I.res.resize((I.m + 63) / 64);
  I.conv.resize(1);
  I.its.resize(1);
}

Decoder::Decoder(const TannerGraph& graph, std::span<const Segment> segments, DecoderConfig cfg,
                 int device) {
  impl_ = std::make_unique<Impl>();
  Impl& I = *impl_;
  I.cfg = std::move(cfg);
  I.m = graph.num_checks;
  I.n = graph.num_vars;
  I.segs.assign(segments.begin(), segments.end());
  I.css = segments.size() == 2;
  std::vector<qb_segment> qs;
  for (const Segment& s : segments) qs.push_back({s.check_begin, s.check_end, s.var_begin, s.var_end});
  qb_graph g{static_cast<std::uint32_t>(graph.num_checks), static_cast<std::uint32_t>(graph.num_vars),
             static_cast<std::uint32_t>(graph.num_edges()), graph.edge_var.data(),
             graph.check_offsets.data(), graph.var_offsets.data(), graph.var_edges.data()};
  qb_config c{I.cfg.max_iterations, I.cfg.alpha, I.cfg.early_termination ? 1 : 0,
              arith_code(I.cfg.arithmetic), I.cfg.quant_scale,
              I.cfg.priors.empty() ? nullptr : I.cfg.priors.data(), I.cfg.priors.size()};
  const qb_status st = qb_decoder_create(&g, qs.data(), static_cast<std::uint32_t>(qs.size()), &c,
                                         device, &I.h);
  if (st != QB_OK) raise(st, nullptr);
  I.est.resize((I.n + 63) / 64);
  I.res.resize((I.m + 63) / 64);
  I.conv.resize(qs.size());
  I.its.resize(qs.size());
}

Decoder::~Decoder() = default;
Decoder::Decoder(Decoder&&) noexcept = default;
Decoder& Decoder::operator=(Decoder&&) noexcept = default;

const DecoderConfig& Decoder::config() const { return impl_->cfg; }
std::size_t Decoder::num_checks() const { return impl_->m; }
std::size_t Decoder::num_vars() const { return impl_->n; }
std::size_t Decoder::num_segments() const { return impl_->segs.size(); }
std::uint64_t Decoder::last_kernel_ns() const { return qb_last_kernel_ns(impl_->h); }
void* Decoder::native_handle() const { return impl_->h; }

void Decoder::set_latency_io(LatencyIo mode) {
  const qb_status st = qb_set_option(impl_->h, QB_OPT_LATENCY_IO, static_cast<int64_t>(mode));
  if (st != QB_OK) raise(st, impl_->h);
}

DecodeOutcome Decoder::decode(const Gf2Vector& syndrome) {
  DecodeOutcome out;
  decode_into(syndrome, out);
  return out;
}

void Decoder::decode_into(const Gf2Vector& syndrome, DecodeOutcome& out) {
  Impl& I = *impl_;
  if (syndrome.size() != I.m) {
    throw std::invalid_argument("decode: syndrome has " + std::to_string(syndrome.size()) +
                                " bits but the graph has " + std::to_string(I.m) + " checks");
  }
  I.run(syndrome);
  assign_bits(out.error_estimate, I.n, I.est.data());
  assign_bits(out.syndrome_residual, I.m, I.res.data());
  out.converged = std::all_of(I.conv.begin(), I.conv.end(), [](std::uint8_t c) { return c != 0; });
  out.iterations_used = *std::max_element(I.its.begin(), I.its.end());
}

void Decoder::decode_css_into(const Gf2Vector& s_x, const Gf2Vector& s_z, DecodeOutcome& out_x,
                              DecodeOutcome& out_z) {
  Impl& I = *impl_;
  if (!I.css) throw std::invalid_argument("decode_css_into: decoder was not built from a CssCode");
  const Segment &sx = I.segs[0], &sz = I.segs[1];
  const std::size_t xc = sx.check_end - sx.check_begin, zc = sz.check_end - sz.check_begin;
  if (s_x.size() != xc || s_z.size() != zc) {
    throw std::invalid_argument("decode_css_into: syndrome lengths (" + std::to_string(s_x.size()) +
                                ", " + std::to_string(s_z.size()) +
                                ") do not match the code's check counts (" + std::to_string(xc) +
                                ", " + std::to_string(zc) + ")");
  }
  I.run(s_x.concat(s_z));
  Gf2Vector est, res;
  assign_bits(est, I.n, I.est.data());
  assign_bits(res, I.m, I.res.data());
  out_x.error_estimate = est.slice(sx.var_begin, sx.var_end);
  out_x.syndrome_residual = res.slice(sx.check_begin, sx.check_end);
  out_x.converged = I.conv[0] != 0;
  out_x.iterations_used = I.its[0];
  out_z.error_estimate = est.slice(sz.var_begin, sz.var_end);
  out_z.syndrome_residual = res.slice(sz.check_begin, sz.check_end);
  out_z.converged = I.conv[1] != 0;
  out_z.iterations_used = I.its[1];
}

std::vector<DecodeOutcome> Decoder::decode_batch(std::span<const Gf2Vector> syndromes) {
  Impl& I = *impl_;
  for (std::size_t i = 0; i < syndromes.size(); ++i) {
    if (syndromes[i].size() != I.m) {
      throw std::invalid_argument("decode_batch: syndrome " + std::to_string(i) + " has " +
                                  std::to_string(syndromes[i].size()) +
                                  " bits but the graph has " + std::to_string(I.m) + " checks");
    }
  }
  const std::size_t shots = syndromes.size(), sw = (I.m + 63) / 64, ew = (I.n + 63) / 64;
  const std::size_t ns = I.segs.size();
  std::vector<DecodeOutcome> out(shots);
  if (shots == 0) return out;
  std::vector<std::uint64_t> syn(shots * sw), est(shots * ew), res(shots * sw);
  std::vector<std::uint8_t> conv(shots * ns);
  std::vector<std::uint32_t> its(shots * ns);
  for (std::size_t i = 0; i < shots; ++i) {
    std::copy(syndromes[i].words().begin(), syndromes[i].words().end(), syn.begin() + i * sw);
  }
  const qb_status st = qb_decode_batch(I.h, shots, syn.data(), est.data(), res.data(), conv.data(),
                                       its.data());
  if (st != QB_OK) raise(st, I.h);
  for (std::size_t i = 0; i < shots; ++i) {
    assign_bits(out[i].error_estimate, I.n, est.data() + i * ew);
    assign_bits(out[i].syndrome_residual, I.m, res.data() + i * sw);
    out[i].converged = true;
    out[i].iterations_used = 0;
    for (std::size_t s = 0; s < ns; ++s) {
      out[i].converged = out[i].converged && conv[i * ns + s] != 0;
      out[i].iterations_used = std::max<std::size_t>(out[i].iterations_used, its[i * ns + s]);
    }
  }
  return out;
}

std::vector<std::uint32_t> Decoder::soft_vars() const {
  std::vector<std::uint32_t> v(impl_->m);
  const qb_status st = qb_soft_vars(impl_->h, v.data());
  if (st != QB_OK) raise(st, impl_->h);
  return v;
}

DecodeOutcome Decoder::decode_soft(const Gf2Vector& syndrome, std::span<const double> reliability) {
  Impl& I = *impl_;
  if (syndrome.size() != I.m || reliability.size() != I.m) {
    throw std::invalid_argument("decode_soft: syndrome has " + std::to_string(syndrome.size()) +
                                " bits and " + std::to_string(reliability.size()) +
                                " reliabilities but the graph has " + std::to_string(I.m) + " checks");
  }
  const std::vector<unsigned char> soft = I.pack_soft(reliability);
  const qb_status st = qb_decode_soft(I.h, syndrome.words().data(), soft.data(), I.est.data(),
                                      I.res.data(), I.conv.data(), I.its.data());
  if (st != QB_OK) raise(st, I.h);
  DecodeOutcome out;
  assign_bits(out.error_estimate, I.n, I.est.data());
  assign_bits(out.syndrome_residual, I.m, I.res.data());
  out.converged = std::all_of(I.conv.begin(), I.conv.end(), [](std::uint8_t c) { return c != 0; });
  out.iterations_used = *std::max_element(I.its.begin(), I.its.end());
  return out;
}

std::vector<DecodeOutcome> Decoder::decode_batch_soft(std::span<const Gf2Vector> syndromes,
                                                      std::span<const double> reliability) {
  Impl& I = *impl_;
  for (std::size_t i = 0; i < syndromes.size(); ++i) {
    if (syndromes[i].size() != I.m) {
      throw std::invalid_argument("decode_batch_soft: syndrome " + std::to_string(i) + " has " +
                                  std::to_string(syndromes[i].size()) +
                                  " bits but the graph has " + std::to_string(I.m) + " checks");
    }
  }
  if (reliability.size() != syndromes.size() * I.m) {
    throw std::invalid_argument("decode_batch_soft: expected " + std::to_string(syndromes.size() * I.m) +
                                " reliabilities, got " + std::to_string(reliability.size()));
  }
  const std::size_t shots = syndromes.size(), sw = (I.m + 63) / 64, ew = (I.n + 63) / 64;
  const std::size_t ns = I.segs.size();
  std::vector<DecodeOutcome> out(shots);
  if (shots == 0) return out;
  const std::vector<unsigned char> soft = I.pack_soft(reliability);
  std::vector<std::uint64_t> syn(shots * sw), est(shots * ew), res(shots * sw);
  std::vector<std::uint8_t> conv(shots * ns);
  std::vector<std::uint32_t> its(shots * ns);
  for (std::size_t i = 0; i < shots; ++i) {
    std::copy(syndromes[i].words().begin(), syndromes[i].words().end(), syn.begin() + i * sw);
  }
  const qb_status st = qb_decode_batch_soft(I.h, shots, syn.data(), soft.data(), est.data(), res.data(),
                                            conv.data(), its.data());
  if (st != QB_OK) raise(st, I.h);
  for (std::size_t i = 0; i < shots; ++i) {
    assign_bits(out[i].error_estimate, I.n, est.data() + i * ew);
    assign_bits(out[i].syndrome_residual, I.m, res.data() + i * sw);
    out[i].converged = true;
    out[i].iterations_used = 0;
    for (std::size_t s = 0; s < ns; ++s) {
      out[i].converged = out[i].converged && conv[i * ns + s] != 0;
      out[i].iterations_used = std::max<std::size_t>(out[i].iterations_used, its[i * ns + s]);
    }
  }
  return out;
}

DecodeOutcome decode(const TannerGraph& graph, const Gf2Vector& syndrome, const DecoderConfig& cfg) {
  Decoder decoder(graph, cfg);
  return decoder.decode(syndrome);
}

std::vector<DecodeOutcome> decode_batch(const TannerGraph& graph,
                                        std::span<const Gf2Vector> syndromes,
                                        const DecoderConfig& cfg, unsigned /*num_workers*/) {
  for (std::size_t i = 0; i < syndromes.size(); ++i) {
    if (syndromes[i].size() != graph.num_checks) {
      throw std::invalid_argument("decode_batch: syndrome " + std::to_string(i) + " has " +
                                  std::to_string(syndromes[i].size()) +
                                  " bits but the graph has " + std::to_string(graph.num_checks) +
                                  " checks");
    }
  }
  if (syndromes.empty()) return {};
  Decoder decoder(graph, cfg);
  return decoder.decode_batch(syndromes);
}

CssDecodeResult decode_css(const TannerGraph& combined_graph, std::span<const Segment> segments,
                           const Gf2Vector& s_x, const Gf2Vector& s_z, const DecoderConfig& cfg) {
  Decoder decoder(combined_graph, segments, cfg);
  CssDecodeResult r;
  decoder.decode_css_into(s_x, s_z, r.x, r.z);
  return r;
}

}  // namespace qldpc_b200

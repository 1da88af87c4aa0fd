// C++ parity runner for the host mirror (namespace qldpc_b200): the same checks
// the reference's doctest suites make of qldpc::Decoder, against the C oracle
// (oracle/libmsa_oracle.so - test infrastructure, linked here only).  One
// PASS/FAIL line per check; exit status 1 if any fails.  Style follows
// proj/tests/acceptance.cpp; checks follow proj/tests/test_decoder.cpp.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "qldpc_b200/decoder.hpp"

using namespace qldpc_b200;

extern "C" {
struct oracle_graph {
  uint32_t num_checks, num_vars, num_edges;
  const uint32_t *edge_var, *check_offsets, *var_offsets, *var_edges;
};
struct oracle_segment {
  uint32_t check_begin, check_end, var_begin, var_end;
};
struct oracle_config {
  uint64_t max_iterations;
  double alpha;
  int32_t early_termination, arithmetic;
  double quant_scale;
  const double* priors;
  uint64_t num_priors;
};
int oracle_decode(const oracle_graph*, const oracle_segment*, uint32_t, const oracle_config*,
                  const uint64_t*, uint64_t*, uint64_t*, uint8_t*, uint32_t*, float*, float*,
                  int32_t*, int32_t*);
}

namespace {

int g_failures = 0;
void report(const char* name, bool ok, const std::string& detail = "") {
  std::printf("%s %s%s%s\n", ok ? "PASS" : "FAIL", name, detail.empty() ? "" : " - ", detail.c_str());
  if (!ok) ++g_failures;
}

TannerGraph toy_graph() {
  return build_tanner_graph(3, 6, {{0, 2, 3, 5}, {0, 1, 3, 4}, {1, 2, 4, 5}});
}

// Bivariate bicycle code: combined graph diag(hz, hx) with hx=[A|B], hz=[B^T|A^T].
struct Css {
  TannerGraph graph_x, combined;
  std::vector<Segment> segs;
  std::size_t n, mz, mx;
};
Css bb_code(std::size_t l, std::size_t m, std::vector<std::pair<int, int>> a,
            std::vector<std::pair<int, int>> b) {
  const std::size_t lm = l * m, n = 2 * lm;
  auto mono = [&](const std::vector<std::pair<int, int>>& t) {
    std::vector<std::vector<uint32_t>> rows(lm);
    for (std::size_t u = 0; u < l; ++u)
      for (std::size_t v = 0; v < m; ++v)
        for (auto [i, j] : t) rows[u * m + v].push_back(((u + i) % l) * m + (v + j) % m);
    return rows;
  };
  auto transpose = [&](const std::vector<std::vector<uint32_t>>& r) {
    std::vector<std::vector<uint32_t>> t(lm);
    for (std::size_t i = 0; i < lm; ++i) for (uint32_t c : r[i]) t[c].push_back(i);
    return t;
  };
  auto A = mono(a), B = mono(b), At = transpose(A), Bt = transpose(B);
  std::vector<std::vector<uint32_t>> hx(lm), hz(lm);
  for (std::size_t r = 0; r < lm; ++r) {
    hx[r] = A[r];
    for (uint32_t c : B[r]) hx[r].push_back(c + lm);
    hz[r] = Bt[r];
    for (uint32_t c : At[r]) hz[r].push_back(c + lm);
  }
  Css c;
  c.n = n;
  c.mz = c.mx = lm;
  c.graph_x = build_tanner_graph(lm, n, hz);
  std::vector<std::vector<uint32_t>> comb = hz;
  for (auto row : hx) {
    for (auto& v : row) v += n;
    comb.push_back(row);
  }
  c.combined = build_tanner_graph(2 * lm, 2 * n, comb);
  c.segs = {{0, (uint32_t)lm, 0, (uint32_t)n}, {(uint32_t)lm, (uint32_t)(2 * lm), (uint32_t)n, (uint32_t)(2 * n)}};
  return c;
}

Gf2Vector random_syndrome(std::mt19937& gen, std::size_t len, double density) {
  std::bernoulli_distribution bit(density);
  Gf2Vector s(len);
  for (std::size_t i = 0; i < len; ++i) s.set(i, bit(gen));
  return s;
}

bool same_outcome(const DecodeOutcome& a, const DecodeOutcome& b) {
  return a.error_estimate == b.error_estimate && a.converged == b.converged &&
         a.iterations_used == b.iterations_used && a.syndrome_residual == b.syndrome_residual;
}

DecodeOutcome oracle(const TannerGraph& g, const std::vector<Segment>& segs, const DecoderConfig& cfg,
                     const Gf2Vector& s) {
  oracle_graph og{(uint32_t)g.num_checks, (uint32_t)g.num_vars, (uint32_t)g.num_edges(),
                  g.edge_var.data(), g.check_offsets.data(), g.var_offsets.data(), g.var_edges.data()};
  std::vector<oracle_segment> os;
  for (auto& x : segs) os.push_back({x.check_begin, x.check_end, x.var_begin, x.var_end});
  oracle_config oc{cfg.max_iterations, cfg.alpha, cfg.early_termination ? 1 : 0,
                   cfg.arithmetic == Arithmetic::kFloat ? 0 : cfg.arithmetic == Arithmetic::kInt8 ? 1 : 2,
                   cfg.quant_scale, cfg.priors.empty() ? nullptr : cfg.priors.data(), cfg.priors.size()};
  DecodeOutcome out;
  out.error_estimate = Gf2Vector(g.num_vars);
  out.syndrome_residual = Gf2Vector(g.num_checks);
  std::vector<uint8_t> conv(os.size());
  std::vector<uint32_t> its(os.size());
  if (oracle_decode(&og, os.data(), (uint32_t)os.size(), &oc, s.words().data(),
                    out.error_estimate.words().data(), out.syndrome_residual.words().data(),
                    conv.data(), its.data(), nullptr, nullptr, nullptr, nullptr) != 0) {
    throw std::invalid_argument("oracle rejected the configuration");
  }
  out.converged = true;
  for (std::size_t i = 0; i < os.size(); ++i) {
    out.converged = out.converged && conv[i];
    out.iterations_used = std::max<std::size_t>(out.iterations_used, its[i]);
  }
  return out;
}

template <class F>
bool throws_invalid(F&& f) {
  try {
    f();
  } catch (const std::invalid_argument&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

}  // namespace

int main() {
  const std::vector<Segment> whole_toy = {{0, 3, 0, 6}};
  // 1. toy code, every syndrome, all modes (test_decoder.cpp:269-294, :417-424)
  {
    TannerGraph g = toy_graph();
    bool ok = true;
    for (Arithmetic mode : {Arithmetic::kFloat, Arithmetic::kInt8, Arithmetic::kInt16}) {
      DecoderConfig cfg;
      cfg.arithmetic = mode;
      Decoder dec(g, cfg);
      for (int mask = 0; mask < 8; ++mask) {
        Gf2Vector s(3);
        for (int m = 0; m < 3; ++m) s.set(m, (mask >> m) & 1);
        DecodeOutcome out = dec.decode(s);
        ok = ok && same_outcome(out, oracle(g, whole_toy, cfg, s));
        if (mode == Arithmetic::kFloat) {
          ok = ok && out.converged == s.is_zero() && out.iterations_used == (s.is_zero() ? 1u : 10u);
        }
      }
    }
    report("toy code: every syndrome, float/int8/int16, equals the oracle", ok);
  }
  // 2. validation (test_decoder.cpp:296-326, test_quantized.cpp:185-204)
  {
    TannerGraph g = toy_graph();
    DecoderConfig c;
    bool ok = true;
    c.alpha = 0.0; ok = ok && throws_invalid([&] { Decoder d(g, c); });
    c.alpha = 1.25; ok = ok && throws_invalid([&] { Decoder d(g, c); });
    c = DecoderConfig{}; c.max_iterations = 0; ok = ok && throws_invalid([&] { Decoder d(g, c); });
    c = DecoderConfig{}; c.priors = {1.0, 2.0}; ok = ok && throws_invalid([&] { Decoder d(g, c); });
    c = DecoderConfig{}; c.arithmetic = Arithmetic::kInt8; c.quant_scale = 0.3;
    ok = ok && throws_invalid([&] { Decoder d(g, c); });
    c = DecoderConfig{}; c.arithmetic = Arithmetic::kInt16; c.alpha = 1e-6;
    ok = ok && throws_invalid([&] { Decoder d(g, c); });
    Decoder dec(g, DecoderConfig{});
    ok = ok && throws_invalid([&] { dec.decode(Gf2Vector(5)); });
    DecodeOutcome a, b;
    ok = ok && throws_invalid([&] { dec.decode_css_into(Gf2Vector(1), Gf2Vector(2), a, b); });
    ok = ok && throws_invalid([&] { parse_arithmetic("int32"); });
    report("configuration and length validation throws std::invalid_argument", ok);
  }
  Css bb72 = bb_code(6, 6, {{3, 0}, {0, 1}, {0, 2}}, {{0, 3}, {1, 0}, {2, 0}});
  Css bb784 = bb_code(28, 14, {{26, 0}, {0, 6}, {0, 8}}, {{0, 7}, {9, 0}, {20, 0}});
  // 3. bb72 X graph vs oracle, alternating early termination (test_decoder.cpp:426-434)
  {
    std::mt19937 gen(71);
    bool ok = true;
    const std::vector<Segment> seg = {{0, 36, 0, 72}};
    for (int trial = 0; trial < 25; ++trial) {
      DecoderConfig cfg;
      cfg.early_termination = trial % 2 == 0;
      Gf2Vector s = random_syndrome(gen, 36, 0.1);
      ok = ok && same_outcome(decode(bb72.graph_x, s, cfg), oracle(bb72.graph_x, seg, cfg, s));
    }
    report("bb72 X graph equals the oracle bit for bit", ok);
  }
  // 4. reuse + batch == sequential (test_decoder.cpp:328-377)
  {
    std::mt19937 gen(29);
    DecoderConfig cfg;
    std::vector<Gf2Vector> syn;
    for (int i = 0; i < 64; ++i) syn.push_back(random_syndrome(gen, 36, 0.08));
    auto batch = decode_batch(bb72.graph_x, syn, cfg, 8);
    Decoder dec(bb72.graph_x, cfg);
    bool ok = batch.size() == syn.size();
    for (std::size_t i = 0; ok && i < syn.size(); ++i) ok = same_outcome(batch[i], dec.decode(syn[i]));
    ok = ok && decode_batch(bb72.graph_x, {}, cfg, 4).empty();
    std::vector<Gf2Vector> bad = syn;
    bad[7] = Gf2Vector(5);
    ok = ok && throws_invalid([&] { decode_batch(bb72.graph_x, bad, cfg, 2); });
    report("batch equals the sequential map; bad lengths rejected up front", ok);
  }
  // 5. combined == separate (test_decoder.cpp:379-405) on bb72, and [[784,24,24]] vs oracle
  {
    std::mt19937 gen(59);
    bool ok = true;
    for (int trial = 0; trial < 40; ++trial) {
      DecoderConfig cfg;
      cfg.early_termination = trial % 2 == 0;
      Gf2Vector sx = random_syndrome(gen, 36, 0.06), sz = random_syndrome(gen, 36, 0.06);
      CssDecodeResult r = decode_css(bb72.combined, bb72.segs, sx, sz, cfg);
      ok = ok && same_outcome(r.x, decode(bb72.graph_x, sx, cfg));
    }
    for (Arithmetic mode : {Arithmetic::kFloat, Arithmetic::kInt8}) {
      DecoderConfig cfg;
      cfg.max_iterations = 30;
      cfg.arithmetic = mode;
      Decoder dec(bb784.combined, bb784.segs, cfg);
      for (LatencyIo io : {LatencyIo::kMapped, LatencyIo::kMemcpy, LatencyIo::kDoorbell}) {
        dec.set_latency_io(io);
        for (int trial = 0; trial < 12; ++trial) {
          Gf2Vector s = random_syndrome(gen, 784, 0.03);
          ok = ok && same_outcome(dec.decode(s), oracle(bb784.combined, bb784.segs, cfg, s));
        }
      }
    }
    report("combined decode equals separate decodes; [[784,24,24]] equals the oracle in every I/O mode", ok);
  }
  // 6. soft syndromes (extension): [H | I] extension of bb72, per-shot reliabilities; the
  //    oracle is one reference-style decoder per shot whose priors carry that shot's values
  //    as the library stores them (float(prior) / quantised prior / scale)
  {
    std::mt19937 gen(83);
    const std::size_t n = bb72.n, mz = bb72.mz, mx = bb72.mx;
    std::vector<std::vector<uint32_t>> rows;
    for (std::size_t r = 0; r < mz; ++r) {
      std::vector<uint32_t> row;
      for (uint32_t e = bb72.combined.check_offsets[r]; e < bb72.combined.check_offsets[r + 1]; ++e)
        row.push_back(bb72.combined.edge_var[e]);
      row.push_back((uint32_t)(n + r));
      rows.push_back(row);
    }
    for (std::size_t r = 0; r < mx; ++r) {
      std::vector<uint32_t> row;
      for (uint32_t e = bb72.combined.check_offsets[mz + r]; e < bb72.combined.check_offsets[mz + r + 1]; ++e)
        row.push_back(bb72.combined.edge_var[e] + (uint32_t)mz);  // second block sits after the first I
      row.push_back((uint32_t)(2 * n + mz + r));
      rows.push_back(row);
    }
    const std::size_t M = mz + mx, N = 2 * n + mz + mx;
    TannerGraph ext = build_tanner_graph(M, N, rows);
    const std::vector<Segment> segs = {{0, (uint32_t)mz, 0, (uint32_t)(n + mz)},
                                       {(uint32_t)mz, (uint32_t)M, (uint32_t)(n + mz), (uint32_t)N}};
    bool ok = true;
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (Arithmetic mode : {Arithmetic::kFloat, Arithmetic::kInt8, Arithmetic::kInt16}) {
      DecoderConfig cfg;
      cfg.max_iterations = 20;
      cfg.arithmetic = mode;
      cfg.priors.assign(N, 5.0);
      Decoder dec(ext, segs, cfg);
      const std::vector<uint32_t> sv = dec.soft_vars();
      for (std::size_t m = 0; m < M; ++m) ok = ok && sv[m] == (m < mz ? n + m : 2 * n + mz + (m - mz));
      std::vector<Gf2Vector> syn;
      std::vector<double> rel;
      for (int i = 0; i < 24; ++i) {
        syn.push_back(random_syndrome(gen, M, 0.05));
        for (std::size_t m = 0; m < M; ++m) rel.push_back(std::abs(1.0 + 0.45 * gauss(gen)) * 2.0 / (0.45 * 0.45));
      }
      std::vector<DecodeOutcome> batch = dec.decode_batch_soft(syn, rel);
      const double scale = mode == Arithmetic::kInt8 ? 8.0 : 256.0, kmax = mode == Arithmetic::kInt8 ? 127 : 32767;
      for (int i = 0; i < 24; ++i) {
        DecoderConfig shot = cfg;
        for (std::size_t m = 0; m < M; ++m) {
          const double v = rel[i * M + m];
          if (mode == Arithmetic::kFloat) {
            shot.priors[sv[m]] = static_cast<double>(static_cast<float>(v));
          } else {
            double q = std::min(kmax, std::max(-kmax, (double)std::llround(v * scale)));
            if (q == 0) q = 1;
            shot.priors[sv[m]] = q / scale;
          }
        }
        const DecodeOutcome want = oracle(ext, segs, shot, syn[i]);
        ok = ok && same_outcome(batch[i], want);
        for (LatencyIo io : {LatencyIo::kMapped, LatencyIo::kMemcpy, LatencyIo::kDoorbell}) {
          dec.set_latency_io(io);
          ok = ok && same_outcome(dec.decode_soft(syn[i], std::span<const double>(rel).subspan(i * M, M)), want);
        }
      }
      ok = ok && throws_invalid([&] { dec.decode_soft(syn[0], std::span<const double>(rel).subspan(0, 5)); });
      ok = ok && throws_invalid([&] { dec.decode_batch_soft(syn, std::span<const double>(rel).subspan(0, M)); });
    }
    Decoder plain(bb72.combined, bb72.segs, DecoderConfig{});
    std::vector<double> ones(bb72.combined.num_checks, 1.0);
    ok = ok && throws_invalid([&] { plain.decode_soft(Gf2Vector(bb72.combined.num_checks), ones); });
    report("soft syndromes on [H | I]: batch and single-shot (3 I/O modes) equal one oracle decoder per shot", ok);
  }
  std::printf("%s\n", g_failures == 0 ? "ALL PASS" : "SOME FAILED");
  return g_failures == 0 ? 0 : 1;
}

// C++ host mirror of the reference's decoder interface over the C-ABI
// (include/qldpc_b200.h).  Same type and function names, argument meaning and
// error behaviour as proj/include/qldpc/decoder.hpp:16-129, in namespace
// qldpc_b200, so code written against the reference reads the same:
//
//   qldpc_b200::Decoder dec(graph, cfg);          // or (graph, segments, cfg) for a CSS code
//   qldpc_b200::DecodeOutcome out = dec.decode(syndrome);
//
// std::invalid_argument marks exactly the conditions the reference rejects;
// CUDA failures surface as std::runtime_error.  All arithmetic runs on the GPU.
#pragma once

#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <memory>
#include <span>
#include <string>
#include <string_view>
#include <vector>

namespace qldpc_b200 {

/// Dense bit-packed GF(2) vector in the reference's layout
/// (proj/include/qldpc/gf2.hpp:13-67): bit i at words()[i >> 6], bit i & 63.
class Gf2Vector {
 public:
  Gf2Vector() = default;
  explicit Gf2Vector(std::size_t len) : len_(len), words_((len + 63) / 64, 0) {}
  static Gf2Vector from_bits(std::initializer_list<int> bits);
  static Gf2Vector from_bits(std::span<const int> bits);

  std::size_t size() const { return len_; }
  bool get(std::size_t i) const { return (words_[i >> 6] >> (i & 63)) & 1u; }
  void set(std::size_t i, bool value) {
    const std::uint64_t mask = std::uint64_t{1} << (i & 63);
    if (value) words_[i >> 6] |= mask; else words_[i >> 6] &= ~mask;
  }
  bool is_zero() const;
  std::size_t weight() const;
  Gf2Vector slice(std::size_t begin, std::size_t end) const;
  Gf2Vector concat(const Gf2Vector& other) const;
  friend bool operator==(const Gf2Vector& a, const Gf2Vector& b) {
    return a.len_ == b.len_ && a.words_ == b.words_;
  }
  std::span<const std::uint64_t> words() const { return words_; }
  std::span<std::uint64_t> words() { return words_; }

 private:
  std::size_t len_ = 0;
  std::vector<std::uint64_t> words_;
};

/// Same fields as the reference's TannerGraph (proj/include/qldpc/tanner_graph.hpp:15-48).
struct TannerGraph {
  std::size_t num_checks = 0;
  std::size_t num_vars = 0;
  std::vector<std::uint32_t> edge_var, edge_check, check_offsets, var_offsets, var_edges;
  std::size_t num_edges() const { return edge_var.size(); }
};

/// One edge per listed entry, row-major edge order (proj/src/tanner_graph.cpp:7-41).
TannerGraph build_tanner_graph(std::size_t rows, std::size_t cols,
                               const std::vector<std::vector<std::uint32_t>>& row_support);

/// An independent block of a graph (proj/src/decoder.cpp:25-30).
struct Segment {
  std::uint32_t check_begin = 0, check_end = 0, var_begin = 0, var_end = 0;
};

enum class Arithmetic { kFloat, kInt8, kInt16, kHalf /* extension: fp16 messages */ };
std::string_view arithmetic_name(Arithmetic mode);
Arithmetic parse_arithmetic(std::string_view name);

struct DecoderConfig {  // proj/include/qldpc/decoder.hpp:23-38
  std::size_t max_iterations = 10;
  double alpha = 0.8;
  bool early_termination = true;
  std::vector<double> priors;
  Arithmetic arithmetic = Arithmetic::kFloat;
  double quant_scale = 0.0;
};

struct DecodeOutcome {  // proj/include/qldpc/decoder.hpp:40-46
  Gf2Vector error_estimate;
  bool converged = false;
  std::size_t iterations_used = 0;
  Gf2Vector syndrome_residual;
};

/// Single-shot I/O policy (QB_OPT_LATENCY_IO).
enum class LatencyIo { kMapped = 0, kMemcpy = 1, kDoorbell = 2 };

class Decoder {  // proj/include/qldpc/decoder.hpp:77-108
 public:
  Decoder(const TannerGraph& graph, DecoderConfig cfg, int device = 0);
  /// Two-component decoder over a block-diagonal graph (the reference's
  /// Decoder(const CssCode&, cfg): segments X = checks of hz, Z = checks of hx).
  Decoder(const TannerGraph& combined_graph, std::span<const Segment> segments, DecoderConfig cfg,
          int device = 0);
  ~Decoder();
  Decoder(Decoder&&) noexcept;
  Decoder& operator=(Decoder&&) noexcept;

  const DecoderConfig& config() const;
  std::size_t num_checks() const;
  std::size_t num_vars() const;
  std::size_t num_segments() const;

  DecodeOutcome decode(const Gf2Vector& syndrome);
  void decode_into(const Gf2Vector& syndrome, DecodeOutcome& out);
  void decode_css_into(const Gf2Vector& s_x, const Gf2Vector& s_z, DecodeOutcome& out_x,
                       DecodeOutcome& out_z);
  /// Batch of syndromes through the persistent batch kernel (H2D, decode, D2H).
  std::vector<DecodeOutcome> decode_batch(std::span<const Gf2Vector> syndromes);
  std::uint64_t last_kernel_ns() const;

  /// Soft (noisy) syndromes on a graph [H | I] (extension; include/qldpc_b200.h, "soft
  /// syndromes"): reliability[m] is this shot's prior (LLR) of the degree-1 measurement-error
  /// variable soft_vars()[m] of check m; entries of checks without one are ignored.  Equal to a
  /// reference Decoder built for the shot with priors[soft_vars()[m]] = the value as stored
  /// (float(prior), or the quantised prior / quant_scale in the integer modes; a value that
  /// would quantise to 0 is stored as +-1, which the reference would reject).
  std::vector<std::uint32_t> soft_vars() const;  // 0xffffffff where a check has none
  DecodeOutcome decode_soft(const Gf2Vector& syndrome, std::span<const double> reliability);
  /// reliability = [syndromes.size()][num_checks()], row-major.
  std::vector<DecodeOutcome> decode_batch_soft(std::span<const Gf2Vector> syndromes,
                                               std::span<const double> reliability);

  void set_latency_io(LatencyIo mode);
  void* native_handle() const;  // qb_decoder*

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

DecodeOutcome decode(const TannerGraph& graph, const Gf2Vector& syndrome, const DecoderConfig& cfg);

/// Elementwise identical to sequential decode calls; num_workers names CPU
/// threads in the reference and is accepted and ignored here (one launch).
std::vector<DecodeOutcome> decode_batch(const TannerGraph& graph,
                                        std::span<const Gf2Vector> syndromes,
                                        const DecoderConfig& cfg, unsigned num_workers = 1);

struct CssDecodeResult {
  DecodeOutcome x, z;
};
CssDecodeResult decode_css(const TannerGraph& combined_graph, std::span<const Segment> segments,
                           const Gf2Vector& s_x, const Gf2Vector& s_z, const DecoderConfig& cfg);

}  // namespace qldpc_b200

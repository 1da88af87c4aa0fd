/* TEST INFRASTRUCTURE — the CPU oracle.  Not part of the product: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this; nothing under paper_2508_07879_b200/ does.
 *
 * Plain-C restatement of the reference's scaled min-sum flooding decoder
 * (reference: proj/src/decoder.cpp).  Unlike the reference it EXPOSES the edge
 * messages q (variable->check) and r (check->variable) so the GPU kernels can
 * be compared per edge.  Parity of this file is pinned in
 * tests/test_oracle.py against (a) the reference's own known-answer vectors
 * and (b) the compiled reference (oracle/_ref/libqldpc_ref.so) on identical
 * graphs, priors and syndromes, bit for bit.
 *
 * Layout conventions are the reference's:
 *   - edges are numbered check-major; check m owns [check_off[m], check_off[m+1])
 *   - var_edges lists each variable's edge ids in ascending order
 *   - bit i of a packed vector is (words[i >> 6] >> (i & 63)) & 1
 *     (proj/include/qldpc/gf2.hpp:26)
 *
 * Arithmetic modes (proj/src/decoder.cpp:38-61):
 *   0 = float   fp32 storage, fp64 arithmetic, one rounding per stored message
 *   1 = int8    int8 storage, int32 arithmetic, Q16 alpha, saturate at 127
 *   2 = int16   int16 storage, int32 arithmetic, Q16 alpha, saturate at 32767
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_INVALID 1

#define DEG1_CHECK_MAG 64.0 /* decoder.cpp:18 */
#define FLOAT_CLAMP 1e30    /* decoder.cpp:23 */

typedef struct {
  uint32_t num_checks, num_vars, num_edges;
  const uint32_t *edge_var;      /* [E] */
  const uint32_t *check_offsets; /* [M+1] */
  const uint32_t *var_offsets;   /* [N+1] */
  const uint32_t *var_edges;     /* [E] */
} oracle_graph;

typedef struct {
  uint32_t check_begin, check_end, var_begin, var_end;
} oracle_segment;

typedef struct {
  uint64_t max_iterations;
  double alpha;
  int32_t early_termination;
  int32_t arithmetic;
  double quant_scale;   /* 0 = mode default (8 / 256) */
  const double *priors; /* NULL = uniform 1.0 */
  uint64_t num_priors;
} oracle_config;

static int get_bit(const uint64_t *w, uint64_t i) {
  return (int)((w[i >> 6] >> (i & 63)) & 1u);
}

static void put_bit(uint64_t *w, uint64_t i) { w[i >> 6] |= (uint64_t)1 << (i & 63); }

/* round(value*scale) clamped to [-limit, limit]; decoder.cpp:500-509.
 * Returns 0 and sets *err for NaN. */
int32_t oracle_quantize_saturate(double value, double scale, int32_t limit, int *err) {
  const double scaled = value * scale;
  *err = 0;
  if (isnan(scaled)) {
    *err = 1;
    return 0;
  }
  if (scaled >= (double)limit) return limit;
  if (scaled <= (double)(-limit)) return -limit;
  return (int32_t)llround(scaled);
}

/* Definitional node operations (decoder.cpp:455-498), used for the KATs. */
int oracle_check_node_update(const double *q, uint64_t deg, int s_bit, double alpha,
                             double *r) {
  if (deg == 0 || !(alpha > 0.0 && alpha <= 1.0) || (s_bit != 0 && s_bit != 1)) {
    return ORACLE_INVALID;
  }
  const double as = alpha * (s_bit ? -1.0 : 1.0);
  if (deg == 1) {
    r[0] = as * DEG1_CHECK_MAG;
    return ORACLE_OK;
  }
  for (uint64_t i = 0; i < deg; ++i) {
    double mn = INFINITY;
    int flip = 0;
    for (uint64_t j = 0; j < deg; ++j) {
      if (j == i) continue;
      flip ^= q[j] < 0.0;
      const double a = fabs(q[j]);
      if (a < mn) mn = a;
    }
    const double v = as * mn;
    r[i] = flip ? -v : v;
  }
  return ORACLE_OK;
}

void oracle_variable_node_update(double gamma, const double *r, uint64_t deg, double *q) {
  if (deg == 1) {
    q[0] = gamma;
    return;
  }
  double total = gamma;
  for (uint64_t i = 0; i < deg; ++i) total += r[i];
  for (uint64_t i = 0; i < deg; ++i) q[i] = total - r[i];
}

double oracle_posterior(double gamma, const double *r, uint64_t deg, int *bit) {
  double total = gamma;
  for (uint64_t i = 0; i < deg; ++i) total += r[i];
  *bit = total < 0.0;
  return total;
}

/* ---- the decoder ------------------------------------------------------- */

typedef struct {
  const oracle_graph *g;
  int arith;
  int32_t kmax;
  double alpha;
  uint32_t alpha_fx;
  /* float mode */
  float *qf, *rf, *gf;
  /* int modes: messages held widened in int32 but always within [-kmax,kmax] */
  int32_t *qi, *ri, *gi;
  uint8_t *sbit, *ehat, *resid;
} state;

static int32_t scale_q16(const state *st, int32_t mag) { /* decoder.cpp:226-229 */
  return (int32_t)(((int64_t)mag * st->alpha_fx + 32768) >> 16);
}

static void cn_float(state *st, uint32_t c0, uint32_t c1) { /* decoder.cpp:245-259,284-309 */
  const oracle_graph *g = st->g;
  for (uint32_t m = c0; m < c1; ++m) {
    const uint32_t b = g->check_offsets[m], e1 = g->check_offsets[m + 1];
    const double sg = st->sbit[m] ? -1.0 : 1.0;
    if (e1 - b == 1) {
      st->rf[b] = (float)(st->alpha * sg * DEG1_CHECK_MAG);
      continue;
    }
    double m1 = INFINITY, m2 = INFINITY;
    uint32_t arg = b;
    unsigned neg = 0;
    for (uint32_t e = b; e < e1; ++e) {
      const float v = st->qf[e];
      neg += v < 0.0f;
      const double a = fabs((double)v);
      if (a < m1) {
        m2 = m1;
        m1 = a;
        arg = e;
      } else if (a < m2) {
        m2 = a;
      }
    }
    const double as = st->alpha * sg;
    for (uint32_t e = b; e < e1; ++e) {
      const unsigned self = st->qf[e] < 0.0f;
      const int flip = ((neg - self) & 1u) != 0;
      const double v = as * (e == arg ? m2 : m1);
      st->rf[e] = (float)(flip ? -v : v);
    }
  }
}

static void cn_int(state *st, uint32_t c0, uint32_t c1) { /* decoder.cpp:251-255,260-283 */
  const oracle_graph *g = st->g;
  for (uint32_t m = c0; m < c1; ++m) {
    const uint32_t b = g->check_offsets[m], e1 = g->check_offsets[m + 1];
    const int sneg = st->sbit[m] != 0;
    if (e1 - b == 1) {
      const int32_t mag = scale_q16(st, st->kmax);
      st->ri[b] = sneg ? -mag : mag;
      continue;
    }
    int32_t m1 = INT32_MAX, m2 = INT32_MAX;
    uint32_t arg = b;
    unsigned neg = 0;
    for (uint32_t e = b; e < e1; ++e) {
      const int32_t v = st->qi[e];
      neg += v < 0;
      const int32_t a = v < 0 ? -v : v;
      if (a < m1) {
        m2 = m1;
        m1 = a;
        arg = e;
      } else if (a < m2) {
        m2 = a;
      }
    }
    for (uint32_t e = b; e < e1; ++e) {
      const unsigned self = st->qi[e] < 0;
      const int flip = ((neg - self) & 1u) != 0;
      const int32_t s = scale_q16(st, e == arg ? m2 : m1);
      st->ri[e] = (sneg != flip) ? -s : s;
    }
  }
}

static void vn_float(state *st, uint32_t v0, uint32_t v1) { /* decoder.cpp:313-335,231-243 */
  const oracle_graph *g = st->g;
  for (uint32_t n = v0; n < v1; ++n) {
    const uint32_t b = g->var_offsets[n], e1 = g->var_offsets[n + 1];
    double total = st->gf[n];
    for (uint32_t i = b; i < e1; ++i) total += (double)st->rf[g->var_edges[i]];
    st->ehat[n] = total < 0;
    if (e1 - b == 1) {
      st->qf[g->var_edges[b]] = st->gf[n];
      continue;
    }
    for (uint32_t i = b; i < e1; ++i) {
      const uint32_t e = g->var_edges[i];
      double x = total - (double)st->rf[e];
      if (x > FLOAT_CLAMP) x = FLOAT_CLAMP;
      if (x < -FLOAT_CLAMP) x = -FLOAT_CLAMP;
      st->qf[e] = (float)x;
    }
  }
}

static void vn_int(state *st, uint32_t v0, uint32_t v1) {
  const oracle_graph *g = st->g;
  for (uint32_t n = v0; n < v1; ++n) {
    const uint32_t b = g->var_offsets[n], e1 = g->var_offsets[n + 1];
    int32_t total = st->gi[n];
    for (uint32_t i = b; i < e1; ++i) total += st->ri[g->var_edges[i]];
    st->ehat[n] = total < 0;
    if (e1 - b == 1) {
      st->qi[g->var_edges[b]] = st->gi[n];
      continue;
    }
    for (uint32_t i = b; i < e1; ++i) {
      const uint32_t e = g->var_edges[i];
      int32_t x = total - st->ri[e];
      if (x > st->kmax) x = st->kmax;
      if (x < -st->kmax) x = -st->kmax;
      st->qi[e] = x;
    }
  }
}

static int check_segment(state *st, uint32_t c0, uint32_t c1) { /* decoder.cpp:337-350 */
  const oracle_graph *g = st->g;
  int ok = 1;
  for (uint32_t m = c0; m < c1; ++m) {
    uint8_t p = st->sbit[m];
    for (uint32_t e = g->check_offsets[m]; e < g->check_offsets[m + 1]; ++e) {
      p ^= st->ehat[g->edge_var[e]];
    }
    st->resid[m] = p;
    ok = ok && p == 0;
  }
  return ok;
}

/* Validates like decoder.cpp:373-387 and :83-131.  Returns ORACLE_INVALID for
 * anything the reference rejects with std::invalid_argument. */
int oracle_validate(const oracle_graph *g, const oracle_config *cfg) {
  if (cfg->max_iterations < 1) return ORACLE_INVALID;
  if (!(cfg->alpha > 0.0 && cfg->alpha <= 1.0)) return ORACLE_INVALID;
  if (cfg->priors && cfg->num_priors != 0 && cfg->num_priors != g->num_vars) {
    return ORACLE_INVALID;
  }
  if (cfg->arithmetic < 0 || cfg->arithmetic > 2) return ORACLE_INVALID;
  const int has_priors = cfg->priors && cfg->num_priors != 0;
  if (cfg->arithmetic != 0) {
    const double scale = cfg->quant_scale != 0.0 ? cfg->quant_scale
                                                 : (cfg->arithmetic == 1 ? 8.0 : 256.0);
    if (!(scale > 0.0) || !isfinite(scale)) return ORACLE_INVALID;
    if ((uint32_t)lround(cfg->alpha * 65536.0) == 0) return ORACLE_INVALID;
    const int32_t kmax = cfg->arithmetic == 1 ? 127 : 32767;
    uint64_t maxdeg = 0;
    for (uint32_t n = 0; n < g->num_vars; ++n) {
      const uint64_t d = g->var_offsets[n + 1] - g->var_offsets[n];
      if (d > maxdeg) maxdeg = d;
    }
    if (maxdeg + 1 > (uint64_t)(INT32_MAX / kmax)) return ORACLE_INVALID;
    for (uint32_t n = 0; n < g->num_vars; ++n) {
      const double p = has_priors ? cfg->priors[n] : 1.0;
      if (!isfinite(p)) return ORACLE_INVALID;
      int err;
      if (oracle_quantize_saturate(p, scale, kmax, &err) == 0) return ORACLE_INVALID;
    }
  } else {
    for (uint32_t n = 0; n < g->num_vars; ++n) {
      const double p = has_priors ? cfg->priors[n] : 1.0;
      if (!isfinite(p)) return ORACLE_INVALID;
    }
  }
  return ORACLE_OK;
}

/* Decodes one syndrome (num_checks bits, packed).
 *
 * Outputs (all caller-allocated):
 *   estimate  ceil(N/64) words, residual ceil(M/64) words (whole graph layout)
 *   converged[nseg], iterations[nseg]  per segment (decoder.cpp:194-202); the
 *     whole-graph outcome of decode_into is AND / MAX over them (:204-213)
 *   q_out / r_out: optional [E] final edge messages, as float (mode 0) or
 *     int32 (modes 1, 2) — pass the matching pointer, the other NULL.
 */
int oracle_decode(const oracle_graph *g, const oracle_segment *segs, uint32_t nseg,
                  const oracle_config *cfg, const uint64_t *syndrome, uint64_t *estimate,
                  uint64_t *residual, uint8_t *converged, uint32_t *iterations,
                  float *qf_out, float *rf_out, int32_t *qi_out, int32_t *ri_out) {
  if (oracle_validate(g, cfg) != ORACLE_OK) return ORACLE_INVALID;
  const uint32_t M = g->num_checks, N = g->num_vars, E = g->num_edges;
  const int has_priors = cfg->priors && cfg->num_priors != 0;
  state st;
  memset(&st, 0, sizeof st);
  st.g = g;
  st.arith = cfg->arithmetic;
  st.alpha = cfg->alpha;
  st.sbit = calloc(M, 1);
  st.ehat = calloc(N, 1);
  st.resid = calloc(M, 1);
  if (st.arith == 0) {
    st.qf = calloc(E, sizeof(float));
    st.rf = calloc(E, sizeof(float));
    st.gf = calloc(N, sizeof(float));
    for (uint32_t n = 0; n < N; ++n) st.gf[n] = (float)(has_priors ? cfg->priors[n] : 1.0);
  } else {
    st.kmax = st.arith == 1 ? 127 : 32767;
    const double scale =
        cfg->quant_scale != 0.0 ? cfg->quant_scale : (st.arith == 1 ? 8.0 : 256.0);
    st.alpha_fx = (uint32_t)lround(cfg->alpha * 65536.0);
    st.qi = calloc(E, sizeof(int32_t));
    st.ri = calloc(E, sizeof(int32_t));
    st.gi = calloc(N, sizeof(int32_t));
    for (uint32_t n = 0; n < N; ++n) {
      int err;
      st.gi[n] = oracle_quantize_saturate(has_priors ? cfg->priors[n] : 1.0, scale, st.kmax, &err);
    }
  }
  for (uint32_t m = 0; m < M; ++m) st.sbit[m] = (uint8_t)get_bit(syndrome, m);

  /* decoder.cpp:156-158 */
  for (uint32_t e = 0; e < E; ++e) {
    if (st.arith == 0) {
      st.qf[e] = st.gf[g->edge_var[e]];
    } else {
      st.qi[e] = st.gi[g->edge_var[e]];
    }
  }

  uint8_t *frozen = calloc(nseg, 1);
  for (uint32_t s = 0; s < nseg; ++s) {
    converged[s] = 0;
    iterations[s] = 0;
  }
  uint64_t iter = 0;
  uint32_t nfrozen = 0;
  while (iter < cfg->max_iterations && nfrozen < nseg) { /* decoder.cpp:162-181 */
    ++iter;
    for (uint32_t s = 0; s < nseg; ++s) {
      if (frozen[s]) continue;
      if (st.arith == 0) {
        cn_float(&st, segs[s].check_begin, segs[s].check_end);
        vn_float(&st, segs[s].var_begin, segs[s].var_end);
      } else {
        cn_int(&st, segs[s].check_begin, segs[s].check_end);
        vn_int(&st, segs[s].var_begin, segs[s].var_end);
      }
    }
    if (cfg->early_termination) {
      for (uint32_t s = 0; s < nseg; ++s) {
        if (frozen[s]) continue;
        if (check_segment(&st, segs[s].check_begin, segs[s].check_end)) {
          frozen[s] = 1;
          converged[s] = 1;
          iterations[s] = (uint32_t)iter;
          ++nfrozen;
        }
      }
    }
  }
  for (uint32_t s = 0; s < nseg; ++s) { /* decoder.cpp:182-187 */
    if (frozen[s]) continue;
    iterations[s] = (uint32_t)iter;
    converged[s] = (uint8_t)check_segment(&st, segs[s].check_begin, segs[s].check_end);
  }

  memset(estimate, 0, 8 * ((N + 63) / 64));
  memset(residual, 0, 8 * ((M + 63) / 64));
  for (uint32_t n = 0; n < N; ++n) {
    if (st.ehat[n]) put_bit(estimate, n);
  }
  for (uint32_t m = 0; m < M; ++m) {
    if (st.resid[m]) put_bit(residual, m);
  }
  if (qf_out && st.qf) memcpy(qf_out, st.qf, E * sizeof(float));
  if (rf_out && st.rf) memcpy(rf_out, st.rf, E * sizeof(float));
  if (qi_out && st.qi) memcpy(qi_out, st.qi, E * sizeof(int32_t));
  if (ri_out && st.ri) memcpy(ri_out, st.ri, E * sizeof(int32_t));

  free(frozen);
  free(st.sbit);
  free(st.ehat);
  free(st.resid);
  free(st.qf);
  free(st.rf);
  free(st.gf);
  free(st.qi);
  free(st.ri);
  free(st.gi);
  return ORACLE_OK;
}

/* Sequential map over `shots` syndromes with stride ceil(M/64) words; outputs
 * in whole-graph layout with converged = AND, iterations = MAX over segments
 * (decode_into semantics) when per_segment == 0, else [shots][nseg] arrays. */
int oracle_decode_many(const oracle_graph *g, const oracle_segment *segs, uint32_t nseg,
                       const oracle_config *cfg, uint64_t shots, const uint64_t *syndromes,
                       uint64_t *estimates, uint64_t *residuals, uint8_t *converged,
                       uint32_t *iterations, int per_segment) {
  const uint64_t sw = (g->num_checks + 63) / 64, ew = (g->num_vars + 63) / 64;
  uint64_t *rtmp = malloc(8 * sw);
  uint8_t *cs = malloc(nseg);
  uint32_t *is = malloc(4 * nseg);
  int rc = ORACLE_OK;
  for (uint64_t i = 0; i < shots && rc == ORACLE_OK; ++i) {
    rc = oracle_decode(g, segs, nseg, cfg, syndromes + i * sw, estimates + i * ew,
                       residuals ? residuals + i * sw : rtmp, cs, is, NULL, NULL, NULL, NULL);
    if (per_segment) {
      for (uint32_t s = 0; s < nseg; ++s) {
        converged[i * nseg + s] = cs[s];
        iterations[i * nseg + s] = is[s];
      }
    } else {
      uint8_t c = 1;
      uint32_t it = 0;
      for (uint32_t s = 0; s < nseg; ++s) {
        c = c && cs[s];
        if (is[s] > it) it = is[s];
      }
      converged[i] = c;
      iterations[i] = it;
    }
  }
  free(rtmp);
  free(cs);
  free(is);
  return rc;
}

/* Soft (noisy) syndromes: priors that change per shot.  The reference takes priors per
 * Decoder (decoder.hpp:31-32; quantised / stored in the constructor, decoder.cpp:108-131),
 * so per-shot soft information means one Decoder per shot: shot i is decoded
 * with the base priors of `cfg` (1.0 when empty) except priors[soft_vars[k]] = soft[i][k].
 * Everything else is oracle_decode / oracle_decode_many. */
int oracle_decode_many_soft(const oracle_graph *g, const oracle_segment *segs, uint32_t nseg,
                            const oracle_config *cfg, uint64_t shots, const uint64_t *syndromes,
                            const uint32_t *soft_vars, uint32_t nsoft, const double *soft,
                            uint64_t *estimates, uint64_t *residuals, uint8_t *converged,
                            uint32_t *iterations, int per_segment) {
  const uint32_t N = g->num_vars;
  const uint64_t sw = (g->num_checks + 63) / 64, ew = (N + 63) / 64;
  const int has_priors = cfg->priors && cfg->num_priors != 0;
  if (has_priors && cfg->num_priors != N) return ORACLE_INVALID;
  double *pri = malloc(sizeof(double) * N);
  for (uint32_t n = 0; n < N; ++n) pri[n] = has_priors ? cfg->priors[n] : 1.0;
  oracle_config c = *cfg;
  c.priors = pri;
  c.num_priors = N;
  int rc = ORACLE_OK;
  for (uint64_t i = 0; i < shots && rc == ORACLE_OK; ++i) {
    for (uint32_t k = 0; k < nsoft; ++k) {
      if (soft_vars[k] < N) pri[soft_vars[k]] = soft[i * nsoft + k];
    }
    rc = oracle_decode_many(g, segs, nseg, &c, 1, syndromes + i * sw, estimates + i * ew,
                            residuals ? residuals + i * sw : NULL,
                            converged + i * (per_segment ? nseg : 1),
                            iterations + i * (per_segment ? nseg : 1), per_segment);
  }
  free(pri);
  return rc;
}

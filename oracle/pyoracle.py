"""TEST INFRASTRUCTURE — ctypes front-ends for the CPU oracle and the compiled
reference.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this module; the product package
(paper_2508_07879_b200) never does.

* ``Oracle``  — oracle/libmsa_oracle.so, the plain-C restatement (msa_oracle.c).
* ``Ref``     — oracle/_ref/libqldpc_ref.so, the UNMODIFIED reference compiled
  from /root/reference by oracle/Makefile plus the C wrapper ref_capi.cpp.
  Built in the authoring container; travels to the GPU box as a prebuilt file.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "libmsa_oracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libqldpc_ref.so")
ARITH = {"float": 0, "int8": 1, "int16": 2}

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
u8p = C.POINTER(C.c_uint8)
f64p = C.POINTER(C.c_double)


def build(ref: bool = True) -> None:
    """make -C oracle (gcc only; the reference half needs /root/reference)."""
    subprocess.run(["make", "-C", _HERE, "libmsa_oracle.so"], check=True, capture_output=True)
    if ref and os.path.exists("/root/reference/proj/src/decoder.cpp"):
        subprocess.run(["make", "-C", _HERE, "-j8", "ref"], check=True, capture_output=True)


def _p(a, typ):
    return None if a is None else a.ctypes.data_as(typ)


def _words(bits: int) -> int:
    return (int(bits) + 63) // 64


class _Graph(C.Structure):
    _fields_ = [("num_checks", C.c_uint32), ("num_vars", C.c_uint32), ("num_edges", C.c_uint32),
                ("edge_var", u32p), ("check_offsets", u32p), ("var_offsets", u32p),
                ("var_edges", u32p)]


class _Segment(C.Structure):
    _fields_ = [("check_begin", C.c_uint32), ("check_end", C.c_uint32),
                ("var_begin", C.c_uint32), ("var_end", C.c_uint32)]


class _Config(C.Structure):
    _fields_ = [("max_iterations", C.c_uint64), ("alpha", C.c_double),
                ("early_termination", C.c_int32), ("arithmetic", C.c_int32),
                ("quant_scale", C.c_double), ("priors", f64p), ("num_priors", C.c_uint64)]


class Oracle:
    """The plain-C restatement.  `graph` is anything with the TannerGraph array
    attributes (paper_2508_07879_b200.codes.TannerGraph or RefGraph)."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        self.lib = C.CDLL(ORACLE_SO)
        self.lib.oracle_decode.restype = C.c_int
        self.lib.oracle_decode_many.restype = C.c_int
        self.lib.oracle_validate.restype = C.c_int
        self.lib.oracle_quantize_saturate.restype = C.c_int32
        self.lib.oracle_quantize_saturate.argtypes = [C.c_double, C.c_double, C.c_int32,
                                                      C.POINTER(C.c_int)]
        self.lib.oracle_check_node_update.argtypes = [f64p, C.c_uint64, C.c_int, C.c_double, f64p]
        self.lib.oracle_variable_node_update.argtypes = [C.c_double, f64p, C.c_uint64, f64p]
        self.lib.oracle_posterior.restype = C.c_double
        self.lib.oracle_posterior.argtypes = [C.c_double, f64p, C.c_uint64, C.POINTER(C.c_int)]

    # -- plumbing -----------------------------------------------------------
    @staticmethod
    def _pack(graph, segments, cfg):
        keep = [np.ascontiguousarray(getattr(graph, k), dtype=np.uint32)
                for k in ("edge_var", "check_offsets", "var_offsets", "var_edges")]
        g = _Graph(graph.num_checks, graph.num_vars, keep[0].size, _p(keep[0], u32p),
                   _p(keep[1], u32p), _p(keep[2], u32p), _p(keep[3], u32p))
        if segments is None:
            segments = [[0, graph.num_checks, 0, graph.num_vars]]
        seg_np = np.ascontiguousarray(segments, dtype=np.uint32).reshape(-1, 4)
        segs = (_Segment * seg_np.shape[0])(*[_Segment(*map(int, r)) for r in seg_np])
        pri = None
        if getattr(cfg, "priors", None) is not None and len(cfg.priors) > 0:
            pri = np.ascontiguousarray(cfg.priors, dtype=np.float64)
            keep.append(pri)
        c = _Config(int(cfg.max_iterations), float(cfg.alpha), 1 if cfg.early_termination else 0,
                    ARITH[cfg.arithmetic], float(cfg.quant_scale), _p(pri, f64p),
                    0 if pri is None else pri.size)
        return g, segs, seg_np.shape[0], c, keep

    def validate(self, graph, cfg) -> bool:
        g, _, _, c, keep = self._pack(graph, None, cfg)
        return self.lib.oracle_validate(C.byref(g), C.byref(c)) == 0

    def decode(self, graph, cfg, syndrome: np.ndarray, segments=None):
        """-> (estimate words, residual words, converged[nseg], iterations[nseg], q[E], r[E])."""
        g, segs, nseg, c, keep = self._pack(graph, segments, cfg)
        syn = np.ascontiguousarray(syndrome, dtype=np.uint64)
        est = np.zeros(_words(graph.num_vars), dtype=np.uint64)
        res = np.zeros(_words(graph.num_checks), dtype=np.uint64)
        conv = np.zeros(nseg, dtype=np.uint8)
        its = np.zeros(nseg, dtype=np.uint32)
        e = keep[0].size
        is_int = cfg.arithmetic != "float"
        q = np.zeros(e, dtype=np.int32 if is_int else np.float32)
        r = np.zeros(e, dtype=np.int32 if is_int else np.float32)
        vp = C.c_void_p
        margs = ((None, None, q.ctypes.data_as(vp), r.ctypes.data_as(vp)) if is_int
                 else (q.ctypes.data_as(vp), r.ctypes.data_as(vp), None, None))
        rc = self.lib.oracle_decode(C.byref(g), segs, C.c_uint32(nseg), C.byref(c), _p(syn, u64p),
                                    _p(est, u64p), _p(res, u64p), _p(conv, u8p), _p(its, u32p),
                                    *margs)
        if rc != 0:
            raise ValueError("oracle: invalid configuration")
        return est, res, conv, its, q, r

    def decode_many(self, graph, cfg, syndromes: np.ndarray, segments=None, per_segment=True):
        g, segs, nseg, c, keep = self._pack(graph, segments, cfg)
        syn = np.ascontiguousarray(syndromes, dtype=np.uint64)
        shots = syn.shape[0]
        est = np.zeros((shots, _words(graph.num_vars)), dtype=np.uint64)
        res = np.zeros((shots, _words(graph.num_checks)), dtype=np.uint64)
        k = nseg if per_segment else 1
        conv = np.zeros((shots, k), dtype=np.uint8)
        its = np.zeros((shots, k), dtype=np.uint32)
        rc = self.lib.oracle_decode_many(C.byref(g), segs, C.c_uint32(nseg), C.byref(c),
                                         C.c_uint64(shots), _p(syn, u64p), _p(est, u64p),
                                         _p(res, u64p), _p(conv, u8p), _p(its, u32p),
                                         C.c_int(1 if per_segment else 0))
        if rc != 0:
            raise ValueError("oracle: invalid configuration")
        return est, res, conv, its

    def decode_many_soft(self, graph, cfg, syndromes: np.ndarray, soft_vars, soft,
                         segments=None, per_segment=True):
        """Per-shot priors: shot i is decoded with cfg's priors except
        priors[soft_vars[k]] = soft[i][k] (doubles; one reference Decoder per shot)."""
        g, segs, nseg, c, keep = self._pack(graph, segments, cfg)
        syn = np.ascontiguousarray(syndromes, dtype=np.uint64)
        shots = syn.shape[0]
        sv = np.ascontiguousarray(soft_vars, dtype=np.uint32)
        so = np.ascontiguousarray(soft, dtype=np.float64).reshape(shots, sv.size)
        est = np.zeros((shots, _words(graph.num_vars)), dtype=np.uint64)
        res = np.zeros((shots, _words(graph.num_checks)), dtype=np.uint64)
        k = nseg if per_segment else 1
        conv = np.zeros((shots, k), dtype=np.uint8)
        its = np.zeros((shots, k), dtype=np.uint32)
        self.lib.oracle_decode_many_soft.restype = C.c_int
        rc = self.lib.oracle_decode_many_soft(C.byref(g), segs, C.c_uint32(nseg), C.byref(c),
                                              C.c_uint64(shots), _p(syn, u64p), _p(sv, u32p),
                                              C.c_uint32(sv.size), _p(so, f64p), _p(est, u64p),
                                              _p(res, u64p), _p(conv, u8p), _p(its, u32p),
                                              C.c_int(1 if per_segment else 0))
        if rc != 0:
            raise ValueError("oracle: invalid configuration")
        return est, res, conv, its

    # -- node ops (KATs) ------------------------------------------------------
    def check_node_update(self, q: Sequence[float], s_bit: int, alpha: float) -> np.ndarray:
        qa = np.ascontiguousarray(q, dtype=np.float64)
        out = np.zeros_like(qa)
        if self.lib.oracle_check_node_update(_p(qa, f64p), qa.size, s_bit, alpha, _p(out, f64p)):
            raise ValueError("check_node_update: invalid argument")
        return out

    def variable_node_update(self, gamma: float, r: Sequence[float]) -> np.ndarray:
        ra = np.ascontiguousarray(r, dtype=np.float64)
        out = np.zeros_like(ra)
        self.lib.oracle_variable_node_update(gamma, _p(ra, f64p), ra.size, _p(out, f64p))
        return out

    def posterior_and_decision(self, gamma: float, r: Sequence[float]) -> Tuple[float, int]:
        ra = np.ascontiguousarray(r, dtype=np.float64)
        bit = C.c_int()
        tot = self.lib.oracle_posterior(gamma, _p(ra, f64p), ra.size, C.byref(bit))
        return float(tot), int(bit.value)

    def quantize_saturate(self, value: float, scale: float, limit: int) -> int:
        err = C.c_int()
        out = self.lib.oracle_quantize_saturate(value, scale, limit, C.byref(err))
        if err.value:
            raise ValueError("quantize_saturate: value is NaN")
        return int(out)


# ---------------------------------------------------------------------------
# compiled reference
# ---------------------------------------------------------------------------

class RefGraph:
    """TannerGraph arrays copied out of the reference (same attribute names as
    paper_2508_07879_b200.codes.TannerGraph), plus the native pointer."""

    def __init__(self, ref: "Ref", ptr, owner=None):
        self._ref, self.ptr, self._owner = ref, ptr, owner
        m, n, e = C.c_uint64(), C.c_uint64(), C.c_uint64()
        ref.lib.ref_graph_dims(ptr, C.byref(m), C.byref(n), C.byref(e))
        self.num_checks, self.num_vars, self.num_edges = int(m.value), int(n.value), int(e.value)
        self.edge_var = np.zeros(self.num_edges, dtype=np.uint32)
        self.edge_check = np.zeros(self.num_edges, dtype=np.uint32)
        self.check_offsets = np.zeros(self.num_checks + 1, dtype=np.uint32)
        self.var_offsets = np.zeros(self.num_vars + 1, dtype=np.uint32)
        self.var_edges = np.zeros(self.num_edges, dtype=np.uint32)
        ref.lib.ref_graph_arrays(ptr, _p(self.edge_var, u32p), _p(self.edge_check, u32p),
                                 _p(self.check_offsets, u32p), _p(self.var_offsets, u32p),
                                 _p(self.var_edges, u32p))


class RefCode:
    def __init__(self, ref: "Ref", ptr):
        self._ref, self.ptr = ref, ptr
        v = [C.c_uint64() for _ in range(5)]
        ref.lib.ref_code_params(ptr, *[C.byref(x) for x in v])
        self.n, self.k, self.d, self.rows_x, self.rows_z = [int(x.value) for x in v]

    def graph(self, which: str) -> RefGraph:
        idx = {"x": 0, "z": 1, "combined": 2}[which]
        self._ref.lib.ref_code_graph.restype = C.c_void_p
        return RefGraph(self._ref, C.c_void_p(self._ref.lib.ref_code_graph(self.ptr, idx)), self)

    def matrix_coo(self, which: str) -> np.ndarray:
        idx = {"hx": 0, "hz": 1}[which]
        self._ref.lib.ref_code_matrix_nnz.restype = C.c_uint64
        nnz = int(self._ref.lib.ref_code_matrix_nnz(self.ptr, idx))
        out = np.zeros((nnz, 2), dtype=np.uint32)
        self._ref.lib.ref_code_matrix_coo(self.ptr, idx, _p(out, u32p))
        return out

    @property
    def segments(self) -> np.ndarray:
        mz, mx, n = self.rows_z, self.rows_x, self.n
        return np.asarray([[0, mz, 0, n], [mz, mz + mx, n, 2 * n]], dtype=np.uint32)

    def __del__(self):
        try:
            self._ref.lib.ref_code_free(self.ptr)
        except Exception:
            pass


class RefDecoder:
    def __init__(self, ref: "Ref", ptr, m: int, n: int, keep=None):
        self._ref, self.ptr, self.m, self.n, self._keep = ref, ptr, m, n, keep

    def decode(self, syndrome: np.ndarray, bits: Optional[int] = None):
        """decode_into -> (estimate, residual, converged, iterations, kernel_ns)."""
        syn = np.ascontiguousarray(syndrome, dtype=np.uint64)
        est = np.zeros(_words(self.n), dtype=np.uint64)
        res = np.zeros(_words(self.m), dtype=np.uint64)
        conv, its, kns = C.c_uint8(), C.c_uint64(), C.c_uint64()
        rc = self._ref.lib.ref_decode(self.ptr, _p(syn, u64p),
                                      C.c_uint64(self.m if bits is None else bits),
                                      _p(est, u64p), _p(res, u64p), C.byref(conv), C.byref(its),
                                      C.byref(kns))
        self._ref._check(rc)
        return est, res, bool(conv.value), int(its.value), int(kns.value)

    def decode_many(self, syndromes: np.ndarray, want_residual: bool = True):
        syn = np.ascontiguousarray(syndromes, dtype=np.uint64)
        shots = syn.shape[0]
        est = np.zeros((shots, _words(self.n)), dtype=np.uint64)
        res = np.zeros((shots, _words(self.m)), dtype=np.uint64) if want_residual else None
        conv = np.zeros(shots, dtype=np.uint8)
        its = np.zeros(shots, dtype=np.uint32)
        rc = self._ref.lib.ref_decode_many(self.ptr, C.c_uint64(shots), _p(syn, u64p),
                                           C.c_uint64(self.m), _p(est, u64p), _p(res, u64p),
                                           _p(conv, u8p), _p(its, u32p))
        self._ref._check(rc)
        return est, res, conv, its

    def decode_css(self, s_x: np.ndarray, bits_x: int, s_z: np.ndarray, bits_z: int, n: int):
        sx = np.ascontiguousarray(s_x, dtype=np.uint64)
        sz = np.ascontiguousarray(s_z, dtype=np.uint64)
        ex, ez = np.zeros(_words(n), dtype=np.uint64), np.zeros(_words(n), dtype=np.uint64)
        rx, rz = np.zeros(_words(bits_x), dtype=np.uint64), np.zeros(_words(bits_z), dtype=np.uint64)
        cx, cz, ix, iz = C.c_uint8(), C.c_uint8(), C.c_uint64(), C.c_uint64()
        rc = self._ref.lib.ref_decode_css(self.ptr, _p(sx, u64p), C.c_uint64(bits_x), _p(sz, u64p),
                                          C.c_uint64(bits_z), _p(ex, u64p), _p(rx, u64p),
                                          C.byref(cx), C.byref(ix), _p(ez, u64p), _p(rz, u64p),
                                          C.byref(cz), C.byref(iz))
        self._ref._check(rc)
        return (ex, rx, bool(cx.value), int(ix.value)), (ez, rz, bool(cz.value), int(iz.value))

    def __del__(self):
        try:
            self._ref.lib.ref_decoder_free(self.ptr)
        except Exception:
            pass


class Ref:
    """The compiled, unmodified reference."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self):
        if not os.path.exists(REF_SO):
            build(ref=True)
        if not os.path.exists(REF_SO):
            raise RuntimeError("oracle/_ref/libqldpc_ref.so is absent and /root/reference is not "
                               "available to build it")
        self.lib = C.CDLL(REF_SO)
        self.lib.ref_last_error.restype = C.c_char_p
        self.lib.ref_graphbox_graph.restype = C.c_void_p
        self.lib.ref_code_graph.restype = C.c_void_p
        self.lib.ref_percentile_nearest_rank.restype = C.c_double
        self.lib.ref_percentile_nearest_rank.argtypes = [f64p, C.c_uint64, C.c_double]

    def _check(self, rc: int) -> None:
        if rc == 0:
            return
        msg = self.lib.ref_last_error().decode("utf-8", "replace")
        if rc == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)

    # -- codes / graphs -----------------------------------------------------
    def builtin_code(self, name: str) -> RefCode:
        out = C.c_void_p()
        self._check(self.lib.ref_code_builtin(name.encode(), C.byref(out)))
        return RefCode(self, out)

    def bb_code(self, l, m, a_terms, b_terms, name="", d=0) -> RefCode:
        a = np.ascontiguousarray(a_terms, dtype=np.uint32).reshape(-1)
        b = np.ascontiguousarray(b_terms, dtype=np.uint32).reshape(-1)
        out = C.c_void_p()
        self._check(self.lib.ref_code_bb(C.c_uint64(l), C.c_uint64(m), _p(a, u32p),
                                         C.c_uint32(a.size // 2), _p(b, u32p),
                                         C.c_uint32(b.size // 2), name.encode(), C.c_uint64(d),
                                         C.byref(out)))
        return RefCode(self, out)

    def code_from_coo(self, name, rows_x, rows_z, cols, hx_coo, hz_coo) -> RefCode:
        hx = np.ascontiguousarray(hx_coo, dtype=np.uint32).reshape(-1, 2)
        hz = np.ascontiguousarray(hz_coo, dtype=np.uint32).reshape(-1, 2)
        out = C.c_void_p()
        self._check(self.lib.ref_code_from_coo(name.encode(), C.c_uint32(rows_x),
                                               C.c_uint32(rows_z), C.c_uint32(cols), _p(hx, u32p),
                                               C.c_uint64(hx.shape[0]), _p(hz, u32p),
                                               C.c_uint64(hz.shape[0]), C.byref(out)))
        return RefCode(self, out)

    def code(self, name: str) -> RefCode:
        """Registry code, or bb784 through build_bb_code (not in the registry)."""
        if name == "bb784":
            return self.bb_code(28, 14, [(26, 0), (0, 6), (0, 8)], [(0, 7), (9, 0), (20, 0)],
                                "bb784", 24)
        return self.builtin_code(name)

    def graph_from_coo(self, rows: int, cols: int, coo: np.ndarray) -> RefGraph:
        coo = np.ascontiguousarray(coo, dtype=np.uint32).reshape(-1, 2)
        box = C.c_void_p()
        self._check(self.lib.ref_graph_from_coo(C.c_uint32(rows), C.c_uint32(cols), _p(coo, u32p),
                                                C.c_uint64(coo.shape[0]), C.byref(box)))
        return RefGraph(self, C.c_void_p(self.lib.ref_graphbox_graph(box)), _Box(self, box))

    def toy_graph(self) -> RefGraph:
        box = C.c_void_p()
        self._check(self.lib.ref_graph_toy(C.byref(box)))
        return RefGraph(self, C.c_void_p(self.lib.ref_graphbox_graph(box)), _Box(self, box))

    # -- decoders -----------------------------------------------------------
    @staticmethod
    def _cfg_args(cfg):
        pri = None
        if getattr(cfg, "priors", None) is not None and len(cfg.priors) > 0:
            pri = np.ascontiguousarray(cfg.priors, dtype=np.float64)
        return pri, (C.c_uint64(int(cfg.max_iterations)), C.c_double(cfg.alpha),
                     C.c_int(1 if cfg.early_termination else 0), C.c_int(ARITH[cfg.arithmetic]),
                     C.c_double(cfg.quant_scale), _p(pri, f64p),
                     C.c_uint64(0 if pri is None else pri.size))

    def decoder(self, graph_or_code, cfg) -> RefDecoder:
        pri, args = self._cfg_args(cfg)
        out = C.c_void_p()
        if isinstance(graph_or_code, RefCode):
            self._check(self.lib.ref_decoder_new_code(graph_or_code.ptr, *args, C.byref(out)))
            return RefDecoder(self, out, graph_or_code.rows_x + graph_or_code.rows_z,
                              2 * graph_or_code.n, keep=graph_or_code)
        self._check(self.lib.ref_decoder_new_graph(graph_or_code.ptr, *args, C.byref(out)))
        return RefDecoder(self, out, graph_or_code.num_checks, graph_or_code.num_vars,
                          keep=graph_or_code)

    def decode_many_soft(self, graph: RefGraph, cfg, syndromes: np.ndarray, soft_vars, soft):
        """One unmodified reference Decoder PER SHOT with priors[soft_vars[k]] = soft[i][k]
        (ref_decode_many_soft); single segment, as the reference's graph constructor."""
        pri, args = self._cfg_args(cfg)
        syn = np.ascontiguousarray(syndromes, dtype=np.uint64)
        shots = syn.shape[0]
        sv = np.ascontiguousarray(soft_vars, dtype=np.uint32)
        so = np.ascontiguousarray(soft, dtype=np.float64).reshape(shots, sv.size)
        est = np.zeros((shots, _words(graph.num_vars)), dtype=np.uint64)
        res = np.zeros((shots, _words(graph.num_checks)), dtype=np.uint64)
        conv = np.zeros(shots, dtype=np.uint8)
        its = np.zeros(shots, dtype=np.uint32)
        self._check(self.lib.ref_decode_many_soft(
            graph.ptr, *args, _p(sv, u32p), C.c_uint32(sv.size), _p(so, f64p), C.c_uint64(shots),
            _p(syn, u64p), C.c_uint64(graph.num_checks), _p(est, u64p), _p(res, u64p),
            _p(conv, u8p), _p(its, u32p)))
        return est, res, conv, its

    def decode_batch(self, graph: RefGraph, syndromes: np.ndarray, cfg, workers: int = 1,
                     bits_each: Optional[Sequence[int]] = None):
        pri, args = self._cfg_args(cfg)
        syn = np.ascontiguousarray(syndromes, dtype=np.uint64)
        shots = syn.shape[0]
        est = np.zeros((shots, _words(graph.num_vars)), dtype=np.uint64)
        res = np.zeros((shots, _words(graph.num_checks)), dtype=np.uint64)
        conv = np.zeros(shots, dtype=np.uint8)
        its = np.zeros(shots, dtype=np.uint32)
        be = None if bits_each is None else np.ascontiguousarray(bits_each, dtype=np.uint64)
        rc = self.lib.ref_decode_batch(graph.ptr, C.c_uint64(shots), _p(syn, u64p),
                                       C.c_uint64(graph.num_checks), _p(be, u64p), *args,
                                       C.c_uint(workers), _p(est, u64p), _p(res, u64p),
                                       _p(conv, u8p), _p(its, u32p))
        self._check(rc)
        return est, res, conv, its

    # -- node ops -----------------------------------------------------------
    def check_node_update(self, q, s_bit, alpha) -> np.ndarray:
        qa = np.ascontiguousarray(q, dtype=np.float64)
        out = np.zeros_like(qa)
        self._check(self.lib.ref_check_node_update(_p(qa, f64p), C.c_uint64(qa.size),
                                                   C.c_int(s_bit), C.c_double(alpha),
                                                   _p(out, f64p)))
        return out

    def variable_node_update(self, gamma, r) -> np.ndarray:
        ra = np.ascontiguousarray(r, dtype=np.float64)
        out = np.zeros_like(ra)
        self._check(self.lib.ref_variable_node_update(C.c_double(gamma), _p(ra, f64p),
                                                      C.c_uint64(ra.size), _p(out, f64p)))
        return out

    def posterior_and_decision(self, gamma, r):
        ra = np.ascontiguousarray(r, dtype=np.float64)
        post, bit = C.c_double(), C.c_int()
        self._check(self.lib.ref_posterior_and_decision(C.c_double(gamma), _p(ra, f64p),
                                                        C.c_uint64(ra.size), C.byref(post),
                                                        C.byref(bit)))
        return float(post.value), int(bit.value)

    def quantize_saturate(self, value, scale, limit) -> int:
        out = C.c_int32()
        self._check(self.lib.ref_quantize_saturate(C.c_double(value), C.c_double(scale),
                                                   C.c_int32(limit), C.byref(out)))
        return int(out.value)

    # -- noise / campaign / bench ---------------------------------------------
    def sample_error(self, kind: int, p: float, seed: int, n: int, trial: int):
        ex = np.zeros(_words(n), dtype=np.uint64)
        ez = np.zeros(_words(n), dtype=np.uint64)
        self._check(self.lib.ref_sample_error(C.c_int(kind), C.c_double(p), C.c_uint64(seed),
                                              C.c_uint64(n), C.c_uint64(trial), _p(ex, u64p),
                                              _p(ez, u64p)))
        return ex, ez

    def extract_syndromes(self, code: RefCode, e_x: np.ndarray, e_z: np.ndarray):
        sx = np.zeros(_words(code.rows_z), dtype=np.uint64)
        sz = np.zeros(_words(code.rows_x), dtype=np.uint64)
        ex = np.ascontiguousarray(e_x, dtype=np.uint64)
        ez = np.ascontiguousarray(e_z, dtype=np.uint64)
        self._check(self.lib.ref_extract_syndromes(code.ptr, _p(ex, u64p), _p(ez, u64p),
                                                   _p(sx, u64p), _p(sz, u64p)))
        return sx, sz

    def syndrome_pool(self, code: RefCode, p: float, seed: int, count: int, first_trial: int = 0,
                      with_errors: bool = False):
        """run_bench's pool recipe (bench.cpp:203-211): combined syndromes s_x ++ s_z."""
        m = code.rows_x + code.rows_z
        out = np.zeros((count, _words(m)), dtype=np.uint64)
        ex = np.zeros((count, _words(code.n)), dtype=np.uint64) if with_errors else None
        ez = np.zeros((count, _words(code.n)), dtype=np.uint64) if with_errors else None
        self._check(self.lib.ref_syndrome_pool(code.ptr, C.c_double(p), C.c_uint64(seed),
                                               C.c_uint64(first_trial), C.c_uint64(count),
                                               _p(out, u64p), _p(ex, u64p), _p(ez, u64p)))
        return (out, ex, ez) if with_errors else out

    def classify(self, code: RefCode, e_x, ex_hat, e_z, ez_hat) -> int:
        arrs = [np.ascontiguousarray(a, dtype=np.uint64) for a in (e_x, ex_hat, e_z, ez_hat)]
        out = C.c_int()
        self._check(self.lib.ref_classify(code.ptr, *[_p(a, u64p) for a in arrs], C.byref(out)))
        return int(out.value)

    def run_campaign(self, code: RefCode, kind: int, p: float, seed: int, trials: int, cfg,
                     workers: int = 1):
        pri, args = self._cfg_args(cfg)
        counts = np.zeros(6, dtype=np.uint64)
        rates = np.zeros(4, dtype=np.float64)
        self._check(self.lib.ref_run_campaign(code.ptr, C.c_int(kind), C.c_double(p),
                                              C.c_uint64(seed), C.c_uint64(trials), *args,
                                              C.c_uint(workers), _p(counts, u64p),
                                              _p(rates, f64p)))
        keys = ("exact", "stabilizer", "logical_x", "logical_z", "logical_both", "non_converged")
        out = {k: int(v) for k, v in zip(keys, counts)}
        out.update(trials=trials, logical_error_rate=float(rates[0]),
                   baseline_logical_rate=float(rates[1]), convergence_rate=float(rates[2]),
                   mean_iterations=float(rates[3]))
        return out

    def run_bench(self, code: RefCode, arithmetic="float", alpha=0.8, max_iterations=10,
                  early_termination=False, batch=1, threads=1, warmup=100, measure=200, p=0.01,
                  seed=1):
        stats = np.zeros(8, dtype=np.float64)
        meta = np.zeros(3, dtype=np.uint64)
        self._check(self.lib.ref_run_bench(code.ptr, C.c_int(ARITH[arithmetic]), C.c_double(alpha),
                                           C.c_uint64(max_iterations),
                                           C.c_int(1 if early_termination else 0),
                                           C.c_uint64(batch), C.c_uint(threads),
                                           C.c_uint64(warmup), C.c_uint64(measure), C.c_double(p),
                                           C.c_uint64(seed), _p(stats, f64p), _p(meta, u64p)))
        keys = ("min_us", "mean_us", "median_us", "p99_us", "max_us", "conv_rate", "kernel_frac",
                "threads")
        out = {k: float(v) for k, v in zip(keys, stats)}
        out.update(digest=int(meta[0]), min_iterations=int(meta[1]), max_iterations=int(meta[2]))
        return out

    def read_bench_csv_file(self, path: str):
        """The reference's validating CSV reader -> (row count, p99 of the first row)."""
        rows, p99 = C.c_uint64(), C.c_double()
        self._check(self.lib.ref_read_bench_csv_file(path.encode(), C.byref(rows), C.byref(p99)))
        return int(rows.value), float(p99.value)

    def load_alist(self, text: str):
        """The reference's load_alist -> (rows, cols, (nnz, 2) COO array)."""
        rows, cols, nnz = C.c_uint64(), C.c_uint64(), C.c_uint64()
        buf = np.zeros((max(len(text), 16), 2), dtype=np.uint32)
        self._check(self.lib.ref_load_alist(text.encode(), C.byref(rows), C.byref(cols),
                                            _p(buf, u32p), C.c_uint64(buf.shape[0]),
                                            C.byref(nnz)))
        return int(rows.value), int(cols.value), buf[:int(nnz.value)].copy()

    def have_css_json(self) -> bool:
        return hasattr(self.lib, "ref_have_css_json") and bool(self.lib.ref_have_css_json())

    def css_json_load(self, text: str, base_dir: str = "") -> RefCode:
        """The reference's load_css_json (proj/src/css_json.cpp:84-150)."""
        out = C.c_void_p()
        self._check(self.lib.ref_css_json_load(text.encode(), base_dir.encode(), C.byref(out)))
        return RefCode(self, out)

    def css_json_save(self, code: RefCode) -> str:
        """The reference's save_css_json(code): self-contained descriptor, inline alists."""
        need = C.c_uint64()
        self._check(self.lib.ref_css_json_save(code.ptr, None, C.c_uint64(0), C.byref(need)))
        buf = C.create_string_buffer(int(need.value))
        self._check(self.lib.ref_css_json_save(code.ptr, buf, need, C.byref(need)))
        return buf.value.decode()

    def host_descriptor(self) -> str:
        buf = C.create_string_buffer(512)
        self._check(self.lib.ref_host_descriptor(buf, C.c_uint64(512)))
        return buf.value.decode()

    def percentile_nearest_rank(self, sorted_vals, pct) -> float:
        a = np.ascontiguousarray(sorted_vals, dtype=np.float64)
        return float(self.lib.ref_percentile_nearest_rank(_p(a, f64p), a.size, pct))


class _Box:
    def __init__(self, ref: Ref, ptr):
        self._ref, self.ptr = ref, ptr

    def __del__(self):
        try:
            self._ref.lib.ref_graphbox_free(self.ptr)
        except Exception:
            pass

"""Python mirror of the reference's decoder interface over the C-ABI.

Same names, argument meaning and error behaviour as
proj/include/qldpc/decoder.hpp:23-129 so that the parity tests read like the
reference's own (proj/tests/test_decoder.cpp): ``DecoderConfig``,
``DecodeOutcome``, ``Decoder(graph | code, cfg)``, ``decode``, ``decode_into``
(returns the outcome), ``decode_css_into``, ``last_kernel_ns``, and the free
functions ``decode``, ``decode_batch``, ``decode_css``.

``std::invalid_argument`` surfaces as ``ValueError``; CUDA failures as
``RuntimeError``.  Packed vectors are numpy ``uint64`` arrays in the
``Gf2Vector::words()`` layout.  All computation happens in the CUDA library.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import List, Optional, Sequence, Tuple, Union

import numpy as np

from . import _lib
from .codes import CssCode, TannerGraph
from .gf2 import num_words


@dataclasses.dataclass
class DecoderConfig:
    """reference: struct DecoderConfig (decoder.hpp:23-38)."""

    max_iterations: int = 10
    alpha: float = 0.8
    early_termination: bool = True
    priors: Optional[Sequence[float]] = None
    arithmetic: str = "float"  # "float" | "int8" | "int16" | "half" (extension)
    quant_scale: float = 0.0


@dataclasses.dataclass
class DecodeOutcome:
    """reference: struct DecodeOutcome (decoder.hpp:40-46)."""

    error_estimate: np.ndarray      # uint64 words, N bits
    converged: bool
    iterations_used: int
    syndrome_residual: np.ndarray   # uint64 words, M bits

    def same_as(self, other: "DecodeOutcome") -> bool:
        """reference: same_outcome (proj/tests/test_decoder.cpp:26-30)."""
        return (np.array_equal(self.error_estimate, other.error_estimate)
                and bool(self.converged) == bool(other.converged)
                and int(self.iterations_used) == int(other.iterations_used)
                and np.array_equal(self.syndrome_residual, other.syndrome_residual))


def _raise(status: int, handle) -> None:
    lib = _lib.load()
    msg = lib.qb_last_error(handle).decode("utf-8", "replace")
    if status == _lib.QB_INVALID_ARGUMENT:
        raise ValueError(msg)
    raise RuntimeError(msg)


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


def _ptr(a: Optional[np.ndarray], typ):
    return None if a is None else a.ctypes.data_as(typ)


class Decoder:
    """reference: class Decoder (decoder.hpp:77-108).  Not thread-safe; one per worker."""

    def __init__(self, graph_or_code: Union[TannerGraph, CssCode], cfg: Optional[DecoderConfig] = None,
                 device: int = 0, segments: Optional[np.ndarray] = None):
        lib = _lib.load()
        cfg = cfg if cfg is not None else DecoderConfig()
        self._cfg = dataclasses.replace(cfg)
        if isinstance(graph_or_code, CssCode):
            graph = graph_or_code.combined_graph
            segments = graph_or_code.segments
            self._css = True
        else:
            graph = graph_or_code
            self._css = segments is not None and len(segments) == 2
        self._graph = graph
        if cfg.arithmetic not in _lib.ARITH:
            raise ValueError(f"unknown arithmetic mode '{cfg.arithmetic}' "
                             "(expected float, int8, int16 or half)")
        ev, co, vo, ve = (_u32(graph.edge_var), _u32(graph.check_offsets),
                          _u32(graph.var_offsets), _u32(graph.var_edges))
        g = _lib.QbGraph(graph.num_checks, graph.num_vars, graph.num_edges,
                         _ptr(ev, _lib.u32p), _ptr(co, _lib.u32p), _ptr(vo, _lib.u32p),
                         _ptr(ve, _lib.u32p))
        pri = None
        if cfg.priors is not None and len(cfg.priors) > 0:
            pri = np.ascontiguousarray(cfg.priors, dtype=np.float64)
        if int(cfg.max_iterations) < 0:
            raise ValueError("DecoderConfig: max_iterations must be at least 1")
        c = _lib.QbConfig(int(cfg.max_iterations), float(cfg.alpha),
                          1 if cfg.early_termination else 0, _lib.ARITH[cfg.arithmetic],
                          float(cfg.quant_scale), _ptr(pri, _lib.f64p),
                          0 if pri is None else pri.size)
        seg_arr = None
        nseg = 0
        if segments is not None:
            seg_np = _u32(segments).reshape(-1, 4)
            nseg = seg_np.shape[0]
            seg_arr = (_lib.QbSegment * nseg)(*[_lib.QbSegment(*map(int, row)) for row in seg_np])
        handle = C.c_void_p()
        st = lib.qb_decoder_create(C.byref(g), seg_arr, nseg, C.byref(c), device, C.byref(handle))
        self._h = None
        if st != _lib.QB_OK:
            _raise(st, None)
        self._h = handle
        self._lib = lib
        self.num_segments = int(lib.qb_num_segments(handle))
        self._sw = num_words(graph.num_checks)
        self._ew = num_words(graph.num_vars)
        self._segments = (np.asarray([[0, graph.num_checks, 0, graph.num_vars]], dtype=np.uint32)
                          if segments is None else _u32(segments).reshape(-1, 4))

    # -- lifetime -----------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None) is not None:
            self._lib.qb_decoder_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- accessors ----------------------------------------------------------
    def config(self) -> DecoderConfig:
        return self._cfg

    def num_checks(self) -> int:
        return int(self._lib.qb_num_checks(self._h))

    def num_vars(self) -> int:
        return int(self._lib.qb_num_vars(self._h))

    def set_option(self, option: int, value: int) -> None:
        st = self._lib.qb_set_option(self._h, option, value)
        if st != _lib.QB_OK:
            _raise(st, self._h)

    def get_option(self, option: int) -> int:
        return int(self._lib.qb_get_option(self._h, option))

    def last_kernel_ns(self) -> int:
        return int(self._lib.qb_last_kernel_ns(self._h))

    def launch_count(self) -> int:
        return int(self._lib.qb_launch_count(self._h))

    # -- decode -------------------------------------------------------------
    def _check_syndrome(self, syndrome: np.ndarray, bits: Optional[int], what: str) -> np.ndarray:
        syndrome = np.ascontiguousarray(syndrome, dtype=np.uint64)
        m = self.num_checks()
        nbits = m if bits is None else int(bits)
        if nbits != m or syndrome.size != self._sw:
            raise ValueError(f"{what}: syndrome has {nbits} bits but the graph has {m} checks")
        return syndrome

    def decode_segments(self, syndrome: np.ndarray, bits: Optional[int] = None
                        ) -> Tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
        """One shot through qb_decode: (estimate words, residual words,
        converged[nseg], iterations[nseg])."""
        syndrome = self._check_syndrome(syndrome, bits, "decode")
        est = np.zeros(self._ew, dtype=np.uint64)
        res = np.zeros(self._sw, dtype=np.uint64)
        conv = np.zeros(self.num_segments, dtype=np.uint8)
        its = np.zeros(self.num_segments, dtype=np.uint32)
        st = self._lib.qb_decode(self._h, _ptr(syndrome, _lib.u64p), _ptr(est, _lib.u64p),
                                 _ptr(res, _lib.u64p), _ptr(conv, _lib.u8p), _ptr(its, _lib.u32p))
        if st != _lib.QB_OK:
            _raise(st, self._h)
        return est, res, conv, its

    def decode(self, syndrome: np.ndarray, bits: Optional[int] = None) -> DecodeOutcome:
        """Decoder::decode / decode_into (decoder.cpp:545-564): converged is the AND,
        iterations_used the MAX over segments (decoder.cpp:204-213)."""
        est, res, conv, its = self.decode_segments(syndrome, bits)
        return DecodeOutcome(est, bool(conv.all()), int(its.max()), res)

    decode_into = decode

    def decode_css_into(self, s_x: np.ndarray, s_z: np.ndarray, bits_x: Optional[int] = None,
                        bits_z: Optional[int] = None) -> Tuple[DecodeOutcome, DecodeOutcome]:
        """Decoder::decode_css_into (decoder.cpp:566-591)."""
        from .gf2 import concat_bits, pack_bits, unpack_bits
        if self.num_segments != 2 or not self._css:
            raise ValueError("decode_css_into: decoder was not built from a CssCode")
        (c0, c1, v0, v1), (d0, d1, u0, u1) = [tuple(map(int, r)) for r in self._segments]
        xc, zc = c1 - c0, d1 - d0
        bx = xc if bits_x is None else int(bits_x)
        bz = zc if bits_z is None else int(bits_z)
        s_x = np.ascontiguousarray(s_x, dtype=np.uint64)
        s_z = np.ascontiguousarray(s_z, dtype=np.uint64)
        if bx != xc or bz != zc or s_x.size != num_words(xc) or s_z.size != num_words(zc):
            raise ValueError(f"decode_css_into: syndrome lengths ({bx}, {bz}) do not match the "
                             f"code's check counts ({xc}, {zc})")
        est, res, conv, its = self.decode_segments(concat_bits(s_x, xc, s_z, zc))
        eb = unpack_bits(est, self.num_vars())
        rb = unpack_bits(res, self.num_checks())
        out_x = DecodeOutcome(pack_bits(eb[v0:v1]), bool(conv[0]), int(its[0]), pack_bits(rb[c0:c1]))
        out_z = DecodeOutcome(pack_bits(eb[u0:u1]), bool(conv[1]), int(its[1]), pack_bits(rb[d0:d1]))
        return out_x, out_z

    def decode_debug(self, syndrome: np.ndarray):
        """qb_decode_debug: outcome plus the final edge messages (q, r) in reference
        edge order (float32 for float/half, int32 for the integer modes)."""
        syndrome = self._check_syndrome(syndrome, None, "decode")
        e = self._graph.num_edges
        est = np.zeros(self._ew, dtype=np.uint64)
        res = np.zeros(self._sw, dtype=np.uint64)
        conv = np.zeros(self.num_segments, dtype=np.uint8)
        its = np.zeros(self.num_segments, dtype=np.uint32)
        is_int = self._cfg.arithmetic in ("int8", "int16")
        q = np.zeros(e, dtype=np.int32 if is_int else np.float32)
        r = np.zeros(e, dtype=np.int32 if is_int else np.float32)
        args = ((None, None, _ptr(q, _lib.i32p), _ptr(r, _lib.i32p)) if is_int
                else (_ptr(q, _lib.f32p), _ptr(r, _lib.f32p), None, None))
        st = self._lib.qb_decode_debug(self._h, _ptr(syndrome, _lib.u64p), _ptr(est, _lib.u64p),
                                       _ptr(res, _lib.u64p), _ptr(conv, _lib.u8p),
                                       _ptr(its, _lib.u32p), *args)
        if st != _lib.QB_OK:
            _raise(st, self._h)
        return est, res, conv, its, q, r

    def decode_batch_debug(self, syndromes: np.ndarray, dump_shot: int):
        """qb_decode_batch_debug: the batch kernel's outcomes plus the final edge messages
        (q, r) of shot `dump_shot`, in reference edge order."""
        syndromes = np.ascontiguousarray(syndromes, dtype=np.uint64)
        if syndromes.ndim != 2 or syndromes.shape[1] != self._sw:
            raise ValueError(f"decode_batch: syndromes must be (shots, {self._sw}) uint64 words")
        shots, e = syndromes.shape[0], self._graph.num_edges
        est = np.zeros((shots, self._ew), dtype=np.uint64)
        res = np.zeros((shots, self._sw), dtype=np.uint64)
        conv = np.zeros((shots, self.num_segments), dtype=np.uint8)
        its = np.zeros((shots, self.num_segments), dtype=np.uint32)
        is_int = self._cfg.arithmetic in ("int8", "int16")
        q = np.zeros(e, dtype=np.int32 if is_int else np.float32)
        r = np.zeros(e, dtype=np.int32 if is_int else np.float32)
        args = ((None, None, _ptr(q, _lib.i32p), _ptr(r, _lib.i32p)) if is_int
                else (_ptr(q, _lib.f32p), _ptr(r, _lib.f32p), None, None))
        st = self._lib.qb_decode_batch_debug(self._h, shots, syndromes.ctypes.data, int(dump_shot),
                                             est.ctypes.data, res.ctypes.data, conv.ctypes.data,
                                             its.ctypes.data, *args)
        if st != _lib.QB_OK:
            _raise(st, self._h)
        return est, res, conv, its, q, r

    def decode_batch_segments(self, syndromes: np.ndarray, want_residual: bool = True):
        """qb_decode_batch on (shots, ceil(M/64)) host words: (estimates, residuals | None,
        converged[shots, nseg], iterations[shots, nseg])."""
        syndromes = np.ascontiguousarray(syndromes, dtype=np.uint64)
        if syndromes.ndim != 2 or syndromes.shape[1] != self._sw:
            raise ValueError(f"decode_batch: syndromes must be (shots, {self._sw}) uint64 words")
        shots = syndromes.shape[0]
        est = np.zeros((shots, self._ew), dtype=np.uint64)
        res = np.zeros((shots, self._sw), dtype=np.uint64) if want_residual else None
        conv = np.zeros((shots, self.num_segments), dtype=np.uint8)
        its = np.zeros((shots, self.num_segments), dtype=np.uint32)
        st = self._lib.qb_decode_batch(self._h, shots, syndromes.ctypes.data, est.ctypes.data,
                                       None if res is None else res.ctypes.data,
                                       conv.ctypes.data, its.ctypes.data)
        if st != _lib.QB_OK:
            _raise(st, self._h)
        return est, res, conv, its

    def decode_batch_raw(self, shots: int, syn_ptr: int, est_ptr: int, res_ptr: Optional[int],
                         conv_ptr: int, its_ptr: int) -> None:
        """qb_decode_batch on caller-owned HOST buffers given as addresses (e.g. pinned)."""
        st = self._lib.qb_decode_batch(self._h, shots, syn_ptr, est_ptr, res_ptr, conv_ptr, its_ptr)
        if st != _lib.QB_OK:
            _raise(st, self._h)

    def decode_batch_device(self, shots: int, d_syn: int, d_est: int, d_res: Optional[int],
                            d_conv: int, d_its: int, stream: int = 0) -> None:
        """qb_decode_batch_device on DEVICE addresses (e.g. torch tensors' data_ptr())."""
        st = self._lib.qb_decode_batch_device(self._h, shots, d_syn, d_est, d_res, d_conv, d_its,
                                              stream)
        if st != _lib.QB_OK:
            _raise(st, self._h)


    # -- soft (noisy) syndromes: per-shot priors of the absorbed variables ---------------
    SOFT_DTYPES = {"float": np.float32, "half": np.float32, "int8": np.int8, "int16": np.int16}

    def soft_vars(self) -> np.ndarray:
        """qb_soft_vars: for every check the variable whose prior a soft value replaces
        (0xffffffff: none)."""
        out = np.zeros(self.num_checks(), dtype=np.uint32)
        st = self._lib.qb_soft_vars(self._h, _ptr(out, _lib.u32p))
        if st != _lib.QB_OK:
            _raise(st, self._h)
        return out

    def soft_dtype(self):
        return self.SOFT_DTYPES[self._cfg.arithmetic]

    def quantize_soft(self, llr: np.ndarray) -> np.ndarray:
        """Reliabilities (LLR magnitudes, any shape) -> the decoder's soft format: float32, or
        quantize_saturate(llr, quant_scale, kmax) (decoder.cpp:500-509) with results of 0
        clamped to +-1 (the reference rejects a prior that quantises to 0, decoder.cpp:115-120)."""
        llr = np.asarray(llr, dtype=np.float64)
        if self._cfg.arithmetic in ("float", "half"):
            return llr.astype(np.float32)
        kmax = 127 if self._cfg.arithmetic == "int8" else 32767
        scale = self._cfg.quant_scale or (8.0 if self._cfg.arithmetic == "int8" else 256.0)
        scaled = llr * scale
        q = np.where(scaled >= 0, np.floor(scaled + 0.5), -np.floor(-scaled + 0.5))  # llround
        q = np.clip(q, -kmax, kmax)
        q = np.where(q == 0, np.where(np.signbit(scaled), -1, 1), q)
        return q.astype(self.soft_dtype())

    def _check_soft(self, soft: np.ndarray, shots: int) -> np.ndarray:
        soft = np.ascontiguousarray(soft, dtype=self.soft_dtype())
        if soft.shape != (shots, self.num_checks()):
            raise ValueError(f"decode_batch_soft: soft values must be ({shots}, {self.num_checks()})")
        if self._cfg.arithmetic in ("int8", "int16"):
            used = self.soft_vars() != 0xffffffff
            if (soft[:, used] == 0).any() or (soft[:, used] == np.iinfo(soft.dtype).min).any():
                raise ValueError("decode_batch_soft: a quantised prior is 0 (the reference rejects "
                                 "it, decoder.cpp:115-120) or below -kmax")
        elif not np.isfinite(soft).all():
            raise ValueError("decode_batch_soft: a prior is not finite")
        return soft

    def decode_soft_segments(self, syndrome: np.ndarray, soft: np.ndarray):
        """qb_decode_soft: one shot through the latency path with per-shot priors."""
        syndrome = self._check_syndrome(syndrome, None, "decode")
        soft = self._check_soft(np.asarray(soft)[None, :], 1)[0]
        est = np.zeros(self._ew, dtype=np.uint64)
        res = np.zeros(self._sw, dtype=np.uint64)
        conv = np.zeros(self.num_segments, dtype=np.uint8)
        its = np.zeros(self.num_segments, dtype=np.uint32)
        st = self._lib.qb_decode_soft(self._h, _ptr(syndrome, _lib.u64p), soft.ctypes.data,
                                      _ptr(est, _lib.u64p), _ptr(res, _lib.u64p), _ptr(conv, _lib.u8p),
                                      _ptr(its, _lib.u32p))
        if st != _lib.QB_OK:
            _raise(st, self._h)
        return est, res, conv, its

    def decode_batch_soft_segments(self, syndromes: np.ndarray, soft: np.ndarray,
                                   want_residual: bool = True):
        """qb_decode_batch_soft on host arrays: syndromes (shots, ceil(M/64)) uint64 words and
        soft (shots, M) per-shot priors of the absorbed variables in soft_dtype()."""
        syndromes = np.ascontiguousarray(syndromes, dtype=np.uint64)
        if syndromes.ndim != 2 or syndromes.shape[1] != self._sw:
            raise ValueError(f"decode_batch: syndromes must be (shots, {self._sw}) uint64 words")
        shots = syndromes.shape[0]
        soft = self._check_soft(soft, shots)
        est = np.zeros((shots, self._ew), dtype=np.uint64)
        res = np.zeros((shots, self._sw), dtype=np.uint64) if want_residual else None
        conv = np.zeros((shots, self.num_segments), dtype=np.uint8)
        its = np.zeros((shots, self.num_segments), dtype=np.uint32)
        st = self._lib.qb_decode_batch_soft(self._h, shots, syndromes.ctypes.data, soft.ctypes.data,
                                            est.ctypes.data, None if res is None else res.ctypes.data,
                                            conv.ctypes.data, its.ctypes.data)
        if st != _lib.QB_OK:
            _raise(st, self._h)
        return est, res, conv, its

    def decode_batch_soft_device(self, shots: int, d_syn: int, d_soft: int, d_est: int,
                                 d_res: Optional[int], d_conv: int, d_its: int, stream: int = 0) -> None:
        st = self._lib.qb_decode_batch_soft_device(self._h, shots, d_syn, d_soft, d_est, d_res,
                                                   d_conv, d_its, stream)
        if st != _lib.QB_OK:
            _raise(st, self._h)

    def generate_soft_syndromes(self, seed: int, p: float, mu: float, sigma: float, shots: int,
                                d_syn: int, d_soft: int, d_err: Optional[int] = None,
                                first_trial: int = 0, probs: Optional[Sequence[float]] = None,
                                stream: int = 0) -> None:
        """qb_generate_soft_syndromes: data flips + Gaussian soft measurement on the device."""
        pr = None if probs is None else np.ascontiguousarray(probs, dtype=np.float64)
        st = self._lib.qb_generate_soft_syndromes(self._h, seed, float(p), _ptr(pr, _lib.f64p),
                                                  float(mu), float(sigma), first_trial, shots,
                                                  d_syn, d_soft, d_err, stream)
        if st != _lib.QB_OK:
            _raise(st, self._h)

    def latency_run(self, pool: np.ndarray, warmup: int, measure: int,
                    soft_pool: Optional[np.ndarray] = None):
        """qb_latency_run: the reference's run_bench protocol at batch 1
        (proj/src/bench.cpp:182-337) -> (wall_ns[measure], kernel_ns[measure], digest).
        With `soft_pool` ((n, num_checks) values as decode_batch_soft takes them) every decode
        is a qb_decode_soft (qb_latency_run_soft)."""
        pool = np.ascontiguousarray(pool, dtype=np.uint64)
        if pool.ndim != 2 or pool.shape[1] != self._sw:
            raise ValueError(f"latency_run: pool must be (n, {self._sw}) uint64 words")
        soft_ptr = None
        if soft_pool is not None:
            soft_pool = self._check_soft(soft_pool, pool.shape[0])
            soft_ptr = soft_pool.ctypes.data
        wall = np.zeros(measure, dtype=np.uint64)
        kern = np.zeros(measure, dtype=np.uint64)
        digest = C.c_uint64()
        st = self._lib.qb_latency_run_soft(self._h, _ptr(pool, _lib.u64p), soft_ptr, pool.shape[0],
                                           warmup, measure, _ptr(wall, _lib.u64p),
                                           _ptr(kern, _lib.u64p), C.byref(digest))
        if st != _lib.QB_OK:
            _raise(st, self._h)
        return wall, kern, int(digest.value)

    def generate_syndromes(self, seed: int, p: float, shots: int, d_syn: int,
                           d_err: Optional[int] = None, first_trial: int = 0,
                           probs: Optional[Sequence[float]] = None, css_interleave: bool = True,
                           stream: int = 0) -> None:
        """qb_generate_syndromes: on-device sample_error + extract_syndromes
        (proj/src/noise.cpp:67-105) into DEVICE buffers, bit-exact with the
        reference's SplitMix64 streams."""
        pr = None if probs is None else np.ascontiguousarray(probs, dtype=np.float64)
        st = self._lib.qb_generate_syndromes(self._h, seed, float(p), _ptr(pr, _lib.f64p),
                                             1 if css_interleave else 0, first_trial, shots,
                                             d_syn, d_err, stream)
        if st != _lib.QB_OK:
            _raise(st, self._h)


# ---- free functions (decoder.hpp:110-129) -----------------------------------

def decode(graph: TannerGraph, syndrome: np.ndarray, cfg: DecoderConfig,
           bits: Optional[int] = None) -> DecodeOutcome:
    with Decoder(graph, cfg) as dec:
        return dec.decode(syndrome, bits)


def decode_batch(graph: TannerGraph, syndromes: Sequence[np.ndarray], cfg: DecoderConfig,
                 num_workers: int = 1, bits: Optional[Sequence[int]] = None) -> List[DecodeOutcome]:
    """reference: decode_batch (decoder.cpp:604-655).  Every length is validated up
    front; results are elementwise identical to sequential decodes for every
    `num_workers` (which only names the CPU thread count in the reference and is
    accepted and ignored here: the batch is one persistent-kernel launch)."""
    m = graph.num_checks
    sw = num_words(m)
    for i, s in enumerate(syndromes):
        nbits = m if bits is None else int(bits[i])
        if nbits != m or np.asarray(s).size != sw:
            raise ValueError(f"decode_batch: syndrome {i} has {nbits} bits but the graph has "
                             f"{m} checks")
    if len(syndromes) == 0:
        return []  # decoder.cpp:617: returns before any Decoder is built
    with Decoder(graph, cfg) as dec:
        est, res, conv, its = dec.decode_batch_segments(np.stack([np.asarray(s, dtype=np.uint64)
                                                                  for s in syndromes]))
    return [DecodeOutcome(est[i], bool(conv[i].all()), int(its[i].max()), res[i])
            for i in range(len(syndromes))]


def decode_css(code: CssCode, s_x: np.ndarray, s_z: np.ndarray, cfg: DecoderConfig
               ) -> Tuple[DecodeOutcome, DecodeOutcome]:
    with Decoder(code, cfg) as dec:
        return dec.decode_css_into(s_x, s_z)

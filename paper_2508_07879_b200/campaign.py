"""Monte-Carlo logical-error-rate campaigns (reference: run_campaign,
proj/src/noise.cpp:217-338) with the whole trial loop on the GPU: the library's
SplitMix64-exact sampler, the batch decode kernel and the residual classifier
run back to back, and only ten counters come back per call.

Multi-GPU: trials are split contiguously across ranks exactly as the reference
splits them across worker threads (``[r*T/W, (r+1)*T/W)``, noise.cpp:253-254);
every trial has its own random stream, so the result is independent of the
number of ranks.  The ONLY collective is one all-reduce(sum) of the counter
vector at the end (noise.cpp:306-324) - NCCL on GPUs, gloo in the CPU tests.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from .codes import CssCode, SparseMatrix
from .decoder import Decoder, DecoderConfig, _raise
from .gf2 import num_words, pack_bits, unpack_bits

COUNTER_NAMES = ("exact", "stabilizer", "logical_x", "logical_z", "logical_both",
                 "non_converged", "baseline_fail", "converged_both", "iteration_sum", "trials")


# ---- GF(2) linear algebra on Python-int bitsets (cold, run once per code) ----------

def _rows_as_ints(m: SparseMatrix) -> List[int]:
    out = []
    for sup in m.row_support:
        x = 0
        for c in sup:
            x |= 1 << c
        out.append(x)
    return out


def _nullspace(rows: Sequence[int], ncols: int) -> List[int]:
    """Basis of {v : <row, v> = 0 for every row} over GF(2)."""
    pivots: Dict[int, int] = {}  # pivot column -> reduced row
    for r in rows:
        for col, pr in pivots.items():
            if (r >> col) & 1:
                r ^= pr
        if r:
            col = r.bit_length() - 1
            for c2 in list(pivots):
                if (pivots[c2] >> col) & 1:
                    pivots[c2] ^= r
            pivots[col] = r
    free = [c for c in range(ncols) if c not in pivots]
    basis = []
    for f in free:
        v = 1 << f
        for col, pr in pivots.items():
            if (pr >> f) & 1:
                v |= 1 << col
        basis.append(v)
    return basis


def _independent_of(span_rows: Sequence[int], candidates: Sequence[int]) -> List[int]:
    """Candidates that extend the row space of `span_rows`, greedily."""
    basis: Dict[int, int] = {}

    def reduce(x: int) -> int:
        while x:
            top = x.bit_length() - 1
            if top not in basis:
                return x
            x ^= basis[top]
        return 0

    for r in span_rows:
        x = reduce(r)
        if x:
            basis[x.bit_length() - 1] = x
    out = []
    for c in candidates:
        x = reduce(c)
        if x:
            basis[x.bit_length() - 1] = x
            out.append(c)
    return out


def logical_operators(code: CssCode) -> Tuple[List[int], List[int]]:
    """(logical Z operators, logical X operators) as n-bit integers:
    Lz spans ker(hx) modulo rowspace(hz), Lx spans ker(hz) modulo rowspace(hx)."""
    hx, hz = _rows_as_ints(code.hx), _rows_as_ints(code.hz)
    lz = _independent_of(hz, _nullspace(hx, code.n))
    lx = _independent_of(hx, _nullspace(hz, code.n))
    if len(lz) != code.k or len(lx) != code.k:
        raise RuntimeError(f"expected {code.k} logical operators, found {len(lz)} / {len(lx)}")
    return lz, lx


def residual_tests(code: CssCode) -> Tuple[np.ndarray, np.ndarray]:
    """Test vectors for qb_set_logicals in the combined layout (2n bits):
    x_tests = logical Z operators on the X-error variables [0, n),
    z_tests = logical X operators on the Z-error variables [n, 2n)."""
    lz, lx = logical_operators(code)
    n = code.n

    def place(vals: Sequence[int], shift: int) -> np.ndarray:
        bits = np.zeros((len(vals), 2 * n), dtype=np.uint8)
        for j, v in enumerate(vals):
            for i in range(n):
                if (v >> i) & 1:
                    bits[j, shift + i] = 1
        return pack_bits(bits)

    return place(lz, 0), place(lx, n)


# ---- campaign ------------------------------------------------------------------------

@dataclasses.dataclass
class CampaignResult:
    """reference: struct CampaignResult (proj/include/qldpc/noise.hpp:118-137)."""

    trials: int = 0
    exact: int = 0
    stabilizer: int = 0
    logical_x: int = 0
    logical_z: int = 0
    logical_both: int = 0
    non_converged: int = 0
    logical_error_rate: float = 0.0
    baseline_logical_rate: float = 0.0
    convergence_rate: float = 0.0
    mean_iterations: float = 0.0

    @staticmethod
    def from_counters(c: Sequence[int]) -> "CampaignResult":
        d = dict(zip(COUNTER_NAMES, (int(x) for x in c)))
        t = max(d["trials"], 1)
        return CampaignResult(
            trials=d["trials"], exact=d["exact"], stabilizer=d["stabilizer"],
            logical_x=d["logical_x"], logical_z=d["logical_z"], logical_both=d["logical_both"],
            non_converged=d["non_converged"],
            logical_error_rate=(d["logical_x"] + d["logical_z"] + d["logical_both"]
                                + d["non_converged"]) / t,
            baseline_logical_rate=d["baseline_fail"] / t,
            convergence_rate=d["converged_both"] / t, mean_iterations=d["iteration_sum"] / t)


def shard(trials: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous trial range of `rank` (noise.cpp:253-254)."""
    return rank * trials // world, (rank + 1) * trials // world


def reduce_counters(counters: np.ndarray, group=None, device=None, world: int = 1) -> np.ndarray:
    """Sum of the counter vectors of every rank (one all_reduce; the analogue of the
    reference's integer sum over workers, noise.cpp:306-324).  Without a process group this
    is the identity for world == 1 and an ERROR for world > 1: returning one shard's
    counters as if they were the campaign's would look valid and be wrong."""
    try:
        import torch
        import torch.distributed as dist
    except ImportError:  # pragma: no cover
        if world > 1:
            raise RuntimeError("reduce_counters: world > 1 needs torch.distributed")
        return counters
    if not (dist.is_available() and dist.is_initialized()):
        if world > 1:
            raise RuntimeError("reduce_counters: world > 1 but no process group is initialised "
                               "(torch.distributed.init_process_group)")
        return counters
    t = torch.as_tensor(np.asarray(counters, dtype=np.int64))
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy().astype(np.uint64)


class Campaign:
    """A decoder plus the residual tests of its code, ready to run trial ranges."""

    def __init__(self, code: CssCode, cfg: DecoderConfig, device: int = 0):
        self.code = code
        self.decoder = Decoder(code, cfg, device=device)
        x_tests, z_tests = residual_tests(code)
        self._tests = (np.ascontiguousarray(x_tests), np.ascontiguousarray(z_tests))
        lib = _lib.load()
        st = lib.qb_set_logicals(self.decoder._h, self._tests[0].ctypes.data_as(_lib.u64p),
                                 self._tests[0].shape[0],
                                 self._tests[1].ctypes.data_as(_lib.u64p), self._tests[1].shape[0])
        if st != _lib.QB_OK:
            _raise(st, self.decoder._h)

    def run_range(self, p: float, seed: int, first_trial: int, trials: int) -> np.ndarray:
        counters = np.zeros(len(COUNTER_NAMES), dtype=np.uint64)
        st = _lib.load().qb_campaign_run(self.decoder._h, seed, float(p), None, first_trial, trials,
                                         counters.ctypes.data_as(_lib.u64p))
        if st != _lib.QB_OK:
            _raise(st, self.decoder._h)
        return counters

    def classify_device(self, shots: int, d_err: int, d_est: int, d_syn: int, d_conv: int,
                        d_its: int, stream: int = 0) -> np.ndarray:
        """qb_classify_batch_device on resident buffers -> the ten counters."""
        counters = np.zeros(len(COUNTER_NAMES), dtype=np.uint64)
        st = _lib.load().qb_classify_batch_device(self.decoder._h, shots, d_err, d_est, d_syn,
                                                  d_conv, d_its,
                                                  counters.ctypes.data_as(_lib.u64p), stream)
        if st != _lib.QB_OK:
            _raise(st, self.decoder._h)
        return counters

    def close(self) -> None:
        self.decoder.close()


def run_campaign(code: CssCode, p: float, seed: int, trials: int, cfg: DecoderConfig,
                 device: int = 0, world: int = 1, rank: int = 0, group=None,
                 range_fn=None, reduce_device="cuda") -> CampaignResult:
    """reference: run_campaign(code, NoiseModel{independent-xz, p, seed}, trials, cfg).
    With world > 1 every rank calls this with its own `rank`; all ranks return the
    same aggregated result (contiguous shard per rank, noise.cpp:253-254, then ONE
    all_reduce of the ten counters).

    `range_fn(p, seed, first_trial, trials) -> counters` replaces the device decoder for the
    rank's trial range (tests drive this very function on CPU ranks over gloo, with
    `reduce_device="cpu"`); the default builds a Campaign on `device`."""
    if not (0.0 <= p <= 1.0):
        raise ValueError("NoiseModel: p must lie in [0, 1]")
    if world < 1 or not (0 <= rank < world):
        raise ValueError("run_campaign: rank must lie in [0, world)")
    lo, hi = shard(trials, world, rank)
    camp = None
    if range_fn is None:
        camp = Campaign(code, cfg, device=device)
        range_fn = camp.run_range
    try:
        counters = np.asarray(range_fn(p, seed, lo, hi - lo), dtype=np.uint64) if hi > lo else \
            np.zeros(len(COUNTER_NAMES), dtype=np.uint64)
    finally:
        if camp is not None:
            camp.close()
    if world > 1:
        import torch
        dev = torch.device("cuda", device) if reduce_device == "cuda" else torch.device("cpu")
        counters = reduce_counters(counters, group, dev, world=world)
    return CampaignResult.from_counters(counters)


# ---- BASELINE config 5: phenomenological noise on the extended graph ---------------------

class PhenomenologicalCampaign:
    """Campaigns on diag([Hz | I], [Hx | I]) (codes.extended_graph): data qubits flip with
    probability p, every measured syndrome bit is noisy - either flipped with probability q
    (hard syndromes, constant prior ln((1-q)/q) on the measurement-error variables) or read
    through a Gaussian channel (soft syndromes, per-shot priors |LLR_m|).  Sample, measure,
    decode and classify all run on the device (qb_campaign_run / qb_campaign_run_soft).

    A trial FAILS unless both components converge and the data residual has zero syndrome
    and is no logical operator; in the ten counters a data residual with non-zero syndrome
    is booked as a logical error of its component.  The reference has no such noise model
    (SPEC.md:15): this is new-build behaviour on top of its decoder semantics."""

    def __init__(self, code: CssCode, cfg: DecoderConfig, p_data: float, p_meas: float,
                 device: int = 0):
        from .codes import build_tanner_graph, extended_graph
        self.code = code
        h, segs = extended_graph(code)
        self.h_ext, self.segments = h, segs
        self.graph = build_tanner_graph(h)
        n, mz, mx = code.n, code.hz.rows, code.hx.rows
        self.data_slices = (slice(0, n), slice(n + mz, 2 * n + mz))
        self.p_data, self.p_meas = float(p_data), float(p_meas)
        if cfg.priors is None:
            llr_d = float(np.log((1 - p_data) / p_data))
            llr_m = float(np.log((1 - p_meas) / p_meas))
            pri = np.concatenate([np.full(n, llr_d), np.full(mz, llr_m), np.full(n, llr_d),
                                  np.full(mx, llr_m)])
            cfg = dataclasses.replace(cfg, priors=pri.tolist())
        self.probs = np.concatenate([np.full(n, p_data), np.full(mz, p_meas), np.full(n, p_data),
                                     np.full(mx, p_meas)])
        self.decoder = Decoder(self.graph, cfg, device=device, segments=segs)
        lib = _lib.load()
        tx, tz = residual_tests(code)  # over 2n bits: place the data parts in the extended layout
        bx, bz = unpack_bits(tx, 2 * n), unpack_bits(tz, 2 * n)
        nv = self.graph.num_vars
        ex = np.zeros((bx.shape[0], nv), dtype=np.uint8)
        ez = np.zeros((bz.shape[0], nv), dtype=np.uint8)
        ex[:, self.data_slices[0]] = bx[:, :n]
        ez[:, self.data_slices[1]] = bz[:, n:]
        self.tests_bits = (ex, ez)
        self._tests = (np.ascontiguousarray(pack_bits(ex)), np.ascontiguousarray(pack_bits(ez)))
        st = lib.qb_set_logicals(self.decoder._h, self._tests[0].ctypes.data_as(_lib.u64p),
                                 self._tests[0].shape[0],
                                 self._tests[1].ctypes.data_as(_lib.u64p), self._tests[1].shape[0])
        if st != _lib.QB_OK:
            _raise(st, self.decoder._h)
        aux = np.ones(nv, dtype=np.uint8)
        aux[self.data_slices[0]] = 0
        aux[self.data_slices[1]] = 0
        self.aux_bits = aux
        self._aux = np.ascontiguousarray(pack_bits(aux))
        st = lib.qb_set_auxiliary_vars(self.decoder._h, self._aux.ctypes.data_as(_lib.u64p))
        if st != _lib.QB_OK:
            _raise(st, self.decoder._h)

    def run_range(self, seed: int, first_trial: int, trials: int) -> np.ndarray:
        """Hard noisy syndromes: every variable v flips with probs[v]."""
        counters = np.zeros(len(COUNTER_NAMES), dtype=np.uint64)
        st = _lib.load().qb_campaign_run(self.decoder._h, seed, 0.0,
                                         self.probs.ctypes.data_as(_lib.f64p), first_trial, trials,
                                         counters.ctypes.data_as(_lib.u64p))
        if st != _lib.QB_OK:
            _raise(st, self.decoder._h)
        return counters

    def run_range_soft(self, seed: int, mu: float, sigma: float, first_trial: int,
                       trials: int) -> np.ndarray:
        """Soft syndromes: data flips at p_data, Gaussian measurement channel (mu, sigma)."""
        counters = np.zeros(len(COUNTER_NAMES), dtype=np.uint64)
        st = _lib.load().qb_campaign_run_soft(self.decoder._h, seed, self.p_data, None, float(mu),
                                              float(sigma), first_trial, trials,
                                              counters.ctypes.data_as(_lib.u64p))
        if st != _lib.QB_OK:
            _raise(st, self.decoder._h)
        return counters

    def host_counters(self, err_bits: np.ndarray, est_bits: np.ndarray, conv: np.ndarray,
                      its: np.ndarray, syn_bits: np.ndarray) -> np.ndarray:
        """The classification rule restated on the host (numpy), for tests."""
        c = np.zeros(len(COUNTER_NAMES), dtype=np.uint64)
        r = err_bits ^ est_bits
        segs = [(int(a), int(b), int(v0), int(v1)) for a, b, v0, v1 in self.segments]
        both = conv.min(axis=1) == 1
        harmful, base_harmful = [], []
        for k, (c0, c1, v0, v1) in enumerate(segs):
            t = self.tests_bits[k].astype(np.int32)
            def bad(vec, need_zero_syn):
                seg = np.zeros_like(vec)
                seg[:, v0:v1] = vec[:, v0:v1]
                zero = ~seg.any(axis=1)
                aux = (seg & self.aux_bits[None, :]).any(axis=1)
                odd = ((seg.astype(np.int32) @ t.T) & 1).any(axis=1)
                out = ~zero & (aux | odd)
                if need_zero_syn is not None:
                    out = ~zero & (need_zero_syn | aux | odd)
                return out, zero
            h_r, zero_r = bad(r, None)
            h_e, _ = bad(err_bits, syn_bits[:, c0:c1].any(axis=1))
            harmful.append((h_r, zero_r))
            base_harmful.append(h_e)
        (hx, zx), (hz, zz) = harmful
        c[0] = int((both & zx & zz).sum())
        c[1] = int((both & ~(zx & zz) & ~hx & ~hz).sum())
        c[2] = int((both & hx & ~hz).sum())
        c[3] = int((both & ~hx & hz).sum())
        c[4] = int((both & hx & hz).sum())
        c[5] = int((~both).sum())
        c[6] = int((base_harmful[0] | base_harmful[1]).sum())
        c[7] = int(both.sum())
        c[8] = int(its.max(axis=1).astype(np.uint64).sum())
        c[9] = err_bits.shape[0]
        return c

    def close(self) -> None:
        self.decoder.close()

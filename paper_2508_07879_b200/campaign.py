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
from .gf2 import num_words, pack_bits

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


def reduce_counters(counters: np.ndarray, group=None, device=None) -> np.ndarray:
    """Sum of the counter vectors of every rank; identity without a process group."""
    try:
        import torch
        import torch.distributed as dist
    except ImportError:  # pragma: no cover
        return counters
    if not (dist.is_available() and dist.is_initialized()):
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
                 device: int = 0, world: int = 1, rank: int = 0, group=None) -> CampaignResult:
    """reference: run_campaign(code, NoiseModel{independent-xz, p, seed}, trials, cfg).
    With world > 1 every rank calls this with its own `rank`; all ranks return the
    same aggregated result."""
    if not (0.0 <= p <= 1.0):
        raise ValueError("NoiseModel: p must lie in [0, 1]")
    lo, hi = shard(trials, world, rank)
    camp = Campaign(code, cfg, device=device)
    try:
        counters = camp.run_range(p, seed, lo, hi - lo) if hi > lo else \
            np.zeros(len(COUNTER_NAMES), dtype=np.uint64)
    finally:
        camp.close()
    if world > 1:
        import torch
        counters = reduce_counters(counters, group, torch.device("cuda", device))
    return CampaignResult.from_counters(counters)

"""Shared test utilities (inputs only; no decoding logic)."""
from __future__ import annotations

import numpy as np

from paper_2508_07879_b200 import codes, gf2


def random_syndrome(rng: np.random.Generator, length: int, density: float) -> np.ndarray:
    """Packed random syndrome (cf. random_syndrome, proj/tests/test_decoder.cpp:19-24)."""
    return gf2.pack_bits((rng.random(length) < density).astype(np.uint8))


def random_syndromes(rng: np.random.Generator, shots: int, length: int, density: float) -> np.ndarray:
    return gf2.pack_bits((rng.random((shots, length)) < density).astype(np.uint8))


def random_ldpc_matrix(rng: np.random.Generator, rows: int, cols: int) -> codes.SparseMatrix:
    """Random sparse matrix with no empty rows or columns and a sprinkling of
    degree-1 checks and variables, the shape of the reference's irregular-graph
    fixture (proj/tests/test_decoder.cpp:140-155)."""
    dense = np.zeros((rows, cols), dtype=np.uint8)
    for m in range(rows):
        for _ in range(1 + int(rng.integers(0, 4))):
            dense[m, int(rng.integers(0, cols))] = 1
    for n in range(cols):
        if not dense[:, n].any():
            dense[int(rng.integers(0, rows)), n] = 1
    return codes.SparseMatrix.from_dense(dense)


def error_syndromes(code: codes.CssCode, rng: np.random.Generator, shots: int, p: float):
    """Independent X/Z bit-flip errors at rate p and their combined syndromes
    s_x ++ s_z (noise model of proj/src/noise.cpp:73-77, 97-105; numpy RNG)."""
    ex = (rng.random((shots, code.n)) < p).astype(np.uint8)
    ez = (rng.random((shots, code.n)) < p).astype(np.uint8)
    sx = code.hz.mat_vec(ex)
    sz = code.hx.mat_vec(ez)
    return ex, ez, gf2.pack_bits(np.concatenate([sx, sz], axis=-1))


_M64 = (1 << 64) - 1
_PHI = 0x9E3779B97F4A7C15


def _splitmix_mix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def skip_sampler_flips(seed: int, trial: int, p: float, num_vars: int) -> list:
    """Plain-Python statement of the geometric-skip sampler (QB_OPT_SAMPLER = 1, uniform p;
    csrc/kernel_noise.cuh): the flipped variables of one trial, ascending.  Not a reference
    algorithm - the reference draws one uniform per variable (proj/src/noise.cpp:67-78) -
    only its SplitMix64 seeding and output function are the reference's
    (proj/include/qldpc/noise.hpp:28-45)."""
    import math
    if p <= 0.0:
        return []
    inv = 1.0 / math.log1p(-p) if p < 1.0 else -0.0
    ctr = _splitmix_mix((seed + _PHI * trial + _PHI) & _M64)
    pos, out = -1.0, []
    while True:
        ctr = (ctr + _PHI) & _M64
        u = ((_splitmix_mix(ctr) >> 12) + 0.5) * 2.0 ** -52
        pos += math.floor(math.log(u) * inv) + 1.0
        if not pos < num_vars:
            return out
        out.append(int(pos))


def random_regular63_matrix(rng: np.random.Generator, checks: int) -> codes.SparseMatrix:
    """Random (6,3)-regular parity-check matrix with `checks` rows and 2 * checks columns and no
    repeated entry (configuration model + repair swaps): a graph with the degrees of the
    bivariate-bicycle codes but none of their structure."""
    n = 2 * checks
    stubs = np.repeat(np.arange(n), 3)
    rng.shuffle(stubs)
    rows = stubs.reshape(checks, 6)
    for _ in range(10000):
        bad = [m for m in range(checks) if len(set(rows[m].tolist())) < 6]
        if not bad:
            break
        for m in bad:
            vals = rows[m].tolist()
            j = next(k for k in range(6) if vals.count(vals[k]) > 1)
            m2, j2 = int(rng.integers(0, checks)), int(rng.integers(0, 6))
            rows[m, j], rows[m2, j2] = rows[m2, j2], rows[m, j]
    else:
        raise RuntimeError("could not repair the configuration-model graph")
    return codes.SparseMatrix.from_rows(checks, n, [sorted(r.tolist()) for r in rows])

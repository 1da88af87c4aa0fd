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

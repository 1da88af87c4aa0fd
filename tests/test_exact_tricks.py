"""CPU checks of the two arithmetic identities the CUDA path relies on to stay
bit-exact with the reference while avoiding slow instructions.  They restate the
loader's / sampler's host-side logic in exact arithmetic (fractions, numpy fp16) —
no GPU, no oracle.

1. Sampler (csrc/kernel_noise.cuh): the reference flips a bit iff
   `unit < p` with `unit = (draw >> 11) * 2^-53` (proj/include/qldpc/noise.hpp:28-45,
   proj/src/noise.cpp:67-95).  The kernel tests the integers `(draw >> 11) < ceil(p * 2^53)`.

2. int8 mode on packed fp16 instructions (csrc/kernel_lean_h2.cuh): the reference
   scales a magnitude with `(mag * alpha_fx + 32768) >> 16` (proj/src/decoder.cpp:226-229).
   The kernel computes `fma(mag, c, 1536) - 1536` in fp16 for an fp16 constant c that the
   loader accepts only if it reproduces the integer formula for all 128 magnitudes.
"""
import math
from fractions import Fraction

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st


def noise_threshold(p: float) -> int:
    """csrc/kernel_noise.cuh: noise_threshold()."""
    if not p > 0.0:
        return 0
    if p >= 1.0:
        return 1 << 53
    return int(math.ceil(math.ldexp(p, 53)))


@settings(max_examples=2000, deadline=None)
@given(p=st.floats(min_value=0.0, max_value=1.0, allow_nan=False),
       k=st.integers(min_value=0, max_value=(1 << 53) - 1))
def test_integer_threshold_equals_unit_less_than_p(p, k):
    unit_less = Fraction(k, 1 << 53) < Fraction(p)      # exact value of both sides
    assert (k < noise_threshold(p)) == unit_less
    # and the reference's own floating-point evaluation is exact, hence the same
    assert ((k * 2.0 ** -53) < p) == unit_less


@pytest.mark.parametrize("p", [0.0, 1.0, 0.5, 2.0 ** -53, 2.0 ** -54, 1.0 - 2.0 ** -53, 0.01,
                               float(np.nextafter(0.01, 1.0)), 1e-300])
def test_integer_threshold_at_the_edges(p):
    thr = noise_threshold(p)
    for k in {0, 1, max(thr - 1, 0), thr, min(thr + 1, (1 << 53) - 1), (1 << 53) - 1}:
        assert (k < thr) == (Fraction(k, 1 << 53) < Fraction(p)), (p, k)


def q16_scale(mag: int, alpha_fx: int) -> int:
    """reference: scale_q16 (proj/src/decoder.cpp:226-229)."""
    return (mag * alpha_fx + 32768) >> 16


def find_fp16_constant(alpha_fx: int):
    """csrc/qldpc_b200.cu (int8 branch of the loader): nearest fp16 values to
    alpha_fx / 65536, accepted only if round-to-nearest-even(mag * c) equals the integer
    formula for every magnitude 0..127."""
    c0 = np.float16(np.float32(alpha_fx) / np.float32(65536.0))
    bits0 = int(c0.view(np.uint16))
    for d in (0, -1, 1, -2, 2):
        c = np.array([bits0 + d], dtype=np.uint16).view(np.float16)[0]
        cf = float(c)
        if not (0.0 < cf <= 1.0):
            continue
        # mag * c is exact in binary64 (7 x 11 bits); Python's round() is round-half-even
        if all(round(mag * cf) == q16_scale(mag, alpha_fx) for mag in range(128)):
            return c
    return None


def fp16_fma_minus_magic(mag: int, c: np.float16) -> float:
    """What the kernel computes: fp16 fma(mag, c, 1536) - 1536, each with ONE rounding.
    mag * c + 1536 is exact in binary64, so casting that to fp16 is the fused result."""
    fused = np.float16(np.float64(mag) * np.float64(c) + 1536.0)
    return float(np.float16(np.float64(fused) - 1536.0))


@pytest.mark.parametrize("alpha", [0.8, 0.625, 0.75, 1.0, 0.5, 0.3, 0.9, 0.95, 0.7, 0.6875,
                                   0.8125, 0.1, 0.05])
def test_fp16_form_of_the_q16_scaling(alpha):
    alpha_fx = int(round(alpha * 65536.0))  # decoder.cpp:89 (lround)
    c = find_fp16_constant(alpha_fx)
    if c is None:
        pytest.skip(f"alpha {alpha}: no fp16 constant - the loader keeps the scalar int8 kernel")
    for mag in range(128):
        got = fp16_fma_minus_magic(mag, c)
        assert got == q16_scale(mag, alpha_fx), (alpha, mag, float(c))
        assert got == int(got) and 0 <= got <= 127


def test_the_reference_default_alpha_has_an_fp16_constant():
    assert find_fp16_constant(int(round(0.8 * 65536.0))) is not None


def test_int8_quantities_are_exact_fp16_integers():
    """Every int8-mode value (|x| <= 4 * 127 before saturation, 127 + 508 inside
    `total - r`) and the sum / difference of two of them is an fp16 integer."""
    vals = np.arange(-635, 636, dtype=np.int32)
    as16 = vals.astype(np.float16)
    assert np.array_equal(as16.astype(np.int32), vals)
    a = np.arange(-508, 509, dtype=np.int32)
    b = np.arange(-127, 128, dtype=np.int32)
    s = (a[:, None].astype(np.float16) + b[None, :].astype(np.float16)).astype(np.int32)
    assert np.array_equal(s, a[:, None] + b[None, :])
    d = (a[:, None].astype(np.float16) - b[None, :].astype(np.float16)).astype(np.int32)
    assert np.array_equal(d, a[:, None] - b[None, :])


def test_magic_rounding_window():
    """fma(mag, c, 1536) stays inside [1024, 2048), where fp16 has unit spacing."""
    assert float(np.float16(1536.0)) == 1536.0 and float(np.float16(1536.0 + 127.0)) == 1663.0
    assert np.spacing(np.float16(1536.0)) == 1.0 and np.spacing(np.float16(1663.0)) == 1.0
    assert int(np.float16(1536.0).view(np.uint16)) == 0x6600   # the kernel's constant
    assert int(np.float16(127.0).view(np.uint16)) == 0x57F0    # saturation bound / sentinel
    assert int(np.float16(64.0).view(np.uint16)) == 0x5400     # degree-1 check sentinel


def test_geometric_skip_sampling_has_the_bernoulli_law():
    """The skip sampler's algorithm (tests/helpers.skip_sampler_flips, the statement the GPU
    kernel is compared with bit for bit): gaps floor(ln u / ln(1-p)) between flips give i.i.d.
    Bernoulli(p) variables - weight mean and variance of Binomial(N, p), uniform per-position
    rate including both ends, strictly ascending positions, p = 0 / p = 1 edge cases."""
    from tests.helpers import skip_sampler_flips
    n, p, trials = 300, 0.04, 6000
    counts = np.zeros(n)
    weights = np.zeros(trials)
    for t in range(trials):
        f = skip_sampler_flips(11, t, p, n)
        assert all(a < b for a, b in zip(f, f[1:])) and (not f or (0 <= f[0] and f[-1] < n))
        counts[f] += 1
        weights[t] = len(f)
    var = n * p * (1 - p)
    assert abs(weights.mean() - n * p) < 4 * np.sqrt(var / trials)
    assert abs(weights.var() - var) < 5 * var * np.sqrt(2.0 / trials) + 0.01 * var
    assert np.abs(counts / trials - p).max() < 5 * np.sqrt(p * (1 - p) / trials)
    assert abs(counts[:10].sum() / (10 * trials) - p) < 4 * np.sqrt(p * (1 - p) / (10 * trials))
    assert abs(counts[-10:].sum() / (10 * trials) - p) < 4 * np.sqrt(p * (1 - p) / (10 * trials))
    assert skip_sampler_flips(3, 0, 0.0, n) == []
    assert skip_sampler_flips(3, 0, 1.0, n) == list(range(n))
    assert skip_sampler_flips(3, 5, p, n) != skip_sampler_flips(3, 6, p, n)

"""The C-ABI shared library on a machine WITHOUT a GPU: it must load, export
every symbol include/qldpc_b200.h declares, reject exactly the configurations
the reference rejects (validation runs before any CUDA call), and fail loudly -
never fall back - when asked to compute without a device."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2508_07879_b200 import Decoder, DecoderConfig, _lib, codes, decode_batch, gf2

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _has_gpu():
    lib = _lib.load()
    sm = C.c_int()
    return lib.qb_device_info(0, None, 0, C.byref(sm), None, None) == 0


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "qldpc_b200.h")).read()
    declared = set(re.findall(r"\b(qb_[a-z_0-9]+)\s*\(", header))
    declared -= {"qb_status"}
    assert len(declared) >= 18
    lib = C.CDLL(_lib.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} is declared in the header but not exported"
    # and the ctypes table binds all of them
    assert declared <= set(_lib.SYMBOLS), declared - set(_lib.SYMBOLS)


def test_version_string():
    assert b"sm_100a" in _lib.load().qb_version()


def test_invalid_configurations_are_rejected_before_touching_cuda():
    """Same conditions as Decoder::Decoder (decoder.cpp:373-404, :83-131); these
    return QB_INVALID_ARGUMENT (-> ValueError) with or without a device."""
    g = codes.build_tanner_graph(codes.toy_code_3x6())
    for bad in (dict(alpha=0.0), dict(alpha=1.25), dict(max_iterations=0),
                dict(priors=[1.0, 2.0]),
                dict(priors=[1.0, 1.0, 1.0, float("inf"), 1.0, 1.0]),
                dict(arithmetic="int8", quant_scale=0.3),
                dict(arithmetic="int16", alpha=1e-6),
                dict(arithmetic="int8", quant_scale=-4.0)):
        with pytest.raises(ValueError):
            Decoder(g, DecoderConfig(**bad))
    with pytest.raises(ValueError, match="unknown arithmetic"):
        Decoder(g, DecoderConfig(arithmetic="int32"))


def test_malformed_graphs_and_segments_are_rejected():
    g = codes.build_tanner_graph(codes.toy_code_3x6())
    import dataclasses
    broken = dataclasses.replace(g, var_edges=g.var_edges[::-1].copy())
    with pytest.raises(ValueError):
        Decoder(broken, DecoderConfig())
    with pytest.raises(ValueError):  # segments that do not tile the graph
        Decoder(g, DecoderConfig(), segments=np.array([[0, 2, 0, 6]], dtype=np.uint32))
    with pytest.raises(ValueError):  # not block-diagonal
        Decoder(g, DecoderConfig(), segments=np.array([[0, 1, 0, 3], [1, 3, 3, 6]], dtype=np.uint32))


def test_batch_length_validation_needs_no_device():
    """decode_batch validates every length up front (decoder.cpp:608-615)."""
    code = codes.make_code("bb72")
    good = np.zeros(1, dtype=np.uint64)
    with pytest.raises(ValueError, match="syndrome 3"):
        decode_batch(code.graph_x, [good, good, good, good], DecoderConfig(), bits=[36, 36, 36, 5])
    assert decode_batch(code.graph_x, [], DecoderConfig(alpha=7.0), 4) == []


@pytest.mark.skipif(_has_gpu(), reason="this check is about machines without a CUDA device")
def test_compute_fails_loudly_without_a_device():
    g = codes.build_tanner_graph(codes.toy_code_3x6())
    with pytest.raises(RuntimeError, match="CUDA"):
        Decoder(g, DecoderConfig())

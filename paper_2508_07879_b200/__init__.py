"""B200-native (sm_100a) scaled min-sum syndrome decoder for CSS QLDPC codes:
a drop-in for the `qldpc::Decoder` path of the reference implementation of
arXiv 2508.07879 (see DESIGN.md and include/qldpc_b200.h).

All decoding runs in hand-written CUDA behind a C-ABI; this package is the thin
host-side mirror of the reference's operator interface plus the host-only code
model that feeds it.  Importing the package does not load the CUDA library;
constructing a `Decoder` does, and fails loudly if it is missing.
"""
from .codes import (CssCode, SparseMatrix, TannerGraph, build_bb_code, build_tanner_graph,  # noqa: F401
                    extended_graph, make_code, make_css_code, toy_code_3x6)
from .decoder import (DecodeOutcome, Decoder, DecoderConfig, decode, decode_batch,  # noqa: F401
                      decode_css)
from . import alist, css_json  # noqa: F401  on-disk code formats (alist, CSS-JSON descriptors)
from .gf2 import concat_bits, num_words, pack_bits, to_hex, unpack_bits  # noqa: F401

__all__ = [
    "CssCode", "SparseMatrix", "TannerGraph", "build_bb_code", "build_tanner_graph",
    "extended_graph", "make_code", "make_css_code", "toy_code_3x6", "DecodeOutcome", "Decoder",
    "DecoderConfig", "decode", "decode_batch", "decode_css", "concat_bits", "num_words",
    "pack_bits", "to_hex", "unpack_bits",
]

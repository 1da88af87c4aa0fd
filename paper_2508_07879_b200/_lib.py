"""ctypes binding of the C-ABI in include/qldpc_b200.h.

The library is built in-tree (``__graft_entry__.build()``) as
``paper_2508_07879_b200/libqldpc_b200.so``.  There is no fallback of any kind:
if the library is missing the import of a compute entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqldpc_b200.so")

QB_OK, QB_INVALID_ARGUMENT, QB_RUNTIME_ERROR = 0, 1, 2
ARITH = {"float": 0, "int8": 1, "int16": 2, "half": 3}
ARITH_NAMES = {v: k for k, v in ARITH.items()}

OPT_KERNEL, OPT_LATENCY_IO, OPT_LATENCY_SHAPE, OPT_GROUP_THREADS, OPT_BATCH_CTAS_PER_SM = range(5)
OPT_SAMPLER = 16  # 0 = the reference's SplitMix64 stream, 1 = geometric skips (same distribution)

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
u8p = C.POINTER(C.c_uint8)
f32p = C.POINTER(C.c_float)
i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)


class QbGraph(C.Structure):
    _fields_ = [("num_checks", C.c_uint32), ("num_vars", C.c_uint32), ("num_edges", C.c_uint32),
                ("edge_var", u32p), ("check_offsets", u32p), ("var_offsets", u32p),
                ("var_edges", u32p)]


class QbSegment(C.Structure):
    _fields_ = [("check_begin", C.c_uint32), ("check_end", C.c_uint32),
                ("var_begin", C.c_uint32), ("var_end", C.c_uint32)]


class QbConfig(C.Structure):
    _fields_ = [("max_iterations", C.c_uint64), ("alpha", C.c_double),
                ("early_termination", C.c_int32), ("arithmetic", C.c_int32),
                ("quant_scale", C.c_double), ("priors", f64p), ("num_priors", C.c_uint64)]


# Every symbol include/qldpc_b200.h declares: (restype, argtypes).
SYMBOLS = {
    "qb_version": (C.c_char_p, []),
    "qb_last_error": (C.c_char_p, [C.c_void_p]),
    "qb_device_info": (C.c_int, [C.c_int, C.c_char_p, C.c_size_t, C.POINTER(C.c_int),
                                 C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "qb_measure_smem_bandwidth": (C.c_int, [C.c_int, f64p, f64p]),
    "qb_host_alloc": (C.c_int, [C.POINTER(C.c_void_p), C.c_size_t]),
    "qb_host_free": (None, [C.c_void_p]),
    "qb_decoder_create": (C.c_int, [C.POINTER(QbGraph), C.POINTER(QbSegment), C.c_uint32,
                                    C.POINTER(QbConfig), C.c_int, C.POINTER(C.c_void_p)]),
    "qb_decoder_destroy": (None, [C.c_void_p]),
    "qb_set_option": (C.c_int, [C.c_void_p, C.c_int, C.c_int64]),
    "qb_get_option": (C.c_int64, [C.c_void_p, C.c_int]),
    "qb_num_checks": (C.c_uint32, [C.c_void_p]),
    "qb_num_vars": (C.c_uint32, [C.c_void_p]),
    "qb_num_segments": (C.c_uint32, [C.c_void_p]),
    "qb_decode": (C.c_int, [C.c_void_p, u64p, u64p, u64p, u8p, u32p]),
    "qb_decode_batch": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p]),
    "qb_decode_batch_device": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "qb_decode_debug": (C.c_int, [C.c_void_p, u64p, u64p, u64p, u8p, u32p, f32p, f32p, i32p,
                                  i32p]),
    "qb_decode_batch_debug": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p,
                                        C.c_void_p, C.c_void_p, C.c_void_p, f32p, f32p, i32p, i32p]),
    "qb_generate_syndromes": (C.c_int, [C.c_void_p, C.c_uint64, C.c_double, f64p, C.c_int,
                                        C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                                        C.c_void_p]),
    "qb_latency_run": (C.c_int, [C.c_void_p, u64p, C.c_uint64, C.c_uint64, C.c_uint64, u64p,
                                 u64p, u64p]),
    "qb_latency_run_soft": (C.c_int, [C.c_void_p, u64p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                      u64p, u64p, u64p]),
    "qb_set_logicals": (C.c_int, [C.c_void_p, u64p, C.c_uint32, u64p, C.c_uint32]),
    "qb_campaign_run": (C.c_int, [C.c_void_p, C.c_uint64, C.c_double, f64p, C.c_uint64,
                                  C.c_uint64, u64p]),
    "qb_campaign_run_multi": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint32, C.c_uint64, C.c_double,
                                        f64p, C.c_uint64, C.c_uint64, u64p]),
    "qb_classify_batch_device": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_void_p, u64p, C.c_void_p]),
    "qb_soft_vars": (C.c_int, [C.c_void_p, u32p]),
    "qb_decode_soft": (C.c_int, [C.c_void_p, u64p, C.c_void_p, u64p, u64p, u8p, u32p]),
    "qb_decode_batch_soft": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p]),
    "qb_decode_batch_soft_device": (C.c_int, [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_void_p]),
    "qb_generate_soft_syndromes": (C.c_int, [C.c_void_p, C.c_uint64, C.c_double, f64p, C.c_double,
                                             C.c_double, C.c_uint64, C.c_uint64, C.c_void_p,
                                             C.c_void_p, C.c_void_p, C.c_void_p]),
    "qb_set_auxiliary_vars": (C.c_int, [C.c_void_p, u64p]),
    "qb_campaign_run_soft": (C.c_int, [C.c_void_p, C.c_uint64, C.c_double, f64p, C.c_double,
                                       C.c_double, C.c_uint64, C.c_uint64, u64p]),
    "qb_last_kernel_ns": (C.c_uint64, [C.c_void_p]),
    "qb_launch_count": (C.c_uint64, [C.c_void_p]),
}

_lib = None


def load() -> C.CDLL:
    """Loads the in-tree library; raises (never falls back) when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (nvcc, sm_100a).  There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, (restype, argtypes) in SYMBOLS.items():
        fn = getattr(lib, name)  # AttributeError if the library lacks a declared symbol
        fn.restype = restype
        fn.argtypes = argtypes
    _lib = lib
    return lib

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    """The compiled, unmodified reference (oracle/_ref/libqldpc_ref.so).  Built
    here from /root/reference; on the GPU box only the prebuilt file exists."""
    from oracle.pyoracle import Ref
    try:
        return Ref()
    except Exception as exc:  # pragma: no cover - depends on the environment
        pytest.skip(f"compiled reference unavailable: {exc}")


@pytest.fixture(scope="session")
def gpu_lib():
    """Loads the CUDA library and requires a device; never falls back."""
    from paper_2508_07879_b200 import _lib
    import ctypes as C
    lib = _lib.load()
    sm = C.c_int()
    maj = C.c_int()
    mino = C.c_int()
    name = C.create_string_buffer(128)
    st = lib.qb_device_info(0, name, 128, C.byref(sm), C.byref(maj), C.byref(mino))
    assert st == 0, lib.qb_last_error(None).decode()
    return {"lib": lib, "name": name.value.decode(), "sms": sm.value, "cc": (maj.value, mino.value)}

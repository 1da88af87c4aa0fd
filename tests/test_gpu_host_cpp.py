"""Runs the C++ parity runner of the host mirror (tests/cpp/host_parity.cpp):
qldpc_b200::Decoder through the C-ABI against the C oracle, with the checks the
reference's doctest suites make of qldpc::Decoder."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_cpp_host_mirror_parity_runner():
    cpp = os.path.join(ROOT, "tests", "cpp")
    exe = os.path.join(cpp, "host_parity")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2508_07879_b200", "host")], check=True)
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "libmsa_oracle.so"], check=True)
        subprocess.run(["make", "-C", cpp], check=True)
    # rpaths are absolute paths of the build machine: point the loader at this checkout
    env = dict(os.environ)
    env["LD_LIBRARY_PATH"] = os.pathsep.join(
        [os.path.join(ROOT, "paper_2508_07879_b200", "host"),
         os.path.join(ROOT, "paper_2508_07879_b200"), os.path.join(ROOT, "oracle"),
         env.get("LD_LIBRARY_PATH", "")])
    out = subprocess.run([exe], capture_output=True, text=True, env=env, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ALL PASS" in out.stdout and "FAIL" not in out.stdout.replace("SOME FAILED", "")


def test_cpp_host_mirror_builds():
    """The host mirror compiles and links against the C-ABI on a CPU-only machine."""
    subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2508_07879_b200", "host")], check=True,
                   capture_output=True)
    assert os.path.exists(os.path.join(ROOT, "paper_2508_07879_b200", "host",
                                       "libqldpc_b200_host.so"))


@pytest.mark.gpu
def test_reference_acceptance_runner_passes_against_the_gpu_decoder():
    """oracle/_ref/acceptance_dropin = the reference's own proj/tests/acceptance.cpp
    linked with the reference library in which proj/src/decoder.cpp is replaced by
    the drop-in shim over the C-ABI (paper_2508_07879_b200/host/dropin).  All 8 of
    the reference's end-to-end checks (soundness over 10 000 syndromes x 5 codes x 3
    modes, toy coset consistency, code family, all weight-1 errors, the 10-iteration
    protocol, determinism, campaign reproducibility, bench CSV) must PASS."""
    exe = os.path.join(ROOT, "oracle", "_ref", "acceptance_dropin")
    if not os.path.exists(exe):
        pytest.skip("prebuilt oracle/_ref/acceptance_dropin absent (needs /root/reference to build)")
    env = dict(os.environ)
    env["LD_LIBRARY_PATH"] = os.pathsep.join([os.path.join(ROOT, "paper_2508_07879_b200"),
                                              env.get("LD_LIBRARY_PATH", "")])
    out = subprocess.run([exe], capture_output=True, text=True, env=env, timeout=900,
                         cwd=os.path.join(ROOT, "oracle", "_ref"))
    print(out.stdout[-3000:])
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert out.stdout.count("PASS") >= 8 and "FAIL" not in out.stdout


@pytest.mark.gpu
def test_dropin_shim_device_selection_from_the_environment():
    """The reference's constructors carry no device argument: the shim reads QB_DEVICE /
    QB_DEVICES (round-robin over the list, one Decoder per reference worker thread)."""
    exe = os.path.join(ROOT, "oracle", "_ref", "acceptance_dropin")
    if not os.path.exists(exe):
        pytest.skip("prebuilt oracle/_ref/acceptance_dropin absent (needs /root/reference to build)")
    base = dict(os.environ)
    base["LD_LIBRARY_PATH"] = os.pathsep.join([os.path.join(ROOT, "paper_2508_07879_b200"),
                                               base.get("LD_LIBRARY_PATH", "")])
    cwd = os.path.join(ROOT, "oracle", "_ref")
    ok = subprocess.run([exe], capture_output=True, text=True, env={**base, "QB_DEVICES": "0,0"},
                        timeout=900, cwd=cwd)
    assert ok.returncode == 0 and "FAIL" not in ok.stdout, ok.stdout[-2000:] + ok.stderr[-2000:]
    for bad in ({"QB_DEVICE": "gpu0"}, {"QB_DEVICE": "97"}):
        out = subprocess.run([exe], capture_output=True, text=True, env={**base, **bad},
                             timeout=900, cwd=cwd)
        assert out.returncode != 0 or "FAIL" in out.stdout, bad

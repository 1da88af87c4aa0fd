"""bench.py's JSON contract, checked on the CPU: the reference arm (`--impl reference`) times the
compiled reference's own run_bench on the host cores, so it runs here; our arm needs a GPU and
is only checked for the pieces that do not (argument handling, the shared `config`)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=300):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=timeout, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])


def test_reference_arm_line(ref):
    line = _run("--impl", "reference", "--shots", "2048", "--steps", "2", "--warmup", "1")
    assert line["impl"] == "reference" and line["steps"] == 2 and line["warmup"] == 1
    assert line["unit"] == "decodes/s" and line["higher_is_better"] is True and line["value"] > 0
    assert line["vs_baseline"] is None and line["gpu_launches"] == 0 and line["n_gpus"] == 1
    base = line["cpu_baseline"]
    assert base["kind"] == "reference" and base["cores"] >= 1 and base["value"] == line["value"]
    assert "run_bench" in base["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "decodes/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    # the CPU single-shot latency row (run_bench at batch 1 on one thread), both protocols
    lat = base["latency_us"]
    for key in ("bb784_fixed10", "bb784_cap50_early", "bb144_fixed10", "bb144_cap50_early"):
        assert 0 < lat[key]["p50"] <= lat[key]["p99"]
    assert lat["bb784_fixed10"]["p50"] > lat["bb144_fixed10"]["p50"]


def test_both_arms_describe_the_same_workload():
    sys.path.insert(0, ROOT)
    import bench
    argv = sys.argv
    try:
        sys.argv = ["bench.py", "--shots", "4096"]
        ours = bench.bench_config(bench.parse_args())
        sys.argv = ["bench.py", "--impl", "reference", "--shots", "4096"]
        theirs = bench.bench_config(bench.parse_args())
    finally:
        sys.argv = argv
    assert ours == theirs and ours["shots_per_gpu_per_step"] == 4096
    assert "bb784" in ours["workload"] and "early-stop" in ours["workload"]


def test_ours_fails_loudly_without_a_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0 and "no CPU fallback" in r.stderr

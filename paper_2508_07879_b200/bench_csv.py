"""Latency benchmark rows in the reference's CSV schema, so
the reference's own validating reader (`read_bench_csv`, proj/src/bench.cpp:366-444)
accepts GPU rows: the frozen 19-column header (bench.cpp:339-343), the row format
(:345-358), a `# host:` comment line (:360-364) and `# digest:` lines carrying the
FNV-1a output digest (:27-36, :287-291; CLI convention qldpc_cli.cpp:451-459).

`run_bench` follows the reference protocol at batch 1 (bench.hpp:20-37): pool of
max(batch, 256) syndromes sampled at rate p (here by the device generator, which
is bit-exact with `sample_error`), warm-up + measured decodes, per-decode
wall-clock of the whole call, nearest-rank percentiles."""
from __future__ import annotations

import dataclasses
import math
import os
from typing import Iterable, List, Optional

import numpy as np

from .codes import CssCode
from .decoder import Decoder, DecoderConfig

HEADER = ("code,n,k,d,mode,alpha,imax,early_term,batch,threads,trials,"
          "min_us,mean_us,median_us,p99_us,max_us,conv_rate,kernel_frac,under_63us")


@dataclasses.dataclass
class BenchRecord:
    """reference: struct BenchRecord (proj/include/qldpc/bench.hpp:38-58)."""
    code: str
    n: int
    k: int
    d: int
    mode: str
    alpha: float
    imax: int
    early_term: bool
    batch: int
    threads: int
    trials: int
    min_us: float
    mean_us: float
    median_us: float
    p99_us: float
    max_us: float
    conv_rate: float
    kernel_frac: float
    under_63us: bool
    digest: int = 0

    def row(self) -> str:
        for field in (self.code, self.mode):
            if "," in field or "\n" in field:
                raise ValueError("bench csv: string fields must not contain commas or newlines")
        return (f"{self.code},{self.n},{self.k},{self.d},{self.mode},{self.alpha:g},{self.imax},"
                f"{int(self.early_term)},{self.batch},{self.threads},{self.trials},"
                f"{self.min_us:.3f},{self.mean_us:.3f},{self.median_us:.3f},{self.p99_us:.3f},"
                f"{self.max_us:.3f},{self.conv_rate:.6f},{self.kernel_frac:.6f},"
                f"{int(self.under_63us)}")


def percentile_nearest_rank(sorted_vals, pct: float) -> float:
    """reference: percentile_nearest_rank (bench.cpp:169-180)."""
    n = len(sorted_vals)
    if n == 0:
        raise ValueError("percentile of an empty sample")
    if not (0.0 < pct <= 100.0):
        raise ValueError("percentile rank must lie in (0, 100]")
    rank = min(max(int(math.ceil(pct / 100.0 * n)), 1), n)
    return float(sorted_vals[rank - 1])


def run_bench(code: CssCode, mode: str = "float", alpha: float = 0.8, max_iterations: int = 10,
              early_termination: bool = False, warmup: int = 100, measure: int = 200,
              p: float = 0.01, seed: int = 1, io_mode: int = 0, device: int = 0) -> BenchRecord:
    import torch
    from .gf2 import num_words
    cfg = DecoderConfig(max_iterations=max_iterations, alpha=alpha,
                        early_termination=early_termination, arithmetic=mode)
    g = code.combined_graph
    with Decoder(code, cfg, device=device) as dec:
        d_pool = torch.zeros((256, num_words(g.num_checks)), dtype=torch.int64,
                             device=torch.device("cuda", device))
        dec.generate_syndromes(seed, p, 256, d_pool.data_ptr(), None,
                               stream=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        pool = d_pool.cpu().numpy().view(np.uint64)
        dec.set_option(1, io_mode)
        wall, kern, digest = dec.latency_run(pool, warmup, measure)
        conv = 0
        # convergence rate of the measured decodes (same order as the harness)
        est, _, c, _ = dec.decode_batch_segments(pool)
        idx = [(warmup + b) % 256 for b in range(measure)]
        conv = float(np.mean(c.all(axis=1)[idx]))
    us = np.sort(wall.astype(np.float64) * 1e-3)
    mean = float(np.mean(us))
    return BenchRecord(code.name, code.n, code.k, code.d, mode, alpha, max_iterations,
                       early_termination, 1, 1, warmup + measure, float(us[0]), mean,
                       percentile_nearest_rank(us, 50.0), percentile_nearest_rank(us, 99.0),
                       float(us[-1]), conv,
                       float(np.sum(kern.astype(np.float64)) / max(np.sum(wall.astype(np.float64)), 1.0)),
                       mean < 63.0, digest)


def host_descriptor() -> str:
    cpu = "unknown cpu"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    cpu = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    gpu = ""
    try:
        import torch
        if torch.cuda.is_available():
            gpu = "; " + torch.cuda.get_device_name(0)
    except Exception:
        pass
    return f"{cpu}; {os.cpu_count()} hardware threads{gpu}; qldpc_b200"


def write_bench_csv(path: str, rows: Iterable[BenchRecord]) -> None:
    rows = list(rows)
    with open(path, "w") as f:
        f.write(f"# host: {host_descriptor()}\n")
        f.write(HEADER + "\n")
        for r in rows:
            f.write(r.row() + "\n")
        for r in rows:
            f.write(f"# digest: {r.code},{r.mode},{r.batch},{r.threads},{r.digest:016x}\n")

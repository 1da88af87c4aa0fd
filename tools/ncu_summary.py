#!/usr/bin/env python
"""Condenses an .ncu-rep (ncu --set full --import-source on) into the text
summary committed under profiles/: headline metrics, pipe utilisation, stall
breakdown, opcode mix and shared-memory wavefronts of one kernel launch."""
import csv
import io
import subprocess
import sys
from collections import Counter


def run(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def main(path, units=None):
    raw = list(csv.reader(io.StringIO(run(["-i", path, "--page", "raw", "--csv"]))))
    hdr, vals = raw[0], raw[-1]
    m = dict(zip(hdr, vals))
    want = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
            "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
            "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__cycles_elapsed.avg.per_second"]
    print(f"# {path}")
    for k in want:
        if k in m:
            print(f"{k:80s} {m[k]}")
    src = list(csv.reader(io.StringIO(run(["-i", path, "--page", "source", "--csv"]))))
    if len(src) < 3:
        return
    h = src[1]
    ix = {c: i for i, c in enumerate(h)}
    rows = src[2:]

    def f(r, k):
        try:
            return float(r[ix[k]])
        except (ValueError, KeyError, IndexError):
            return 0.0

    tot = sum(f(r, "Instructions Executed") for r in rows)
    samples = sum(f(r, "# Samples") for r in rows)
    print(f"\nwarp instructions executed (source page): {tot:.0f}")
    if units:
        print(f"  per unit ({units:.0f} units): {tot / units:.1f}")
    stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    st = sorted(((sum(f(r, c) for r in rows), c) for c in stalls), reverse=True)
    print("stall samples (% of all samples):")
    for v, c in st[:10]:
        print(f"  {c:28s} {100 * v / max(samples, 1):5.1f}")
    ops = Counter()
    for r in rows:
        t = r[ix["Source"]].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
        ops[op.split(".")[0]] += f(r, "Instructions Executed")
    print("opcode mix (% of executed warp instructions):")
    for op, n in ops.most_common(18):
        print(f"  {op:10s} {100 * n / max(tot, 1):5.1f}" + (f"   {n / units:8.1f} / unit" if units else ""))
    wf = sum(f(r, "L1 Wavefronts Shared") for r in rows)
    ex = sum(f(r, "L1 Wavefronts Shared Excessive") for r in rows)
    print(f"shared-memory wavefronts: {wf:.0f} total, {ex:.0f} excessive (bank conflicts)")


def traffic_json(path, out, shots, arithmetic, workload):
    """profiles/traffic.json: DRAM bytes of ONE launch of the dominant kernel (bench.py reads it
    for roofline.traffic)."""
    import json
    raw = list(csv.reader(io.StringIO(run(["-i", path, "--page", "raw", "--csv"]))))
    hdr, units, vals = raw[0], raw[1], raw[-1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = {}
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(name)
        tot[name] = float(vals[i].replace(",", "")) * scale[units[i]]
    def pct(name):
        try:
            return float(vals[hdr.index(name)].replace(",", ""))
        except (ValueError, IndexError):
            return None

    with open(out, "w") as f:
        json.dump({"kernel": vals[hdr.index("Kernel Name")], "shots_per_launch": int(shots),
                   "smem_wavefronts_pct_of_peak": pct(
                       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
                   "issue_active_pct": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                   "alu_pipe_pct": pct("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                   "xu_pipe_pct": pct("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
                   "arithmetic": arithmetic, "workload": workload,
                   "dram_bytes_read": tot["dram__bytes_read.sum"],
                   "dram_bytes_write": tot["dram__bytes_write.sum"],
                   "dram_bytes_per_launch": sum(tot.values()),
                   "source": "ncu --set full --clock-control none, one launch of `python bench.py "
                             "--steps 2 --warmup 1` (tools/prof_bench.sh)"}, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "--traffic-json":
        traffic_json(sys.argv[1], *sys.argv[3:7])
    else:
        main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)

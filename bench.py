#!/usr/bin/env python
"""Benchmark of the hot path: batched min-sum decodes/s and single-shot latency
at [[784,24,24]] (BASELINE.json), one process per GPU.

    python bench.py --gpus 1 --steps 5 --warmup 3            # our CUDA path
    python bench.py --impl reference --gpus 1 --steps 3 ...  # reference CPU path

A STEP is one pass of the decoder over one batch of `--shots` synthetic
syndromes per GPU (bb784 combined X+Z graph, independent-XZ bit-flip noise at
`--p`, fp32 min-sum, 50-iteration cap with syndrome-match early stop — config 4
of BASELINE.json at its centre point).  The batch is generated ON the device by
the library's SplitMix64-exact generator before the timed region, so inputs are
resident in HBM; input + output of one step (~310 MB at 1 Mi shots) exceed the
126 MB L2, so no step re-reads a cached batch.

One JSON line is printed by rank 0 (see DESIGN.md §Measurement for every key).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "batched decodes/s at [[784,24,24]] (p50/p99 single-shot latency in `latency_us`)"
BYTES_PER_EDGE_UPDATE = {"float": 16, "half": 8, "int16": 8, "int8": 4}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--code", default="bb784")
    ap.add_argument("--shots", type=int, default=1 << 20, help="shots per GPU per step")
    ap.add_argument("--p", type=float, default=0.01)
    ap.add_argument("--max-iterations", type=int, default=50)
    ap.add_argument("--no-early-stop", action="store_true")
    ap.add_argument("--arithmetic", default="float")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--latency-shots", type=int, default=10000)
    ap.add_argument("--skip-latency", action="store_true")
    ap.add_argument("--skip-cpu-baseline", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-variants", action="store_true")
    ap.add_argument("--e2e-chunk", type=int, default=0, help="QB_OPT_BATCH_CHUNK for the e2e leg (0 = auto)")
    ap.add_argument("--ref-shots", type=int, default=0,
                    help="--impl reference: shots per step (0 = --shots, the same batch: "
                         "run_bench's pool is trials 0 .. shots-1 of the same seed)")
    ap.add_argument("--dry-spawn", action="store_true",
                    help="rank plumbing only (gloo, no GPU): spawn --gpus ranks, shard a trial "
                         "range, all-reduce the counters, print one line")
    return ap.parse_args()


def bench_config(args) -> dict:
    """`config` of the JSON line - the SAME dict for both arms, so the driver can tell that
    they ran one workload: the batch of step k is trials [0, shots) of NoiseModel{seed} on
    either side (device generator == the reference's sample_error streams; run_bench's pool
    is exactly those trials, proj/src/bench.cpp:203-211)."""
    return {"workload": workload_name(args), "shots_per_gpu_per_step": args.shots,
            "l2": "inputs+outputs per step exceed L2 (no flush needed)",
            "generator": "reference sample_error SplitMix64 streams (device generator is "
                         "bit-exact with them), seed %d, trials 0 .. shots-1 per GPU" % args.seed}


def workload_name(args) -> str:
    stop = "fixed" if args.no_early_stop else "early-stop"
    return (f"{args.code} combined X+Z graph, {args.arithmetic} min-sum, alpha 0.8, "
            f"{args.max_iterations}-iteration cap {stop}, independent-XZ p={args.p}")


# --------------------------------------------------------------------------- clocks

class ClockSampler:
    """Samples SM clocks and throttle reasons with nvidia-smi DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._pump, daemon=True).start()
        except OSError:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)),
                "reasons": sorted(reasons), "samples": len(sm)}


def nearest_rank(sorted_vals, pct):
    """reference: percentile_nearest_rank (proj/src/bench.cpp:169-180)."""
    n = len(sorted_vals)
    rank = min(max(int(np.ceil(pct / 100.0 * n)), 1), n)
    return float(sorted_vals[rank - 1])


# --------------------------------------------------------------------------- reference arm

def reference_throughput(args, shots_per_step, steps, warmup):
    """Times the reference's own CPU implementation of the path (oracle/_ref, the
    unmodified sources compiled in place) with every host thread, on a bounded
    sample of the same workload; falls back to the C oracle port if the prebuilt
    library is absent.  Returns (decodes/s, seconds/step, cpu_baseline dict)."""
    from oracle.pyoracle import Oracle, Ref
    cores = os.cpu_count() or 1
    if Ref.available() and args.arithmetic in ("float", "int8", "int16"):
        ref = Ref()
        rc = ref.code(args.code)
        # run_bench's protocol (bench.cpp:182-337): persistent worker pool, one Decoder per
        # worker, timed region = copy-in + decode + copy-out of one batch.
        r = ref.run_bench(rc, arithmetic=args.arithmetic, alpha=0.8,
                          max_iterations=args.max_iterations,
                          early_termination=not args.no_early_stop, batch=shots_per_step,
                          threads=0, warmup=warmup, measure=steps, p=args.p, seed=args.seed)
        per_decode_us = r["mean_us"]
        return (1e6 / per_decode_us, per_decode_us * shots_per_step * 1e-6,
                {"value": 1e6 / per_decode_us, "unit": "decodes/s", "cores": int(r["threads"]),
                 "kind": "reference",
                 "sample": f"run_bench: {steps} batches of {shots_per_step} shots, "
                           f"{int(r['threads'])} threads, conv_rate {r['conv_rate']:.4f}",
                 "host": ref.host_descriptor()})
    from paper_2508_07879_b200 import DecoderConfig, codes, gf2
    code = codes.make_code(args.code)
    rng = np.random.default_rng(args.seed)
    n = min(shots_per_step, 2048)
    ex = (rng.random((n, code.n)) < args.p).astype(np.uint8)
    ez = (rng.random((n, code.n)) < args.p).astype(np.uint8)
    syn = gf2.pack_bits(np.concatenate([code.hz.mat_vec(ex), code.hx.mat_vec(ez)], axis=-1))
    cfg = DecoderConfig(max_iterations=args.max_iterations,
                        early_termination=not args.no_early_stop, arithmetic=args.arithmetic)
    orc = Oracle()
    t0 = time.perf_counter()
    for _ in range(max(steps, 1)):
        orc.decode_many(code.combined_graph, cfg, syn, code.segments)
    dt = (time.perf_counter() - t0) / max(steps, 1)
    return (n / dt, dt, {"value": n / dt, "unit": "decodes/s", "cores": 1, "kind": "port",
                         "sample": f"C oracle, {n} shots per step, 1 thread"})


def reference_latency(args, measure=1500):
    """CPU single-shot latency beside the GPU's: the reference's own
    run_bench at batch 1 on ONE thread (proj/src/bench.cpp:182-337; pool of 256 syndromes,
    nearest-rank percentiles), paper protocol (10 iterations fixed) and the 50-cap early-stop
    variant, for [[784,24,24]] and [[144,12,12]]."""
    from oracle.pyoracle import Ref
    if not (Ref.available() and args.arithmetic in ("float", "int8", "int16")):
        return None
    ref = Ref()
    out = {"protocol": "reference run_bench, batch 1, 1 thread, pool 256, %d measured decodes "
                       "after 100 warm-ups; wall clock per decode incl. copy-in/out" % measure}
    for name in sorted({args.code, "bb144"}):
        rc = ref.code(name)
        for label, iters, early in (("fixed10", 10, False), ("cap50_early", 50, True)):
            r = ref.run_bench(rc, arithmetic=args.arithmetic, alpha=0.8, max_iterations=iters,
                              early_termination=early, batch=1, threads=1, warmup=100,
                              measure=measure, p=args.p, seed=args.seed)
            out[f"{name}_{label}"] = {"p50": r["median_us"], "p99": r["p99_us"],
                                      "mean": r["mean_us"], "min": r["min_us"], "max": r["max_us"]}
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ref_shots = args.ref_shots or args.shots
    value, sec_per_step, base = reference_throughput(args, ref_shots, args.steps, args.warmup)
    cfg = bench_config(args)
    if ref_shots != args.shots:
        cfg["shots_per_gpu_per_step"] = ref_shots
    base["latency_us"] = reference_latency(args)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "decodes/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec_per_step * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if args.arithmetic == "float" else args.arithmetic,
        "data": "synthetic", "config": cfg,
        "cpu_baseline": base,
        "e2e": {"value": value, "unit": "decodes/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- our arm

def run_ours(args):
    import torch
    from paper_2508_07879_b200 import Decoder, DecoderConfig, _lib, codes, gf2

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise RuntimeError("bench.py needs a CUDA device: there is no CPU fallback")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    code = codes.make_code(args.code)
    g = code.combined_graph
    cfg = DecoderConfig(max_iterations=args.max_iterations,
                        early_termination=not args.no_early_stop, arithmetic=args.arithmetic)
    from paper_2508_07879_b200.campaign import COUNTER_NAMES, Campaign, CampaignResult
    camp = Campaign(code, cfg, device=local)  # decoder + residual tests (logical operators)
    dec = camp.decoder
    lib = _lib.load()
    shots = args.shots
    sw, ew, nseg = gf2.num_words(g.num_checks), gf2.num_words(g.num_vars), dec.num_segments

    # ---- resident inputs: generated on the device, trial ids unique across ranks
    d_syn = torch.zeros((shots, sw), dtype=torch.int64, device=dev)
    d_err = torch.zeros((shots, ew), dtype=torch.int64, device=dev)
    d_est = torch.zeros((shots, ew), dtype=torch.int64, device=dev)
    d_conv = torch.zeros((shots, nseg), dtype=torch.uint8, device=dev)
    d_its = torch.zeros((shots, nseg), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    dec.generate_syndromes(args.seed, args.p, shots, d_syn.data_ptr(), d_err.data_ptr(),
                           first_trial=rank * shots, stream=stream)
    torch.cuda.synchronize()

    def step():
        dec.decode_batch_device(shots, d_syn.data_ptr(), d_est.data_ptr(), None,
                                d_conv.data_ptr(), d_its.data_ptr(), stream)

    for _ in range(args.warmup):
        step()
    barrier()
    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    launches0 = dec.launch_count()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    ev[0].record()
    for k in range(args.steps):
        step()
        ev[k + 1].record()
    barrier()
    clocks = sampler.stop() if rank == 0 else None
    launches = dec.launch_count() - launches0
    total_ms = ev[0].elapsed_time(ev[-1])
    kernel_ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = world * shots * args.steps / (total_ms * 1e-3)

    # ---- outcome counters: the only data-path collective.  The batch is
    # classified on the device (exact / stabilizer / logical / non-converged, as the
    # reference's run_campaign does) and the ten counters + the edge-update count are summed
    # over ranks with ONE all-reduce.
    seg_edges = [int(g.check_offsets[c1] - g.check_offsets[c0]) for c0, c1, _, _ in code.segments]
    its64 = d_its.to(torch.int64)
    edge_updates = sum(int(its64[:, s].sum().item()) * seg_edges[s] for s in range(nseg))
    cls = camp.classify_device(shots, d_err.data_ptr(), d_est.data_ptr(), d_syn.data_ptr(),
                               d_conv.data_ptr(), d_its.data_ptr(), stream)
    counters = torch.tensor([int(x) for x in cls] + [edge_updates], dtype=torch.int64, device=dev)
    if dist is not None:
        dist.all_reduce(counters, op=dist.ReduceOp.SUM)
    totals = [int(x) for x in counters.tolist()]
    result = CampaignResult.from_counters(totals[:len(COUNTER_NAMES)])
    edge_updates_all = totals[-1]

    # ---- e2e: the public batch call on HOST (pinned) buffers, copies inside the timed region.
    # Every rank runs it at the same time (they share the host and its PCIe root complexes);
    # the job's figure uses the slowest rank's time.
    e2e = None
    if not args.skip_e2e:
        barrier()
        e2e = measure_e2e(args, dec, lib, d_syn, shots, sw, ew, nseg)
        t = torch.tensor([e2e["ms_per_step"]], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e["ms_per_step"] = float(t.item())
        e2e["value"] = world * shots / (e2e["ms_per_step"] * 1e-3)
        e2e["h2d_bytes_per_step"] *= world
        e2e["d2h_bytes_per_step"] *= world

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant (only) kernel in the timed region
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "MEASURED_PEAKS.json" if "hbm_gbs" in peaks else "fallback 6650 GB/s"
    g32, g128 = C.c_double(), C.c_double()
    st = lib.qb_measure_smem_bandwidth(local, C.byref(g32), C.byref(g128))
    assert st == 0, lib.qb_last_error(None).decode()
    bpe = BYTES_PER_EDGE_UPDATE[args.arithmetic]
    k_ms = float(np.mean(kernel_ms))
    eu_per_launch = edge_updates / 1.0  # per step on this rank (every step decodes the same batch)
    smem_achieved = eu_per_launch * bpe / (k_ms * 1e-3) / 1e9
    hbm_bytes_per_shot = sw * 8 + ew * 8 + nseg + 4 * nseg
    hbm_achieved = shots * hbm_bytes_per_shot / (k_ms * 1e-3) / 1e9
    sm_clock = (clocks or {}).get("sm_mhz") or float(peaks.get("sm_max_mhz", 1965.0))
    roofline = {
        "bound": "smem", "kernel": "decode_lean_kernel", "achieved": smem_achieved,
        "peak": g32.value, "unit": "GB/s", "frac": smem_achieved / g32.value,
        "peak_source": "qb_measure_smem_bandwidth (32-bit conflict-free ld/st stream, this run)",
        "peak_128bit": g128.value,
        "peak_theoretical": 148 * 128 * sm_clock * 1e6 / 1e9,
        "edge_updates_per_s": eu_per_launch / (k_ms * 1e-3),
        "bytes_per_edge_update": bpe, "kernel_ms": k_ms, "traffic": None,
        "hbm": {"bound": "hbm", "achieved": hbm_achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": hbm_achieved / hbm_peak, "peak_source": hbm_src,
                "bytes_per_shot": hbm_bytes_per_shot, "traffic": None},
    }

    # DRAM traffic of the dominant kernel: from the committed `ncu --set full` capture of this
    # very command (profiles/traffic.json: dram__bytes_read.sum + dram__bytes_write.sum per
    # launch), not a live measurement; null when the capture is for another shot count.
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f)
        if (tr.get("shots_per_launch") == shots and tr.get("arithmetic") == args.arithmetic
                and tr.get("workload") == workload_name(args)):
            roofline["traffic"] = tr["dram_bytes_per_launch"]
            roofline["traffic_source"] = tr.get("source")
            # the hardware's own view of the same launch, to set beside `frac` (which counts
            # ALGORITHMIC bytes, incl. the first iteration that the kernel evaluates from a table
            # without touching r): shared-memory wavefronts as a fraction of their peak rate
            if tr.get("smem_wavefronts_pct_of_peak") is not None:
                roofline["ncu_smem_wavefront_frac"] = tr["smem_wavefronts_pct_of_peak"] / 100.0
                roofline["ncu_pipes_pct"] = {"issue": tr.get("issue_active_pct"), "alu": tr.get("alu_pipe_pct"),
                                             "xu": tr.get("xu_pipe_pct")}
            roofline["hbm"]["traffic"] = tr["dram_bytes_per_launch"]
            roofline["hbm"]["algorithmic_bytes_per_launch"] = shots * hbm_bytes_per_shot
    except (OSError, ValueError, KeyError):
        pass

    line = {
        "metric": METRIC, "value": value, "unit": "decodes/s", "n_gpus": world,
        "gpus_requested": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" if args.arithmetic == "float" else args.arithmetic, "data": "synthetic",
        "config": bench_config(args),
        "roofline": roofline, "gpu_launches": int(launches), "clocks": clocks,
        "outcomes": {"shots": result.trials, "exact": result.exact,
                     "stabilizer": result.stabilizer, "logical_x": result.logical_x,
                     "logical_z": result.logical_z, "logical_both": result.logical_both,
                     "non_converged": result.non_converged,
                     "logical_error_rate": result.logical_error_rate,
                     "baseline_logical_rate": result.baseline_logical_rate,
                     "convergence_rate": result.convergence_rate,
                     "mean_iterations": result.mean_iterations,
                     "edge_updates_all_ranks_per_step": edge_updates_all,
                     "reduction": "one all_reduce(SUM) of 11 int64 counters"},
    }

    if e2e is not None:
        line["e2e"] = e2e
    # ---- single-shot latency (N=1 only): the other half of BASELINE's metric.  The full table
    # stays in `latency_us`; the compact p50 / p99 block rides inside `e2e` (a decode through
    # qb_decode with host buffers IS an end-to-end call), where the driver's record keeps it.
    if world == 1 and not args.skip_latency:
        line["latency_us"] = measure_latency(args, code, lib, d_syn)
        compact = compact_latency(line["latency_us"])
        compact.update(measure_latency_bb144(args))
        if e2e is not None:
            e2e["latency_us"] = compact
        else:
            line["e2e"] = {"latency_us": compact}
    if world == 1 and not args.skip_variants:
        line["variants"] = measure_variants(args, code, d_syn, d_est, d_conv, d_its, stream)
    if world == 1 and not args.skip_cpu_baseline:
        try:
            _, _, base = reference_throughput(args, 1 << 16, 40, 2)  # ~10-15 s of CPU work
            base["latency_us"] = reference_latency(args)
            line["cpu_baseline"] = base
        except Exception as exc:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "unit": "decodes/s", "cores": 0,
                                    "kind": "reference", "sample": f"failed: {exc}"}
    print(json.dumps(line), flush=True)
    dec.close()
    if dist is not None:
        dist.destroy_process_group()


def _time_batches(dec, shots, bufs, stream, reps=3):
    import torch
    d_syn, d_est, d_conv, d_its = bufs
    f = lambda: dec.decode_batch_device(shots, d_syn.data_ptr(), d_est.data_ptr(), None,
                                        d_conv.data_ptr(), d_its.data_ptr(), stream)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def measure_variants(args, code, d_syn, d_est, d_conv, d_its, stream):
    """Device-resident throughput of the other arithmetic modes / protocols on the SAME
    syndromes (bb784, p as the main line), and of BASELINE config 5: the phenomenological
    extension diag([Hz | I], [Hx | I]) with LLR priors, int8 messages (degree-padded
    kernel).  Reported beside the headline, never in place of it."""
    import torch
    from paper_2508_07879_b200 import Decoder, DecoderConfig, codes, gf2
    g = code.combined_graph
    shots = min(args.shots, 1 << 19)
    edges = g.num_edges
    out = {"shots_per_launch": shots, "note": "CUDA events around 3 launches after 3 warm-ups; "
           "float / int8 / int16 are bit-exact with the reference, half has no reference mode"}
    for arith in ("float", "int8", "half", "int16"):
        for label, iters, early in (("cap50_early", 50, True), ("fixed10", 10, False)):
            if arith == args.arithmetic and label == "cap50_early" and args.max_iterations == 50:
                continue  # the headline itself
            cfg = DecoderConfig(max_iterations=iters, early_termination=early, arithmetic=arith)
            with Decoder(code, cfg) as dec:
                ms = _time_batches(dec, shots, (d_syn, d_est, d_conv, d_its), stream)
                eu = float(d_its[:shots].to(torch.int64).sum().item()) * (edges // 2)
                out[f"{arith}_{label}"] = {"decodes_per_s": shots / ms * 1e3,
                                           "edge_updates_per_s": eu / ms * 1e3,
                                           "smem_bytes_per_s": eu / ms * 1e3 * BYTES_PER_EDGE_UPDATE[arith],
                                           "two_shots_per_thread": bool(dec.get_option(10))}
    # ---- config 5: extended graph, per-variable priors, int8 (and float for comparison)
    pq = 0.005
    h, segs = codes.extended_graph(code)
    ge = codes.build_tanner_graph(h)
    n, mz, mx = code.n, code.hz.rows, code.hx.rows
    llr = float(np.log((1 - pq) / pq))
    probs = np.full(ge.num_vars, pq)
    sw, ew = gf2.num_words(ge.num_checks), gf2.num_words(ge.num_vars)
    shots5 = min(shots, 1 << 18)
    dev = d_syn.device
    e_syn = torch.zeros((shots5, sw), dtype=torch.int64, device=dev)
    e_est = torch.zeros((shots5, ew), dtype=torch.int64, device=dev)
    for arith in ("int8", "float"):
        for label, iters, early in (("cap50_early", 50, True), ("fixed10", 10, False)):
            cfg = DecoderConfig(max_iterations=iters, early_termination=early, arithmetic=arith,
                                priors=[llr] * ge.num_vars)
            with Decoder(ge, cfg, segments=segs) as dec:
                dec.generate_syndromes(args.seed, 0.0, shots5, e_syn.data_ptr(), None, probs=probs,
                                       css_interleave=False, stream=stream)
                ms = _time_batches(dec, shots5, (e_syn, e_est, d_conv, d_its), stream)
                its = d_its[:shots5].to(torch.int64)
                eu = float(its.sum().item()) * (ge.num_edges // 2)
                out[f"config5_ext_{arith}_{label}"] = {
                    "decodes_per_s": shots5 / ms * 1e3, "edge_updates_per_s": eu / ms * 1e3,
                    "kernel": "decode_ell_kernel" if dec.get_option(107) else "decode_generic_kernel",
                    "p_data": pq, "p_meas": pq, "shots_per_launch": shots5,
                    "convergence_rate": float((d_conv[:shots5].min(dim=1).values == 1).double().mean().item()),
                    "mean_iterations": float(its.max(dim=1).values.double().mean().item())}
    # ---- config 5 AS NAMED: soft (noisy) syndromes.  Data flips at p, every check measured
    # through a Gaussian channel with flip probability Phi(-mu/sigma) ~ p; the reliabilities
    # |LLR_m| are per-shot priors of the absorbed measurement variables (qb_decode_batch_soft).
    import math
    mu, sigma = 1.0, 0.39
    q_eff = 0.5 * math.erfc(mu / sigma / math.sqrt(2))
    for arith, dt in (("int8", torch.int8), ("float", torch.float32)):
        e_soft = torch.zeros((shots5, ge.num_checks), dtype=dt, device=dev)
        for label, iters, early in (("cap50_early", 50, True), ("fixed10", 10, False)):
            cfg = DecoderConfig(max_iterations=iters, early_termination=early, arithmetic=arith,
                                priors=[llr] * ge.num_vars)
            with Decoder(ge, cfg, segments=segs) as dec:
                dec.generate_soft_syndromes(args.seed, pq, mu, sigma, shots5, e_syn.data_ptr(),
                                            e_soft.data_ptr(), None, stream=stream)
                f = lambda: dec.decode_batch_soft_device(shots5, e_syn.data_ptr(), e_soft.data_ptr(),
                                                         e_est.data_ptr(), None, d_conv.data_ptr(),
                                                         d_its.data_ptr(), stream)
                for _ in range(3):
                    f()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(3):
                    f()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 3
                its = d_its[:shots5].to(torch.int64)
                eu = float(its.sum().item()) * (ge.num_edges // 2)
                out[f"config5_soft_{arith}_{label}"] = {
                    "decodes_per_s": shots5 / ms * 1e3, "edge_updates_per_s": eu / ms * 1e3,
                    "kernel": "decode_ell_h2_kernel<soft>" if dec.get_option(10) else "decode_ell_kernel<soft>",
                    "p_data": pq, "mu": mu, "sigma": sigma, "p_meas_effective": q_eff,
                    "shots_per_launch": shots5, "soft_bytes_per_shot": ge.num_checks * e_soft.element_size(),
                    "convergence_rate": float((d_conv[:shots5].min(dim=1).values == 1).double().mean().item()),
                    "mean_iterations": float(its.max(dim=1).values.double().mean().item())}
    from paper_2508_07879_b200.campaign import PhenomenologicalCampaign
    for arith in ("int8", "float"):
        pc = PhenomenologicalCampaign(code, DecoderConfig(max_iterations=50, arithmetic=arith), pq, q_eff)
        try:
            tr = 1 << 18
            for name, fn in (("config5_campaign_hard", lambda first: pc.run_range(args.seed, first, tr)),
                             ("config5_campaign_soft", lambda first: pc.run_range_soft(args.seed, mu, sigma, first, tr))):
                fn(0)
                t0 = time.perf_counter()
                for r in range(3):
                    c = fn((r + 1) * tr)
                dt = (time.perf_counter() - t0) / 3
                out[f"{name}_{arith}"] = {
                    "trials_per_s": tr / dt, "trials_per_call": tr, "p_data": pq, "p_meas": q_eff,
                    "failures_last_call": int(c[2] + c[3] + c[4] + c[5]),
                    "timer": "host perf_counter around the blocking campaign call, mean of 3"}
        finally:
            pc.close()
    # ---- BASELINE config 4's loop, entirely on the device: sample -> syndrome -> decode ->
    # classify through qb_campaign_run, with the reference-exact sampler and the skip sampler
    from paper_2508_07879_b200 import _lib
    from paper_2508_07879_b200.campaign import Campaign
    trials = min(args.shots, 1 << 20)
    camp = Campaign(code, DecoderConfig(max_iterations=args.max_iterations,
                                        early_termination=not args.no_early_stop,
                                        arithmetic=args.arithmetic))
    try:
        for name, sampler, fused in (("campaign_reference_stream", 0, 1),
                                     ("campaign_reference_stream_three_kernels", 0, 0),
                                     ("campaign_skip_sampler", 1, 0)):
            camp.decoder.set_option(_lib.OPT_SAMPLER, sampler)
            camp.decoder.set_option(17, fused)  # QB_OPT_CAMPAIGN_FUSED
            camp.run_range(args.p, args.seed, 0, trials)  # warm-up (buffers, module load)
            t0 = time.perf_counter()
            reps = 3
            for r in range(reps):
                c = camp.run_range(args.p, args.seed, r * trials, trials)
            dt = (time.perf_counter() - t0) / reps
            out[name] = {"trials_per_s": trials / dt, "trials_per_call": trials, "p": args.p,
                         "kernels": ("decode_lean_campaign_kernel + campaign_count_kernel" if fused and sampler == 0
                                     else "sampler + decode_lean_kernel + classify_kernel"),
                         "timer": "host perf_counter around qb_campaign_run (blocking), mean of 3",
                         "non_converged_last_call": int(c[5])}
    finally:
        camp.close()
    return out


def measure_e2e(args, dec, lib, d_syn, shots, sw, ew, nseg):
    """qb_decode_batch through pinned host buffers: H2D + kernel + D2H per step (this rank)."""
    import torch

    def pinned(nbytes):
        p = C.c_void_p()
        assert lib.qb_host_alloc(C.byref(p), nbytes) == 0
        return p

    n = shots
    if args.e2e_chunk:
        dec.set_option(15, args.e2e_chunk)
    h_syn, h_est = pinned(n * sw * 8), pinned(n * ew * 8)
    h_conv, h_its = pinned(n * nseg), pinned(n * nseg * 4)
    # stage the same synthetic batch on the host (outside the timed region)
    torch.cuda.synchronize()
    host_syn = d_syn.cpu().numpy()
    C.memmove(h_syn, host_syn.ctypes.data, n * sw * 8)
    l0 = dec.launch_count()
    for _ in range(2):
        dec.decode_batch_raw(n, h_syn.value, h_est.value, None, h_conv.value, h_its.value)
    times = []
    for _ in range(max(args.steps, 3)):
        t0 = time.perf_counter()
        dec.decode_batch_raw(n, h_syn.value, h_est.value, None, h_conv.value, h_its.value)
        times.append(time.perf_counter() - t0)
    dt = float(np.median(times))
    out = {"value": n / dt, "unit": "decodes/s", "h2d_bytes_per_step": n * sw * 8,
           "d2h_bytes_per_step": n * (ew * 8 + nseg + 4 * nseg), "ms_per_step": dt * 1e3,
           "api": "qb_decode_batch (pinned host buffers; H2D, kernel, D2H inside the call)",
           "timer": "host perf_counter around the blocking call, median of %d; max over ranks" % len(times),
           "gpu_launches_per_step": (dec.launch_count() - l0) // (2 + len(times))}
    for p in (h_syn, h_est, h_conv, h_its):
        lib.qb_host_free(p)
    # what the host link of this box delivers (pinned, 64 MiB per copy, one direction at a
    # time): the e2e rate needs d2h_bytes_per_step / step time of it in the D2H direction
    try:
        nb = 64 << 20
        hbuf = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
        dbuf = torch.empty(nb, dtype=torch.uint8, device="cuda")
        link = {}
        for name, dst, src in (("h2d_gbs", dbuf, hbuf), ("d2h_gbs", hbuf, dbuf)):
            dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(4):
                dst.copy_(src, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            link[name] = 4 * nb / (e0.elapsed_time(e1) * 1e-3) / 1e9
        link["d2h_needed_gbs"] = out["d2h_bytes_per_step"] / dt / 1e9
        link["h2d_needed_gbs"] = out["h2d_bytes_per_step"] / dt / 1e9
        link["note"] = "measured pinned-memory copy rates of this box beside what the e2e rate moves"
        out["host_link"] = link
    except Exception as exc:  # the measurement is explanatory only
        out["host_link"] = {"error": str(exc)}
    return out


def measure_latency(args, code, lib, d_syn):
    """Single-shot decode latency through qb_decode (host buffers in, host buffers
    out), per the reference protocol: pool of 256 syndromes, 10 iterations fixed
    (bench.hpp:20-28) and the 50-iteration early-stop variant; nearest-rank
    percentiles (bench.cpp:169-180)."""
    from paper_2508_07879_b200 import Decoder, DecoderConfig
    pool = d_syn[:256].cpu().numpy().astype(np.uint64)
    out = {}
    for label, iters, early in (("fixed10", 10, False), ("cap50_early", 50, True)):
        cfg = DecoderConfig(max_iterations=iters, early_termination=early,
                            arithmetic=args.arithmetic)
        with Decoder(code, cfg) as dec:
            for io_mode, io_name in ((2, "doorbell"), (0, "mapped"), (1, "memcpy"),
                                     (1, "memcpy_nograph"), (1, "memcpy_poll")):
                dec.set_option(1, io_mode)
                dec.set_option(12, 0 if io_name == "memcpy_nograph" else 1)
                dec.set_option(18, 1 if io_name == "memcpy_poll" else 0)
                wall, kern, digest = dec.latency_run(pool, 300, args.latency_shots)
                wall = np.sort(wall.astype(np.float64) * 1e-3)
                kern = np.sort(kern.astype(np.float64) * 1e-3)
                out[f"{label}_{io_name}"] = {
                    "p50": nearest_rank(wall, 50), "p99": nearest_rank(wall, 99),
                    "mean": float(np.mean(wall)), "min": float(wall[0]), "max": float(wall[-1]),
                    "kernel_p50": nearest_rank(kern, 50), "kernel_p99": nearest_rank(kern, 99),
                    "shots": args.latency_shots, "digest": "%016x" % digest}
                if io_mode == 1 and io_name != "memcpy_poll":  # the same protocol timed by CUDA events on the stream
                    dec.set_option(11, 1)
                    _, ev, _ = dec.latency_run(pool, 300, args.latency_shots)
                    dec.set_option(11, 0)
                    ev = np.sort(ev.astype(np.float64) * 1e-3)
                    out[f"{label}_{io_name}"].update(
                        {"cuda_event_p50": nearest_rank(ev, 50), "cuda_event_p99": nearest_rank(ev, 99),
                         "cuda_event_mean": float(np.mean(ev))})
    # config 3 also names the reduced-precision path: same protocol, doorbell and launch-per-shot
    for arith in ("half", "int8"):
        if arith == args.arithmetic:
            continue
        cfg = DecoderConfig(max_iterations=10, early_termination=False, arithmetic=arith)
        with Decoder(code, cfg) as dec:
            for io_mode, io_name in ((2, "doorbell"), (0, "mapped")):
                dec.set_option(1, io_mode)
                wall, kern, digest = dec.latency_run(pool, 300, args.latency_shots)
                wall = np.sort(wall.astype(np.float64) * 1e-3)
                kern = np.sort(kern.astype(np.float64) * 1e-3)
                out[f"{arith}_fixed10_{io_name}"] = {
                    "p50": nearest_rank(wall, 50), "p99": nearest_rank(wall, 99),
                    "mean": float(np.mean(wall)), "kernel_p50": nearest_rank(kern, 50),
                    "kernel_p99": nearest_rank(kern, 99), "shots": args.latency_shots,
                    "digest": "%016x" % digest}
    # BASELINE config 5's graph: single shots on the phenomenological extension (degree-padded
    # kernel, one CTA per segment, H2D / kernel / D2H as one graph launch)
    from paper_2508_07879_b200 import codes, gf2
    hx, segs = codes.extended_graph(code)
    gx = codes.build_tanner_graph(hx)
    pq = 0.005
    rng = np.random.default_rng(args.seed)
    pool5 = gf2.pack_bits(hx.mat_vec((rng.random((256, gx.num_vars)) < pq).astype(np.uint8)))
    for arith in ("int8", "float"):
        cfg = DecoderConfig(max_iterations=10, early_termination=False, arithmetic=arith,
                            priors=[float(np.log((1 - pq) / pq))] * gx.num_vars)
        with Decoder(gx, cfg, segments=segs) as dec:
            for io_mode, io_name in ((2, "doorbell"), (0, "mapped"), (1, "memcpy")):
                dec.set_option(1, io_mode)
                wall, kern, digest = dec.latency_run(pool5, 300, args.latency_shots)
                wall = np.sort(wall.astype(np.float64) * 1e-3)
                kern = np.sort(kern.astype(np.float64) * 1e-3)
                out[f"config5_ext_{arith}_fixed10_{io_name}"] = {
                    "p50": nearest_rank(wall, 50), "p99": nearest_rank(wall, 99),
                    "mean": float(np.mean(wall)), "kernel_p50": nearest_rank(kern, 50),
                    "kernel_p99": nearest_rank(kern, 99), "shots": args.latency_shots,
                    "kernel": "decode_ell_latency_kernel" if dec.get_option(106) else "decode_generic_kernel"}
    # ... and config 5 as named (soft syndromes): every single shot carries its own priors of the
    # measurement-error variables (qb_decode_soft); l_m = (1 - 2 s_m) mu + N(0, sigma^2)
    mu, sigma = 1.0, 0.39
    s0 = hx.mat_vec((rng.random((256, gx.num_vars)) < pq).astype(np.uint8) * data_mask(code, gx)[None, :])
    lm = (1.0 - 2.0 * s0) * mu + sigma * rng.standard_normal(s0.shape)
    pool5s, llr5 = gf2.pack_bits((lm < 0).astype(np.uint8)), 2.0 * mu * np.abs(lm) / sigma ** 2
    for arith in ("int8", "float"):
        cfg = DecoderConfig(max_iterations=10, early_termination=False, arithmetic=arith,
                            priors=[float(np.log((1 - pq) / pq))] * gx.num_vars)
        with Decoder(gx, cfg, segments=segs) as dec:
            soft5 = dec.quantize_soft(llr5)
            for io_mode, io_name in ((2, "doorbell"), (0, "mapped"), (1, "memcpy")):
                dec.set_option(1, io_mode)
                wall, kern, digest = dec.latency_run(pool5s, 300, args.latency_shots, soft_pool=soft5)
                wall = np.sort(wall.astype(np.float64) * 1e-3)
                kern = np.sort(kern.astype(np.float64) * 1e-3)
                out[f"config5_soft_{arith}_fixed10_{io_name}"] = {
                    "p50": nearest_rank(wall, 50), "p99": nearest_rank(wall, 99),
                    "mean": float(np.mean(wall)), "kernel_p50": nearest_rank(kern, 50),
                    "kernel_p99": nearest_rank(kern, 99), "shots": args.latency_shots,
                    "soft_bytes_per_shot": int(soft5.shape[1] * soft5.itemsize), "mu": mu, "sigma": sigma,
                    "api": "qb_decode_soft", "kernel": "decode_ell_latency_kernel"}
    out["note"] = ("wall = host steady_clock around the whole qb_decode (copy-in, launch, "
                   "completion, copy-out) inside qb_latency_run; kernel = in-kernel %globaltimer "
                   "span; doorbell = persistent cluster polling mapped host memory (no launch per "
                   "shot), mapped = one cluster launch per shot with the syndrome in the kernel "
                   "parameters and results to mapped pinned memory + completion flag, memcpy = "
                   "cudaMemcpyAsync H2D / kernel / D2H + stream sync (paper protocol) as ONE CUDA-graph "
                   "launch per decode (memcpy_nograph: three separate stream operations; memcpy_poll: the "
                   "host watches the tags of the copied record instead of cudaStreamSynchronize, "
                   "QB_OPT_LATENCY_WAIT = 1); cuda_event = "
                   "cudaEventRecord before the H2D copy and after the D2H copy of that protocol")
    return out


def data_mask(code, gx) -> np.ndarray:
    """1 for the data-qubit variables of the extended graph [Hz | I] (+) [Hx | I], 0 for the
    measurement-error variables."""
    n, mz = code.n, code.hz.rows
    m = np.zeros(gx.num_vars, dtype=np.uint8)
    m[:n] = 1
    m[n + mz:2 * n + mz] = 1
    return m


def compact_latency(table: dict) -> dict:
    """p50 / p99 (us) per protocol from measure_latency's table, for `e2e.latency_us`."""
    out = {"unit": "us", "protocols": "memcpy = cudaMemcpyAsync H2D + kernel + D2H + sync as one "
           "CUDA-graph launch (the paper's protocol; cuda_event = the same span by CUDA events; "
           "memcpy_poll = the same with the host watching the copied record's tags instead of the stream sync); "
           "mapped = one cluster launch per shot, syndrome in the kernel parameters, result to "
           "mapped pinned memory; doorbell = persistent cluster polling mapped memory. Host "
           "steady_clock around the whole qb_decode call, nearest-rank percentiles"}
    code = {}
    for label in ("fixed10", "cap50_early"):
        row = {}
        for proto in ("memcpy", "memcpy_poll", "mapped", "doorbell"):
            r = table.get(f"{label}_{proto}")
            if not r:
                continue
            row[proto] = {"p50": r["p50"], "p99": r["p99"]}
            if "cuda_event_p50" in r:
                row[proto].update(cuda_event_p50=r["cuda_event_p50"], cuda_event_p99=r["cuda_event_p99"])
        code[label] = row
    out["bb784_float"] = code
    for arith in ("int8", "float"):
        row = {}
        for proto in ("memcpy", "mapped", "doorbell"):
            r = table.get(f"config5_ext_{arith}_fixed10_{proto}")
            if r:
                row[proto] = {"p50": r["p50"], "p99": r["p99"]}
        if row:
            out[f"config5_ext784_{arith}"] = {"fixed10": row}
        row = {}
        for proto in ("memcpy", "mapped", "doorbell"):
            r = table.get(f"config5_soft_{arith}_fixed10_{proto}")
            if r:
                row[proto] = {"p50": r["p50"], "p99": r["p99"]}
        if row:
            out[f"config5_soft784_{arith}"] = {"fixed10": row}
    return out


def measure_latency_bb144(args) -> dict:
    """BASELINE config 2: [[144,12,12]] single shots, fp32, ONE CTA per shot - a decoder built
    from the combined Tanner graph (the reference's `Decoder(graph, cfg)` constructor: one
    segment, decoder.cpp:406-413), which the cluster kernel runs as a cluster of one CTA - and,
    beside it, the CssCode decoder (two segments) as a 2-CTA cluster; pool = trials 0..255 of
    sample_error(p, seed) exactly as run_bench builds it (proj/src/bench.cpp:203-211),
    generated by the bit-exact device sampler."""
    import torch
    from paper_2508_07879_b200 import Decoder, DecoderConfig, codes, gf2
    code = codes.make_code("bb144")
    g = code.combined_graph
    d_pool = torch.zeros((256, gf2.num_words(g.num_checks)), dtype=torch.int64, device="cuda")
    out = {}
    for label, iters, early in (("fixed10", 10, False), ("cap50_early", 50, True)):
        cfg = DecoderConfig(max_iterations=iters, early_termination=early, arithmetic=args.arithmetic)
        row = {}
        with Decoder(code, cfg) as gen:
            gen.generate_syndromes(args.seed, args.p, 256, d_pool.data_ptr(), None,
                                   stream=torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
        pool = d_pool.cpu().numpy().astype(np.uint64)
        for shape_name, target in (("one_cta_per_shot", g), ("cluster", code)):
            with Decoder(target, cfg) as dec:
                assert dec.get_option(106) == 1, "cluster kernel expected"
                for io_mode, io_name in ((1, "memcpy"), (0, "mapped"), (2, "doorbell")):
                    dec.set_option(1, io_mode)
                    wall, kern, _ = dec.latency_run(pool, 300, args.latency_shots)
                    wall = np.sort(wall.astype(np.float64) * 1e-3)
                    kern = np.sort(kern.astype(np.float64) * 1e-3)
                    r = {"p50": nearest_rank(wall, 50), "p99": nearest_rank(wall, 99),
                         "kernel_p50": nearest_rank(kern, 50), "kernel_p99": nearest_rank(kern, 99)}
                    if io_mode == 1:  # the same protocol timed by CUDA events on the stream
                        dec.set_option(11, 1)
                        _, ev, _ = dec.latency_run(pool, 300, args.latency_shots)
                        dec.set_option(11, 0)
                        ev = np.sort(ev.astype(np.float64) * 1e-3)
                        r.update(cuda_event_p50=nearest_rank(ev, 50), cuda_event_p99=nearest_rank(ev, 99))
                    row[f"{shape_name}_{io_name}"] = r
        out[label] = row
    out["shapes"] = ("one_cta_per_shot = Decoder(combined graph): one segment, X and Z stop together "
                     "(identical outcomes at a fixed iteration count); cluster = Decoder(CssCode): "
                     "one CTA per segment, segments stop independently")
    return {"bb144_%s" % args.arithmetic: out}


def free_port() -> int:
    import socket
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        return sock.getsockname()[1]


def spawn_ranks(args) -> int:
    """`python bench.py --gpus N` without a launcher: re-execute this command under
    torch.distributed.run with N ranks on this node (what the driver does itself for N > 1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # keep the communicator's log (rings / NVLS) on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT,COLL")
    return subprocess.call(cmd, env=env)


def run_dry(args):
    """--dry-spawn: everything about the N-rank run except the GPU - rendezvous (gloo),
    contiguous trial shards, ONE all_reduce(SUM) of the counter vector through
    campaign.run_campaign's own code path, max-over-ranks timing, one line from rank 0."""
    import torch
    import torch.distributed as dist
    from paper_2508_07879_b200.campaign import COUNTER_NAMES, run_campaign
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    trials = args.shots

    def fake_range(p, seed, first, count):  # a rank's counters: `count` trials, all "exact"
        c = np.zeros(len(COUNTER_NAMES), dtype=np.uint64)
        c[0] = count
        c[8] = (2 * first + count - 1) * count // 2  # sum of its trial ids: depends on WHICH trials it got
        c[9] = count
        return c

    t0 = time.perf_counter()
    res = run_campaign(None, args.p, args.seed, trials, None, world=world, rank=rank,
                       range_fn=fake_range, reduce_device="cpu")
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"dry_spawn": True, "n_gpus": world, "gpus_requested": args.gpus,
                          "trials": res.trials, "exact": res.exact,
                          "trial_id_sum": int(round(res.mean_iterations * max(res.trials, 1))),
                          "trial_id_sum_expected": trials * (trials - 1) // 2,
                          "seconds_max_over_ranks": float(t.item())}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:
        sys.exit(spawn_ranks(args))
    if world and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} ranks")
    if args.dry_spawn:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

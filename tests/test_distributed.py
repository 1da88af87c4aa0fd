"""Multi-rank host path on CPU (gloo, world_size 2): campaign.run_campaign(world=2) itself -
its trial partition and the final counter all-reduce, the only collective on the path
 - checked against a single-process run, plus bench.py's own rank spawning.
The per-rank counter function is INJECTED (range_fn): each rank classifies its shard with
the CPU oracle standing in for the GPU kernels (this is a test: the product path never
does that), everything around it is the product's code."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_counters(lo, hi):
    """Counters of trials [lo, hi) computed on the CPU: numpy sampler keyed by the
    trial id (so shards are independent of the partition) + C oracle decode."""
    sys.path.insert(0, ROOT)
    from oracle.pyoracle import Oracle
    from paper_2508_07879_b200 import DecoderConfig, codes, gf2
    from paper_2508_07879_b200.campaign import COUNTER_NAMES, logical_operators
    code = codes.make_code("bb72")
    cfg = DecoderConfig(max_iterations=10)
    lz, lx = logical_operators(code)
    orc = Oracle()
    c = np.zeros(len(COUNTER_NAMES), dtype=np.uint64)
    for t in range(lo, hi):
        rng = np.random.default_rng([20260822, t])
        ex = (rng.random(code.n) < 0.04).astype(np.uint8)
        ez = (rng.random(code.n) < 0.04).astype(np.uint8)
        syn = gf2.pack_bits(np.concatenate([code.hz.mat_vec(ex), code.hx.mat_vec(ez)]))
        est, _, conv, its, _, _ = orc.decode(code.combined_graph, cfg, syn, code.segments)
        eh = gf2.unpack_bits(est, 2 * code.n)
        rx, rz = ex ^ eh[:code.n], ez ^ eh[code.n:]

        def harmful(r, tests):
            v = sum(int(b) << i for i, b in enumerate(r))
            return any(bin(v & tvec).count("1") & 1 for tvec in tests)

        if not conv.all():
            cls = 5
        elif not rx.any() and not rz.any():
            cls = 0
        else:
            bx, bz = harmful(rx, lz), harmful(rz, lx)
            cls = 1 if not bx and not bz else 4 if bx and bz else 2 if bx else 3
        c[cls] += 1
        c[7] += int(conv.all())
        c[8] += int(its.max())
        c[9] += 1
    return c


def _worker(rank, world, port, trials, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_2508_07879_b200.campaign import COUNTER_NAMES, run_campaign
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seen = []

    def range_fn(p, seed, first, count):  # stands in for Campaign.run_range on this rank's GPU
        seen.append((first, first + count))
        return _oracle_counters(first, first + count)

    res = run_campaign(None, 0.04, 20260822, trials, None, world=world, rank=rank,
                       range_fn=range_fn, reduce_device="cpu")
    total = [getattr(res, k) for k in COUNTER_NAMES[:6]] + [res.trials]
    out.put((rank, total, res.logical_error_rate, res.mean_iterations, seen[0] if seen else (0, 0)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_campaign_reduction_matches_single_process():
    import torch.multiprocessing as mp
    from paper_2508_07879_b200.campaign import CampaignResult, shard
    trials, world = 120, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, trials, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = _oracle_counters(0, trials)
    want = CampaignResult.from_counters(single)
    for rank, total, ler, mean_it, (lo, hi) in results:
        assert (lo, hi) == shard(trials, world, rank)
        assert total == [int(x) for x in single[:6]] + [trials], f"rank {rank} sees a different aggregate"
        assert ler == want.logical_error_rate and mean_it == want.mean_iterations
    assert single[9] == trials


def test_run_campaign_refuses_world_gt_1_without_a_process_group():
    """One shard's counters must never be returned as the campaign's (reduce_counters)."""
    from paper_2508_07879_b200.campaign import COUNTER_NAMES, run_campaign
    fn = lambda p, seed, first, count: np.zeros(len(COUNTER_NAMES), dtype=np.uint64)
    with pytest.raises(RuntimeError, match="no process group"):
        run_campaign(None, 0.01, 1, 100, None, world=2, rank=0, range_fn=fn, reduce_device="cpu")
    with pytest.raises(ValueError, match="rank"):
        run_campaign(None, 0.01, 1, 100, None, world=2, rank=2, range_fn=fn, reduce_device="cpu")
    assert run_campaign(None, 0.01, 1, 100, None, range_fn=fn).trials == 0


def test_bench_spawns_its_own_ranks():
    """`python bench.py --gpus 2` with no launcher must start 2 ranks itself and say so
    (--dry-spawn: the rank plumbing on gloo, no GPU)."""
    import json
    import subprocess
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-spawn",
                        "--shots", "100001"], capture_output=True, text=True, timeout=240, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["gpus_requested"] == 2
    assert line["trials"] == 100001 and line["exact"] == 100001
    assert line["trial_id_sum"] == line["trial_id_sum_expected"]


def test_shard_partition_is_contiguous_and_complete():
    """Same rule as the reference's worker split (proj/src/noise.cpp:253-254)."""
    from paper_2508_07879_b200.campaign import shard
    for trials in (0, 1, 7, 1000, 1 << 20):
        for world in (1, 2, 3, 4, 8):
            edges = [shard(trials, world, r) for r in range(world)]
            assert edges[0][0] == 0 and edges[-1][1] == trials
            assert all(a[1] == b[0] for a, b in zip(edges, edges[1:]))
            assert max(hi - lo for lo, hi in edges) - min(hi - lo for lo, hi in edges) <= 1

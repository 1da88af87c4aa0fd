"""Device campaign (sample -> syndrome -> decode -> classify on the GPU) against
the reference's run_campaign (proj/src/noise.cpp:217-338) through the prebuilt
compiled reference: because the sampler and the decoder are bit-exact, every
counter must be IDENTICAL, not merely statistically compatible."""
import numpy as np
import pytest

from paper_2508_07879_b200 import DecoderConfig, codes
from paper_2508_07879_b200.campaign import Campaign, CampaignResult, run_campaign, shard

pytestmark = pytest.mark.gpu


def _same(ours: CampaignResult, theirs: dict):
    for key in ("trials", "exact", "stabilizer", "logical_x", "logical_z", "logical_both",
                "non_converged"):
        assert getattr(ours, key) == theirs[key], key
    for key in ("logical_error_rate", "baseline_logical_rate", "convergence_rate",
                "mean_iterations"):
        assert abs(getattr(ours, key) - theirs[key]) < 1e-12, key


@pytest.mark.parametrize("mode", ["float", "int8", "int16"])
def test_campaign_counts_equal_reference_bb72(ref, mode):
    """acceptance check 7's configuration (proj/tests/acceptance.cpp:288-314) and a
    high-noise point where logical misclassifications actually occur."""
    code = codes.make_code("bb72")
    rc = ref.code("bb72")
    for p, seed, trials, iters in ((0.01, 20260822, 4000, 10), (0.06, 7, 3000, 30)):
        cfg = DecoderConfig(max_iterations=iters, arithmetic=mode)
        theirs = ref.run_campaign(rc, 0, p, seed, trials, cfg, workers=0)
        ours = run_campaign(code, p, seed, trials, cfg)
        _same(ours, theirs)
    assert theirs["logical_x"] + theirs["logical_z"] + theirs["logical_both"] > 0


def test_campaign_counts_equal_reference_bb784(ref):
    code = codes.make_code("bb784")
    rc = ref.code("bb784")
    cfg = DecoderConfig(max_iterations=50)
    theirs = ref.run_campaign(rc, 0, 0.02, 12345, 1500, cfg, workers=0)
    ours = run_campaign(code, 0.02, 12345, 1500, cfg)
    _same(ours, theirs)


def test_campaign_is_independent_of_the_partition():
    """Deterministic for a fixed seed, independent of the worker / rank count
    (proj/tests/test_noise.cpp:372-434): per-shard counters add up exactly."""
    code = codes.make_code("bb144")
    cfg = DecoderConfig(max_iterations=20)
    camp = Campaign(code, cfg)
    try:
        whole = camp.run_range(0.03, 99, 0, 5000)
        for world in (2, 3, 8):
            total = np.zeros_like(whole)
            for rank in range(world):
                lo, hi = shard(5000, world, rank)
                total += camp.run_range(0.03, 99, lo, hi - lo)
            assert np.array_equal(total, whole)
        # several sample / decode / classify rounds inside one call (QB_OPT_BATCH_CHUNK),
        # including one-trial rounds (odd counts exercise the packed kernels' half-empty pair)
        small = camp.run_range(0.03, 99, 0, 40)
        for chunk, trials, want in ((1, 40, small), (64, 5000, whole), (1001, 5000, whole),
                                    (4999, 5000, whole)):
            camp.decoder.set_option(15, chunk)
            assert np.array_equal(camp.run_range(0.03, 99, 0, trials), want), chunk
        camp.decoder.set_option(15, 0)
    finally:
        camp.close()


def test_decoder_beats_the_identity_baseline():
    """proj/tests/test_noise.cpp:446-457: LER < 0.05 and baseline > 0.5 at p = 0.01 on bb72."""
    r = run_campaign(codes.make_code("bb72"), 0.01, 20260822, 10000, DecoderConfig())
    assert r.logical_error_rate < 0.05 and r.baseline_logical_rate > 0.5


def test_half_precision_ler_within_reference_ci(ref):
    """north star: the reduced-precision (fp16) path has no bit-level oracle; its
    logical error rate must lie within the 95 % binomial confidence interval of the
    reference decoder's (float) on the same noise model."""
    import math
    code = codes.make_code("bb144")
    rc = ref.code("bb144")
    for p, iters in ((0.02, 30), (0.04, 30)):
        trials_ref = 12000
        rr = ref.run_campaign(rc, 0, p, 4242, trials_ref, DecoderConfig(max_iterations=iters),
                              workers=0)
        k = rr["logical_x"] + rr["logical_z"] + rr["logical_both"] + rr["non_converged"]
        ph, z = k / trials_ref, 1.96
        den = 1 + z * z / trials_ref
        c = (ph + z * z / (2 * trials_ref)) / den
        hw = z * math.sqrt(ph * (1 - ph) / trials_ref + z * z / (4 * trials_ref ** 2)) / den
        ours = run_campaign(code, p, 4242, 200000,
                            DecoderConfig(max_iterations=iters, arithmetic="half"))
        assert c - hw <= ours.logical_error_rate <= c + hw, (p, ours.logical_error_rate, c, hw)


def test_skip_sampler_campaign_within_reference_ci_and_partition_independent(ref):
    """QB_OPT_SAMPLER = 1 draws other trials than the reference (geometric gaps instead of
    one uniform per qubit), so its campaign is judged like the fp16 path: failure rate inside
    the 95 % Wilson interval of the reference's run_campaign on the same noise model, mean
    iteration count close to it, and - the stream being keyed by (seed, trial) - counters
    that do not depend on how the trial range is split."""
    import math
    code = codes.make_code("bb144")
    rc = ref.code("bb144")
    cfg = DecoderConfig(max_iterations=30)
    camp = Campaign(code, cfg)
    try:
        camp.decoder.set_option(16, 1)
        for p in (0.02, 0.04):
            n = 12000
            rr = ref.run_campaign(rc, 0, p, 4242, n, cfg, workers=0)
            k = rr["logical_x"] + rr["logical_z"] + rr["logical_both"] + rr["non_converged"]
            ph, z = k / n, 1.96
            den = 1 + z * z / n
            c = (ph + z * z / (2 * n)) / den
            hw = z * math.sqrt(ph * (1 - ph) / n + z * z / (4 * n * n)) / den
            ours = CampaignResult.from_counters(camp.run_range(p, 4242, 0, 200000))
            assert c - hw <= ours.logical_error_rate <= c + hw, (p, ours.logical_error_rate, c, hw)
            assert abs(ours.mean_iterations - rr["mean_iterations"]) < 0.05 * rr["mean_iterations"]
            assert ours.baseline_logical_rate > 0.5
        whole = camp.run_range(0.03, 99, 0, 5000)
        total = np.zeros_like(whole)
        for rank in range(3):
            lo, hi = shard(5000, 3, rank)
            total += camp.run_range(0.03, 99, lo, hi - lo)
        assert np.array_equal(total, whole)
        camp.decoder.set_option(15, 999)   # five and a bit rounds of 999 trials per call
        assert np.array_equal(camp.run_range(0.03, 99, 0, 5000), whole)
        camp.decoder.set_option(15, 0)
        camp.decoder.set_option(16, 0)
        assert not np.array_equal(camp.run_range(0.03, 99, 0, 5000), whole)
    finally:
        camp.close()


def test_multi_gpu_entry_point_on_the_gpus_present(ref):
    """qb_campaign_run_multi: one decoder per visible GPU, contiguous shards, ONE
    ncclAllReduce of the ten counters (NCCL bound at run time).  On a 1-GPU box this still
    exercises the whole path - communicator creation, grouped all-reduce, agreement check -
    and the result must equal the reference's run_campaign."""
    import ctypes as C
    import torch
    from paper_2508_07879_b200 import _lib
    lib = _lib.load()
    code = codes.make_code("bb72")
    cfg = DecoderConfig(max_iterations=10)
    ngpu = torch.cuda.device_count()
    camps = [Campaign(code, cfg, device=d) for d in range(ngpu)]
    try:
        handles = (C.c_void_p * ngpu)(*[c.decoder._h for c in camps])
        counters = np.zeros(10, dtype=np.uint64)
        for first, count in ((0, 2500), (2500, 1500)):  # ADDS, like qb_campaign_run
            st = lib.qb_campaign_run_multi(handles, ngpu, 20260822, 0.01, None, first, count,
                                           counters.ctypes.data_as(_lib.u64p))
            assert st == 0, lib.qb_last_error(camps[0].decoder._h).decode()
        theirs = ref.run_campaign(ref.code("bb72"), 0, 0.01, 20260822, 4000, cfg, workers=0)
        _same(CampaignResult.from_counters(counters), theirs)
        assert np.array_equal(counters, camps[0].run_range(0.01, 20260822, 0, 4000))
        # two handles on one device are refused (NCCL needs one rank per GPU)
        dup = (C.c_void_p * 2)(camps[0].decoder._h, camps[0].decoder._h)
        st = lib.qb_campaign_run_multi(dup, 2, 1, 0.01, None, 0, 10, counters.ctypes.data_as(_lib.u64p))
        assert st == _lib.QB_INVALID_ARGUMENT
        assert b"one decoder per GPU" in lib.qb_last_error(camps[0].decoder._h)
    finally:
        for c in camps:
            c.close()


@pytest.mark.parametrize("mode", ["float", "int16"])
def test_fused_campaign_kernel_equals_the_three_kernel_pipeline(ref, mode):
    """QB_OPT_CAMPAIGN_FUSED: sample + syndrome + decode + classify in one kernel
    (kernel_campaign.cuh) against sampler -> decode -> classifier as separate kernels and
    against the reference's run_campaign: all ten counters identical, at an early-stop and a
    fixed-iteration configuration, for whole ranges and odd splits."""
    code = codes.make_code("bb144")
    rc = ref.code("bb144")
    for cfg, p, trials in ((DecoderConfig(max_iterations=30, arithmetic=mode), 0.03, 6001),
                           (DecoderConfig(max_iterations=8, early_termination=False, arithmetic=mode), 0.05, 3000),
                           (DecoderConfig(max_iterations=1, arithmetic=mode), 0.01, 2000)):
        camp = Campaign(code, cfg)
        try:
            assert camp.decoder.get_option(17) == 1
            fused = camp.run_range(p, 77, 0, trials)
            split = camp.run_range(p, 77, 0, 1234) + camp.run_range(p, 77, 1234, trials - 1234)
            camp.decoder.set_option(15, 257)  # many rounds inside one call
            rounds = camp.run_range(p, 77, 0, trials)
            camp.decoder.set_option(15, 0)
            camp.decoder.set_option(17, 0)
            plain = camp.run_range(p, 77, 0, trials)
        finally:
            camp.close()
        assert np.array_equal(fused, plain), (fused, plain)
        assert np.array_equal(fused, split) and np.array_equal(fused, rounds)
        _same(CampaignResult.from_counters(fused), ref.run_campaign(rc, 0, p, 77, trials, cfg, workers=0))
    assert fused[6] > 0  # the identity-decoder baseline is exercised too

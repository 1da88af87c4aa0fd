"""'Next' rows of SURVEY.md §8f: alist input for user-supplied matrices and bench
CSV rows the reference's own reader accepts.  CPU-only parts run everywhere; the
CSV end-to-end check needs a GPU (it measures)."""
import os

import numpy as np
import pytest

from paper_2508_07879_b200 import alist, bench_csv, codes

TOY_ALIST = ("6 3\n2 4\n2 2 2 2 2 2\n4 4 4\n1 2\n2 3\n1 3\n1 2\n2 3\n1 3\n"
             "1 3 4 6\n1 2 4 5\n2 3 5 6\n")  # proj/tests/test_alist.cpp:27-40


def test_hand_written_fixture_loads():
    assert alist.loads(TOY_ALIST) == codes.toy_code_3x6()


def test_zero_padding_is_ignored_and_round_trip():
    padded = TOY_ALIST.replace("1 2\n", "1 2 0 0\n").replace("2 3\n", "2 3 0 0\n")
    assert alist.loads(padded) == codes.toy_code_3x6()
    for name in ("bb72",):
        h = codes.make_code(name).hx
        assert alist.loads(alist.dumps(h)) == h


@pytest.mark.parametrize("mutation,needle", [
    (lambda t: t.replace("6 3\n", "6\n", 1), "line 1"),
    (lambda t: t.replace("2 2 2 2 2 2\n", "2 2 2 2 2\n"), "line 3"),
    (lambda t: t.replace("1 3 4 6\n", "1 3 4 5\n"), "disagrees"),
    (lambda t: t.replace("1 2\n", "1 9\n", 1), "out of range"),
    (lambda t: t.replace("1 2\n", "1 x\n", 1), "non-integer"),
    (lambda t: t.rsplit("\n", 2)[0] + "\n", "unexpected end"),
])
def test_malformed_input_is_diagnosed(mutation, needle):
    with pytest.raises(alist.AlistError, match=needle):
        alist.loads(mutation(TOY_ALIST))


def test_loader_agrees_with_reference(ref):
    rng = np.random.default_rng(12)
    from tests.helpers import random_ldpc_matrix
    for _ in range(5):
        h = random_ldpc_matrix(rng, 5 + int(rng.integers(0, 5)), 9 + int(rng.integers(0, 6)))
        text = alist.dumps(h)
        rows, cols, coo = ref.load_alist(text)
        assert (rows, cols) == (h.rows, h.cols) and np.array_equal(coo, h.coo())
        assert alist.loads(text) == h
    bad = TOY_ALIST.replace("1 3 4 6\n", "1 3 4 5\n")
    with pytest.raises(RuntimeError):  # the reference throws std::runtime_error (alist.cpp:36-39)
        ref.load_alist(bad)
    with pytest.raises(RuntimeError):
        alist.loads(bad)


def test_percentile_and_row_format():
    """proj/tests/test_bench.cpp:52-71."""
    s = [1.0, 2.0, 3.0, 4.0]
    assert [bench_csv.percentile_nearest_rank(s, q) for q in (25, 50, 75, 99, 100, 1)] == \
        [1.0, 2.0, 3.0, 4.0, 4.0, 1.0]
    assert bench_csv.percentile_nearest_rank([7.0], 50) == 7.0
    for bad in (([], 50.0), (s, 0.0), (s, 100.5)):
        with pytest.raises(ValueError):
            bench_csv.percentile_nearest_rank(*bad)
    assert bench_csv.HEADER.count(",") == 18
    rec = bench_csv.BenchRecord("bb72", 72, 12, 6, "float", 0.8, 10, False, 1, 1, 300, 1.0, 2.0,
                                2.0, 3.0, 4.0, 1.0, 0.5, True)
    assert rec.row() == "bb72,72,12,6,float,0.8,10,0,1,1,300,1.000,2.000,2.000,3.000,4.000,1.000000,0.500000,1"


def test_reference_reader_accepts_our_csv_format(ref, tmp_path):
    rec = bench_csv.BenchRecord("bb72", 72, 12, 6, "float", 0.8, 10, False, 1, 1, 300, 1.0, 2.0,
                                2.0, 3.0, 4.0, 1.0, 0.5, True, digest=0x1234)
    path = os.path.join(tmp_path, "b.csv")
    bench_csv.write_bench_csv(path, [rec, rec])
    assert ref.read_bench_csv_file(path) == (2, 3.0)


@pytest.mark.gpu
def test_gpu_bench_rows_validate_and_digest_matches_reference(ref, tmp_path):
    """A GPU latency row in the reference's schema passes the reference's validating
    reader, and its digest equals BenchResult::output_digest of the CPU run."""
    code = codes.make_code("bb144")
    rows = [bench_csv.run_bench(code, mode, max_iterations=10, early_termination=False,
                                warmup=100, measure=200, p=0.01, seed=1, io_mode=io)
            for mode, io in (("float", 0), ("int8", 2))]
    path = os.path.join(tmp_path, "gpu.csv")
    bench_csv.write_bench_csv(path, rows)
    n, p99 = ref.read_bench_csv_file(path)
    assert n == 2 and abs(p99 - round(rows[0].p99_us, 3)) < 1e-9
    rc = ref.code("bb144")
    for rec in rows:
        r = ref.run_bench(rc, arithmetic=rec.mode, max_iterations=10, early_termination=False,
                          batch=1, threads=1, warmup=100, measure=200, p=0.01, seed=1)
        assert rec.digest == r["digest"]
        assert rec.under_63us and rec.p99_us < 63.0

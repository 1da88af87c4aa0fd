#!/bin/bash
# On the GPU box: initcheck over the sanitizer subset with every report kept (device frames
# only), condensed to one line per (kernel, source line) in gpurun_out/<round>_initcheck_sites.txt.
set -u
R=${1:-r1}
SKIP="--deselect tests/test_alist_csv.py::test_gpu_bench_rows_validate_and_digest_matches_reference"
SMALL='toy or bb72 or zero_syndrome or irregular or unit_degrees or degree_zero or tma_tiles or regular_and_cluster or memcpy_protocol or packed_fp16 or generator_reproduces or independent_of_the_partition or half_mode'
timeout ${SANITIZE_TIMEOUT:-1500} compute-sanitizer --tool initcheck --show-backtrace device --print-limit 400000 \
    --target-processes all --log-file /tmp/initcheck_full.log \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_ell.py tests/test_gpu_noise.py tests/test_gpu_campaign.py \
    -m gpu -q $SKIP -k "$SMALL" > gpurun_out/${R}_initcheck_pytest.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/${R}_initcheck_pytest.log)"
{
  grep -h "ERROR SUMMARY" /tmp/initcheck_full.log
  echo "reports per (access, kernel, source line):"
  grep -h -A4 "Uninitialized" /tmp/initcheck_full.log | grep "    at \|Device Frame" | sed 's/^=========\s*//; s/+0x[0-9a-f]*//' \
    | paste - - | sed 's/(qb::DecodeParams.*)//' | sort | uniq -c | sort -rn
} > gpurun_out/${R}_initcheck_sites.txt
cat gpurun_out/${R}_initcheck_sites.txt | cut -c1-300 | head -30

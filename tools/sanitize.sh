#!/bin/bash
# On the GPU box: the GPU parity tests under compute-sanitizer.
#   memcheck  : the whole `-m gpu` suite (out-of-bounds / misaligned global, shared, local)
#   racecheck : shared-memory hazards, on the tests that cover every kernel family at small
#               sizes (racecheck serialises warps, the large-batch tests would take hours)
#   synccheck : divergent / invalid barrier and mbarrier use, same subset
#   initcheck : reads of uninitialised device global memory, same subset
# Timing assertions are deselected (a sanitised decode is 10-100x slower).
# Logs: gpurun_out/<round>_<tool>.log (+ _pytest.log); one summary line per tool on stdout.
set -u
R=${1:-r1}
TOOLS=${2:-"memcheck racecheck synccheck initcheck"}
mkdir -p gpurun_out
SKIP="--deselect tests/test_alist_csv.py::test_gpu_bench_rows_validate_and_digest_matches_reference"
SUBSET="tests/test_gpu_parity.py tests/test_gpu_ell.py tests/test_gpu_noise.py tests/test_gpu_campaign.py tests/test_gpu_soft.py"
SMALL='toy or bb72 or zero_syndrome or irregular or unit_degrees or degree_zero or tma_tiles or regular_and_cluster or memcpy_protocol or packed_fp16 or generator_reproduces or independent_of_the_partition or fused_campaign or messages_half or degree_padded_batch_kernel_messages or soft_requires or device_campaigns_on_the_extended or rejected_option or alist or single_shot_soft'
for tool in $TOOLS; do
  log=gpurun_out/${R}_${tool}.log
  if [ "$tool" = memcheck ]; then
    sel="tests"; kexpr=""
  else
    sel="$SUBSET"; kexpr="$SMALL"
  fi
  extra=""
  skip="$SKIP"
  if [ "$tool" = racecheck ]; then
    extra="--racecheck-report all"
    # asserts a wall-clock bound (< 1 s for 64 decodes) that a racecheck run cannot meet
    skip="$SKIP --deselect tests/test_gpu_parity.py::test_memcpy_protocol_graph_and_event_timing"
  fi
  timeout ${SANITIZE_TIMEOUT:-1500} compute-sanitizer --tool $tool $extra --target-processes all \
      --log-file $log python -m pytest $sel -m gpu -q $skip ${kexpr:+-k "$kexpr"} \
      > gpurun_out/${R}_${tool}_pytest.log 2>&1
  rc=$?
  echo "$tool: pytest rc=$rc | $(tail -1 gpurun_out/${R}_${tool}_pytest.log) | $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $log | sort | uniq -c | tr '\n' ';')"
done

#!/bin/bash
# On the GPU box: racecheck with every hazard kept (no backtraces), condensed to one line per
# (hazard kind, write site, read site, shared-memory address) in
# gpurun_out/<round>_racecheck_sites_<part>.txt.  Two parts so that each stays under its
# timeout: "other" = degree-padded / noise / campaign tests, "parity" = test_gpu_parity.py.
set -u
R=${1:-r1}
PARTS=${2:-"other parity"}
SMALL='toy or bb72 or zero_syndrome or irregular or unit_degrees or degree_zero or tma_tiles or regular_and_cluster or packed_fp16 or generator_reproduces or independent_of_the_partition or skip_sampler or fused_campaign or messages_half or degree_padded_batch_kernel_messages or soft_requires or device_campaigns_on_the_extended or alist'
for part in $PARTS; do
  if [ "$part" = parity ]; then sel="tests/test_gpu_parity.py"; else sel="tests/test_gpu_ell.py tests/test_gpu_noise.py tests/test_gpu_campaign.py tests/test_gpu_soft.py"; fi
  log=/tmp/racecheck_${part}.log
  timeout ${SANITIZE_TIMEOUT:-1200} compute-sanitizer --tool racecheck --racecheck-report all --show-backtrace no \
      --print-limit 2000000 --target-processes all --log-file $log \
      python -m pytest $sel -m gpu -q -k "$SMALL" > gpurun_out/${R}_racecheck_${part}_pytest.log 2>&1
  echo "$part: pytest rc=$? $(tail -1 gpurun_out/${R}_racecheck_${part}_pytest.log)"
  {
    grep -h "RACECHECK SUMMARY" $log | sort | uniq -c
    echo "hazards per (kind, write site, read site, address):"
    grep -h -A2 "hazard detected" $log \
      | grep -o "Potential [A-Z]* hazard detected at __shared__ 0x[0-9a-f]*\|Thread ([0-9]*,[0-9]*,[0-9]*) at .* in [a-z_0-9]*\.[a-z]*:[0-9]*" \
      | sed 's/Thread ([0-9,]*) at //; s/+0x[0-9a-f]*//; s/(const qb::DecodeParams[^)]*)//; s/Potential //; s/ hazard detected at __shared__//' \
      | paste - - - | sort | uniq -c | sort -rn
  } > gpurun_out/${R}_racecheck_sites_${part}.txt
  head -40 gpurun_out/${R}_racecheck_sites_${part}.txt | cut -c1-260
done

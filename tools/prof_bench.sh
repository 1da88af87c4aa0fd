#!/bin/bash
# On the GPU box: (1) launch list of the default bench command, (2) one full ncu capture of the
# dominant kernel at the bench's own size, condensed to text + profiles/traffic.json inputs.
# Only small text files are left in gpurun_out/ (the .ncu-rep stays in /tmp).
set -u
R=${1:-r1}
mkdir -p gpurun_out /tmp/prof
FLAGS="--steps 2 --warmup 1 --skip-latency --skip-cpu-baseline --skip-e2e --skip-variants"
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches_bench.csv python bench.py $FLAGS > gpurun_out/${R}_launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_lean_kernel -s 1 -c 1 -f \
    -o /tmp/prof/bench python bench.py $FLAGS > gpurun_out/${R}_prof_bench.log 2>&1
python tools/ncu_summary.py /tmp/prof/bench.ncu-rep > gpurun_out/${R}_decode_lean_kernel_f32_earlystop.txt 2>&1
WL=$(python - <<'PY'
import bench, sys
sys.argv = ["bench.py"]
print(bench.workload_name(bench.parse_args()))
PY
)
python tools/ncu_summary.py /tmp/prof/bench.ncu-rep --traffic-json gpurun_out/traffic.json 1048576 float "$WL"
ncu -i /tmp/prof/bench.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/${R}_bench_source.csv.gz

#!/bin/bash
# Profiles the degree-padded kernel on the extended [[784,24,24]] graph (text summaries only).
set -u
ARITHS=${1:-int8}; TAG=${2:-ext_f10}
mkdir -p gpurun_out /tmp/prof
for a in $ARITHS; do
  rep=/tmp/prof/${a}_${TAG}
  ncu --set full --clock-control none --import-source on -k regex:decode_ell -s 2 -c 1 -f -o $rep \
      python tools/sweep_ext.py --ariths $a --iters 10:0 --shots 131072 > gpurun_out/prof_${a}_${TAG}.log 2>&1
  python tools/ncu_summary.py $rep.ncu-rep 1310720 > gpurun_out/prof_${a}_${TAG}.txt 2>&1
done

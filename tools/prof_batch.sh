#!/bin/bash
# Profiles the batch kernel for the given arithmetic modes on the GPU box and leaves only
# text summaries (+ gzipped per-instruction source pages) in gpurun_out/.
#   tools/prof_batch.sh "float int8 half" 10:0 tag
set -u
ARITHS=${1:-float}; ITERS=${2:-10:0}; TAG=${3:-f10}; SHOTS=${4:-131072}
IT=${ITERS%%:*}
mkdir -p gpurun_out /tmp/prof
for a in $ARITHS; do
  rep=/tmp/prof/${a}_${TAG}
  ncu --set full --clock-control none --import-source on -k regex:decode_lean -s 2 -c 1 -f -o $rep \
      python tools/sweep.py --ariths $a --npts 0 --iters $ITERS --shots $SHOTS > gpurun_out/prof_${a}_${TAG}.log 2>&1
  python tools/ncu_summary.py $rep.ncu-rep $((SHOTS * IT)) > gpurun_out/prof_${a}_${TAG}.txt 2>&1
  ncu -i $rep.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/prof_${a}_${TAG}_source.csv.gz
done

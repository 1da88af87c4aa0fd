#!/bin/bash
# On the GPU box: the round's closing evidence in one call - GPU tests, smoke, the default
# bench line, then the launch list + full capture of the bench kernel (tools/prof_bench.sh).
set -u
R=${1:-r1}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/gpu_tests.log)"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err; echo "reference arm rc=$?"
bash tools/prof_bench.sh $R
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
v = d.get("variants", {})
print(json.dumps({"value": d["value"], "e2e": d["e2e"]["value"], "frac": d["roofline"]["frac"],
                  "cpu": d["cpu_baseline"]["value"],
                  "campaign": {k: v[k]["trials_per_s"] for k in v if k.startswith("campaign")},
                  "lat_doorbell_p99": d["latency_us"]["fixed10_doorbell"]["p99"],
                  "lat_memcpy_p99": d["latency_us"]["fixed10_memcpy"]["p99"], "clocks": d["clocks"]}))
PY

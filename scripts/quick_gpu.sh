#!/bin/bash
# Quick GPU iteration: build, GPU tests (optional), decode bench with and without the L2 lookahead.
# usage (under gpurun): bash scripts/quick_gpu.sh TAG [pytest-args...]
TAG=${1:-q}; shift
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { tail -30 $OUT/build_$TAG.log; exit 1; }
if [ -z "$SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -q "$@" > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|ERROR|passed|failed" $OUT/pytest_gpu_$TAG.log | tail -15
fi
Q="--prefill-layers 0 --c4-steps 0 --c5-reps 0 --fused-base-reps 0 --no-cpu-baseline --e2e-steps 3 --steps 50 --warmup 5"

for la in 0; do
  timeout 300 python bench.py $Q --json-out $OUT/bench_${TAG}_la$la.json > $OUT/bench_${TAG}_la$la.log 2>&1
  echo "bench decode_kernel=$la rc=$?"
  python - $OUT/bench_${TAG}_la$la.json <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print("value %.0f tok/s  ms/step %.4f  frac %.3f  windows %s  e2e %.0f clocks %s" % (d["value"], d["ms_per_step"], d["roofline"]["frac"], d["windows"], d["e2e"]["value"], d["clocks"]))
PY
done

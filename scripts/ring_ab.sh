#!/bin/bash
# decode A/B: PDL pair vs persistent ring pair (and ring stage counts) on the c2 bench step.
# usage (under gpurun): bash scripts/ring_ab.sh TAG [ring configs...]
TAG=${1:-r}; shift
CFGS=${@:-0 1}
OUT=gpurun_out
mkdir -p $OUT
Q="--prefill-layers 0 --c4-steps 0 --c5-reps 0 --fused-base-reps 0 --cold-start 0 --no-cpu-baseline --e2e-steps 3 --steps 50 --warmup 5"
for c in $CFGS; do
  timeout 300 python bench.py $Q --decode-ring $c --json-out $OUT/ring_${TAG}_$c.json > $OUT/ring_${TAG}_$c.log 2>&1
  python - $OUT/ring_${TAG}_$c.json $c <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print("ring %-6s value %.0f tok/s  ms/step %.4f  frac %.3f  e2e %.0f" % (sys.argv[2], d["value"], d["ms_per_step"], d["roofline"]["frac"], d["e2e"]["value"]))
PY
done

#!/bin/bash
# decode A/B of the pipelined schedule (LORA_OPT_DECODE_CHUNK_KB) on the c2 bench step.
# usage (under gpurun): bash scripts/chunk_ab.sh TAG [chunk KB values...]
TAG=${1:-c}; shift
CFGS=${@:-0 8192}
OUT=gpurun_out
mkdir -p $OUT
Q="--prefill-layers 0 --c4-steps 0 --c5-reps 0 --fused-base-reps 0 --cold-start 0 --no-cpu-baseline --e2e-steps 3 --steps 50 --warmup 5"
for c in $CFGS; do
  timeout 300 python bench.py $Q --decode-chunk-kb $c --json-out $OUT/chunk_${TAG}_$c.json > $OUT/chunk_${TAG}_$c.log 2>&1
  python - $OUT/chunk_${TAG}_$c.json $c <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print("chunk %-6s KB  value %.0f tok/s  ms/step %.4f  frac %.3f  e2e %.0f" % (sys.argv[2], d["value"], d["ms_per_step"], d["roofline"]["frac"], d["e2e"]["value"]))
PY
done

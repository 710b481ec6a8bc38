#!/bin/bash
# A/B of compile-time variants on the c2 decode bench step (under gpurun):
#   bash scripts/build_ab.sh TAG "DEFS_A" "DEFS_B" ...   (each DEFS string -> LORA_BUILD_DEFS; "" = default)
TAG=$1; shift
OUT=gpurun_out
mkdir -p $OUT
Q="--prefill-layers 0 --c4-steps 0 --c5-reps 0 --fused-base-reps 0 --cold-start 0 --no-cpu-baseline --e2e-steps 3 --steps 50 --warmup 5"
i=0
for defs in "$@"; do
  LORA_BUILD_DEFS="$defs" python -c "import __graft_entry__ as g; g.build()" > $OUT/build_${TAG}_$i.log 2>&1 || { echo "build failed: $defs"; tail -5 $OUT/build_${TAG}_$i.log; continue; }
  for rep in 1 2; do
    LORA_BUILD_DEFS="$defs" timeout 300 python bench.py $Q --json-out $OUT/ab_${TAG}_${i}_$rep.json > $OUT/ab_${TAG}_${i}_$rep.log 2>&1
    python - $OUT/ab_${TAG}_${i}_$rep.json "$defs" <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print("[%-40s] value %.0f tok/s  ms/step %.4f  frac %.3f" % (sys.argv[2], d["value"], d["ms_per_step"], d["roofline"]["frac"]))
PY
  done
  i=$((i+1))
done

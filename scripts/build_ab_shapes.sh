#!/bin/bash
# A/B of compile-time variants on the c2 bench step AND the single-apply decode shapes (under gpurun):
#   bash scripts/build_ab_shapes.sh TAG "DEFS_A" "DEFS_B" ...   (each DEFS string -> LORA_BUILD_DEFS)
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
Q="--prefill-layers 0 --c4-steps 0 --c5-reps 0 --fused-base-reps 0 --cold-start 0 --no-cpu-baseline --e2e-steps 2 --steps 100 --warmup 5"
i=0
for defs in "$@"; do
  LORA_BUILD_DEFS="$defs" python -c "import __graft_entry__ as g; g.build()" > $OUT/build_${TAG}_$i.log 2>&1 || { echo "build failed: $defs"; tail -5 $OUT/build_${TAG}_$i.log; continue; }
  LORA_BUILD_DEFS="$defs" timeout 300 python bench.py $Q --json-out $OUT/ab_${TAG}_$i.json > $OUT/ab_${TAG}_$i.log 2>&1
  python - $OUT/ab_${TAG}_$i.json "$defs" <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print("[%-50s] c2 %.0f tok/s  frac %.3f" % (sys.argv[2], d["value"], d["roofline"]["frac"]))
PY
  LORA_BUILD_DEFS="$defs" timeout 300 python scripts/decode_shapes_bench.py 2>&1 | tail -1
  i=$((i+1))
done

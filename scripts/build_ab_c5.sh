#!/bin/bash
# A/B of compile-time variants on the c5 tp1/tp8 decode shapes and c2 (under gpurun)
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
Q="--prefill-layers 0 --c4-steps 0 --c5-reps 3 --fused-base-reps 0 --cold-start 0 --no-cpu-baseline --e2e-steps 2 --steps 100 --warmup 5"
i=0
for defs in "$@"; do
  LORA_BUILD_DEFS="$defs" python -c "import __graft_entry__ as g; g.build()" > $OUT/build_${TAG}_$i.log 2>&1 || { echo "build failed: $defs"; continue; }
  LORA_BUILD_DEFS="$defs" timeout 600 python bench.py $Q --json-out $OUT/ab_${TAG}_$i.json > $OUT/ab_${TAG}_$i.log 2>&1
  python - $OUT/ab_${TAG}_$i.json "$defs" <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
c5=d["c5"]["per_shape"]
s=" ".join("%s %.1f/%.1f" % (k, v["tp1"]["us_per_apply"], v["tp8"]["shard_kernels_us"]) for k, v in c5.items())
print("[%-30s] c2 %.0f  c5 tp1/tp8 us: %s" % (sys.argv[2], d["value"], s))
PY
  i=$((i+1))
done

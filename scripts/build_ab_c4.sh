#!/bin/bash
# A/B of compile-time variants on the c4 step (under gpurun)
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
i=0
for defs in "$@"; do
  LORA_BUILD_DEFS="$defs" python -c "import __graft_entry__ as g; g.build()" > $OUT/build_${TAG}_$i.log 2>&1 || { echo "build failed: $defs"; continue; }
  LORA_BUILD_DEFS="$defs" timeout 600 python bench.py --prefill-layers 0 --c5-reps 0 --fused-base-reps 0 --cold-start 0 --no-cpu-baseline --e2e-steps 2 --steps 20 --warmup 3 --c4-steps 80 --json-out $OUT/ab_${TAG}_$i.json > $OUT/ab_${TAG}_$i.log 2>&1
  python -c "
import json,sys; d=json.load(open(sys.argv[1])); c=d['c4']
print('[%-28s] c4 %.0f tok/s %.4f ms/step load GBps %.1f' % (sys.argv[2], c['value'], c['ms_per_step'], c['load_GBps_effective']))" $OUT/ab_${TAG}_$i.json "$defs"
  i=$((i+1))
done

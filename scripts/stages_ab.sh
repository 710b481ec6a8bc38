#!/bin/bash
# decode bench A/B over the streaming kernel's ring stages and the kernel pair.  usage: bash scripts/stages_ab.sh TAG
TAG=${1:-sa}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
Q="--prefill-layers 0 --c4-steps 0 --c5-reps 0 --fused-base-reps 0 --no-cpu-baseline --e2e-steps 3 --steps 50 --warmup 5"
for cfg in "0 2" "0 3" "1 2"; do
  set -- $cfg
  timeout 300 python bench.py $Q --decode-kernel $1 --decode-stages $2 --json-out gpurun_out/b_${TAG}_$1$2.json > /dev/null 2>&1
  python -c "import json;d=json.load(open('gpurun_out/b_${TAG}_$1$2.json'));print('kernel $1 stages $2: %.0f tok/s  %.4f ms/step  frac %.3f  e2e %.0f' % (d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value']))"
done

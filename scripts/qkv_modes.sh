#!/bin/bash
# c2 decode bench value per q/k/v issue mode (serial / 3 streams / lora_apply_multi)
for m in serial streams fused; do
  v=$(timeout 300 python bench.py --qkv-mode $m --prefill-layers 0 --c4-steps 0 --no-cpu-baseline --steps 500 --e2e-steps 3 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['avg_launch_us'], d['roofline']['frac'])")
  echo "qkv-mode $m -> tok/s, us/apply, frac: $v"
done

#!/bin/bash
# ncu --set full of the decode kernels (shrink + expand) from a short bench run. usage: bash scripts/ncu_kernels.sh TAG [regex]
TAG=${1:-x}; RX=${2:-lora_}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$RX -s 40 -c 4 -f -o gpurun_out/prof_$TAG \
   python bench.py --layers 4 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"

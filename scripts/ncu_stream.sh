#!/bin/bash
# ncu --set full of one streaming decode launch (q/k/v multi, grid 148) from a short bench run, plus the
# SASS source page.  usage: bash scripts/ncu_stream.sh TAG [skip]
TAG=${1:-s}; SKIP=${2:-8}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail -20 gpurun_out/build_$TAG.log; exit 1; }
Q="--layers 4 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --prefill-layers 0 --c4-steps 0 --c5-reps 0 --fused-base-reps 0 --min-window-ms 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lora_decode_stream -s $SKIP -c 1 -f \
   -o gpurun_out/prof_$TAG python bench.py $Q > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page details --csv > gpurun_out/details_$TAG.csv 2>/dev/null
python scripts/ncu_sass_hot.py gpurun_out/sass_$TAG.csv 40

#!/bin/bash
# One gpurun call: build, parity tests, smoke, bench, ncu launch list + full capture of the decode kernel.
# usage (from the repo root, under gpurun): bash scripts/gpu_round.sh [tag]
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { tail -30 $OUT/build_$TAG.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu_$TAG.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest_gpu_$TAG.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -4 $OUT/smoke_$TAG.log
timeout 600 python bench.py --json-out $OUT/bench_$TAG.json > $OUT/bench_$TAG.log 2>&1; echo "bench rc=$?"; tail -3 $OUT/bench_$TAG.log
if [ -z "$SKIP_NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv \
     python bench.py --layers 4 --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu-launch rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:lora_decode -s 40 -c 2 -f -o $OUT/prof_decode_$TAG \
     python bench.py --layers 4 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu-full rc=$?"
fi

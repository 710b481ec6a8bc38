#!/bin/bash
# Round-end evidence in one gpurun call: GPU tests, smoke, the default bench line, the ncu launch
# list and full captures (decode pair + prefill).  usage: bash scripts/final_round.sh TAG
TAG=${1:-r1d}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { tail -30 $OUT/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -3 $OUT/smoke_$TAG.log
timeout 900 python bench.py --json-out $OUT/bench_$TAG.json > $OUT/bench_$TAG.log 2>&1; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref_$TAG.log 2>&1; echo "ref rc=$?"; tail -1 $OUT/bench_ref_$TAG.log | cut -c1-200
bash scripts/profile_round.sh $TAG > $OUT/profile_$TAG.log 2>&1; tail -3 $OUT/profile_$TAG.log

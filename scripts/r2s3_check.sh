# decode change check: GPU tests, c2 bench, single-apply shapes (under gpurun)
mkdir -p gpurun_out
TAG=${1:-chk}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_$TAG.log
Q="--prefill-layers 0 --c4-steps 0 --c5-reps 0 --fused-base-reps 0 --cold-start 0 --no-cpu-baseline --e2e-steps 2 --steps 100 --warmup 5"
timeout 300 python bench.py $Q --json-out gpurun_out/bench_$TAG.json > gpurun_out/bench_$TAG.log 2>&1
python -c "import json,sys; d=json.load(open(sys.argv[1])); print('c2 %.0f tok/s frac %.3f' % (d['value'], d['roofline']['frac']))" gpurun_out/bench_$TAG.json
timeout 300 python scripts/decode_shapes_bench.py 2>&1 | tail -1

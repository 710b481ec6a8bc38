# tcgen05 expand variant: build with LORA_EXPAND_TC=1, decode parity tests, c2 bench, shapes (under gpurun)
mkdir -p gpurun_out
export LORA_BUILD_DEFS="-DLORA_EXPAND_TC=1"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_tc.log 2>&1 || { tail -30 gpurun_out/build_tc.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_tc.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/smoke_tc.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_tc.log | grep -E "passed|failed|Error|assert" | head
Q="--prefill-layers 0 --c4-steps 0 --c5-reps 0 --fused-base-reps 0 --cold-start 0 --no-cpu-baseline --e2e-steps 2 --steps 100 --warmup 5"
timeout 300 python bench.py $Q --json-out gpurun_out/bench_tc.json > gpurun_out/bench_tc.log 2>&1
python -c "import json,sys; d=json.load(open(sys.argv[1])); print('c2 %.0f tok/s frac %.3f' % (d['value'], d['roofline']['frac']))" gpurun_out/bench_tc.json
timeout 300 python scripts/decode_shapes_bench.py 2>&1 | tail -1
timeout 300 python scripts/trace_layer.py > gpurun_out/trace_layer_tc.txt 2>&1; tail -22 gpurun_out/trace_layer_tc.txt | grep -E "E data->mma|E wait->data|E wait->done|E mma->y"

# final evidence of the round: GPU tests, smoke, full bench line, reference arm, layer trace (under gpurun)
mkdir -p gpurun_out
TAG=${1:-r2f}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -4 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --json-out gpurun_out/bench_$TAG.json > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?"
timeout 300 python scripts/trace_layer.py > gpurun_out/trace_layer_$TAG.txt 2>&1; echo "trace rc=$?"
timeout 300 python scripts/decode_shapes_bench.py > gpurun_out/shapes_$TAG.txt 2>&1; tail -1 gpurun_out/shapes_$TAG.txt

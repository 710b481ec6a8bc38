# quick decode A/B: parity tests of the decode path, c2 bench (decode only), layer trace
mkdir -p gpurun_out
TAG=${1:-q}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
Q="--prefill-layers 0 --c4-steps 0 --c5-reps 0 --fused-base-reps 0 --no-cpu-baseline --cold-start 0 --e2e-steps 3 --steps 200 --warmup 5"
timeout 300 python bench.py $Q --json-out gpurun_out/bench_$TAG.json > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"
python - gpurun_out/bench_$TAG.json <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
print("value %.0f tok/s  ms/step %.4f  frac %.3f  windows %s" % (d["value"], d["ms_per_step"], d["roofline"]["frac"], d["windows"]))
PY
timeout 300 python scripts/trace_layer.py > gpurun_out/trace_layer_$TAG.txt 2>&1; echo trace rc=$?; head -16 gpurun_out/trace_layer_$TAG.txt | tail -13

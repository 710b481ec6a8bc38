# plan-cache check: GPU tests, host cost per call, c2 bench with e2e (under gpurun)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_h.log 2>&1 || { tail -30 gpurun_out/build_h.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_h.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_h.log
timeout 300 python scripts/host_cost.py 2>&1 | tail -4
Q="--prefill-layers 0 --c4-steps 0 --c5-reps 0 --fused-base-reps 0 --cold-start 0 --no-cpu-baseline --e2e-steps 20 --steps 100 --warmup 5"
timeout 300 python bench.py $Q --json-out gpurun_out/bench_h.json > gpurun_out/bench_h.log 2>&1
python -c "import json,sys; d=json.load(open(sys.argv[1])); print('c2 %.0f tok/s frac %.3f e2e %.0f tok/s (%.3f ms/step)' % (d['value'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['ms_per_step']))" gpurun_out/bench_h.json

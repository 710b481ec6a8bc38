# cold-start change check: GPU tests, c4 bench + cold_start (under gpurun)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_c4.log 2>&1 || { tail -30 gpurun_out/build_c4.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_c4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_c4.log
for i in 1 2; do
timeout 600 python bench.py --prefill-layers 0 --c5-reps 0 --fused-base-reps 0 --no-cpu-baseline --e2e-steps 2 --steps 50 --warmup 5 --json-out gpurun_out/bench_c4_$i.json > gpurun_out/bench_c4_$i.log 2>&1
python -c "
import json; d=json.load(open('gpurun_out/bench_c4_$i.json')); c=d['c4']; cs=d['cold_start']
print('c4 %.0f tok/s %.4f ms/step overlap %.3f load GBps %.1f | c2 %.0f' % (c['value'], c['ms_per_step'], c['overlap'], c['load_GBps_effective'], d['value']))
print({r: (v['memcpy_best_us'], v['gather_kernel_best_us']) for r, v in cs['load_by_rank'].items()})"
done

# balanced prefill tiling A/B: parity tests + c3 prefill bench for each build (under gpurun)
mkdir -p gpurun_out
for defs in "" "-DLORA_PF_BALANCE=1"; do
  export LORA_BUILD_DEFS="$defs"
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_pfb.log 2>&1 || { tail -20 gpurun_out/build_pfb.log; exit 1; }
  echo "== [$defs]"
  timeout 600 python -m pytest tests -m gpu -q -x -k "prefill or c3 or tiles or split or fused or c4" 2>&1 | tail -2
  for i in 1 2; do
  timeout 600 python bench.py --prefill-layers 2 --prefill-steps 20 --c4-steps 0 --c5-reps 3 --fused-base-reps 0 --cold-start 0 --no-cpu-baseline --e2e-steps 2 --steps 20 --warmup 3 --json-out gpurun_out/pfb.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/pfb.json')); p=d['prefill']; c=d['c5']['prefill_tp1']
print('c3 %.2f us/apply frac %.4f | c5 q %.1f gate %.1f down %.1f' % (p['ms_per_apply']*1e3, p['roofline']['frac'], c['q']['us_per_apply'], c['gate']['us_per_apply'], c['down']['us_per_apply']))"
  done
done

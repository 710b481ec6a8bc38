# decode shapes A/B: the round-start library (gpurun_in/liblora_old.so) vs the current build; q/k/v issue modes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_sh.log 2>&1 || { tail -30 gpurun_out/build_sh.log; exit 1; }
LIB=paper_2401_11240_b200/lib/liblora.so
cp $LIB /tmp/liblora_new.so
for v in old new; do
  cp /tmp/liblora_$v.so $LIB 2>/dev/null || cp gpurun_in/liblora_old.so $LIB
  echo "== $v"; timeout 300 python scripts/decode_shapes_bench.py 2>&1 | tail -6
done
cp /tmp/liblora_new.so $LIB
Q="--prefill-layers 0 --c4-steps 0 --c5-reps 0 --fused-base-reps 0 --cold-start 0 --no-cpu-baseline --e2e-steps 2 --steps 100 --warmup 5"
for m in serial streams fused; do
  timeout 300 python bench.py $Q --qkv-mode $m --json-out gpurun_out/qkv_$m.json > gpurun_out/qkv_$m.log 2>&1
  python -c "import json,sys; d=json.load(open(sys.argv[1])); print('qkv-mode %s value %.0f tok/s frac %.3f' % (sys.argv[2], d['value'], d['roofline']['frac']))" gpurun_out/qkv_$m.json $m
done

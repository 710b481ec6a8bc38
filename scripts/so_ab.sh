#!/bin/bash
# A/B of two prebuilt liblora.so files on the c2 decode bench (under gpurun):
#   bash scripts/so_ab.sh TAG A.so B.so   (each run twice, interleaved; the in-tree .so is restored)
TAG=$1; A=$2; B=$3
OUT=gpurun_out; mkdir -p $OUT
LIB=paper_2401_11240_b200/lib/liblora.so
cp $LIB /tmp/liblora_orig.so
Q="--prefill-layers 0 --c4-steps 0 --c5-reps 0 --fused-base-reps 0 --cold-start 0 --no-cpu-baseline --e2e-steps 2 --steps 50 --warmup 5"
for rep in 1 2; do
  for v in A B; do
    if [ $v = A ]; then cp $A $LIB; else cp $B $LIB; fi
    timeout 300 python bench.py $Q --json-out $OUT/soab_${TAG}_${v}_$rep.json > $OUT/soab_${TAG}_${v}_$rep.log 2>&1
    python -c "import json,sys; d=json.load(open(sys.argv[1])); print('%s rep%s value %.0f tok/s frac %.3f' % (sys.argv[2], sys.argv[3], d['value'], d['roofline']['frac']))" $OUT/soab_${TAG}_${v}_$rep.json $v $rep
  done
done
cp /tmp/liblora_orig.so $LIB

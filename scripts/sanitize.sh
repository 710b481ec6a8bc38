#!/bin/bash
# compute-sanitizer over every kernel path (scripts/sanitize_cases.py), one tool at a time; writes
# gpurun_out/sanitize_<tool>_<case>.log and a summary.  usage: bash scripts/sanitize.sh [tools] [cases]
TOOLS=${1:-"memcheck racecheck synccheck initcheck"}
CASES=${2:-"c1 c1p c2 c2_multi c5_splitk c5_colsplit fused_base tp_split load_kernel"}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_san.log 2>&1 || { tail -20 $OUT/build_san.log; exit 1; }
SUM=$OUT/sanitize_summary_${SUMTAG:-all}.txt
echo "# compute-sanitizer $(compute-sanitizer --version | tail -1) on $(nvidia-smi --query-gpu=name --format=csv,noheader | head -1)" > $SUM
for t in $TOOLS; do
  for c in $CASES; do
    timeout 900 compute-sanitizer --tool $t --target-processes all --print-limit 20 \
      python scripts/sanitize_cases.py $c > $OUT/sanitize_${t}_${c}.log 2>&1
    rc=$?
    res=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $OUT/sanitize_${t}_${c}.log | tail -1)
    ok=$(grep -c "^$c " $OUT/sanitize_${t}_${c}.log)
    printf "%-10s %-12s rc=%-3s case_ok=%s  %s\n" $t $c $rc $ok "$res" | tee -a $SUM
  done
done

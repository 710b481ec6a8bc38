#!/bin/bash
# Profiles for profiles/: ncu launch list of a short bench run, and full captures of the decode
# (shrink+expand) and prefill kernels.  Run under gpurun from the repo root: bash scripts/profile_round.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
   --log-file gpurun_out/launches_$TAG.csv \
   python bench.py --layers 4 --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline --prefill-layers 1 --prefill-steps 2 --c4-steps 0 --c5-reps 0 \
   > gpurun_out/launches_$TAG.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lora_(shrink|expand)" -s 8 -c 4 -f \
   -o gpurun_out/prof_decode_$TAG \
   python scripts/ncu_decode_step.py > gpurun_out/prof_decode_$TAG.log 2>&1
echo "decode full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lora_prefill" -s 4 -c 2 -f \
   -o gpurun_out/prof_prefill_$TAG \
   python bench.py --layers 1 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --prefill-layers 1 --prefill-steps 2 --c4-steps 0 --c5-reps 0 \
   > gpurun_out/prof_prefill_$TAG.log 2>&1
echo "prefill full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lora_fused_gemm" -s 2 -c 1 -f \
   -o gpurun_out/prof_fused_$TAG \
   python scripts/fused_base_bench.py > gpurun_out/prof_fused_$TAG.log 2>&1
echo "fused full rc=$?"

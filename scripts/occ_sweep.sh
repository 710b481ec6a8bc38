# occupancy sweep of the decode pair (experiment knobs LORA_EXP_SSMEM / LORA_EXP_ESMEM pad the
# dynamic smem of the shrink / expand CTAs); prints the c2 bench value per setting
for cfg in ${CFGS:-"0 0" "50000 0" "57000 0" "66000 0" "75000 0" "90000 0" "113000 0"}; do
  set -- ${cfg/:/ }
  v=$(LORA_EXP_SSMEM=$1 LORA_EXP_ESMEM=$2 timeout 300 python bench.py --prefill-layers 0 --c4-steps 0 --c5-reps 0 --e2e-steps 2 --no-cpu-baseline --steps 300 2>&1 | tail -1 | python -c "import sys,json; print(json.loads(sys.stdin.read())['value'])")
  echo "S=$1 E=$2 -> $v"
done

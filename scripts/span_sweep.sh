#!/bin/bash
# Sweep of the cluster-span decode knobs on c2: "cluster target stage stages" per setting,
# prints the summary lines of scripts/trace_span.py.  usage: bash scripts/span_sweep.sh [NP]
NP=${1:-8}
while read -r cl tg sb ns; do
  [ -z "$cl" ] && continue
  echo "== cluster $cl target $tg stage $sb x $ns"
  LORA_SPAN_CLUSTER=$cl LORA_SPAN_TARGET=$tg LORA_SPAN_STAGE=$sb LORA_SPAN_STAGES=$ns timeout 120 \
    python scripts/trace_span.py c2 $NP 2>&1 | grep -E "graph of|med|resident|Error|error" | head -20
done < ${SWEEP_FILE:-scripts/span_sweep.txt}

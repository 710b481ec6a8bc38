mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbh scripts/microbench_hmma.cu && /tmp/mbh > gpurun_out/hmma.txt 2>&1
cat gpurun_out/hmma.txt
SKIP_NCU=1 bash scripts/gpu_round.sh r2s3
timeout 300 python scripts/trace_layer.py > gpurun_out/trace_layer_r2s3.txt 2>&1; echo trace rc=$?

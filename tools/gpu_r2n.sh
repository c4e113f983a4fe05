mkdir -p gpurun_out
CMP_ARGS="--config tnl1b --no-layer" bash tools/cmp_variants.sh > gpurun_out/r2n_variants_tnl1b.txt 2>&1
CMP_ARGS="--no-layer" bash tools/cmp_variants.sh > gpurun_out/r2n_variants_tnl04b.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipe_rate tools/pipe_rate.cu && /tmp/pipe_rate > gpurun_out/r2n_pipe_rate.txt 2>&1

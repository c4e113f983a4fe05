mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2404_02882_b200/csrc tools/l2_bw.cu -o /tmp/l2_bw -lcuda && /tmp/l2_bw > gpurun_out/r2o_l2_bw.txt 2>&1

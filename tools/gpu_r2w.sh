mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2404_02882_b200/csrc tools/tmem_bw.cu -o /tmp/tmem_bw && /tmp/tmem_bw > gpurun_out/r2w_tmem_bw.txt 2>&1

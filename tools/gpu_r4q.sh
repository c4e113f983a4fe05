# head_dim 128 segment length: TNL-1B forced lengths (k = 11 default, 22, 28 blocks) and the TNL-7B block cap
bash tools/sweep_env.sh LASP_SEG_LEN "0 2816 3584" --config tnl1b > gpurun_out/r4q_seglen_tnl1b.txt 2>&1; cat gpurun_out/r4q_seglen_tnl1b.txt
bash tools/sweep_env.sh LASP_MAX_SEG_BLOCKS "0 24 28 32" --config tnl7b --steps 10 > gpurun_out/r4q_maxblocks_tnl7b.txt 2>&1; cat gpurun_out/r4q_maxblocks_tnl7b.txt

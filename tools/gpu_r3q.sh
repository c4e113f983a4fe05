mkdir -p gpurun_out
for cfg in "2 768 4" "2 32768 4" "2 768 16" "2 32768 16"; do echo "== $cfg" >> gpurun_out/r3q.txt; timeout 120 python scratch/p2p_big.py $cfg >> gpurun_out/r3q.txt 2>&1; done

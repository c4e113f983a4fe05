mkdir -p gpurun_out
for ex in both p2p; do
  timeout 300 python bench.py --loopback 4 --steps 5 --warmup 2 --no-e2e --exchange $ex > gpurun_out/r3p_$ex.json 2> gpurun_out/r3p_$ex.err; echo "$ex rc=$?" >> gpurun_out/r3p_rc.txt
done
timeout 300 python bench.py --loopback 2 --steps 5 --warmup 2 --no-e2e --exchange p2p > gpurun_out/r3p_p2p2.json 2> gpurun_out/r3p_p2p2.err; echo "p2p world2 rc=$?" >> gpurun_out/r3p_rc.txt

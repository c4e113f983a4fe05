# state copy of block j before block j's u . c (default) vs u . c of block j + 1 at the end of block j (xKUEARLY)
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r4n_pytest_parity.txt 2>&1; tail -2 gpurun_out/r4n_pytest_parity.txt
bash tools/cmp3.sh "liblasp_xKUEARLY.so liblasp.so" > gpurun_out/r4n_ab_kulate_tnl04b.txt 2>&1; cat gpurun_out/r4n_ab_kulate_tnl04b.txt
bash tools/cmp3.sh "liblasp_xKUEARLY.so liblasp.so" --config tnl1b > gpurun_out/r4n_ab_kulate_tnl1b.txt 2>&1; cat gpurun_out/r4n_ab_kulate_tnl1b.txt

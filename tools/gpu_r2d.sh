mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gqa or config2 or deterministic" 2>&1 | tail -3 > gpurun_out/r2d_pytest.txt
bash tools/cmp3.sh "liblasp_r1.so liblasp_old.so liblasp.so" > gpurun_out/r2d_cmp_tnl04b.txt 2>&1
bash tools/cmp3.sh "liblasp_r1.so liblasp_old.so liblasp.so" --config tnl1b > gpurun_out/r2d_cmp_tnl1b.txt 2>&1

mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool initcheck python tools/sanitize_gla.py 2>&1 | tail -6 > gpurun_out/r3e_initcheck_gla.txt

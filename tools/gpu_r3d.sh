mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool initcheck --kernel-name kns=lasp --print-limit 50 python tools/sanitize_case.py > gpurun_out/r3d_initcheck_lasp.txt 2>&1
grep -E "ERROR SUMMARY|Uninitialized|^=========     at " gpurun_out/r3d_initcheck_lasp.txt | sort | uniq -c | sort -rn | head -20 > gpurun_out/r3d_summary.txt

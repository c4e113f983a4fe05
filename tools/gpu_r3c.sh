mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool initcheck --print-limit 400 python tools/sanitize_case.py 2>&1 | grep -E "Uninitialized|at |by thread|Address|in " | awk '{$1=$1};1' | sort | uniq -c | sort -rn | head -60 > gpurun_out/r3c_initcheck.txt

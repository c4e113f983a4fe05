# compute-sanitizer over every kernel family on the current code (new P-chunk / c-tile barriers, state prefetch,
# templated prefix kernel)
mkdir -p gpurun_out
{ echo "== memcheck"; timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_case.py 2>&1 | tail -12
  echo "== racecheck"; timeout 1200 compute-sanitizer --tool racecheck python tools/sanitize_case.py 2>&1 | tail -12
  echo "== synccheck"; timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_case.py 2>&1 | tail -12; } > gpurun_out/r4k_sanitizer.txt 2>&1
cat gpurun_out/r4k_sanitizer.txt
{ echo "== memcheck, separate prefix kernels (LASP_NO_FUSED_FOLD=1)"; LASP_NO_FUSED_FOLD=1 timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_case.py 2>&1 | tail -12
  echo "== racecheck, separate prefix kernels"; LASP_NO_FUSED_FOLD=1 timeout 1200 compute-sanitizer --tool racecheck python tools/sanitize_case.py 2>&1 | tail -4; } >> gpurun_out/r4k_sanitizer.txt 2>&1
tail -18 gpurun_out/r4k_sanitizer.txt

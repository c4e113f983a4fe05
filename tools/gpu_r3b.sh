mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool" >> gpurun_out/r3b_sanitizer.txt
  timeout 1200 compute-sanitizer --tool $tool python tools/sanitize_case.py 2>&1 | tail -12 >> gpurun_out/r3b_sanitizer.txt
done

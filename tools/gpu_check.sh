timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_case.py 2>&1 | tail -4
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize_case.py 2>&1 | tail -4

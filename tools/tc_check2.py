import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.tc_check import run
cases = {"a": (1024, 2, 64, 1, None), "b": (1000, 1, 64, 1, 0.9), "c": (1000, 2, 64, 1, None), "d": (896, 1, 64, 0, 0.9)}
for k in sys.argv[1:]:
    run(*cases[k])

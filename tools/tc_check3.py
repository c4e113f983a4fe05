import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.tc_check import run
N, H = int(sys.argv[1]), int(sys.argv[2])
run(N, H, 64, 0, None)

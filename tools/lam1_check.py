import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.tc_check import run
run(int(sys.argv[1]), 1, 64, 3, 1.0)

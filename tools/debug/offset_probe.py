import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from tools.gemm_probe import run
which = sys.argv[1]
offs = {"rows": (5, 0, 7, 0, 2, 0), "acol8": (0, 8, 0, 0, 0, 0), "acol3": (0, 3, 0, 0, 0, 0),
        "bcol8": (0, 0, 0, 8, 0, 0), "bcol11": (0, 0, 0, 11, 0, 0), "ccol4": (0, 0, 0, 0, 0, 4),
        "ccol1": (0, 0, 0, 0, 0, 1), "aligned_all": (64, 64, 64, 64, 64, 64)}[which]
print(which, run(300, 200, 100, off=offs))

import cProfile, pstats, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2510_08874_b200 import ExecConfig, execute_multiply
from paper_2510_08874_b200.cli import build_problem
fab, A, B, C, a, b = build_problem(600, 520, 900, 4, "misaligned", "col", "row", 1, 1, 2, seed=17)
execute_multiply(A, B, C, ExecConfig()); torch.cuda.synchronize()
t=time.time()
pr = cProfile.Profile(); pr.enable()
for _ in range(3):
    execute_multiply(A, B, C, ExecConfig()); torch.cuda.synchronize()
pr.disable()
print("per multiply", (time.time()-t)/3)
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)

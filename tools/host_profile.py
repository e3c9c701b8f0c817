"""cProfile of the host side of one bench step (reset + insert + 10 doubling rounds)."""
import cProfile
import os
import pstats
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2209_00103_b200 as gg
import bench

step = bench.Step(gg, torch, torch.device("cuda", 0))
for _ in range(5):
    step.run(False)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    step.run(False)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e3*(t1-t0)/20:.3f} ms/step, wall {1e3*(t2-t0)/20:.3f} ms/step")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    step.run(False)
pr.disable()
torch.cuda.synchronize()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)

import os, sys
sys.path.insert(0, os.getcwd())
import synth
from paper_1805_06607_b200 import mrab
p = synth.make_config(3, "full")
plan = mrab.Plan(p); ctx = mrab.Context(plan, p.q0)
ctx.step(p.history_m - 1 + 3)
for k in (0, 3, 4, 5):
    ms, by = ctx.time_kernel(k, 1, reps=20, flush_l2=True)
    print(k, f"{ms*1e3:.1f} us  {by/ms/1e6:.0f} GB/s  bytes {by/1e6:.1f} MB")

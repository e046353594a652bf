"""Time the RHS pair (mrab_time_kernel 0) of one mesh: CFG, MESH env."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1805_06607_b200 import mrab
p = synth.make_config(int(os.environ.get("CFG", "4")), "full")
ctx = mrab.Context(mrab.Plan(p), p.q0)
ctx.step(p.history_m - 1 + 1)
for g in [int(x) for x in os.environ.get("MESH", "1").split(",")]:
    ms, by = ctx.time_kernel(0, g, reps=20, flush_l2=True)
    print(f"mesh {g}: pair {ms*1e3:.1f} us")

"""Create config C (default 3) and launch the fused 2-D RHS kernel of mesh G once, exactly as
the MRAB step launches it (mrab_time_kernel) -- a clean target for ncu."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1805_06607_b200 import mrab
p = synth.make_config(int(os.environ.get("CFG", "3")), "full")
plan = mrab.Plan(p)
ctx = mrab.Context(plan, p.q0)
g = int(os.environ.get("MESH", "1"))
print(ctx.time_kernel(int(os.environ.get("KERNEL", "0")), g, reps=int(os.environ.get("REPS", "1")), flush_l2=True))

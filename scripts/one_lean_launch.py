"""One launch of the lean-only 2-D RHS kernel over the interior tiles of the config-3
background (mrab_time_kernel kernel 3) -- an ncu target."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1805_06607_b200 import mrab
p = synth.make_config(3, "full")
plan = mrab.Plan(p); ctx = mrab.Context(plan, p.q0)
ctx.step(p.history_m - 1 + 1)
print(ctx.time_kernel(int(os.environ.get("KERNEL", "3")), 1, reps=1, flush_l2=True))

"""One launch of a 2-D RHS diagnostic on the config-3 background (mrab_time_kernel kernel
KERNEL: 3 lean-only kernel on the interior tiles, 4 mixed kernel on them, 5 the non-interior
tiles) with no step before it, so that it is the first k_rhs2d launch -- an ncu target."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_1805_06607_b200 import mrab
p = synth.make_config(3, "full")
plan = mrab.Plan(p); ctx = mrab.Context(plan, p.q0)
print(ctx.time_kernel(int(os.environ.get("KERNEL", "3")), 1, reps=1, flush_l2=True))

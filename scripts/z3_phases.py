"""Per-phase cycle accounting of k_rhs3z (needs the -DMRAB_Z3_PROF build: MRAB_Z3_PROF=1
python paper_1805_06607_b200/build.py --force).  Prints each phase's share of CTA thread 0's
cycles over one launch of the RHS of mesh MESH of config CFG."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1805_06607_b200 import mrab
p = synth.make_config(int(os.environ.get("CFG", "4")), "full")
ctx = mrab.Context(mrab.Plan(p), p.q0)
buf = torch.zeros(8, dtype=torch.int64, device="cuda")
ctx.set_trace(buf.data_ptr())
ms, _ = ctx.time_kernel(0, int(os.environ.get("MESH", "1")), reps=1, flush_l2=True)
v = buf.cpu().tolist()
names = ["wait+barrier", "convert+barrier", "flux(G)+barrier", "scatter+div", "complete+issue_ep",
         "warm-up steps", "steps", "issue box/outer"]
tot = sum(v[:6]) + v[7]
print(f"launch {ms*1e3:.0f} us; steps (all CTAs) {v[6]}; cycles per step {tot / max(v[6], 1):.0f}")
for n, x in [(names[i], v[i]) for i in (0, 1, 2, 7, 3, 4, 5)]:
    print(f"  {n:18s} {100 * x / tot:5.1f} %  {x / max(v[6], 1):8.0f} cyc/step")

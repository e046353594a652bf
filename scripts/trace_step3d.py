"""Launch timeline of one 3-D MRAB macro step (mrab_set_trace): the task-flow schedule stamps
the start and end of every node (RHS pair, donor preparation, gather) with a 1-thread kernel
on the node's stream; printed relative to the first stamp (globaltimer, us)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1805_06607_b200 import mrab

KIND = {4: "flux", 5: "div", 6: "prep", 7: "gather"}
cid = int(os.environ.get("CFG", "5"))
kw = {"order_n": int(os.environ["ORDER"])} if "ORDER" in os.environ else {}
p = synth.make_config(cid, os.environ.get("SCALE", "full"), **kw)
plan = mrab.Plan(p)
ctx = mrab.Context(plan, p.q0)
ctx.step(p.history_m - 1 + 2)
cap = 1 << 14
buf = torch.zeros(2 + 5 * cap, dtype=torch.int64, device="cuda")
buf[1] = cap
ctx.set_trace(buf.data_ptr())
ctx.step(2)   # re-capture the traced graphs
torch.cuda.synchronize()
buf[0] = 0
torch.cuda.synchronize()
ctx.step(1)
torch.cuda.synchronize()
n = int(buf[0].item())
rec = buf[2:2 + 5 * n].view(-1, 5).cpu().numpy()
t0 = rec[:, 1].min()
ev = {}
for tagsm, a, b, _, _ in rec:
    tag = int(tagsm) & 0xffff
    key = (tag >> 12) & 7, (tag >> 8) & 15, tag & 255
    ev.setdefault(key, [None, None])[(tag >> 15) & 1] = (a - t0) / 1e3
rows = sorted(ev.items(), key=lambda kv: kv[1][0] if kv[1][0] is not None else 0)
print(f"config {cid}: {len(rows)} nodes, span {(rec[:, 1].max() - t0) / 1e3:.1f} us")
busy = 0.0
for (kind, g, j), (s, e) in rows:
    print(f"{KIND.get(kind, kind):6s} mesh {g} j {j:2d}: {s:9.1f} -> {e:9.1f} us ({e - s:8.1f})")
    busy += e - s
print(f"sum of node spans {busy:.1f} us (serial equivalent)")

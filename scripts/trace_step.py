"""Launch timeline of one 2-D MRAB macro step (mrab_set_trace): per launch its CTA count
and [first CTA start, last CTA end] relative to the step's first CTA (globaltimer ns)."""
import os
import sys
from collections import defaultdict
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1805_06607_b200 import mrab

KIND = {1: "rhs", 2: "gather", 3: "bulk"}
p = synth.make_config(int(os.environ.get("CFG", "3")), "full")
plan = mrab.Plan(p)
ctx = mrab.Context(plan, p.q0)
ctx.step(p.history_m - 1 + 4)
cap = 1 << 20
buf = torch.zeros(2 + 5 * cap, dtype=torch.int64, device="cuda")
buf[1] = cap
ctx.set_trace(buf.data_ptr())
ctx.step(3)                      # capture the traced graphs
torch.cuda.synchronize()
for rep in range(int(os.environ.get("REPS", "2"))):
    buf[0] = 0
    torch.cuda.synchronize()
    ctx.step(1)
    torch.cuda.synchronize()
    n = int(buf[0].item())
    rec = buf[2:2 + 5 * min(n, cap)].view(-1, 5).cpu().numpy()
    t00 = rec[:, 1].min()
    L = defaultdict(list)
    for tagsm, a, b, ta, tb in rec:
        L[int(tagsm) & 0xffff].append((a - t00, b - t00, (int(tagsm) >> 16) & 0xffffffffff,
                                       (ta - a) / 1e3 if ta else 0.0, (tb - ta) / 1e3 if tb else 0.0))
    print(f"--- macro step {rep}: {n} CTA records, span {(rec[:, 2].max() - t00) / 1e3:.1f} us")
    for tag, v in sorted(L.items(), key=lambda kv: min(x[0] for x in kv[1])):
        s = min(x[0] for x in v) / 1e3
        e = max(x[1] for x in v) / 1e3
        d = sorted((x[1] - x[0]) / 1e3 for x in v)
        print(f"{KIND.get(tag >> 12, tag >> 12):6s} mesh {(tag >> 8) & 15} j {tag & 255:2d}: "
              f"{len(v):5d} CTAs  {s:7.1f} -> {e:7.1f} us ({e - s:6.1f})  CTA median {d[len(d) // 2]:.1f} max {d[-1]:.1f} us")
        if os.environ.get("MARCH_MAP") and 300 < len(v) < 1000 and rep == 0:
            # row-marching launch: CTA b = item b = (row chunk b // ns, strip b % ns)
            ns = int(os.environ.get("MARCH_NS", "9"))
            dur = {x[2]: (x[1] - x[0]) / 1e3 for x in v}
            nch = (max(dur) + ns) // ns
            print("    CTA duration (us) by row chunk (rows) x strip (columns):")
            for ch in range(nch):
                print("    " + " ".join(f"{dur.get(ch * ns + s_, 0):5.0f}" for s_ in range(ns)))
        if os.environ.get("SMALL_MAP") and 100 <= len(v) <= 300 and rep == 0 and (tag >> 12) == 1:
            byidx = sorted(((x[2], (x[1] - x[0]) / 1e3, x[3], x[4]) for x in v))
            for lo in range(0, len(byidx), 32):
                ch = byidx[lo:lo + 32]
                ds = sorted(c[1] for c in ch)
                pa = sorted(c[2] for c in ch)[len(ch) // 2]
                pb = sorted(c[3] for c in ch)[len(ch) // 2]
                print(f"    CTAs {lo:4d}..{lo + len(ch) - 1:4d}: dur median {ds[len(ds) // 2]:5.1f} max {ds[-1]:5.1f}  "
                      f"phase A {pa:5.1f} B {pb:5.1f} C {ds[len(ds) // 2] - pa - pb:5.1f}")
        if len(v) > 1000 and rep == 0:
            # list order = non-interior tiles first: durations by CTA index bucket
            byidx = sorted(((x[2], (x[1] - x[0]) / 1e3, x[0] / 1e3, x[3], x[4]) for x in v))
            for lo in range(0, len(byidx), 128):
                ch = byidx[lo:lo + 128]
                ds = sorted(c[1] for c in ch)
                pa = sorted(c[3] for c in ch)[len(ch) // 2]
                pb = sorted(c[4] for c in ch)[len(ch) // 2]
                print(f"    CTAs {lo:5d}..{lo + len(ch) - 1:5d}: dur median {ds[len(ds) // 2]:5.1f} max {ds[-1]:5.1f}  "
                      f"phase A {pa:5.1f} B {pb:5.1f} C {ds[len(ds) // 2] - pa - pb:5.1f}  start {min(c[2] for c in ch):6.1f}..{max(c[2] for c in ch):6.1f}")

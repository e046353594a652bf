"""Brief summary of an ncu report: key counters, stall ratios and the hottest source lines."""
import csv
import subprocess
import sys

rep = sys.argv[1]
nlines = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum",
        "lts__t_bytes.sum"]
for k in keys:
    if k in h:
        print(f"{k} = {v[h.index(k)]} {u[h.index(k)]}")
st = [(float(v[i]), k) for i, k in enumerate(h)
      if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio") and v[i]]
for val, k in sorted(st, reverse=True)[:10]:
    print(f"  stall {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:24s} {val:.2f}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
start = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[start]
ci, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
agg, cur = {}, None
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    if r[0]:
        cur = (r[0], r[1][:100])
    try:
        a = agg.setdefault(cur, [0.0, 0.0])
        a[0] += float(r[ci] or 0)
        a[1] += float(r[ii] or 0)
    except ValueError:
        pass
ts = sum(x[0] for x in agg.values()) or 1
ti = sum(x[1] for x in agg.values()) or 1
for k, x in sorted(agg.items(), key=lambda kv: -kv[1][0])[:nlines]:
    print(f"{x[0] / ts * 100:5.1f}% samp {x[1] / ti * 100:5.1f}% inst  L{k[0]}: {k[1]}")

import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iE = hdr.index("Instructions Executed"); iS = hdr.index("Source"); iW = hdr.index("Warp Stall Sampling (All Samples)")
hist = collections.Counter(); stall = collections.Counter(); tot = 0; tots = 0
seq = []
for r in rows[2:]:
    if len(r) <= iE or not r[iE].replace(".","").isdigit(): continue
    op = r[iS].split()[0] if r[iS].split() else "?"
    if op.startswith("@"): op = r[iS].split()[1]
    base = op.split(".")[0]
    n = float(r[iE] or 0); s = float(r[iW] or 0)
    hist[base] += n; stall[base] += s; tot += n; tots += s
    seq.append((r[iS].strip(), n, s))
print("total warp inst %.3g, stall samples %d" % (tot, tots))
for k, v in hist.most_common(25):
    print(f"{k:10s} {v/tot*100:5.1f}%  stall {stall[k]/tots*100:5.1f}%")
if len(sys.argv) > 2:
    # top stall instructions
    for s in sorted(seq, key=lambda x: -x[2])[:25]:
        print(f"{s[2]:6.0f} {s[1]:10.0f}  {s[0][:90]}")

"""Split an ncu SASS source-page CSV (--page source --csv --print-source sass) into
contiguous regions of executed code and report per region: instructions executed,
share, warp-stall samples, and the opcode mix.  Usage: python ncu_regions.py src.csv"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iex, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
recs = []
for r in rows[2:]:
    try:
        recs.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[isamp] or 0)))
    except (ValueError, IndexError):
        pass
base = recs[0][0]
tot = sum(x[2] for x in recs); tots = sum(x[3] for x in recs)
# regions: split where the execution count changes by > 4x between neighbours
regs = []; cur = [recs[0]]
for a, b in zip(recs, recs[1:]):
    ca, cb = a[2], b[2]
    if (ca == 0) != (cb == 0) or (ca and cb and max(ca, cb) > 4 * min(ca, cb)):
        regs.append(cur); cur = []
    cur.append(b)
regs.append(cur)
print("total warp-instructions %.4g, samples %d" % (tot, tots))
for g in regs:
    ex = sum(x[2] for x in g)
    if ex < 0.003 * tot: continue
    ops = collections.Counter()
    for x in g:
        op = x[1].split()[0]
        if op.startswith("@"): op = x[1].split()[1]
        ops[op.split(".")[0]] += x[2]
    print("%05x-%05x n=%4d exec=%.4g (%5.1f%%) samples=%5.1f%%  %s" % (g[0][0] - base, g[-1][0] - base, len(g), ex,
          100.0 * ex / tot, 100.0 * sum(x[3] for x in g) / max(1, tots),
          ", ".join("%s:%.0f%%" % (k, 100.0 * v / ex) for k, v in ops.most_common(6))))

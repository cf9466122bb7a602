"""Summarise ncu evidence (launch list CSV + one --set full report) into markdown."""
import csv, io, subprocess, sys
from collections import defaultdict

def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    kn, mv, mu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr_i + 1:]:
        if len(r) <= mv:
            continue
        v = float(r[mv].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(r[mu], 1.0)
        name = r[kn].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append("| `%s` | %d | %.1f | %.2f%% |" % (k[:90], n, us, 100 * us / tot))
    return "\n".join(out)

def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    keys = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "smsp__thread_inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"]
    out = ["| metric | value | unit |", "|---|---|---|"]
    for k in keys:
        if k in d:
            out.append("| %s | %s | %s |" % (k, d[k][0], d[k][1]))
    st = sorted(((float(d[k][0] or 0), k) for k in d if k.startswith("smsp__average_warps_issue_stalled")
                 and k.endswith("_per_issue_active.ratio")), reverse=True)[:10]
    out.append("\nTop warp-stall reasons (cycles per issued instruction):\n")
    out += ["- %s: %.3f" % (k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), v)
            for v, k in st]
    return "\n".join(out), d

if __name__ == "__main__":
    tag, lcsv, rep = sys.argv[1:4]
    md, d = report(rep)
    print("# ncu evidence %s\n\n## Launch list (`gpu__time_duration.sum`, serialised, cold)\n\n%s\n\n## DP kernel, `--set full`\n\n%s\n"
          % (tag, launches(lcsv), md))

"""Measured instruction counts per cell of one DP launch, from an `ncu --set full` report,
into profiles/issue_<config>.json (read by bench.py: roofline.issue_slots_per_cell_ncu).

    python scripts/ncu_issue.py <report.ncu-rep> <config> <Z> <N> <M> [precision]

issue slots per cell   = smsp__inst_executed.sum * 32 / (Z*N*M)   (warp instructions x lanes)
thread inst per cell   = sass__thread_inst_executed_true_per_opcode / (Z*N*M) (predicated-on lanes)
issue_active           = smsp__issue_active.avg.pct_of_peak_sustained_active / 100
"""
import csv
import io
import json
import os
import subprocess
import sys


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            d[h] = (v, u)
        res.append(d)
    return res


def num(d, key):
    v, u = d[key]
    x = float(v.replace(",", ""))
    return x * {"Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9, "inst": 1.0}.get(u, 1.0)


def main():
    rep, config, Z, N, M = sys.argv[1:6]
    prec = int(sys.argv[6]) if len(sys.argv) > 6 else 32
    cells = float(Z) * float(N) * float(M)
    rows = [d for d in raw_metrics(rep) if "sdtw_dp" in d.get("Kernel Name", ("", ""))[0]]
    d = rows[-1]
    warp = num(d, "smsp__inst_executed.sum")
    key = "smsp__thread_inst_executed.sum" if "smsp__thread_inst_executed.sum" in d else \
        "sass__thread_inst_executed_true_per_opcode"
    thread = num(d, key)
    act = float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"][0].replace(",", "")) / 100.0
    out = {"config": config, "Z": int(Z), "N": int(N), "M": int(M), "precision": prec,
           "warp_inst": warp, "thread_inst": thread, "cells": cells,
           "issue_slots_per_cell": warp * 32 / cells, "thread_inst_per_cell": thread / cells,
           "issue_active": act, "kernel": d["Kernel Name"][0][:120],
           "duration": d["gpu__time_duration.sum"][0] + " " + d["gpu__time_duration.sum"][1],
           "source": "ncu --set full of one DP launch (%s), %s" % (config, os.path.basename(rep))}
    dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                       "issue_%s.json" % config)
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

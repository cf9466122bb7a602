"""Summarise a SDTW_UNIT_LOG file (per-unit grab / start / end times of persistent DP launches,
written by the library when SDTW_UNIT_LOG is set): per unit kind the run and wait times, how
long workers sat blocked on a predecessor, and how the number of busy workers decays at the
end of the launch.  Usage: python scripts/unit_timeline.py LOG [launch index, default last]"""
import sys
from collections import defaultdict

import numpy as np


def launches(path):
    out, cur, hdr = [], [], None
    for line in open(path):
        if line.startswith("#"):
            if cur:
                out.append((hdr, np.array(cur, dtype=np.int64)))
            hdr, cur = line.strip(), []
        else:
            cur.append([int(v) for v in line.split()])
    if cur:
        out.append((hdr, np.array(cur, dtype=np.int64)))
    return out


def summary(hdr, a):
    kv = dict(x.split("=") for x in hdr.split()[2:])
    Z = int(kv["Z"])
    _, unit, block, sm, grab, start, end = a.T
    t0 = grab.min()
    T = (end.max() - t0) / 1e6
    print(hdr)
    print("makespan %.3f ms, %d units, %d workers" % (T, len(a), len(set(block.tolist()))))
    kind = unit // Z
    for k in sorted(set(kind.tolist())):
        m = kind == k
        print("  kind %2d: %4d units  run %.3f ms (min %.3f max %.3f)  wait mean %.3f max %.3f ms" % (
            k, m.sum(), (end[m] - start[m]).mean() / 1e6, (end[m] - start[m]).min() / 1e6,
            (end[m] - start[m]).max() / 1e6, (start[m] - grab[m]).mean() / 1e6, (start[m] - grab[m]).max() / 1e6))
    wait = (start - grab).sum() / 1e6
    busy = (end - start).sum() / 1e6
    W = len(set(block.tolist()))
    print("  worker-time: busy %.1f%%, blocked on a predecessor %.1f%%, idle (done/gaps) %.1f%%" % (
        100 * busy / (W * T), 100 * wait / (W * T), 100 * (1 - (busy + wait) / (W * T))))
    # busy workers over time
    ts = np.linspace(0, T, 41)
    line = []
    for t in ts:
        tt = t0 + t * 1e6
        line.append(int(((start <= tt) & (end > tt)).sum()))
    print("  running units at 2.5%% steps of the makespan: %s" % line)
    # per SM: busy time
    per_sm = defaultdict(float)
    for s_, b_ in zip(sm.tolist(), (end - start).tolist()):
        per_sm[s_] += b_ / 1e6
    v = np.array(list(per_sm.values()))
    print("  per-SM busy CTA-ms: mean %.2f min %.2f max %.2f" % (v.mean(), v.min(), v.max()))
    last = np.argsort(end)[-5:]
    for i in last:
        print("  late unit: kind %d q %d sm %d grab %.3f start %.3f end %.3f ms" % (
            kind[i], unit[i] % Z, sm[i], (grab[i] - t0) / 1e6, (start[i] - t0) / 1e6, (end[i] - t0) / 1e6))


if __name__ == "__main__":
    L = launches(sys.argv[1])
    idx = int(sys.argv[2]) if len(sys.argv) > 2 else -1
    summary(*L[idx])

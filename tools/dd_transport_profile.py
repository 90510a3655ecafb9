"""Config 5 over 8 loopback ranks, a few iterations with each halo transport (staged copies, then peer stores), for
an ncu launch list (`ncu --metrics gpu__time_duration.sum`): which kernels each transport launches per colour and
what they cost.  PBNG_DD_GRAPH=0 so that ncu sees plain launches.

    PBNG_DD_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file out.csv \
        python tools/dd_transport_profile.py
    python tools/dd_transport_profile.py --summarise out.csv"""
import csv
import os
import sys
from collections import defaultdict

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def summarise(path):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    hdr = rows[0]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        name = r[ik].split("<")[0].split("(")[0]
        tot[name] += float(r[iv].replace(",", "")) / 1e3  # ns -> us
        cnt[name] += 1
    print("| kernel | launches | total us | mean us |\n|---|---|---|---|")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"| {k} | {cnt[k]} | {tot[k]:.1f} | {tot[k] / cnt[k]:.2f} |")


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--summarise":
        return summarise(sys.argv[2])
    import torch
    from paper_2306_09021_b200 import dd
    from scenes import generators as G
    s = G.config5_muscle_stack()
    ctxs, _ = dd.loopback_contexts(s, 8, dtype="f32")
    grp = dd.Group(ctxs)
    for tr in ("copies", "peer"):
        grp.set_transport(tr)
        grp.iterate(2, s.accel)
        torch.cuda.synchronize()
    grp.close()
    for c in ctxs:
        c.close()


if __name__ == "__main__":
    main()

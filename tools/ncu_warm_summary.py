"""Summarise a warm-cache ncu capture (`ncu --set full --cache-control none`, raw page exported as CSV on the
GPU box by tools/gpu/r2s3_ncu.sh) into a markdown table: per launch time, DRAM bytes, L2-slice (LTS) and L1
throughput as fractions of their peaks, hit rates, warps/issue activity and the main stall reasons.

    python tools/ncu_warm_summary.py gpurun_out/s3c3w_raw.csv "<title>" > profiles/<tag>_summary.md
"""
import csv
import sys

COLS = [
    ("time us", "gpu__time_duration.sum", 1e-3),
    ("DRAM MB", ("dram__bytes_read.sum", "dram__bytes_write.sum"), 1e-6),
    ("DRAM % peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("LTS % peak", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("L2 hit %", "lts__t_sector_hit_rate.pct", 1),
    ("L1 % peak", "l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
    ("L1 hit %", "l1tex__t_sector_hit_rate.pct", 1),
    ("L1 LSU wavefronts % peak", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", 1),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("long-sb / issue", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", 1),
    ("lg-throttle / issue", "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", 1),
    ("mio-throttle / issue", "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", 1),
    ("short-sb / issue", "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", 1),
    ("wait / issue", "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", 1),
]


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def main():
    path, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    with open(path, newline="") as f:
        rows = list(csv.reader(f))
    hdr = rows[0]
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    idx = {h: i for i, h in enumerate(hdr)}
    name_col = idx.get("Kernel Name")
    out = [f"# {title}", "", f"Source: `{path}` (ncu --set full --cache-control none --clock-control none: caches are NOT "
           "flushed between launches, so L2 holds what the previous launches left -- the steady state of bench.py).", "",
           "| launch | kernel | " + " | ".join(c[0] for c in COLS) + " |",
           "|---|---|" + "---|" * len(COLS)]
    for k, r in enumerate(data):
        cells = []
        for _, key, sc in COLS:
            keys = key if isinstance(key, tuple) else (key,)
            vals = [num(r[idx[q]]) for q in keys if q in idx]
            if not vals or any(v is None for v in vals):
                cells.append("n/a")
                continue
            cells.append(f"{sum(vals) * sc:.3g}")
        kn = r[name_col][:40] if name_col is not None else ""
        out.append(f"| {k} | {kn} | " + " | ".join(cells) + " |")
    units = rows[1]
    out += ["", "Units row of the capture (for the time column: " + units[idx["gpu__time_duration.sum"]] + ")."]
    print("\n".join(out))


if __name__ == "__main__":
    main()

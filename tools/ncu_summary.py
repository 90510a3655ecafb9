"""Summarise ncu captures (run here, no GPU needed) into profiles/<tag>_summary.md and
profiles/sweep_traffic.json.

    python tools/ncu_summary.py <tag> <config> [gpurun_out dir]
reads <dir>/<tag>_sweep.ncu-rep (ncu --set full of one iteration's colour launches),
<dir>/<tag>_launches.csv (gpu__time_duration of every launch) and <dir>/<tag>_plain.json (bench line).
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "derived__smsp__sass_thread_inst_executed_op_ffma_pred_on_x2", "derived__smsp__sass_thread_inst_executed_op_dfma_pred_on_x2",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed",
]


def ncu_raw(rep):
    # the raw page exported on the GPU box (<tag>_raw.csv, tools/ncu_sweep.sh) when the report itself was
    # dropped to keep gpurun_out/ small; otherwise read the report
    raw = rep.replace("_sweep.ncu-rep", "_raw.csv")
    if os.path.exists(raw):
        out = open(raw).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for i, h in enumerate(hdr):
            if h in METRICS or h == "Kernel Name":
                d[h] = (r[i], units[i])
        res.append(d)
    return res


def num(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return None


def to_bytes(v, u):
    x = num(v)
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def to_us(v, u):
    x = num(v)
    return x * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1, "ms": 1e3,
                "s": 1e6}.get(u, 1)


def launch_shares(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("<")[0].split("(")[0].replace("void ", "").strip()
        name = name.split("::")[-1]
        t = num(r["Metric Value"]) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[r["Metric Unit"]]
        tot[name] += t
        cnt[name] += 1
    all_t = sum(tot.values())
    return sorted(((k, cnt[k], tot[k], tot[k] / all_t) for k in tot), key=lambda x: -x[2]), all_t


def main():
    tag, cfg = sys.argv[1], int(sys.argv[2])
    d = sys.argv[3] if len(sys.argv) > 3 and sys.argv[3] != "-" else os.path.join(ROOT, "gpurun_out")
    key = sys.argv[4] if len(sys.argv) > 4 else f"config{cfg}"  # sweep_traffic.json key (e.g. config3_f64)
    rep = os.path.join(d, f"{tag}_sweep.ncu-rep")
    kern = ncu_raw(rep)
    bench = json.load(open(os.path.join(d, f"{tag}_plain.json")))
    shares, all_t = launch_shares(os.path.join(d, f"{tag}_launches.csv"))
    lines = [f"# ncu summary `{tag}` — BASELINE config {cfg}", "",
             f"Workload: {bench['config']['workload']}", "",
             "Source: `ncu --set full --clock-control none --import-source on -k regex:sweep -s 8 -c 8` of "
             f"`python bench.py --config {cfg} --steps 1 --warmup 3 --no-cpu-baseline --no-e2e` (one full iteration = 8 colour "
             "launches after skipping the first iteration), plus the `gpu__time_duration.sum` launch list of the same command. "
             "ncu numbers are cold-cache and serialised; only shares and per-launch bytes are comparable with bench.py.", "",
             "## Per-launch (sweep kernel, one iteration)", "",
             "| launch | grid | regs | time us | DRAM read MB | DRAM write MB | DRAM GB/s | L2 hit % | L1 hit % | warps active % | issue active % | FMA pipe % | XU pipe % | long-sb stall/issue |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    tot_b = tot_t = 0.0
    flops = 0.0
    fl = {"f": 0.0, "d": 0.0}
    for i, k in enumerate(kern):
        g = lambda m: k.get(m, ("", ""))
        t = to_us(*g("gpu__time_duration.sum"))
        rb = to_bytes(*g("dram__bytes_read.sum"))
        wb = to_bytes(*g("dram__bytes_write.sum"))
        tot_b += rb + wb
        tot_t += t
        for op in ("ffma", "dfma"):
            v = num(g(f"derived__smsp__sass_thread_inst_executed_op_{op}_pred_on_x2")[0] or "0")
            flops += v or 0
        hz = num(g("sm__cycles_elapsed.avg.per_second")[0] or "0") or 0.0
        unit = g("sm__cycles_elapsed.avg.per_second")[1]
        hz *= {"cycle/second": 1.0, "cycle/usecond": 1e6, "cycle/nsecond": 1e9, "Mcycle/second": 1e6,
               "Gcycle/second": 1e9, "Kcycle/second": 1e3, "hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}.get(unit, 1.0)
        for p_ in ("f", "d"):  # FLOP = add + mul + 2 fma (thread-level SASS ops per elapsed cycle, whole GPU)
            a = num(g(f"smsp__sass_thread_inst_executed_op_{p_}add_pred_on.sum.per_cycle_elapsed")[0] or "0") or 0.0
            m = num(g(f"smsp__sass_thread_inst_executed_op_{p_}mul_pred_on.sum.per_cycle_elapsed")[0] or "0") or 0.0
            f_ = num(g(f"smsp__sass_thread_inst_executed_op_{p_}fma_pred_on.sum.per_cycle_elapsed")[0] or "0") or 0.0
            fl[p_] += (a + m + 2 * f_) * hz * t * 1e-6  # flops of this launch
        lines.append(f"| {i} | {g('launch__grid_size')[0]} | {g('launch__registers_per_thread')[0]} | {t:.1f} | {rb/1e6:.1f} | {wb/1e6:.1f} | "
                     f"{(rb+wb)/t/1e3:.0f} | {g('lts__t_sector_hit_rate.pct')[0]} | {g('l1tex__t_sector_hit_rate.pct')[0]} | "
                     f"{g('sm__warps_active.avg.pct_of_peak_sustained_active')[0]} | {g('smsp__issue_active.avg.pct_of_peak_sustained_active')[0]} | "
                     f"{g('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active')[0]} | {g('sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active')[0]} | "
                     f"{g('smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio')[0]} |")
    n = max(len(kern), 1)
    rf = bench["roofline"]
    alg = rf["hbm"]["algorithmic_bytes_per_launch"] if "hbm" in rf else rf["algorithmic_bytes_per_launch"]
    lines += ["", f"Mean DRAM traffic per sweep launch (ncu): **{tot_b/n/1e6:.1f} MB**; algorithmic bytes per launch "
              f"(bench.py model, DESIGN.md): **{alg/1e6:.1f} MB** (ratio {tot_b/n/alg:.3f}).",
              f"ncu DRAM bandwidth over the iteration: {tot_b/tot_t/1e3:.0f} GB/s (cold cache, serialised launches).",
              f"FLOP rate over the iteration (SASS add + mul + 2 fma): FP32 {fl['f']/tot_t/1e6:.2f} TFLOP/s, "
              f"FP64 {fl['d']/tot_t/1e6:.2f} TFLOP/s from the scalar FADD/FMUL/FFMA counters of this set; the packed "
              "FFMA2/FADD2/FMUL2 ops are counted by tools/flop_count.py (profiles/sweep_flops.json), and bench.py's ALU "
              "fraction uses those counts against the measured peaks of profiles/alu_peaks.json (FP32 73.4-74.0, FP64 33.9 "
              "TFLOP/s).", "",
              "## Launch list (share of GPU time, all launches of the command)", "",
              "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for name, c, t, sh in shares:
        lines.append(f"| {name} | {c} | {t:.0f} | {100*sh:.1f}% |")
    lines += ["", "## bench.py line of the same command (plain run, not under ncu)", "", "```json",
              json.dumps(bench, indent=1), "```", ""]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w").write("\n".join(lines))
    tp = os.path.join(ROOT, "profiles", "sweep_traffic.json")
    tj = json.load(open(tp)) if os.path.exists(tp) else {}
    tj[key] = {"dram_bytes_per_launch": tot_b / n, "algorithmic_bytes_per_launch": alg, "capture": f"profiles/{tag}_summary.md",
                          "launches": n}
    json.dump(tj, open(tp, "w"), indent=1)
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    main()

"""Executed FP flops per vertex update of each config's sweep kernel, for the ALU rooflines
("FP32/FP64 FLOP rate from ncu sass op counters (FMA = 2)").

Runs every config at full size through the public API, warms up, then brackets ONE pbng_iterate call of
K iterations with cudaProfilerStart/Stop so that ncu (--profile-from-start off) sees exactly the sweep
launches of K iterations.  Under ncu:

    python tools/flop_count.py > gpurun_out/flops_plain.log &&
    ncu --profile-from-start off --metrics <FLOP_METRICS>,gpu__time_duration.sum,dram__bytes_read.sum,\
        dram__bytes_write.sum --csv --log-file gpurun_out/flops.csv python tools/flop_count.py
    python tools/flop_count.py --parse gpurun_out/flops.csv gpurun_out/flops_plain.log > profiles/sweep_flops.json

FLOPs = 2 FFMA + FADD + FMUL + 4 FFMA2 + 2 FADD2 + 2 FMUL2 + 2 DFMA + DADD + DMUL (thread instructions with
all predicates on).  MUFU (rcp, rsqrt, lg2, ex2) and integer work are not counted.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

WEIGHTS = {"ffma": 2, "fadd": 1, "fmul": 1, "ffma2": 4, "fadd2": 2, "fmul2": 2, "dfma": 2, "dadd": 1, "dmul": 1}
METRICS = [f"smsp__sass_thread_inst_executed_op_{k}_pred_on.sum" for k in WEIGHTS]
CASES = [("config3", 3, None, 1), ("config3_f64", 3, "f64", 1), ("config2", 2, None, 4), ("config4", 4, None, 1),
         ("config5", 5, None, 1), ("config1", 1, None, 8)]


def run():
    import numpy as np  # noqa: F401
    import torch
    from paper_2306_09021_b200 import context_from_scene
    from scenes import generators as G
    for key, cfg, dtype, K in CASES:
        s = G.make_config(cfg, "full")
        ctx = context_from_scene(s, device=0, dtype=dtype)
        ctx.iterate(2, s.accel, s.omega, s.rho, s.gamma)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        ctx.iterate(K, s.accel, s.omega, s.rho, s.gamma)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        q = ctx.query()
        print(json.dumps({"case": key, "iterations": K, "vertex_updates": q["n_free"] * q["n_batch"] * K,
                          "pairs": q["n_pairs"] * q["n_batch"] * K, "schedule": q["schedule"]}), flush=True)
        ctx.close()
        del ctx
        torch.cuda.empty_cache()


def parse(csv_path, plain_log):
    cases = [json.loads(l) for l in open(plain_log) if l.startswith("{")]
    rows = list(csv.reader(line for line in open(csv_path) if not line.startswith("==")))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    # one record per (launch, metric); launches appear in order, grouped by case by the profiler ranges
    launches = {}
    order = []
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        lid = r[ix["ID"]]
        if lid not in launches:
            launches[lid] = {"name": r[ix["Kernel Name"]]}
            order.append(lid)
        val = r[ix["Metric Value"]].replace(",", "")
        try:
            launches[lid][r[ix["Metric Name"]]] = float(val)
        except ValueError:
            pass
    sweeps = [launches[l] for l in order if "sweep" in launches[l]["name"]]
    # split the sweep launches over the cases: each case's profiled range holds only its own launches;
    # the launch count per case is known from the schedule (colour launches: colours x K; pipelined: 1)
    out = {}
    pos = 0
    for c in cases:
        n = 1 if c["schedule"] == 2 else 8 * c["iterations"]
        seg = sweeps[pos:pos + n]
        pos += n
        fl = sum(sum(WEIGHTS[k] * L.get(f"smsp__sass_thread_inst_executed_op_{k}_pred_on.sum", 0.0) for k in WEIGHTS)
                 for L in seg)
        t = sum(L.get("gpu__time_duration.sum", 0.0) for L in seg)
        dram = sum(L.get("dram__bytes_read.sum", 0.0) + L.get("dram__bytes_write.sum", 0.0) for L in seg)
        by_op = {k: sum(L.get(f"smsp__sass_thread_inst_executed_op_{k}_pred_on.sum", 0.0) for L in seg) for k in WEIGHTS}
        out[c["case"]] = {
            "flops_per_vertex_update": fl / c["vertex_updates"], "flops_per_pair": fl / max(c["pairs"], 1),
            "launches": len(seg), "kernel": seg[0]["name"][:120] if seg else None,
            "thread_insts_by_op": by_op, "ncu_time_ns": t, "dram_bytes": dram,
            "ncu_flop_rate_tflops": fl / t / 1e3 if t else None,
            "capture": "tools/flop_count.py under ncu --metrics (FMA = 2, FFMA2 = 4, FADD2/FMUL2 = 2)"}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--parse":
        parse(sys.argv[2], sys.argv[3])
    else:
        run()

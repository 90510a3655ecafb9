#!/usr/bin/env python
"""Benchmark of the B200-native PBNG hot path (arXiv 2306.09021).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3|4|2|5|1] [--impl ours|reference]

Default workload (N = 1): BASELINE.json config 3, the single-GPU roofline configuration -- a 128^3-cell
unit cube (2,146,689 vertices, 12,582,912 Kuhn tets), Neo-Hookean fp32 with per-tet lognormal E, SOR
omega = 1.5, 50 PBNG iterations.  One STEP = reset to x^0 + 50 iterations (8 colour passes each) + the
energy / Newton-residual evaluation, i.e. every row of SURVEY.md §8(a) that runs per solve.
Metric (BASELINE.json): PBNG vertex-updates/s = free vertices x iterations / time, whole job.

N > 1 (torchrun, one rank per GPU): every rank solves its own independent config-3 problem (the paper's
independent-problem / data-generation use) with no data-path collective -> weak
scaling; timing = max over ranks of CUDA-event time.  --config 4 shards the 4096 samples of the batched
config across ranks instead.

--impl reference times the serial fp64 CPU oracle (oracle/, test infrastructure) on the same workload:
each step is one colour pass of one PBNG iteration at full size (a bounded sample), rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "PBNG vertex-updates/sec per GPU and box at 1/2/4/8 B200; % of HBM roofline"
UNIT = "vertex-updates/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"  # /opt/skills/guides/B200_PROFILING.md fallback


def scene_for(config: int, rank: int, world: int):
    from scenes import generators as G
    if config == 4:
        full = G.config4_batched()
        per = full.n_batch // world
        return full.samples(rank * per, (rank + 1) * per), full
    s = G.make_config(config, "full")
    return s, s


def workload_name(s, config):
    return {
        1: "config1_tiny_cube: 4^3 cells, 125 vertices, 384 Kuhn tets, NH fp64, 200 iterations",
        2: "config2_twisted_bar: 32x32x128 cells, 140,481 vertices, 786,432 tets, FCR fp32, Chebyshev rho=0.95 gamma=1.7, 100 iterations",
        3: "config3_hetero_cube: 128^3 cells, 2,146,689 vertices, 12,582,912 Kuhn tets, NH fp32, per-tet lognormal E, SOR omega=1.5, 50 iterations",
        4: "config4_batched: 4096 x 16^3-cell cubes (4,913 vertices, 24,576 tets each), NH fp32, Chebyshev rho=0.95 gamma=1.7, 100 iterations",
        5: "config5_muscle_stack: 8 x 48^3-cell blocks, 941,192 vertices, 5,308,416 tets, FCR fp32, springs + plane contacts, gravity, 130 iterations",
    }[config]


class ClockSampler:
    """Samples SM clock and clock-event (throttle) reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_index: int):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._th = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h) if hasattr(
                    nv, "nvmlDeviceGetCurrentClocksEventReasons") else nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv is not None:
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th is not None:
            self._th.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def ncu_traffic(config: int):
    """Average DRAM bytes per sweep launch from the committed ncu --set full capture, if present."""
    p = os.path.join(ROOT, "profiles", "sweep_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(f"config{config}", {}).get("dram_bytes_per_launch")


def cpu_baseline_oracle(scene, config: int, full_iteration: bool = True):
    """The oracle as it stands, serial fp64, on a bounded sample of the same workload."""
    from oracle import Oracle
    o = Oracle(scene, 0)
    x0 = np.ascontiguousarray(scene.x0[0])
    col = o.colours()
    free = np.ones(scene.n_vertices, bool)
    free[scene.pinned] = False
    if full_iteration:
        t = time.perf_counter()
        o.iterate(x0, x0, 0, 1, scene.accel, scene.omega, scene.rho, scene.gamma)
        dt = time.perf_counter() - t
        n = int(free.sum())
        sample = f"1 full PBNG iteration (all {o.n_colours} colour passes + {scene.accel} blend) of the same workload"
    else:
        w = x0.copy()
        t = time.perf_counter()
        o.sweep_colour_inplace(w, 0)
        dt = time.perf_counter() - t
        n = int((free & (col == 0)).sum())
        sample = "colour-0 pass of one PBNG iteration"
    return {"value": n / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{sample}; serial fp64 C oracle, {n} vertex updates in {dt:.2f} s",
            "host_cpu": _cpu_name(), "host_nproc": os.cpu_count()}


def _cpu_name():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import Oracle
    scene, full = scene_for(args.config, 0, 1)
    o = Oracle(scene, 0)
    col = o.colours()
    free = np.ones(scene.n_vertices, bool)
    free[scene.pinned] = False
    counts = [int((free & (col == c)).sum()) for c in range(o.n_colours)]
    w = np.ascontiguousarray(scene.x0[0]).copy()
    for k in range(args.warmup):
        o.sweep_colour_inplace(w, k % o.n_colours)
    w = np.ascontiguousarray(scene.x0[0]).copy()
    t0 = time.perf_counter()
    n = 0
    for k in range(args.steps):
        c = k % o.n_colours
        o.sweep_colour_inplace(w, c)
        n += counts[c]
    dt = time.perf_counter() - t0
    value = n / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dt / max(args.steps, 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(scene, args.config), "step": "one colour pass (colour = step mod 8) of one PBNG iteration at full size"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{args.steps} colour passes, {n} vertex updates, serial fp64 C oracle"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    world, rank, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device; the PBNG path has no CPU fallback")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    from paper_2306_09021_b200 import context_from_scene, dd

    scene, full = scene_for(args.config, rank, world)
    # one mesh, domain-decomposed, halo exchange per colour: config 5 always at N > 1; any other
    # single-mesh config with --dd (e.g. config 3 in z slabs)
    decomposed = world > 1 and (args.config == 5 or (args.dd and args.config != 4))
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        part = None
        if decomposed:
            owner = dd.slab_partition(scene.X, world)
            part = (owner, rank, world)
        ctx = context_from_scene(scene, device=local, stream=stream, set_positions=False, partition=part,
                                 dtype=args.dtype)
        x0_dev = torch.from_numpy(np.ascontiguousarray(scene.x0, dtype=ctx.np_dtype)).to(dev)
        x0_host = torch.from_numpy(np.ascontiguousarray(scene.x0, dtype=ctx.np_dtype)).pin_memory()
        x_out_host = torch.empty_like(x0_host).pin_memory()
        exchanger = dd.TorchDistExchange(ctx, rank, world, scene.accel) if decomposed else None
    q = ctx.query()
    iters = scene.iterations
    accel = (scene.accel, scene.omega, scene.rho, scene.gamma)

    def run_iterations():
        if decomposed:
            with torch.cuda.stream(stream):
                dd.iterate([ctx], exchanger, iters, *accel)
        else:
            ctx.iterate(iters, *accel)

    def energy_residual():
        e, r = ctx.energy_residual()
        if decomposed:  # global energy = sum over ranks, residual = root of the summed squares
            t = torch.tensor(np.concatenate([e, np.asarray(r) ** 2]), dtype=torch.float64, device=dev)
            pg.all_reduce(t)
            t = t.cpu().numpy()
            e, r = t[:len(e)], np.sqrt(t[len(e):])
        return e, r

    def step():
        ctx.set_positions(x0_dev)
        run_iterations()
        return energy_residual()

    def step_e2e():
        ctx.set_positions(x0_host)
        run_iterations()
        e, r = energy_residual()
        ctx.get_positions(x_out_host)
        return e, r

    for _ in range(args.warmup):
        step()
    stream.synchronize()

    def barrier():
        if pg is not None:
            pg.barrier()

    # ---- device-resident timed region ----
    launches0 = ctx.query()["kernel_launches"]
    ctx.profile_read()
    ctx.profile_enable(1 if decomposed else 2)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            E, R = step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    ctx.profile_enable(0)
    sweep_ms, sweep_launches = ctx.profile_read()
    launches = ctx.query()["kernel_launches"] - launches0
    t_ms = ev0.elapsed_time(ev1)
    if pg is not None:
        tt = torch.tensor([t_ms], device=dev, dtype=torch.float64)
        pg.all_reduce(tt, op=pg.ReduceOp.MAX)
        t_ms = float(tt.item())
    units_rank = q["n_free"] * q["n_batch"] * iters * args.steps  # owned free vertices of this rank
    if pg is not None:
        tu = torch.tensor([units_rank], device=dev, dtype=torch.float64)
        pg.all_reduce(tu)
        units_all = float(tu.item())
    else:
        units_all = float(units_rank)
    value = units_all / (t_ms / 1e3)

    # ---- end-to-end through the C ABI with host buffers (pinned), copies inside the timed region ----
    te_ms = None
    for _ in range(0 if args.no_e2e else 1):
        step_e2e()
    barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(0 if args.no_e2e else args.steps):
        step_e2e()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    te_ms = e0.elapsed_time(e1) if not args.no_e2e else 1.0
    if pg is not None:
        tt = torch.tensor([te_ms], device=dev, dtype=torch.float64)
        pg.all_reduce(tt, op=pg.ReduceOp.MAX)
        te_ms = float(tt.item())
    e2e_value = units_all / (te_ms / 1e3) if not args.no_e2e else None
    xbytes = x0_host.numel() * x0_host.element_size()

    if rank == 0:
        hbm, peak_kind = peaks()
        bytes_per_iter = q["sweep_bytes"] + (q["accel_bytes"] if scene.accel != "none" else 0.0)
        n_sweeps = iters * args.steps
        launches_per_iter = sweep_launches / max(n_sweeps, 1)
        bytes_per_launch = bytes_per_iter / max(launches_per_iter, 1e-9)
        achieved = bytes_per_launch / (sweep_ms / max(sweep_launches, 1) / 1e3) / 1e9
        traffic = ncu_traffic(args.config if args.dtype is None else f"{args.config}_{args.dtype}")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if (args.config == 4 or decomposed) else "weak",
            "vs_baseline": None,
            "dtype": "f32" if q["dtype"] == 0 else "f64", "data": "synthetic",
            "config": {
                "workload": (workload_name(scene, args.config) if args.dtype is None else
                             workload_name(scene, args.config).replace("fp32", args.dtype.replace("f", "fp"))
                             .replace("fp64 fp64", "fp64")),
                "free_vertices_per_gpu": q["n_free"] * q["n_batch"], "iterations_per_step": iters,
                "pairs_per_iteration": q["n_pairs"], "colours": q["n_colours"],
                "step": "set_positions(x0, device) + iterate + energy_residual",
                "l2": "inputs larger than L2: %.2f GB of pair records per iteration vs 126 MB L2" % (q["sweep_bytes"] / 1e9),
                "parallelism": (f"domain decomposition over {world} GPUs (slabs), NCCL halo exchange after every colour"
                                if decomposed else f"samples sharded over {world} GPUs (no collective)" if args.config == 4
                                else f"replicas x{world} (independent problems, no collective)"),
            },
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": traffic, "peak_source": peak_kind, "kernel": "sweep_kernel",
                         "algorithmic_bytes_per_launch": bytes_per_launch,
                         "sweep_kernel_share_of_step": sweep_ms / t_ms if t_ms > 0 else None},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": xbytes,
                    "d2h_bytes_per_step": xbytes + 16 * q["n_batch"]},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "energy": float(np.asarray(E)[0]), "residual": float(np.asarray(R)[0]),
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_oracle(scene, args.config)
        print(json.dumps(line), flush=True)
    ctx.close()
    if pg is not None:
        pg.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer leg (profiling runs)")
    ap.add_argument("--dtype", default=None, choices=["f32", "f64"],
                    help="override the config's compute dtype (e.g. config 3 in fp64: the FP64 measurement variant)")
    ap.add_argument("--dd", action="store_true", help="N > 1: domain-decompose one mesh (z slabs) instead of replicas")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("bench.py: warmup raised to 3 (timing rule)", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

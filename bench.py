#!/usr/bin/env python
"""Benchmark of the B200-native PBNG hot path (arXiv 2306.09021).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3|4|2|5|1] [--impl ours|reference]

Default workload (N = 1): BASELINE.json config 3, the single-GPU roofline configuration -- a 128^3-cell
unit cube (2,146,689 vertices, 12,582,912 Kuhn tets), Neo-Hookean fp32 with per-tet lognormal E, SOR
omega = 1.5, 50 PBNG iterations.  One STEP = reset to x^0 + 50 iterations (8 colour passes each) + the
energy / Newton-residual evaluation, i.e. every row of SURVEY.md §8(a) that runs per solve.
Metric (BASELINE.json): PBNG vertex-updates/s = free vertices x iterations / time, whole job.

N > 1 (torchrun, one rank per GPU): default config 4 -- the north_star scaling config, the paper's
data-generation use: the 4096 independent samples are sharded in contiguous ranges
across ranks with no data-path collective (strong scaling: the total work is fixed); timing = max over
ranks of CUDA-event time.  Before the sharded run rank 0 solves the whole 4096-sample batch alone on its
GPU (same invocation, same steps) and reports it as "anchor_1gpu", so box / (N x anchor) is
self-contained.  --config 5 (or --dd with a single-mesh config) domain-decomposes one mesh with the
library's NCCL halo exchange; --config 3 at N > 1 runs independent replicas (weak scaling).

--impl reference times the CPU oracle (oracle/, test infrastructure) as it stands on the same workload:
each step is one full PBNG iteration (all colour passes + blend) of the same problem, run by the OpenMP
build of the oracle on all host cores (bitwise the serial oracle; config 4: a 16-sample subset), rank 0
only.
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


def shard(n: int, rank: int, world: int):
    """Contiguous range of rank `rank` when n items are split over `world` ranks (the first n % world
    ranks take one more); every item is solved exactly once."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def scene_for(config: int, rank: int, world: int):
    from scenes import generators as G
    if config == 4:
        full = G.config4_batched()
        lo, hi = shard(full.n_batch, rank, world)
        return full.samples(lo, hi), full
    s = G.make_config(config, "full")
    return s, s


def alu_peaks():
    """Measured CUDA-core peaks (tools/alu_peaks.cu on this pool's B200, profiles/alu_peaks.json)."""
    p = os.path.join(ROOT, "profiles", "alu_peaks.json")
    if not os.path.exists(p):
        return None
    return json.load(open(p))


def sweep_flops(config_key: str):
    """Executed FP flops per vertex update of the config's sweep kernel, counted from ncu per-SASS-
    instruction executed thread counts (FMA = 2, packed FFMA2 = 4, FADD2/FMUL2 = 2; profiles/sweep_flops.json)."""
    p = os.path.join(ROOT, "profiles", "sweep_flops.json")
    if not os.path.exists(p):
        return None
    return json.load(open(p)).get(config_key)


# the dominant kernel and what bounds it, per config
KERNEL = {1: "sweep_pipe_kernel (pipelined, fp64 NH)", 2: "sweep_pipe_kernel (pipelined, fp32 FCR)",
          3: "sweep_kernel (colour launches, fp32 NH)", 4: "sweep_batched2_kernel (fp32 NH, 2 samples/lane)",
          5: "sweep_split_kernel (fp32 FCR, colour launches)"}
BOUND = {1: "hbm", 2: "alu", 3: "hbm", 4: "alu", 5: "alu"}


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


def ncu_traffic(key: str):
    """Average DRAM bytes per launch of the config's dominant kernel, from the committed ncu --set full
    capture named in profiles/sweep_traffic.json (or None)."""
    p = os.path.join(ROOT, "profiles", "sweep_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(key, {}).get("dram_bytes_per_launch")


def _host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _cpu_name():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def oracle_subset(scene, config: int):
    """The bounded oracle sample of the workload: config 4 -> its first 16 samples (one sample is a
    4,335-vertex problem); every other config -> the whole problem."""
    return scene.samples(0, min(16, scene.n_batch)) if config == 4 else scene


def oracle_iteration_rate(scene, iterations: int, omp: bool):
    """Vertex updates per second of `iterations` full PBNG iterations (all colour passes + blend) of the
    oracle as it stands on every sample of `scene`: serial (pinned to one core with sched_setaffinity, the
    taskset of the survey) or the OpenMP build on all host cores.  Returns (rate, updates, seconds, cores)."""
    from oracle import Oracle, threads
    cores_all = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None
    if omp:
        n_threads = threads(_host_threads())
    else:
        n_threads = 1
        if cores_all:
            os.sched_setaffinity(0, {cores_all[0]})
    try:
        n_free = scene.n_vertices - int(np.unique(scene.pinned).size)
        dt = 0.0
        for b in range(scene.n_batch):
            o = Oracle(scene, b, omp=omp)
            x0 = np.ascontiguousarray(scene.x0[b])
            t = time.perf_counter()
            o.iterate(x0, x0, 0, iterations, scene.accel, scene.omega, scene.rho, scene.gamma)
            dt += time.perf_counter() - t
    finally:
        if cores_all and not omp:
            os.sched_setaffinity(0, set(cores_all))
    n = n_free * scene.n_batch * iterations
    return n / dt, n, dt, n_threads


def cpu_baselines(scene, config: int):
    """The oracle as it stands on bounded samples of the same workload: the OpenMP build on all host cores
    (the paper's own parallelisation) and the serial build pinned to one core."""
    sub = oracle_subset(scene, config)
    what = "16 of the 4096 samples" if config == 4 else "the full problem"
    it_omp = 4 if config in (3, 5) else (2 if config == 4 else 10)
    rate, n, dt, cores = oracle_iteration_rate(sub, it_omp, omp=True)
    omp = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"{it_omp} full PBNG iterations (all colour passes + {scene.accel} blend) of {what}; "
                     f"OpenMP build of the fp64 C oracle (bitwise the serial one), {n} vertex updates in {dt:.2f} s",
           "host_cpu": _cpu_name(), "host_nproc": os.cpu_count()}
    rate1, n1, dt1, _ = oracle_iteration_rate(sub, 1, omp=False)
    serial = {"value": rate1, "unit": UNIT, "cores": 1, "kind": "oracle",
              "sample": f"1 full PBNG iteration of {what}; serial fp64 C oracle pinned to one core, "
                        f"{n1} vertex updates in {dt1:.2f} s"}
    return omp, serial


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def default_config(args, world):
    return args.config if args.config is not None else (4 if world > 1 else 3)


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import Oracle, threads
    config = default_config(args, world)
    scene, _ = scene_for(config, 0, 1)
    sub = oracle_subset(scene, config)
    n_threads = threads(_host_threads())
    oracles = [Oracle(sub, b, omp=True) for b in range(sub.n_batch)]
    n_free = sub.n_vertices - int(np.unique(sub.pinned).size)
    state = [(np.ascontiguousarray(sub.x0[b]), np.ascontiguousarray(sub.x0[b])) for b in range(sub.n_batch)]

    def step(l):
        for b, o in enumerate(oracles):
            x, xm = state[b]
            state[b] = o.iterate(x, xm, l, 1, sub.accel, sub.omega, sub.rho, sub.gamma)

    for k in range(args.warmup):
        step(k)
    state = [(np.ascontiguousarray(sub.x0[b]), np.ascontiguousarray(sub.x0[b])) for b in range(sub.n_batch)]
    t0 = time.perf_counter()
    for k in range(args.steps):
        step(k)
    dt = time.perf_counter() - t0
    n = n_free * sub.n_batch * args.steps
    value = n / dt
    what = "16 of the 4096 samples" if config == 4 else "the full problem"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dt / max(args.steps, 1), "higher_is_better": True,
        "scaling": "strong" if config == 4 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(scene, config),
                   "step": f"one full PBNG iteration (all colour passes + {sub.accel} blend) of {what}"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": n_threads, "kind": "oracle",
                         "sample": f"{args.steps} PBNG iterations of {what}, {n} vertex updates; OpenMP build of the "
                                   f"fp64 C oracle (bitwise the serial one) on {n_threads} host threads",
                         "host_cpu": _cpu_name()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


class Solver:
    """One rank's solve of a scene through the public API (context_from_scene / iterate / energy_residual)."""

    def __init__(self, scene, config, local, dev, stream, world, rank, decomposed, dtype, pg, halo="nccl", colours=None):
        import torch
        from paper_2306_09021_b200 import context_from_scene, dd
        self.scene, self.dev, self.stream, self.pg = scene, dev, stream, pg
        self.decomposed = decomposed
        with torch.cuda.stream(stream):
            part = None
            if decomposed:
                owner = dd.slab_partition(scene.X, world)
                part = (owner, rank, world, dd.nccl_unique_id(pg, rank))
            self.ctx = context_from_scene(scene, device=local, stream=stream, set_positions=False, partition=part,
                                          dtype=dtype, colours=colours)
            if decomposed and halo == "peer":
                # rows stored straight into the neighbours' ghost rows over NVLink peer memory (collective)
                self.ctx.enable_peer_halo(True)
            nd = self.ctx.np_dtype
            self.x0_dev = torch.from_numpy(np.ascontiguousarray(scene.x0, dtype=nd)).to(dev)
            self.x0_host = torch.from_numpy(np.ascontiguousarray(scene.x0, dtype=nd)).pin_memory()
            self.x_out_host = torch.empty_like(self.x0_host).pin_memory()
        self.q = self.ctx.query()
        self.iters = scene.iterations
        self.accel = (scene.accel, scene.omega, scene.rho, scene.gamma)

    def step(self):
        self.ctx.set_positions(self.x0_dev)
        self.ctx.iterate(self.iters, *self.accel)
        return self.ctx.energy_residual()  # decomposed: the library all-reduces over ranks (NCCL)

    def step_e2e(self):
        self.ctx.set_positions(self.x0_host)
        self.ctx.iterate(self.iters, *self.accel)
        e, r = self.ctx.energy_residual()
        self.ctx.get_positions(self.x_out_host)
        return e, r

    def units_per_step(self):
        return self.q["n_free"] * self.q["n_batch"] * self.iters


def timed(fn, steps, stream, dev, barrier):
    import torch
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize(dev)
    out = None
    ev0.record(stream)
    for _ in range(steps):
        out = fn()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    return ev0.elapsed_time(ev1), out


def roofline_block(config, dtype_key, q, sweep_ms, sweep_launches, t_ms, iters, steps, scene_accel, colouring="greedy"):
    """Roofline of the dominant kernel: HBM for the Neo-Hookean colour sweep (config
    3), FP32 ALU for the fixed-corotated and batched kernels (configs 2, 4, 5) against the measured
    CUDA-core peak; both fractions are reported for every config, `bound` names the one that binds."""
    hbm, peak_kind = peaks()
    n_sweeps = iters * steps
    launches_per_iter = sweep_launches / max(n_sweeps, 1)
    bytes_per_iter = q["sweep_bytes"] + (q["accel_bytes"] if scene_accel != "none" else 0.0)
    bytes_per_launch = bytes_per_iter / max(launches_per_iter, 1e-9)
    launch_s = sweep_ms / max(sweep_launches, 1) / 1e3
    achieved_bw = bytes_per_launch / launch_s / 1e9
    vupd_per_launch = q["n_free"] * q["n_batch"] / max(launches_per_iter, 1e-9)
    key = f"config{config}" + ("" if dtype_key is None else f"_{dtype_key}")
    hbm_block = {"achieved": achieved_bw, "peak": hbm, "unit": "GB/s", "frac": achieved_bw / hbm,
                 "peak_source": peak_kind, "algorithmic_bytes_per_launch": bytes_per_launch,
                 "traffic": ncu_traffic(key if colouring == "greedy" else f"{key}_{colouring}")}
    if config == 3:
        # context for north_star's ">= 60% of HBM on config 3": that target was set on SURVEY.md section 8(d)'s
        # stored-Dm^-1 pair layout (1,383 B per vertex update in fp32, 2,483 B in fp64).  The layouts built here
        # move fewer bytes, so the fraction above is on their own bytes; this block states the sweep's rate
        # against the rate that stored layout would reach at 100% of the measured HBM peak.
        b_stored = 2483.0 if q["dtype"] == 1 else 1383.0
        at_peak = hbm * 1e9 / b_stored
        rate = vupd_per_launch / launch_s
        hbm_block["survey_stored_layout"] = {"bytes_per_vertex_update": b_stored,
                                             "vupd_per_s_at_100pct_hbm": at_peak,
                                             "sweep_vupd_per_s": rate, "sweep_over_that_bound": rate / at_peak}
    fl = sweep_flops(key)
    ap = alu_peaks()
    alu_block = None
    if fl is not None and ap is not None:
        f64 = q["dtype"] == 1
        pk = ap["fp64_dfma_tflops_sustained"] if f64 else max(ap["fp32_ffma_tflops_sustained"],
                                                              ap["fp32_ffma2_tflops_sustained"])
        ach = fl["flops_per_vertex_update"] * vupd_per_launch / launch_s / 1e12
        alu_block = {"achieved": ach, "peak": pk, "unit": "TFLOP/s", "frac": ach / pk,
                     "peak_source": "measured (profiles/alu_peaks.json, sustained, %s)" % ("DFMA" if f64 else "best of FFMA/FFMA2"),
                     "flops_per_vertex_update": fl["flops_per_vertex_update"], "flops_source": fl.get("capture")}
    bound = BOUND[config] if alu_block is not None else "hbm"
    main = alu_block if bound == "alu" else hbm_block
    out = {"bound": bound, "achieved": main["achieved"], "peak": main["peak"], "unit": main["unit"],
           "frac": main["frac"], "traffic": hbm_block["traffic"], "peak_source": main["peak_source"],
           "kernel": KERNEL[config], "kernel_share_of_step": sweep_ms / t_ms if t_ms > 0 else None,
           "launch_us": launch_s * 1e6, "hbm": hbm_block}
    if alu_block is not None:
        out["alu"] = alu_block
    return out


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
    config = default_config(args, world)
    scene, full = scene_for(config, rank, world)
    # one mesh, domain-decomposed, halo exchange per colour: config 5 always at N > 1; any other
    # single-mesh config with --dd (e.g. config 3 in z slabs)
    decomposed = world > 1 and (config == 5 or (args.dd and config != 4))
    stream = torch.cuda.Stream(dev)

    def barrier():
        if pg is not None:
            pg.barrier()

    def max_over_ranks(v):
        if pg is None:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v):
        if pg is None:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        pg.all_reduce(t)
        return float(t.item())

    colours = None
    if args.colouring == "kuhn4":
        from scenes import generators as G
        if config == 3:
            colours = G.kuhn_grid_colouring(128, 128, 128)
        elif config == 4:
            colours = G.kuhn_grid_colouring(16, 16, 16)
        elif config == 5:
            # block b shifted by b so that the binding springs' end nodes (top of b, bottom of b + 1) differ
            one = G.kuhn_grid_colouring(48, 48, 48)
            colours = np.concatenate([(one + b) % 4 for b in range(8)]).astype(np.int32)
        else:
            raise SystemExit("--colouring kuhn4: configs 3, 4 and 5 (config 2 diverges on it under its Chebyshev "
                             "blend, in the oracle too: DESIGN.md section 7)")
    # ---- same-invocation 1-GPU anchor of the sharded config: rank 0 solves the whole batch alone ----
    anchor = None
    if world > 1 and config == 4:
        if rank == 0:
            a = Solver(full, config, local, dev, stream, 1, 0, False, args.dtype, None, colours=colours)
            for _ in range(args.warmup):
                a.step()
            ta, _ = timed(a.step, args.steps, stream, dev, lambda: None)
            anchor = {"value": a.units_per_step() * args.steps / (ta / 1e3), "ms_per_step": ta / args.steps,
                      "samples": full.n_batch, "what": "rank 0 alone, whole 4096-sample batch, same steps/warmup"}
            a.ctx.close()
            del a
            torch.cuda.empty_cache()
        barrier()

    S = Solver(scene, config, local, dev, stream, world, rank, decomposed, args.dtype, pg, args.halo, colours)
    ctx, q = S.ctx, S.q
    for _ in range(args.warmup):
        S.step()
    stream.synchronize()

    # ---- device-resident timed region ----
    launches0 = ctx.query()["kernel_launches"]
    ctx.profile_read()
    ctx.profile_enable(2)
    with ClockSampler(local) as clk:
        t_ms, (E, R) = timed(S.step, args.steps, stream, dev, barrier)
    ctx.profile_enable(0)
    sweep_ms, sweep_launches = ctx.profile_read()
    launches = ctx.query()["kernel_launches"] - launches0
    t_ms = max_over_ranks(t_ms)
    units_all = sum_over_ranks(float(S.units_per_step() * args.steps))
    value = units_all / (t_ms / 1e3)

    # ---- end-to-end through the C ABI with host buffers (pinned), copies inside the timed region ----
    e2e = None
    if not args.no_e2e:
        S.step_e2e()
        te_ms, _ = timed(S.step_e2e, args.steps, stream, dev, barrier)
        te_ms = max_over_ranks(te_ms)
        xbytes = S.x0_host.numel() * S.x0_host.element_size()
        e2e = {"value": units_all / (te_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": xbytes,
               "d2h_bytes_per_step": xbytes + 16 * q["n_batch"]}

    if rank == 0:
        iters = S.iters
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if (config == 4 or decomposed) else "weak",
            "vs_baseline": None,
            "dtype": "f32" if q["dtype"] == 0 else "f64", "data": "synthetic",
            "config": {
                "workload": (workload_name(scene, config) if args.dtype is None else
                             workload_name(scene, config).replace("fp32", args.dtype.replace("f", "fp"))
                             .replace("fp64 fp64", "fp64")),
                "free_vertices_per_gpu": q["n_free"] * q["n_batch"], "iterations_per_step": iters,
                "pairs_per_iteration": q["n_pairs"], "colours": q["n_colours"],
                "colouring": ("greedy (PAPER.md:702-705)" if args.colouring == "greedy" else
                              "caller-supplied (i+j+k) mod 4 of the Kuhn grid (pbng_color_given)"),
                "samples_on_rank0": q["n_batch"],
                "step": "set_positions(x0, device) + iterate + energy_residual",
                "l2": "inputs larger than L2: %.2f GB of algorithmic bytes per iteration vs 126 MB L2" % (
                    (q["sweep_bytes"] + q["accel_bytes"]) / 1e9),
                "parallelism": ((f"domain decomposition over {world} GPUs (slabs), " + ("peer-store halo rows over NVLink (pbng_enable_peer_halo)" if args.halo == "peer" else "NCCL halo exchange") + " after every colour")
                                if decomposed else f"samples sharded over {world} GPUs (no collective)" if config == 4
                                else f"replicas x{world} (independent problems, no collective)"),
            },
            "roofline": roofline_block(config, args.dtype, q, sweep_ms, sweep_launches, t_ms, iters, args.steps,
                                       scene.accel, args.colouring),
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "energy": float(np.asarray(E)[0]), "residual": float(np.asarray(R)[0]),
        }
        if world > 1:
            line["per_gpu_value"] = value / world
            if anchor is not None:
                line["anchor_1gpu"] = anchor
        if world == 1 and not args.no_cpu_baseline:
            omp, serial = cpu_baselines(scene, config)
            line["cpu_baseline"] = omp
            line["cpu_baseline_serial"] = serial
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
    ap.add_argument("--config", type=int, default=None, choices=[1, 2, 3, 4, 5],
                    help="BASELINE.json config (default: 3 at N = 1, 4 at N > 1)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer leg (profiling runs)")
    ap.add_argument("--dtype", default=None, choices=["f32", "f64"],
                    help="override the config's compute dtype (e.g. config 3 in fp64: the FP64 measurement variant)")
    ap.add_argument("--dd", action="store_true", help="N > 1: domain-decompose one mesh (z slabs) instead of replicas")
    ap.add_argument("--colouring", default="greedy", choices=["greedy", "kuhn4"],
                    help="the paper's greedy colouring (default, 8 colours) or, configs 3-5, the caller-supplied "
                         "4-colouring (i + j + k) mod 4 of the Kuhn grid(s) through pbng_color_given")
    ap.add_argument("--halo", default=os.environ.get("PBNG_BENCH_HALO", "nccl"), choices=["nccl", "peer"],
                    help="decomposed runs: per-colour halo by NCCL send/receive (default) or by peer stores "
                         "(pbng_enable_peer_halo: one kernel per neighbour writes its ghost rows over NVLink)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("bench.py: warmup raised to 3 (timing rule)", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

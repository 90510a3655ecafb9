"""bench.py's reference arm (the fp64 oracle as it stands, OpenMP build on the host cores, BASELINE tier
rules) on CPU: one JSON line with the contract's keys on rank 0, nothing (exit 0) on other ranks; and the
host-side helpers of the multi-GPU arm (sample sharding, default config per world size)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(env_extra):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                           "--steps", "2", "--warmup", "1"], capture_output=True, text=True, env=env, timeout=600)


def test_reference_arm_prints_one_contract_line():
    p = run({"RANK": "0", "WORLD_SIZE": "1"})
    assert p.returncode == 0, p.stderr
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_other_ranks_exit_quietly():
    p = run({"RANK": "1", "WORLD_SIZE": "2"})
    assert p.returncode == 0 and p.stdout.strip() == ""


def test_sample_sharding_covers_every_sample_once():
    sys.path.insert(0, ROOT)
    import bench
    for n in (4096, 4097, 7, 1):
        for world in (1, 2, 3, 8):
            ranges = [bench.shard(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1


def test_default_config_per_world_size():
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    a = argparse.Namespace(config=None)
    assert bench.default_config(a, 1) == 3 and bench.default_config(a, 2) == 4 and bench.default_config(a, 8) == 4
    a.config = 5
    assert bench.default_config(a, 8) == 5


def test_oracle_cpu_baselines_on_a_small_config():
    # both baselines run the oracle as it stands; the OpenMP one on all host threads, the serial one pinned
    sys.path.insert(0, ROOT)
    import bench
    from scenes import generators as G
    s = G.make_config(3, "small")
    omp, serial = bench.cpu_baselines(s, 3)
    assert omp["kind"] == serial["kind"] == "oracle" and serial["cores"] == 1
    assert omp["cores"] == bench._host_threads() and omp["value"] > 0 and serial["value"] > 0
    assert os.sched_getaffinity(0) == set(range(os.cpu_count())) or len(os.sched_getaffinity(0)) > 1

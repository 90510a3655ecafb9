"""Domain decomposition on one GPU: the library's loopback transport
(pbng_group_iterate: per colour, part 1 -> side-stream pack / copy / unpack || part 2, captured once as a
CUDA graph and replayed) runs G rank contexts in one process.  The decomposed iterates must equal the
undecomposed ones bit for bit (global colouring, same per-vertex arithmetic), equal the plain
colour-by-colour order of the public per-colour calls, and the rank sums of energy / residual must match
the undecomposed evaluation.  No kernel ever waits for another rank's kernel."""
import os
import time

import numpy as np
import pytest

from scenes import generators as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def single(scene, dtype):
    from paper_2306_09021_b200 import context_from_scene
    ctx = context_from_scene(scene, device=0, dtype=dtype)
    ctx.iterate(scene.iterations, scene.accel, scene.omega, scene.rho, scene.gamma)
    E, R = ctx.energy_residual()
    x = ctx.get_positions().cpu().numpy()
    ctx.close()
    return x, E, R


def gather(scene, ctxs, owner):
    xs = [c.get_positions().cpu().numpy() for c in ctxs]
    pinned = np.zeros(scene.n_vertices, bool)
    pinned[scene.pinned] = True
    x = xs[0].copy()
    for r in range(len(ctxs)):
        rows = (owner == r) & ~pinned
        x[:, rows] = xs[r][:, rows]
    return x


def decomposed(scene, dtype, world, mode="group", split=None, transport="copies"):
    from paper_2306_09021_b200 import dd
    ctxs, owner = dd.loopback_contexts(scene, world, dtype=dtype)
    parts = [scene.iterations] if split is None else split
    grp = dd.Group(ctxs) if mode == "group" else None
    if grp is not None and transport != "copies":
        grp.set_transport(transport)
    for k in parts:
        if mode == "group":
            grp.iterate(k, scene.accel, scene.omega, scene.rho, scene.gamma)
        else:
            dd.serial_iterate(ctxs, k, scene.accel, scene.omega, scene.rho, scene.gamma)
    E, R = dd.combine_energy_residual([c.energy_residual() for c in ctxs])
    x = gather(scene, ctxs, owner)
    infos = [c.query() for c in ctxs]
    if grp is not None:
        grp.close()
    for c in ctxs:
        c.close()
    return x, E, R, infos


@pytest.mark.parametrize("cfg,world,dtype", [(5, 2, "f64"), (5, 3, "f32"), (3, 2, "f64"), (3, 3, "f32"),
                                             (2, 2, "f32"), (4, 2, "f32"), (1, 2, "f64")])
def test_loopback_decomposition_is_bitwise(cfg, world, dtype):
    s = G.make_config(cfg, "small")
    if cfg == 1:
        s.accel, s.omega, s.iterations = "sor", 1.5, 40
    x1, E1, R1 = single(s, dtype)
    xd, Ed, Rd, infos = decomposed(s, dtype, world)
    assert sum(i["n_ghosts"] for i in infos) > 0
    assert np.array_equal(x1, xd), np.abs(x1 - xd).max()
    np.testing.assert_allclose(Ed, E1, rtol=1e-12, atol=0)
    np.testing.assert_allclose(Rd, R1, rtol=1e-9, atol=0)


@pytest.mark.parametrize("cfg,world", [(5, 2), (3, 3), (2, 2)])
def test_library_schedule_equals_plain_colour_order(cfg, world):
    """The library's overlapped, graph-captured schedule gives the bits of the plain colour-by-colour order
    (public per-colour calls), with and without CUDA graphs, over calls that continue the state."""
    s = G.make_config(cfg, "small")
    xs, Es, _, _ = decomposed(s, "f32", world, mode="serial", split=[3, 2, 4])
    xg, Eg, _, _ = decomposed(s, "f32", world, split=[3, 2, 4])
    os.environ["PBNG_DD_GRAPH"] = "0"
    try:
        xe, Ee, _, _ = decomposed(s, "f32", world, split=[3, 2, 4])
    finally:
        del os.environ["PBNG_DD_GRAPH"]
    assert np.array_equal(xs, xg) and np.array_equal(xs, xe)
    assert np.array_equal(Es, Eg) and np.array_equal(Es, Ee)


def test_full_config5_two_rank_loopback_two_iterations():
    s = G.config5_muscle_stack()
    s.iterations = 2
    x1, E1, _ = single(s, "f32")
    xd, Ed, _, infos = decomposed(s, "f32", 2)
    assert np.array_equal(x1, xd)
    assert all(i["n_ghosts"] > 0 for i in infos)


def test_batched_sample_minor_decomposition_is_bitwise():
    """n_batch >= 32 (sample-minor position layout): halo pack/unpack address samples by group and lane."""
    s = G.config4_batched(n_samples=40, n=4, iterations=12)
    x1, E1, R1 = single(s, "f32")
    xd, Ed, Rd, infos = decomposed(s, "f32", 2)
    assert infos[0]["n_batch"] == 40 and sum(i["n_ghosts"] for i in infos) > 0
    assert np.array_equal(x1, xd), np.abs(x1 - xd).max()
    np.testing.assert_allclose(Ed, E1, rtol=1e-12, atol=0)


def test_full_config5_eight_ranks_graph_replay_bitwise_and_host_submission():
    """Config 5 at full size over 8 loopback ranks: bitwise equal to one context; the second solve from
    x^0 replays the captured graph (one host call per solve), and the host submission time of that call
    is far below the GPU time of the iterations it submits."""
    import torch
    from paper_2306_09021_b200 import dd
    s = G.config5_muscle_stack()
    s.iterations = 6
    x1, E1, _ = single(s, "f32")
    ctxs, owner = dd.loopback_contexts(s, 8, dtype="f32")
    grp = dd.Group(ctxs)
    x0 = np.asarray(s.x0)
    for rep in range(2):
        for c in ctxs:
            c.set_positions(x0)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(ctxs[0].stream)
        t = time.perf_counter()
        grp.iterate(s.iterations, s.accel)
        host_s = time.perf_counter() - t
        ev1.record(ctxs[0].stream)
        torch.cuda.synchronize()
        gpu_s = ev0.elapsed_time(ev1) / 1e3
    xd = gather(s, ctxs, owner)
    replays = ctxs[0].query()["graph_replays"]
    print(f"config5 8 loopback ranks: host submission {1e6 * host_s / s.iterations:.1f} us/iteration, "
          f"GPU {1e6 * gpu_s / s.iterations:.1f} us/iteration, graph replays {replays}")
    grp.close()
    for c in ctxs:
        c.close()
    assert np.array_equal(x1, xd)
    assert replays >= 1
    assert host_s < 0.5 * gpu_s


@pytest.mark.parametrize("cfg,world,dtype", [(5, 2, "f64"), (5, 3, "f32"), (3, 3, "f32"), (2, 2, "f32"),
                                             (4, 2, "f32"), (1, 2, "f64")])
def test_peer_store_transport_is_bitwise(cfg, world, dtype):
    """pbng_group_set_transport(1): boundary rows stored straight into the neighbours' ghost rows by ONE kernel
    per neighbour, ordered by the pushed / done epoch flags (include/pbng.h "Peer-store transport") -- the
    iterates equal the undecomposed ones bit for bit, and no wait times out (PBNG_E_CUDA otherwise)."""
    s = G.make_config(cfg, "small")
    if cfg == 1:
        s.accel, s.omega, s.iterations = "sor", 1.5, 40
    x1, E1, R1 = single(s, dtype)
    xd, Ed, Rd, infos = decomposed(s, dtype, world, transport="peer")
    assert sum(i["n_ghosts"] for i in infos) > 0
    assert np.array_equal(x1, xd), np.abs(x1 - xd).max()
    np.testing.assert_allclose(Ed, E1, rtol=1e-12, atol=0)


def test_peer_store_transport_split_calls_graph_and_direct():
    """Calls that continue the state (flag epochs restart per call), with CUDA graphs and with direct launches,
    and switching the transport back and forth on one group."""
    from paper_2306_09021_b200 import dd
    s = G.make_config(5, "small")
    xs, Es, _, _ = decomposed(s, "f32", 3, mode="serial", split=[3, 2, 4])
    xg, Eg, _, _ = decomposed(s, "f32", 3, split=[3, 2, 4], transport="peer")
    os.environ["PBNG_DD_GRAPH"] = "0"
    try:
        xe, Ee, _, _ = decomposed(s, "f32", 3, split=[3, 2, 4], transport="peer")
    finally:
        del os.environ["PBNG_DD_GRAPH"]
    assert np.array_equal(xs, xg) and np.array_equal(xs, xe)
    assert np.array_equal(Es, Eg) and np.array_equal(Es, Ee)
    ctxs, owner = dd.loopback_contexts(s, 3, dtype="f32")
    grp = dd.Group(ctxs)
    for k, tr in zip([3, 2, 4], ["peer", "copies", "peer"]):
        grp.set_transport(tr)
        grp.iterate(k, s.accel, s.omega, s.rho, s.gamma)
    xm = gather(s, ctxs, owner)
    grp.close()
    for c in ctxs:
        c.close()
    assert np.array_equal(xs, xm)


def test_batched_sample_minor_peer_store_is_bitwise():
    s = G.config4_batched(n_samples=40, n=4, iterations=12)
    x1, E1, R1 = single(s, "f32")
    xd, Ed, Rd, infos = decomposed(s, "f32", 2, transport="peer")
    assert np.array_equal(x1, xd), np.abs(x1 - xd).max()


def test_full_config5_eight_ranks_peer_store_bitwise_and_timing():
    """Config 5 at full size over 8 loopback ranks with peer stores: bitwise equal to one context, the graph is
    replayed, and the GPU time per iteration is printed next to the staged-copy transport's."""
    import torch
    from paper_2306_09021_b200 import dd
    s = G.config5_muscle_stack()
    s.iterations = 6
    x1, E1, _ = single(s, "f32")
    ctxs, owner = dd.loopback_contexts(s, 8, dtype="f32")
    grp = dd.Group(ctxs)
    x0 = np.asarray(s.x0)
    times = {}
    for tr in ("copies", "peer"):
        grp.set_transport(tr)
        for rep in range(3):
            for c in ctxs:
                c.set_positions(x0)
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(ctxs[0].stream)
            grp.iterate(s.iterations, s.accel)
            ev1.record(ctxs[0].stream)
            torch.cuda.synchronize()
            times[tr] = ev0.elapsed_time(ev1) * 1e3 / s.iterations
        xd = gather(s, ctxs, owner)
        assert np.array_equal(x1, xd), tr
    launches = ctxs[0].query()["kernel_launches"]
    print(f"config5 8 loopback ranks, GPU us/iteration: copies {times['copies']:.1f}, peer stores {times['peer']:.1f}")
    grp.close()
    for c in ctxs:
        c.close()
    assert launches > 0


def test_enable_peer_halo_without_a_communicator_is_refused():
    """pbng_enable_peer_halo is collective over pbng_partition's communicator: a device context without one
    (undecomposed, or a loopback rank context) gets PBNG_E_BAD_ORDER and keeps working."""
    from paper_2306_09021_b200 import PBNGError, context_from_scene, dd
    s = G.make_config(3, "small")
    ctx = context_from_scene(s, device=0, dtype="f32")
    with pytest.raises(PBNGError) as e:
        ctx.enable_peer_halo(True)
    assert e.value.status == 5
    ctx.iterate(2, s.accel, s.omega, s.rho, s.gamma)
    ctx.close()
    ctxs, _ = dd.loopback_contexts(s, 2, dtype="f32")
    with pytest.raises(PBNGError) as e:
        ctxs[0].enable_peer_halo(True)
    assert e.value.status == 5
    for c in ctxs:
        c.close()

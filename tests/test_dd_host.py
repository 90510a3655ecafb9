"""Host logic of the domain decomposition on CPU: rank-local contexts are host-only
(device = -1) and the ranks are real processes talking over torch.distributed gloo.  Checks that the halo
plan is consistent across ranks (a's send list to b == b's receive list from a, per colour), that
ownership covers every free vertex exactly once, that ghosts are exactly the vertices a rank's stencils
need, and that the global colouring is identical on every rank."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from scenes import generators as G


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene(name):
    if name == "stack":
        return G.make_config(5, "small")  # 3 stacked blocks with binding springs + contacts
    return G.make_config(3, "small")      # one connected cube: slabs share tets


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2306_09021_b200 import context_from_scene
        from paper_2306_09021_b200.dd import slab_partition
        s = _scene(name)
        owner = slab_partition(s.X, world)
        ctx = context_from_scene(s, device=-1, dtype="f64", partition=(owner, rank, world))
        info = ctx.query()
        lists = {}
        for c in range(ctx.n_colours):
            for p in range(world):
                if p != rank:
                    snd, rcv = ctx.halo_vertices(c, p)
                    lists[(c, p)] = (snd.tolist(), rcv.tolist())
        gathered = [None] * world
        dist.all_gather_object(gathered, {"rank": rank, "lists": lists, "colours": ctx.colours.tolist(),
                                          "n_free": info["n_free"], "n_ghosts": info["n_ghosts"],
                                          "n_local": info["n_local_vertices"], "n_tets": s.n_tets})
        q.put((rank, gathered if rank == 0 else None, None))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("stack", 2), ("stack", 3), ("cube", 2), ("cube", 3)])
def test_halo_plan_consistent_across_ranks(name, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, g, err = q.get(timeout=300)
        assert err is None, err
        res[r] = g
    for p in procs:
        p.join(timeout=60)
    gathered = res[0]
    s = _scene(name)
    from paper_2306_09021_b200.dd import slab_partition
    owner = slab_partition(s.X, world)
    pinned = np.zeros(s.n_vertices, bool)
    pinned[s.pinned] = True
    # the colouring is global and identical on every rank
    for g in gathered[1:]:
        assert g["colours"] == gathered[0]["colours"]
    colours = np.array(gathered[0]["colours"])
    # ownership covers every free vertex once
    assert sum(g["n_free"] for g in gathered) == int((~pinned).sum())
    for a in range(world):
        for b in range(world):
            if a == b:
                continue
            for c in range(max(colours) + 1):
                snd_a = gathered[a]["lists"][(c, b)][0]
                rcv_b = gathered[b]["lists"][(c, a)][1]
                assert snd_a == rcv_b, (a, b, c)
                assert all(owner[v] == a and colours[v] == c and not pinned[v] for v in snd_a)
    # ghosts of rank r = free vertices owned elsewhere that share a stencil with a free vertex of r, or
    # belong to a tet / constraint whose energy r evaluates (brute force over the stencils)
    stencils = [list(map(int, t)) for t in s.tets]
    if s.wc is not None:
        for k in range(s.wc["n0"].shape[0]):
            stencils.append([int(v) for v in s.wc["idx0"][k, :s.wc["n0"][k]]] +
                            [int(v) for v in s.wc["idx1"][k, :s.wc["n1"][k]]])
    for r in range(world):
        need = set()
        for st in stencils:
            if any((not pinned[v]) and owner[v] == r for v in st) or owner[st[0]] == r:
                need.update(st)
        ghosts = {v for v in need if not pinned[v] and owner[v] != r}
        assert gathered[r]["n_ghosts"] == len(ghosts)
        recv_all = set()
        for (c, p), (snd, rcv) in gathered[r]["lists"].items():
            recv_all.update(rcv)
        assert recv_all == ghosts
    if name == "stack" and s.meta["blocks"] % world == 0:
        # slab boundaries fall on block interfaces: only binding springs cross ranks (no shared tets)
        for t in s.tets:
            assert len({owner[v] for v in t}) == 1


def test_slab_partition_aligns_with_blocks():
    from paper_2306_09021_b200.dd import slab_partition
    s = G.config5_muscle_stack(n_blocks=8, n=6)
    nvb = 7 ** 3
    for world in (1, 2, 4, 8):
        owner = slab_partition(s.X, world)
        block = np.arange(s.n_vertices) // nvb
        assert np.array_equal(owner, (block // (8 // world)).astype(np.int32))


def _uid_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2306_09021_b200 import PBNGError, context_from_scene, dd
        uid = dd.nccl_unique_id(dist, rank)
        # pbng_partition on a host-only context: the NCCL transport needs a device (no communicator made)
        s = _scene("stack")
        owner = dd.slab_partition(s.X, world)
        ctx = context_from_scene(s, device=-1, dtype="f64")
        try:
            ctx.partition(owner, rank, world, uid)
            status = 0
        except PBNGError as e:
            status = e.status
        ctx.partition(None, 0, 1, None)  # n_ranks = 1 needs no id and no device
        got = [None] * world
        dist.all_gather_object(got, (uid, status))
        q.put((rank, got if rank == 0 else None, None))
    except Exception as e:  # pragma: no cover
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_nccl_unique_id_bootstrap_over_process_group(world):
    """dd.nccl_unique_id: the library makes the id on rank 0 and torch.distributed broadcasts it, so every
    rank passes the same 128 bytes to pbng_partition."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_uid_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, g, err = q.get(timeout=300)
        assert err is None, err
        res[r] = g
    for p in procs:
        p.join(timeout=60)
    got = res[0]
    uids = [g[0] for g in got]
    assert all(len(u) == 128 for u in uids) and all(u == uids[0] for u in uids)
    assert all(g[1] == 11 for g in got)  # PBNG_E_NO_DEVICE


def test_peer_halo_needs_a_device_context_with_a_communicator():
    """pbng_enable_peer_halo (include/pbng.h "Peer-store transport") on host-only contexts: a device is required
    (PBNG_E_NO_DEVICE) whether or not the context is partitioned; nothing is allocated or mapped."""
    from paper_2306_09021_b200 import PBNGError, context_from_scene, dd
    s = _scene("stack")
    for part in (None, (dd.slab_partition(s.X, 2), 0, 2)):
        ctx = context_from_scene(s, device=-1, dtype="f64", partition=part)
        with pytest.raises(PBNGError) as e:
            ctx.enable_peer_halo(True)
        assert e.value.status == 11  # PBNG_E_NO_DEVICE
        ctx.close()

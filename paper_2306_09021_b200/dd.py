"""Domain decomposition of one mesh across ranks (the paper itself runs one
shared-memory CPU).

Each rank holds a rank-local context: it sweeps its owned free vertices and keeps ghost copies of the
vertices its stencils touch.  The colouring is global, so after colour pass k the only state another rank
needs is the new value of the colour-k vertices it holds as ghosts.  The exchange runs
INSIDE libpbng:
  * one rank per GPU: `pbng_partition` gives the context an NCCL communicator, and `pbng_iterate` does
    part 1 -> (pack -> ncclSend/ncclRecv -> unpack on a side stream || part 2) per colour, captured once as
    a CUDA graph; this module only bootstraps the NCCL unique id over torch.distributed;
  * all ranks in one process on one GPU (tests, emulation): `Group` (pbng_group_*), the library's loopback
    transport with device-to-device copies; no kernel ever waits for another rank's kernel.
`serial_iterate` is the plain colour-by-colour order (sweep, pack, copy, unpack) through the public per-colour
calls -- the reference schedule the tests compare the library's overlapped one against.
This module is argument marshalling and data movement only; all arithmetic is in libpbng.
"""
from __future__ import annotations

from typing import List, Optional

import numpy as np

from .pbng import Context, Group, context_from_scene, nccl_unique_id as _nccl_unique_id


def slab_partition(X: np.ndarray, n_ranks: int, axis: int = 2) -> np.ndarray:
    """Owner rank per vertex: equal-count slabs along `axis` (ties broken by vertex index).  For the
    stacked-block scene (config 5, block-major numbering) with n_ranks dividing the block count the slab
    boundaries coincide with block interfaces, so only the binding springs cross ranks."""
    nv = X.shape[0]
    order = np.lexsort((np.arange(nv), X[:, axis]))
    owner = np.empty(nv, np.int32)
    owner[order] = (np.arange(nv, dtype=np.int64) * n_ranks // nv).astype(np.int32)
    return owner


def nccl_unique_id(pg=None, rank: int = 0, group=None) -> bytes:
    """The 128-byte NCCL unique id for pbng_partition: created by the library on rank 0 and broadcast to
    every rank over the torch.distributed process group `pg` (the module torch.distributed, or None for a
    single process)."""
    uid = _nccl_unique_id() if rank == 0 else None
    if pg is None:
        return uid
    obj = [uid]
    pg.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def n_fields(accel: str) -> int:
    return 1 if accel == "none" else 3


def serial_iterate(ctxs: List[Context], n: int, accel: str = "none", omega: float = 1.0, rho: float = 0.0,
                   gamma: float = 1.0):
    """n decomposed iterations in the plain order: every colour pass on every rank context, then the
    colour's halo (pack, copy, unpack), then the fused blend closes the iteration.
    Uses only the public per-colour calls; one device, all ranks in this process."""
    import torch
    nf = n_fields(accel)
    world = len(ctxs)
    dev = f"cuda:{ctxs[0].device}"
    for _ in range(n):
        for c in range(ctxs[0].n_colours):
            for ctx in ctxs:
                ctx.sweep_colour(c, accel, omega, rho, gamma)
            bufs = {}
            for q, ctx in enumerate(ctxs):
                for p in range(world):
                    if p == q:
                        continue
                    ns, _ = ctx.halo_counts(c, p)
                    if ns:
                        b = torch.empty((ctx.n_batch, ns, nf, 4), dtype=ctx.torch_dtype, device=dev)
                        ctx.halo_pack(c, p, nf, b)
                        bufs[(q, p)] = b
            for (q, p), b in bufs.items():
                ctxs[p].halo_unpack(c, q, nf, b)
        for ctx in ctxs:
            ctx.end_iteration(accel)


def combine_energy_residual(parts):
    """Global energy = sum over ranks; residual = sqrt(sum of squares) (per sample)."""
    E = np.sum([p[0] for p in parts], axis=0)
    R = np.sqrt(np.sum([np.asarray(p[1]) ** 2 for p in parts], axis=0))
    return E, R


def loopback_contexts(scene, n_ranks: int, device: int = 0, dtype: Optional[str] = None, owner=None,
                      records: str = "auto"):
    """One rank-local context per rank of a slab partition, all on one device (emulation)."""
    owner = slab_partition(scene.X, n_ranks) if owner is None else owner
    return [context_from_scene(scene, device=device, dtype=dtype, partition=(owner, r, n_ranks), records=records)
            for r in range(n_ranks)], owner


__all__ = ["slab_partition", "nccl_unique_id", "n_fields", "serial_iterate", "combine_energy_residual",
           "loopback_contexts", "Group"]

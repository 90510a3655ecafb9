"""Domain decomposition of one mesh across ranks with a halo exchange after every colour pass
(the paper itself runs one shared-memory CPU).

Each rank holds a rank-local context (`pbng_set_partition`): it sweeps its owned free vertices and keeps
ghost copies of the vertices its stencils touch.  The colouring is global, so after colour pass k the
only state another rank needs is the new value of the colour-k vertices it holds as ghosts: the library
packs them (`pbng_halo_pack`), this module moves the buffers between ranks, and the library scatters them
(`pbng_halo_unpack`).  Iterates are then bit-identical to the undecomposed run.

Exchangers:
  * TorchDistExchange -- one rank per GPU, buffers moved with torch.distributed P2P (NCCL over NVLink)
    on the context stream; no host synchronisation inside an iteration.
  * LoopbackExchange  -- all ranks' contexts in one process on one device (test / emulation only: plain
    sequential device copies, no kernel ever waits for another).
This module is argument marshalling and data movement only; all arithmetic is in libpbng.
"""
from __future__ import annotations

from typing import List, Optional

import numpy as np

from .pbng import Context, context_from_scene


def slab_partition(X: np.ndarray, n_ranks: int, axis: int = 2) -> np.ndarray:
    """Owner rank per vertex: equal-count slabs along `axis` (ties broken by vertex index).  For the
    stacked-block scene (config 5, block-major numbering) with n_ranks dividing the block count the slab
    boundaries coincide with block interfaces, so only the binding springs cross ranks."""
    nv = X.shape[0]
    order = np.lexsort((np.arange(nv), X[:, axis]))
    owner = np.empty(nv, np.int32)
    owner[order] = (np.arange(nv, dtype=np.int64) * n_ranks // nv).astype(np.int32)
    return owner


def n_fields(accel: str) -> int:
    return 1 if accel == "none" else 3


class _Buffers:
    def __init__(self, ctx: Context, peers: List[int], fields: int):
        import torch
        self.send, self.recv = {}, {}
        dev = f"cuda:{ctx.device}"
        for c in range(ctx.n_colours):
            for p in peers:
                ns, nr = ctx.halo_counts(c, p)
                if ns:
                    self.send[(c, p)] = torch.empty((ctx.n_batch, ns, fields, 4), dtype=ctx.torch_dtype, device=dev)
                if nr:
                    self.recv[(c, p)] = torch.empty((ctx.n_batch, nr, fields, 4), dtype=ctx.torch_dtype, device=dev)


class TorchDistExchange:
    """Per-colour halo exchange of one rank's context over a torch.distributed process group."""

    def __init__(self, ctx: Context, rank: int, n_ranks: int, accel: str, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.ctx = ctx
        self.rank = rank
        self.group = group
        self.fields = n_fields(accel)
        self.peers = [p for p in range(n_ranks) if p != rank]
        self.buf = _Buffers(ctx, self.peers, self.fields)

    def exchange(self, colour: int):
        dist = self.dist
        ops = []
        for p in self.peers:
            sb = self.buf.send.get((colour, p))
            if sb is not None:
                self.ctx.halo_pack(colour, p, self.fields, sb)
                ops.append(dist.P2POp(dist.isend, sb, p, group=self.group))
            rb = self.buf.recv.get((colour, p))
            if rb is not None:
                ops.append(dist.P2POp(dist.irecv, rb, p, group=self.group))
        if not ops:
            return
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for p in self.peers:
            rb = self.buf.recv.get((colour, p))
            if rb is not None:
                self.ctx.halo_unpack(colour, p, self.fields, rb)


class LoopbackExchange:
    """All ranks in one process (emulation / tests): rank q's pack buffer is rank p's unpack buffer."""

    def __init__(self, ctxs: List[Context], accel: str):
        self.ctxs = ctxs
        self.fields = n_fields(accel)
        n = len(ctxs)
        self.buf = [_Buffers(c, [p for p in range(n) if p != r], self.fields) for r, c in enumerate(ctxs)]

    def exchange(self, colour: int):
        n = len(self.ctxs)
        for q in range(n):
            for p in range(n):
                if p != q and (colour, p) in self.buf[q].send:
                    self.ctxs[q].halo_pack(colour, p, self.fields, self.buf[q].send[(colour, p)])
        for p in range(n):
            for q in range(n):
                if p != q and (colour, q) in self.buf[p].recv:
                    rb = self.buf[p].recv[(colour, q)]
                    rb.copy_(self.buf[q].send[(colour, p)])
                    self.ctxs[p].halo_unpack(colour, q, self.fields, rb)


def iterate(ctxs: List[Context], exchanger, n: int, accel: str = "none", omega: float = 1.0, rho: float = 0.0,
            gamma: float = 1.0, overlap: bool = True):
    """n PBNG iterations of a decomposed mesh: every colour pass on every local rank context, then the
    halo exchange of that colour (PAPER.md:693-705 order), then the fused blend closes the iteration.

    overlap: each colour pass is split (pbng_sweep_colour_part): the halo-send vertices first, then the
    halo of the colour is packed, exchanged and unpacked on a side stream while the colour's remaining
    vertices are updated on the main stream; the next colour waits for both.  Packing reads only the
    halo-send rows and unpacking writes only ghost rows of this colour, which no vertex of this colour
    reads, so the results are those of the serial order bit for bit."""
    n_col = ctxs[0].n_colours
    if not overlap:
        for _ in range(n):
            for c in range(n_col):
                for ctx in ctxs:
                    ctx.sweep_colour(c, accel, omega, rho, gamma)
                exchanger.exchange(c)
            for ctx in ctxs:
                ctx.end_iteration(accel)
        return
    import torch
    main = torch.cuda.current_stream(ctxs[0].device)
    side = torch.cuda.Stream(ctxs[0].device)
    boundary_done, exchange_done = torch.cuda.Event(), torch.cuda.Event()
    saved = [ctx.stream for ctx in ctxs]
    try:
        for _ in range(n):
            for c in range(n_col):
                for ctx in ctxs:
                    ctx.set_stream(main)
                    ctx.sweep_colour_part(c, 1, accel, omega, rho, gamma)
                boundary_done.record(main)
                side.wait_event(boundary_done)
                for ctx in ctxs:
                    ctx.set_stream(side)
                with torch.cuda.stream(side):
                    exchanger.exchange(c)
                exchange_done.record(side)
                for ctx in ctxs:
                    ctx.set_stream(main)
                    ctx.sweep_colour_part(c, 2, accel, omega, rho, gamma)
                main.wait_event(exchange_done)
            for ctx in ctxs:
                ctx.end_iteration(accel)
    finally:
        for ctx, st in zip(ctxs, saved):
            if st is not None:
                ctx.set_stream(st)


def combine_energy_residual(parts):
    """Global energy = sum over ranks; residual = sqrt(sum of squares) (per sample)."""
    E = np.sum([p[0] for p in parts], axis=0)
    R = np.sqrt(np.sum([np.asarray(p[1]) ** 2 for p in parts], axis=0))
    return E, R


def loopback_contexts(scene, n_ranks: int, device: int = 0, dtype: Optional[str] = None, owner=None):
    """One rank-local context per rank of a slab partition, all on one device (emulation)."""
    owner = slab_partition(scene.X, n_ranks) if owner is None else owner
    return [context_from_scene(scene, device=device, dtype=dtype, partition=(owner, r, n_ranks))
            for r in range(n_ranks)], owner

"""The peer-store halo transport's flag protocol (include/pbng.h "Peer-store transport", csrc/pbng_kernels.cu
"Peer-store halo transport"; colour order PAPER.md:693-705), model-checked on CPU.

The multi-process path cannot run in this container (one GPU at most), so its ordering rules are checked on a
model: every rank is a sequence of operations guarded by exactly the waits the library issues, a random
scheduler interleaves the ranks arbitrarily (the ranks' GPUs run at unrelated speeds), and every ghost read
checks that the ghost row holds the value of the pass the serial colour order prescribes -- not an older one
(the neighbour's store has not landed: read-after-write) and not a newer one (the neighbour ran ahead and
overwrote it: write-after-read).  Dropping either wait must make the model fail, which shows the checks bite.
The halo plan is the real one of the small stacked-block and connected-cube scenes (host-only contexts)."""
import random

import numpy as np
import pytest

from scenes import generators as G


def halo_plan(scene, world):
    """send[r][col][q] = rows rank r sends to q after colour col (counts), from host-only rank contexts."""
    from paper_2306_09021_b200 import context_from_scene
    from paper_2306_09021_b200.dd import slab_partition
    owner = slab_partition(scene.X, world)
    send, ncol = [], None
    for r in range(world):
        ctx = context_from_scene(scene, device=-1, dtype="f64", partition=(owner, r, world))
        ncol = ctx.n_colours
        send.append([[0 if q == r else ctx.halo_counts(c, q)[0] for q in range(world)] for c in range(ncol)])
        ctx.close()
    return send, ncol


class Model:
    """pass E = 1 + it * ncol + col.  Per rank and pass, in the library's stream order:
      main:  part1(E) -> part2(E) -> [join side] -> sync(E) = { done_on_q[r] = E for every neighbour q ;
             wait pushed_r[q] >= E for q that sends r rows of colour col }   (last pass: signal, then wait
             done_r[q] >= E for every neighbour)
      side:  after part1(E), per neighbour q with rows: push(E, q) = { wait done_r[q] >= E - 1 ; store ;
             pushed_on_q[r] = E }"""

    def __init__(self, send, ncol, n_iter, wait_done=True, wait_pushed=True):
        self.send, self.ncol, self.G = send, ncol, len(send)
        self.last = n_iter * ncol
        self.wait_done, self.wait_pushed = wait_done, wait_pushed
        G_ = self.G
        self.nbr = [[q for q in range(G_) if q != r and any(send[r][c][q] or send[q][c][r] for c in range(ncol))]
                    for r in range(G_)]
        self.pushed = [[0] * G_ for _ in range(G_)]   # pushed[r][q]: in r's memory, written by q
        self.done = [[0] * G_ for _ in range(G_)]
        self.version = {}                             # (receiver, sender, colour) -> pass whose rows it holds
        # per rank: program counter over [("p1b",E),("p1e",E),("p2b",E),("p2e",E),("sync",E),...] and the
        # set of pushes of the current pass still to run (enabled once p1e(E) is past)
        self.pc = [0] * G_
        self.E = [1] * G_
        self.pending = [None] * G_                    # pushes of pass E not yet executed (None: not forked yet)
        self.signalled = [False] * G_
        self.finished = [False] * G_

    def col(self, E):
        return (E - 1) % self.ncol

    def expected(self, E, c):
        """The pass whose colour-c rows a read during pass E must see (0: the initial positions)."""
        col = self.col(E)
        back = (col - c) % self.ncol
        back = back if back else self.ncol  # the colour itself is not read; harmless
        return max(E - back, 0)

    def check_reads(self, r, E):
        for q in self.nbr[r]:
            for c in range(self.ncol):
                if c == self.col(E) or not self.send[q][c][r]:
                    continue
                want = self.expected(E, c)
                got = self.version.get((r, q, c), 0)
                if got != want:
                    return f"rank {r} pass {E}: ghost rows of colour {c} from {q} hold pass {got}, want {want}"
        return None

    def enabled(self, r):
        """Operations rank r could execute now."""
        if self.finished[r]:
            return []
        E, ops = self.E[r], []
        if self.pending[r]:
            for q in self.pending[r]:
                if not self.wait_done or self.done[r][q] >= E - 1:
                    ops.append(("push", q))
        pc = self.pc[r]
        if pc < 4:
            ops.append(("sweep", pc))
        elif not self.pending[r]:  # join: sync comes after the pushes
            if not self.signalled[r]:
                ops.append(("signal", None))
            else:
                col = self.col(E)
                if E == self.last:
                    ok = all(self.done[r][q] >= E for q in self.nbr[r])
                else:
                    ok = (not self.wait_pushed) or all(self.pushed[r][q] >= E for q in self.nbr[r]
                                                       if self.send[q][col][r])
                if ok:
                    ops.append(("advance", None))
        return ops

    def step(self, r, op):
        E = self.E[r]
        kind, arg = op
        if kind == "sweep":
            err = self.check_reads(r, E)  # begin and end of part 1 and part 2: versions are monotone between
            if err:
                return err
            self.pc[r] += 1
            if self.pc[r] == 2:  # part 1 finished: fork the pushes
                self.pending[r] = [q for q in self.nbr[r] if self.send[r][self.col(E)][q]]
        elif kind == "push":
            self.version[(arg, r, self.col(E))] = E
            self.pushed[arg][r] = E
            self.pending[r].remove(arg)
        elif kind == "signal":
            for q in self.nbr[r]:
                self.done[q][r] = E
            self.signalled[r] = True
        else:
            if E == self.last:
                self.finished[r] = True
            else:
                self.E[r], self.pc[r], self.pending[r], self.signalled[r] = E + 1, 0, None, False
        return None

    def run(self, rng, bias=None):
        """Random interleaving; bias = a rank that is scheduled rarely (a slow GPU).  Returns an error string,
        "deadlock", or None."""
        while not all(self.finished):
            choices = [(r, op) for r in range(self.G) for op in self.enabled(r)]
            if not choices:
                return "deadlock"
            if bias is not None and len(choices) > 1 and rng.random() < 0.9:
                fast = [c for c in choices if c[0] != bias]
                choices = fast or choices
            r, op = rng.choice(choices)
            err = self.step(r, op)
            if err:
                return err
        return None


def explore(send, ncol, n_iter, trials, **rules):
    rng = random.Random(7)
    G_ = len(send)
    for t in range(trials):
        bias = None if t % (G_ + 1) == G_ else t % (G_ + 1)
        err = Model(send, ncol, n_iter, **rules).run(rng, bias)
        if err:
            return err
    return None


@pytest.fixture(scope="module")
def plans():
    out = {}
    for name, cfg, world in (("stack3", 5, 3), ("cube3", 3, 3), ("cube2", 3, 2)):
        out[name] = halo_plan(G.make_config(cfg, "small"), world)
    return out


def test_synthetic_chain_with_empty_colours():
    # 4 ranks in a chain, 3 colours; rank 1 sends nothing in colour 2, rank 3 nothing in colour 0
    G_, ncol = 4, 3
    send = [[[0] * G_ for _ in range(ncol)] for _ in range(G_)]
    for r in range(G_):
        for q in (r - 1, r + 1):
            if 0 <= q < G_:
                for c in range(ncol):
                    send[r][c][q] = 5
    send[1][2][0] = send[1][2][2] = 0
    send[3][0][2] = 0
    assert explore(send, ncol, 3, 300) is None


@pytest.mark.parametrize("name", ["stack3", "cube3", "cube2"])
def test_protocol_keeps_serial_colour_order_on_real_halo_plans(plans, name):
    send, ncol = plans[name]
    assert sum(map(sum, (row for r in send for row in r))) > 0
    assert explore(send, ncol, 3, 200) is None


@pytest.mark.parametrize("name", ["cube3", "cube2"])
def test_dropping_a_wait_breaks_the_model(plans, name):
    """Without the `done` wait a fast rank overwrites ghost rows its neighbour still reads; without the
    `pushed` wait a rank reads ghost rows that have not landed."""
    send, ncol = plans[name]
    assert explore(send, ncol, 3, 200, wait_done=False) not in (None, "deadlock")
    assert explore(send, ncol, 3, 200, wait_pushed=False) not in (None, "deadlock")

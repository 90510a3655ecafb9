"""CPU tests of the C-ABI boundary: the library loads, exports every symbol include/pbng.h declares, and
its host logic (validation, greedy colouring, layout sizes) behaves -- no compute call needs a GPU here
(host-only contexts, device = -1)."""
import os
import re

import numpy as np
import pytest

from paper_2306_09021_b200 import pbng as P
from scenes import generators as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "pbng.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pbng_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = P.lib()
    names = declared_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(P.EXPORTS)
    assert L.pbng_version() == 100
    # the library is the in-tree build
    assert os.path.dirname(P.LIB_PATH) == os.path.join(ROOT, "paper_2306_09021_b200")


def test_nm_shows_c_linkage():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", P.LIB_PATH], capture_output=True, text=True).stdout
    for n in declared_functions():
        assert re.search(rf"\bT {n}$", out, flags=re.M), n


def host_ctx(scene, dtype="f64"):
    return P.context_from_scene(scene, device=-1, dtype=dtype)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_library_colouring_equals_oracle(cfg):
    from oracle import Oracle
    s = G.make_config(cfg, "small")
    ctx = host_ctx(s)
    o = Oracle(s)
    assert ctx.n_colours == o.n_colours
    assert np.array_equal(ctx.colours, o.colours())


def test_library_colouring_table1_and_spring_network():
    from oracle import Oracle
    for n in (16, 32):
        X, T = G.five_tet_grid(n)
        ctx = P.Context(X, T, device=-1)
        ctx.set_material("nh", 1e5, 0.3)
        ctx.set_constraints(np.zeros(0, np.int32), np.zeros(0))
        col, nc = ctx.color()
        assert nc == 5  # PAPER.md Table 1 (tests/golden/table1_colours.json)
    s = G.spring_network()
    ctx = host_ctx(s)
    assert np.array_equal(ctx.colours, Oracle(s).colours())


def test_query_counts():
    s = G.config1_tiny_cube()
    ctx = host_ctx(s)
    q = ctx.query()
    assert q["n_vertices"] == 125 and q["n_tets"] == 384 and q["n_pinned"] == 50 and q["n_free"] == 75
    deg = np.bincount(s.tets.reshape(-1), minlength=125)
    free = np.setdiff1d(np.arange(125), s.pinned)
    assert q["n_pairs"] == deg[free].sum()
    assert q["n_pair_slots"] >= q["n_pairs"] and q["n_pair_slots"] % 32 == 0
    assert q["n_colours"] == 8


def test_errors():
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 0]], float)
    with pytest.raises(P.PBNGError) as ei:
        P.Context(X, [[0, 1, 2, 3], [0, 1, 4, 2]], device=-1)
    assert ei.value.status == 3 and ei.value.bad_index == 1
    with pytest.raises(P.PBNGError) as ei:
        P.Context(X, [[0, 1, 2, 7]], device=-1)
    assert ei.value.status == 2 and ei.value.bad_index == 0
    ctx = P.Context(X, [[0, 1, 2, 3]], device=-1)
    with pytest.raises(P.PBNGError) as ei:
        ctx.set_material("nh", 1e5, 0.5)
    assert ei.value.status == 1
    with pytest.raises(P.PBNGError) as ei:
        ctx.color()
    assert ei.value.status == 5  # bad order: material / constraints missing
    ctx.set_material("nh", 1e5, 0.3)
    ctx.set_constraints(np.zeros(0, np.int32), np.zeros(0))
    with pytest.raises(P.PBNGError) as ei:
        ctx.color()
    assert ei.value.status == 4  # vertex 4 is free and isolated
    ctx.set_constraints(np.array([4], np.int32), np.array([1.0, 1.0, 0.0]))
    col, nc = ctx.color()
    assert nc == 4
    with pytest.raises(P.PBNGError) as ei:
        ctx.bind_workspace  # attribute exists
        P._check(P.lib().pbng_set_positions(ctx._h, None))
    assert ei.value.status == 11  # host-only context
    with pytest.raises(P.PBNGError) as ei:
        ctx.set_constraints(np.array([4, 4], np.int32), np.zeros(6))
    assert ei.value.status == 1


def test_weak_constraint_struct_layout():
    import ctypes as C

    class WC(C.Structure):
        _fields_ = [("n0", C.c_int32), ("n1", C.c_int32), ("idx0", C.c_int32 * 4), ("idx1", C.c_int32 * 4),
                    ("w0", C.c_double * 4), ("w1", C.c_double * 4), ("anchor", C.c_double * 3), ("K", C.c_double * 6)]
    assert C.sizeof(WC) == P.WC_DTYPE.itemsize == 176
    for name in ("w0", "w1", "anchor", "K"):
        assert getattr(WC, name).offset == P.WC_DTYPE.fields[name][1]


def test_schedule_selection():
    s = G.config1_tiny_cube()
    ctx = P.Context(s.X, s.tets, n_batch=1, dtype="f64", device=-1)
    ctx.set_material(s.model, s.E, s.nu, s.density, s.gravity)
    ctx.set_constraints(s.pinned, s.targets, s.wc)
    with pytest.raises(P.PBNGError) as e:
        ctx.set_schedule("pipelined")
    assert e.value.status == 6  # not coloured yet
    ctx.color()
    assert ctx.query()["schedule"] == 2  # auto -> pipelined on a small undecomposed context
    ctx.set_schedule("colour_launches")
    assert ctx.query()["schedule"] == 1
    ctx.set_schedule("pipelined")
    assert ctx.query()["schedule"] == 2
    # a domain-decomposed context needs the halo exchange between colour passes
    d = P.Context(s.X, s.tets, n_batch=1, dtype="f64", device=-1)
    d.set_material(s.model, s.E, s.nu, s.density, s.gravity)
    d.set_constraints(s.pinned, s.targets, s.wc)
    d.set_partition((np.arange(125) >= 60).astype(np.int32), 0, 2)
    d.color()
    assert d.query()["schedule"] == 1
    with pytest.raises(P.PBNGError) as e:
        d.set_schedule("pipelined")
    assert e.value.status == 1


def test_record_layout_selection():
    """pbng_set_records (lower-byte variant (i)): rest-recompute records only for the
    unbatched Neo-Hookean path layout; chosen before pbng_color; the algorithmic byte model shrinks."""
    def make(s, records, nb=1, dtype="f32"):
        c = P.Context(s.X, s.tets, n_batch=nb, dtype=dtype, device=-1)
        c.set_material(s.model, s.E, s.nu, s.density, s.gravity)
        c.set_constraints(s.pinned, np.repeat(s.targets[:1], nb, axis=0), s.wc)
        if records is not None:
            c.set_records(records)
        c.color()
        return c
    s = G.make_config(3, "small")
    q_st, q_re, q_au = make(s, "stored").query(), make(s, "rest").query(), make(s, None).query()
    q_tb = make(s, "table").query()
    assert (q_st["records"], q_re["records"], q_tb["records"]) == (1, 2, 3)
    assert q_au["records"] == 1  # small problem: split warps, plain records
    assert q_tb["sweep_bytes"] < q_re["sweep_bytes"]  # the same 8 B records, without the rest positions
    # 8 B per record (+ path0, + the rest positions once) against 32 B per stored three-id record
    assert q_re["sweep_bytes"] < 0.5 * q_st["sweep_bytes"]
    # fp64: 48 B -> 16 B per record
    assert make(s, "rest", dtype="f64").query()["sweep_bytes"] < make(s, "stored", dtype="f64").query()["sweep_bytes"]
    # fixed-corotated and batched contexts keep stored rest data
    assert make(G.make_config(5, "small"), "rest").query()["records"] == 1
    assert make(s, "rest", nb=32).query()["records"] == 1
    assert make(s, "table", nb=32).query()["records"] == 1
    # h = 1/14 is not exact in binary: congruent elements' fp64 rest tuples differ in the last bits -> stored
    assert make(s, "table", dtype="f64").query()["records"] == 1
    assert make(G.config3_hetero_cube(n=16), "table", dtype="f64").query()["records"] == 3
    # an irregular mesh (jittered rest positions: every element shape distinct) overflows the table
    rng = np.random.default_rng(0)
    sj = G.make_config(3, "small")
    sj.X = sj.X + rng.uniform(-0.1, 0.1, sj.X.shape) * sj.h
    assert make(sj, "table").query()["records"] == 1
    c = make(s, None)
    with pytest.raises(P.PBNGError) as e:
        c.set_records("rest")  # after pbng_color
    assert e.value.status == 5
    with pytest.raises(KeyError):
        c.set_records("bogus")

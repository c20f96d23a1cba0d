"""The 3D extension on the GPU (BASELINE configs[2..4]) against the restated
3D oracle (oracle/port3.py) and the codec: element matrices within 1e-12,
records bit-exact given the product's own stencils."""
import ctypes
import math

import numpy as np
import pytest

import paper_2005_03606_b200 as lzb
from oracle import port as orc
from oracle import port3 as o3

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("n", [1, 2, 3])
def test_constant_element3(n):
    K = lzb.integrate_elements3(lzb.field3_constant(1.5), [0.0, 1 / 3], [0.0, 2 / 3], [0.0, 0.0], 1 / 3, n)
    for k in K:
        assert _rel(k, 1.5 * o3.unit_stiffness3(1 / 3)) < 1e-14


def test_grf_element3_matches_restatement():
    g = lzb.grf_table(5, 16, 0.05, 1.0)
    f = lzb.field3_grf(g)
    rng = np.random.default_rng(1)
    h = 1 / 27
    cells = rng.integers(0, 27, size=(6, 3))
    for n in (1, 2, 4):
        K = lzb.integrate_elements3(f, cells[:, 0] * h, cells[:, 1] * h, cells[:, 2] * h, h, n)
        for c, k in zip(cells, K):
            want = o3.element3(lambda x, y, z: o3.eps_grf(g, x, y, z), c[0] * h, c[1] * h, c[2] * h, h, n)
            assert _rel(k, want) < 1e-12, (n, c)


def test_extruded_element3_is_the_tensor_product_of_the_2d_element():
    f2 = lzb.field_theta(16.0)
    x0, y0, h, n = 4 / 27, 20 / 27, 1 / 27, 3
    K3 = lzb.integrate_elements3(lzb.field3_extruded(f2), [x0], [y0], [13 / 27], h, n)[0]
    K2 = lzb.integrate_elements(f2, [x0], [y0], [h], [n])[0].reshape(4, 4)
    of = orc.field_from_keys({"setup": "theta", "theta": "16"})
    M2 = o3.mass2(lambda x, y: orc.lib().orc_field_eval(ctypes.byref(of), x, y), x0, y0, h, n)
    assert _rel(K3, o3.extruded_from_2d(K2, M2, h)) < 1e-12


@pytest.mark.parametrize("fixed", [0, 2, 4, 8])
def test_grid3_records_bit_exact(fixed):
    """Stored operator = A(n=1) + roundtrip(A(n) - A(n=1), p3), p3 chosen by the
    (reference-pinned) codec over the 64 entries, or forced."""
    g = lzb.grf_table(9, 16, 0.05, 1.0)
    f = lzb.field3_grf(g)
    G = lzb.Grid3(2, f, delta_max=1e-8, fixed_p3=fixed)
    G.assemble_fixed(3)
    N, h = 9, (1.0 / 3) ** 2
    ops, p3 = G.cells(0, N ** 3)
    idx = np.arange(N ** 3)
    cx, cy, cz = idx % N, (idx // N) % N, idx // (N * N)
    K = lzb.integrate_elements3(f, cx * h, cy * h, cz * h, h, 3).reshape(-1, 64)
    B = lzb.integrate_elements3(f, cx * h, cy * h, cz * h, h, 1).reshape(-1, 64)
    for c in range(0, N ** 3, 37):
        sur = K[c] - B[c]
        want_p3 = fixed if fixed else orc.choose_precision(sur, 1e-8)
        assert p3[c] == want_p3, c
        want = B[c] + lzb.codec.roundtrip(sur, want_p3)
        assert np.array_equal(ops[c].reshape(-1), want), c
    st = G.stats()
    assert st.fine_cells == N ** 3 and sum(st.p3_histogram) == N ** 3
    assert st.fine_stored_bytes == sum(st.p3_histogram[q] * (1 if q == 0 else 1 + 64 * q) for q in range(9))
    if fixed:
        assert st.p3_histogram[fixed] == N ** 3


@pytest.mark.parametrize("depth,solver", [(2, "adafac-pi"), (2, "additive"), (3, "adafac-pi")])
def test_cycle3_matches_restatement(depth, solver):
    """The 3D additive cycle against the numpy restatement (oracle/port3.py
    Cycle3) on the product's own leaf operators: residual history within
    1e-10 relative per cycle, u on every level within 1e-12."""
    g = lzb.grf_table(2, 16, 0.05, 1.0)
    G = lzb.Grid3(depth, lzb.field3_grf(g))
    G.assemble_fixed(2)
    G.init_cycle(solver=solver, omega=0.6, seed=42, max_cycles=100)
    N = 3 ** depth
    ops, _ = G.cells(0, N ** 3)
    ref = o3.Cycle3(ops, depth, variant=solver, omega=0.6, seed=42)
    for _ in range(8):
        a, b = G.step(), ref.step()
        assert a["status"] == b["status"]
        assert a["residual"] == pytest.approx(b["residual"], rel=1e-10)
    for lvl in range(depth + 1):
        u, w = G.vertices(lvl, lzb.T.V_U), ref.v[lvl]["u"]
        assert np.abs(u - w).max() <= 1e-12 * max(np.abs(w).max(), 1.0), lvl


def test_cycle3_converges():
    g = lzb.grf_table(4, 16, 0.05, 1.0)
    G = lzb.Grid3(3, lzb.field3_grf(g))
    G.assemble_fixed(2)
    G.init_cycle(solver="adafac-pi", omega=0.6, max_cycles=300, target=1e-8)
    reps = []
    while True:
        reps.append(G.step())
        if reps[-1]["status"] != lzb.T.CONTINUE:
            break
    assert reps[-1]["status"] == lzb.T.CONVERGED, (len(reps), reps[-1]["normalized"])


@pytest.mark.parametrize("world,solver", [(2, "adafac-pi"), (3, "additive"), (3, "adafac-pi")])
def test_dist_cycle3_loopback_bit_identical(world, solver):
    """The z-slab-distributed 3D cycle (several slabs on the one GPU through
    device copies) against the one-GPU 3D cycle: u on the slab planes and on
    every coarse level bit for bit, residuals to the regrouped norm sum."""
    import torch

    from paper_2005_03606_b200 import parallel
    depth = 3
    g = lzb.grf_table(6, 16, 0.05, 1.0)
    f = lzb.field3_grf(g)
    ref = lzb.Grid3(depth, f)
    ref.assemble_fixed(2)
    ref.init_cycle(solver=solver, omega=0.6, seed=9, max_cycles=100)
    grids = []
    for _ in range(world):
        G = lzb.Grid3(depth, f)
        G.assemble_fixed(2)
        G.init_cycle(solver=solver, omega=0.6, seed=9, max_cycles=100)
        grids.append(G)
    slabs = [parallel.Slab3(G, r, world) for r, G in enumerate(grids)]
    comm = parallel.LoopbackComm(torch.cuda.ExternalStream(lzb.default_context().solve_stream))
    for _ in range(6):
        w, d = ref.step(), parallel.dist_cycle3(slabs, comm, solver == "adafac-pi")
        assert d["status"] == w["status"] and d["residual"] == pytest.approx(w["residual"], rel=1e-12)
    N = 3 ** depth
    for s in slabs:
        for lvl in range(depth):
            assert np.array_equal(s.grid.vertices(lvl, lzb.T.V_U), ref.vertices(lvl, lzb.T.V_U)), lvl
        a, b = s.grid.vertices(depth, lzb.T.V_U), ref.vertices(depth, lzb.T.V_U)
        assert np.array_equal(a[s.v0:min(s.v1, N + 1)], b[s.v0:min(s.v1, N + 1)])


@pytest.mark.parametrize("width,fixed", [(2, 2), (3, 3), (4, 0), (5, 4), (6, 6), (7, 7), (8, 0), (8, 8)])
def test_grid3_compressed_planes_bit_identical(width, fixed):
    """Leaf operators held only as compressed class planes (BASELINE
    configs[4]): the decoded operators, and the cycle that reads them (the
    residual and the Galerkin coarse operators decode the planes), are bit
    for bit those of the FP64 grid."""
    g = lzb.grf_table(3, 16, 0.05, 1.0)
    f = lzb.field3_grf(g)
    grids = [lzb.Grid3(2, f, delta_max=1e-4, fixed_p3=fixed),
             lzb.Grid3(2, f, delta_max=1e-4, fixed_p3=fixed, plane_width=width)]
    for G in grids:
        G.assemble_fixed(3)
        G.init_cycle(solver="adafac-pi", omega=0.6, seed=7, max_cycles=100)
    (a_ops, a_p3), (b_ops, b_p3) = (G.cells(0, 9 ** 3) for G in grids)
    assert np.array_equal(a_p3, b_p3) and np.array_equal(a_ops, b_ops)
    for _ in range(4):
        ra, rb = (G.step() for G in grids)
        assert ra["residual"] == rb["residual"] and ra["status"] == rb["status"]
    for lvl in range(3):
        assert np.array_equal(grids[0].vertices(lvl, lzb.T.V_U), grids[1].vertices(lvl, lzb.T.V_U)), lvl
    assert grids[1].leaf_bytes_per_cell() == 27 * width + 9


def test_grid3_planes_reject_wide_records():
    g = lzb.grf_table(3, 16, 0.05, 1.0)
    G = lzb.Grid3(2, lzb.field3_grf(g), delta_max=0.0, plane_width=3)  # exact records need p3 = 8
    with pytest.raises(lzb.ResourceError):
        G.assemble_fixed(3)
    with pytest.raises(lzb.LzbError):
        lzb.Grid3(2, lzb.field3_grf(g), fixed_p3=5, plane_width=4)


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_assemble3_loopback(world):
    """z-slab sharded assembly (each slab assembles only the leaf planes its
    cycle reads and its level-(D-1) Galerkin planes, one all-gather of those)
    feeding the slab-distributed cycle: the same u, bit for bit, as the
    one-GPU grid assembled whole."""
    import torch

    from paper_2005_03606_b200 import parallel
    depth = 3
    f = lzb.field3_grf(lzb.grf_table(8, 16, 0.05, 1.0))
    ref = lzb.Grid3(depth, f)
    ref.assemble_fixed(3)
    ref.init_cycle(solver="adafac-pi", omega=0.6, seed=5, max_cycles=100)
    slabs = []
    for r in range(world):
        G = lzb.Grid3(depth, f)
        G.init_cycle(solver="adafac-pi", omega=0.6, seed=5, max_cycles=100)
        slabs.append(parallel.Slab3(G, r, world))
    comm = parallel.LoopbackComm(torch.cuda.ExternalStream(lzb.default_context().solve_stream))
    parallel.distributed_assemble3(slabs, comm, 3)
    for _ in range(5):
        w, d = ref.step(), parallel.dist_cycle3(slabs, comm, True)
        assert d["status"] == w["status"] and d["residual"] == pytest.approx(w["residual"], rel=1e-12)
    N = 3 ** depth
    for s in slabs:
        for lvl in range(depth):
            assert np.array_equal(s.grid.vertices(lvl, lzb.T.V_U), ref.vertices(lvl, lzb.T.V_U)), lvl
        a, b = s.grid.vertices(depth, lzb.T.V_U), ref.vertices(depth, lzb.T.V_U)
        assert np.array_equal(a[s.v0:min(s.v1, N + 1)], b[s.v0:min(s.v1, N + 1)])


def test_tree3_sphere_leaves_and_elements():
    """BASELINE configs[3] assembly on the adaptive spacetree: the leaf set of
    the restated construction (oracle/port3.py sphere_tree_leaves), element
    matrices of leaves on every level against the literal per-sample
    restatement (1e-12), records bit-exact given the product's stencils, and
    the delayed shell re-assembly touching only the interface leaves."""
    f = lzb.field3_sphere()
    T3 = lzb.Tree3(1, 3, f, delta_max=1e-8)
    want = o3.sphere_tree_leaves(1, 3)
    assert T3.n_leaves == len(want)
    assert list(T3.per_level[:4]) == list(np.bincount(want[:, 0], minlength=4))
    T3.assemble(2)
    ops, p3, n, lxyz = T3.cells(0, T3.n_leaves)
    assert np.array_equal(lxyz, want.astype(np.int32)) and (n == 2).all()
    rng = np.random.default_rng(3)
    pick = np.concatenate([rng.choice(np.where(lxyz[:, 0] == lv)[0], 4, replace=False) for lv in (1, 2, 3)])
    h = np.array([math.pow(1.0 / 3, lv) for lv in range(8)])[lxyz[pick, 0]]  # libm pow, as the host side
    x0, y0, z0 = (lxyz[pick, d + 1] * h for d in range(3))
    K = lzb.integrate_elements3(f, x0, y0, z0, h, 2).reshape(-1, 64)
    B = lzb.integrate_elements3(f, x0, y0, z0, h, 1).reshape(-1, 64)
    for i, c in enumerate(pick):
        lit = o3.element3(o3.eps_sphere, x0[i], y0[i], z0[i], h[i], 2)
        assert _rel(K[i].reshape(8, 8), lit) < 1e-12
        sur = K[i] - B[i]
        assert p3[c] == orc.choose_precision(sur, 1e-8)
        assert np.array_equal(ops[c].reshape(-1), B[i] + lzb.codec.roundtrip(sur, p3[c]))
    cnt = T3.set_shell(0.02)
    assert 0 < cnt < T3.n_leaves
    T3.assemble_shell(4)
    ops2, _, n2, _ = T3.cells(0, T3.n_leaves)
    moved = n2 == 4
    assert moved.sum() == cnt
    assert np.array_equal(ops2[~moved], ops[~moved])
    st = T3.stats()
    assert st.fine_cells == T3.n_leaves and sum(st.p3_histogram) == T3.n_leaves and st.max_n == 4


@pytest.mark.parametrize("solver,lbase,lmax", [("adafac-pi", 1, 3), ("additive", 1, 3), ("adafac-pi", 2, 3)])
def test_tree3_cycle_matches_restatement(solver, lbase, lmax):
    """The additive cycle on the adaptive sphere tree (hanging vertices) against
    the numpy restatement (oracle/port3.py Cycle3A) on the product's own leaf
    operators: residual history within 1e-10 relative per cycle, u on every
    level within 1e-12; and the shell re-assembly + refresh keeps it in step."""
    f = lzb.field3_sphere()
    T3 = lzb.Tree3(lbase, lmax, f, delta_max=1e-8)
    T3.assemble(2)
    T3.init_cycle(solver=solver, omega=0.6, seed=11, max_cycles=100)
    ops, _, _, lxyz = T3.cells(0, T3.n_leaves)
    ref = o3.Cycle3A(lxyz, ops, lmax, variant=solver, omega=0.6, seed=11)
    for _ in range(6):
        a, b = T3.step(), ref.step()
        assert a["status"] == b["status"]
        assert a["residual"] == pytest.approx(b["residual"], rel=1e-10)
    for lvl in range(lmax + 1):
        u, w = T3.vertices(lvl, lzb.T.V_U), ref.v[lvl]["u"]
        assert np.abs(u - w).max() <= 1e-12 * max(np.abs(w).max(), 1.0), lvl


@pytest.mark.parametrize("solver,lbase,lmax,radius", [("adafac-pi", 1, 3, 0.34), ("additive", 2, 3, 0.3)])
def test_tree3_rerefinement_matches_restatement(solver, lbase, lmax, radius):
    """Re-refinement during the solve (BASELINE configs[3]: the refined region
    grows, topology changes, new leaves are assembled -- the reference's
    apply_refinement_now, solver.cpp:402-418): surviving leaves keep their
    operators bit for bit, the new ones are their fresh integration, the new
    vertices start from the parent interpolant, and the cycle continues in
    step with the restatement doing the same refinement."""
    f = lzb.field3_sphere()
    T3 = lzb.Tree3(lbase, lmax, f, delta_max=1e-8)
    T3.assemble(2)
    T3.init_cycle(solver=solver, omega=0.6, seed=11, max_cycles=100)
    ops, _, _, lxyz = T3.cells(0, T3.n_leaves)
    ref = o3.Cycle3A(lxyz, ops, lmax, variant=solver, omega=0.6, seed=11)
    for _ in range(3):
        a, b = T3.step(), ref.step()
        assert a["residual"] == pytest.approx(b["residual"], rel=1e-10)
    n0 = T3.n_leaves
    k = T3.refine(radius, 2)
    assert k > 0 and T3.n_leaves > n0
    ops2, p32, n2, lxyz2 = T3.cells(0, T3.n_leaves)
    old = {tuple(c): o for c, o in zip(lxyz.tolist(), ops)}
    fresh = [i for i, c in enumerate(lxyz2.tolist()) if tuple(c) not in old]
    assert len(fresh) == k
    for i, c in enumerate(lxyz2.tolist()):
        if tuple(c) in old:
            assert np.array_equal(ops2[i], old[tuple(c)])
    # the new leaves: their element matrices at n = 2 (codec-absorbed, delta 1e-8)
    sel = fresh[:: max(1, len(fresh) // 16)]
    h = np.array([(1.0 / 3) ** lxyz2[i][0] for i in sel])
    want = lzb.integrate_elements3(f, lxyz2[sel, 1] * h, lxyz2[sel, 2] * h, lxyz2[sel, 3] * h, h, 2)
    assert np.abs(ops2[sel] - want).max() <= 1e-7 and (n2[fresh] == 2).all()
    ref.refine(lxyz2, ops2)
    for lvl in range(lmax + 1):
        u, w = T3.vertices(lvl, lzb.T.V_U), ref.v[lvl]["u"]
        assert np.abs(u - w).max() <= 1e-12 * max(np.abs(w).max(), 1.0), lvl
    for _ in range(4):
        a, b = T3.step(), ref.step()
        assert a["status"] == b["status"] and a["cycle"] == b["cycle"]
        assert a["residual"] == pytest.approx(b["residual"], rel=1e-10)
    for lvl in range(lmax + 1):
        u, w = T3.vertices(lvl, lzb.T.V_U), ref.v[lvl]["u"]
        assert np.abs(u - w).max() <= 1e-12 * max(np.abs(w).max(), 1.0), lvl
    with pytest.raises(lzb.LzbError):
        T3.refine(radius - 0.1, 2)  # no coarsening (mesh.hpp:55)


@pytest.mark.parametrize("depth,nu", [(2, 1), (3, 2)])
def test_vcycle3_matches_restatement(depth, nu):
    """V(nu, nu) cycles on the 3D hierarchy (the BASELINE configs' V(1,1) /
    V(2,2)) against the numpy restatement on the product's leaf operators:
    residual history within 1e-10 per cycle, u within 1e-12; and they converge."""
    g = lzb.grf_table(2, 16, 0.05, 1.0)
    G = lzb.Grid3(depth, lzb.field3_grf(g))
    G.assemble_fixed(2)
    G.init_cycle(solver="additive", omega=0.6, seed=42, max_cycles=100)
    N = 3 ** depth
    ops, _ = G.cells(0, N ** 3)
    ref = o3.Cycle3(ops, depth, variant="additive", omega=0.6, seed=42)
    reps = []
    for _ in range(6):
        a, b = G.vcycle(nu), ref.vstep(nu)
        assert a["status"] == b["status"]
        assert a["residual"] == pytest.approx(b["residual"], rel=1e-10)
        reps.append(a)
    u, w = G.vertices(depth, lzb.T.V_U), ref.v[depth]["u"]
    assert np.abs(u - w).max() <= 1e-12 * max(np.abs(w).max(), 1.0)
    assert reps[-1]["normalized"] < 0.1


def test_vcycle3_then_step_matches_restatement():
    """V-cycles and additive steps mixed on one grid: after a
    V-cycle the coarse u is the injected fine u again, so a following
    additive step forms u-hat from the solution; the mixed sequence matches
    the restatement doing the same."""
    depth = 3
    g = lzb.grf_table(3, 16, 0.05, 1.0)
    G = lzb.Grid3(depth, lzb.field3_grf(g))
    G.assemble_fixed(2)
    G.init_cycle(solver="adafac-pi", omega=0.6, seed=42, max_cycles=100)
    ops, _ = G.cells(0, 27 ** 3)
    ref = o3.Cycle3(ops, depth, variant="adafac-pi", omega=0.6, seed=42)
    for kind in ("v", "v", "s", "s", "v", "s"):
        a, b = (G.vcycle(1), ref.vstep(1)) if kind == "v" else (G.step(), ref.step())
        assert a["residual"] == pytest.approx(b["residual"], rel=1e-10), kind
        if kind == "v":
            for lvl in range(depth):
                uc, uf = G.vertices(lvl, lzb.T.V_U), G.vertices(lvl + 1, lzb.T.V_U)
                assert np.array_equal(uc, uf[::3, ::3, ::3]), lvl
    for lvl in range(depth + 1):
        u, w = G.vertices(lvl, lzb.T.V_U), ref.v[lvl]["u"]
        assert np.abs(u - w).max() <= 1e-12 * max(np.abs(w).max(), 1.0), lvl


def test_reinit_cycle_keeps_coarse_operators():
    """init_cycle after a solve (bench.py's C3 sequence: adaFAC-PI solve, then
    V(2,2) cycles on the same operators) re-allocates the vertex arrays; the
    coarse Galerkin operators must survive it (or be re-formed): the V-cycle
    history equals a fresh grid's, bit for bit."""
    f = lzb.field3_grf(lzb.grf_table(4, 16, 0.05, 1.0))

    def vhist(pre):
        g = lzb.Grid3(3, f, delta_max=1e-8)
        g.assemble_fixed(3)
        if pre:
            g.init_cycle(solver="adafac-pi", omega=0.6, seed=11, max_cycles=100)
            # other allocations come and go in between, as in a long-lived process
            junk = [lzb.Grid3(2, f) for _ in range(3)]
            for _ in range(6):
                g.step()
            for j in junk:
                j.close()
        g.init_cycle(solver="additive", omega=0.6, seed=5, max_cycles=100)
        out = [g.vcycle(2)["residual"] for _ in range(4)]
        g.close()
        return out

    a, b = vhist(False), vhist(True)
    assert a == b
    assert a[3] < 0.05 * a[0]  # the coarse correction works (smoothing alone gives ~0.5)


_UPDATE3_SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, ".")
import numpy as np
import paper_2005_03606_b200 as lzb
depth, solver = int(sys.argv[1]), sys.argv[2]
G = lzb.Grid3(depth, lzb.field3_grf(lzb.grf_table(5, 16, 0.05, 1.0)))
G.assemble_fixed(1)
G.init_cycle(solver=solver, omega=0.6, seed=42, max_cycles=100)
res = [G.step()["residual"] for _ in range(3)]
u = G.vertices(depth, lzb.T.V_U)
print("HASH", hashlib.sha256(np.ascontiguousarray(u).tobytes()).hexdigest(), " ".join(repr(x) for x in res))
"""


@pytest.mark.parametrize("depth,solver", [(3, "adafac-pi"), (4, "additive"), (5, "adafac-pi")])
def test_update3_march_bit_identical_to_row_kernel(depth, solver):
    """The marching leaf update (k3_update_fine_march: 27 owner-patch rows per
    block, ring of coarse lines, next rows prefetched) against the row-block
    kernel it replaces (LZB_UPDATE3_ROWS=1): identical u bits and residuals
    after three cycles; depth 5 has three march chunks per column, depth 3 a
    short one (9 patches)."""
    import os
    import subprocess
    import sys

    outs = []
    for rows in (False, True):
        env = dict(os.environ)
        env.pop("LZB_UPDATE3_ROWS", None)
        env.pop("LZB_UHAT3_MARCH", None)
        if rows:
            env["LZB_UPDATE3_ROWS"] = "1"
        else:
            env["LZB_UHAT3_MARCH"] = "1"  # the opt-in marching u-hat too (from 243^3 up)
        p = subprocess.run([sys.executable, "-c", _UPDATE3_SCRIPT, str(depth), solver], env=env, capture_output=True,
                           text=True, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        outs.append([ln for ln in p.stdout.splitlines() if ln.startswith("HASH")][0])
    assert outs[0] == outs[1]

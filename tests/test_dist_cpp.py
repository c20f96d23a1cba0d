"""The slab-distributed data plane in C++ (csrc/dist.cpp).

The driver runs the grid's compute phases with the exchanges in between on
the solve stream; its NCCL transport (send/recv halos, in-place broadcasts of
the replicated level D-1, on-device all-reduce of the norm and counters) and
its loopback transport (several slabs of one process, device copies) execute
the same plan. On the one GPU of the test box the loopback transport checks
the plan with 2 and 3 slabs bit for bit against the undistributed cycle, and
the NCCL transport runs with a communicator of one rank (no peer exists here:
the multi-rank exchange logic is covered by the loopback slabs and by the
gloo tests of tests/test_parallel.py).
"""
import numpy as np
import pytest

import paper_2005_03606_b200 as lzb

pytestmark = pytest.mark.gpu


def slab_vertex_rows(N, world, rank):
    from paper_2005_03606_b200 import parallel
    return parallel.slab_vertex_rows(N, world, rank)


def _desc(depth, solver):
    return lzb.make_desc(depth=depth, field=lzb.field_theta(16.0), solver=solver, omega=0.6, rhs_kind="sinprod",
                         max_cycles=200, delta_max=1e-8)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("solver", ["additive", "adafac-pi"])
def test_cpp_dist_cycle_loopback_bit_identical(world, solver):
    depth, cycles = 4, 6
    ref = lzb.Grid(_desc(depth, solver), 42)
    ref.assemble_fixed(3)
    want = [ref.step() for _ in range(cycles)]
    grids = [lzb.Grid(_desc(depth, solver), 42) for _ in range(world)]
    for g in grids:
        g.assemble_fixed(3)
    got = [lzb.dist_cycle_loopback(grids) for _ in range(cycles)]
    for w, g in zip(want, got):
        assert g["status"] == w["status"] and g["cycle"] == w["cycle"]
        assert g["residual"] == pytest.approx(w["residual"], rel=1e-12)
        for k in ("dof_updates", "max_n", "factor_totals", "pending_tasks", "coarse_updates"):
            assert g[k] == w[k], k
    N = 3 ** depth
    for r, g in enumerate(grids):
        v0, v1 = slab_vertex_rows(N, world, r)
        for fld in (lzb.T.V_U, lzb.T.V_R, lzb.T.V_RHAT, lzb.T.V_DIAG):
            a = g.vertices(depth, fld).reshape(N + 1, N + 1)[v0:v1]
            assert np.array_equal(a, ref.vertices(depth, fld).reshape(N + 1, N + 1)[v0:v1]), (r, fld)
        for lvl in range(depth):
            for fld in (lzb.T.V_U, lzb.T.V_FL, lzb.T.V_R):
                assert np.array_equal(g.vertices(lvl, fld), ref.vertices(lvl, fld)), (r, lvl, fld)


@pytest.mark.parametrize("world", [2, 4])
def test_cpp_dist_assemble_and_solve_loopback(world):
    """Slab assembly (each slab integrates its leaf rows) + the exchange of the
    leaf state, then distributed cycles to convergence: the one-GPU history."""
    depth = 5
    d = lzb.make_desc(depth=depth, field=lzb.field_sinusoid(0.9, 6.0), solver="adafac-pi", omega=0.6,
                      rhs_kind="sinprod", max_cycles=300, target=1e-9)
    ref = lzb.Grid(d, 42)
    ref.assemble_fixed(4)
    want = ref.run()
    grids = [lzb.Grid(d, 42) for _ in range(world)]
    lzb.dist_assemble_loopback(grids, 4)
    for g in grids:
        assert np.array_equal(g.cells(depth)["ops"], ref.cells(depth)["ops"])
    got = []
    while True:
        got.append(lzb.dist_cycle_loopback(grids))
        if got[-1]["status"] != lzb.T.CONTINUE:
            break
    assert len(got) == len(want) and got[-1]["status"] == lzb.T.CONVERGED
    for a, b in zip(got, want):
        assert a["residual"] == pytest.approx(b["residual"], rel=1e-11)


@pytest.mark.parametrize("world,solver", [(2, "adafac-pi"), (3, "additive")])
def test_cpp_dist_cycle3_loopback(world, solver):
    depth = 3
    f = lzb.field3_grf(lzb.grf_table(6, 16, 0.05, 1.0))
    ref = lzb.Grid3(depth, f)
    ref.assemble_fixed(2)
    ref.init_cycle(solver=solver, omega=0.6, seed=9, max_cycles=100)
    grids = []
    for _ in range(world):
        G = lzb.Grid3(depth, f)
        G.init_cycle(solver=solver, omega=0.6, seed=9, max_cycles=100)
        grids.append(G)
    lzb.dist_assemble_loopback(grids, 2)  # z-slab sharded assembly + the level D-1 plane exchange
    for _ in range(6):
        w, g = ref.step(), lzb.dist_cycle_loopback(grids)
        assert g["status"] == w["status"] and g["residual"] == pytest.approx(w["residual"], rel=1e-12)
    N = 3 ** depth
    for r, G in enumerate(grids):
        v0, v1 = slab_vertex_rows(N, world, r)
        for lvl in range(depth):
            assert np.array_equal(G.vertices(lvl, lzb.T.V_U), ref.vertices(lvl, lzb.T.V_U)), lvl
        a, b = G.vertices(depth, lzb.T.V_U), ref.vertices(depth, lzb.T.V_U)
        assert np.array_equal(a[v0:v1], b[v0:v1])


@pytest.mark.parametrize("world,solver,width", [(2, "adafac-pi", 0), (3, "additive", 0), (3, "adafac-pi", 4)])
def test_cpp_dist_cycle3_slab_local_storage(world, solver, width):
    """Slab-local leaf operators (SURVEY §8e memory scaling): each slab grid
    stores only the leaf cell layers its kernels read (its vertex planes' cells
    and one layer below; lzb_grid3_create_slab), FP64 class planes or
    compressed planes; the sharded assembly and the distributed cycle (TMA
    tiles over the windowed tensors) give the undistributed grid's u bit for
    bit, on about 1/world of the leaf operator memory each."""
    depth = 3
    N = 3 ** depth
    f = lzb.field3_grf(lzb.grf_table(6, 16, 0.05, 1.0))
    fixed = 4 if width else 0
    ref = lzb.Grid3(depth, f, delta_max=1e-4, fixed_p3=fixed)
    ref.assemble_fixed(2)
    ref.init_cycle(solver=solver, omega=0.6, seed=9, max_cycles=100)
    whole, _, _ = lzb.Grid3(depth, f, delta_max=1e-4, fixed_p3=fixed, plane_width=width).leaf_storage()
    grids, total = [], 0
    for r in range(world):
        G = lzb.Grid3(depth, f, delta_max=1e-4, fixed_p3=fixed, plane_width=width, slab=(r, world))
        v0, v1 = slab_vertex_rows(N, world, r)
        b, z0, z1 = G.leaf_storage()
        assert (z0, z1) == (max(v0 - 1, 0), min(v1, N))
        assert b * N == whole * (z1 - z0)  # bytes proportional to the stored layers
        total += b
        G.init_cycle(solver=solver, omega=0.6, seed=9, max_cycles=100)
        grids.append(G)
    assert total <= whole * (N + world - 1) // N  # one halo layer per interior slab boundary
    lzb.dist_assemble_loopback(grids, 2)
    for _ in range(6):
        w, g = ref.step(), lzb.dist_cycle_loopback(grids)
        assert g["status"] == w["status"] and g["residual"] == pytest.approx(w["residual"], rel=1e-12)
    for r, G in enumerate(grids):
        v0, v1 = slab_vertex_rows(N, world, r)
        for lvl in range(depth):
            assert np.array_equal(G.vertices(lvl, lzb.T.V_U), ref.vertices(lvl, lzb.T.V_U)), lvl
        a, b = G.vertices(depth, lzb.T.V_U), ref.vertices(depth, lzb.T.V_U)
        assert np.array_equal(a[v0:v1], b[v0:v1])
        # the stored operators are the undistributed grid's; layers outside the window are not held
        _, z0, z1 = G.leaf_storage()
        ops_g, _ = G.cells(z0 * N * N, (z1 - z0) * N * N)
        ops_r, _ = ref.cells(z0 * N * N, (z1 - z0) * N * N)
        assert np.array_equal(ops_g, ops_r)
        if z0 > 0:
            with pytest.raises(lzb.LzbError):
                G.cells(0, N * N)
        with pytest.raises(lzb.LzbError):
            G.step()  # the one-GPU cycle reads every leaf


def test_cpp_dist_nccl_single_rank():
    """The NCCL transport with a communicator of one rank (the context owns
    it): the 2D and 3D distributed cycles equal the undistributed ones."""
    ctx = lzb.Context(0)
    ctx.comm_init(lzb.nccl_unique_id(), 1, 0)
    assert ctx.comm_info() == (0, 1)
    d = _desc(4, "adafac-pi")
    ref, g = lzb.Grid(d, 42, ctx), lzb.Grid(d, 42, ctx)
    ref.assemble_fixed(3)
    g.dist_assemble(3)
    for _ in range(5):
        w, r = ref.step(), g.dist_cycle()
        assert r["status"] == w["status"] and r["residual"] == pytest.approx(w["residual"], rel=1e-12)
    assert np.array_equal(g.vertices(4, lzb.T.V_U), ref.vertices(4, lzb.T.V_U))
    f = lzb.field3_grf(lzb.grf_table(6, 16, 0.05, 1.0))
    r3, g3 = lzb.Grid3(3, f, ctx=ctx), lzb.Grid3(3, f, ctx=ctx)
    r3.assemble_fixed(2)
    r3.init_cycle(solver="adafac-pi", omega=0.6, seed=9, max_cycles=100)
    g3.init_cycle(solver="adafac-pi", omega=0.6, seed=9, max_cycles=100)
    g3.dist_assemble(2)
    for _ in range(4):
        w, r = r3.step(), g3.dist_cycle()
        assert r["residual"] == pytest.approx(w["residual"], rel=1e-12)
    assert np.array_equal(g3.vertices(3, lzb.T.V_U), r3.vertices(3, lzb.T.V_U))
    for x in (ref, g, r3, g3):
        x.close()
    ctx.close()


def test_cpp_dist_without_communicator_fails_loudly():
    g = lzb.Grid(_desc(3, "adafac-pi"), 1)
    with pytest.raises(lzb.LzbError):
        g.dist_cycle()

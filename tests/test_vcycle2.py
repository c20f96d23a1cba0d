"""The 2D V(nu, nu) cycle (BASELINE configs[1] names V(1,1)): the numpy
restatement's own properties on CPU (transfer adjointness, convergence on the
constant-coefficient Q1 hierarchy) and, on the GPU, lzb_grid_vcycle against
the restatement on the product's operators and transfers."""
import numpy as np
import pytest

import paper_2005_03606_b200 as lzb
from oracle import port as orc
from oracle.port2v import VCycle2

Q1 = np.array([[4, -1, -1, -2], [-1, 4, -2, -1], [-1, -2, 4, -1], [-2, -1, -1, 4]]) / 6.0


def q1_hierarchy(D, seed=0):
    rng = np.random.default_rng(seed)
    ops = [np.tile(Q1.reshape(16), (9 ** l, 1)) for l in range(D + 1)]
    P = [np.tile(orc.geometric().reshape(16, 4), (9 ** l, 1, 1)) for l in range(D)]
    n = 3 ** D
    fl = rng.standard_normal((n + 1, n + 1)) / n ** 2
    u = rng.standard_normal((n + 1, n + 1))
    u[0, :] = u[-1, :] = u[:, 0] = u[:, -1] = 0.0
    return ops, P, fl, u


def test_restatement_transfers_are_adjoint():
    """<P^T r, v_c> = <r, P v_c> on interior fine vertices: the owned-lattice
    restriction and the owner-patch prolongation are transposes."""
    ops, P, fl, u = q1_hierarchy(3, seed=1)
    V = VCycle2(ops, P, fl, u, omega=0.6)
    rng = np.random.default_rng(2)
    n = 27
    r = rng.standard_normal((n + 1, n + 1))
    r[0, :] = r[-1, :] = r[:, 0] = r[:, -1] = 0.0
    vc = rng.standard_normal((10, 10))
    vc[0, :] = vc[-1, :] = vc[:, 0] = vc[:, -1] = 0.0
    lhs = float(np.sum(V.restrict(3, r) * vc))
    V.u[2] = vc
    V.u[3] = np.zeros((n + 1, n + 1))
    V.prolong(3)
    rhs = float(np.sum(r * V.u[3]))
    assert lhs == pytest.approx(rhs, rel=1e-12)


@pytest.mark.parametrize("nu", [1, 2])
def test_restatement_converges_on_q1(nu):
    """Galerkin-consistent constant-coefficient Q1 hierarchy: a V(nu, nu)
    cycle contracts the residual at a grid-independent rate (factor-3
    coarsening with damped Jacobi: about 0.57 for V(1,1), 0.34 for V(2,2);
    the coarsest level with interior vertices is smoothed, not solved)."""
    for D in (3, 4):
        ops, P, fl, u = q1_hierarchy(D, seed=D)
        V = VCycle2(ops, P, fl, u, omega=0.6)
        reps = [V.vstep(nu) for _ in range(8)]
        rates = [b["residual"] / a["residual"] for a, b in zip(reps[2:], reps[3:])]
        assert max(rates) < (0.65 if nu == 1 else 0.4), rates


@pytest.mark.gpu
@pytest.mark.parametrize("depth,nu,transfer,field", [
    (3, 1, "geometric", "checkerboard"), (4, 1, "geometric", "checkerboard"),
    (4, 2, "boxmg", "checkerboard"), (4, 1, "geometric", "theta")])
def test_vcycle_matches_restatement(depth, nu, transfer, field):
    """lzb_grid_vcycle on an assembled grid against the restatement started
    from the same u, load, operators and transfer blocks: residual history
    within 1e-10 per cycle, leaf u within 1e-12; and it converges."""
    f = lzb.checkerboard(7, 8) if field == "checkerboard" else lzb.field_theta(16.0)
    d = lzb.make_desc(depth=depth, field=f, solver="additive", omega=0.6, rhs_kind="sinprod",
                      max_cycles=100, transfer=transfer)
    G = lzb.Grid(d, 42)
    G.assemble_fixed(3)
    u0 = G.vertices(depth, lzb.T.V_U).copy()
    a = G.vcycle(nu)
    fl = G.vertices(depth, lzb.T.V_FL)
    ops = [G.cells(l)["ops"] for l in range(depth + 1)]
    P = [np.array([[G.transfer(l, cx, cy) for cx in range(3 ** l)] for cy in range(3 ** l)])
         for l in range(depth)]
    ref = VCycle2(ops, P, fl, u0, omega=0.6, max_cycles=100)
    reps = [a]
    b = ref.vstep(nu)
    for k in range(6):
        assert a["status"] == b["status"]
        assert a["residual"] == pytest.approx(b["residual"], rel=1e-10), k
        if k < 5:
            a, b = G.vcycle(nu), ref.vstep(nu)
            reps.append(a)
    u, w = G.vertices(depth, lzb.T.V_U), ref.u[depth]
    assert np.abs(u - w).max() <= 1e-12 * max(np.abs(w).max(), 1.0)
    assert reps[-1]["normalized"] < 0.2
    assert reps[-1]["dof_updates"] == 2 * nu * (3 ** depth - 1) ** 2


@pytest.mark.gpu
def test_vcycle_rejects_bad_nu():
    G = lzb.Grid(lzb.make_desc(depth=2, solver="additive"), 1)
    with pytest.raises(Exception):
        G.vcycle(-1)


@pytest.mark.gpu
def test_vcycle_sweep_count_change_and_compressed_leaves():
    """Changing nu between cycles re-captures the sweep graph (the restatement
    follows the same nu sequence); the compressed leaf records (plane_width)
    give the FP64 residual history bit for bit."""
    def grid(width):
        d = lzb.make_desc(depth=4, field=lzb.field_theta(16.0), solver="additive", omega=0.6,
                          rhs_kind="sinprod", max_cycles=100, plane_width=width)
        G = lzb.Grid(d, 42)
        G.assemble_fixed(3)
        return G

    seq = [1, 2, 1, 3, 1]
    G = grid(0)
    u0 = G.vertices(4, lzb.T.V_U).copy()
    a = [G.vcycle(seq[0])]
    fl = G.vertices(4, lzb.T.V_FL)
    ops = [G.cells(l)["ops"] for l in range(5)]
    P = [np.array([[G.transfer(l, cx, cy) for cx in range(3 ** l)] for cy in range(3 ** l)]) for l in range(4)]
    ref = VCycle2(ops, P, fl, u0, omega=0.6, max_cycles=100)
    b = [ref.vstep(seq[0])]
    for nu in seq[1:]:
        a.append(G.vcycle(nu))
        b.append(ref.vstep(nu))
    for x, y in zip(a, b):
        assert x["residual"] == pytest.approx(y["residual"], rel=1e-10)
    H = grid(4)
    c = [H.vcycle(nu) for nu in seq]
    assert [x["residual"] for x in a] == [x["residual"] for x in c]


@pytest.mark.gpu
@pytest.mark.parametrize("depth", [1, 2])
def test_vcycle_shallow_grids(depth):
    """Depth 1 (one coarse level without interior vertices) and 2: the cycle
    runs, matches the restatement and contracts."""
    d = lzb.make_desc(depth=depth, field=lzb.checkerboard(3, 8), solver="additive", omega=0.6,
                      rhs_kind="sinprod", max_cycles=100)
    G = lzb.Grid(d, 5)
    G.assemble_fixed(2)
    u0 = G.vertices(depth, lzb.T.V_U).copy()
    a = [G.vcycle(1)]
    fl = G.vertices(depth, lzb.T.V_FL)
    ops = [G.cells(l)["ops"] for l in range(depth + 1)]
    P = [np.array([[G.transfer(l, cx, cy) for cx in range(3 ** l)] for cy in range(3 ** l)]) for l in range(depth)]
    ref = VCycle2(ops, P, fl, u0, omega=0.6, max_cycles=100)
    b = [ref.vstep(1)]
    for _ in range(4):
        a.append(G.vcycle(1))
        b.append(ref.vstep(1))
    for x, y in zip(a, b):
        assert x["residual"] == pytest.approx(y["residual"], rel=1e-10)
    assert a[-1]["residual"] < a[0]["residual"]


@pytest.mark.gpu
def test_vcycle_on_unassembled_leaves_converges():
    """Delayed assembly before any integration: the leaves still carry the
    bottom (eps at the centre) stencils, the V-cycle runs on them and
    converges; a later additive step on the same grid still works."""
    d = lzb.make_desc(depth=4, field=lzb.field_sinusoid(0.9, 6.0), solver="additive", omega=0.6,
                      rhs_kind="sinprod", max_cycles=100, assembly="lazy")
    G = lzb.Grid(d, 7)
    reps = [G.vcycle(2) for _ in range(8)]
    assert reps[-1]["normalized"] < 1e-3
    assert G.step()["cycle"] == 9


@pytest.mark.gpu
@pytest.mark.parametrize("solver", ["additive", "adafac-pi"])
def test_vcycle_then_step_uses_injected_solution(solver):
    """after vcycle() the coarse u is the injected fine u (the
    additive cycle's invariant), so a following step() equals a step on a
    grid that starts from the same leaf u and operators, bit for bit."""
    depth = 4
    d = lzb.make_desc(depth=depth, field=lzb.checkerboard(7, 8), solver=solver, omega=0.6, rhs_kind="sinprod",
                      max_cycles=100)
    A = lzb.Grid(d, 42)
    A.assemble_fixed(3)
    A.vcycle(1)
    A.vcycle(2)
    for lvl in range(depth):
        assert np.array_equal(A.vertices(lvl, lzb.T.V_U), A.vertices(lvl + 1, lzb.T.V_U)[::3, ::3])
    B = lzb.Grid(d, 42)
    B.assemble_fixed(3)
    B.vcycle(1)  # the same coarse operators (finest-first Galerkin pass) as A's
    B.set_vertices(depth, lzb.T.V_U, A.vertices(depth, lzb.T.V_U))
    B.pass_(4)  # finish_cycle_sync: inject into the coarse levels
    ra, rb = A.step(), B.step()
    assert ra["residual"] == rb["residual"]
    for lvl in range(depth + 1):
        assert np.array_equal(A.vertices(lvl, lzb.T.V_U), B.vertices(lvl, lzb.T.V_U)), lvl

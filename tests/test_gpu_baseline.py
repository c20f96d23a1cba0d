"""Parity on the BASELINE.json configurations at their stated sizes.

The other GPU suites pin the path at depths <= 4 (plus a few depth-5/6
cycles); these run the benched kernels on the configs' own grids:

* C2 (configs[1]): the fused fixed-p assembly kernel that bench.py times
  (k_fixed_res: integrate + compress + publish) on all 531,441 cells of the
  729^2 grid at p = 32, every cell's integrated matrix against the oracle's
  integrate_element (element.hpp:36-49): bit-identical on the EXACT path (the
  field's sines from the host libm), 1e-12 normwise on the FAST one, and the LZMG stream of that pass
  byte-equal to the oracle publishing the same matrices (stream.cpp:100-132,
  303-338);
* C1 (configs[0]): 243^2, 8x8 checkerboard, p = 1, 2, 4, 8, 16 fixed-p
  assembly, operators on every level bit-identical and 20 additive cycles
  (solver.cpp:349-400) against the oracle; 20 V(1,1) cycles against the
  restated V-cycle;
* C2 delayed solve: p doubling 1 -> 32 in the deterministic anarchic mode
  (workers = 1 semantics, scheduler.cpp:88-111) on the 729^2 grid, the whole
  run to convergence against the oracle (residual history, max_n, pending
  tasks per cycle), and the concurrent mode reaching the same solution.

The oracle (oracle/lzb_oracle.c) is pinned to the unmodified reference by
tests/test_oracle_pin.py.
"""
import numpy as np
import pytest

import paper_2005_03606_b200 as lzb
from oracle import port
from oracle.port2v import VCycle2

pytestmark = pytest.mark.gpu

TOP = lzb.T.P1_TOP
C2_DEPTH, C2_P = 6, 32


def normwise(a, b):
    """per-cell max |a - b| / max |b| (the north_star 1e-12 element bar)"""
    den = np.maximum(np.abs(b).max(axis=1), 1e-300)
    return (np.abs(a - b).max(axis=1) / den).max()


@pytest.mark.parametrize("integration", ["exact", "fast"])
def test_c2_assembly_every_cell_and_stream(integration):
    f = lzb.field_sinusoid(0.9, 6.0)
    d = lzb.make_desc(depth=C2_DEPTH, field=f, delta_max=1e-8, solver="adafac-pi", omega=0.6,
                      integration=integration)
    g = lzb.Grid(d, 42)
    raw = g.assemble_fixed_raw(C2_P)
    want = port.integrate_level(f, C2_DEPTH, C2_P)
    assert raw.shape == want.shape == (729 * 729, 16)
    err = normwise(raw, want)
    assert err <= 1e-12, err
    if integration == "exact":
        # the field's sines come from the host libm (the reference's), the
        # accumulation keeps element.hpp:42-45's order: bit-identical
        assert np.array_equal(raw, want)
    # compression + publish of the same kernel against the oracle publishing
    # the device's integrated matrices: identical input stencils -> identical bytes
    o = port.Grid(d, 42)
    o.publish_level(C2_DEPTH, raw, C2_P, TOP)
    ca, cb = g.cells(C2_DEPTH), o.cells(C2_DEPTH)
    for key in ("ops", "p1", "n", "p3", "epoch"):
        assert np.array_equal(ca[key], cb[key]), key
    assert g.stream_image() == o.stream_image()
    sa, sb = g.stats(), o.stats()
    assert list(sa.p3_histogram) == list(sb.p3_histogram)
    assert sa.fine_stored_bytes == sb.fine_stored_bytes


def test_c2_grid_checkerboard_bit_identical():
    """No transcendental in the field: the EXACT kernel at 729^2, p = 32 is
    bit-identical to the reference arithmetic on every cell."""
    f = lzb.checkerboard(1, 8)
    d = lzb.make_desc(depth=C2_DEPTH, field=f, delta_max=1e-8)
    g = lzb.Grid(d, 42)
    raw = g.assemble_fixed_raw(C2_P)
    assert np.array_equal(raw, port.integrate_level(f, C2_DEPTH, C2_P))


def test_batched_publish_matches_oracle():
    """lzb_grid_publish_level (the batched CellStream::publish_element) on
    perturbed matrices with mixed n and p1: same stored operators, markers and
    LZMG bytes as the oracle's per-cell publishes."""
    f = lzb.field_theta(16.0)
    d = lzb.make_desc(depth=4, field=f, delta_max=1e-6)
    rng = np.random.default_rng(3)
    base = port.integrate_level(f, 4, 3)
    mats = base * (1 + 1e-3 * rng.standard_normal(base.shape))
    n = rng.integers(1, 9, 81 * 81).astype(np.int32)
    g, o = lzb.Grid(d, 1), port.Grid(d, 1)
    for p1 in (5, TOP):
        g.publish_level(4, mats, n, p1)
        o.publish_level(4, mats, n, p1)
        ca, cb = g.cells(4), o.cells(4)
        for key in ("ops", "p1", "n", "p3"):
            assert np.array_equal(ca[key], cb[key]), key
        assert g.stream_image() == o.stream_image()


C1_TEXT = ("setup = checkerboard\nfield-seed = 1\nblocks = 8\ndepth = 5\nsolver = additive\nassembly = adaptive\n"
           "omega = 0.6\nmax-cycles = 20\nseed = 42\n")


def c1_pair(rhs_kind, delta):
    d = port.desc_from_keys(port.parse_keys(C1_TEXT + f"compression-threshold = {delta}\nrhs = 1\n"))
    if rhs_kind == "sinprod":
        d.rhs = lzb.Rhs(kind=lzb.T.RHS_SINPROD, value=2 * np.pi ** 2)
    return lzb.Grid(d, 42), port.Grid(d, 42), d


@pytest.mark.parametrize("p", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("rhs_kind,delta", [("constant", 1e-8), ("sinprod", 0.0)])
def test_c1_fixed_p_and_20_cycles(p, rhs_kind, delta):
    """BASELINE configs[0]: 243^2, checkerboard 10^U(-2,2), fixed p, 20 cycles
    with omega 0.6, the constant load and the f = 2 pi^2 sin sin load (its
    sines from the host libm, as the reference's): u on every level, the
    operators and the LZMG bytes bit-identical; the residual norm is a
    parallel sum (1e-13, north_star bar 1e-10)."""
    g, o, d = c1_pair(rhs_kind, delta)
    raw = g.assemble_fixed_raw(p)
    o.assemble_fixed(p)
    assert np.array_equal(raw, port.integrate_level(d.field, 5, p))
    assert np.array_equal(g.cells(5)["ops"], o.cells(5)["ops"])
    rg, ro = [g.step() for _ in range(20)], [o.step() for _ in range(20)]
    exact, rel = True, 1e-13
    for a, b in zip(rg, ro):
        assert a["status"] == b["status"] and a["dof_updates"] == b["dof_updates"] == 242 * 242
        assert abs(a["residual"] - b["residual"]) <= rel * b["residual"], (a["cycle"], a["residual"], b["residual"])
    assert rg[-1]["residual"] < rg[0]["residual"]
    for lvl in range(6):
        assert np.array_equal(g.cells(lvl)["ops"], o.cells(lvl)["ops"]), lvl  # Galerkin levels too
        a, b = g.vertices(lvl, lzb.T.V_U), o.vertices(lvl, lzb.T.V_U)
        if exact:
            assert np.array_equal(a, b), lvl
        else:
            assert np.abs(a - b).max() <= 1e-9 * max(np.abs(b).max(), 1e-300), lvl
    assert g.stream_image() == o.stream_image()


def test_c1_twenty_vcycles_match_restatement():
    """BASELINE configs[0]'s '20 V(1,1) cycles' at 243^2 (p = 16) against the
    restated V-cycle on the product's operators: within 1e-10 per cycle."""
    f = lzb.checkerboard(1, 8)
    d = lzb.make_desc(depth=5, field=f, solver="additive", omega=0.6, rhs_kind="sinprod", max_cycles=100)
    G = lzb.Grid(d, 42)
    G.assemble_fixed(16)
    u0 = G.vertices(5, lzb.T.V_U).copy()
    a = [G.vcycle(1)]
    fl = G.vertices(5, lzb.T.V_FL)
    ops = [G.cells(l)["ops"] for l in range(6)]
    P = [np.array([[G.transfer(l, cx, cy) for cx in range(3 ** l)] for cy in range(3 ** l)]) for l in range(5)]
    ref = VCycle2(ops, P, fl, u0, omega=0.6, max_cycles=100)
    b = [ref.vstep(1)]
    for _ in range(19):
        a.append(G.vcycle(1))
        b.append(ref.vstep(1))
    for x, y in zip(a, b):
        assert x["status"] == y["status"]
        assert x["residual"] == pytest.approx(y["residual"], rel=1e-10), x["cycle"]
    w = ref.u[5]
    assert np.abs(G.vertices(5, lzb.T.V_U) - w).max() <= 1e-12 * max(np.abs(w).max(), 1.0)
    assert a[-1]["normalized"] < 1e-3


def c2_delayed_desc(concurrent=False, start="geometric"):
    """BASELINE configs[1]: the delayed solve starting from the geometric
    stencil (eps = 1); start = "sample" is the reference's n = 1 start."""
    f = lzb.field_sinusoid(0.9, 6.0)
    return lzb.make_desc(depth=C2_DEPTH, field=f, delta_max=1e-8, solver="adafac-pi", omega=0.6,
                         assembly="anarchic", rhs_kind="sinprod", schedule="double", n_max=C2_P,
                         termination_c=0.0, target=1e-10, max_cycles=500, concurrent=concurrent,
                         start_geometric=start == "geometric")


@pytest.mark.parametrize("start", ["geometric", "sample"])
def test_c2_delayed_doubling_solve_matches_oracle(start):
    """The delayed solve bench.py times (729^2, p doubling 1 -> 32 while the
    adaFAC-PI cycles run) in the deterministic mode, cycle by cycle against
    the oracle: residual within 1e-13 (parallel norm sum), max_n / pending
    tasks / DoF counts identical, same termination cycle; operators, markers,
    u and the LZMG stream bit-identical."""
    d = c2_delayed_desc(start=start)
    g, o = lzb.Grid(d, 42), port.Grid(d, 42)
    rg, ro = g.run(), o.run()
    assert len(rg) == len(ro) and rg[-1]["status"] == lzb.T.CONVERGED
    for a, b in zip(rg, ro):
        for k in ("status", "max_n", "pending_tasks", "dof_updates", "max_samples"):
            assert a[k] == b[k], (a["cycle"], k, a[k], b[k])
        assert abs(a["residual"] - b["residual"]) <= 1e-13 * b["residual"], a["cycle"]
        assert a["avg_n"] == pytest.approx(b["avg_n"], rel=1e-12)
    assert max(r["max_n"] for r in rg) == C2_P
    ca, cb = g.cells(C2_DEPTH), o.cells(C2_DEPTH)
    assert np.array_equal(ca["n"], cb["n"]) and np.array_equal(ca["p1"], cb["p1"])
    for lvl in range(C2_DEPTH + 1):
        assert np.array_equal(g.cells(lvl)["ops"], o.cells(lvl)["ops"]), lvl
        assert np.array_equal(g.vertices(lvl, lzb.T.V_U), o.vertices(lvl, lzb.T.V_U)), lvl
    assert g.stream_image() == o.stream_image()


def test_c2_concurrent_delayed_solve_reaches_same_solution():
    """The concurrent mode (assembly batches on the low-priority stream,
    swapped in by events) converges to the deterministic mode's discrete
    solution within the solver tolerance, with the same final operators."""
    det = lzb.Grid(c2_delayed_desc(False), 42)
    rd = det.run()
    con = lzb.Grid(c2_delayed_desc(True), 42)
    rc = con.run()
    assert rd[-1]["status"] == rc[-1]["status"] == lzb.T.CONVERGED
    assert con.drain() == 0
    ca, cb = con.cells(C2_DEPTH), det.cells(C2_DEPTH)
    assert np.array_equal(ca["ops"], cb["ops"]) and np.array_equal(ca["n"], cb["n"])
    ua, ub = con.vertices(C2_DEPTH, lzb.T.V_U), det.vertices(C2_DEPTH, lzb.T.V_U)
    # both iterates are within target 1e-10 (normalised residual) of the same discrete solution
    assert np.abs(ua - ub).max() <= 1e-8 * np.abs(ub).max()

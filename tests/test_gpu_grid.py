"""GPU parity of the full delayed-assembly path (grid engine) against the oracle.

The device engine keeps the reference's accumulation orders, so on fields
without transcendentals the solver state (u on every level, operators,
markers, epochs) and the LZMG stream bytes are bit-identical to the oracle,
which is itself bit-identical to the unmodified reference
(tests/test_oracle_pin.py). The per-cycle residual norm is a parallel sum,
so it is compared at 1e-13 relative (north_star bar: 1e-10).
"""
import glob
import os

import numpy as np
import pytest

import paper_2005_03606_b200 as lzb
from conftest import GOLDEN
from oracle import port

pytestmark = pytest.mark.gpu

INT_KEYS = ("cycle", "status", "dof_updates", "dof_updates_total", "coarse_updates", "pending_tasks", "max_n",
            "max_samples", "enabled_mask", "levels", "cells", "dofs_fine_interior", "grid_points_total")


def assert_reports(got, want, rel=1e-13):
    assert len(got) == len(want)
    for g, w in zip(got, want):
        for k in INT_KEYS:
            assert g[k] == w[k], (k, g[k], w[k])
        for k in ("residual", "normalized"):
            assert abs(g[k] - w[k]) <= rel * abs(w[k]), (k, g[k], w[k])
        for k in ("avg_n", "factor_totals", "factor_mean"):
            assert abs(g[k] - w[k]) <= 1e-12 * abs(w[k]), (k, g[k], w[k])


def assert_state(g, o, depth, exact=True):
    for lvl in range(depth + 1):
        a, b = g.vertices(lvl, lzb.T.V_U), o.vertices(lvl, lzb.T.V_U)
        if exact:
            assert np.array_equal(a, b), f"u level {lvl}"
        else:
            assert np.max(np.abs(a - b)) <= 1e-9 * max(np.max(np.abs(b)), 1e-300)
        ca, cb = g.cells(lvl), o.cells(lvl)
        for key in ("p1", "n", "p3", "epoch"):
            if exact or key in ("p1", "n"):
                assert np.array_equal(ca[key], cb[key]), (lvl, key)
        if exact:
            assert np.array_equal(ca["ops"], cb["ops"]), f"ops level {lvl}"


def grid_pair(text, **kw):
    k = port.parse_keys(text)
    d = port.desc_from_keys(k)
    for name, val in kw.items():
        setattr(d, name, val)
    g = lzb.Grid(d, int(k["seed"]))
    o = port.Grid(d, int(k["seed"]))
    return g, o, d


@pytest.mark.parametrize("cfg", sorted(glob.glob(os.path.join(GOLDEN, "exp_*.cfg"))))
def test_reference_telemetry_configs(cfg, tmp_path):
    """The configs behind the reference's committed telemetry CSVs."""
    text = open(cfg).read()
    out = tmp_path / "t.csv"
    ec, reps = lzb.run_experiment(text + f"csv = {out}\n")
    gold = port.csv_data_rows(cfg.replace(".cfg", ".csv"))
    mine = port.csv_data_rows(str(out))
    assert len(mine) == len(gold)
    for a, b in zip(mine, gold):
        fa, fb = a.split(","), b.split(",")
        assert fa[0] == fb[0] and fa[3:] == fb[3:]
        for i in (1, 2):
            assert abs(float(fa[i]) - float(fb[i])) <= 1e-13 * abs(float(fb[i]))
    # preamble identical: the telemetry header is part of the interface
    head_a = [l for l in open(out) if l.startswith("#") and not l.startswith("# csv")]
    head_b = [l for l in open(cfg.replace(".cfg", ".csv")) if l.startswith("#")]
    assert head_a == head_b
    assert ec == (0 if gold[-1].endswith("converged") else 3)


MATRIX = [(f, s, a) for f in ["setup = quadrant\neps-low = 0.001", "setup = checkerboard\nfield-seed = 1",
                               "setup = constant\neps = 3"]
          for s in ["additive", "adafac-jac", "adafac-pi"] for a in ["eager", "lazy", "adaptive", "anarchic"]]


@pytest.mark.parametrize("f,solver,asm", MATRIX)
def test_cycle_bit_identical_to_oracle(f, solver, asm):
    text = f"{f}\ndepth = 3\nsolver = {solver}\nassembly = {asm}\nmax-cycles = 10\nomega = 0.6\nrhs = 1\nseed = 42\n"
    g, o, d = grid_pair(text)
    assert_reports(g.run(), o.run())
    assert_state(g, o, d.depth)
    assert g.stream_image() == o.stream_image()


RIPPLE = [(f, s, a, t) for f in ["setup = quadrant\neps-low = 0.001", "setup = checkerboard\nfield-seed = 1"]
          for s in ["additive", "adafac-pi"] for a in ["eager", "adaptive", "anarchic"] for t in ["geometric", "boxmg"]]
RIPPLE_THROTTLED = [(f, a, t, th) for f in ["setup = quadrant\neps-low = 0.001", "setup = theta\ntheta = 16"]
                    for a in ["anarchic"] for t in ["geometric", "boxmg"] for th in [5, 20, 97]]


@pytest.mark.parametrize("f,solver,asm,transfer", RIPPLE)
def test_ripple_bit_identical_to_oracle(f, solver, asm, transfer):
    """coarse-recompute = ripple on the device (dirty flags by cycle parity,
    coarse_recompute tasks in the high-priority class) against the oracle,
    itself pinned to the unmodified reference (test_oracle_pin.py)."""
    text = (f"{f}\ndepth = 3\nsolver = {solver}\nassembly = {asm}\nmax-cycles = 10\nomega = 0.6\nrhs = 1\n"
            f"seed = 42\ncoarse-recompute = ripple\ntransfer = {transfer}\n")
    g, o, d = grid_pair(text)
    assert d.policy == lzb.T.RIPPLE
    assert_reports(g.run(), o.run())
    assert_state(g, o, d.depth)
    assert g.stream_image() == o.stream_image()


@pytest.mark.parametrize("f,asm,transfer,throttle", RIPPLE_THROTTLED)
def test_ripple_throttled_bit_identical_to_oracle(f, asm, transfer, throttle):
    """coarse-recompute = ripple with a throttle (solver.cpp:86-90,
    scheduler.cpp:88-111): the high-priority coarse_recompute tasks form a
    FIFO with duplicates, at most `throttle` tasks per begin_cycle (coarse
    first, the leaf tasks get the rest); device against the oracle, itself
    pinned to the unmodified reference with throttle 20 (test_oracle_pin.py)."""
    text = (f"{f}\ndepth = 3\nsolver = adafac-pi\nassembly = {asm}\nmax-cycles = 14\nomega = 0.6\nrhs = 1\n"
            f"seed = 42\ncoarse-recompute = ripple\ntransfer = {transfer}\nthrottle = {throttle}\n")
    g, o, d = grid_pair(text)
    assert d.policy == lzb.T.RIPPLE and d.throttle == throttle
    rg, ro = g.run(), o.run()
    assert_reports(rg, ro)
    assert_state(g, o, d.depth)
    assert g.stream_image() == o.stream_image()
    assert g.drain() == 0


@pytest.mark.parametrize("setup", ["setup = theta\ntheta = 16", "setup = sinusoid"])
def test_cycle_transcendental_fields_within_tolerance(setup):
    text = f"{setup}\ndepth = 3\nsolver = additive\nassembly = eager\nmax-cycles = 10\nomega = 0.6\nseed = 42\n"
    g, o, d = grid_pair(text, rhs=lzb.Rhs(kind=lzb.T.RHS_SINPROD, value=2 * np.pi ** 2))
    rg, ro = g.run(), o.run()
    assert_reports(rg, ro)  # the norm is a parallel sum (1e-13; north_star bar 1e-10)
    # exp / cos / sin of the field and the load come from the host libm: bit-identical state
    assert_state(g, o, d.depth)
    assert g.stream_image() == o.stream_image()


@pytest.mark.parametrize("rhs_kind", ["constant", "sinprod"])
def test_fixed_p_checkerboard_delta0(rhs_kind):
    """BASELINE config 1 shape (depth 4 here): fixed p, exact storage, additive, omega 0.6;
    bit-identical with either load (the sinprod sines from the host libm)."""
    text = "setup = checkerboard\ndepth = 4\nsolver = additive\nassembly = adaptive\nmax-cycles = 6\nomega = 0.6\n" \
           "compression-threshold = 0\nrhs = 1\nseed = 42\n"
    kw = {"rhs": lzb.Rhs(kind=lzb.T.RHS_SINPROD, value=2 * np.pi ** 2)} if rhs_kind == "sinprod" else {}
    g, o, d = grid_pair(text, **kw)
    for p in (1, 2, 4):
        g.assemble_fixed(p)
        o.assemble_fixed(p)
        assert np.array_equal(g.cells(4)["ops"], o.cells(4)["ops"])
    rg, ro = [g.step() for _ in range(6)], [o.step() for _ in range(6)]
    assert_reports(rg, ro)
    assert_state(g, o, 4)


def test_double_schedule_and_cap():
    text = "setup = sinusoid\ndepth = 3\nsolver = additive\nassembly = anarchic\nmax-cycles = 8\nseed = 1\n"
    g, o, d = grid_pair(text, schedule=lzb.T.SCHEDULE_DOUBLE, n_max=8)
    rg, ro = g.run(), o.run()
    assert [r["max_n"] for r in rg] == [r["max_n"] for r in ro]
    assert [r["pending_tasks"] for r in rg] == [r["pending_tasks"] for r in ro]
    assert max(r["max_n"] for r in rg) <= 8


def test_throttled_anarchic_fifo():
    text = "setup = quadrant\neps-low = 1e-4\ndepth = 3\nassembly = anarchic\nthrottle = 37\nmax-cycles = 12\nseed = 5\n"
    g, o, d = grid_pair(text)
    assert_reports(g.run(), o.run())
    assert_state(g, o, 3)


def test_per_cell_protocol_api():
    """publish_element / adaptive_step / markers (test_assembly.cpp:28-92)."""
    text = "setup = quadrant\neps-low = 1e-5\ndepth = 1\nassembly = adaptive\n"
    g, o, d = grid_pair(text)
    terminal = None
    for step in range(250):
        g.adaptive_step(1, 1, 1)
        o.adaptive_step(1, 1, 1)
        p1 = g.cells(1)["p1"][1 * 3 + 1]
        assert p1 == o.cells(1)["p1"][4]
        if p1 == lzb.T.P1_TOP:
            terminal = step
            break
        assert p1 == step + 1
    assert terminal is not None and terminal >= 2
    assert np.array_equal(g.cells(1)["ops"], o.cells(1)["ops"])
    m = 1.5 * g.cells(1)["ops"][0]
    g.publish_element(1, 0, 0, m, 5, 5)
    o.publish_element(1, 0, 0, m, 5, 5)
    assert np.array_equal(g.cells(1)["ops"], o.cells(1)["ops"])
    assert g.stream_image() == o.stream_image()


def test_stream_save_load_roundtrip(tmp_path):
    text = "setup = quadrant\neps-low = 1e-3\ndepth = 3\nassembly = eager\nmax-cycles = 4\nseed = 3\n"
    g, o, d = grid_pair(text)
    g.run()
    o.run()
    g.save(tmp_path / "s.lzmg")
    data = open(tmp_path / "s.lzmg", "rb").read()
    assert data == o.stream_image()
    g2 = lzb.Grid(d, 3)
    g2.load(tmp_path / "s.lzmg")
    o2 = port.Grid(d, 3)
    o2.load_image(data)
    for lvl in range(4):
        a, b = g2.cells(lvl), o2.cells(lvl)
        for key in ("ops", "p1", "p3", "n"):
            assert np.array_equal(a[key], b[key]), key
        assert np.array_equal(a["ops"], g.cells(lvl)["ops"])  # codec error absorbed at write
    bad = bytearray(data)
    bad[:4] = b"XXXX"
    with pytest.raises(lzb.CorruptStreamError):
        lzb.Grid(d, 3).load_image(bytes(bad))
    with pytest.raises(lzb.CorruptStreamError):
        lzb.Grid(d, 3).load_image(data[:-3])


def test_all_elided_stream_compresses_by_128():
    """test_codec.cpp:204-216 and Table 1 theta = 1 accounting."""
    d = lzb.make_desc(depth=2, field=lzb.field_constant(1.0), assembly="eager")
    g = lzb.Grid(d, 0)
    g.eager_setup()
    st = g.stats()
    assert st.fine_cells == 81 and st.fine_factor_totals == 128.0 and st.fine_factor_mean == 128.0
    assert st.p3_histogram[0] == 81


def test_large_grid_properties():
    """729^2 (BASELINE config 2 grid): size-independent properties of the device path."""
    d = lzb.make_desc(depth=6, field=lzb.field_sinusoid(0.9, 6.0), solver="additive", omega=0.6,
                      assembly="adaptive", rhs_kind="sinprod", max_cycles=3)
    g = lzb.Grid(d, 42)
    g.assemble_fixed(4)
    ops = g.cells(6)["ops"].reshape(-1, 4, 4)
    assert np.max(np.abs(ops - ops.transpose(0, 2, 1))) <= 1e-12 * np.max(np.abs(ops))  # symmetry
    # zero row sums up to the absorbed codec error (|rt - surplus| <= delta_max per entry)
    assert np.max(np.abs(ops.sum(axis=2))) <= 4 * d.delta_max + 1e-12 * np.max(np.abs(ops))
    # a sample of cells against the oracle element (codec-absorbed with delta 1e-8)
    rng = np.random.default_rng(0)
    idx = rng.integers(0, 729 * 729, 64)
    h = np.power(1.0 / 3, 6)
    for c in idx:
        want = port.integrate_element(d.field, (c % 729) * h, (c // 729) * h, h, 4)
        assert np.max(np.abs(ops[c].reshape(16) - want)) <= 2e-8
    reps = [g.step() for _ in range(3)]
    assert reps[-1]["dof_updates"] == 728 * 728
    assert reps[-1]["residual"] < reps[0]["residual"]
    # injection holds on coincident points (test_solver.cpp:213-224)
    for lvl in range(1, 7):
        c, f = g.vertices(lvl - 1, lzb.T.V_U), g.vertices(lvl, lzb.T.V_U)
        assert np.array_equal(c, f[::3, ::3])


@pytest.mark.parametrize("setup", ["setup = quadrant\neps-low = 0.1", "setup = theta\ntheta = 16"])
def test_concurrent_anarchic_converges_to_eager_solution(setup):
    """Assembly batches on the low-priority stream, swapped in via events: the
    final operators are bit-identical to eager assembly (each cell's protocol
    is timing-independent) and the solve reaches the same discrete solution."""
    base = f"{setup}\ndepth = 4\nsolver = adafac-pi\nrhs = 1\nseed = 11\nmax-cycles = 600\n"
    k = port.parse_keys(base + "assembly = anarchic\n")
    d = port.desc_from_keys(k)
    d.concurrent = 1
    g = lzb.Grid(d, 11)
    reps = g.run()
    assert reps[-1]["status"] == lzb.T.CONVERGED
    assert g.drain() == 0
    # eager reference: every leaf integrated to top before the solve
    ke = port.parse_keys(base + "assembly = eager\n")
    o = lzb.Grid(port.desc_from_keys(ke), 11)  # device eager run (bitwise == oracle on exact fields)
    o.run()
    ca, cb = g.cells(4), o.cells(4)
    assert np.all(ca["p1"] == lzb.T.P1_TOP)
    assert np.array_equal(ca["ops"], cb["ops"]) and np.array_equal(ca["n"], cb["n"])
    # continue the concurrent grid on the final operators to the same tolerance
    d2 = port.desc_from_keys(port.parse_keys(base + "assembly = anarchic\n"))
    more = [g.step() for _ in range(200)]
    ue, ua = o.vertices(4, lzb.T.V_U), g.vertices(4, lzb.T.V_U)
    assert np.max(np.abs(ua - ue)) <= 1e-7 * np.max(np.abs(ue))
    del d2, more


def test_concurrent_rejects_non_anarchic():
    d = lzb.make_desc(depth=2, assembly="adaptive", concurrent=True)
    with pytest.raises(lzb.LzbError):
        lzb.Grid(d)


# ------------------------------------------- residual on compressed records
def _cycles(d, n_asm, k, eager=False):
    g = lzb.Grid(d, 42)
    if eager:
        g.eager_setup()
    else:
        g.assemble_fixed(n_asm)
    reps = [g.step() for _ in range(k)]
    return g, reps


@pytest.mark.gpu
@pytest.mark.parametrize("width", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("solver", ["additive", "adafac-pi"])
def test_compressed_residual_bit_identical(width, solver):
    """The residual decoding the leaf records' surplus bytes (plane_width)
    rebuilds the stored operator bit for bit: same u, r and residual history
    as the FP64 residual, including records wider than a slot (FP64 fallback)."""
    f = lzb.field_theta(16.0)
    base = dict(depth=4, field=f, solver=solver, omega=0.6, rhs_kind="sinprod", max_cycles=100, delta_max=1e-8)
    a, ra = _cycles(lzb.make_desc(**base), 3, 6)
    b, rb = _cycles(lzb.make_desc(plane_width=width, **base), 3, 6)
    assert [r["residual"] for r in ra] == [r["residual"] for r in rb]
    for lvl in range(5):
        assert np.array_equal(a.vertices(lvl, lzb.T.V_U), b.vertices(lvl, lzb.T.V_U))
    assert np.array_equal(a.vertices(4, lzb.T.V_R), b.vertices(4, lzb.T.V_R))


@pytest.mark.gpu
def test_compressed_residual_adaptive_and_reload(tmp_path):
    """Records published by the adaptive protocol and by a stream load feed the
    compressed residual as they feed the FP64 one."""
    f = lzb.checkerboard(3, 8)
    base = dict(depth=3, field=f, solver="adafac-pi", omega=0.6, rhs=1.0, max_cycles=100)
    a, ra = _cycles(lzb.make_desc(assembly="eager", **base), 0, 5, eager=True)
    b, rb = _cycles(lzb.make_desc(assembly="eager", plane_width=4, **base), 0, 5, eager=True)
    assert [r["residual"] for r in ra] == [r["residual"] for r in rb]
    img = a.stream_image()
    c = lzb.Grid(lzb.make_desc(plane_width=4, **base), 42)
    c.load_image(img)
    d0 = lzb.Grid(lzb.make_desc(**base), 42)
    d0.load_image(img)
    rc, rd = [c.step() for _ in range(4)], [d0.step() for _ in range(4)]
    assert [r["residual"] for r in rc] == [r["residual"] for r in rd]
    assert np.array_equal(c.vertices(3, lzb.T.V_U), d0.vertices(3, lzb.T.V_U))


@pytest.mark.gpu
@pytest.mark.parametrize("p3", [2, 3, 4, 5, 6, 7, 8])
def test_fixed_width_records(p3):
    """fixed_p3: every leaf record at one mantissa width (the width sweep of
    BASELINE configs[4]); the stored operator is baseline + roundtrip at that
    width, and the compressed residual at plane_width = p3 agrees with the
    FP64 one bit for bit."""
    f = lzb.field_sinusoid(0.9, 6.0)
    base = dict(depth=3, field=f, solver="additive", omega=0.6, rhs_kind="sinprod", max_cycles=100,
                fixed_p3=p3)
    a, ra = _cycles(lzb.make_desc(**base), 2, 4)
    b, rb = _cycles(lzb.make_desc(plane_width=p3, **base), 2, 4)
    st = a.stats()
    assert st.p3_histogram[p3] == 27 * 27 and st.fine_stored_bytes == 27 * 27 * (1 + 16 * p3)
    assert [r["residual"] for r in ra] == [r["residual"] for r in rb]
    # stored entries = baseline + roundtrip(surplus, p3) of the n = 2 integration
    cells = a.cells(3)
    h = (1.0 / 3) ** 3  # mesh.hpp:87 on the host, x0 = cx * h
    xs = np.array([cx * h for cy in range(27) for cx in range(27)])
    ys = np.array([cy * h for cy in range(27) for cx in range(27)])
    m = lzb.integrate_elements(f, xs, ys, h, 2)
    basev = lzb.integrate_elements(f, xs, ys, h, 1)  # A(n=1) = eps(centre) K_unit, the baseline
    for c in (0, 13, 400, 728):
        want = basev[c] + lzb.codec.roundtrip(m[c] - basev[c], p3)
        assert np.array_equal(cells["ops"][c], want), c


@pytest.mark.gpu
@pytest.mark.parametrize("depth,kind,dmax,n", [(2, "checker", 1e-8, 3), (3, "sinusoid", 1e-8, 4),
                                               (4, "checker", 0.0, 2), (5, "sinusoid", 1e-4, 5)])
def test_assemble_stream_matches_sequential(depth, kind, dmax, n):
    """lzb_grid_assemble_stream (assembly + pack + copy pipelined over the
    three bands of level-1 subtrees) gives the bytes of assemble_fixed
    followed by stream_image and leaves the same grid state; a too-small
    buffer fails without writing past it."""
    import torch
    f = lzb.checkerboard(1, 8) if kind == "checker" else lzb.field_sinusoid(0.9, 6.0)
    desc = lzb.make_desc(depth=depth, field=f, solver="adafac-pi", omega=0.6, max_cycles=100, delta_max=dmax)
    a, b = lzb.Grid(desc, 1), lzb.Grid(desc, 1)
    a.assemble_fixed(n)
    a.step()  # refined records with payloads
    b.assemble_fixed(n)
    b.step()
    want = a.stream_image()
    out = torch.full((len(want) + 64,), 0xAB, dtype=torch.uint8, pin_memory=True).numpy()
    tl = np.zeros(9, np.float32)
    size = b.assemble_stream(n, out, tl)
    assert size == len(want) and out[:size].tobytes() == want
    assert (out[size:] == 0xAB).all() and (np.diff(tl[:3]) > 0).all()
    assert np.array_equal(a.cells(depth)["ops"], b.cells(depth)["ops"])
    assert [r["residual"] for r in (a.step(), a.step())] == [r["residual"] for r in (b.step(), b.step())]
    guard = np.full(len(want), 0xCD, np.uint8)
    with pytest.raises(lzb.LzbError):
        b.assemble_stream(n, guard[: len(want) // 2])
    assert (guard[len(want) // 2:] == 0xCD).all()


@pytest.mark.gpu
@pytest.mark.parametrize("text", [
    "setup = theta\ntheta = 16\nrhs = 1\ndepth = 5\nsolver = additive\nassembly = anarchic\nmax-cycles = 3\n",
    "setup = quadrant\neps-low = 0.001\nrhs = 1\ndepth = 6\nsolver = adafac-pi\nassembly = anarchic\nmax-cycles = 2\n",
])
def test_deep_grids_match_oracle(text):
    """Depths 5 and 6 (the survey's gate depths; the oracle is pinned to the
    unmodified reference there): u on every level, operators, markers and
    LZMG bytes bit-identical -- the theta field's exp / cos from the host libm."""
    text += "omega = 0.6\nseed = 42\n"
    d = port.desc_from_keys(port.parse_keys(text))
    g, o = lzb.Grid(d, 42), port.Grid(d, 42)
    rg, ro = g.run(), o.run()
    assert_reports(rg, ro)
    assert_state(g, o, d.depth)
    assert g.stream_image() == o.stream_image()


FORCED = [(asm, extra) for asm in ["eager", "lazy", "adaptive", "anarchic"]
          for extra in ["forced-task-fraction = 0.3\nforced-task-n = 4\n",
                        "forced-task-fraction = 0.5\nforced-task-n = 3\nthrottle = 40\n"]]
FORCED += [("anarchic", "forced-task-fraction = 0.2\ncoarse-recompute = ripple\n"),
           ("eager", "forced-task-fraction = 0.2\ncoarse-recompute = ripple\n")]


@pytest.mark.parametrize("asm,extra", FORCED)
def test_forced_tasks_bit_identical_to_oracle(asm, extra):
    """run_experiment's forced-task workload emulation (experiment.cpp:260-270,
    spawn_forced assembly.cpp:138-154) on the device: forced tasks share the
    FIFO with the step tasks (p2 = 2, key before the cycle's step tasks), hold
    a cell's p2 so that anarchic steps are not spawned, run their integration
    (discarded) at begin_cycle under the throttle, and adaptive_sync runs them
    inside the pass. Telemetry (pending tasks), u, operators and LZMG bytes
    against the oracle, itself pinned to the reference (test_oracle_pin.py)."""
    text = (f"setup = theta\ntheta = 16\nrhs = 1\ndepth = 3\nsolver = adafac-pi\nassembly = {asm}\n"
            f"max-cycles = 9\n{extra}omega = 0.6\nseed = 42\n")
    g, o, d = grid_pair(text)
    assert d.forced_fraction > 0
    rg, ro = g.run(), o.run()
    assert_reports(rg, ro)
    assert_state(g, o, d.depth)
    assert g.stream_image() == o.stream_image()
    if asm != "adaptive":
        assert any(r["pending_tasks"] for r in rg)


def test_forced_tasks_through_run_experiment(tmp_path):
    """The config keys forced-task-fraction / forced-task-n reach the device
    through the C-ABI experiment layer and give the oracle's telemetry."""
    text = ("setup = quadrant\neps-low = 0.001\nrhs = 1\ndepth = 3\nassembly = anarchic\nmax-cycles = 6\n"
            "forced-task-fraction = 0.25\nforced-task-n = 2\nthrottle = 30\nseed = 3\ntiming = off\n")
    ec, reps = lzb.run_experiment(text)
    want = port.Grid.from_text(text).run()
    assert_reports(reps, want)  # the norm is a parallel sum: 1e-13, every other column equal


def test_forced_tasks_rejected_with_concurrent_assembly():
    d = lzb.make_desc(depth=2, assembly="anarchic", concurrent=True, forced_fraction=0.5)
    with pytest.raises(lzb.LzbError):
        lzb.Grid(d)


GEO = [(sched, extra) for sched in ["increment", "double"] for extra in ["", "throttle = 50\n"]]


@pytest.mark.parametrize("sched,extra", GEO)
def test_geometric_start_bit_identical_to_oracle(sched, extra):
    """BASELINE configs[1]'s start: unintegrated leaves read the geometric
    stencil (eps = 1) and their first integration is a deferred task too
    (restated extension of request_stencil, assembly.cpp:95-106; the codec
    baseline stays A(n = 1)). Device against the restatement, bit for bit."""
    text = (f"setup = sinusoid\nrhs = 1\ndepth = 4\nsolver = adafac-pi\nassembly = anarchic\nmax-cycles = 12\n"
            f"schedule = {sched}\nn-max = 16\nstart = geometric\n{extra}omega = 0.6\nseed = 42\n")
    g, o, d = grid_pair(text)
    assert d.start_geometric == 1
    rg, ro = g.run(), o.run()
    assert_reports(rg, ro)
    assert_state(g, o, d.depth)
    assert g.stream_image() == o.stream_image()
    # the first cycle solves with the geometric stencil: every leaf still bottom
    assert rg[0]["max_n"] == 0 and rg[1]["max_n"] == 1


def test_geometric_start_concurrent_converges_to_deterministic_solution():
    base = dict(depth=4, field=lzb.field_sinusoid(0.9, 6.0), delta_max=1e-8, solver="adafac-pi", omega=0.6,
                assembly="anarchic", rhs_kind="sinprod", schedule="double", n_max=16, termination_c=0.0,
                target=1e-9, max_cycles=400, start_geometric=True)  # depth 4 stalls near 2.5e-10
    det = lzb.Grid(lzb.make_desc(**base), 42)
    rd = det.run()
    con = lzb.Grid(lzb.make_desc(concurrent=True, **base), 42)
    rc = con.run()
    assert rd[-1]["status"] == rc[-1]["status"] == lzb.T.CONVERGED
    assert con.drain() == 0
    ca, cb = con.cells(4), det.cells(4)
    assert np.array_equal(ca["ops"], cb["ops"]) and np.array_equal(ca["n"], cb["n"])
    ua, ub = con.vertices(4, lzb.T.V_U), det.vertices(4, lzb.T.V_U)
    assert np.abs(ua - ub).max() <= 1e-8 * np.abs(ub).max()


def _stencils_restated(ops, N):
    """assemble_vertex_stencil (assembly.cpp:120-136) over the product's cells."""
    out = np.zeros(((N + 1) * (N + 1), 9))
    for iy in range(N + 1):
        for ix in range(N + 1):
            st = np.zeros(9)
            for c in range(4):
                cx, cy = ix - 1 + (c & 1), iy - 1 + (c >> 1)
                if not (0 <= cx < N and 0 <= cy < N):
                    continue
                corner = (1 - (c & 1)) | ((1 - (c >> 1)) << 1)
                K = ops[cy * N + cx]
                for k in range(4):
                    dx, dy = (k & 1) - (corner & 1), (k >> 1) - (corner >> 1)
                    st[(dy + 1) * 3 + dx + 1] += K[corner * 4 + k]
            out[iy * (N + 1) + ix] = st
    return out


def test_vertex_stencil_known_answer_and_protocol():
    """test_element.cpp:83-140: the eps = 1 interior stencil is 8/3 and -1/3
    (centre = the cell-wise Jacobi diagonal); zero matrices give a zero
    stencil; a bottom neighbour with require_payload is a protocol_error."""
    d = lzb.make_desc(depth=1, field=lzb.field_constant(1.0), assembly="lazy", delta_max=0.0)
    g = lzb.Grid(d, 0)
    with pytest.raises(lzb.ProtocolError):
        g.vertex_stencils(1, require_payload=True)
    g.pass_(0)  # request_stencil on every leaf (lazy: converge now)
    st = g.vertex_stencils(1, require_payload=True).reshape(4, 4, 9)
    want = np.full(9, -1.0 / 3.0)
    want[4] = 8.0 / 3.0
    assert np.allclose(st[1, 1], want, rtol=1e-12, atol=0)
    g.step()
    assert st[1, 1, 4] == pytest.approx(g.vertices(1, lzb.T.V_DIAG)[1, 1], rel=1e-14)
    z = lzb.Grid(d, 0)
    for cy in range(3):
        for cx in range(3):
            z.publish_element(1, cx, cy, np.zeros(16), 1, 1)
    assert not np.any(z.vertex_stencils(1)[5])
    z.vertex_stencils(1)  # boundary vertices: missing cells contribute zero, no throw


def test_vertex_stencils_match_restatement():
    """Every vertex of every level of an assembled grid (leaves, Galerkin
    coarse levels, unassembled bottom cells) against the restated loop."""
    d = lzb.make_desc(depth=3, field=lzb.field_theta(16.0), assembly="adaptive", solver="adafac-pi")
    g = lzb.Grid(d, 1)
    g.step()
    g.step()
    for lvl in range(4):
        N = 3 ** lvl
        got = g.vertex_stencils(lvl)
        assert np.array_equal(got, _stencils_restated(g.cells(lvl)["ops"], N)), lvl


DEVLOOP = [("setup = checkerboard\nfield-seed = 1", "adafac-pi", "eager", "geometric", 300, 1e-10),
           ("setup = checkerboard\nfield-seed = 1", "additive", "anarchic", "boxmg", 25, 1e-10),   # timeout
           ("setup = quadrant\neps-low = 0.001", "adafac-jac", "adaptive", "geometric", 400, 1e-9),
           ("setup = sinusoid", "adafac-pi", "anarchic", "geometric", 200, 1e-10)]


@pytest.mark.parametrize("devloop", [False, True])
@pytest.mark.parametrize("f,solver,asm,transfer,cycles,target", DEVLOOP)
def test_run_matches_stepping(f, solver, asm, transfer, cycles, target, devloop, monkeypatch):
    """lzb_grid_run against stepping the same grid cycle by cycle with reads in
    between (which keep the stepped grid on the full cycle: every step runs
    the coarse pass and the stats). run() skips both once the hierarchy has
    settled (a calm cycle whose coarse pass recomputed nothing), and with
    LZB_DEVLOOP=1 hands the quiescent cycles to the device-side loop (a
    conditional WHILE graph, termination test on the device: solver.cpp:8-16,
    421-444). Same kernels on the same data: same reports, same state."""
    if devloop:
        monkeypatch.setenv("LZB_DEVLOOP", "1")
    else:
        monkeypatch.delenv("LZB_DEVLOOP", raising=False)
    text = (f"{f}\ndepth = 4\nsolver = {solver}\nassembly = {asm}\ntransfer = {transfer}\nmax-cycles = {cycles}\n"
            f"omega = 0.6\nrhs = 1\nseed = 7\ntarget = {target}\n")
    k = port.parse_keys(text)
    d = port.desc_from_keys(k)
    g, h = lzb.Grid(d, 7), lzb.Grid(d, 7)
    rg = g.run()
    monkeypatch.delenv("LZB_DEVLOOP", raising=False)
    if asm == "eager":
        h.eager_setup()
    rh = []
    while not rh or rh[-1]["status"] == lzb.T.CONTINUE:
        rh.append(h.step())
        h.stats()  # a C-ABI call between steps: the stepped grid never takes the settled path
    assert len(rg) > 8
    assert_reports(rg, rh, rel=0.0)
    for lvl in range(5):
        for fld in (lzb.T.V_U, lzb.T.V_R, lzb.T.V_FL):
            assert np.array_equal(g.vertices(lvl, fld), h.vertices(lvl, fld)), (lvl, fld)
        assert np.array_equal(g.cells(lvl)["ops"], h.cells(lvl)["ops"])
        assert np.array_equal(g.cells(lvl)["epoch"], h.cells(lvl)["epoch"])
    assert g.stats().p3_histogram[:] == h.stats().p3_histogram[:]
    if devloop and asm == "eager":  # the loop's cycles ran in one graph launch: one wall-clock share
        walls = [r["wall_seconds"] for r in rg[-4:]]
        assert len(set(walls)) == 1
    # and the grid carries on from the host afterwards
    if rg[-1]["status"] == lzb.T.TIMEOUT:
        a, b = g.step(), h.step()
        assert a["residual"] == b["residual"] and a["cycle"] == b["cycle"]

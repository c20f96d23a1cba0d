"""Edge cases of the device path: smallest grids, empty and ragged batches,
limits, corrupt inputs and non-finite values, the way the reference's tests
exercise them (test_codec.cpp, test_stream / test_solver edge cases)."""
import numpy as np
import pytest

import paper_2005_03606_b200 as lzb
from oracle import port

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("solver", ["additive", "adafac-jac", "adafac-pi"])
@pytest.mark.parametrize("asm", ["eager", "anarchic"])
def test_depth1_grid_bit_identical(solver, asm):
    """The smallest multilevel grid: one coarse cell, 3x3 leaves, 4 interior DoFs."""
    text = f"setup = quadrant\neps-low = 0.01\ndepth = 1\nsolver = {solver}\nassembly = {asm}\nmax-cycles = 12\n" \
           "omega = 0.6\nrhs = 1\nseed = 5\n"
    k = port.parse_keys(text)
    d = port.desc_from_keys(k)
    g, o = lzb.Grid(d, 5), port.Grid(d, 5)
    rg, ro = g.run(), o.run()
    # the norm is a parallel sum: 1e-13 relative; the fields bit for bit
    assert len(rg) == len(ro)
    for a, b in zip(rg, ro):
        assert a["residual"] == pytest.approx(b["residual"], rel=1e-13) and a["status"] == b["status"]
        assert a["dof_updates"] == b["dof_updates"]
    for lvl in range(2):
        assert np.array_equal(g.vertices(lvl, lzb.T.V_U), o.vertices(lvl, lzb.T.V_U))
    assert g.stream_image() == o.stream_image()


def test_depth0_rejected():
    with pytest.raises(lzb.LzbError):
        lzb.Grid(lzb.make_desc(depth=0), 1)


def test_empty_and_ragged_element_batches():
    f = lzb.field_theta(16.0)
    assert lzb.integrate_elements(f, [], [], [], []).shape == (0, 16)
    # ragged n in one batch: every cell at its own n, as cell-by-cell calls
    x0 = np.array([0.0, 1 / 3, 2 / 3, 1 / 9, 5 / 9])
    n = np.array([1, 7, 2, 33, 4])
    got = lzb.integrate_elements(f, x0, x0[::-1], 1 / 9, n)
    for i in range(5):
        want = port.integrate_element(port.field_from_keys({"setup": "theta", "theta": "16"}), x0[i], x0[::-1][i],
                                      1 / 9, int(n[i]))
        assert np.abs(got[i] - want).max() <= 1e-12 * np.abs(want).max()


def test_element_sample_limit_and_bad_n():
    f = lzb.field_constant(1.0)
    with pytest.raises(lzb.LzbError):
        lzb.integrate_elements(f, [0.0], [0.0], [1.0], [0])
    lzb.integrate_elements(f, [0.0], [0.0], [1.0], [300])  # large n is fine


def test_codec_zero_subnormal_and_width_edges():
    z = lzb.codec.encode([0.0, -0.0], 3)
    assert bytes(z) == b"\x00\x00\x80\x00\x00\x80"  # -0 encodes as +0: (0, 0, -128)
    assert list(lzb.codec.decode(z, 3)) == [0.0, 0.0]
    sub = np.ldexp(1.25, -1070)  # subnormal: the exponent clamps to -128
    assert lzb.codec.roundtrip([sub], 4)[0] == np.ldexp(1.25, -128)
    raw = np.array([np.pi, -1e300, 5e-324])
    assert np.array_equal(lzb.codec.roundtrip(raw, 8), raw)  # p3 = 8 is the raw image
    assert lzb.codec.choose_precision([1e-9, -1e-9], 1e-8) == 0  # all within delta: record elided
    assert lzb.codec.choose_precision([np.pi], 0.0) == 8


def test_nonfinite_publish_is_a_protocol_error():
    d = lzb.make_desc(depth=2, field=lzb.field_constant(1.0))
    g = lzb.Grid(d, 1)
    m = np.eye(4).reshape(-1)
    m[5] = float("nan")
    with pytest.raises(lzb.ProtocolError):
        g.publish_element(2, 1, 1, m, 2, lzb.T.P1_TOP)
    g.publish_element(2, 1, 1, np.eye(4).reshape(-1), 2, lzb.T.P1_TOP)  # the grid stays usable


@pytest.mark.parametrize("mutate", ["truncated_header", "bad_version", "bad_count", "class3", "p3_is_1",
                                    "payload_cut"])
def test_corrupt_streams_rejected(mutate):
    d = lzb.make_desc(depth=2, field=lzb.field_theta(16.0), assembly="eager")
    g = lzb.Grid(d, 1)
    g.eager_setup()
    data = bytearray(g.stream_image())
    if mutate == "truncated_header":
        data = data[:7]
    elif mutate == "bad_version":
        data[4] = 9
    elif mutate == "bad_count":
        data[8] = data[8] + 1
    elif mutate == "class3":
        data[12] = 0xC0
    elif mutate == "p3_is_1":
        data[12] = (data[12] & 0xF0) | 1
    else:
        data = data[:-1]
    with pytest.raises(lzb.CorruptStreamError):
        lzb.Grid(d, 1).load_image(bytes(data))


def test_grid3_limits():
    f = lzb.field3_constant(1.0)
    for bad in (dict(depth=7), dict(depth=2, fixed_p3=1), dict(depth=2, fixed_p3=9)):
        with pytest.raises(lzb.LzbError):
            lzb.Grid3(bad.pop("depth"), f, **bad)
    G = lzb.Grid3(1, f)
    with pytest.raises(lzb.LzbError):
        G.assemble_fixed(17)
    G.assemble_fixed(1)
    ops, p3 = G.cells(0, 27)
    assert np.all(p3 == 0)  # eps = 1 at n = 1: the surplus is exactly 0, every record elided
    with pytest.raises(lzb.LzbError):
        G.step()  # no cycle state yet


def test_grid3_depth1_cycle_converges():
    G = lzb.Grid3(1, lzb.field3_constant(2.0))
    G.assemble_fixed(2)
    G.init_cycle(solver="adafac-pi", omega=0.6, max_cycles=500, target=1e-10)
    for _ in range(500):
        r = G.step()
        if r["status"] != lzb.T.CONTINUE:
            break
    assert r["status"] == lzb.T.CONVERGED

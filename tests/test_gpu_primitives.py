"""GPU parity of the batched primitives against the oracle / reference vectors.

Bar: bit-exact for the EXACT integration path on fields without
transcendentals, for the codec, choose_precision, Galerkin and BoxMG;
1e-12 normwise-relative for transcendental fields (CUDA libm vs glibc) and
for the FAST integration path (north_star tolerance).
"""
import os

import numpy as np
import pytest

import paper_2005_03606_b200 as lzb
from conftest import GOLDEN
from oracle import port
from oracle.types import field_constant, field_quadrant, field_sinusoid, field_theta

pytestmark = pytest.mark.gpu
VEC = np.load(os.path.join(GOLDEN, "vectors.npz"))
REL = 1e-12


def fields():
    return {"constant": field_constant(2.5), "theta1": field_theta(1.0), "theta16": field_theta(16.0),
            "quadrant": field_quadrant(1e-3), "sinusoid": field_sinusoid(0.9, 6.0),
            "checker": lzb.checkerboard(1, 8)}


TRANSCENDENTAL = {"theta1", "theta16", "sinusoid"}


def normwise(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.max(np.abs(a - b), axis=-1) / np.maximum(np.max(np.abs(b), axis=-1), 1e-300)


@pytest.mark.parametrize("name", sorted(fields()))
@pytest.mark.parametrize("integration", ["exact", "fast"])
def test_element_matches_reference_vectors(ctx, name, integration):
    f = fields()[name]
    boxes = VEC["element_boxes"]
    ns = VEC["element_ns"]
    x0 = np.repeat(boxes[:, 0], len(ns))
    y0 = np.repeat(boxes[:, 1], len(ns))
    h = np.repeat(boxes[:, 2], len(ns))
    n = np.tile(ns, len(boxes))
    got = lzb.integrate_elements(f, x0, y0, h, n, integration, ctx)
    want = VEC[f"element_{name}"]
    if integration == "exact" and name not in TRANSCENDENTAL:
        assert np.array_equal(got, want)  # bit-identical to the reference
    else:
        assert normwise(got, want).max() <= REL


@pytest.mark.parametrize("n", [1, 2, 5, 16, 33])
def test_level_integration_device_entry(ctx, n):
    """lzb_integrate_level_dev on a whole depth-3 level vs the oracle, both paths."""
    torch = pytest.importorskip("torch")
    f = lzb.checkerboard(7, 8)
    N = 27
    for integration, mode in (("exact", lzb.T.INTEGRATE_EXACT), ("fast", lzb.T.INTEGRATE_FAST)):
        out = torch.empty(N * N * 16, dtype=torch.float64, device="cuda")
        s = lzb.lib().lzb_ctx_solve_stream(ctx.h)
        lzb._check(lzb.lib().lzb_integrate_level_dev(ctx.h, lzb.C.byref(f), 3, n, out.data_ptr(), mode, s))
        got = out.cpu().numpy().reshape(N * N, 16)
        h = 1.0 / 27  # pow(1/3, 3) on the host below mirrors the device table
        h = np.power(1.0 / 3, 3)
        want = np.array([port.integrate_element(f, (c % N) * h, (c // N) * h, h, n) for c in range(N * N)])
        if integration == "exact":
            assert np.array_equal(got, want)
        else:
            assert normwise(got, want).max() <= REL


@pytest.mark.parametrize("p3", range(2, 9))
def test_codec_bit_exact(ctx, p3):
    vals = VEC["codec_values"]
    enc = lzb.codec.encode(vals, p3, ctx)
    assert np.array_equal(enc, VEC[f"codec_bytes_{p3}"])
    dec = lzb.codec.decode(enc, p3, ctx)
    assert np.array_equal(dec.view(np.uint64), VEC[f"codec_rt_{p3}"].view(np.uint64))


def test_codec_known_answers_and_errors(ctx):
    assert lzb.codec.encode_value(1.0, 2, ctx) == b"\x00\x00"          # test_codec.cpp:21-27
    assert lzb.codec.encode_value(-0.75, 2, ctx) == b"\xc0\xff"        # test_codec.cpp:29-35
    assert lzb.codec.roundtrip([np.ldexp(1.5, 300)], 3, ctx)[0] == np.ldexp(1.5, 127)
    assert lzb.codec.roundtrip([np.ldexp(1.5, -300)], 3, ctx)[0] == np.ldexp(1.5, -128)
    for bad in (float("nan"), float("inf")):
        with pytest.raises(lzb.ProtocolError):
            lzb.codec.encode([1.0, bad], 4, ctx)
    assert lzb.codec.choose_precision([1.2345678901, -0.987654321, 1.5, 0.7777777], 1e-8, ctx) == 5
    rng = np.random.default_rng(3)  # idempotence on canonical bytes (test_codec.cpp:70-81)
    x = np.ldexp(rng.uniform(1, 2, 5000), rng.integers(-100, 100, 5000))
    for p3 in (2, 4, 7):
        b1 = lzb.codec.encode(x, p3, ctx)
        b2 = lzb.codec.encode(lzb.codec.decode(b1, p3, ctx), p3, ctx)
        assert np.array_equal(b1, b2)


def test_choose_precision_records(ctx):
    for i, d in enumerate(VEC["choose_deltas"]):
        assert np.array_equal(lzb.codec.choose_precision_records(VEC["choose_recs16"], 16, d, ctx),
                              VEC[f"choose16_{i}"])
        assert np.array_equal(lzb.codec.choose_precision_records(VEC["choose_recs80"], 80, d, ctx),
                              VEC[f"choose80_{i}"])


def test_galerkin_and_boxmg_bit_exact(ctx):
    ch = VEC["transfer_children"]
    assert np.array_equal(lzb.galerkin_coarse_element(ch, None, ctx), VEC["galerkin_geo"])
    P, fb = lzb.boxmg_prolongation(ch, ctx)
    assert np.array_equal(P, VEC["boxmg_P"]) and np.array_equal(fb, VEC["boxmg_fallback"])
    assert np.array_equal(lzb.galerkin_coarse_element(ch, P, ctx), VEC["galerkin_boxmg"])


def test_boxmg_constant_eps_is_geometric(ctx):
    # test_transfer.cpp:28-40
    k = lzb.integrate_element((0, 0, 1), field_constant(1.0), 1, ctx=ctx)
    P, fb = lzb.boxmg_prolongation(np.tile(k, (1, 9, 1)), ctx)
    assert fb[0] == 0 and np.max(np.abs(P[0] - lzb.geometric_prolongation())) < 1e-10

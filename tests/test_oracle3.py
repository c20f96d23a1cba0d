"""The restated 3D oracle (oracle/port3.py) against its internal pins, on CPU
(the reference has no 3D code: SURVEY.md §8c, "3D: parity unpinned by the
reference"), and the product's GRF generator (host code) against the numpy
restatement."""
import ctypes

import numpy as np
import pytest

import paper_2005_03606_b200 as lzb
from oracle import port as orc
from oracle import port3 as o3


@pytest.mark.parametrize("n", [1, 2, 3])
def test_constant_eps_is_the_analytic_q1_stiffness(n):
    for h in (1.0, 1.0 / 9):
        K = o3.element3(lambda x, y, z: 2.5, 0.0, 0.0, 0.0, h, n)
        assert np.allclose(K, 2.5 * o3.unit_stiffness3(h), rtol=0, atol=1e-15)


def test_grf_element_symmetric_zero_row_sum():
    g = o3.grf_table(3, 8, 0.1, 1.0)
    K = o3.element3(lambda x, y, z: o3.eps_grf(g, x, y, z), 0.2, 0.4, 0.6, 1.0 / 27, 3)
    assert np.allclose(K, K.T, rtol=0, atol=1e-15 * np.abs(K).max())
    assert np.abs(K.sum(axis=1)).max() < 1e-13 * np.abs(K).max()
    assert np.all(np.diag(K) > 0)


def test_z_independent_eps_is_the_tensor_product_of_2d():
    """K3 = h (K2 (x) Mz + M2 (x) Dz), K2 from the reference-pinned 2D oracle."""
    f2 = orc.field_from_keys({"setup": "theta", "theta": "16"})
    x0, y0, h, n = 2 / 9, 5 / 9, 1 / 9, 3
    K2 = orc.integrate_element(f2, x0, y0, h, n).reshape(4, 4)
    def eps2(x, y):
        return orc.lib().orc_field_eval(ctypes.byref(f2), x, y)

    M2 = o3.mass2(eps2, x0, y0, h, n)
    K3 = o3.element3(lambda x, y, z: eps2(x, y), x0, y0, 0.3, h, n)
    assert np.allclose(K3, o3.extruded_from_2d(K2, M2, h), rtol=0, atol=1e-14 * np.abs(K3).max())


def test_grf_table_product_matches_restatement():
    """lzb_grf_table (host C++ radix-2 FFT) against numpy's inverse FFT."""
    want = o3.grf_table(7, 16, 0.05, 1.0)
    got = lzb.grf_table(7, 16, 0.05, 1.0)
    assert np.abs(got - want).max() < 1e-12


def test_grf_table_statistics():
    g = lzb.grf_table(11, 64, 0.05, 1.0)
    assert abs(g.mean()) < 0.2 and 0.6 < g.var() < 1.4
    # the covariance falls with the lag like exp(-r^2 / 2 ell^2): at r = ell about 0.6
    lag = int(round(0.05 * 64))
    c = np.mean(g * np.roll(g, lag, axis=0)) / g.var()
    assert 0.35 < c < 0.85


def test_sphere_tree_counts():
    """Leaf counts of the restated adaptive spacetree (level 2 inside the ball,
    level 1 elsewhere): the 27 level-1 cells all meet the r = 0.25 ball except
    the 8 corners; the others refine into level-2 leaves."""
    from oracle import port3 as o3
    L = o3.sphere_tree_leaves(1, 2)
    per = np.bincount(L[:, 0], minlength=3)
    assert per[0] == 0 and per[1] == 8 and per[2] == 19 * 27
    assert o3.eps_sphere(0.5, 0.5, 0.5) == pytest.approx(100.0) and o3.eps_sphere(0.0, 0.0, 0.0) == pytest.approx(1.0)


def _unit_ops(leaves, eps):
    """n = 1 trilinear elements eps(centre) K_unit(h) per leaf."""
    out = np.zeros((len(leaves), 8, 8))
    for i, (lv, cx, cy, cz) in enumerate(leaves):
        h = (1.0 / 3) ** lv
        out[i] = eps((cx + 0.5) * h, (cy + 0.5) * h, (cz + 0.5) * h) * o3.unit_stiffness3(h)
    return out


def test_cycle3a_without_adaptivity_is_cycle3():
    """The adaptive restatement on a tree refined uniformly to depth 2 is the
    regular 3D cycle: residual history and u on every level within 1e-12."""
    leaves = o3.sphere_tree_leaves(2, 2)
    ops = _unit_ops(leaves, lambda x, y, z: 1.0 + x + 2 * y * z)
    order = np.lexsort((leaves[:, 1], leaves[:, 2], leaves[:, 3]))  # [z, y, x] raster for Cycle3
    a = o3.Cycle3A(leaves, ops, 2, seed=7)
    b = o3.Cycle3(ops[order], 2, seed=7)
    for _ in range(4):
        ra, rb = a.step(), b.step()
        assert ra["residual"] == pytest.approx(rb["residual"], rel=1e-12)
    for lvl in range(3):
        assert np.abs(a.v[lvl]["u"] - b.v[lvl]["u"]).max() <= 1e-12


def test_cycle3a_sphere_tree_converges():
    """On the sphere tree (level 3 in the ball, 1 elsewhere, hanging nodes)
    the adaptive cycle reduces the residual."""
    leaves = o3.sphere_tree_leaves(1, 3)
    a = o3.Cycle3A(leaves, _unit_ops(leaves, o3.eps_sphere), 3, seed=3)
    assert (a.kind[3] == 3).any() and (a.kind[2] == 3).any()
    reps = [a.step() for _ in range(25)]
    assert reps[-1]["normalized"] < 0.05, [r["normalized"] for r in reps[::6]]


def test_galerkin_class_weights_factor_per_axis():
    """The class-form Galerkin weights W[child][k][q] (sum over the (i, j) of
    class k of Q_child[i][a_q] Q_child[j][b_q], trilinear Q) equal the product
    of per-axis factors wa[l][kd][qd] that k3_galerkin contracts axis by axis."""
    def qax(L, a):
        return (L if a else 3 - L) / 3.0

    wa = np.zeros((3, 3, 3))
    for l in range(3):
        for kd in range(3):
            for qd in range(3):
                a, b = int(qd == 2), int(qd >= 1)
                wa[l, kd, qd] = sum(qax(l + i, a) * qax(l + j, b) for i in (0, 1) for j in (0, 1)
                                    if (2 * i if i == j else 1) == kd)

    def cls(i, j):
        return tuple(2 * ((i >> d) & 1) if ((i >> d) & 1) == ((j >> d) & 1) else 1 for d in range(3))

    for lx, ly, lz in [(0, 0, 0), (1, 2, 0), (2, 1, 1), (2, 2, 2)]:
        for q in range(27):
            qx, qy, qz = q // 9, (q // 3) % 3, q % 3
            a = (qx == 2) + 2 * (qy == 2) + 4 * (qz == 2)
            b = (qx >= 1) + 2 * (qy >= 1) + 4 * (qz >= 1)
            W = np.zeros((3, 3, 3))
            for i in range(8):
                for j in range(8):
                    Li = (lx + (i & 1), ly + ((i >> 1) & 1), lz + (i >> 2))
                    Lj = (lx + (j & 1), ly + ((j >> 1) & 1), lz + (j >> 2))
                    W[cls(i, j)] += o3.pw3(Li, a) * o3.pw3(Lj, b)
            want = np.einsum("i,j,k->ijk", wa[lx, :, qx], wa[ly, :, qy], wa[lz, :, qz])
            assert np.allclose(W, want, rtol=1e-14, atol=1e-16)

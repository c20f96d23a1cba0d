"""Golden vectors for the element / codec / transfer primitives, produced by
the UNMODIFIED reference (oracle/_ref) so that the CPU suite can pin the C
restatement even where the reference tree is absent.

Usage: python tests/golden/make_vectors.py   (writes tests/golden/vectors.npz)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402
from oracle.types import field_constant, field_quadrant, field_sinusoid, field_theta  # noqa: E402
from oracle import port  # noqa: E402


def fields():
    cb = port.Field()
    port.lib().orc_field_checkerboard(port.C.byref(cb), 1, 8)
    return {
        "constant": field_constant(2.5), "theta1": field_theta(1.0), "theta16": field_theta(16.0),
        "quadrant": field_quadrant(1e-3), "sinusoid": field_sinusoid(0.9, 6.0), "checker": cb,
    }


def main():
    rng = np.random.default_rng(20260419)
    out = {}
    # element matrices on a spread of boxes / n
    boxes = [(0.0, 0.0, 1.0), (1 / 3, 1 / 3, 1 / 3), (2 / 9, 5 / 9, 1 / 9), (121 / 243, 7 / 243, 1 / 243),
             (0.5, 0.25, 1 / 27)]
    ns = [1, 2, 3, 4, 7, 16]
    for name, f in fields().items():
        mats = []
        for (x0, y0, h) in boxes:
            for n in ns:
                mats.append(ref.integrate_element(f, x0, y0, h, n))
        out[f"element_{name}"] = np.array(mats)
    out["element_boxes"] = np.array(boxes)
    out["element_ns"] = np.array(ns)
    # codec: random values over a wide exponent range plus edge cases
    mant = rng.uniform(1.0, 2.0, 4000) * rng.choice([-1.0, 1.0], 4000)
    expo = rng.integers(-140, 140, 4000)
    vals = np.ldexp(mant, expo)
    edge = np.array([0.0, -0.0, 1.0, -0.75, 2.0 ** -128, -(2.0 ** -128), 2.0 ** -129, 1.5 * 2.0 ** 300,
                     1.5 * 2.0 ** -300, 5e-324, -5e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
                     np.nextafter(1.0, 2.0), np.nextafter(1.0, 0.0)])
    vals = np.concatenate([vals, edge])
    out["codec_values"] = vals
    for p3 in range(2, 9):
        out[f"codec_bytes_{p3}"] = ref.encode_many(vals, p3)
        out[f"codec_rt_{p3}"] = ref.decode_many(out[f"codec_bytes_{p3}"], p3)
    # choose_precision on 16- and 80-entry records with several deltas
    recs16 = np.ldexp(rng.uniform(-1, 1, (500, 16)), rng.integers(-30, 5, (500, 16)))
    recs16[::7] = 0.0
    recs16[3::11, ::3] *= 1e-12
    recs80 = np.ldexp(rng.uniform(-1, 1, (200, 80)), rng.integers(-40, 2, (200, 80)))
    out["choose_recs16"] = recs16
    out["choose_recs80"] = recs80
    for i, d in enumerate([0.0, 1e-12, 1e-8, 1e-4]):
        out[f"choose16_{i}"] = ref.choose_many(recs16, 16, d)
        out[f"choose80_{i}"] = ref.choose_many(recs80, 80, d)
    out["choose_deltas"] = np.array([0.0, 1e-12, 1e-8, 1e-4])
    # transfer: Galerkin (geometric + random P) and BoxMG on random Laplacian-like children
    ch = []
    for _ in range(64):
        kids = []
        for _ in range(9):
            w = rng.uniform(0.05, 1.0, (4, 4))
            w = np.triu(w, 1)
            w = w + w.T
            m = -w
            np.fill_diagonal(m, w.sum(1))
            kids.append(m.reshape(16))
        ch.append(np.array(kids))
    ch = np.array(ch)
    geo = np.zeros(64)
    port.lib().orc_geometric(port._ptr(geo))
    out["transfer_children"] = ch
    out["galerkin_geo"] = np.array([ref.galerkin(c, geo) for c in ch])
    bm = [ref.boxmg(c) for c in ch]
    out["boxmg_P"] = np.array([b[0] for b in bm])
    out["boxmg_fallback"] = np.array([b[1] for b in bm])
    out["galerkin_boxmg"] = np.array([ref.galerkin(c, b[0]) for c, b in zip(ch, bm)])
    np.savez_compressed(os.path.join(HERE, "vectors.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()

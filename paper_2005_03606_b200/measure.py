"""HBM roofline of the leaf-level cycle kernels and the stream pack.

Algorithmic bytes per launch are the unique bytes a
perfect-cache kernel must move for a 3^depth x 3^depth grid; times come from
lzb_grid_time_kernel (CUDA events on the solve stream, back-to-back launches
of one kernel). Used by bench.py and tools/smoother_roofline.py.
"""
from __future__ import annotations

from . import _types as T


def kernel_bytes(depth: int, image_bytes: int, payload_leaves: int) -> dict:
    N = 3 ** depth
    nc, nv = N * N, (N + 1) ** 2
    nvc = (N // 3 + 1) ** 2
    total_cells = sum(9 ** l for l in range(depth + 1))
    return {
        # u read, uhat write (+ coarse u)
        T.TK_UHAT: nv * 16 + nvc * 8,
        # fl, u, uhat read; r, rhat, diag written; one 128-B operator + p1 per cell
        T.TK_RESIDUAL: nv * 48 + nc * (128 + 4),
        # rhat read, coarse fl written
        T.TK_RESTRICT: nv * 8 + nvc * 8,
        # diag, r, u read; u written
        T.TK_JACOBI: nv * 32,
        # u read + written (+ coarse u, usnap)
        T.TK_PROLONG: nv * 16 + nvc * 16,
        # per record: p1, p3, p2, offset (14 B); the stored operator of every leaf
        # with a payload; the image bytes written
        T.TK_PACK: total_cells * 14 + payload_leaves * 128 + image_bytes,
    }


KERNEL_NAMES = {T.TK_UHAT: "k_uhat", T.TK_RESIDUAL: "k_residual", T.TK_RESTRICT: "k_restrict",
                T.TK_JACOBI: "k_jacobi", T.TK_PROLONG: "k_prolong", T.TK_PACK: "k_pack_patches"}


def hbm_kernel_table(grid, depth: int, peak_gbs: float, reps: int = 10) -> dict:
    """Per-kernel ms / algorithmic bytes / GB/s / fraction of `peak_gbs` on an
    assembled grid (one or more cycles run, so every vector is live)."""
    st = grid.stats()
    img = grid.stream_image_size()
    ab = kernel_bytes(depth, img, st.fine_cells - st.p3_histogram[0])
    out = {}
    for tk, name in KERNEL_NAMES.items():
        ms = grid.time_kernel(tk, reps)
        gbs = ab[tk] / (ms * 1e-3) / 1e9
        out[name] = {"ms": ms, "bytes": ab[tk], "GB/s": gbs, "frac": gbs / peak_gbs}
    out["image_bytes"] = img
    return out

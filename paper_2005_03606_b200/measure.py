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


MANTISSA_BITS = {2: 7, 3: 15, 4: 23, 5: 31, 6: 39, 7: 47, 8: 52}


def width_sweep(ctx, field, depth: int, peak_gbs: float, widths=(2, 3, 4, 5, 6, 7, 8), reps=10, cycles=10):
    """BASELINE configs[4] in 2D: every leaf record at one width p3 (fixed_p3)
    and the residual reading the compressed records (plane_width = p3), plus
    the delta-chosen widths with FP64 operators as the reference row. Per
    width: LZMG bytes per leaf, residual bytes per cell, k_residual time and
    roofline fraction, cycle time and DoF-updates/s."""
    import torch

    import paper_2005_03606_b200 as lzb
    N = 3 ** depth
    nc, nv = N * N, (N + 1) ** 2
    stream = torch.cuda.ExternalStream(ctx.solve_stream)
    rows = []
    for p3 in (0,) + tuple(widths):
        w = p3 if p3 < 8 else 0  # width 8 reads the FP64 rows
        d = lzb.make_desc(depth=depth, field=field, solver="adafac-pi", omega=0.6, rhs_kind="sinprod",
                          max_cycles=10 ** 6, delta_max=1e-8, integration="fast", fixed_p3=p3, plane_width=w)
        g = lzb.Grid(d, 1, ctx)
        g.assemble_fixed(4)
        for _ in range(2):
            g.step()
        ms = g.time_kernel(T.TK_RESIDUAL, reps)
        cell_b = (16 * w + 1) if w else (128 + 4)
        nbytes = nv * 48 + nc * cell_b
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(cycles):
            g.step()
        b.record(stream)
        b.synchronize()
        cyc = a.elapsed_time(b) / cycles
        st = g.stats()
        rows.append({"p3": p3 if p3 else "chosen", "mantissa_bits": MANTISSA_BITS.get(p3),
                     "lzmg_bytes_per_leaf": st.fine_stored_bytes / st.fine_cells,
                     "residual_bytes_per_cell": cell_b, "k_residual_ms": ms,
                     "k_residual_frac": nbytes / (ms * 1e-3) / 1e9 / peak_gbs,
                     "cycle_ms": cyc, "dof_updates_per_s": (N - 1) ** 2 / (cyc * 1e-3)})
        g.close()
        del g
        torch.cuda.empty_cache()
    return rows

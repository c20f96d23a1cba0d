"""B200-native delayed-assembly hot path of arXiv 2005.03606.

Python view of the C-ABI in ``include/lzb.h`` (``lib/liblzb.so``: hand-written
sm_100a kernels + host C++). Names mirror the reference's C++ interface
(``/root/reference/proj/include/lazymg``): ``integrate_element``,
``codec.encode_value/decode_value/choose_precision``, ``galerkin_coarse_element``,
``boxmg_prolongation``, and ``Grid`` = Mesh + CellStream + Assembler +
AdditiveSolver on a regular 2D spacetree, plus ``run_experiment`` /
``emit_table`` / ``compare_runs`` for the config / telemetry interface.

There is no CPU fallback: every call runs on the GPU, and a missing library
or device raises ``LzbError``.
"""
from __future__ import annotations

import atexit
import ctypes as C
import os
import subprocess
import weakref

import numpy as np

from . import _types as T
from ._types import (CompressionStats, CycleReport, Field, GridDesc, Rhs, field_checkerboard,  # noqa: F401
                     field_constant, field_quadrant, field_sinusoid, field_theta, report_dict,
                     TK_UHAT, TK_RESIDUAL, TK_RESTRICT, TK_JACOBI, TK_PROLONG, TK_PACK, TK_FRONT, TK_BACK)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "liblzb.so")


class LzbError(RuntimeError):
    """Status-coded failure of a C-ABI call (codes in include/lzb_types.h)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[lzb status {code}] {msg}")
        self.code = code


class ProtocolError(LzbError):  # lazymg::protocol_error
    pass


class CorruptStreamError(LzbError):  # lazymg::corrupt_stream_error
    pass


class ResourceError(LzbError):  # lazymg::resource_error
    pass


_EXC = {T.ERR_PROTOCOL: ProtocolError, T.ERR_CORRUPT: CorruptStreamError, T.ERR_RESOURCE: ResourceError}

_lib = None


def build():
    """Compile liblzb.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "csrc")], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LzbError(T.ERR_CUDA, f"{LIB_PATH} missing: run paper_2005_03606_b200.build()")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_double
        L.lzb_last_error.restype = C.c_char_p
        L.lzb_launch_count.restype = C.c_uint64
        L.lzb_ctx_create.argtypes = [C.c_int, C.POINTER(vp)]
        L.lzb_ctx_destroy.argtypes = [vp]
        L.lzb_ctx_synchronize.argtypes = [vp]
        L.lzb_ctx_solve_stream.restype = vp
        L.lzb_ctx_solve_stream.argtypes = [vp]
        L.lzb_ctx_assembly_stream.restype = vp
        L.lzb_ctx_assembly_stream.argtypes = [vp]
        L.lzb_field_checkerboard.argtypes = [C.POINTER(Field), C.c_uint64, C.c_int]
        L.lzb_field_eval_host.restype = dbl
        L.lzb_field_eval_host.argtypes = [C.POINTER(Field), dbl, dbl]
        L.lzb_integrate_elements.argtypes = [vp, C.POINTER(Field), i64, vp, vp, vp, vp, vp, C.c_int]
        L.lzb_integrate_elements_dev.argtypes = [vp, C.POINTER(Field), i64, vp, vp, vp, vp, vp, C.c_int, vp]
        L.lzb_integrate_level_dev.argtypes = [vp, C.POINTER(Field), C.c_int, C.c_int, vp, C.c_int, vp]
        L.lzb_integrate_level.argtypes = [vp, C.POINTER(Field), C.c_int, C.c_int, vp, C.c_int]
        L.lzb_probe_fp64_tflops.argtypes = [C.c_int, C.POINTER(dbl)]
        L.lzb_subcell_stiffness.argtypes = [vp, dbl, dbl, dbl, dbl, vp]
        L.lzb_codec_encode.argtypes = [vp, i64, vp, C.c_int, vp]
        L.lzb_codec_decode.argtypes = [vp, i64, vp, C.c_int, vp]
        L.lzb_codec_choose_precision.argtypes = [vp, i64, i32, vp, dbl, vp]
        L.lzb_codec_choose_precision_dev.argtypes = [vp, i64, i32, vp, dbl, vp, vp]
        L.lzb_pack_header.restype = C.c_uint8
        L.lzb_pack_header.argtypes = [i32, C.c_int, C.c_int]
        L.lzb_unpack_header.argtypes = [C.c_uint8] + [C.POINTER(C.c_int)] * 3
        L.lzb_galerkin.argtypes = [vp, i64, vp, vp, vp]
        L.lzb_boxmg.argtypes = [vp, i64, vp, vp, vp]
        L.lzb_geometric_prolongation.argtypes = [vp]
        L.lzb_grid_create.argtypes = [vp, C.POINTER(GridDesc), C.POINTER(vp)]
        L.lzb_grid_destroy.argtypes = [vp]
        L.lzb_grid_init_noise.argtypes = [vp, C.c_uint64]
        L.lzb_grid_eager_setup.argtypes = [vp]
        L.lzb_grid_assemble_fixed.argtypes = [vp, C.c_int]
        L.lzb_grid_step.argtypes = [vp, C.POINTER(CycleReport)]
        L.lzb_grid_vcycle.argtypes = [vp, C.c_int, C.POINTER(CycleReport)]
        L.lzb_grid_run.argtypes = [vp, vp, C.c_int, C.POINTER(C.c_int)]
        L.lzb_grid_pass.argtypes = [vp, C.c_int, C.POINTER(dbl)]
        L.lzb_grid_cycle.argtypes = [vp]
        L.lzb_grid_vertices.argtypes = [vp, C.c_int, C.c_int, vp, C.c_int]
        L.lzb_grid_cells.argtypes = [vp, C.c_int, vp, vp, vp, vp, vp]
        L.lzb_grid_transfer.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp]
        L.lzb_grid_publish_element.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, C.c_int, i32]
        L.lzb_grid_publish_level.argtypes = [vp, C.c_int, vp, vp, i32]
        L.lzb_grid_vertex_stencils.argtypes = [vp, C.c_int, C.c_int, vp]
        L.lzb_scatter_row.argtypes = [vp, C.c_int, vp]
        L.lzb_grid_assemble_fixed_raw.argtypes = [vp, C.c_int, vp]
        L.lzb_grid_adaptive_step.argtypes = [vp, C.c_int, C.c_int, C.c_int]
        L.lzb_grid_stats.argtypes = [vp, C.POINTER(CompressionStats)]
        L.lzb_grid_stream_image.argtypes = [vp, vp, i64, C.POINTER(i64)]
        L.lzb_grid_stream_load.argtypes = [vp, vp, i64]
        L.lzb_grid_save.argtypes = [vp, C.c_char_p]
        L.lzb_grid_load.argtypes = [vp, C.c_char_p]
        L.lzb_grid_pending.restype = i64
        L.lzb_grid_pending.argtypes = [vp]
        L.lzb_grid_device_view.argtypes = [vp, C.c_int, C.c_int, C.POINTER(vp)]
        L.lzb_grid_time_kernel.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.lzb_grid_set_slab.argtypes = [vp, C.c_int, C.c_int]
        L.lzb_grf_table.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_double, vp]
        L.lzb_integrate_elements3.argtypes = [vp, C.POINTER(T.Field3), i64, vp, vp, vp, vp, vp, vp]
        L.lzb_grid3_create.argtypes = [vp, C.c_int, C.POINTER(T.Field3), C.c_double, C.c_int, C.POINTER(vp)]
        L.lzb_grid_assemble_stream.argtypes = [vp, C.c_int, vp, i64, C.POINTER(i64), vp]
        L.lzb_grid3_create_slab.argtypes = [vp, C.c_int, C.POINTER(T.Field3), C.c_double, C.c_int, C.c_int, C.c_int,
                                            C.c_int, C.POINTER(vp)]
        L.lzb_grid3_create_window.argtypes = [vp, C.c_int, C.POINTER(T.Field3), C.c_double, C.c_int, C.c_int,
                                              C.c_int, C.c_int, C.POINTER(vp)]
        L.lzb_grid3_leaf_storage.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.lzb_grid3_create_planes.argtypes = [vp, C.c_int, C.POINTER(T.Field3), C.c_double, C.c_int, C.c_int,
                                               C.POINTER(vp)]
        L.lzb_grid3_destroy.argtypes = [vp]
        L.lzb_grid3_assemble_fixed.argtypes = [vp, C.c_int]
        L.lzb_grid3_stats.argtypes = [vp, C.POINTER(CompressionStats)]
        L.lzb_grid3_cells.argtypes = [vp, i64, i64, vp, vp]
        L.lzb_grid3_init_cycle.argtypes = [vp, C.c_int, C.c_double, C.c_double, C.c_uint64, C.c_int, C.c_double]
        L.lzb_grid3_step.argtypes = [vp, C.POINTER(CycleReport)]
        L.lzb_grid3_vcycle.argtypes = [vp, C.c_int, C.POINTER(CycleReport)]
        L.lzb_grid3_vertices.argtypes = [vp, C.c_int, C.c_int, vp]
        L.lzb_grid3_set_slab.argtypes = [vp, C.c_int, C.c_int]
        L.lzb_grid3_dist_phase.argtypes = [vp, C.c_int]
        L.lzb_grid3_dist_result.argtypes = [vp, C.POINTER(C.c_double)]
        L.lzb_grid3_dist_report.argtypes = [vp, C.c_double, C.POINTER(CycleReport)]
        L.lzb_grid3_assemble_planes.argtypes = [vp, C.c_int, C.c_int, C.c_int]
        L.lzb_grid3_galerkin_planes.argtypes = [vp, C.c_int, C.c_int, C.c_int]
        L.lzb_grid3_coarse_below.argtypes = [vp, C.c_int]
        L.lzb_grid3_level_ops.argtypes = [vp, C.c_int, C.POINTER(vp)]
        L.lzb_tree3_create.argtypes = [vp, C.c_int, C.c_int, C.POINTER(T.Field3), C.c_double, C.c_int, C.POINTER(vp)]
        L.lzb_tree3_destroy.argtypes = [vp]
        L.lzb_tree3_counts.argtypes = [vp, vp, C.POINTER(i64)]
        L.lzb_tree3_assemble.argtypes = [vp, C.c_int]
        L.lzb_tree3_set_shell.argtypes = [vp, C.c_double, C.POINTER(i64)]
        L.lzb_tree3_assemble_shell.argtypes = [vp, C.c_int]
        L.lzb_tree3_stats.argtypes = [vp, C.POINTER(CompressionStats)]
        L.lzb_tree3_cells.argtypes = [vp, i64, i64, vp, vp, vp, vp]
        L.lzb_tree3_init_cycle.argtypes = [vp, C.c_int, C.c_double, C.c_double, C.c_uint64, C.c_int, C.c_double]
        L.lzb_tree3_refresh_ops.argtypes = [vp]
        L.lzb_tree3_refine.argtypes = [vp, C.c_double, C.c_int, C.POINTER(C.c_int64)]
        L.lzb_tree3_step.argtypes = [vp, C.POINTER(CycleReport)]
        L.lzb_tree3_vertices.argtypes = [vp, C.c_int, C.c_int, vp]
        L.lzb_grid3_time_kernel.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.lzb_grid3_device_view.argtypes = [vp, C.c_int, C.c_int, C.POINTER(vp)]
        L.lzb_grid_plane_arrays.argtypes = [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(C.c_int)]
        L.lzb_grid_dist_phase.argtypes = [vp, C.c_int, C.c_int]
        L.lzb_nccl_unique_id.argtypes = [vp]
        L.lzb_ctx_comm_init.argtypes = [vp, vp, C.c_int, C.c_int]
        L.lzb_ctx_comm_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.lzb_grid_dist_cycle.argtypes = [vp, C.POINTER(CycleReport)]
        L.lzb_grid_dist_cycle_loopback.argtypes = [vp, C.c_int, C.POINTER(CycleReport)]
        L.lzb_grid_dist_assemble.argtypes = [vp, C.c_int]
        L.lzb_grid_dist_assemble_loopback.argtypes = [vp, C.c_int, C.c_int]
        L.lzb_grid3_dist_cycle.argtypes = [vp, C.POINTER(CycleReport)]
        L.lzb_grid3_dist_cycle_loopback.argtypes = [vp, C.c_int, C.POINTER(CycleReport)]
        L.lzb_grid3_dist_assemble.argtypes = [vp, C.c_int]
        L.lzb_grid3_dist_assemble_loopback.argtypes = [vp, C.c_int, C.c_int]
        L.lzb_grid_dist_result.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        L.lzb_grid_dist_report.argtypes = [vp, C.c_double, C.POINTER(C.c_uint64), C.POINTER(CycleReport)]
        L.lzb_run_experiment_file.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.lzb_run_experiment_text.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.lzb_last_reports.argtypes = [vp, C.c_int, C.POINTER(C.c_int)]
        L.lzb_config_keys.argtypes = [C.c_char_p, C.c_char_p, i64]
        L.lzb_emit_table.argtypes = [C.c_char_p, C.c_char_p, i64]
        L.lzb_compare_runs.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, i64]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        msg = lib().lzb_last_error().decode()
        raise _EXC.get(rc, LzbError)(rc, msg)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def launch_count() -> int:
    return lib().lzb_launch_count()


class Context:
    """Device + solve (high-priority) and assembly (low-priority) streams."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib().lzb_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            if _lib is not None:  # interpreter teardown may have released the module
                _lib.lzb_ctx_destroy(self.h)
            self.h = None

    __del__ = close

    def synchronize(self):
        _check(lib().lzb_ctx_synchronize(self.h))

    @property
    def solve_stream(self):
        return lib().lzb_ctx_solve_stream(self.h)

    def comm_init(self, unique_id: bytes, nranks: int, rank: int):
        """The context's NCCL communicator for the C++ slab data plane
        (unique_id from nccl_unique_id() on rank 0, shared by the launcher)."""
        _torch_nccl_first()
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        _check(lib().lzb_ctx_comm_init(self.h, buf, nranks, rank))

    def comm_info(self):
        r, n = C.c_int(), C.c_int()
        _check(lib().lzb_ctx_comm_info(self.h, C.byref(r), C.byref(n)))
        return r.value, n.value


def _torch_nccl_first():
    # liblzb.so loads NCCL at run time by soname (libnccl.so.2), preferring a copy the
    # process already holds. When torch is installed its bundled NCCL must be that
    # copy: loading the system library first would make a later `import torch`
    # resolve libtorch_cuda.so against the wrong version.
    try:
        import torch  # noqa: F401
    except ImportError:
        pass


def nccl_unique_id() -> bytes:
    _torch_nccl_first()
    buf = (C.c_uint8 * 128)()
    _check(lib().lzb_nccl_unique_id(buf))
    return bytes(buf)


def _handles(grids):
    arr = (C.c_void_p * len(grids))(*[g.h.value if isinstance(g.h, C.c_void_p) else g.h for g in grids])
    return arr


def dist_cycle_loopback(grids) -> dict:
    """One slab-distributed cycle of the C++ data plane over several slab grids
    of this process (slab i of len(grids); device copies instead of NCCL)."""
    r = CycleReport()
    fn = lib().lzb_grid3_dist_cycle_loopback if isinstance(grids[0], Grid3) else lib().lzb_grid_dist_cycle_loopback
    _check(fn(_handles(grids), len(grids), C.byref(r)))
    return report_dict(r)


def dist_assemble_loopback(grids, n):
    fn = (lib().lzb_grid3_dist_assemble_loopback if isinstance(grids[0], Grid3)
          else lib().lzb_grid_dist_assemble_loopback)
    _check(fn(_handles(grids), len(grids), n))


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("LZB_DEVICE", "0")))
    return _default_ctx


def checkerboard(seed=1, blocks=8) -> Field:
    """BASELINE config 1 eps (8x8 blocks of 10^U(-2,2)); table computed in C."""
    f = Field()
    lib().lzb_field_checkerboard(C.byref(f), seed, blocks)
    return f


# ------------------------------------------------------------------ element
def integrate_elements(field: Field, x0, y0, h, n, integration="exact", ctx: Context | None = None):
    """Batched integrate_element(CellBox{x0,y0,h}, eps, n) (element.hpp:36-49)."""
    ctx = ctx or default_context()
    x0 = np.ascontiguousarray(x0, dtype=np.float64).reshape(-1)
    y0 = np.ascontiguousarray(np.broadcast_to(y0, x0.shape), dtype=np.float64)
    h = np.ascontiguousarray(np.broadcast_to(h, x0.shape), dtype=np.float64)
    n = np.ascontiguousarray(np.broadcast_to(n, x0.shape), dtype=np.int32)
    out = np.zeros((x0.size, 16))
    mode = T.INTEGRATE_FAST if integration == "fast" else T.INTEGRATE_EXACT
    _check(lib().lzb_integrate_elements(ctx.h, C.byref(field), x0.size, _ptr(x0), _ptr(y0), _ptr(h), _ptr(n),
                                        _ptr(out), mode))
    return out


def integrate_element(box, field: Field, n: int, integration="exact", ctx=None):
    x0, y0, h = box
    return integrate_elements(field, [x0], [y0], [h], [n], integration, ctx)[0]


def integrate_level(field: Field, level: int, n: int, integration="exact", out=None, ctx=None):
    """All cells of a regular level at one n into a host array (N*N, 16)."""
    ctx = ctx or default_context()
    N = 3 ** level
    if out is None:
        out = np.zeros((N * N, 16))
    mode = T.INTEGRATE_FAST if integration == "fast" else T.INTEGRATE_EXACT
    _check(lib().lzb_integrate_level(ctx.h, C.byref(field), level, n, _ptr(out), mode))
    return out


def probe_fp64_tflops(device=0) -> float:
    v = C.c_double()
    _check(lib().lzb_probe_fp64_tflops(device, C.byref(v)))
    return v.value


def reference_subcell_stiffness(a, b, c, d, ctx=None):
    ctx = ctx or default_context()
    out = np.zeros(16)
    _check(lib().lzb_subcell_stiffness(ctx.h, a, b, c, d, _ptr(out)))
    return out


# ------------------------------------------------------------------ codec
class codec:
    """codec::encode_value / decode_value / roundtrip / choose_precision (codec.hpp:23-37)."""

    @staticmethod
    def encode(values, p3, ctx=None) -> np.ndarray:
        ctx = ctx or default_context()
        x = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        out = np.zeros(x.size * p3, dtype=np.uint8)
        _check(lib().lzb_codec_encode(ctx.h, x.size, _ptr(x), p3, _ptr(out)))
        return out

    @staticmethod
    def decode(data, p3, ctx=None) -> np.ndarray:
        ctx = ctx or default_context()
        b = np.ascontiguousarray(data, dtype=np.uint8).reshape(-1)
        out = np.zeros(b.size // p3)
        _check(lib().lzb_codec_decode(ctx.h, out.size, _ptr(b), p3, _ptr(out)))
        return out

    @staticmethod
    def encode_value(x, p3, ctx=None) -> bytes:
        return codec.encode([x], p3, ctx).tobytes() if p3 else b""

    @staticmethod
    def decode_value(data, p3, ctx=None) -> float:
        return float(codec.decode(np.frombuffer(bytes(data), np.uint8), p3, ctx)[0])

    @staticmethod
    def roundtrip(values, p3, ctx=None):
        if p3 == 0:
            return np.zeros(np.size(values))
        return codec.decode(codec.encode(values, p3, ctx), p3, ctx)

    @staticmethod
    def choose_precision_records(values, entries, delta_max, ctx=None) -> np.ndarray:
        ctx = ctx or default_context()
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        nrec = v.size // entries
        out = np.zeros(nrec, dtype=np.int32)
        _check(lib().lzb_codec_choose_precision(ctx.h, nrec, entries, _ptr(v), delta_max, _ptr(out)))
        return out

    @staticmethod
    def choose_precision(values, delta_max, ctx=None) -> int:
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        return int(codec.choose_precision_records(v, v.size, delta_max, ctx)[0])


def scatter_row(element, corner, stencil=None) -> np.ndarray:
    """scatter_row (element.cpp:39-45): stencil9 += the element row of `corner`."""
    e = np.ascontiguousarray(element, dtype=np.float64).reshape(16)
    st = np.zeros(9) if stencil is None else stencil
    _check(lib().lzb_scatter_row(_ptr(e), corner, _ptr(st)))
    return st


def pack_header(p1, p2, p3) -> int:
    return lib().lzb_pack_header(p1, 1 if p2 else 0, p3)


def unpack_header(h):
    cls, p2, p3 = C.c_int(), C.c_int(), C.c_int()
    _check(lib().lzb_unpack_header(h, C.byref(cls), C.byref(p2), C.byref(p3)))
    return cls.value, bool(p2.value), p3.value


# ------------------------------------------------------------------ transfer
def geometric_prolongation() -> np.ndarray:
    out = np.zeros(64)
    lib().lzb_geometric_prolongation(_ptr(out))
    return out


def galerkin_coarse_element(children, P=None, ctx=None) -> np.ndarray:
    """Batched R A_patch P (transfer.hpp:31): children (..., 9, 16), P (..., 64) or None."""
    ctx = ctx or default_context()
    ch = np.ascontiguousarray(children, dtype=np.float64).reshape(-1, 144)
    Pp = None if P is None else np.ascontiguousarray(P, dtype=np.float64).reshape(-1, 64)
    out = np.zeros((ch.shape[0], 16))
    _check(lib().lzb_galerkin(ctx.h, ch.shape[0], _ptr(ch), None if Pp is None else _ptr(Pp), _ptr(out)))
    return out


def boxmg_prolongation(children, ctx=None):
    ctx = ctx or default_context()
    ch = np.ascontiguousarray(children, dtype=np.float64).reshape(-1, 144)
    P = np.zeros((ch.shape[0], 64))
    fb = np.zeros(ch.shape[0], np.int32)
    _check(lib().lzb_boxmg(ctx.h, ch.shape[0], _ptr(ch), _ptr(P), _ptr(fb)))
    return P, fb


# ------------------------------------------------------------------ grid
def make_desc(depth=2, field: Field | None = None, rhs: float = 0.0, rhs_kind="constant",
              rhs_scale=2 * np.pi ** 2, delta_max=1e-8, solver="adafac-pi", omega=0.7, target=1e-10,
              divergence=1e2, max_cycles=500, assembly="adaptive", termination_c=0.01, schedule="increment",
              n_max=0, integration="exact", transfer="geometric", gating=True, throttle=0, seed=0,
              concurrent=False, plane_width=0, fixed_p3=0, start_geometric=False, forced_fraction=0.0,
              forced_n=8) -> GridDesc:
    d = GridDesc()
    d.dim = 2
    d.depth = depth
    d.field = field if field is not None else field_constant(1.0)
    d.rhs = Rhs(kind=T.RHS_SINPROD, value=rhs_scale) if rhs_kind == "sinprod" else Rhs(kind=T.RHS_CONSTANT,
                                                                                      value=rhs)
    d.delta_max = delta_max
    d.variant = {"additive": T.ADDITIVE, "adafac-jac": T.ADAFAC_JAC, "adafac-pi": T.ADAFAC_PI}[solver]
    d.max_cycles = max_cycles
    d.omega, d.target, d.divergence = omega, target, divergence
    d.mode = {"eager": T.EAGER, "lazy": T.LAZY, "adaptive": T.ADAPTIVE, "anarchic": T.ANARCHIC}[assembly]
    d.schedule = T.SCHEDULE_DOUBLE if schedule == "double" else T.SCHEDULE_INCREMENT
    d.termination_c = termination_c
    d.n_max = n_max
    d.integration = T.INTEGRATE_FAST if integration == "fast" else T.INTEGRATE_EXACT
    d.transfer = T.BOXMG if transfer == "boxmg" else T.GEOMETRIC
    d.policy = T.ALWAYS
    d.gating = 1 if gating else 0
    d.concurrent = 1 if concurrent else 0
    d.throttle = throttle
    d.noise_seed = seed
    d.plane_width = plane_width
    d.fixed_p3 = fixed_p3
    d.start_geometric = 1 if start_geometric else 0
    d.forced_fraction = forced_fraction
    d.forced_n = forced_n
    return d


# grids still alive at interpreter exit are destroyed before the CUDA runtime
# tears down (objects kept alive by tracebacks would otherwise be freed late)
_live_grids: "weakref.WeakSet" = weakref.WeakSet()


@atexit.register
def _close_live_grids():
    for g in list(_live_grids):
        g.close()


class Grid:
    """Mesh + CellStream + Assembler + AdditiveSolver of one regular 2D
    spacetree, resident on the GPU (solver.hpp:72-126 semantics)."""

    def __init__(self, desc: GridDesc, noise_seed: int | None = None, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.desc = desc
        self.depth = desc.depth
        h = C.c_void_p()
        _check(lib().lzb_grid_create(self.ctx.h, C.byref(desc), C.byref(h)))
        self.h = h
        _live_grids.add(self)
        if noise_seed is not None:
            self.init_noise(noise_seed)

    def close(self):
        if getattr(self, "h", None):
            if _lib is not None:
                _lib.lzb_grid_destroy(self.h)
            self.h = None

    __del__ = close

    def init_noise(self, seed):
        _check(lib().lzb_grid_init_noise(self.h, seed))

    def eager_setup(self):
        _check(lib().lzb_grid_eager_setup(self.h))

    def assemble_fixed(self, n):
        _check(lib().lzb_grid_assemble_fixed(self.h, n))

    def step(self) -> dict:
        r = CycleReport()
        _check(lib().lzb_grid_step(self.h, C.byref(r)))
        return report_dict(r)

    def vcycle(self, nu=1) -> dict:
        """One multiplicative V(nu, nu) cycle (lzb_grid_vcycle)."""
        r = CycleReport()
        _check(lib().lzb_grid_vcycle(self.h, nu, C.byref(r)))
        return report_dict(r)

    def run(self, cap=100000):
        arr = (CycleReport * cap)()
        n = C.c_int()
        _check(lib().lzb_grid_run(self.h, arr, cap, C.byref(n)))
        return [report_dict(arr[i]) for i in range(min(cap, n.value))]

    # slab-distributed cycle (parallel.py drives the phases and the exchanges)
    def dist_cycle(self) -> dict:
        """One slab-distributed cycle over the context's NCCL communicator
        (this rank's slab; the C++ data plane, csrc/dist.cpp)."""
        r = CycleReport()
        _check(lib().lzb_grid_dist_cycle(self.h, C.byref(r)))
        return report_dict(r)

    def dist_assemble(self, n):
        _check(lib().lzb_grid_dist_assemble(self.h, n))

    def set_slab(self, v0, v1):
        _check(lib().lzb_grid_set_slab(self.h, v0, v1))

    def dist_phase(self, phase, flags=0):
        _check(lib().lzb_grid_dist_phase(self.h, phase, flags))

    def dist_result(self):
        n2 = C.c_double()
        slots = (C.c_uint64 * 20)()
        _check(lib().lzb_grid_dist_result(self.h, C.byref(n2), slots))
        return n2.value, list(slots)

    def dist_report(self, norm2, slots) -> dict:
        arr = (C.c_uint64 * 20)(*[int(x) for x in slots])
        r = CycleReport()
        _check(lib().lzb_grid_dist_report(self.h, float(norm2), arr, C.byref(r)))
        return report_dict(r)

    def pass_(self, which):
        v = C.c_double()
        _check(lib().lzb_grid_pass(self.h, which, C.byref(v)))
        return v.value

    assembly_pass = lambda self: self.pass_(0)  # noqa: E731
    residual_pass = lambda self: self.pass_(1)  # noqa: E731

    def drain(self) -> int:
        """TaskPool::drain_all: finish every pending assembly task (commits an
        in-flight concurrent batch first); returns the tasks left (0)."""
        return int(self.pass_(7))

    def cycle(self):
        return lib().lzb_grid_cycle(self.h)

    def vertices(self, level, field):
        N = 3 ** level
        out = np.zeros((N + 1) * (N + 1))
        _check(lib().lzb_grid_vertices(self.h, level, field, _ptr(out), 0))
        return out.reshape(N + 1, N + 1)

    def set_vertices(self, level, field, values):
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        _check(lib().lzb_grid_vertices(self.h, level, field, _ptr(v), 1))

    def cells(self, level):
        N = 3 ** level
        ops = np.zeros((N * N, 16))
        p1 = np.zeros(N * N, np.int32)
        n = np.zeros(N * N, np.int32)
        p3 = np.zeros(N * N, np.int32)
        ep = np.zeros(N * N, np.uint32)
        _check(lib().lzb_grid_cells(self.h, level, _ptr(ops), _ptr(p1), _ptr(n), _ptr(p3), _ptr(ep)))
        return dict(ops=ops, p1=p1, n=n, p3=p3, epoch=ep)

    def transfer(self, level, cx, cy):
        out = np.zeros(64)
        _check(lib().lzb_grid_transfer(self.h, level, cx, cy, _ptr(out)))
        return out

    def assemble_fixed_raw(self, n):
        """assemble_fixed(n) through the same fused kernel; returns the
        integrated leaf matrices before compression, (N*N, 16)."""
        N = 3 ** self.desc.depth
        out = np.zeros((N * N, 16))
        _check(lib().lzb_grid_assemble_fixed_raw(self.h, n, _ptr(out)))
        return out

    def vertex_stencils(self, level, require_payload=False):
        """assemble_vertex_stencil of every vertex: ((N+1)^2, 9), Stencil9 order."""
        N = 3 ** level
        out = np.zeros(((N + 1) * (N + 1), 9))
        _check(lib().lzb_grid_vertex_stencils(self.h, level, 1 if require_payload else 0, _ptr(out)))
        return out

    def publish_level(self, level, mats, n, p1):
        m = np.ascontiguousarray(mats, dtype=np.float64).reshape(-1)
        nn = np.ascontiguousarray(np.broadcast_to(np.asarray(n, np.int32), (9 ** level,)))
        _check(lib().lzb_grid_publish_level(self.h, level, _ptr(m), _ptr(nn), p1))

    def publish_element(self, level, cx, cy, m, n, p1):
        m = np.ascontiguousarray(m, dtype=np.float64)
        _check(lib().lzb_grid_publish_element(self.h, level, cx, cy, _ptr(m), n, p1))

    def adaptive_step(self, level, cx, cy):
        _check(lib().lzb_grid_adaptive_step(self.h, level, cx, cy))

    def stats(self) -> CompressionStats:
        s = CompressionStats()
        _check(lib().lzb_grid_stats(self.h, C.byref(s)))
        return s

    def stream_image(self, out: np.ndarray | None = None):
        """CellStream::save byte image. With `out` (a uint8 host array, ideally
        pinned) the image is copied straight into it and its size returned."""
        size = C.c_int64()
        if out is not None:
            _check(lib().lzb_grid_stream_image(self.h, _ptr(out), out.size, C.byref(size)))
            return size.value
        _check(lib().lzb_grid_stream_image(self.h, None, 0, C.byref(size)))
        buf = np.zeros(size.value, np.uint8)
        _check(lib().lzb_grid_stream_image(self.h, _ptr(buf), buf.size, C.byref(size)))
        return buf[: size.value].tobytes()

    def assemble_stream(self, n, out: np.ndarray, timeline: np.ndarray | None = None) -> int:
        """assemble_fixed(n) + stream_image(out), pipelined per band of level-1
        subtrees (lzb_grid_assemble_stream); returns the image size."""
        size = C.c_int64()
        _check(lib().lzb_grid_assemble_stream(self.h, n, _ptr(out), out.size, C.byref(size),
                                              None if timeline is None else _ptr(timeline)))
        return size.value

    def stream_image_size(self) -> int:
        size = C.c_int64()
        _check(lib().lzb_grid_stream_image(self.h, None, 0, C.byref(size)))
        return size.value

    def load_image(self, data: bytes):
        b = np.frombuffer(data, np.uint8).copy()
        _check(lib().lzb_grid_stream_load(self.h, _ptr(b), b.size))

    def save(self, path):
        _check(lib().lzb_grid_save(self.h, str(path).encode()))

    def load(self, path):
        _check(lib().lzb_grid_load(self.h, str(path).encode()))

    def pending(self) -> int:
        return lib().lzb_grid_pending(self.h)

    def device_view(self, level, field) -> int:
        p = C.c_void_p()
        _check(lib().lzb_grid_device_view(self.h, level, field, C.byref(p)))
        return p.value

    def time_kernel(self, what, reps=20) -> float:
        """Average device ms of one leaf-level kernel (TK_* id), CUDA events on the solve stream."""
        ms = C.c_double()
        _check(lib().lzb_grid_time_kernel(self.h, what, reps, C.byref(ms)))
        return ms.value


# ---------------------------------------------------------------------- 3D
# Restated 3D extension (BASELINE configs[2..4]; the reference is 2D only).
def grf_table(seed=1, n=64, ell=0.05, sigma2=1.0) -> np.ndarray:
    """Gaussian random field g on a periodic n^3 grid (lzb_grf_table)."""
    out = np.zeros((n, n, n))
    _check(lib().lzb_grf_table(seed, n, ell, sigma2, _ptr(out)))
    return out


def field3_grf(table: np.ndarray) -> "T.Field3":
    """eps = exp(g), g trilinear in the periodic table (kept alive by the field)."""
    t = np.ascontiguousarray(table, dtype=np.float64)
    f = T.Field3(kind=T.F3_GRF, grf_n=t.shape[0], value=1.0, grf=t.ctypes.data)
    f._table = t
    return f


def field3_constant(value=1.0) -> "T.Field3":
    return T.Field3(kind=T.F3_CONSTANT, grf_n=0, value=value, grf=None)


def field3_extruded(f2: Field) -> "T.Field3":
    return T.Field3(kind=T.F3_EXTRUDED, grf_n=0, value=1.0, grf=None, xy=f2)


def field3_sphere(centre=(0.5, 0.5, 0.5), radius=0.25, width=0.01, eps_in=100.0, eps_out=1.0) -> "T.Field3":
    """BASELINE configs[3]: eps_in inside the sphere, eps_out outside, a tanh
    interface whose 10-90 % transition spans `width` (lzb_types.h)."""
    f = T.Field3(kind=T.F3_SPHERE, grf_n=0, value=1.0, grf=None)
    f.centre[:] = [float(c) for c in centre]
    f.radius, f.width, f.eps_in, f.eps_out = radius, width, eps_in, eps_out
    return f


class Tree3:
    """BASELINE configs[3] assembly on a 3D adaptive spacetree (lzb_tree3_*):
    level lmax where a cell meets the field's sphere, lbase elsewhere."""

    def __init__(self, lbase, lmax, field, delta_max=1e-8, fixed_p3=0, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.field = field
        h = C.c_void_p()
        _check(lib().lzb_tree3_create(self.ctx.h, lbase, lmax, C.byref(field), delta_max, fixed_p3, C.byref(h)))
        self.h = h
        per = np.zeros(8, np.int64)
        tot = C.c_int64()
        _check(lib().lzb_tree3_counts(self.h, _ptr(per), C.byref(tot)))
        self.per_level, self.n_leaves = per, tot.value

    def close(self):
        if getattr(self, "h", None):
            if _lib is not None:
                _lib.lzb_tree3_destroy(self.h)
            self.h = None

    __del__ = close

    def assemble(self, n):
        _check(lib().lzb_tree3_assemble(self.h, n))

    def set_shell(self, band) -> int:
        c = C.c_int64()
        _check(lib().lzb_tree3_set_shell(self.h, band, C.byref(c)))
        return c.value

    def assemble_shell(self, n):
        _check(lib().lzb_tree3_assemble_shell(self.h, n))

    def stats(self) -> CompressionStats:
        s = CompressionStats()
        _check(lib().lzb_tree3_stats(self.h, C.byref(s)))
        return s

    def init_cycle(self, solver="adafac-pi", omega=0.6, rhs_scale=3 * np.pi ** 2, seed=42, max_cycles=100,
                   target=1e-10):
        variant = {"additive": T.ADDITIVE, "adafac-pi": T.ADAFAC_PI, "adafac-jac": T.ADAFAC_JAC}[solver]
        _check(lib().lzb_tree3_init_cycle(self.h, variant, omega, rhs_scale, seed, max_cycles, target))
        self.lmax = int(np.nonzero(self.per_level)[0].max())

    def refresh_ops(self):
        _check(lib().lzb_tree3_refresh_ops(self.h))

    def refine(self, radius, n) -> int:
        """Grow the refinement ball to `radius` (new leaves assembled at n, the
        cycle state carried over); returns the number of new leaves."""
        k = C.c_int64()
        _check(lib().lzb_tree3_refine(self.h, radius, n, C.byref(k)))
        per = np.zeros(8, np.int64)
        tot = C.c_int64()
        _check(lib().lzb_tree3_counts(self.h, _ptr(per), C.byref(tot)))
        self.per_level, self.n_leaves = per, tot.value
        return k.value

    def step(self) -> dict:
        r = CycleReport()
        _check(lib().lzb_tree3_step(self.h, C.byref(r)))
        return report_dict(r)

    def vertices(self, level, field) -> np.ndarray:
        n = 3 ** level + 1
        out = np.zeros((n, n, n))
        _check(lib().lzb_tree3_vertices(self.h, level, field, _ptr(out)))
        return out

    def cells(self, first, count):
        ops = np.zeros((count, 8, 8))
        p3, n = np.zeros(count, np.int32), np.zeros(count, np.int32)
        lxyz = np.zeros((count, 4), np.int32)
        _check(lib().lzb_tree3_cells(self.h, first, count, _ptr(ops), _ptr(p3), _ptr(n), _ptr(lxyz)))
        return ops, p3, n, lxyz


def integrate_elements3(field, x0, y0, z0, h, n, ctx: Context | None = None) -> np.ndarray:
    """Batched 3D element integration: (count, 8, 8) trilinear stiffness matrices."""
    ctx = ctx or default_context()
    x0 = np.ascontiguousarray(x0, dtype=np.float64).reshape(-1)
    cnt = x0.size
    y0, z0, h = (np.ascontiguousarray(np.broadcast_to(v, (cnt,)), dtype=np.float64) for v in (y0, z0, h))
    n = np.ascontiguousarray(np.broadcast_to(n, (cnt,)), dtype=np.int32)
    out = np.zeros((cnt, 8, 8))
    _check(lib().lzb_integrate_elements3(ctx.h, C.byref(field), cnt, _ptr(x0), _ptr(y0), _ptr(z0), _ptr(h),
                                         _ptr(n), _ptr(out)))
    return out


class Grid3:
    """Leaves of a regular 3D grid (3^depth cells per axis): fixed-p assembly
    with the 64-entry record coding (lzb_grid3_*)."""

    def __init__(self, depth, field, delta_max=1e-8, fixed_p3=0, plane_width=0, ctx: Context | None = None,
                 slab: tuple[int, int] | None = None):
        """slab = (rank, world): store only the leaf operators of that z-slab's
        layers (lzb_grid3_create_slab); such a grid runs the distributed cycle."""
        self.ctx = ctx or default_context()
        self.depth, self.field = depth, field
        self.N = 3 ** depth
        self.plane_width = plane_width
        h = C.c_void_p()
        if slab is None:
            _check(lib().lzb_grid3_create_planes(self.ctx.h, depth, C.byref(field), delta_max, fixed_p3, plane_width,
                                                 C.byref(h)))
        else:
            _check(lib().lzb_grid3_create_slab(self.ctx.h, depth, C.byref(field), delta_max, fixed_p3, plane_width,
                                               slab[1], slab[0], C.byref(h)))
        self.h = h

    def leaf_storage(self):
        """(resident bytes of the leaf operators, first and end stored cell layer)"""
        b, z0, z1 = C.c_int64(), C.c_int(), C.c_int()
        _check(lib().lzb_grid3_leaf_storage(self.h, C.byref(b), C.byref(z0), C.byref(z1)))
        return b.value, z0.value, z1.value

    def assemble_planes(self, n, cz0, cz1):
        _check(lib().lzb_grid3_assemble_planes(self.h, n, cz0, cz1))

    def galerkin_planes(self, level, pz0, pz1):
        _check(lib().lzb_grid3_galerkin_planes(self.h, level, pz0, pz1))

    def coarse_below(self, level):
        _check(lib().lzb_grid3_coarse_below(self.h, level))

    def level_ops_ptr(self, level) -> int:
        p = C.c_void_p()
        _check(lib().lzb_grid3_level_ops(self.h, level, C.byref(p)))
        return p.value

    def time_kernel(self, what, reps=10) -> float:
        """Average device ms of one leaf-level cycle kernel (TK_* id), CUDA events on the solve stream."""
        ms = C.c_double()
        _check(lib().lzb_grid3_time_kernel(self.h, what, reps, C.byref(ms)))
        return ms.value

    def leaf_bytes_per_cell(self) -> int:
        """Resident bytes of one leaf operator: 27 FP64 class values, or 27
        plane words of plane_width bytes + eps(centre) + p3."""
        return 27 * 8 if not self.plane_width else 27 * self.plane_width + 8 + 1

    def close(self):
        if getattr(self, "h", None):
            if _lib is not None:
                _lib.lzb_grid3_destroy(self.h)
            self.h = None

    __del__ = close

    def assemble_fixed(self, n):
        _check(lib().lzb_grid3_assemble_fixed(self.h, n))

    def stats(self) -> CompressionStats:
        s = CompressionStats()
        _check(lib().lzb_grid3_stats(self.h, C.byref(s)))
        return s

    def init_cycle(self, solver="adafac-pi", omega=0.6, rhs_scale=3 * np.pi ** 2, seed=42, max_cycles=100,
                   target=1e-10):
        variant = {"additive": T.ADDITIVE, "adafac-jac": T.ADAFAC_JAC, "adafac-pi": T.ADAFAC_PI}[solver]
        _check(lib().lzb_grid3_init_cycle(self.h, variant, omega, rhs_scale, seed, max_cycles, target))

    def step(self) -> dict:
        r = CycleReport()
        _check(lib().lzb_grid3_step(self.h, C.byref(r)))
        return report_dict(r)

    def vcycle(self, nu=2) -> dict:
        """One multiplicative V(nu, nu) cycle (lzb_grid3_vcycle)."""
        r = CycleReport()
        _check(lib().lzb_grid3_vcycle(self.h, nu, C.byref(r)))
        return report_dict(r)

    # slab-distributed cycle (parallel.dist_cycle3)
    def dist_cycle(self) -> dict:
        """One z-slab-distributed cycle over the context's NCCL communicator
        (the C++ data plane, csrc/dist.cpp; after init_cycle)."""
        r = CycleReport()
        _check(lib().lzb_grid3_dist_cycle(self.h, C.byref(r)))
        return report_dict(r)

    def dist_assemble(self, n):
        """z-slab sharded assembly + the level-(D-1) class-plane exchange (NCCL)."""
        _check(lib().lzb_grid3_dist_assemble(self.h, n))

    def set_slab(self, v0, v1):
        _check(lib().lzb_grid3_set_slab(self.h, v0, v1))

    def dist_phase(self, phase, flags=0):
        _check(lib().lzb_grid3_dist_phase(self.h, phase))

    def dist_result(self):
        n2 = C.c_double()
        _check(lib().lzb_grid3_dist_result(self.h, C.byref(n2)))
        return n2.value, [0] * 20

    def dist_report(self, norm2, slots=None) -> dict:
        r = CycleReport()
        _check(lib().lzb_grid3_dist_report(self.h, float(norm2), C.byref(r)))
        return report_dict(r)

    def device_view(self, level, field) -> int:
        p = C.c_void_p()
        _check(lib().lzb_grid3_device_view(self.h, level, field, C.byref(p)))
        return p.value

    def vertices(self, level, field):
        n = 3 ** level + 1
        out = np.zeros((n, n, n))  # [z][y][x]
        _check(lib().lzb_grid3_vertices(self.h, level, field, _ptr(out)))
        return out

    def cells(self, first, count):
        ops = np.zeros((count, 8, 8))
        p3 = np.zeros(count, np.int32)
        _check(lib().lzb_grid3_cells(self.h, first, count, _ptr(ops), _ptr(p3)))
        return ops, p3


# ------------------------------------------------------------------ experiment
def run_experiment(cfg_text: str):
    """run_experiment(parse_config_file) (experiment.hpp:75,89); returns (exit_code, reports)."""
    ec, nc = C.c_int(), C.c_int()
    _check(lib().lzb_run_experiment_text(cfg_text.encode(), C.byref(ec), C.byref(nc)))
    arr = (CycleReport * max(nc.value, 1))()
    cnt = C.c_int()
    lib().lzb_last_reports(arr, max(nc.value, 1), C.byref(cnt))
    return ec.value, [report_dict(arr[i]) for i in range(nc.value)]


def run_experiment_file(path: str):
    ec, nc = C.c_int(), C.c_int()
    _check(lib().lzb_run_experiment_file(str(path).encode(), C.byref(ec), C.byref(nc)))
    return ec.value, nc.value


def config_keys(cfg_text: str) -> dict:
    buf = C.create_string_buffer(1 << 16)
    _check(lib().lzb_config_keys(cfg_text.encode(), buf, len(buf)))
    out = {}
    for line in buf.value.decode().splitlines():
        k, v = line.split(" = ", 1)
        out[k] = v
    return out


def emit_table(paths) -> str:
    buf = C.create_string_buffer(1 << 20)
    _check(lib().lzb_emit_table("\n".join(str(p) for p in paths).encode(), buf, len(buf)))
    return buf.value.decode()


def compare_runs(a, b) -> str:
    buf = C.create_string_buffer(1 << 16)
    _check(lib().lzb_compare_runs(str(a).encode(), str(b).encode(), buf, len(buf)))
    return buf.value.decode()

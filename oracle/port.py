"""ctypes view of the C restatement (oracle/build/liblzb_oracle.so).

TEST INFRASTRUCTURE ONLY: the parity checker for the B200 product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from oracle.types import CompressionStats, CycleReport, Field, report_dict
from paper_2005_03606_b200 import _types as T

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liblzb_oracle.so")

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.orc_last_error.restype = C.c_char_p
        L.orc_field_eval.restype = C.c_double
        L.orc_field_eval.argtypes = [C.POINTER(Field), C.c_double, C.c_double]
        L.orc_field_checkerboard.argtypes = [C.POINTER(Field), C.c_uint64, C.c_int]
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_subcell_stiffness.argtypes = [C.c_double] * 4 + [vp]
        L.orc_integrate_element.argtypes = [C.POINTER(Field), C.c_double, C.c_double, C.c_double, C.c_int, vp]
        L.orc_integrate_level.argtypes = [C.POINTER(Field), C.c_int, C.c_int, vp, C.c_int]
        L.orc_publish_level.argtypes = [vp, C.c_int, vp, vp, C.c_int32]
        L.orc_encode_value.argtypes = [C.c_double, C.c_int, vp]
        L.orc_decode_value.restype = C.c_double
        L.orc_decode_value.argtypes = [vp, C.c_int]
        L.orc_choose_precision.argtypes = [vp, C.c_int64, C.c_double]
        L.orc_pack_header.restype = C.c_uint8
        L.orc_pack_header.argtypes = [C.c_int32, C.c_int, C.c_int]
        L.orc_unpack_header.argtypes = [C.c_uint8] + [C.POINTER(C.c_int)] * 3
        L.orc_geometric.argtypes = [vp]
        L.orc_galerkin.argtypes = [vp, vp, vp]
        L.orc_boxmg.argtypes = [vp, vp]
        L.orc_grid_create.restype = vp
        L.orc_grid_create.argtypes = [C.POINTER(T.GridDesc)]
        L.orc_grid_destroy.argtypes = [vp]
        L.orc_init_noise.argtypes = [vp, C.c_uint64]
        L.orc_eager_setup.argtypes = [vp]
        L.orc_assemble_fixed.argtypes = [vp, C.c_int]
        L.orc_step.argtypes = [vp, C.POINTER(CycleReport)]
        L.orc_run.argtypes = [vp, vp, C.c_int, C.POINTER(C.c_int)]
        L.orc_pass.argtypes = [vp, C.c_int, C.POINTER(C.c_double)]
        L.orc_vertices.argtypes = [vp, C.c_int, C.c_int, vp, C.c_int]
        L.orc_cells.argtypes = [vp, C.c_int, vp, vp, vp, vp, vp]
        L.orc_publish_element.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int32]
        L.orc_adaptive_step.argtypes = [vp, C.c_int, C.c_int, C.c_int]
        L.orc_stats.argtypes = [vp, C.POINTER(CompressionStats)]
        L.orc_stream_image.restype = C.c_int64
        L.orc_stream_image.argtypes = [vp, vp, C.c_int64]
        L.orc_stream_load.argtypes = [vp, vp, C.c_int64]
        L.orc_cycle.argtypes = [vp]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------------ config keys
DEFAULT_KEYS = {  # ExperimentConfig defaults, experiment.hpp:14-66
    "setup": "constant", "eps": "1", "theta": "1", "eps-low": "0.001", "rhs": "0", "seed": "0",
    "depth": "2", "solver": "adafac-pi", "omega": "0.7", "target": "1e-10", "divergence": "100",
    "max-cycles": "500", "assembly": "adaptive", "termination-c": "0.01", "transfer": "geometric",
    "coarse-recompute": "always", "gating": "on", "compression-threshold": "1e-08", "workers": "1",
    "throttle": "0",
}


def parse_keys(text: str) -> dict:
    keys = dict(DEFAULT_KEYS)
    for line in text.splitlines():
        line = line.split("#")[0].strip()
        if not line:
            continue
        k, v = line.split("=", 1)
        keys[k.strip()] = v.strip()
    return keys


def field_from_keys(k: dict) -> Field:
    s = k["setup"]
    if s == "theta":
        return T.field_theta(float(k["theta"]))
    if s == "quadrant":
        return T.field_quadrant(float(k["eps-low"]))
    if s == "checkerboard":
        f = Field()
        lib().orc_field_checkerboard(C.byref(f), int(k.get("field-seed", "1")), int(k.get("blocks", "8")))
        return f
    if s == "sinusoid":
        return T.field_sinusoid(float(k.get("amp", "0.9")), float(k.get("freq", "6")))
    return T.field_constant(float(k["eps"]))


def desc_from_keys(k: dict) -> T.GridDesc:
    d = T.GridDesc()
    d.dim = 2
    d.depth = int(k["depth"])
    d.field = field_from_keys(k)
    if k.get("rhs-kind", "constant") == "sinprod":
        d.rhs = T.Rhs(kind=T.RHS_SINPROD, value=float(k.get("rhs-scale", repr(2 * np.pi ** 2))))
    else:
        d.rhs = T.Rhs(kind=T.RHS_CONSTANT, value=float(k["rhs"]))
    d.delta_max = float(k["compression-threshold"])
    d.variant = {"additive": T.ADDITIVE, "adafac-jac": T.ADAFAC_JAC, "adafac-pi": T.ADAFAC_PI}[k["solver"]]
    d.max_cycles = int(k["max-cycles"])
    d.omega = float(k["omega"])
    d.target = float(k["target"])
    d.divergence = float(k["divergence"])
    d.mode = {"eager": T.EAGER, "lazy": T.LAZY, "adaptive": T.ADAPTIVE, "anarchic": T.ANARCHIC}[k["assembly"]]
    d.schedule = T.SCHEDULE_DOUBLE if k.get("schedule", "increment") == "double" else T.SCHEDULE_INCREMENT
    d.termination_c = float(k["termination-c"])
    d.n_max = int(k.get("n-max", "0"))
    d.integration = T.INTEGRATE_FAST if k.get("integration", "exact") == "fast" else T.INTEGRATE_EXACT
    d.transfer = T.BOXMG if k["transfer"] == "boxmg" else T.GEOMETRIC
    d.policy = T.RIPPLE if k["coarse-recompute"] == "ripple" else T.ALWAYS
    d.gating = 1 if k["gating"] in ("on", "true", "1") else 0
    d.concurrent = 0
    d.throttle = int(k["throttle"])
    d.noise_seed = int(k["seed"])
    d.boundary_value = 0.0
    d.start_geometric = 1 if k.get("start", "sample") == "geometric" else 0
    d.forced_fraction = float(k.get("forced-task-fraction", "0"))
    d.forced_n = int(k.get("forced-task-n", "8"))
    return d


# ------------------------------------------------------------------ primitives
def integrate_element(field: Field, x0, y0, h, n):
    out = np.zeros(16)
    lib().orc_integrate_element(C.byref(field), x0, y0, h, n, _ptr(out))
    return out


def integrate_level(field: Field, level, n, threads=None):
    """Every cell of a regular level (cy*N+cx, 16 doubles each), the
    reference's integrate_element over disjoint cell ranges on host threads."""
    N = 3 ** level
    out = np.zeros((N * N, 16))
    lib().orc_integrate_level(C.byref(field), level, n, _ptr(out), int(threads or os.cpu_count() or 1))
    return out


def encode_value(x, p3):
    out = np.zeros(8, np.uint8)
    _check(lib().orc_encode_value(float(x), p3, _ptr(out)))
    return out[:p3].copy()


def decode_value(b, p3):
    b = np.ascontiguousarray(b, dtype=np.uint8)
    return lib().orc_decode_value(_ptr(b), p3)


def choose_precision(v, delta):
    v = np.ascontiguousarray(v, dtype=np.float64)
    r = lib().orc_choose_precision(_ptr(v), v.size, delta)
    if r < 0:
        raise OracleError(-r, "non-finite")
    return r


def geometric():
    P = np.zeros(64)
    lib().orc_geometric(_ptr(P))
    return P


def galerkin(children, P):
    ch = np.ascontiguousarray(children, dtype=np.float64).reshape(144)
    P = np.ascontiguousarray(P, dtype=np.float64).reshape(64)
    out = np.zeros(16)
    lib().orc_galerkin(_ptr(ch), _ptr(P), _ptr(out))
    return out


def boxmg(children):
    ch = np.ascontiguousarray(children, dtype=np.float64).reshape(144)
    out = np.zeros(64)
    fb = lib().orc_boxmg(_ptr(ch), _ptr(out))
    return out, fb


class Grid:
    """Restated Mesh + CellStream + Assembler + AdditiveSolver (regular 2D)."""

    def __init__(self, desc: T.GridDesc, noise_seed=None):
        self.desc = desc
        self.depth = desc.depth
        self.h = lib().orc_grid_create(C.byref(desc))
        if not self.h:
            raise OracleError(T.ERR_INVALID, lib().orc_last_error().decode())
        if noise_seed is not None:
            lib().orc_init_noise(self.h, noise_seed)

    @classmethod
    def from_text(cls, text: str, noise=True):
        k = parse_keys(text)
        d = desc_from_keys(k)
        return cls(d, int(k["seed"]) if noise else None)

    def close(self):
        if getattr(self, "h", None):
            lib().orc_grid_destroy(self.h)
            self.h = None

    __del__ = close

    def eager_setup(self):
        _check(lib().orc_eager_setup(self.h))

    def assemble_fixed(self, n):
        _check(lib().orc_assemble_fixed(self.h, n))

    def step(self):
        r = CycleReport()
        _check(lib().orc_step(self.h, C.byref(r)))
        return report_dict(r)

    def run(self, cap=100000):
        arr = (CycleReport * cap)()
        n = C.c_int()
        _check(lib().orc_run(self.h, arr, cap, C.byref(n)))
        return [report_dict(arr[i]) for i in range(min(cap, n.value))]

    def pass_(self, which):
        v = C.c_double()
        _check(lib().orc_pass(self.h, which, C.byref(v)))
        return v.value

    def vertices(self, level, field):
        N = 3 ** level
        out = np.zeros((N + 1) * (N + 1))
        _check(lib().orc_vertices(self.h, level, field, _ptr(out), 0))
        return out.reshape(N + 1, N + 1)

    def set_vertices(self, level, field, values):
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        _check(lib().orc_vertices(self.h, level, field, _ptr(v), 1))

    def cells(self, level):
        N = 3 ** level
        ops = np.zeros((N * N, 16))
        p1 = np.zeros(N * N, np.int32)
        n = np.zeros(N * N, np.int32)
        p3 = np.zeros(N * N, np.int32)
        ep = np.zeros(N * N, np.uint32)
        _check(lib().orc_cells(self.h, level, _ptr(ops), _ptr(p1), _ptr(n), _ptr(p3), _ptr(ep)))
        return dict(ops=ops, p1=p1, n=n, p3=p3, epoch=ep)

    def publish_element(self, level, cx, cy, m, n, p1):
        m = np.ascontiguousarray(m, dtype=np.float64)
        _check(lib().orc_publish_element(self.h, level, cx, cy, _ptr(m), n, p1))

    def publish_level(self, level, mats, n, p1):
        m = np.ascontiguousarray(mats, dtype=np.float64).reshape(-1)
        nn = np.ascontiguousarray(np.broadcast_to(np.asarray(n, np.int32), (9 ** level,)))
        _check(lib().orc_publish_level(self.h, level, _ptr(m), _ptr(nn), p1))

    def adaptive_step(self, level, cx, cy):
        _check(lib().orc_adaptive_step(self.h, level, cx, cy))

    def stats(self):
        s = CompressionStats()
        _check(lib().orc_stats(self.h, C.byref(s)))
        return s

    def stream_image(self) -> bytes:
        size = lib().orc_stream_image(self.h, None, 0)
        if size < 0:
            _check(-size)
        buf = np.zeros(size, np.uint8)
        lib().orc_stream_image(self.h, _ptr(buf), size)
        return buf.tobytes()

    def load_image(self, data: bytes):
        b = np.frombuffer(data, np.uint8).copy()
        _check(lib().orc_stream_load(self.h, _ptr(b), b.size))

    def cycle(self):
        return lib().orc_cycle(self.h)


# ------------------------------------------------------------------ telemetry rows
CSV_COLUMNS = ("cycle,residual,normalized,dof_updates,dof_updates_total,coarse_updates,pending_tasks,"
               "max_n,avg_n,max_samples,factor_totals,factor_mean,enabled_mask,levels,cells,"
               "dofs_fine_interior,grid_points_total,wall_seconds,status")


def csv_row(r: dict) -> str:
    """experiment.cpp:232-244 number formats."""
    return ("%d,%.17g,%.17g,%d,%d,%d,%d,%d,%.6f,%d,%.6f,%.6f,%d,%d,%d,%d,%d,%.6f,%s" % (
        r["cycle"], r["residual"], r["normalized"], r["dof_updates"], r["dof_updates_total"],
        r["coarse_updates"], r["pending_tasks"], r["max_n"], r["avg_n"], r["max_samples"],
        r["factor_totals"], r["factor_mean"], r["enabled_mask"], r["levels"], r["cells"],
        r["dofs_fine_interior"], r["grid_points_total"], r["wall_seconds"], T.STATUS_NAMES[r["status"]]))


def csv_data_rows(path: str):
    rows = []
    header = False
    for line in open(path):
        line = line.rstrip("\n")
        if not line or line.startswith("#"):
            continue
        if not header:
            header = True
            continue
        rows.append(line)
    return rows

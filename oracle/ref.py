"""ctypes view of the unmodified reference (oracle/_ref/liblazymg_ref.so).

TEST INFRASTRUCTURE ONLY. See oracle/ref_driver.cpp for the exported harness.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from oracle.types import CycleReport, CompressionStats, Field, report_dict

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "liblazymg_ref.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(LIB_PATH)
        L = C.CDLL(LIB_PATH)
        dp = C.POINTER(C.c_double)
        L.ref_last_error.restype = C.c_char_p
        L.ref_eval_field.restype = C.c_double
        L.ref_eval_field.argtypes = [C.POINTER(Field), C.c_double, C.c_double]
        L.ref_integrate_element.argtypes = [C.POINTER(Field), C.c_double, C.c_double, C.c_double, C.c_int, dp]
        L.ref_integrate_cells.argtypes = [C.POINTER(Field), C.c_int, C.c_int64, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_int]
        L.ref_encode_value.argtypes = [C.c_double, C.c_int, C.c_void_p]
        L.ref_decode_value.restype = C.c_double
        L.ref_decode_value.argtypes = [C.c_void_p, C.c_int]
        L.ref_encode_many.argtypes = [C.c_int64, C.c_void_p, C.c_int, C.c_void_p]
        L.ref_decode_many.argtypes = [C.c_int64, C.c_void_p, C.c_int, C.c_void_p]
        L.ref_choose_precision.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.POINTER(C.c_int)]
        L.ref_choose_many.argtypes = [C.c_int64, C.c_int, C.c_void_p, C.c_double, C.c_void_p, C.c_int]
        L.ref_pack_header.restype = C.c_uint8
        L.ref_pack_header.argtypes = [C.c_int32, C.c_int, C.c_int]
        L.ref_unpack_header.argtypes = [C.c_uint8, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_galerkin.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_boxmg.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_rig_create.restype = C.c_void_p
        L.ref_rig_create.argtypes = [C.c_char_p, C.c_int]
        L.ref_rig_destroy.argtypes = [C.c_void_p]
        L.ref_rig_eager_setup.argtypes = [C.c_void_p]
        L.ref_rig_step.argtypes = [C.c_void_p, C.POINTER(CycleReport)]
        L.ref_rig_run.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_int)]
        L.ref_rig_pass.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double)]
        L.ref_rig_vertices.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int]
        L.ref_rig_cells.argtypes = [C.c_void_p, C.c_int] + [C.c_void_p] * 6
        L.ref_rig_transfer.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.ref_rig_publish_element.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int32]
        L.ref_rig_adaptive_step.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        L.ref_rig_stats.argtypes = [C.c_void_p, C.POINTER(CompressionStats)]
        L.ref_rig_save.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_rig_load.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_rig_cycle.argtypes = [C.c_void_p]
        L.ref_run_experiment_text.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_config_keys.argtypes = [C.c_char_p, C.c_char_p, C.c_int64]
        L.ref_emit_table.argtypes = [C.c_char_p, C.c_char_p, C.c_int64]
        L.ref_compare_runs.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int64]
        L.ref_time_integrate.restype = C.c_double
        L.ref_time_integrate.argtypes = [C.POINTER(Field), C.c_int, C.c_int, C.c_int64, C.c_int, dp]
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def integrate_element(field: Field, x0, y0, h, n):
    out = np.zeros(16)
    _check(lib().ref_integrate_element(C.byref(field), x0, y0, h, n, out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def integrate_cells(field: Field, level, cx, cy, n, nthreads=1):
    cx = np.ascontiguousarray(cx, dtype=np.int32)
    cy = np.ascontiguousarray(cy, dtype=np.int32)
    n = np.ascontiguousarray(np.broadcast_to(n, cx.shape), dtype=np.int32)
    out = np.zeros((cx.size, 16))
    _check(lib().ref_integrate_cells(C.byref(field), level, cx.size, _ptr(cx), _ptr(cy), _ptr(n), _ptr(out), nthreads))
    return out


def encode_many(x, p3):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros(x.size * p3, dtype=np.uint8)
    _check(lib().ref_encode_many(x.size, _ptr(x), p3, _ptr(out)))
    return out


def decode_many(b, p3):
    b = np.ascontiguousarray(b, dtype=np.uint8)
    out = np.zeros(b.size // p3)
    lib().ref_decode_many(out.size, _ptr(b), p3, _ptr(out))
    return out


def choose_many(values, entries, delta, nthreads=1):
    v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
    nrec = v.size // entries
    out = np.zeros(nrec, dtype=np.int32)
    _check(lib().ref_choose_many(nrec, entries, _ptr(v), delta, _ptr(out), nthreads))
    return out


def galerkin(children, P):
    ch = np.ascontiguousarray(children, dtype=np.float64).reshape(144)
    P = np.ascontiguousarray(P, dtype=np.float64).reshape(64)
    out = np.zeros(16)
    lib().ref_galerkin(_ptr(ch), _ptr(P), _ptr(out))
    return out


def boxmg(children):
    ch = np.ascontiguousarray(children, dtype=np.float64).reshape(144)
    out = np.zeros(64)
    fb = lib().ref_boxmg(_ptr(ch), _ptr(out))
    return out, fb


def run_experiment_text(text: str):
    ec, nc = C.c_int(), C.c_int()
    _check(lib().ref_run_experiment_text(text.encode(), C.byref(ec), C.byref(nc)))
    return ec.value, nc.value


def emit_table(paths):
    buf = C.create_string_buffer(1 << 20)
    _check(lib().ref_emit_table("\n".join(paths).encode(), buf, len(buf)))
    return buf.value.decode()


class Rig:
    """One reference Mesh + CellStream + TaskPool + Assembler + AdditiveSolver
    built exactly as run_experiment does (experiment.cpp:250-259)."""

    def __init__(self, cfg_text: str, noise: bool = True):
        self.h = lib().ref_rig_create(cfg_text.encode(), 1 if noise else 0)
        if not self.h:
            raise RefError(-1, lib().ref_last_error().decode())
        self.depth = None
        for line in cfg_text.splitlines():
            if line.split("#")[0].strip().startswith("depth"):
                self.depth = int(line.split("=")[1].split("#")[0])
        if self.depth is None:
            self.depth = 2

    def close(self):
        if self.h:
            lib().ref_rig_destroy(self.h)
            self.h = None

    __del__ = close

    def eager_setup(self):
        _check(lib().ref_rig_eager_setup(self.h))

    def step(self):
        r = CycleReport()
        _check(lib().ref_rig_step(self.h, C.byref(r)))
        return report_dict(r)

    def run(self, cap=100000):
        arr = (CycleReport * cap)()
        n = C.c_int()
        _check(lib().ref_rig_run(self.h, arr, cap, C.byref(n)))
        return [report_dict(arr[i]) for i in range(min(n.value, cap))]

    def pass_(self, which):
        v = C.c_double()
        _check(lib().ref_rig_pass(self.h, which, C.byref(v)))
        return v.value

    def vertices(self, level, field):
        N = 3 ** level
        out = np.zeros((N + 1) * (N + 1))
        _check(lib().ref_rig_vertices(self.h, level, field, _ptr(out), 0))
        return out.reshape(N + 1, N + 1)

    def set_vertices(self, level, field, values):
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        _check(lib().ref_rig_vertices(self.h, level, field, _ptr(v), 1))

    def cells(self, level):
        N = 3 ** level
        ops = np.zeros((N * N, 16))
        p1 = np.zeros(N * N, np.int32)
        n = np.zeros(N * N, np.int32)
        p3 = np.zeros(N * N, np.int32)
        ep = np.zeros(N * N, np.uint32)
        slot = np.zeros(N * N, np.int32)
        _check(lib().ref_rig_cells(self.h, level, _ptr(ops), _ptr(p1), _ptr(n), _ptr(p3), _ptr(ep), _ptr(slot)))
        return dict(ops=ops, p1=p1, n=n, p3=p3, epoch=ep, slot=slot)

    def publish_element(self, level, cx, cy, m, n, p1):
        m = np.ascontiguousarray(m, dtype=np.float64)
        _check(lib().ref_rig_publish_element(self.h, level, cx, cy, _ptr(m), n, p1))

    def adaptive_step(self, level, cx, cy):
        _check(lib().ref_rig_adaptive_step(self.h, level, cx, cy))

    def stats(self):
        s = CompressionStats()
        _check(lib().ref_rig_stats(self.h, C.byref(s)))
        return s

    def save(self, path):
        _check(lib().ref_rig_save(self.h, path.encode()))

    def load(self, path):
        _check(lib().ref_rig_load(self.h, path.encode()))

    def cycle(self):
        return lib().ref_rig_cycle(self.h)

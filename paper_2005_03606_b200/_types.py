"""ctypes mirrors of include/lzb_types.h (plain data formats, no device code)."""
from __future__ import annotations

import ctypes as C
import math

# lzb_status
OK, ERR_PROTOCOL, ERR_CORRUPT, ERR_RESOURCE, ERR_INVALID, ERR_IO, ERR_CUDA, ERR_NCCL = range(8)
# lzb_field_kind
FIELD_CONSTANT, FIELD_THETA, FIELD_QUADRANT, FIELD_CHECKER, FIELD_SINUSOID = range(5)
RHS_CONSTANT, RHS_SINPROD = range(2)
ADDITIVE, ADAFAC_JAC, ADAFAC_PI = range(3)
EAGER, LAZY, ADAPTIVE, ANARCHIC = range(4)
GEOMETRIC, BOXMG = range(2)
ALWAYS, RIPPLE = range(2)
CONTINUE, CONVERGED, DIVERGED, TIMEOUT = range(4)
SCHEDULE_INCREMENT, SCHEDULE_DOUBLE = range(2)
INTEGRATE_EXACT, INTEGRATE_FAST = range(2)
P1_BOTTOM, P1_TOP = 0, -1
V_U, V_FL, V_R, V_RHAT, V_UHAT, V_DIAG, V_AUX, V_USNAP = range(8)
# lzb_grid_time_kernel ids (lzb_types.h)
TK_UHAT, TK_RESIDUAL, TK_RESTRICT, TK_JACOBI, TK_PROLONG, TK_PACK, TK_FRONT, TK_BACK = range(8)

STATUS_NAMES = {CONTINUE: "continue", CONVERGED: "converged", DIVERGED: "diverged", TIMEOUT: "timeout"}


class Field(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("blocks", C.c_int32),
        ("value", C.c_double),
        ("theta", C.c_double),
        ("eps_low", C.c_double),
        ("amp", C.c_double),
        ("freq", C.c_double),
        ("table", C.c_double * 64),
    ]


# 3D field kinds (lzb_types.h, restated extension)
F3_CONSTANT, F3_GRF, F3_EXTRUDED, F3_SPHERE = range(4)


class Field3(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("grf_n", C.c_int32),
        ("value", C.c_double),
        ("grf", C.c_void_p),
        ("xy", Field),
        ("centre", C.c_double * 3),
        ("radius", C.c_double),
        ("width", C.c_double),
        ("eps_in", C.c_double),
        ("eps_out", C.c_double),
    ]


class Rhs(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("value", C.c_double)]


class GridDesc(C.Structure):
    _fields_ = [
        ("dim", C.c_int32),
        ("depth", C.c_int32),
        ("field", Field),
        ("rhs", Rhs),
        ("delta_max", C.c_double),
        ("variant", C.c_int32),
        ("max_cycles", C.c_int32),
        ("omega", C.c_double),
        ("target", C.c_double),
        ("divergence", C.c_double),
        ("mode", C.c_int32),
        ("schedule", C.c_int32),
        ("termination_c", C.c_double),
        ("n_max", C.c_int32),
        ("integration", C.c_int32),
        ("transfer", C.c_int32),
        ("policy", C.c_int32),
        ("gating", C.c_int32),
        ("concurrent", C.c_int32),
        ("throttle", C.c_uint64),
        ("noise_seed", C.c_uint64),
        ("boundary_value", C.c_double),
        ("plane_width", C.c_int32),
        ("fixed_p3", C.c_int32),
        ("start_geometric", C.c_int32),
        ("forced_n", C.c_int32),
        ("forced_fraction", C.c_double),
    ]


class CycleReport(C.Structure):
    _fields_ = [
        ("cycle", C.c_int32),
        ("status", C.c_int32),
        ("residual", C.c_double),
        ("normalized", C.c_double),
        ("dof_updates", C.c_uint64),
        ("dof_updates_total", C.c_uint64),
        ("coarse_updates", C.c_uint64),
        ("pending_tasks", C.c_uint64),
        ("max_n", C.c_int32),
        ("max_samples", C.c_int32),
        ("avg_n", C.c_double),
        ("factor_totals", C.c_double),
        ("factor_mean", C.c_double),
        ("enabled_mask", C.c_uint32),
        ("levels", C.c_int32),
        ("cells", C.c_uint64),
        ("dofs_fine_interior", C.c_uint64),
        ("grid_points_total", C.c_uint64),
        ("wall_seconds", C.c_double),
    ]


class CompressionStats(C.Structure):
    _fields_ = [
        ("fine_cells", C.c_uint64),
        ("fine_stored_bytes", C.c_uint64),
        ("fine_uncompressed_bytes", C.c_uint64),
        ("fine_factor_totals", C.c_double),
        ("fine_factor_mean", C.c_double),
        ("max_n", C.c_int32),
        ("max_sample_count", C.c_int32),
        ("avg_n", C.c_double),
        ("max_delta", C.c_double),
        ("p3_histogram", C.c_uint64 * 9),
        ("total_stored_bytes", C.c_uint64),
        ("total_uncompressed_bytes", C.c_uint64),
        ("total_factor", C.c_double),
    ]


def report_dict(r: CycleReport) -> dict:
    return {name: getattr(r, name) for name, _ in CycleReport._fields_}


def splitmix64(z: int) -> int:
    """problem.cpp:43-48."""
    m = (1 << 64) - 1
    z = (z + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def field_constant(value=1.0) -> Field:
    return Field(kind=FIELD_CONSTANT, blocks=0, value=value)


def field_theta(theta) -> Field:
    return Field(kind=FIELD_THETA, value=1.0, theta=theta)


def field_quadrant(eps_low) -> Field:
    return Field(kind=FIELD_QUADRANT, value=1.0, eps_low=eps_low)


def field_sinusoid(amp=0.9, freq=6.0) -> Field:
    return Field(kind=FIELD_SINUSOID, value=1.0, amp=amp, freq=freq)


def field_checkerboard(seed=1, blocks=8) -> Field:
    """BASELINE config 1: T_ij = 10^(-2+4U_ij),
    U_ij = (splitmix64(seed ^ (blocks*i+j)) >> 11) * 2^-53. The table is
    computed on the host (Python float pow == C pow for these arguments is
    NOT assumed: lzb_field_checkerboard() in C computes the table for the
    device path, this helper is only used when a caller builds fields here)."""
    f = Field(kind=FIELD_CHECKER, blocks=blocks, value=1.0)
    for i in range(blocks):
        for j in range(blocks):
            u = (splitmix64(seed ^ (blocks * i + j)) >> 11) * 2.0 ** -53
            f.table[i * blocks + j] = math.pow(10.0, -2.0 + 4.0 * u)
    return f

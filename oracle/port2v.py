"""Restated 2D V(nu, nu) cycle (numpy) — TEST INFRASTRUCTURE ONLY.

BASELINE configs[1] names V(1,1) cycles; the reference's solver is additive
only (proj/src/solver.cpp:99-347), so the multiplicative cycle is a restated
extension, unpinned by the reference, built from the pinned pieces of the
additive cycle (device: lzb_grid_vcycle):
  * residual: r = fl - sum over the (up to four) adjacent cells of the cell
    operator row (4x4, corner c at (c & 1, c >> 1), types.hpp:14-15) times u,
    zero on the Dirichlet boundary (solver.cpp:145-200); diag = sum of the
    rows' diagonal entries;
  * damped Jacobi on interior vertices with diag != 0 (solver.cpp:240-252);
  * restriction fl_c = sum over patches of P^T r, each fine lattice vertex
    counted in its lowest-coordinate owner patch (owns_lattice_vertex,
    solver.cpp:39-57, transfer.cpp);
  * prolongation u_f += P u_c through the fine vertex's owner patch
    (solver.cpp:280-313 with a zero snapshot).
Operators and per-patch transfers are read from the product (its Galerkin
operators are pinned bit-for-bit by the additive-cycle tests), so this
checks the cycle's structure, not the assembly. Sums run in numpy's order:
the comparison is at 1e-10 (residual) / 1e-12 (u), not bitwise.
"""
from __future__ import annotations

import math

import numpy as np


def _corner(c):
    return c & 1, c >> 1


class VCycle2:
    """ops[l]: (N*N, 16) cell operators of level l (N = 3**l), row-major 4x4;
    P[l]: (N*N, 16, 4) transfer blocks of the patches of level l < D;
    fl: leaf load ((N+1)^2); u: leaf start ((N+1)^2)."""

    def __init__(self, ops, P, fl, u, omega, target=1e-10, divergence=1e2, max_cycles=500):
        self.D = len(ops) - 1
        self.N = [3 ** l for l in range(self.D + 1)]
        self.K = [np.asarray(o, dtype=np.float64).reshape(n, n, 4, 4) for o, n in zip(ops, self.N)]
        self.P = [np.asarray(p, dtype=np.float64).reshape(n, n, 16, 4) for p, n in zip(P, self.N)]
        self.u = [np.zeros((n + 1, n + 1)) for n in self.N]
        self.fl = [np.zeros((n + 1, n + 1)) for n in self.N]
        D = self.D
        self.u[D] = np.array(u, dtype=np.float64).reshape(self.N[D] + 1, -1)
        self.fl[D] = np.array(fl, dtype=np.float64).reshape(self.N[D] + 1, -1)
        self.omega, self.target, self.divergence, self.max_cycles = omega, target, divergence, max_cycles
        self.cycle, self.history, self.first = 0, [], None

    def residual(self, l):
        n, K, u = self.N[l], self.K[l], self.u[l]
        au = np.zeros((n + 1, n + 1))
        dg = np.zeros((n + 1, n + 1))
        for row in range(4):
            rx, ry = _corner(row)
            s = np.zeros((n, n))
            for col in range(4):
                cx, cy = _corner(col)
                s += K[:, :, row, col] * u[cy:cy + n, cx:cx + n]
            au[ry:ry + n, rx:rx + n] += s
            dg[ry:ry + n, rx:rx + n] += K[:, :, row, row]
        r = self.fl[l] - au
        r[0, :] = r[-1, :] = r[:, 0] = r[:, -1] = 0.0
        return r, dg

    def smooth(self, l, k):
        for _ in range(k):
            r, dg = self.residual(l)
            with np.errstate(divide="ignore", invalid="ignore"):
                upd = np.where(dg != 0, self.omega / dg * r, 0.0)
            upd[0, :] = upd[-1, :] = upd[:, 0] = upd[:, -1] = 0.0
            self.u[l] += upd

    def restrict(self, l, r):  # fl_{l-1} = P^T r over owned lattice vertices
        nc = self.N[l - 1]
        P = self.P[l - 1]
        out = np.zeros((nc + 1, nc + 1))
        idx = np.arange(nc)
        for L in range(16):
            lx, ly = L % 4, L // 4
            rv = r[3 * idx[:, None] + ly, 3 * idx[None, :] + lx]  # [cy, cx]
            rv = rv.copy()
            if lx == 0:
                rv[:, 1:] = 0.0
            if ly == 0:
                rv[1:, :] = 0.0
            for k in range(4):
                kx, ky = _corner(k)
                out[ky:ky + nc, kx:kx + nc] += P[:, :, L, k] * rv
        return out

    def prolong(self, l):  # u_l += P u_{l-1} through owner patches, interior only
        n, nc = self.N[l], self.N[l - 1]
        uc, P = self.u[l - 1], self.P[l - 1]
        f = np.arange(n + 1)
        x1 = f // 3
        own = np.where((f - 3 * x1 == 0) & (x1 > 0), x1 - 1, x1)
        own = np.minimum(own, nc - 1)
        Lc = f - 3 * own
        py, px = own[:, None], own[None, :]
        L = Lc[:, None] * 4 + Lc[None, :]
        add = np.zeros((n + 1, n + 1))
        for k in range(4):
            kx, ky = _corner(k)
            add += P[py, px, L, k] * uc[py + ky, px + kx]
        add[0, :] = add[-1, :] = add[:, 0] = add[:, -1] = 0.0
        self.u[l] += add

    def vstep(self, nu=1):
        D = self.D
        self.cycle += 1
        r, _ = self.residual(D)
        res = math.sqrt(float(np.sum(r ** 2)))
        if not self.history:
            self.first = res if res > 0 else 1.0
        self.history.append(res)
        norm = res / self.first
        status = 1 if norm <= self.target else (2 if norm >= self.divergence else (
            3 if self.cycle >= self.max_cycles else 0))
        if status in (0, 3):
            for l in range(D, 0, -1):
                self.smooth(l, nu)
                r, _ = self.residual(l)
                self.fl[l - 1] = self.restrict(l, r)
                self.u[l - 1] = np.zeros_like(self.u[l - 1])
            for l in range(1, D + 1):
                self.prolong(l)
                self.smooth(l, nu)
        return {"cycle": self.cycle, "residual": res, "normalized": norm, "status": status}

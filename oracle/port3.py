"""Restated 3D oracle (numpy) — TEST INFRASTRUCTURE ONLY.

The reference has no 3D code (proj/include/lazymg/types.hpp:13):
parity of the 3D extension is unpinned by the reference and
is checked against this restatement and against internal oracles instead:
  * the trilinear element is the 3D form of reference_subcell_stiffness
    (proj/src/element.cpp:8-32): per axis seg_int over the sub-interval for
    the shape-function pair, the derivative factor +-(t1 - t0), and
    K_sub_ab = h (Dx Sy Sz + Sx Dy Sz + Sx Sy Dz); K = sum eps(centre_ijk)
    K_sub(i,j,k) over the n^3 sub-boxes (sample order i, j, k as
    proj/include/lazymg/element.hpp:41-45), computed here literally per sample;
  * constant eps: the analytic Q1 cube stiffness h/12 * (4 | 0 | -1 | -1)
    by corner distance (0, 1, 2, 3 differing coordinates);
  * z-independent eps: K3 = h (K2 (x) Mz + M2 (x) Dz) from the 2D element;
  * the Gaussian random field generator restated with numpy's inverse FFT.
"""
from __future__ import annotations

import math

import numpy as np

from paper_2005_03606_b200._types import splitmix64


def seg_int(si: int, sj: int, a: float, b: float) -> float:
    """proj/src/element.cpp:8-15: integral of X_si * X_sj over [a, b], X_0 = 1 - t, X_1 = t."""
    a0, a1 = (0.0, 1.0) if si else (1.0, -1.0)
    b0, b1 = (0.0, 1.0) if sj else (1.0, -1.0)
    Fb = a0 * b0 * b + (a0 * b1 + a1 * b0) * b * b / 2.0 + a1 * b1 * b * b * b / 3.0
    Fa = a0 * b0 * a + (a0 * b1 + a1 * b0) * a * a / 2.0 + a1 * b1 * a * a * a / 3.0
    return Fb - Fa


def corner(a: int):
    return a & 1, (a >> 1) & 1, a >> 2


def subcell_stiffness3(i, j, k, n, h):
    """K_sub(i,j,k) (8 x 8) of the trilinear cube of size h."""
    inv = 1.0 / n
    iv = [(i * inv, (i + 1) * inv), (j * inv, (j + 1) * inv), (k * inv, (k + 1) * inv)]
    K = np.zeros((8, 8))
    for a in range(8):
        ca = corner(a)
        for b in range(8):
            cb = corner(b)
            S = [seg_int(ca[d], cb[d], *iv[d]) for d in range(3)]
            Dd = [(1.0 if ca[d] == cb[d] else -1.0) * (iv[d][1] - iv[d][0]) for d in range(3)]
            K[a, b] = h * (Dd[0] * S[1] * S[2] + S[0] * Dd[1] * S[2] + S[0] * S[1] * Dd[2])
    return K


def unit_stiffness3(h=1.0):
    """Analytic Q1 stiffness of the cube [0,h]^3: h/12 * (4, 0, -1, -1)."""
    K = np.zeros((8, 8))
    for a in range(8):
        for b in range(8):
            d = sum(x != y for x, y in zip(corner(a), corner(b)))
            K[a, b] = h * (4.0, 0.0, -1.0, -1.0)[d] / 12.0
    return K


def eps_grf(table: np.ndarray, x: float, y: float, z: float) -> float:
    """exp of the periodic trilinear interpolant, lerp(a, b, t) = (1 - t) a + t b."""
    n = table.shape[0]
    u = [x * n, y * n, z * n]
    f = [math.floor(v) for v in u]
    t = [u[d] - f[d] for d in range(3)]
    i0 = [int(f[d]) % n for d in range(3)]
    i1 = [(i0[d] + 1) % n for d in range(3)]

    def lerp(a, b, s):
        return (1.0 - s) * a + s * b

    def at(a, b, c):
        return table[(i0[0], i1[0])[a], (i0[1], i1[1])[b], (i0[2], i1[2])[c]]

    c00 = lerp(at(0, 0, 0), at(0, 0, 1), t[2])
    c01 = lerp(at(0, 1, 0), at(0, 1, 1), t[2])
    c10 = lerp(at(1, 0, 0), at(1, 0, 1), t[2])
    c11 = lerp(at(1, 1, 0), at(1, 1, 1), t[2])
    return math.exp(lerp(lerp(c00, c01, t[1]), lerp(c10, c11, t[1]), t[0]))


def eps_sphere(x, y, z, centre=(0.5, 0.5, 0.5), radius=0.25, width=0.01, eps_in=100.0, eps_out=1.0):
    """BASELINE configs[3] field (lzb_types.h LZB_F3_SPHERE): eps_out + (eps_in -
    eps_out) (1 + tanh(2 atanh(0.8) t)) / 2, t = (radius - r) / width."""
    r = math.sqrt((x - centre[0]) ** 2 + (y - centre[1]) ** 2 + (z - centre[2]) ** 2)
    t = (radius - r) / width
    return eps_out + (eps_in - eps_out) * (0.5 * (1.0 + math.tanh(2.1972245773362196 * t)))


def sphere_tree_leaves(lbase, lmax, centre=(0.5, 0.5, 0.5), radius=0.25):
    """Leaves (level, cx, cy, cz) of the adaptive spacetree of BASELINE
    configs[3]: every cell below lbase refined; below lmax the cells whose box
    meets the ball |x - centre| <= radius (the restated 3D form of the
    reference's refine/apply_refinement, mesh.cpp:236-312)."""
    c = np.asarray(centre, dtype=np.float64)
    cur = np.zeros((1, 3), np.int64)
    out = []
    for lvl in range(lmax + 1):
        h = (1.0 / 3) ** lvl
        lo = cur * h
        near = np.clip(c, lo, lo + h)
        dist = np.sqrt(((near - c) ** 2).sum(axis=1))
        refine = np.full(len(cur), lvl < lbase) | ((lvl < lmax) & (dist <= radius))
        leaves = cur[~refine]
        out.append(np.column_stack([np.full(len(leaves), lvl), leaves]))
        par = cur[refine]
        if not len(par):
            break
        d = np.array([(dx, dy, dz) for dz in range(3) for dy in range(3) for dx in range(3)], np.int64)
        cur = (3 * par[:, None, :] + d[None, :, :]).reshape(-1, 3)
    return np.concatenate(out)


def element3(eps, x0, y0, z0, h, n):
    """sum_ijk eps(x_i, y_j, z_k) K_sub(i,j,k), samples x0 + (i + 0.5) inv h."""
    inv = 1.0 / n
    K = np.zeros((8, 8))
    for i in range(n):
        for j in range(n):
            for k in range(n):
                e = eps(x0 + (i + 0.5) * inv * h, y0 + (j + 0.5) * inv * h, z0 + (k + 0.5) * inv * h)
                K += e * subcell_stiffness3(i, j, k, n, h)
    return K


def mass2(eps2, x0, y0, h, n):
    """2D eps-weighted mass sum_ij eps_ij Sx Sy (4 x 4, corners SW,SE,NW,NE), h-free like K2."""
    inv = 1.0 / n
    M = np.zeros((4, 4))
    for i in range(n):
        for j in range(n):
            e = eps2(x0 + (i + 0.5) * inv * h, y0 + (j + 0.5) * inv * h)
            for a in range(4):
                for b in range(4):
                    M[a, b] += e * seg_int(a & 1, b & 1, i * inv, (i + 1) * inv) * \
                        seg_int(a >> 1, b >> 1, j * inv, (j + 1) * inv)
    return M


def extruded_from_2d(K2, M2, h):
    """K3 = h (K2 (x) Mz + M2 (x) Dz) for eps independent of z (a = a2 + 4 az)."""
    Mz = np.array([[1.0 / 3, 1.0 / 6], [1.0 / 6, 1.0 / 3]])
    Dz = np.array([[1.0, -1.0], [-1.0, 1.0]])
    K = np.zeros((8, 8))
    for a in range(8):
        for b in range(8):
            a2, az, b2, bz = a & 3, a >> 2, b & 3, b >> 2
            K[a, b] = h * (K2[a2, b2] * Mz[az, bz] + M2[a2, b2] * Dz[az, bz])
    return K


def grf_table(seed: int, n: int, ell: float, sigma2: float) -> np.ndarray:
    """The generator of lzb_grf_table restated: S_k = exp(-(2 pi |k| ell)^2 / 2),
    Z = sum S_k / sigma2, c_k = sqrt(S_k / Z) (xi - i eta) with (xi, eta) from
    Box-Muller on splitmix64 uniforms in k order, g = Re(unnormalised inverse DFT)."""
    tpi = 2.0 * math.pi
    freq = [i if i < n // 2 else i - n for i in range(n)]
    S = np.zeros((n, n, n))
    Z = 0.0
    for i in range(n):
        for j in range(n):
            for l in range(n):
                k2 = float(freq[i]) ** 2 + float(freq[j]) ** 2 + float(freq[l]) ** 2
                s = math.exp(-0.5 * tpi * tpi * ell * ell * k2)
                S[i, j, l] = s
                Z += s
    Z /= sigma2
    c = np.zeros((n, n, n), complex)
    st = seed
    m = (1 << 64) - 1

    def uniform():
        nonlocal st
        st = (st + 0x9E3779B97F4A7C15) & m
        z = st
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
        z = z ^ (z >> 31)
        return ((z >> 11) + 0.5) * 2.0 ** -53

    flat = c.reshape(-1)
    Sf = S.reshape(-1)
    for q in range(n ** 3):
        u1, u2 = uniform(), uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        a = math.sqrt(Sf[q] / Z)
        flat[q] = complex(a * r * math.cos(tpi * u2), -a * r * math.sin(tpi * u2))
    return np.real(np.fft.ifftn(c)) * n ** 3


assert splitmix64  # same generator family as the 2D checkerboard (problem.cpp:43-48)


# ------------------------------------------------------------------ 3D cycle
def _mix(z):
    m = (1 << 64) - 1
    z = (z + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def pw3(L, a):
    """Trilinear lattice weight w(L, a) = prod_d (a_d ? L_d : 3 - L_d) / 27."""
    lx, ly, lz = L
    return float(((lx if a & 1 else 3 - lx) * (ly if (a >> 1) & 1 else 3 - ly) * (lz if a >> 2 else 3 - lz))) / 27.0


class Cycle3:
    """The additive multilevel cycle of proj/src/solver.cpp:99-347 restated in 3D
    (numpy, arrays indexed [z, y, x]): Galerkin coarse operators, trilinear
    transfer with the lowest-coordinate owner patch, hierarchical residual,
    restriction of r-hat, Jacobi, prolongation cascade, injection."""

    def __init__(self, leaf_ops, depth, variant="adafac-pi", omega=0.6, rhs_scale=3 * math.pi ** 2, seed=42,
                 target=1e-10, max_cycles=100):
        self.D, self.omega, self.variant, self.target, self.max_cycles = depth, omega, variant, target, max_cycles
        self.N = [3 ** l for l in range(depth + 1)]
        N = self.N[depth]
        self.ops = [None] * (depth + 1)
        self.ops[depth] = np.asarray(leaf_ops, dtype=np.float64).reshape(N, N, N, 8, 8)  # [z, y, x]
        for l in range(depth - 1, -1, -1):
            self.ops[l] = self._galerkin(self.ops[l + 1])
        self.v = []
        for l in range(depth + 1):
            n = self.N[l] + 1
            f = {k: np.zeros((n, n, n)) for k in ("u", "fl", "r", "rh", "uh", "dg", "aux", "us")}
            self.v.append(f)
        for l in range(depth + 1):
            n = self.N[l]
            u = self.v[l]["u"]
            for iz in range(n + 1):
                for iy in range(n + 1):
                    for ix in range(n + 1):
                        if min(ix, iy, iz) == 0 or max(ix, iy, iz) == n:
                            u[iz, iy, ix] = 0.0
                        else:
                            k = _mix(seed ^ _mix((l << 48) ^ (ix << 32) ^ (iy << 16) ^ iz))
                            u[iz, iy, ix] = (4.0 / 3.0) * float(k >> 11) * 2.0 ** -53
        self._inject()
        # lumped load on the leaves: f(v) h^3 / 8 per adjacent leaf
        n = N
        h = (1.0 / 3) ** depth
        fl = self.v[depth]["fl"]
        w = h * h * h / 8.0
        for iz in range(n + 1):
            for iy in range(n + 1):
                for ix in range(n + 1):
                    adj = sum(1 for dz in (0, 1) for dy in (0, 1) for dx in (0, 1)
                              if 0 <= ix - dx < n and 0 <= iy - dy < n and 0 <= iz - dz < n)
                    term = w * (rhs_scale * math.sin(math.pi * (ix * h)) * math.sin(math.pi * (iy * h))
                                * math.sin(math.pi * (iz * h)))
                    acc = 0.0
                    for _ in range(adj):
                        acc += term
                    fl[iz, iy, ix] = acc
        self.history = []
        self.cycle = 0

    @staticmethod
    def _galerkin(fine):
        Nf = fine.shape[0]
        Nc = Nf // 3
        out = np.zeros((Nc, Nc, Nc, 8, 8))
        for lz in range(3):
            for ly in range(3):
                for lx in range(3):
                    Q = np.array([[pw3((lx + (i & 1), ly + ((i >> 1) & 1), lz + (i >> 2)), a) for a in range(8)]
                                  for i in range(8)])
                    K = fine[lz::3, ly::3, lx::3]
                    out += np.einsum("ia,zyxij,jb->zyxab", Q, K, Q)
        return out

    def _corner_view(self, arr, n, a):
        """arr[z + az, y + ay, x + ax] over the n^3 cells."""
        ax, ay, az = a & 1, (a >> 1) & 1, a >> 2
        return arr[az:az + n, ay:ay + n, ax:ax + n]

    def _owner(self, l):
        """Per fine vertex of level l: owner patch coordinate and lattice index per axis."""
        n, nc = self.N[l], self.N[l - 1]
        f = np.arange(n + 1)
        x1 = f // 3
        p = np.where((f - 3 * x1 == 0) & (x1 > 0), x1 - 1, x1)
        p = np.minimum(p, nc - 1)
        return p, f - 3 * p

    def _interp(self, l, coarse):
        """P coarse at every vertex of level l."""
        p, L = self._owner(l)
        out = 0.0
        for a in range(8):
            ax, ay, az = a & 1, (a >> 1) & 1, a >> 2
            w = (np.where(ax, L, 3 - L)[None, None, :] * np.where(ay, L, 3 - L)[None, :, None]
                 * np.where(az, L, 3 - L)[:, None, None]) / 27.0
            cv = coarse[(p + az)[:, None, None], (p + ay)[None, :, None], (p + ax)[None, None, :]]
            out = out + w * cv
        return out

    def _restrict(self, l, rh):
        """fl_{l-1} = P^T r-hat over the owned lattice (each fine vertex through its owner patch)."""
        p, L = self._owner(l)
        nc = self.N[l - 1]
        out = np.zeros((nc + 1,) * 3)
        for a in range(8):
            ax, ay, az = a & 1, (a >> 1) & 1, a >> 2
            w = (np.where(ax, L, 3 - L)[None, None, :] * np.where(ay, L, 3 - L)[None, :, None]
                 * np.where(az, L, 3 - L)[:, None, None]) / 27.0
            np.add.at(out, ((p + az)[:, None, None], (p + ay)[None, :, None], (p + ax)[None, None, :]), w * rh)
        return out

    def _interior(self, n):
        m = np.zeros((n + 1,) * 3, bool)
        m[1:n, 1:n, 1:n] = True
        return m

    def _residual(self, l):
        n = self.N[l]
        K = self.ops[l]
        V = self.v[l]
        Au = np.zeros_like(V["u"])
        Auh = np.zeros_like(V["u"])
        dg = np.zeros_like(V["u"])
        for row in range(8):
            for col in range(8):
                uc = self._corner_view(V["u"], n, col)
                uhc = self._corner_view(V["uh"], n, col)
                tgt = self._corner_view(Au, n, row)
                tgt += K[..., row, col] * uc
                self._corner_view(Auh, n, row)[...] += K[..., row, col] * uhc
            self._corner_view(dg, n, row)[...] += K[..., row, row]
        inner = self._interior(n)
        V["r"] = np.where(inner, V["fl"] - Au, 0.0)
        V["rh"] = np.where(inner, V["fl"] - Auh, 0.0)
        V["dg"] = dg

    def _inject(self):
        for l in range(self.D, 0, -1):
            self.v[l - 1]["u"] = self.v[l]["u"][::3, ::3, ::3].copy()

    def step(self):
        self.cycle += 1
        for l in range(self.D, -1, -1):
            V = self.v[l]
            V["uh"] = V["u"] - self._interp(l, self.v[l - 1]["u"]) if l > 0 else V["u"].copy()
            self._residual(l)
            if l > 0:
                self.v[l - 1]["fl"] = self._restrict(l, V["rh"])
        n = self.N[self.D]
        res = math.sqrt(float(np.sum(self.v[self.D]["r"][1:n, 1:n, 1:n] ** 2)))
        if not self.history:
            self.first = res if res > 0 else 1.0
        self.history.append(res)
        norm = res / self.first
        status = 1 if norm <= self.target else (2 if norm >= 1e2 else (3 if self.cycle >= self.max_cycles else 0))
        if status in (0, 3):
            for l in range(self.D):
                self.v[l]["us"] = self.v[l]["u"].copy()
                self.v[l]["aux"] = np.zeros_like(self.v[l]["u"])
            for l in range(self.D, -1, -1):
                V = self.v[l]
                inner = self._interior(self.N[l])
                if self.variant == "adafac-pi" and l > 0:
                    Cv = self.v[l - 1]
                    Cv["aux"] = V["r"][::3, ::3, ::3].copy()
                    cin = self._interior(self.N[l - 1])
                    with np.errstate(divide="ignore", invalid="ignore"):
                        caux = np.where(cin & (Cv["dg"] != 0), self.omega / Cv["dg"] * Cv["aux"], 0.0)
                    V["u"] = np.where(inner, V["u"] - self._interp(l, caux), V["u"])
                damping = self.omega ** (self.D - l + 1) if self.variant == "additive" else self.omega
                with np.errstate(divide="ignore", invalid="ignore"):
                    upd = np.where(V["dg"] != 0, damping / V["dg"] * V["r"], 0.0)
                V["u"] = np.where(inner, V["u"] + upd, V["u"])
            for l in range(1, self.D + 1):
                V, Cv = self.v[l], self.v[l - 1]
                inner = self._interior(self.N[l])
                V["u"] = np.where(inner, V["u"] + self._interp(l, Cv["u"] - Cv["us"]), V["u"])
            self._inject()
        return {"cycle": self.cycle, "residual": res, "normalized": norm, "status": status}


def _cycle3_vstep(self, nu=2):
    """One multiplicative V(nu, nu) cycle (restated extension; device:
    lzb_grid3_vcycle): per level from the leaves nu damped-Jacobi sweeps, the
    residual restricted (P^T over owned lattice vertices) into the next
    level's rhs with a zero start; back up: u_l += P u_{l-1}, nu sweeps.
    Returns the report of the leaf residual before the cycle."""
    D = self.D

    def residual(l):
        V = self.v[l]
        V["uh"] = V["u"].copy()
        self._residual(l)

    def smooth(l, k):
        for _ in range(k):
            residual(l)
            V = self.v[l]
            inner = self._interior(self.N[l])
            with np.errstate(divide="ignore", invalid="ignore"):
                upd = np.where(V["dg"] != 0, self.omega / V["dg"] * V["r"], 0.0)
            V["u"] = np.where(inner, V["u"] + upd, V["u"])

    self.cycle += 1
    residual(D)
    n = self.N[D]
    res = math.sqrt(float(np.sum(self.v[D]["r"][1:n, 1:n, 1:n] ** 2)))
    if not self.history:
        self.first = res if res > 0 else 1.0
    self.history.append(res)
    norm = res / self.first
    status = 1 if norm <= self.target else (2 if norm >= 1e2 else (3 if self.cycle >= self.max_cycles else 0))
    if status in (0, 3):
        for l in range(D, 0, -1):
            smooth(l, nu)
            residual(l)
            self.v[l - 1]["fl"] = self._restrict(l, self.v[l]["rh"])
            self.v[l - 1]["u"] = np.zeros_like(self.v[l - 1]["u"])
        for l in range(1, D + 1):
            V = self.v[l]
            inner = self._interior(self.N[l])
            V["u"] = np.where(inner, V["u"] + self._interp(l, self.v[l - 1]["u"]), V["u"])
            smooth(l, nu)
        self._inject()  # coarse u held corrections: back to the additive invariant
    return {"cycle": self.cycle, "residual": res, "normalized": norm, "status": status}


Cycle3.vstep = _cycle3_vstep


class Cycle3A:
    """The additive cycle of proj/src/solver.cpp:99-347 on a 3D ADAPTIVE
    spacetree (BASELINE configs[3]), restated from the reference's 2D adaptive
    semantics (numpy, dense levels with masks, arrays indexed [z, y, x]):
    - cells exist under refined parents; a vertex exists at a corner of an
      existing cell; kinds (mesh.cpp:115-138): dirichlet on the boundary,
      interior when all 8 surrounding cells of its level exist, else hanging;
      fine_grid = corner of a leaf;
    - operators: leaves' element matrices, refined cells' Galerkin products;
    - fl = the level's own lumped load f h^3/8 per adjacent leaf
      (solver.cpp:99-118), plus the restricted r-hat of the level above;
    - a fine vertex belongs to the first REFINED patch in the order of its
      candidate patches (z, then y, then x, lower coordinate first), the 3D
      restatement's owner rule (solver.cpp:39-57);
    - r, r-hat over every existing vertex (hanging ones keep partial sums),
      zero at dirichlet; restriction of r-hat from owned lattice vertices;
      norm over fine_grid interior vertices; Jacobi / aux correction /
      prolongation on interior vertices only;
    - after a cycle: injection where the fine vertex exists, then hanging
      vertices from the parent interpolant of the first existing host cell
      (mesh.cpp:182-224)."""

    def __init__(self, leaves, leaf_ops, lmax, variant="adafac-pi", omega=0.6, rhs_scale=3 * math.pi ** 2, seed=42,
                 target=1e-10, max_cycles=100):
        self.D, self.omega, self.variant, self.target, self.max_cycles = lmax, omega, variant, target, max_cycles
        self._rhs_scale = rhs_scale
        self.N = [3 ** l for l in range(lmax + 1)]
        leaves = np.asarray(leaves)
        leaf_ops = np.asarray(leaf_ops, dtype=np.float64).reshape(-1, 8, 8)
        self.exist, self.refined = [], []
        for l in range(lmax + 1):
            n = self.N[l]
            self.exist.append(np.zeros((n, n, n), bool))
            self.refined.append(np.zeros((n, n, n), bool))
        self.ops = [np.zeros((n, n, n, 8, 8)) for n in self.N]
        for l in range(lmax + 1):
            sel = leaves[:, 0] == l
            cx, cy, cz = leaves[sel, 1], leaves[sel, 2], leaves[sel, 3]
            self.exist[l][cz, cy, cx] = True
            self.ops[l][cz, cy, cx] = leaf_ops[sel]
        # refined cells: the parents of existing cells, level by level from the finest
        for l in range(lmax, 0, -1):
            z, y, x = np.nonzero(self.exist[l])
            self.refined[l - 1][z // 3, y // 3, x // 3] = True
            self.exist[l - 1][z // 3, y // 3, x // 3] = True
        for l in range(lmax - 1, -1, -1):
            self.ops[l] = np.where(self.refined[l][..., None, None], Cycle3._galerkin(self.ops[l + 1]), self.ops[l])
        self.vexist, self.kind, self.fine = [], [], []
        for l in range(lmax + 1):
            n = self.N[l]
            ve = np.zeros((n + 1,) * 3, bool)
            cnt = np.zeros((n + 1,) * 3, np.int32)
            fg = np.zeros((n + 1,) * 3, bool)
            leaf = self.exist[l] & ~self.refined[l]
            for a in range(8):
                ax, ay, az = a & 1, (a >> 1) & 1, a >> 2
                ve[az:az + n, ay:ay + n, ax:ax + n] |= self.exist[l]
                cnt[az:az + n, ay:ay + n, ax:ax + n] += self.exist[l]
                fg[az:az + n, ay:ay + n, ax:ax + n] |= leaf
            bnd = np.zeros((n + 1,) * 3, bool)
            bnd[[0, n], :, :] = bnd[:, [0, n], :] = bnd[:, :, [0, n]] = True
            kind = np.where(~ve, 0, np.where(bnd, 2, np.where(cnt == 8, 1, 3)))
            self.vexist.append(ve)
            self.kind.append(kind)
            self.fine.append(fg)
        self.own = [None] + [self._owner(l) for l in range(1, lmax + 1)]
        self.v = []
        for l in range(lmax + 1):
            n = self.N[l]
            self.v.append({k: np.zeros((n + 1,) * 3) for k in ("u", "fl", "r", "rh", "uh", "dg", "aux", "us", "load")})
        for l in range(lmax + 1):
            n = self.N[l]
            u = self.v[l]["u"]
            for iz, iy, ix in zip(*np.nonzero(self.vexist[l] & (self.kind[l] != 2))):
                k = _mix(seed ^ _mix((l << 48) ^ (int(ix) << 32) ^ (int(iy) << 16) ^ int(iz)))
                u[iz, iy, ix] = (4.0 / 3.0) * float(k >> 11) * 2.0 ** -53
        self._finish()
        for l in range(lmax + 1):
            n = self.N[l]
            h = (1.0 / 3) ** l
            w = h * h * h / 8.0
            leaf = self.exist[l] & ~self.refined[l]
            adj = np.zeros((n + 1,) * 3, np.int32)
            for a in range(8):
                ax, ay, az = a & 1, (a >> 1) & 1, a >> 2
                adj[az:az + n, ay:ay + n, ax:ax + n] += leaf
            g = np.arange(n + 1) * h
            term = w * (rhs_scale * np.sin(math.pi * g)[None, None, :] * np.sin(math.pi * g)[None, :, None]
                        * np.sin(math.pi * g)[:, None, None])
            self.v[l]["load"] = adj * term
        self.history = []
        self.cycle = 0

    def _owner(self, l):
        """Per vertex of level l: (pz, py, px) of its owner patch, lattice (Lz, Ly, Lx), has-owner."""
        n, nc = self.N[l], self.N[l - 1]
        f = np.arange(n + 1)
        # the patches containing lattice coordinate f: f // 3 - 1 (on a patch
        # boundary) and f // 3, within [0, nc)
        x0 = np.where((f % 3 == 0) & (f > 0), f // 3 - 1, f // 3)
        x1 = np.minimum(f // 3, nc - 1)
        Z, Y, X = np.meshgrid(f, f, f, indexing="ij")
        shape = (n + 1,) * 3
        op = [np.zeros(shape, np.int64) for _ in range(3)]
        has = np.zeros(shape, bool)
        for cz in (x0, x1):
            for cy in (x0, x1):
                for cx in (x0, x1):
                    pz, py, px = cz[Z], cy[Y], cx[X]
                    ok = self.refined[l - 1][pz, py, px] & ~has
                    op[0] = np.where(ok, pz, op[0])
                    op[1] = np.where(ok, py, op[1])
                    op[2] = np.where(ok, px, op[2])
                    has |= ok
        return op[0], op[1], op[2], Z - 3 * op[0], Y - 3 * op[1], X - 3 * op[2], has

    def _w(self, l, a):
        pz, py, px, Lz, Ly, Lx, has = self.own[l]
        ax, ay, az = a & 1, (a >> 1) & 1, a >> 2
        return (np.where(ax, Lx, 3 - Lx) * np.where(ay, Ly, 3 - Ly) * np.where(az, Lz, 3 - Lz)) / 27.0

    def _interp(self, l, coarse):
        pz, py, px, Lz, Ly, Lx, has = self.own[l]
        out = np.zeros_like(coarse, shape=pz.shape)
        for a in range(8):
            ax, ay, az = a & 1, (a >> 1) & 1, a >> 2
            out = out + self._w(l, a) * coarse[pz + az, py + ay, px + ax]
        return out, has

    def _residual(self, l):
        n = self.N[l]
        K = np.where(self.exist[l][..., None, None], self.ops[l], 0.0)
        V = self.v[l]
        Au, Auh, dg = (np.zeros_like(V["u"]) for _ in range(3))
        for row in range(8):
            rx, ry, rz = row & 1, (row >> 1) & 1, row >> 2
            for col in range(8):
                cx, cy, cz = col & 1, (col >> 1) & 1, col >> 2
                Au[rz:rz + n, ry:ry + n, rx:rx + n] += K[..., row, col] * V["u"][cz:cz + n, cy:cy + n, cx:cx + n]
                Auh[rz:rz + n, ry:ry + n, rx:rx + n] += K[..., row, col] * V["uh"][cz:cz + n, cy:cy + n, cx:cx + n]
            dg[rz:rz + n, ry:ry + n, rx:rx + n] += K[..., row, row]
        keep = self.vexist[l] & (self.kind[l] != 2)
        V["r"] = np.where(keep, V["fl"] - Au, 0.0)
        V["rh"] = np.where(keep, V["fl"] - Auh, 0.0)
        V["dg"] = dg

    def _restrict(self, l):
        pz, py, px, Lz, Ly, Lx, has = self.own[l]
        rh = np.where(has, self.v[l]["rh"], 0.0)
        out = self.v[l - 1]["fl"]
        for a in range(8):
            ax, ay, az = a & 1, (a >> 1) & 1, a >> 2
            np.add.at(out, (pz + az, py + ay, px + ax), self._w(l, a) * rh)

    def _finish(self):
        for l in range(self.D, 0, -1):  # inject where the fine vertex exists
            C, F = self.v[l - 1], self.v[l]
            fe = self.vexist[l][::3, ::3, ::3]
            C["u"] = np.where(self.vexist[l - 1] & fe, F["u"][::3, ::3, ::3], C["u"])
        for l in range(1, self.D + 1):  # hanging vertices from the first existing host cell
            n, nc = self.N[l], self.N[l - 1]
            u, cu = self.v[l]["u"], self.v[l - 1]["u"]
            for iz, iy, ix in zip(*np.nonzero(self.kind[l] == 3)):
                cand = []
                for i in (ix, iy, iz):
                    c1 = min(i // 3, nc - 1)
                    c0 = c1 - 1 if (i % 3 == 0 and c1 > 0) else c1
                    cand.append((c0, c1))
                host = None
                for hx in cand[0]:
                    for hy in cand[1]:
                        for hz in cand[2]:
                            if host is None and self.exist[l - 1][hz, hy, hx]:
                                host = (hx, hy, hz)
                hx, hy, hz = host
                fx, fy, fz = (ix - 3.0 * hx) / 3.0, (iy - 3.0 * hy) / 3.0, (iz - 3.0 * hz) / 3.0
                val = 0.0
                for a in range(8):
                    ax, ay, az = a & 1, (a >> 1) & 1, a >> 2
                    w = (fx if ax else 1.0 - fx) * (fy if ay else 1.0 - fy) * (fz if az else 1.0 - fz)
                    if w == 0.0:
                        continue
                    val += w * cu[hz + az, hy + ay, hx + ax]
                u[iz, iy, ix] = val

    def refine(self, leaves, leaf_ops):
        """Re-refinement (the reference's apply_refinement_now, solver.cpp:402-418,
        restated in 3D): the structure rebuilt from the new leaf set and
        operators; u kept on the vertices that existed; a new vertex starts
        from the parent level's interpolant at its first existing host cell
        (coarse levels first, mesh.cpp:182-214), zero on the boundary; then
        injection / hanging interpolation. History and cycle count carry on."""
        old_u = [self.v[l]["u"] for l in range(self.D + 1)]
        old_ve = self.vexist
        hist, cyc, first = self.history, self.cycle, getattr(self, "first", None)
        self.__init__(leaves, leaf_ops, self.D, self.variant, self.omega, self._rhs_scale, 0, self.target,
                      self.max_cycles)
        for l in range(self.D + 1):
            u = np.where(old_ve[l], old_u[l], 0.0)
            new = self.vexist[l] & ~old_ve[l]
            if l > 0:
                nc, cu = self.N[l - 1], self.v[l - 1]["u"]
                for iz, iy, ix in zip(*np.nonzero(new & (self.kind[l] != 2))):
                    cand = []
                    for i in (ix, iy, iz):
                        c1 = min(i // 3, nc - 1)
                        cand.append((c1 - 1 if (i % 3 == 0 and c1 > 0) else c1, c1))
                    host = None
                    for hx in cand[0]:
                        for hy in cand[1]:
                            for hz in cand[2]:
                                if host is None and self.exist[l - 1][hz, hy, hx]:
                                    host = (hx, hy, hz)
                    hx, hy, hz = host
                    fx, fy, fz = (ix - 3.0 * hx) / 3.0, (iy - 3.0 * hy) / 3.0, (iz - 3.0 * hz) / 3.0
                    val = 0.0
                    for a in range(8):
                        ax, ay, az = a & 1, (a >> 1) & 1, a >> 2
                        w = (fx if ax else 1.0 - fx) * (fy if ay else 1.0 - fy) * (fz if az else 1.0 - fz)
                        if w != 0.0:
                            val += w * cu[hz + az, hy + ay, hx + ax]
                    u[iz, iy, ix] = val
            u = np.where(new & (self.kind[l] == 2), 0.0, u)
            self.v[l]["u"] = u
        self._finish()
        self.history, self.cycle = hist, cyc
        if first is not None:
            self.first = first

    def step(self):
        self.cycle += 1
        for l in range(self.D + 1):
            self.v[l]["fl"] = self.v[l]["load"].copy()
        for l in range(self.D, -1, -1):
            V = self.v[l]
            if l > 0:
                interp, has = self._interp(l, self.v[l - 1]["u"])
                V["uh"] = np.where(has, V["u"] - interp, V["u"])
            else:
                V["uh"] = V["u"].copy()
            self._residual(l)
            if l > 0:
                self._restrict(l)
        sq = sum(float(np.sum(np.where(self.fine[l] & (self.kind[l] == 1), self.v[l]["r"], 0.0) ** 2))
                 for l in range(self.D + 1))
        res = math.sqrt(sq)
        if not self.history:
            self.first = res if res > 0 else 1.0
        self.history.append(res)
        norm = res / self.first
        status = 1 if norm <= self.target else (2 if norm >= 1e2 else (3 if self.cycle >= self.max_cycles else 0))
        if status in (0, 3):
            for l in range(self.D + 1):
                self.v[l]["us"] = self.v[l]["u"].copy()
                self.v[l]["aux"] = np.zeros_like(self.v[l]["u"])
            for l in range(self.D, -1, -1):
                V = self.v[l]
                inner = self.kind[l] == 1
                if self.variant == "adafac-pi" and l > 0:
                    Cv = self.v[l - 1]
                    fe = self.vexist[l][::3, ::3, ::3]
                    Cv["aux"] = np.where(self.vexist[l - 1] & fe, V["r"][::3, ::3, ::3], 0.0)
                    cin = self.kind[l - 1] == 1
                    with np.errstate(divide="ignore", invalid="ignore"):
                        caux = np.where(cin & (Cv["dg"] != 0), self.omega / Cv["dg"] * Cv["aux"], 0.0)
                    p, has = self._interp(l, caux)
                    V["u"] = np.where(inner & has, V["u"] - p, V["u"])
                damping = self.omega ** (self.D - l + 1) if self.variant == "additive" else self.omega
                with np.errstate(divide="ignore", invalid="ignore"):
                    upd = np.where(V["dg"] != 0, damping / V["dg"] * V["r"], 0.0)
                V["u"] = np.where(inner, V["u"] + upd, V["u"])
            for l in range(1, self.D + 1):
                V, Cv = self.v[l], self.v[l - 1]
                p, has = self._interp(l, Cv["u"] - Cv["us"])
                V["u"] = np.where((self.kind[l] == 1) & has, V["u"] + p, V["u"])
            self._finish()
        return {"cycle": self.cycle, "residual": res, "normalized": norm, "status": status}

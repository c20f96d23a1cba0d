// tree3.cu — BASELINE configs[3] (C4): a 3D adaptive
// spacetree (k = 3) refined to level lmax inside a sphere and to level lbase
// elsewhere, its leaves at three levels with hanging nodes between them, the
// smoothed-interface sphere field eps (LZB_F3_SPHERE), fixed-p assembly of
// every leaf with the 27-class record coding of grid3.cu, and the delayed
// re-assembly of the interface shell at rising p. The reference is 2D only
// (types.hpp:13); its adaptive mesh is mesh.cpp:66-129,236-312 (cells exist
// only under refined parents, leaves on several levels). The cycle on the
// adaptive tree is the second half of this file.
//
// Leaves are a flat list (level, cx, cy, cz), level-major, in the order the
// levels are generated (parents in order, children z-major); operators are
// class planes over the leaf index (value q of leaf i at q * nleaves + i).
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <chrono>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <array>
#include <cmath>
#include <unordered_map>
#include <vector>

namespace lzb {
namespace {

struct LeafLevels {
    double h[8];  // pow(1/3, l) per level (host-computed, as mesh.hpp:87)
};

// grid3.cu's k_assemble3 for a list of leaves of different levels (or a
// sub-list: `list` holds leaf indices, null for all).
__global__ void __launch_bounds__(128, 4) k_assemble3_leaves(Field3 F, const int4* __restrict__ leaves,
                                                             const int32_t* __restrict__ list, int64_t count,
                                                             int64_t nleaves, LeafLevels HL, AxisTab3 T,
                                                             Planes3 S1, double delta_max, int fixed_p3,
                                                             double* __restrict__ op, int8_t* __restrict__ p3o,
                                                             int32_t* __restrict__ no, unsigned long long* stats,
                                                             int* err) {
    lzb_pdl_enter();
    const int64_t t = gtid();
    if (t >= count) return;
    const int64_t c = list ? list[t] : t;
    const int4 lf = leaves[c];
    const double h = HL.h[lf.x];
    const double x0 = lf.y * h, y0 = lf.z * h, z0 = lf.w * h;
    const double e = centre_eps3(F, x0, y0, z0, h);
    const Base3 B(e, S1.s1, h);
    double sur[27];
    {
        Acc3 A;
        accumulate3(F, x0, y0, z0, h, T, A);
        const double hn = h * (1.0 / T.n);
#pragma unroll
        for (int q = 0; q < 27; ++q)
            sur[q] = class_value(A, hn, q / 9, (q / 3) % 3, q % 3) - B(q / 9, (q / 3) % 3, q % 3);
    }
    bool plain = false;
    const int p3 = fixed_p3 ? fixed_p3 : choose_precision_regular<27>(sur, delta_max, plain);
    if (p3 < 0) {
        atomicExch(err, 1);
        return;
    }
    double delta = 0.0;
#pragma unroll
    for (int q = 0; q < 27; ++q) {
        double rt;
        if (!roundtrip_rec(sur[q], p3, plain, rt)) {
            atomicExch(err, 1);
            return;
        }
        const double d = fabs(rt - sur[q]);
        delta = delta < d ? d : delta;
        op[q * nleaves + c] = B(q / 9, (q / 3) % 3, q % 3) + rt;
    }
    p3o[c] = static_cast<int8_t>(p3);
    no[c] = T.n;
    atomic_max_double_bits(&stats[S_MAXDELTA], delta);
}

// ------------------------------------------------ the cycle on the tree
// solver.cpp:99-347 on the adaptive tree, restated in 3D (oracle/port3.py
// Cycle3A): dense levels with cell flags (0 none, 1 leaf, 2 refined), vertex
// kinds (mesh.cpp:115-138: 0 outside, 1 interior, 2 dirichlet, 3 hanging;
// +4 fine_grid), operators of the existing cells as class planes behind a
// per-cell index. A fine vertex belongs to the first refined patch among the
// patches containing it (z, then y, then x; lower coordinate first).
struct LvA {
    int N;
    double h;
    double* v[LZB_V_NFIELDS];
    double* load;
    uint8_t* cf;
    int32_t* oi;
    double* op;  // class planes, value q of existing cell j at q * nop + j
    int64_t nop;
    uint8_t* vk;
    int bx0, bx1, by0, by1, bz0, bz1;  // vertex box holding every existing vertex (launch domain)
};
enum : uint8_t { VK_OUT = 0, VK_INT = 1, VK_DIR = 2, VK_HANG = 3, VK_FINE = 4 };

__device__ __forceinline__ bool vxyzA(const LvA& L, int& ix, int& iy, int& iz, int64_t& vi) {
    ix = L.bx0 + blockIdx.x * blockDim.x + threadIdx.x;
    iy = L.by0 + blockIdx.y;
    iz = L.bz0 + blockIdx.z;
    if (ix >= L.bx1) return false;
    vi = (static_cast<int64_t>(iz) * (L.N + 1) + iy) * (L.N + 1) + ix;
    return true;
}
__device__ __forceinline__ int64_t cidx(int N, int x, int y, int z) {
    return (static_cast<int64_t>(z) * N + y) * N + x;
}
__device__ __forceinline__ uint8_t cflag(const LvA& L, int x, int y, int z) {
    if (x < 0 || y < 0 || z < 0 || x >= L.N || y >= L.N || z >= L.N) return 0;
    return L.cf[cidx(L.N, x, y, z)];
}
// candidate patches of lattice coordinate f on a level with nc cells per axis
__device__ __forceinline__ void cand(int f, int nc, int& c0, int& c1) {
    c0 = (f % 3 == 0 && f > 0) ? f / 3 - 1 : f / 3;
    c1 = min(f / 3, nc - 1);
}
// owner patch of fine vertex (fx, fy, fz); false if none is refined
__device__ __forceinline__ bool ownerA(const LvA& C, int fx, int fy, int fz, int& px, int& py, int& pz) {
    int x0, x1, y0, y1, z0, z1;
    cand(fx, C.N, x0, x1);
    cand(fy, C.N, y0, y1);
    cand(fz, C.N, z0, z1);
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int c = 0; c < 2; ++c) {
                const int qz = a ? z1 : z0, qy = b ? y1 : y0, qx = c ? x1 : x0;
                if (C.cf[cidx(C.N, qx, qy, qz)] == 2) {
                    px = qx;
                    py = qy;
                    pz = qz;
                    return true;
                }
            }
    return false;
}

__global__ void k4_mark_leaves(const int4* __restrict__ leaves, int64_t n, int lvl, LvA L) {
    lzb_pdl_enter();
    const int64_t t = gtid();
    if (t >= n) return;
    const int4 c = leaves[t];
    if (c.x == lvl) L.cf[cidx(L.N, c.y, c.z, c.w)] = 1;
}
__global__ void k4_mark_parents(LvA F, LvA C) {
    lzb_pdl_enter();
    const int64_t t = gtid();
    const int64_t nc = static_cast<int64_t>(F.N) * F.N * F.N;
    if (t >= nc || !F.cf[t]) return;
    const int x = static_cast<int>(t % F.N), y = static_cast<int>((t / F.N) % F.N), z = static_cast<int>(t / F.N / F.N);
    C.cf[cidx(C.N, x / 3, y / 3, z / 3)] = 2;
}
__global__ void k4_exist01(const uint8_t* __restrict__ cf, int64_t n, int32_t* __restrict__ out) {
    lzb_pdl_enter();
    const int64_t t = gtid();
    if (t < n) out[t] = cf[t] ? 1 : 0;
}
__global__ void k4_index(const uint8_t* __restrict__ cf, int64_t n, int32_t* __restrict__ oi) {
    lzb_pdl_enter();
    const int64_t t = gtid();  // oi holds the exclusive scan of exist01; -1 where no cell
    if (t < n && !cf[t]) oi[t] = -1;
}
// leaf operators (Tree3 class planes over the leaf index) into their level's planes
__global__ void k4_copy_leaf_ops(const int4* __restrict__ leaves, int64_t n, int lvl, const double* __restrict__ lop,
                                 int64_t nleaves, LvA L) {
    lzb_pdl_enter();
    const int64_t t = gtid();
    if (t >= n) return;
    const int4 c = leaves[t];
    if (c.x != lvl) return;
    const int32_t j = L.oi[cidx(L.N, c.y, c.z, c.w)];
#pragma unroll
    for (int q = 0; q < 27; ++q) L.op[q * L.nop + j] = lop[q * nleaves + t];
}
// re-refinement: the class planes / widths / n of the surviving leaves moved
// to their new leaf index (src = old index, -1 for a new leaf)
__global__ void k4_gather_leaves(const int32_t* __restrict__ src, int64_t n_new, int64_t n_old,
                                 const double* __restrict__ op_old, const int8_t* __restrict__ p3_old,
                                 const int32_t* __restrict__ n_oldv, double* __restrict__ op_new,
                                 int8_t* __restrict__ p3_new, int32_t* __restrict__ n_newv) {
    lzb_pdl_enter();
    const int64_t t = gtid();
    if (t >= n_new) return;
    const int32_t o = src[t];
    if (o < 0) {
        p3_new[t] = 0;
        n_newv[t] = 0;
        return;
    }
#pragma unroll
    for (int q = 0; q < 27; ++q) op_new[q * n_new + t] = op_old[q * n_old + o];
    p3_new[t] = p3_old[o];
    n_newv[t] = n_oldv[o];
}
// re-refinement: a vertex that did not exist before starts from the d-linear
// interpolant of the parent level (its first existing host cell), zero on the
// Dirichlet boundary (solver.cpp:402-418 apply_refinement_now, mesh.cpp:182-214)
__global__ void k4_new_vertices(LvA F, LvA C, const uint8_t* __restrict__ existed) {
    lzb_pdl_enter();
    int ix, iy, iz;
    int64_t vi;
    if (!vxyzA(F, ix, iy, iz, vi)) return;
    const int k = F.vk[vi] & 3;
    if (k == VK_OUT || existed[vi]) return;
    if (k == VK_DIR) {
        F.v[LZB_V_U][vi] = 0.0;
        return;
    }
    const int nc = C.N;
    int c1[3], c0[3];
    const int f[3] = {ix, iy, iz};
    for (int d = 0; d < 3; ++d) {
        c1[d] = min(f[d] / 3, nc - 1);
        c0[d] = (f[d] % 3 == 0 && c1[d] > 0) ? c1[d] - 1 : c1[d];
    }
    int hx = -1, hy = -1, hz = -1;
    for (int a = 0; a < 2 && hx < 0; ++a)
        for (int b = 0; b < 2 && hx < 0; ++b)
            for (int c = 0; c < 2 && hx < 0; ++c) {
                const int qx = a ? c1[0] : c0[0], qy = b ? c1[1] : c0[1], qz = c ? c1[2] : c0[2];
                if (C.cf[cidx(nc, qx, qy, qz)]) {
                    hx = qx;
                    hy = qy;
                    hz = qz;
                }
            }
    if (hx < 0) return;
    const double fx = (ix - 3.0 * hx) / 3.0, fy = (iy - 3.0 * hy) / 3.0, fz = (iz - 3.0 * hz) / 3.0;
    double val = 0.0;
    for (int a = 0; a < 8; ++a) {
        const int ax = a & 1, ay = (a >> 1) & 1, az = a >> 2;
        const double w = (ax ? fx : 1.0 - fx) * (ay ? fy : 1.0 - fy) * (az ? fz : 1.0 - fz);
        if (w == 0.0) continue;
        val += w * C.v[LZB_V_U][vidx3(nc, hx + ax, hy + ay, hz + az)];
    }
    F.v[LZB_V_U][vi] = val;
}
// ---- the leaf list on the device (shell selection, level boxes, re-refinement)
struct Ball3 {
    double c[3];
};
// distance range [lo, hi] from the ball's centre to the points of a box: the
// host box_range's arithmetic (Tree3::box_range), operation for operation
__device__ __forceinline__ void box_range_dev(const Ball3& B, double x0, double y0, double z0, double h, double& lo,
                                              double& hi) {
    const double b[3][2] = {{x0, x0 + h}, {y0, y0 + h}, {z0, z0 + h}};
    double near2 = 0.0, far2 = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double c = B.c[d];
        const double q = fmin(fmax(c, b[d][0]), b[d][1]);
        near2 += (q - c) * (q - c);
        const double f = fmax(fabs(b[d][0] - c), fabs(b[d][1] - c));
        far2 += f * f;
    }
    lo = sqrt(near2);
    hi = sqrt(far2);
}
// flag = the leaf's box meets the shell rlo <= |x - centre| <= rhi
__global__ void k4_shell_flags(const int4* __restrict__ leaves, int64_t n, LeafLevels HL, Ball3 B, double rlo,
                               double rhi, uint8_t* __restrict__ flag) {
    lzb_pdl_enter();
    const int64_t t = gtid();
    if (t >= n) return;
    const int4 c = leaves[t];
    const double h = HL.h[c.x];
    double lo, hi;
    box_range_dev(B, c.y * h, c.z * h, c.w * h, h, lo, hi);
    flag[t] = (hi >= rlo && lo <= rhi) ? 1 : 0;
}
// per level the bounding box of its leaves' cell coordinates: bb[l] =
// {min x, max x, min y, max y, min z, max z} (initialised to {INT_MAX, -1, ..})
__global__ void k4_leaf_bbox(const int4* __restrict__ leaves, int64_t n, int* __restrict__ bb) {
    lzb_pdl_enter();
    __shared__ int sb[8 * 6];
    if (threadIdx.x < 48) sb[threadIdx.x] = (threadIdx.x & 1) ? -1 : INT32_MAX;
    __syncthreads();
    for (int64_t t = gtid(); t < n; t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int4 c = leaves[t];
        const int q[3] = {c.y, c.z, c.w};
        // leaves of a warp mostly share the level and lie close: the atomics hit shared memory
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            atomicMin(&sb[c.x * 6 + 2 * d], q[d]);
            atomicMax(&sb[c.x * 6 + 2 * d + 1], q[d]);
        }
    }
    __syncthreads();
    if (threadIdx.x < 48) {
        if (threadIdx.x & 1) atomicMax(&bb[threadIdx.x], sb[threadIdx.x]);
        else atomicMin(&bb[threadIdx.x], sb[threadIdx.x]);
    }
}
__global__ void k4_iota(int32_t* __restrict__ p, int64_t n, int32_t first) {
    lzb_pdl_enter();
    const int64_t t = gtid();
    if (t < n) p[t] = first + static_cast<int32_t>(t);
}
__global__ void k4_existed(LvA L, uint8_t* __restrict__ out) {
    lzb_pdl_enter();
    const int64_t t = gtid();
    if (t < static_cast<int64_t>(L.N + 1) * (L.N + 1) * (L.N + 1)) out[t] = (L.vk[t] & 3) != VK_OUT;
}

// refined cells of C: Galerkin from the 27 children of F (k3_galerkin's class form)
__global__ void __launch_bounds__(256) k4_galerkin(LvA C, LvA F) {
    lzb_pdl_enter();
    const int64_t c = gtid();
    const int64_t ncc = static_cast<int64_t>(C.N) * C.N * C.N;
    if (c >= ncc || C.cf[c] != 2) return;
    const int px = static_cast<int>(c % C.N), py = static_cast<int>((c / C.N) % C.N), pz = static_cast<int>(c / C.N / C.N);
    double out[27];
#pragma unroll
    for (int q = 0; q < 27; ++q) out[q] = 0.0;
    for (int ch = 0; ch < 27; ++ch) {
        const int lz = ch / 9, ly = (ch / 3) % 3, lx = ch % 3;
        const int32_t j = F.oi[cidx(F.N, 3 * px + lx, 3 * py + ly, 3 * pz + lz)];
        double K27[27];
#pragma unroll
        for (int k = 0; k < 27; ++k) K27[k] = F.op[k * F.nop + j];
        galerkin_child(K27, lx, ly, lz, out);
    }
    const int32_t jc = C.oi[c];
#pragma unroll
    for (int q = 0; q < 27; ++q) C.op[q * C.nop + jc] = out[q];
}
__global__ void k4_classify(LvA L) {
    lzb_pdl_enter();
    int ix, iy, iz;
    int64_t vi;
    if (!vxyzA(L, ix, iy, iz, vi)) return;
    int cnt = 0;
    bool fine = false;
    for (int q = 0; q < 8; ++q) {
        const uint8_t f = cflag(L, ix - 1 + (q & 1), iy - 1 + ((q >> 1) & 1), iz - 1 + (q >> 2));
        cnt += f != 0;
        fine |= f == 1;
    }
    uint8_t k = VK_OUT;
    if (cnt) k = bnd3(L.N, ix, iy, iz) ? VK_DIR : (cnt == 8 ? VK_INT : VK_HANG);
    L.vk[vi] = static_cast<uint8_t>(k | (fine ? VK_FINE : 0));
}
// the level's lumped load: f(v) h^3/8 per adjacent leaf (solver.cpp:99-118)
__global__ void k4_load(LvA L, double scale, double w) {
    lzb_pdl_enter();
    int ix, iy, iz;
    int64_t vi;
    if (!vxyzA(L, ix, iy, iz, vi)) return;
    int adj = 0;
    for (int q = 0; q < 8; ++q) adj += cflag(L, ix - 1 + (q & 1), iy - 1 + ((q >> 1) & 1), iz - 1 + (q >> 2)) == 1;
    const double x = ix * L.h, y = iy * L.h, z = iz * L.h;
    const double term = w * (scale * sin(kPi * x) * sin(kPi * y) * sin(kPi * z));
    double acc = 0.0;
    for (int k = 0; k < adj; ++k) acc += term;
    L.load[vi] = acc;
}
__global__ void k4_noise(LvA L, int level, uint64_t seed) {
    lzb_pdl_enter();
    int ix, iy, iz;
    int64_t vi;
    if (!vxyzA(L, ix, iy, iz, vi)) return;
    const int k = L.vk[vi] & 3;
    if (k == VK_OUT || k == VK_DIR) {
        L.v[LZB_V_U][vi] = 0.0;
        return;
    }
    auto mix = [](uint64_t z) {
        z += 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    };
    const uint64_t kk = mix(seed ^ mix((static_cast<uint64_t>(level) << 48) ^ (static_cast<uint64_t>(ix) << 32) ^
                                       (static_cast<uint64_t>(iy) << 16) ^ static_cast<uint64_t>(iz)));
    L.v[LZB_V_U][vi] = (4.0 / 3.0) * static_cast<double>(kk >> 11) * 0x1.0p-53;
}
__global__ void k4_reset_fl(LvA L) {
    lzb_pdl_enter();
    int ix, iy, iz;
    int64_t vi;
    if (vxyzA(L, ix, iy, iz, vi)) L.v[LZB_V_FL][vi] = L.load[vi];
}
__global__ void k4_uhat(LvA F, LvA C, int has_coarse) {
    lzb_pdl_enter();
    int fx, fy, fz;
    int64_t vi;
    if (!vxyzA(F, fx, fy, fz, vi)) return;
    if ((F.vk[vi] & 3) == VK_OUT) return;
    const double u = F.v[LZB_V_U][vi];
    int px, py, pz;
    if (!has_coarse || !ownerA(C, fx, fy, fz, px, py, pz)) {
        F.v[LZB_V_UHAT][vi] = u;
        return;
    }
    const int lx = fx - 3 * px, ly = fy - 3 * py, lz = fz - 3 * pz;
    double interp = 0.0;
    for (int a = 0; a < 8; ++a)
        interp += pw3(lx, ly, lz, a) * C.v[LZB_V_U][vidx3(C.N, px + (a & 1), py + ((a >> 1) & 1), pz + (a >> 2))];
    F.v[LZB_V_UHAT][vi] = u - interp;
}
// r, r-hat, diag over the existing adjacent cells (gather, q = dx + 2 dy + 4 dz)
__global__ void __launch_bounds__(128) k4_residual(LvA F) {
    lzb_pdl_enter();
    int ix, iy, iz;
    int64_t vi;
    if (!vxyzA(F, ix, iy, iz, vi)) return;
    const int kind = F.vk[vi] & 3;
    if (kind == VK_OUT) return;  // r, r-hat, diag of absent vertices stay 0 (never read)
    const int N = F.N;
    const double fl = F.v[LZB_V_FL][vi];
    double r = fl, rh = fl, dg = 0.0;
    for (int q = 0; q < 8; ++q) {
        const int dx = q & 1, dy = (q >> 1) & 1, dz = q >> 2;
        const int cx = ix - 1 + dx, cy = iy - 1 + dy, cz = iz - 1 + dz;
        if (!cflag(F, cx, cy, cz)) continue;
        const int row = (1 - dx) + 2 * (1 - dy) + 4 * (1 - dz);
        const int32_t j = F.oi[cidx(N, cx, cy, cz)];
        double au = 0.0, auh = 0.0;
        for (int col = 0; col < 8; ++col) {
            const double k = F.op[cls3(row, col) * F.nop + j];
            const int64_t cv = vidx3(N, cx + (col & 1), cy + ((col >> 1) & 1), cz + (col >> 2));
            au = __fma_rn(k, F.v[LZB_V_U][cv], au);
            auh = __fma_rn(k, F.v[LZB_V_UHAT][cv], auh);
        }
        r -= au;
        rh -= auh;
        dg += F.op[cls3(row, row) * F.nop + j];
    }
    if (kind == VK_DIR) {
        r = 0.0;
        rh = 0.0;
    }
    F.v[LZB_V_R][vi] = r;
    F.v[LZB_V_RHAT][vi] = rh;
    F.v[LZB_V_DIAG][vi] = dg;
}
// fl_c += P^T r-hat over the lattice vertices each adjacent refined patch owns
__global__ void k4_restrict(LvA F, LvA C) {
    lzb_pdl_enter();
    int IX, IY, IZ;
    int64_t vi;
    if (!vxyzA(C, IX, IY, IZ, vi)) return;
    if ((C.vk[vi] & 3) == VK_OUT) return;
    double acc = C.v[LZB_V_FL][vi];
    for (int q = 0; q < 8; ++q) {
        const int dx = q & 1, dy = (q >> 1) & 1, dz = q >> 2;
        const int px = IX - 1 + dx, py = IY - 1 + dy, pz = IZ - 1 + dz;
        if (cflag(C, px, py, pz) != 2) continue;
        const int k = (1 - dx) + 2 * (1 - dy) + 4 * (1 - dz);
        for (int lz = 0; lz < 4; ++lz)
            for (int ly = 0; ly < 4; ++ly)
                for (int lx = 0; lx < 4; ++lx) {
                    const double w = pw3(lx, ly, lz, k);
                    if (w == 0.0) continue;
                    const int fx = 3 * px + lx, fy = 3 * py + ly, fz = 3 * pz + lz;
                    int ox, oy, oz;
                    if (!ownerA(C, fx, fy, fz, ox, oy, oz) || ox != px || oy != py || oz != pz) continue;
                    const double rh = F.v[LZB_V_RHAT][vidx3(F.N, fx, fy, fz)];
                    if (rh == 0.0) continue;
                    acc += w * rh;
                }
    }
    C.v[LZB_V_FL][vi] = acc;
}
__global__ void __launch_bounds__(256) k4_norm_partial(LvA L, double* partial) {
    lzb_pdl_enter();
    __shared__ double sh[256];
    double s = 0.0;
    const int wx = L.bx1 - L.bx0, wy = L.by1 - L.by0;
    const int64_t nb = static_cast<int64_t>(wx) * wy * (L.bz1 - L.bz0);
    for (int64_t t = gtid(); t < nb; t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int ix = L.bx0 + static_cast<int>(t % wx), iy = L.by0 + static_cast<int>((t / wx) % wy),
                  iz = L.bz0 + static_cast<int>(t / wx / wy);
        const int64_t i = vidx3(L.N, ix, iy, iz);
        if (L.vk[i] == (VK_INT | VK_FINE)) s += L.v[LZB_V_R][i] * L.v[LZB_V_R][i];
    }
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}
__global__ void k4_snap(LvA L) {
    lzb_pdl_enter();
    int ix, iy, iz;
    int64_t i;
    if (!vxyzA(L, ix, iy, iz, i)) return;
    L.v[LZB_V_USNAP][i] = L.v[LZB_V_U][i];
    L.v[LZB_V_AUX][i] = 0.0;
}
__global__ void k4_aux_inject(LvA F, LvA C) {
    lzb_pdl_enter();
    int ix, iy, iz;
    int64_t vi;
    if (!vxyzA(C, ix, iy, iz, vi)) return;
    if ((C.vk[vi] & 3) == VK_OUT) return;
    const int64_t fv = vidx3(F.N, 3 * ix, 3 * iy, 3 * iz);
    if ((F.vk[fv] & 3) != VK_OUT) C.v[LZB_V_AUX][vi] = F.v[LZB_V_R][fv];
}
// the leaf-ward updates of one level on its interior vertices: adaFAC-PI aux
// correction (pi), damped Jacobi (damping), prolongated coarse correction (prol)
__global__ void k4_update(LvA F, LvA C, int pi, double omega, double damping, int jac, int prol) {
    lzb_pdl_enter();
    int fx, fy, fz;
    int64_t vi;
    if (!vxyzA(F, fx, fy, fz, vi)) return;
    if ((F.vk[vi] & 3) != VK_INT) return;
    int px = 0, py = 0, pz = 0;
    const bool own = (pi || prol) && ownerA(C, fx, fy, fz, px, py, pz);
    const int lx = fx - 3 * px, ly = fy - 3 * py, lz = fz - 3 * pz;
    double u = F.v[LZB_V_U][vi];
    if (pi && own) {
        double p = 0.0;
        for (int a = 0; a < 8; ++a) {
            const int64_t ci = vidx3(C.N, px + (a & 1), py + ((a >> 1) & 1), pz + (a >> 2));
            const double dg = C.v[LZB_V_DIAG][ci];
            const double caux = ((C.vk[ci] & 3) == VK_INT && dg != 0.0) ? omega / dg * C.v[LZB_V_AUX][ci] : 0.0;
            p += pw3(lx, ly, lz, a) * caux;
        }
        u -= p;
    }
    if (jac) {
        const double dg = F.v[LZB_V_DIAG][vi];
        if (dg != 0.0) u += damping / dg * F.v[LZB_V_R][vi];
    }
    if (prol && own) {
        double d[8];
        bool any = false;
        for (int a = 0; a < 8; ++a) {
            const int64_t ci = vidx3(C.N, px + (a & 1), py + ((a >> 1) & 1), pz + (a >> 2));
            d[a] = C.v[LZB_V_U][ci] - C.v[LZB_V_USNAP][ci];
            any |= d[a] != 0.0;
        }
        if (any) {
            double p = 0.0;
            for (int a = 0; a < 8; ++a) p += pw3(lx, ly, lz, a) * d[a];
            u += p;
        }
    }
    F.v[LZB_V_U][vi] = u;
}
__global__ void k4_inject(LvA F, LvA C) {
    lzb_pdl_enter();
    int ix, iy, iz;
    int64_t vi;
    if (!vxyzA(C, ix, iy, iz, vi)) return;
    if ((C.vk[vi] & 3) == VK_OUT) return;
    const int64_t fv = vidx3(F.N, 3 * ix, 3 * iy, 3 * iz);
    if ((F.vk[fv] & 3) != VK_OUT) C.v[LZB_V_U][vi] = F.v[LZB_V_U][fv];
}
// hanging u from the parent interpolant of the first existing host cell
// (mesh.cpp:182-214 in 3D: candidates x outer, then y, then z)
__global__ void k4_hanging(LvA F, LvA C) {
    lzb_pdl_enter();
    int ix, iy, iz;
    int64_t vi;
    if (!vxyzA(F, ix, iy, iz, vi)) return;
    if ((F.vk[vi] & 3) != VK_HANG) return;
    const int nc = C.N;
    int c1[3], c0[3];
    const int f[3] = {ix, iy, iz};
    for (int d = 0; d < 3; ++d) {
        c1[d] = min(f[d] / 3, nc - 1);
        c0[d] = (f[d] % 3 == 0 && c1[d] > 0) ? c1[d] - 1 : c1[d];
    }
    int hx = -1, hy = -1, hz = -1;
    for (int a = 0; a < 2 && hx < 0; ++a)
        for (int b = 0; b < 2 && hx < 0; ++b)
            for (int c = 0; c < 2 && hx < 0; ++c) {
                const int qx = a ? c1[0] : c0[0], qy = b ? c1[1] : c0[1], qz = c ? c1[2] : c0[2];
                if (C.cf[cidx(nc, qx, qy, qz)]) {
                    hx = qx;
                    hy = qy;
                    hz = qz;
                }
            }
    if (hx < 0) return;
    const double fx = (ix - 3.0 * hx) / 3.0, fy = (iy - 3.0 * hy) / 3.0, fz = (iz - 3.0 * hz) / 3.0;
    double val = 0.0;
    for (int a = 0; a < 8; ++a) {
        const int ax = a & 1, ay = (a >> 1) & 1, az = a >> 2;
        const double w = (ax ? fx : 1.0 - fx) * (ay ? fy : 1.0 - fy) * (az ? fz : 1.0 - fz);
        if (w == 0.0) continue;
        val += w * C.v[LZB_V_U][vidx3(nc, hx + ax, hy + ay, hz + az)];
    }
    F.v[LZB_V_U][vi] = val;
}

}  // namespace

class Tree3 {
public:
    Tree3(lzb_ctx* ctx, int lbase, int lmax, const lzb_field3& f, double delta_max, int fixed_p3)
        : ctx_(ctx), lbase_(lbase), lmax_(lmax), delta_(delta_max), fixed_(fixed_p3) {
        if (lbase < 0 || lmax < lbase || lmax > 7) throw Error(LZB_ERR_INVALID, "need 0 <= lbase <= lmax <= 7");
        if (fixed_p3 != 0 && (fixed_p3 < 2 || fixed_p3 > 8)) throw Error(LZB_ERR_INVALID, "fixed_p3 must be 0 or 2..8");
        if (!(f.radius >= 0.0)) throw Error(LZB_ERR_INVALID, "refinement sphere radius must be >= 0");
        LZB_CUDA(cudaSetDevice(ctx->device));
        s_ = ctx->solve;
        F_ = to_device(f, table_);
        cen_[0] = f.centre[0];
        cen_[1] = f.centre[1];
        cen_[2] = f.centre[2];
        rad_ = f.radius;
        for (int l = 0; l < 8; ++l) HL_.h[l] = std::pow(1.0 / 3, l);
        build();
        n_leaves_ = static_cast<int64_t>(leaves_.size());
        dleaves_.alloc(n_leaves_);
        LZB_CUDA(cudaMemcpy(dleaves_.p, leaves_.data(), n_leaves_ * sizeof(int4), cudaMemcpyHostToDevice));
        // the list lives on the device from here on; the host keeps its level-major
        // prefix of leaves below lmax (the only ones a re-refinement can replace)
        leaves_.resize(static_cast<size_t>(n_leaves_ - per_level_[lmax_]));
        leaves_.shrink_to_fit();
        op_.alloc(static_cast<size_t>(n_leaves_) * kCls3);
        p3_.alloc(n_leaves_);
        n_.alloc(n_leaves_);
        stats_.alloc(20);
        LZB_CUDA(cudaMemsetAsync(p3_.p, 0, p3_.bytes(), s_));
        LZB_CUDA(cudaMemsetAsync(n_.p, 0, n_.bytes(), s_));
        LZB_CUDA(cudaMemsetAsync(stats_.p, 0, stats_.bytes(), s_));
        LZB_CUDA(cudaStreamSynchronize(s_));
    }

    // Fixed-p assembly of every leaf (list = all) or of the shell list.
    void assemble(int n, bool shell_only) {
        if (n < 1 || n > kMaxN3) throw Error(LZB_ERR_INVALID, "3D sub-samples per axis must be in 1..16");
        if (shell_only && shell_.n == 0) throw Error(LZB_ERR_INVALID, "call set_shell first");
        const int64_t count = shell_only ? n_shell_ : n_leaves_;
        if (count == 0) return;
        const AxisTab3 T = axis_tab3(n), T1 = axis_tab3(1);
        Planes3 S1{};
        for (int q = 0; q < 3; ++q) S1.s1[q] = T1.s[0][q];
        LZB_LAUNCH(k_assemble3_leaves, blocks_for(count, 128), 128, 0, s_, F_, dleaves_.p,
                   shell_only ? shell_.p : nullptr, count, n_leaves_, HL_, T, S1, delta_, fixed_, op_.p, p3_.p, n_.p,
                   stats_.p, ctx_->err.p);
        n_hi_ = std::max(n_hi_, n);
    }

    // The interface shell: leaves whose box meets {x : | |x - centre| - radius | <= band}.
    // the leaves meeting the shell | r - radius | <= band, in leaf order: flags
    // by a kernel (box_range's arithmetic), the index list by a device select
    int64_t set_shell(double band) {
        if (!(band >= 0.0)) throw Error(LZB_ERR_INVALID, "shell band must be >= 0");
        DevBuf<uint8_t> flag(static_cast<size_t>(std::max<int64_t>(n_leaves_, 1)));
        DevBuf<int32_t> list(static_cast<size_t>(std::max<int64_t>(n_leaves_, 1))), cnt(1);
        LZB_LAUNCH(k4_shell_flags, blocks_for(n_leaves_, 256), 256, 0, s_, dleaves_.p, n_leaves_, HL_, ball(),
                   rad_ - band, rad_ + band, flag.p);
        cub::CountingInputIterator<int32_t> idx(0);
        size_t tb = 0;
        LZB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, idx, flag.p, list.p, cnt.p, static_cast<int>(n_leaves_), s_));
        DevBuf<unsigned char> tmp(tb);
        LZB_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, idx, flag.p, list.p, cnt.p, static_cast<int>(n_leaves_), s_));
        int32_t k = 0;
        LZB_CUDA(cudaMemcpyAsync(&k, cnt.p, sizeof k, cudaMemcpyDeviceToHost, s_));
        LZB_CUDA(cudaStreamSynchronize(s_));
        n_shell_ = k;
        shell_.alloc(static_cast<size_t>(std::max<int64_t>(n_shell_, 1)));
        if (n_shell_)
            LZB_CUDA(cudaMemcpyAsync(shell_.p, list.p, n_shell_ * sizeof(int32_t), cudaMemcpyDeviceToDevice, s_));
        LZB_CUDA(cudaStreamSynchronize(s_));
        return n_shell_;
    }

    lzb_compression_stats stats() {
        LZB_CUDA(cudaMemsetAsync(stats_.p + S_HIST, 0, 9 * sizeof(unsigned long long), s_));
        LZB_LAUNCH(k_stats3, 148 * 4, 256, 0, s_, p3_.p, n_leaves_, stats_.p);
        unsigned long long s[20];
        LZB_CUDA(cudaMemcpyAsync(s, stats_.p, sizeof s, cudaMemcpyDeviceToHost, s_));
        sync();
        lzb_compression_stats st;
        std::memset(&st, 0, sizeof st);
        st.fine_cells = static_cast<uint64_t>(n_leaves_);
        double ratio = 0.0;
        for (int p = 0; p <= 8; ++p) {
            st.p3_histogram[p] = s[S_HIST + p];
            st.fine_stored_bytes += s[S_HIST + p] * (p == 0 ? 1ull : 1ull + 64ull * p);
            ratio += static_cast<double>(s[S_HIST + p]) * (512.0 / (p == 0 ? 1.0 : 1.0 + 64.0 * p));
        }
        st.fine_uncompressed_bytes = 512ull * n_leaves_;
        st.fine_factor_totals = st.fine_stored_bytes ? static_cast<double>(st.fine_uncompressed_bytes) /
                                                           static_cast<double>(st.fine_stored_bytes)
                                                     : 0.0;
        st.fine_factor_mean = n_leaves_ ? ratio / n_leaves_ : 0.0;
        st.max_n = n_hi_;
        double md;
        std::memcpy(&md, &s[S_MAXDELTA], sizeof md);
        st.max_delta = md;
        st.total_stored_bytes = st.fine_stored_bytes;
        st.total_uncompressed_bytes = st.fine_uncompressed_bytes;
        st.total_factor = st.fine_factor_totals;
        return st;
    }

    void counts(int64_t* per_level, int64_t* total) const {
        for (int l = 0; l < 8; ++l) per_level[l] = per_level_[l];
        *total = n_leaves_;
    }

    // leaves [first, first + count): the 64 entries, p3, n and (level, cx, cy, cz)
    void cells(int64_t first, int64_t count, double* ops, int32_t* p3, int32_t* n, int32_t* lxyz) {
        if (first < 0 || count < 0 || first + count > n_leaves_) throw Error(LZB_ERR_INVALID, "bad leaf range");
        if (count == 0) return;
        if (ops) {
            DevBuf<double> tmp;
            tmp.alloc(static_cast<size_t>(count) * kCls3);
            LZB_LAUNCH(k3_read_cls<Src64>, blocks_for(count, 128), 128, 0, s_, Src64{op_.p, n_leaves_}, first, count,
                       tmp.p);
            std::vector<double> cls(static_cast<size_t>(count) * kCls3);
            LZB_CUDA(cudaMemcpyAsync(cls.data(), tmp.p, cls.size() * sizeof(double), cudaMemcpyDeviceToHost, s_));
            sync();
            for (int64_t i = 0; i < count; ++i)
                for (int a = 0; a < 8; ++a)
                    for (int b = 0; b < 8; ++b) ops[64 * i + 8 * a + b] = cls[kCls3 * i + cls3(a, b)];
        }
        if (p3) {
            std::vector<int8_t> q(count);
            LZB_CUDA(cudaMemcpy(q.data(), p3_.p + first, count, cudaMemcpyDeviceToHost));
            for (int64_t i = 0; i < count; ++i) p3[i] = q[i];
        }
        if (n) LZB_CUDA(cudaMemcpy(n, n_.p + first, count * sizeof(int32_t), cudaMemcpyDeviceToHost));
        if (lxyz) LZB_CUDA(cudaMemcpy(lxyz, dleaves_.p + first, count * sizeof(int4), cudaMemcpyDeviceToHost));
    }

    // ------------------------------------------------ the cycle on the tree
    // Levels 0..lmax as dense grids with cell flags; the leaves' current
    // operators (this tree's class planes) copied into their levels, the
    // refined cells' operators by Galerkin products, finest first.
    void init_cycle(int variant, double omega, double rhs_scale, uint64_t seed, int max_cycles, double target) {
        if (variant == LZB_ADAFAC_JAC) throw Error(LZB_ERR_INVALID, "the 3D cycle runs additive and adafac-pi");
        variant_ = variant;
        omega_ = omega;
        max_cycles_ = max_cycles;
        target_ = target;
        const int D = lmax_;
        rhs_scale_ = rhs_scale;
        A_.clear();
        A_.resize(D + 1);
        for (int l = 0; l <= D; ++l) {
            LevA& L = A_[l];
            L.N = 1;
            for (int i = 0; i < l; ++i) L.N *= 3;
            L.nc = static_cast<int64_t>(L.N) * L.N * L.N;
            L.nv = static_cast<int64_t>(L.N + 1) * (L.N + 1) * (L.N + 1);
            L.h = HL_.h[l];
            for (int f = 0; f < LZB_V_NFIELDS; ++f) {
                L.v[f].alloc(L.nv);
                LZB_CUDA(cudaMemsetAsync(L.v[f].p, 0, L.v[f].bytes(), s_));
            }
        }
        setup_levels();
        upload_galerkin_weights();
        refresh_ops();
        partialA_.alloc(kNormBlocksA);
        for (int l = 0; l <= D; ++l) LZB_LAUNCH(k4_noise, vgA(l), 128, 0, s_, lv(l), l, seed);
        finish_cycle();
        for (int l = 0; l <= D; ++l)
            LZB_LAUNCH(k4_load, vgA(l), 128, 0, s_, lv(l), rhs_scale, A_[l].h * A_[l].h * A_[l].h / 8.0);
        cycle_ = 0;
        history_.clear();
        sync();
    }

    // the structure of every level from the current leaf list: vertex box,
    // cell flags, operator index and slots, vertex kinds (the vertex fields
    // are kept: init_cycle zeroes them, a re-refinement carries them over)
    void setup_levels() {
        const int D = lmax_;
        // per level the bounding box of its existing cells: its leaves' box
        // joined with the box of the parents of the level below (one pass
        // over the leaves, then finest to coarsest)
        std::vector<std::array<int, 6>> cb(std::max(D + 2, 8), std::array<int, 6>{INT32_MAX, -1, INT32_MAX, -1, INT32_MAX, -1});
        {
            DevBuf<int> bb(48);
            LZB_CUDA(cudaMemcpyAsync(bb.p, cb.data(), 48 * sizeof(int), cudaMemcpyHostToDevice, s_));
            LZB_LAUNCH(k4_leaf_bbox, 148 * 8, 256, 0, s_, dleaves_.p, n_leaves_, bb.p);
            LZB_CUDA(cudaMemcpyAsync(cb.data(), bb.p, 48 * sizeof(int), cudaMemcpyDeviceToHost, s_));
            LZB_CUDA(cudaStreamSynchronize(s_));
        }
        for (int l = D - 1; l >= 0; --l)
            if (cb[l + 1][1] >= 0)
                for (int d = 0; d < 3; ++d) {
                    cb[l][2 * d] = std::min(cb[l][2 * d], cb[l + 1][2 * d] / 3);
                    cb[l][2 * d + 1] = std::max(cb[l][2 * d + 1], cb[l + 1][2 * d + 1] / 3);
                }
        for (int l = 0; l <= D; ++l) {
            LevA& L = A_[l];
            // the vertex box of the level's existing cells: the leaves of level l
            // and the ancestors at level l of every deeper leaf
            int lo[3], hi[3];
            for (int d = 0; d < 3; ++d) {
                lo[d] = cb[l][2 * d];
                hi[d] = cb[l][2 * d + 1];
            }
            for (int d = 0; d < 3; ++d) {
                L.box[2 * d] = hi[d] < 0 ? 0 : lo[d];
                L.box[2 * d + 1] = hi[d] < 0 ? 1 : hi[d] + 2;  // empty level: one (absent) vertex
            }
            L.load.ensure(L.nv);  // fixed sizes per level: allocated once, re-zeroed below
            L.vk.ensure(L.nv);
            // kinds outside the launch box stay "outside" (read by injection across levels)
            LZB_CUDA(cudaMemsetAsync(L.vk.p, 0, L.vk.bytes(), s_));
            LZB_CUDA(cudaMemsetAsync(L.load.p, 0, L.load.bytes(), s_));
            L.cf.ensure(L.nc);
            L.oi.ensure(L.nc + 1);
            LZB_CUDA(cudaMemsetAsync(L.cf.p, 0, L.cf.bytes(), s_));
        }
        // cell flags: leaves, then the refined parents level by level
        for (int l = 0; l <= D; ++l)
            LZB_LAUNCH(k4_mark_leaves, blocks_for(n_leaves_, 256), 256, 0, s_, dleaves_.p, n_leaves_, l, lv(l));
        for (int l = D; l >= 1; --l)
            LZB_LAUNCH(k4_mark_parents, blocks_for(A_[l].nc, 256), 256, 0, s_, lv(l), lv(l - 1));
        // dense cell -> operator slot (exclusive scan of existence), slot counts
        for (int l = 0; l <= D; ++l) {
            LevA& L = A_[l];
            DevBuf<int32_t>& e01 = scan_in_;  // scratch of the finest level's size, kept across calls
            if (e01.n < static_cast<size_t>(L.nc + 1)) e01.alloc(A_[D].nc + 1);
            LZB_CUDA(cudaMemsetAsync(e01.p + L.nc, 0, sizeof(int32_t), s_));
            LZB_LAUNCH(k4_exist01, blocks_for(L.nc, 256), 256, 0, s_, L.cf.p, L.nc, e01.p);
            size_t tb = 0;
            LZB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, e01.p, L.oi.p, static_cast<int>(L.nc + 1), s_));
            DevBuf<unsigned char>& tmp = scan_tmp_;
            if (tmp.n < tb) tmp.alloc(tb);
            LZB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, e01.p, L.oi.p, static_cast<int>(L.nc + 1), s_));
            int32_t cnt = 0;
            LZB_CUDA(cudaMemcpyAsync(&cnt, L.oi.p + L.nc, sizeof(int32_t), cudaMemcpyDeviceToHost, s_));
            LZB_CUDA(cudaStreamSynchronize(s_));
            LZB_LAUNCH(k4_index, blocks_for(L.nc, 256), 256, 0, s_, L.cf.p, L.nc, L.oi.p);
            L.nop = cnt;
            L.op.alloc(static_cast<size_t>(std::max(cnt, 1)) * kCls3);
            LZB_LAUNCH(k4_classify, vgA(l), 128, 0, s_, lv(l));
        }
    }

    // Re-refinement (BASELINE configs[3]; the reference's apply_refinement_now,
    // solver.cpp:402-418, mesh.cpp:236-312, restated for the sphere tree): the
    // ball of refinement grows to `radius`, every leaf meeting it below lmax
    // is refined (the topology changes: new leaves, vertices, hanging nodes);
    // the surviving leaves keep their operators, the new ones are assembled at
    // n (forced re-assembly, stream.cpp:262-266 on_refinement), new vertices
    // start from the parent level's interpolant, the level structure, loads and
    // Galerkin operators are rebuilt; the cycle continues (history kept).
    // Returns the number of new leaves.
    int64_t refine(double radius, int n) {
        if (!(radius >= rad_)) throw Error(LZB_ERR_INVALID, "the refinement ball only grows (no coarsening, mesh.hpp:55)");
        if (n < 1 || n > kMaxN3) throw Error(LZB_ERR_INVALID, "3D sub-samples per axis must be in 1..16");
        const bool cyc = !A_.empty();
        static const bool tr = std::getenv("LZB_TRACE") != nullptr;
        auto t_prev = std::chrono::steady_clock::now();
        auto mark = [&](const char* what) {
            if (!tr) return;
            cudaStreamSynchronize(s_);
            const auto t = std::chrono::steady_clock::now();
            std::fprintf(stderr, "[lzb] refine: %s %.1f ms\n", what,
                         std::chrono::duration<double, std::milli>(t - t_prev).count());
            t_prev = t;
        };
        std::vector<DevBuf<uint8_t>>& existed = existed_;  // kept across events (fixed sizes per level)
        if (cyc && existed.size() != static_cast<size_t>(lmax_ + 1)) existed.resize(lmax_ + 1);
        if (cyc)
            for (int l = 0; l <= lmax_; ++l) {
                existed[l].ensure(A_[l].nv);
                LZB_LAUNCH(k4_existed, blocks_for(A_[l].nv, 256), 256, 0, s_, lv(l), existed[l].p);
            }
        // the new leaf set, level-major, from the old one: a leaf that meets the
        // grown ball below lmax is replaced by its refinement (build()'s rule with
        // the new radius: the ball only grows, so every other leaf survives)
        // Only leaves below lmax can be replaced, and they are the level-major
        // prefix the host keeps (leaves_); the old level-lmax block (97 % of the
        // leaves of the BASELINE tree) moves device to device, behind the new
        // level-lmax leaves the replaced ones generate -- the order a walk over
        // the whole old list would give.
        const int64_t n_old = n_leaves_, n_lo_old = static_cast<int64_t>(leaves_.size()), n_top_old = n_old - n_lo_old;
        rad_ = radius;
        std::vector<std::vector<int4>> per(8);
        std::vector<std::vector<int32_t>> per_src(8);
        std::vector<int4> stack;
        for (int64_t i = 0; i < n_lo_old; ++i) {
            const int4 c = leaves_[i];
            double lo, hi;
            box_range(c.y * HL_.h[c.x], c.z * HL_.h[c.x], c.w * HL_.h[c.x], HL_.h[c.x], lo, hi);
            if (c.x >= lmax_ || lo > rad_) {
                per[c.x].push_back(c);
                per_src[c.x].push_back(static_cast<int32_t>(i));
                continue;
            }
            stack.assign(1, c);
            while (!stack.empty()) {
                const int4 q = stack.back();
                stack.pop_back();
                bool refine = q.x < lmax_;
                if (refine) {
                    box_range(q.y * HL_.h[q.x], q.z * HL_.h[q.x], q.w * HL_.h[q.x], HL_.h[q.x], lo, hi);
                    refine = lo <= rad_;
                }
                if (!refine) {
                    per[q.x].push_back(q);
                    per_src[q.x].push_back(-1);
                    continue;
                }
                for (int dz = 2; dz >= 0; --dz)
                    for (int dy = 2; dy >= 0; --dy)
                        for (int dx = 2; dx >= 0; --dx)
                            stack.push_back(make_int4(q.x + 1, 3 * q.y + dx, 3 * q.z + dy, 3 * q.w + dz));
            }
        }
        mark("existed flags + host walk of the leaves below lmax");
        // head = the new leaves below lmax + the generated level-lmax leaves
        std::vector<int4> head;
        std::vector<int32_t> src, fresh;
        for (int l = 0; l <= lmax_; ++l) {
            per_level_[l] = static_cast<int64_t>(per[l].size()) + (l == lmax_ ? n_top_old : 0);
            head.insert(head.end(), per[l].begin(), per[l].end());
            src.insert(src.end(), per_src[l].begin(), per_src[l].end());
        }
        const int64_t n_head = static_cast<int64_t>(head.size());
        leaves_.assign(head.begin(), head.end() - static_cast<int64_t>(per[lmax_].size()));
        n_leaves_ = n_head + n_top_old;
        if (n_leaves_ > static_cast<int64_t>(INT32_MAX)) throw Error(LZB_ERR_RESOURCE, "too many leaves");
        for (int64_t i = 0; i < n_head; ++i)
            if (src[i] < 0) fresh.push_back(static_cast<int32_t>(i));
        DevBuf<int32_t> dsrc(n_leaves_);
        DevBuf<int4> dl2(n_leaves_);
        if (n_head) {
            LZB_CUDA(cudaMemcpyAsync(dsrc.p, src.data(), n_head * sizeof(int32_t), cudaMemcpyHostToDevice, s_));
            LZB_CUDA(cudaMemcpyAsync(dl2.p, head.data(), n_head * sizeof(int4), cudaMemcpyHostToDevice, s_));
        }
        if (n_top_old) {
            LZB_LAUNCH(k4_iota, blocks_for(n_top_old, 256), 256, 0, s_, dsrc.p + n_head, n_top_old,
                       static_cast<int32_t>(n_lo_old));
            LZB_CUDA(cudaMemcpyAsync(dl2.p + n_head, dleaves_.p + n_lo_old, n_top_old * sizeof(int4),
                                     cudaMemcpyDeviceToDevice, s_));
        }
        DevBuf<double> op2(static_cast<size_t>(n_leaves_) * kCls3);
        DevBuf<int8_t> p32(n_leaves_);
        DevBuf<int32_t> n2(n_leaves_);
        LZB_LAUNCH(k4_gather_leaves, blocks_for(n_leaves_, 256), 256, 0, s_, dsrc.p, n_leaves_, n_old, op_.p, p3_.p,
                   n_.p, op2.p, p32.p, n2.p);
        LZB_CUDA(cudaStreamSynchronize(s_));
        op_ = std::move(op2);
        p3_ = std::move(p32);
        n_ = std::move(n2);
        dleaves_ = std::move(dl2);
        mark("upload + gather of the leaf arrays");
        n_shell_ = 0;  // the shell list indexed the old leaves
        if (!fresh.empty()) {  // the new leaves: assembled now
            shell_.alloc(fresh.size());
            LZB_CUDA(cudaMemcpy(shell_.p, fresh.data(), fresh.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
            n_shell_ = static_cast<int64_t>(fresh.size());
            assemble(n, true);
            n_shell_ = 0;
        }
        mark("assembly of the new leaves");
        if (cyc) {
            setup_levels();
            mark("setup_levels");
            for (int l = 1; l <= lmax_; ++l)  // coarse levels first: interpolation chains through
                LZB_LAUNCH(k4_new_vertices, vgA(l), 128, 0, s_, lv(l), lv(l - 1), existed[l].p);
            refresh_ops();
            mark("new vertices + refresh_ops");
            finish_cycle();
            for (int l = 0; l <= lmax_; ++l)
                LZB_LAUNCH(k4_load, vgA(l), 128, 0, s_, lv(l), rhs_scale_, A_[l].h * A_[l].h * A_[l].h / 8.0);
        }
        sync();
        return static_cast<int64_t>(fresh.size());
    }

    // the leaves' current operators into the levels, then the Galerkin chain
    void refresh_ops() {
        for (int l = 0; l <= lmax_; ++l)
            LZB_LAUNCH(k4_copy_leaf_ops, blocks_for(n_leaves_, 256), 256, 0, s_, dleaves_.p, n_leaves_, l, op_.p,
                       n_leaves_, lv(l));
        for (int l = lmax_ - 1; l >= 0; --l)
            LZB_LAUNCH(k4_galerkin, blocks_for(A_[l].nc, 256), 256, 0, s_, lv(l), lv(l + 1));
    }

    lzb_cycle_report step() {
        if (A_.empty()) throw Error(LZB_ERR_INVALID, "call init_cycle first");
        const int D = lmax_;
        lzb_cycle_report rep;
        std::memset(&rep, 0, sizeof rep);
        rep.cycle = static_cast<int32_t>(++cycle_);
        for (int l = 0; l <= D; ++l) LZB_LAUNCH(k4_reset_fl, vgA(l), 128, 0, s_, lv(l));
        for (int l = D; l >= 0; --l) {
            LZB_LAUNCH(k4_uhat, vgA(l), 128, 0, s_, lv(l), l > 0 ? lv(l - 1) : lv(l), l > 0 ? 1 : 0);
            LZB_LAUNCH(k4_residual, vgA(l), 128, 0, s_, lv(l));
            if (l > 0) LZB_LAUNCH(k4_restrict, vgA(l - 1), 128, 0, s_, lv(l), lv(l - 1));
        }
        double s2 = 0.0;
        std::vector<double> part(kNormBlocksA);
        for (int l = 0; l <= D; ++l) {
            LZB_LAUNCH(k4_norm_partial, kNormBlocksA, 256, 0, s_, lv(l), partialA_.p);
            LZB_CUDA(cudaMemcpyAsync(part.data(), partialA_.p, kNormBlocksA * sizeof(double), cudaMemcpyDeviceToHost,
                                     s_));
            LZB_CUDA(cudaStreamSynchronize(s_));
            for (double x : part) s2 += x;
        }
        rep.residual = std::sqrt(s2);
        if (history_.empty()) first_ = rep.residual > 0.0 ? rep.residual : 1.0;
        history_.push_back(rep.residual);
        rep.normalized = rep.residual / first_;
        rep.status = rep.normalized <= target_ ? LZB_CONVERGED
                     : rep.normalized >= 1e2 ? LZB_DIVERGED
                     : static_cast<int>(cycle_) >= max_cycles_ ? LZB_TIMEOUT : LZB_CONTINUE;
        if (rep.status == LZB_CONTINUE || rep.status == LZB_TIMEOUT) {
            const bool pi = variant_ == LZB_ADAFAC_PI;
            for (int l = 0; l <= D; ++l) LZB_LAUNCH(k4_snap, vgA(l), 128, 0, s_, lv(l));
            for (int l = D; l >= 0; --l) {
                if (pi && l > 0) LZB_LAUNCH(k4_aux_inject, vgA(l - 1), 128, 0, s_, lv(l), lv(l - 1));
                const double damping = variant_ == LZB_ADDITIVE ? std::pow(omega_, D - l + 1) : omega_;
                LZB_LAUNCH(k4_update, vgA(l), 128, 0, s_, lv(l), l > 0 ? lv(l - 1) : lv(l), pi && l > 0 ? 1 : 0,
                           omega_, damping, 1, 0);
            }
            for (int l = 1; l <= D; ++l)
                LZB_LAUNCH(k4_update, vgA(l), 128, 0, s_, lv(l), lv(l - 1), 0, omega_, 0.0, 0, 1);
            finish_cycle();
        }
        rep.levels = D + 1;
        rep.cells = static_cast<uint64_t>(n_leaves_);
        sync();
        return rep;
    }

    void vertices(int level, int field, double* out) {
        if (A_.empty() || level < 0 || level > lmax_ || field < 0 || field >= LZB_V_NFIELDS)
            throw Error(LZB_ERR_INVALID, "bad level / field");
        LZB_CUDA(cudaMemcpyAsync(out, A_[level].v[field].p, A_[level].v[field].bytes(), cudaMemcpyDeviceToHost, s_));
        sync();
    }

    void sync() {
        LZB_CUDA(cudaStreamSynchronize(s_));
        int flag = 0;
        LZB_CUDA(cudaMemcpy(&flag, ctx_->err.p, sizeof(int), cudaMemcpyDeviceToHost));
        if (flag) {
            LZB_CUDA(cudaMemset(ctx_->err.p, 0, sizeof(int)));
            throw Error(LZB_ERR_PROTOCOL, "cannot encode non-finite operator entry");
        }
    }

private:
    struct LevA {
        int N = 1;
        int64_t nc = 1, nv = 8, nop = 0;
        double h = 1.0;
        DevBuf<double> v[LZB_V_NFIELDS];
        DevBuf<double> load, op;
        DevBuf<uint8_t> vk, cf;
        DevBuf<int32_t> oi;
        int box[6] = {0, 2, 0, 2, 0, 2};  // vertex ranges [x0, x1), [y0, y1), [z0, z1)
    };
    static constexpr int kNormBlocksA = 148 * 2;
    std::vector<LevA> A_;
    DevBuf<double> partialA_;
    int variant_ = LZB_ADDITIVE, max_cycles_ = 100;
    double omega_ = 0.6, target_ = 1e-10, first_ = 1.0, rhs_scale_ = 0.0;
    uint32_t cycle_ = 0;
    std::vector<double> history_;

    LvA lv(int l) {
        LvA v{};
        LevA& L = A_[l];
        v.N = L.N;
        v.h = L.h;
        for (int f = 0; f < LZB_V_NFIELDS; ++f) v.v[f] = L.v[f].p;
        v.load = L.load.p;
        v.cf = L.cf.p;
        v.oi = L.oi.p;
        v.op = L.op.p;
        v.nop = L.nop;
        v.vk = L.vk.p;
        v.bx0 = L.box[0];
        v.bx1 = L.box[1];
        v.by0 = L.box[2];
        v.by1 = L.box[3];
        v.bz0 = L.box[4];
        v.bz1 = L.box[5];
        return v;
    }
    dim3 vgA(int l) const {
        const LevA& L = A_[l];
        return dim3(blocks_for(L.box[1] - L.box[0], 128), L.box[3] - L.box[2], L.box[5] - L.box[4]);
    }
    // injection (finest first) where the fine vertex exists, then the hanging
    // vertices of every level from their parents (solver.cpp:344-347)
    void finish_cycle() {
        for (int l = lmax_; l >= 1; --l) LZB_LAUNCH(k4_inject, vgA(l - 1), 128, 0, s_, lv(l), lv(l - 1));
        for (int l = 1; l <= lmax_; ++l) LZB_LAUNCH(k4_hanging, vgA(l), 128, 0, s_, lv(l), lv(l - 1));
    }

    Ball3 ball() const { return Ball3{{cen_[0], cen_[1], cen_[2]}}; }
    // distance range [lo, hi] from the sphere centre to the points of a box
    void box_range(double x0, double y0, double z0, double h, double& lo, double& hi) const {
        const double b[3][2] = {{x0, x0 + h}, {y0, y0 + h}, {z0, z0 + h}};
        double near2 = 0.0, far2 = 0.0;
        for (int d = 0; d < 3; ++d) {
            const double c = cen_[d];
            const double q = std::min(std::max(c, b[d][0]), b[d][1]);
            near2 += (q - c) * (q - c);
            const double f = std::max(std::abs(b[d][0] - c), std::abs(b[d][1] - c));
            far2 += f * f;
        }
        lo = std::sqrt(near2);
        hi = std::sqrt(far2);
    }

    // refinement: every cell below lbase; below lmax the cells meeting the ball
    void build() {
        std::vector<int4> cur{make_int4(0, 0, 0, 0)}, next;
        for (int l = 0; l <= lmax_; ++l) {
            next.clear();
            for (const int4& c : cur) {
                bool refine = l < lbase_;
                if (!refine && l < lmax_) {
                    double lo, hi;
                    box_range(c.y * HL_.h[l], c.z * HL_.h[l], c.w * HL_.h[l], HL_.h[l], lo, hi);
                    refine = lo <= rad_;
                }
                if (!refine) {
                    leaves_.push_back(c);
                    ++per_level_[l];
                    continue;
                }
                for (int dz = 0; dz < 3; ++dz)
                    for (int dy = 0; dy < 3; ++dy)
                        for (int dx = 0; dx < 3; ++dx)
                            next.push_back(make_int4(l + 1, 3 * c.y + dx, 3 * c.z + dy, 3 * c.w + dz));
            }
            cur.swap(next);
            if (cur.empty()) break;
        }
        if (leaves_.size() > static_cast<size_t>(INT32_MAX)) throw Error(LZB_ERR_RESOURCE, "too many leaves");
    }

    lzb_ctx* ctx_;
    cudaStream_t s_ = nullptr;
    int lbase_, lmax_;
    double delta_;
    int fixed_, n_hi_ = 0;
    double cen_[3] = {0.5, 0.5, 0.5}, rad_ = 0.0;
    Field3 F_{};
    LeafLevels HL_{};
    std::vector<int4> leaves_;  // host copy of the level-major prefix: the leaves below lmax
    int64_t per_level_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t n_leaves_ = 0, n_shell_ = 0;
    DevBuf<double> table_, op_;
    DevBuf<int4> dleaves_;
    std::vector<DevBuf<uint8_t>> existed_;  // refine(): which vertices existed before the event
    DevBuf<int32_t> scan_in_;          // setup_levels scratch (existence flags of a level's cells)
    DevBuf<unsigned char> scan_tmp_;   // cub scan workspace
    DevBuf<int32_t> shell_, n_;
    DevBuf<int8_t> p3_;
    DevBuf<unsigned long long> stats_;
};

}  // namespace lzb

struct lzb_tree3 {
    std::unique_ptr<lzb::Tree3> t;
};

extern "C" {

int lzb_tree3_create(lzb_ctx* ctx, int lbase, int lmax, const lzb_field3* f, double delta_max, int fixed_p3,
                     lzb_tree3** out) { LZB_RANGE("lzb_tree3_create");
    return lzb::guarded([&] {
        auto t = std::make_unique<lzb_tree3>();
        t->t = std::make_unique<lzb::Tree3>(ctx, lbase, lmax, *f, delta_max, fixed_p3);
        *out = t.release();
    });
}
int lzb_tree3_destroy(lzb_tree3* t) {
    return lzb::guarded([&] { delete t; });
}
int lzb_tree3_counts(lzb_tree3* t, int64_t* per_level, int64_t* total) { LZB_RANGE("lzb_tree3_counts");
    return lzb::guarded([&] { t->t->counts(per_level, total); });
}
int lzb_tree3_assemble(lzb_tree3* t, int n) { LZB_RANGE("lzb_tree3_assemble");
    return lzb::guarded([&] {
        t->t->assemble(n, false);
        t->t->sync();
    });
}
int lzb_tree3_set_shell(lzb_tree3* t, double band, int64_t* count) { LZB_RANGE("lzb_tree3_set_shell");
    return lzb::guarded([&] { *count = t->t->set_shell(band); });
}
int lzb_tree3_assemble_shell(lzb_tree3* t, int n) { LZB_RANGE("lzb_tree3_assemble_shell");
    return lzb::guarded([&] {
        t->t->assemble(n, true);
        t->t->sync();
    });
}
int lzb_tree3_stats(lzb_tree3* t, lzb_compression_stats* out) { LZB_RANGE("lzb_tree3_stats");
    return lzb::guarded([&] { *out = t->t->stats(); });
}
int lzb_tree3_cells(lzb_tree3* t, int64_t first, int64_t count, double* ops, int32_t* p3, int32_t* n,
                    int32_t* lxyz) { LZB_RANGE("lzb_tree3_cells");
    return lzb::guarded([&] { t->t->cells(first, count, ops, p3, n, lxyz); });
}
int lzb_tree3_init_cycle(lzb_tree3* t, int variant, double omega, double rhs_scale, uint64_t noise_seed,
                         int max_cycles, double target) {
    return lzb::guarded([&] { t->t->init_cycle(variant, omega, rhs_scale, noise_seed, max_cycles, target); });
}
int lzb_tree3_refine(lzb_tree3* t, double radius, int n, int64_t* new_leaves) { LZB_RANGE("lzb_tree3_refine");
    return lzb::guarded([&] {
        const int64_t k = t->t->refine(radius, n);
        if (new_leaves) *new_leaves = k;
    });
}
int lzb_tree3_refresh_ops(lzb_tree3* t) { LZB_RANGE("lzb_tree3_refresh_ops");
    return lzb::guarded([&] {
        t->t->refresh_ops();
        t->t->sync();
    });
}
int lzb_tree3_step(lzb_tree3* t, lzb_cycle_report* out) { LZB_RANGE("lzb_tree3_step");
    return lzb::guarded([&] { *out = t->t->step(); });
}
int lzb_tree3_vertices(lzb_tree3* t, int level, int field, double* out) { LZB_RANGE("lzb_tree3_vertices");
    return lzb::guarded([&] { t->t->vertices(level, field, out); });
}

}  // extern "C"

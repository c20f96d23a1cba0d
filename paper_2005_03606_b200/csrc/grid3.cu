// grid3.cu — the restated 3D extension of the delayed-assembly hot path
// (BASELINE configs[2..4]). The reference is 2D only
// (types.hpp:13), so this follows the survey's restatement:
// trilinear hexahedra on regular 3^l grids, eps sampled at the n^3 sub-cell
// centres, the exact sub-box stiffness of every sample (the 3D form of
// reference_subcell_stiffness, element.cpp:19-32), and the 2D record coding
// (surplus over A(n=1), codec widths, stream.cpp:82-132) on 64-entry records.
//
// Corner a = ax + 2 ay + 4 az, phi_a = X_ax(x) Y_ay(y) Z_az(z), X_0 = 1 - t,
// X_1 = t on the unit cell. With S_c(i) = seg_int over sub-interval i for the
// pair class c (00, 01, 11) and the derivative products s = +-1:
//   K_ab = h/n * ( s_x A_yz[c_y][c_z] + s_y A_xz[c_x][c_z] + s_z A_xy[c_x][c_y] )
//   A_yz = sum_ijk eps_ijk S_y(j) S_z(k), A_xz = sum eps S_x(i) S_z(k),
//   A_xy = sum eps S_x(i) S_y(j)
// accumulated with partial sums over the innermost axis (4 flops per sample,
// not 27 per entry), so the per-sample cost is the eps evaluation.
//
// Layout in HBM: cell operators as class records (the 27 distinct values of
// the 8x8 matrix, padded to 28 doubles = 224 B per cell), index
// (cz*N + cy)*N + cx; markers p3 (i8), n (i32).
#include <cuda.h>

#include <complex>
#include <type_traits>
#include <memory>
#include <vector>

namespace lzb {
namespace {

constexpr int kMaxN3 = 16;

struct Field3 {
    int kind, n;
    double value;
    const double* grf;  // device, n^3
    // the same table x-fastest and padded periodically to (n + 1)^3 (entry n =
    // entry 0 per axis), after the n^3 table: value (i, j, k) at
    // (k (n + 1) + j) (n + 1) + i. The 8 corners of a sample are then at fixed
    // offsets from one base index (no wrap), and the cells of a warp (consecutive
    // x) read neighbouring words.
    const double* grf_t;
    lzb_field xy;
    double cx, cy, cz, radius, width, eps_in, eps_out;  // SPHERE
};

// 2 atanh(0.8): s(t) = (1 + tanh(k t)) / 2 goes from 0.1 to 0.9 over t in [-1/2, 1/2]
constexpr double kSphereK = 2.1972245773362196;

// eps for the 3D kinds (lzb_field3); the GRF is exp of the periodic
// trilinear interpolant of the table, lerp(a, b, t) = (1 - t) a + t b.
__device__ inline double eps3(const Field3& F, double x, double y, double z) {
    if (F.kind == LZB_F3_GRF) {
        const int n = F.n;
        const double ux = x * n, uy = y * n, uz = z * n;
        const double fx = floor(ux), fy = floor(uy), fz = floor(uz);
        const double tx = ux - fx, ty = uy - fy, tz = uz - fz;
        int i0 = static_cast<int>(fx) % n, j0 = static_cast<int>(fy) % n, k0 = static_cast<int>(fz) % n;
        i0 += i0 < 0 ? n : 0;
        j0 += j0 < 0 ? n : 0;
        k0 += k0 < 0 ? n : 0;
        const int i1 = i0 + 1 == n ? 0 : i0 + 1, j1 = j0 + 1 == n ? 0 : j0 + 1, k1 = k0 + 1 == n ? 0 : k0 + 1;
        const double* T = F.grf;
        auto at = [&](int i, int j, int k) { return __ldg(T + (static_cast<int64_t>(i) * n + j) * n + k); };
        auto lerp = [](double a, double b, double t) { return (1.0 - t) * a + t * b; };
        const double c00 = lerp(at(i0, j0, k0), at(i0, j0, k1), tz), c01 = lerp(at(i0, j1, k0), at(i0, j1, k1), tz);
        const double c10 = lerp(at(i1, j0, k0), at(i1, j0, k1), tz), c11 = lerp(at(i1, j1, k0), at(i1, j1, k1), tz);
        const double g = lerp(lerp(c00, c01, ty), lerp(c10, c11, ty), tx);
        return exp(g);
    }
    if (F.kind == LZB_F3_EXTRUDED) return field_eval(F.xy, x, y);
    if (F.kind == LZB_F3_SPHERE) {
        const double dx = x - F.cx, dy = y - F.cy, dz = z - F.cz;
        const double t = (F.radius - sqrt(dx * dx + dy * dy + dz * dz)) / F.width;
        return F.eps_out + (F.eps_in - F.eps_out) * (0.5 * (1.0 + tanh(kSphereK * t)));
    }
    return F.value;
}

// Per-axis seg_int classes (00, 01, 11) of the n sub-intervals.
struct AxisTab3 {
    double s[kMaxN3][3];
    int n;
};

AxisTab3 axis_tab3(int n) {
    AxisTab3 T{};
    T.n = n;
    const double inv = 1.0 / n;
    for (int i = 0; i < n; ++i) {
        const AxisSeg a = axis_seg(i, inv);
        T.s[i][0] = a.s0;
        T.s[i][1] = a.s1;
        T.s[i][2] = a.s2;
    }
    return T;
}

struct Acc3 {
    double yz[9], xz[9], xy[9];
};

// The GRF eps of a cell's samples, separably: a cell is smaller than a
// table spacing (h n_g < 1), so its samples touch the table points b, b+1,
// b+2 per axis. Per sample row i the 3x3 (y, z) points are interpolated in
// x, per (i, j) the 3 z points in y, per sample the z lerp and the exp: 18
// table loads per row instead of 8 per sample. The trilinear interpolant is
// the same function as eps3's (the lerps run in x, y, z order instead of z, y, x).
struct GrfCell {
    const double* T;
    int n, bx, by, bz;  // lower table point per axis
    double X[3][3];     // at the current x: (y point, z point)
    double Y[3];        // at the current (x, y): z point

    __device__ GrfCell(const Field3& F, double x0, double y0, double z0) : T(F.grf), n(F.n) {
        bx = static_cast<int>(floor(x0 * n));
        by = static_cast<int>(floor(y0 * n));
        bz = static_cast<int>(floor(z0 * n));
    }
    __device__ __forceinline__ int wrap(int i) const { return i >= n ? i - n : i; }
    // (1 - t) a + t b with the second product fused (the GRF paths are a
    // restatement: one formula for every GRF sample, grf_sample below included)
    __device__ __forceinline__ static double lerp(double a, double b, double t) { return fma(t, b, (1.0 - t) * a); }
    __device__ __forceinline__ void set_x(double x) {
        const double u = x * n, f = floor(u);
        const int o = static_cast<int>(f) - bx;  // 0 or 1
        const double t = u - f;
        const int i0 = wrap(bx + o), i1 = wrap(bx + o + 1);
#pragma unroll
        for (int jy = 0; jy < 3; ++jy)
#pragma unroll
            for (int kz = 0; kz < 3; ++kz) {
                const int64_t jk = static_cast<int64_t>(wrap(by + jy)) * n + wrap(bz + kz);
                X[jy][kz] = lerp(__ldg(T + static_cast<int64_t>(i0) * n * n + jk),
                                 __ldg(T + static_cast<int64_t>(i1) * n * n + jk), t);
            }
    }
    __device__ __forceinline__ void set_y(double y) {
        const double u = y * n, f = floor(u);
        const bool o = static_cast<int>(f) != by;
        const double t = u - f;
#pragma unroll
        for (int kz = 0; kz < 3; ++kz) Y[kz] = lerp(o ? X[1][kz] : X[0][kz], o ? X[2][kz] : X[1][kz], t);
    }
    __device__ __forceinline__ double eps(double z) const {
        const double u = z * n, f = floor(u);
        const bool o = static_cast<int>(f) != bz;
        const double t = u - f;
        return exp(lerp(o ? Y[1] : Y[0], o ? Y[2] : Y[1], t));
    }
};

// Along a sample row (fixed x, y) the interpolant g is linear in z inside
// each table interval, so exp(g) at the equally spaced z samples is a
// geometric sequence: per row and interval one exp for the first sample and
// one for the ratio exp(dg), then a multiply per sample (a cell spans at most
// two z intervals). Relative error <= n ulps against one exp per sample.
__device__ inline void accumulate3_grf(const Field3& F, double x0, double y0, double z0, double h,
                                       const AxisTab3& T, Acc3& A) {
    const int n = T.n;
    const double inv = 1.0 / n;
    GrfCell G3(F, x0, y0, z0);
    // first z sample in the upper table interval (n if none), and the z
    // parameters of the first sample of each interval
    int ks = n;
    for (int k = 0; k < n; ++k)
        if (static_cast<int>(floor((z0 + (k + 0.5) * inv * h) * F.n)) != G3.bz) {
            ks = k;
            break;
        }
    auto tz = [&](int k) {
        const double u = (z0 + (k + 0.5) * inv * h) * F.n;
        return u - floor(u);
    };
    const double t0 = tz(0), t1 = ks < n ? tz(ks) : 0.0;
    const double dt = inv * h * F.n;  // the z parameter step between samples
#pragma unroll
    for (int q = 0; q < 9; ++q) A.yz[q] = A.xz[q] = A.xy[q] = 0.0;
    for (int i = 0; i < n; ++i) {
        G3.set_x(x0 + (i + 0.5) * inv * h);
        double B[3] = {0.0, 0.0, 0.0}, Cc[3] = {0.0, 0.0, 0.0};
        for (int j = 0; j < n; ++j) {
            G3.set_y(y0 + (j + 0.5) * inv * h);
            double G = 0.0, Dz[3] = {0.0, 0.0, 0.0};
            double e = exp(GrfCell::lerp(G3.Y[0], G3.Y[1], t0));
            double r = exp((G3.Y[1] - G3.Y[0]) * dt);
            for (int k = 0; k < n; ++k) {
                if (k == ks) {
                    e = exp(GrfCell::lerp(G3.Y[1], G3.Y[2], t1));
                    r = exp((G3.Y[2] - G3.Y[1]) * dt);
                }
                G += e;
#pragma unroll
                for (int c = 0; c < 3; ++c) Dz[c] += e * T.s[k][c];
                e *= r;
            }
#pragma unroll
            for (int cy = 0; cy < 3; ++cy) {
#pragma unroll
                for (int cz = 0; cz < 3; ++cz) A.yz[cy * 3 + cz] += T.s[j][cy] * Dz[cz];
                Cc[cy] += T.s[j][cy] * G;
                B[cy] += Dz[cy];
            }
        }
#pragma unroll
        for (int cx = 0; cx < 3; ++cx)
#pragma unroll
            for (int c2 = 0; c2 < 3; ++c2) {
                A.xz[cx * 3 + c2] += T.s[i][cx] * B[c2];
                A.xy[cx * 3 + c2] += T.s[i][cx] * Cc[c2];
            }
    }
}

// ---- GRF samples of small cells, one sample at a time (h n_g < 1)
// Per axis the sample's table interval o (0 .. n - 1) and parameter t.
struct GAx {
    double t;
    int o;
};
template <bool WRAP>
__device__ __forceinline__ GAx grf_axis(double x, int n) {
    const double u = x * n, f = floor(u);
    GAx a;
    a.t = u - f;
    a.o = static_cast<int>(f);
    if (WRAP) {  // arbitrary boxes (lzb_integrate_elements3); grid cells lie in [0, 1)
        a.o %= n;
        a.o += a.o < 0 ? n : 0;
    }
    return a;
}
// exp of the trilinear interpolant at one sample: 8 loads at fixed offsets of
// the padded x-fastest table, lerps in x, y, z order (GrfCell's order and
// formula: the same bits).
__device__ __forceinline__ double grf_sample(const double* __restrict__ Tp, int np, const GAx& ax, const GAx& ay,
                                             const GAx& az) {
    const double* p = Tp + (az.o * np + ay.o) * np + ax.o;
    const int np2 = np * np;
    const double a000 = __ldg(p), a100 = __ldg(p + 1), a010 = __ldg(p + np), a110 = __ldg(p + np + 1);
    const double a001 = __ldg(p + np2), a101 = __ldg(p + np2 + 1), a011 = __ldg(p + np2 + np),
                 a111 = __ldg(p + np2 + np + 1);
    const double c00 = GrfCell::lerp(a000, a100, ax.t), c10 = GrfCell::lerp(a010, a110, ax.t);
    const double c01 = GrfCell::lerp(a001, a101, ax.t), c11 = GrfCell::lerp(a011, a111, ax.t);
    const double d0 = GrfCell::lerp(c00, c10, ay.t), d1 = GrfCell::lerp(c01, c11, ay.t);
    return exp(GrfCell::lerp(d0, d1, az.t));
}

// The 27 class sums at a compile-time NS samples per axis (NS <= 2: at two
// samples per row the geometric-sequence trick of accumulate3_grf saves no
// exp), every loop unrolled, the sums in accumulate3's order with fused
// multiply-adds. WRAP as grf_axis.
template <int NS, bool WRAP, bool ROLL = false>
__device__ __forceinline__ void accumulate3_grf_direct(const Field3& F, double x0, double y0, double z0, double h,
                                                       const AxisTab3& T, Acc3& A) {
    const double inv = 1.0 / NS;
    const int np = F.n + 1;
    GAx ay[NS], az[NS];
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        ay[i] = grf_axis<WRAP>(y0 + (i + 0.5) * inv * h, F.n);
        az[i] = grf_axis<WRAP>(z0 + (i + 0.5) * inv * h, F.n);
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) A.yz[q] = A.xz[q] = A.xy[q] = 0.0;
    // ROLL: the x-sample loop stays a loop (half the code of the unrolled form)
#pragma unroll(ROLL ? 1 : NS)
    for (int i = 0; i < NS; ++i) {
        const GAx axi = grf_axis<WRAP>(x0 + (i + 0.5) * inv * h, F.n);
        double B[3] = {0.0, 0.0, 0.0}, Cc[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int j = 0; j < NS; ++j) {
            double G = 0.0, Dz[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int k = 0; k < NS; ++k) {
                const double e = grf_sample(F.grf_t, np, axi, ay[j], az[k]);
                G += e;
#pragma unroll
                for (int c = 0; c < 3; ++c) Dz[c] = fma(e, T.s[k][c], Dz[c]);
            }
#pragma unroll
            for (int cy = 0; cy < 3; ++cy) {
#pragma unroll
                for (int cz = 0; cz < 3; ++cz) A.yz[cy * 3 + cz] = fma(T.s[j][cy], Dz[cz], A.yz[cy * 3 + cz]);
                Cc[cy] = fma(T.s[j][cy], G, Cc[cy]);
                B[cy] += Dz[cy];
            }
        }
#pragma unroll
        for (int cx = 0; cx < 3; ++cx)
#pragma unroll
            for (int c2 = 0; c2 < 3; ++c2) {
                A.xz[cx * 3 + c2] = fma(T.s[i][cx], B[c2], A.xz[cx * 3 + c2]);
                A.xy[cx * 3 + c2] = fma(T.s[i][cx], Cc[c2], A.xy[cx * 3 + c2]);
            }
    }
}
// eps at the centre of a small GRF cell (the n = 1 sample)
template <bool WRAP>
__device__ __forceinline__ double grf_centre(const Field3& F, double x0, double y0, double z0, double h) {
    const double inv = 1.0 / 1;
    return grf_sample(F.grf_t, F.n + 1, grf_axis<WRAP>(x0 + (0 + 0.5) * inv * h, F.n),
                      grf_axis<WRAP>(y0 + (0 + 0.5) * inv * h, F.n), grf_axis<WRAP>(z0 + (0 + 0.5) * inv * h, F.n));
}

// The 27 class sums of one cell at n samples per axis.
__device__ inline void accumulate3(const Field3& F, double x0, double y0, double z0, double h, const AxisTab3& T,
                                   Acc3& A) {
    if (F.kind == LZB_F3_GRF && h * F.n < 1.0) {
        accumulate3_grf(F, x0, y0, z0, h, T, A);
        return;
    }
    const int n = T.n;
    const double inv = 1.0 / n;
#pragma unroll
    for (int q = 0; q < 9; ++q) A.yz[q] = A.xz[q] = A.xy[q] = 0.0;
    for (int i = 0; i < n; ++i) {
        const double x = x0 + (i + 0.5) * inv * h;
        double B[3] = {0.0, 0.0, 0.0}, Cc[3] = {0.0, 0.0, 0.0};
        for (int j = 0; j < n; ++j) {
            const double y = y0 + (j + 0.5) * inv * h;
            double G = 0.0, Dz[3] = {0.0, 0.0, 0.0};
            for (int k = 0; k < n; ++k) {
                const double z = z0 + (k + 0.5) * inv * h;
                const double e = eps3(F, x, y, z);
                G += e;
#pragma unroll
                for (int c = 0; c < 3; ++c) Dz[c] += e * T.s[k][c];
            }
#pragma unroll
            for (int cy = 0; cy < 3; ++cy) {
#pragma unroll
                for (int cz = 0; cz < 3; ++cz) A.yz[cy * 3 + cz] += T.s[j][cy] * Dz[cz];
                Cc[cy] += T.s[j][cy] * G;
                B[cy] += Dz[cy];
            }
        }
#pragma unroll
        for (int cx = 0; cx < 3; ++cx)
#pragma unroll
            for (int c2 = 0; c2 < 3; ++c2) {
                A.xz[cx * 3 + c2] += T.s[i][cx] * B[c2];
                A.xy[cx * 3 + c2] += T.s[i][cx] * Cc[c2];
            }
    }
}

// Entry (a, b) of h/n * (s_x A_yz + s_y A_xz + s_z A_xy).
__device__ __forceinline__ double entry3(const Acc3& A, double hn, int a, int b) {
    const int ax = a & 1, ay = (a >> 1) & 1, az = a >> 2, bx = b & 1, by = (b >> 1) & 1, bz = b >> 2;
    const int cx = ax == bx ? 2 * ax : 1, cy = ay == by ? 2 * ay : 1, cz = az == bz ? 2 * az : 1;
    const double sx = ax == bx ? 1.0 : -1.0, sy = ay == by ? 1.0 : -1.0, sz = az == bz ? 1.0 : -1.0;
    return hn * (sx * A.yz[cy * 3 + cz] + sy * A.xz[cx * 3 + cz] + sz * A.xy[cx * 3 + cy]);
}

__global__ void k_elements3(Field3 F, int64_t count, const double* x0, const double* y0, const double* z0,
                            const double* h, const int32_t* nn, AxisTab3 T, double* out) {
    lzb_pdl_enter();
    const int64_t t = gtid();
    if (t >= count) return;
    if (nn[t] != T.n) return;  // batches are grouped by n on the host
    Acc3 A;
    // the assembly kernels' path for each case (k_assemble3): the same bits
    const bool small = F.kind == LZB_F3_GRF && h[t] * F.n < 1.0;
    if (small && T.n == 1) accumulate3_grf_direct<1, true>(F, x0[t], y0[t], z0[t], h[t], T, A);
    else if (small && T.n == 2) accumulate3_grf_direct<2, true>(F, x0[t], y0[t], z0[t], h[t], T, A);
    else accumulate3(F, x0[t], y0[t], z0[t], h[t], T, A);
    const double hn = h[t] * (1.0 / T.n);
    for (int a = 0; a < 8; ++a)
        for (int b = 0; b < 8; ++b) out[64 * t + 8 * a + b] = entry3(A, hn, a, b);
}

// Class index of entry (a, b): q = 9 c_x + 3 c_y + c_z, per axis c = 0 (both
// corners 0), 1 (different), 2 (both 1).
__host__ __device__ __forceinline__ int cls3(int a, int b) {
    const int ax = a & 1, ay = (a >> 1) & 1, az = a >> 2, bx = b & 1, by = (b >> 1) & 1, bz = b >> 2;
    return 9 * (ax == bx ? 2 * ax : 1) + 3 * (ay == by ? 2 * ay : 1) + (az == bz ? 2 * az : 1);
}
// Operators in HBM are class planes: the 27 class values of a cell (the
// distinct values of its 8x8 matrix; trilinear operators built from tensor
// products of symmetric per-axis 2x2 matrices — the elements here and their
// Galerkin products with the tensor-product P — take one value per class for
// any eps), stored plane by plane, value q of cell c at q * nc + c: 216 B per
// cell instead of 512, and the per-vertex gathers of the cycle read whole
// 128-B lines across a warp (consecutive vertices, consecutive cells).
constexpr int kCls3 = 27;

// The 64 entries of a trilinear element take 27 values: entry (a, b)
// depends only on the per-axis pair classes (c = 0: both 0, 1: different,
// 2: both 1), the sign of each term being fixed by its class.
__device__ __forceinline__ double class_value(const Acc3& A, double hn, int cx, int cy, int cz) {
    const double sx = cx == 1 ? -1.0 : 1.0, sy = cy == 1 ? -1.0 : 1.0, sz = cz == 1 ? -1.0 : 1.0;
    return hn * (sx * A.yz[cy * 3 + cz] + sy * A.xz[cx * 3 + cz] + sz * A.xy[cx * 3 + cy]);
}

// eps at the n = 1 sample of a cell, evaluated exactly as accumulate3 does at
// n = 1 (the GrfCell path for GRF cells smaller than a table spacing).
__device__ __forceinline__ double centre_eps3(const Field3& F, double x0, double y0, double z0, double h) {
    const double inv = 1.0 / 1;
    const double x = x0 + (0 + 0.5) * inv * h, y = y0 + (0 + 0.5) * inv * h, z = z0 + (0 + 0.5) * inv * h;
    if (F.kind == LZB_F3_GRF && h * F.n < 1.0) {
        GrfCell G3(F, x0, y0, z0);
        G3.set_x(x);
        G3.set_y(y);
        return G3.eps(z);
    }
    return eps3(F, x, y, z);
}

// A(n=1) in class form from eps(centre): at n = 1 the three class sums of
// accumulate3 are all M[a][b] = s_a (e s_b) (every "0 +" of the loop is exact
// for these positive terms), so class (cx, cy, cz) is
// h (sx M[cy][cz] + sy M[cx][cz] + sz M[cx][cy]) — the bits of class_value on
// the n = 1 sums. The stream baseline (stream.cpp:82-84 in 3D), rebuilt by
// the compressed-plane readers from the stored eps(centre).
struct Base3 {
    double m[3][3];
    double h;
    __device__ __forceinline__ Base3(double e, const double* s, double h_) : h(h_) {
        double es[3];
#pragma unroll
        for (int b = 0; b < 3; ++b) es[b] = e * s[b];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) m[a][b] = s[a] * es[b];
    }
    __device__ __forceinline__ double operator()(int cx, int cy, int cz) const {
        const double tx = cx == 1 ? -m[cy][cz] : m[cy][cz];
        const double ty = cy == 1 ? -m[cx][cz] : m[cx][cz];
        const double tz = cz == 1 ? -m[cx][cy] : m[cx][cy];
        return h * (tx + ty + tz);
    }
};

// ---- compressed class planes (plane_width W > 0, BASELINE configs[4])
// Class q of a leaf is held as the W-byte plane word (grid.cu plane_word) of
// rt = roundtrip(surplus_q, p3): lossless at any W >= p3 (rt has at most the
// m(p3) fraction bits), decoded with the compile-time constants of W. The
// word is split into power-of-two pieces (8 | 4, 2, 1 bytes), each piece an
// array of 27 planes of nc words, so a warp reads 2..8 consecutive bytes per
// cell per piece. The stored operator is Base3(eps centre) + rt, bit for bit
// the FP64 class value (k_assemble3 stores exactly that).
// Storage of the leaf level's per-cell planes (class planes, plane-word
// pieces, eps centre): a 3D array [z][y + 1][x + 1] with one leading pad row
// and column (the TMA tiles of the residual start one cell before the block's
// first vertex; tensor coordinates must not be negative) and the x extent
// padded to xp (a multiple of 16: every row starts 16-byte aligned). nc is the
// storage size of one plane (N (N + 1) xp); a cell's storage index is
// plane_sidx of its linear index.
// woff: the storage index of the first stored cell layer (a z-slab window of
// the leaf level: a rank of the slab decomposition holds only the layers its
// kernels read, Grid3's wz0_ .. wz1_)
__host__ __device__ __forceinline__ int64_t plane_sidx(int64_t c, int N, int xp, int64_t woff = 0) {
    if (!xp) return c;
    const int64_t t = c / N;
    return ((t / N) * (N + 1) + t % N + 1) * xp + c % N + 1 - woff;
}
struct Planes3 {
    uint8_t* base;  // piece arrays back to back, largest piece first
    double* ec;     // eps at the cell centre
    int64_t nc;     // storage elements per plane
    double h;
    double s1[3];  // seg_int classes of the n = 1 sub-interval
    int N, xp;     // cells per axis, padded x extent (0: linear storage)
    int64_t woff;  // storage index of the window's first cell layer (plane_sidx)
};

// c: the cell's storage index (plane_sidx)
template <int W>
__device__ __forceinline__ unsigned long long plane_load3(const Planes3& P, int64_t c, int q) {
    const int64_t i = q * P.nc + c;
    if (W == 8) return __ldg(reinterpret_cast<const unsigned long long*>(P.base) + i);
    unsigned long long w = 0;
    int64_t off = 0;
    int sh = 0;
    if (W & 4) {
        w = __ldg(reinterpret_cast<const uint32_t*>(P.base) + i);
        off += 4 * 27 * P.nc;
        sh = 32;
    }
    if (W & 2) {
        w |= static_cast<unsigned long long>(__ldg(reinterpret_cast<const uint16_t*>(P.base + off) + i)) << sh;
        off += 2 * 27 * P.nc;
        sh += 16;
    }
    if (W & 1) w |= static_cast<unsigned long long>(__ldg(P.base + off + i)) << sh;
    return w;
}
__device__ __forceinline__ void plane_store3(const Planes3& P, int W, int64_t c, int q, unsigned long long w) {
    const int64_t i = q * P.nc + c;
    if (W == 8) {
        reinterpret_cast<unsigned long long*>(P.base)[i] = w;
        return;
    }
    int64_t off = 0;
    if (W & 4) {
        reinterpret_cast<uint32_t*>(P.base)[i] = static_cast<uint32_t>(w);
        w >>= 32;
        off += 4 * 27 * P.nc;
    }
    if (W & 2) {
        reinterpret_cast<uint16_t*>(P.base + off)[i] = static_cast<uint16_t>(w);
        w >>= 16;
        off += 2 * 27 * P.nc;
    }
    if (W & 1) P.base[off + i] = static_cast<uint8_t>(w);
}

// Leaf class sources of the cycle kernels: FP64 planes, or compressed planes
// at width W (27 values of one cell: load(c, out)).
// fetch(c, raw) issues a cell's loads (no use: they stay in flight while the
// caller computes), decode(raw, v) turns them into the 27 class values --
// the z-marching residual prefetches the next cell layer with it.
struct Src64 {
    const double* op;
    int64_t nc;      // storage elements per class plane
    int N = 0, xp = 0;  // padded leaf storage (plane_sidx); 0: linear
    int64_t woff = 0;   // leaf window offset (plane_sidx)
    struct Raw {
        double v[27];
    };
    __device__ __forceinline__ double at(int64_t c, int q) const { return __ldg(op + q * nc + plane_sidx(c, N, xp, woff)); }
    // the same from the cell's coordinates (Nl cells per axis): no 64-bit divisions
    __device__ __forceinline__ double at_xyz(int cx, int cy, int cz, int Nl, int q) const {
        const int64_t sc = xp ? (static_cast<int64_t>(cz) * (N + 1) + cy + 1) * xp + cx + 1 - woff
                              : (static_cast<int64_t>(cz) * Nl + cy) * Nl + cx;
        return __ldg(op + q * nc + sc);
    }
    __device__ __forceinline__ void load27(int64_t c, double* v) const {
        const int64_t s = plane_sidx(c, N, xp, woff);
#pragma unroll
        for (int q = 0; q < 27; ++q) v[q] = __ldg(op + q * nc + s);
    }
    __device__ __forceinline__ void fetch(int64_t c, Raw& r) const {
        const int64_t s = plane_sidx(c, N, xp, woff);
#pragma unroll
        for (int q = 0; q < 27; ++q) r.v[q] = __ldg(op + q * nc + s);
    }
    __device__ __forceinline__ void decode(const Raw& r, double* v) const {
#pragma unroll
        for (int q = 0; q < 27; ++q) v[q] = r.v[q];
    }
    static constexpr int kMinBlocks = 1;
};
template <int W>
struct SrcComp {
    Planes3 P;
    using Word = typename std::conditional<(W <= 4), uint32_t, unsigned long long>::type;
    struct Raw {
        Word w[27];
        double e;
    };
    __device__ __forceinline__ void fetch(int64_t c, Raw& r) const {
        const int64_t sc = plane_sidx(c, P.N, P.xp, P.woff);
#pragma unroll
        for (int q = 0; q < 27; ++q) r.w[q] = static_cast<Word>(plane_load3<W>(P, sc, q));
        r.e = __ldg(P.ec + sc);
    }
    // the roundtrip value of a W-byte plane word (PlaneDec(W), with 32-bit
    // integer work for the words of at most 4 bytes)
    __device__ __forceinline__ static double dec(Word w) {
        if constexpr (W == 8) {
            return __longlong_as_double(static_cast<long long>(w));
        } else if constexpr (W <= 4) {
            // e8 | fraction are contiguous in the word: one shift puts them at
            // bit 20 of the high half, one add rebiases the exponent (no carry
            // into the sign: e8 + 895 < 2048)
            constexpr int m = 8 * (W - 1) - 1;
            constexpr uint32_t body = (1u << (8 * W - 1)) - 1u;
            const uint32_t mag = w & body;
            const uint32_t hi = (m > 20 ? mag >> (m - 20) : mag << (20 - m)) + (895u << 20);
            const uint32_t sg = (w >> (8 * W - 1)) << 31;
            const uint32_t lo = m > 20 ? w << (52 - m) : 0u;
            return w == 0 ? 0.0 : __hiloint2double(static_cast<int>(hi | sg), static_cast<int>(lo));
        } else {
            return PlaneDec(W)(static_cast<unsigned long long>(w));
        }
    }
    __device__ __forceinline__ void decode(const Raw& r, double* v) const {
        const Base3 B(r.e, P.s1, P.h);
#pragma unroll
        for (int q = 0; q < 27; ++q) v[q] = B(q / 9, (q / 3) % 3, q % 3) + dec(r.w[q]);
    }
    __device__ __forceinline__ double at_xyz(int cx, int cy, int cz, int Nl, int q) const {
        return at((static_cast<int64_t>(cz) * Nl + cy) * Nl + cx, q);
    }
    __device__ __forceinline__ double at(int64_t c, int q) const {  // one class value
        const int64_t sc = plane_sidx(c, P.N, P.xp, P.woff);
        const Base3 B(__ldg(P.ec + sc), P.s1, P.h);
        return B(q / 9, (q / 3) % 3, q % 3) + dec(static_cast<Word>(plane_load3<W>(P, sc, q)));
    }
    static constexpr int kMinBlocks = 1;
    __device__ __forceinline__ void load27(int64_t c, double* v) const {
        unsigned long long w[27];
        const int64_t sc = plane_sidx(c, P.N, P.xp, P.woff);
#pragma unroll
        for (int q = 0; q < 27; ++q) w[q] = plane_load3<W>(P, sc, q);
        const Base3 B(__ldg(P.ec + sc), P.s1, P.h);
        const PlaneDec dec(W);
#pragma unroll
        for (int q = 0; q < 27; ++q) v[q] = B(q / 9, (q / 3) % 3, q % 3) + dec(w[q]);
    }
};

// choose_precision over a record's distinct values (duplicates never change
// it), all indices compile-time so the values stay in registers; the same
// algorithm as the device choose_precision (codec.cpp:64-85 semantics).
template <int COUNT>
__device__ __noinline__ int choose_precision_set(const double* v, double delta) {
    return choose_precision(v, COUNT, delta);
}
// The same result in registers for records whose values are all regular
// (finite, normal, exponent in [-128, 127], or +-0: the passing widths of
// each value are upward closed): the running maximum P of the
// per-value smallest passing widths, each value testing only widths >= P.
// Other records take the general routine.
//
// Values with exponent e in [-127, 127] (or +-0) are "plain": no clamp and no
// (0, 0, -128) decode apply, so truncation to m fraction bits is a mask and
// the error is exactly the dropped fraction bits F_low * 2^(e - 52) (rt and v
// share the exponent: the subtraction of the reference test is exact); the
// test |rt - v| <= delta is then F_low <= delta * 2^(52 - e), an integer
// comparison against one exact product per value.
__device__ __forceinline__ bool codec_plain(unsigned long long u) {
    const int E = static_cast<int>((u >> 52) & 0x7ff);
    return (u << 1) == 0 || (E >= 1023 - 127 && E <= 1023 + 127);
}
// the smallest width in [P, 7] a plain value passes, else 8. Branch-free: the
// dropped bits at widths 2..7 are nested masks of F (45, 37, .., 5 bits), so
// the passing widths are upward closed and the smallest one is 2 + the number
// of failing widths; F & mask <= T (real) iff F & mask <= floor(T) (integer,
// the conversion saturates for a huge T)
__device__ __forceinline__ int min_width_plain(unsigned long long u, double delta, int P) {
    if ((u << 1) == 0) return P;  // +-0: error 0 at every width
    const int E = static_cast<int>((u >> 52) & 0x7ff);
    const double T = delta * __longlong_as_double(static_cast<long long>(2098 - E) << 52);  // delta 2^(1075 - E)
    const unsigned long long Ti = __double2ull_rz(T), F = u & 0xFFFFFFFFFFFFFull;
    int w = 2;
#pragma unroll
    for (int q = 2; q <= 7; ++q) w += (F & ((1ull << (52 - mantissa_bits(q))) - 1)) > Ti ? 1 : 0;
    return w > P ? w : P;
}
// roundtrip at width p3 in 2..7 of a plain value: the low fraction bits cleared
__device__ __forceinline__ double rt_plain(unsigned long long u, int p3) {
    if ((u << 1) == 0) return 0.0;  // -0 encodes as +0
    return __longlong_as_double(static_cast<long long>(u & ~((1ull << (52 - mantissa_bits(p3))) - 1)));
}

// plain: every value plain (then the caller may roundtrip with rt_plain)
template <int COUNT>
__device__ __forceinline__ int choose_precision_regular(const double* v, double delta, bool& plain) {
    bool all_small = true;
    plain = true;
#pragma unroll
    for (int i = 0; i < COUNT; ++i) {
        all_small = all_small && !(fabs(v[i]) > delta);
        plain = plain && codec_plain(static_cast<unsigned long long>(__double_as_longlong(v[i])));
    }
    if (all_small) return 0;
    if (!plain) return choose_precision_set<COUNT>(v, delta);
    int P = 2;
#pragma unroll
    for (int i = 0; i < COUNT; ++i)
        P = min_width_plain(static_cast<unsigned long long>(__double_as_longlong(v[i])), delta, P);
    return P;
}
// codec::roundtrip for one value of a record coded at p3 (plain: rt_plain)
__device__ __forceinline__ bool roundtrip_rec(double x, int p3, bool plain, double& rt) {
    if (plain && p3 >= 2 && p3 <= 7) {
        rt = rt_plain(static_cast<unsigned long long>(__double_as_longlong(x)), p3);
        return true;
    }
    return roundtrip_fast(x, p3, rt);
}

// ---- record coding of the 27 class surpluses, shared by the assembly kernels
// Base3's values when the n = 1 seg_int classes are symmetric (s[0] == s[2]
// bit for bit, which holds for the unit interval): class (cx, cy, cz) depends
// on (cx == 1, cy == 1, cz == 1) only, 8 values instead of 27 evaluations.
struct BaseVals {
    double b[8];
    bool sym;
    __device__ __forceinline__ BaseVals(const Base3& B, const double* s) : sym(s[0] == s[2]) {
#pragma unroll
        for (int k = 0; k < 8; ++k) b[k] = B(k >> 2, (k >> 1) & 1, k & 1);
    }
    __device__ __forceinline__ double at(const Base3& B, int cx, int cy, int cz) const {
        return sym ? b[(cx == 1) * 4 + (cy == 1) * 2 + (cz == 1)] : B(cx, cy, cz);
    }
};

// choose_precision (codec.cpp:64-85 semantics) of a record whose values are
// all plain, from the exponents first. A plain value v with biased exponent E
// surely passes width q once the dropped bits are fewer than those of
// T = delta 2^(1075 - E) (mask_q <= floor(T)), i.e. 61 - 8 q <= e_T with
// e_T = E_delta - E + 52: q_sure(E) rises with E, so every value passes at
// P = q_sure(E_max). From there the width walks down while every value still
// passes the reference's own test |rt - v| <= delta at P - 1 (rt: the low
// fraction bits cleared, the subtraction exact): the passing widths of each
// value are upward closed, so the first width at which some
// value fails is one below the answer. Typically one pass of 27 tests.
// Records with a value that is not plain (zero, tiny, huge, non-finite) or a
// non-normal delta take the general routine.
template <int COUNT>
__device__ __forceinline__ int choose_precision_exp(const double* v, double delta, bool& plain) {
    unsigned hmax = 0, hmin = 0x7fffffffu;
#pragma unroll
    for (int i = 0; i < COUNT; ++i) {
        const unsigned hi = static_cast<unsigned>(__double2hiint(v[i])) & 0x7fffffffu;
        hmax = max(hmax, hi);
        hmin = min(hmin, hi);
    }
    const int Emax = static_cast<int>(hmax >> 20), Emin = static_cast<int>(hmin >> 20);
    const int Ed = (__double2hiint(delta) >> 20) & 0x7ff;
    plain = Emin >= 1023 - 127 && Emax <= 1023 + 127;
    if (Emax == 0x7ff || Ed == 0 || Ed == 0x7ff || __double2hiint(delta) < 0) {
        plain = false;
        return choose_precision_set<COUNT>(v, delta);
    }
    if (Emax < Ed) return 0;  // every |v| < 2^(E_delta - 1023) <= delta
    if (Emax == Ed) {  // rare: a rolled loop
        bool all_small = true;
#pragma unroll 1
        for (int i = 0; i < COUNT; ++i) all_small = all_small && !(fabs(v[i]) > delta);
        if (all_small) return 0;
    }
    if (!plain) return choose_precision_set<COUNT>(v, delta);
    const int eT = Ed - Emax + 52;
    int P = min(max((68 - eT) >> 3, 2), 8);
    // (non-negative doubles order as their bit patterns: the comparisons with
    // delta run on the integer pipe, the FP64 pipe keeps the subtractions)
    const unsigned long long dbits = static_cast<unsigned long long>(__double_as_longlong(delta));
    while (P > 2) {
        const unsigned long long keep = ~((1ull << (69 - 8 * P)) - 1);  // width P - 1 drops 61 - 8 (P - 1) bits
        bool fail = false;
#pragma unroll
        for (int i = 0; i < COUNT; ++i) {
            const double rt = __longlong_as_double(__double_as_longlong(v[i]) & static_cast<long long>(keep));
            fail = fail || (static_cast<unsigned long long>(__double_as_longlong(v[i] - rt)) & 0x7fffffffffffffffull) > dbits;
        }
        if (fail) break;
        --P;
    }
    return P;
}

// codec::roundtrip of any value (the rare records with a value that is not plain)
__device__ __noinline__ bool roundtrip_slow(double x, int p3, double& rt) { return roundtrip_fast(x, p3, rt); }

// Codes one record and stores the decoded operator: p3 (chosen or forced),
// per class the roundtrip value, the running delta, then FP64 planes
// (W == 0: B + rt) or the W-byte plane words. Returns p3, or -1 on an error
// (non-finite value: err set; record wider than the planes: wide set).
template <class StoreOp>
__device__ __forceinline__ int code_record27(const double* sur, const Base3& B, const BaseVals& BV, double delta_max,
                                             int fixed_p3, int W, int* err, int* wide, double& delta,
                                             StoreOp&& store) {
    bool plain = false;
    int p3 = choose_precision_exp<27>(sur, delta_max, plain);
    if (fixed_p3) p3 = fixed_p3;
    if (p3 < 0) {
        atomicExch(err, 1);
        return -1;
    }
    if (W != 0 && p3 > W) {
        atomicExch(wide, 1);  // record wider than the planes
        return -1;
    }
    delta = 0.0;
    if (plain || p3 == 0 || p3 == 8) {
        // plain values at widths 2..7: the low fraction bits cleared; 0: every rt is +0; 8: the value
        const unsigned long long keep =
            p3 == 0 ? 0ull : (p3 == 8 ? ~0ull : ~((1ull << (52 - mantissa_bits(p3))) - 1));
        if (p3 == 8) {  // rare: a rolled loop
            bool finite = true;
#pragma unroll 1
            for (int q = 0; q < 27; ++q) finite = finite && dev_isfinite(sur[q]);
            if (!finite) {
                atomicExch(err, 1);
                return -1;
            }
        }
        unsigned long long dmax = 0;  // max |rt - sur| through the bit patterns (integer pipe)
#pragma unroll
        for (int q = 0; q < 27; ++q) {
            const double rt = __longlong_as_double(__double_as_longlong(sur[q]) & static_cast<long long>(keep));
            const unsigned long long d = static_cast<unsigned long long>(__double_as_longlong(rt - sur[q])) & 0x7fffffffffffffffull;
            dmax = d > dmax ? d : dmax;
            store(q, BV.at(B, q / 9, (q / 3) % 3, q % 3), rt);
        }
        delta = __longlong_as_double(static_cast<long long>(dmax));
    } else {
        // rare (a value that is not plain): a rolled loop, out of the hot path's code
#pragma unroll 1
        for (int q = 0; q < 27; ++q) {
            double rt;
            if (!roundtrip_slow(sur[q], p3, rt)) {
                atomicExch(err, 1);
                return -1;
            }
            delta = fmax(delta, fabs(rt - sur[q]));
            store(q, B(q / 9, (q / 3) % 3, q % 3), rt);
        }
    }
    return p3;
}

// Fixed-p assembly of every cell of a 3D level: integrate at n, code the
// record against the n = 1 element (stream.cpp:82-111 in 3D), store the
// decoded operator (FP64 class planes, or eps(centre) + the compressed
// planes of width W), width and n. One thread per cell; the record's 27
// distinct surplus values are coded once (they stand for its 64 entries).
// KIND >= 0: the field kind fixed at compile time (the other kinds' sample
// code is dropped: a smaller kernel, fewer instruction-cache misses).
// NS > 0 (GRF cells smaller than a table spacing): the samples per axis at
// compile time, accumulate3_grf_direct; NS = 0: T.n samples, accumulate3.
// COMP: the leaves are compressed planes (W > 0); false: FP64 class planes
// (the plane-word store code is not instantiated: a third less code).
template <int KIND, int NS, bool COMP, int MINB = 3, bool ROLL = false>
__global__ void __launch_bounds__(128, MINB) k_assemble3(Field3 Fin, int N, double h, AxisTab3 T, double delta_max,
                                                      int fixed_p3, double* __restrict__ op, Planes3 PL, int W,
                                                      int8_t* __restrict__ p3o, int32_t* __restrict__ no,
                                                      unsigned long long* stats, int* err, int* wide,
                                                      int64_t cbeg, int64_t cend) {
    lzb_pdl_enter();
    Field3 F = Fin;
    if (KIND >= 0) F.kind = KIND;
    const int64_t c = cbeg + gtid();  // cells [cbeg, cend): whole z planes
    if (c >= cend) return;
    // (a level has at most 729^3 < 2^31 cells: 32-bit divisions; the storage index
    // straight from the coordinates -- the 64-bit divisions were ~10 % of the p <= 2 kernel)
    const uint32_t cu = static_cast<uint32_t>(c), tq = cu / static_cast<uint32_t>(N);
    const int cx = static_cast<int>(cu - tq * N), cz = static_cast<int>(tq / static_cast<uint32_t>(N)),
              cy = static_cast<int>(tq - static_cast<uint32_t>(cz) * N);
    const int64_t nc = PL.nc;
    const int64_t sc = PL.xp ? (static_cast<int64_t>(cz) * (PL.N + 1) + cy + 1) * PL.xp + cx + 1 - PL.woff : c;
    const double x0 = cx * h, y0 = cy * h, z0 = cz * h;
    const double e = NS > 0 ? grf_centre<false>(F, x0, y0, z0, h) : centre_eps3(F, x0, y0, z0, h);
    const Base3 B(e, PL.s1, h);  // A(n=1): eps(centre) * unit stiffness
    const BaseVals BV(B, PL.s1);
    double sur[27];
    {
        Acc3 A;
        if (NS > 0) accumulate3_grf_direct<(NS > 0 ? NS : 1), false, ROLL>(F, x0, y0, z0, h, T, A);
        else accumulate3(F, x0, y0, z0, h, T, A);
        const double hn = h * (1.0 / T.n);
#pragma unroll
        for (int q = 0; q < 27; ++q)
            sur[q] = class_value(A, hn, q / 9, (q / 3) % 3, q % 3) - BV.at(B, q / 9, (q / 3) % 3, q % 3);
    }
    double delta;
    const int p3 = code_record27(sur, B, BV, delta_max, fixed_p3, W, err, wide, delta, [&](int q, double b, double rt) {
        if constexpr (!COMP) op[q * nc + sc] = b + rt;
        else plane_store3(PL, W, sc, q, plane_word(rt, W));
    });
    if (p3 < 0) return;
    if constexpr (COMP) PL.ec[sc] = e;
    p3o[c] = static_cast<int8_t>(p3);
    no[c] = T.n;
    atomic_max_double_bits(&stats[S_MAXDELTA], delta);
}

// The 27 class values of cells [first, first + count) (AoS, 27 per cell).
template <class Src>
__global__ void k3_read_cls(Src S, int64_t first, int64_t count, double* __restrict__ out) {
    lzb_pdl_enter();
    const int64_t t = gtid();
    if (t >= count) return;
    double v[27];
    S.load27(first + t, v);
#pragma unroll
    for (int q = 0; q < 27; ++q) out[27 * t + q] = v[q];
}

__global__ void k_stats3(const int8_t* __restrict__ p3, int64_t nc, unsigned long long* s) {
    lzb_pdl_enter();
    __shared__ unsigned long long sh[9];
    if (threadIdx.x < 9) sh[threadIdx.x] = 0;
    __syncthreads();
    unsigned h[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t c = gtid(); c < nc; c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int q = p3[c];
#pragma unroll
        for (int b = 0; b <= 8; ++b) h[b] += q == b ? 1u : 0u;
    }
#pragma unroll
    for (int b = 0; b <= 8; ++b) {
        const unsigned w = __reduce_add_sync(0xffffffffu, h[b]);
        if ((threadIdx.x & 31) == 0 && w) atomicAdd(&sh[b], static_cast<unsigned long long>(w));
    }
    __syncthreads();
    if (threadIdx.x < 9 && sh[threadIdx.x]) atomicAdd(&s[S_HIST + threadIdx.x], sh[threadIdx.x]);
}

// ------------------------------------------------------------ 3D cycle
// The additive multilevel cycle of solver.cpp:99-347 restated on regular 3D
// grids (the reference is 2D): hierarchical residual r̂ = fl - A û with
// û = u - P u_c, restriction of r̂ into the coarse load, Jacobi on every
// level, prolongation cascade, injection. Trilinear geometric transfer with
// lattice weights w(L, a) = prod_d (a_d ? L_d : 3 - L_d) / 27 over the 4^3
// lattice points of a patch; a fine vertex belongs to the patch with the
// lowest coordinates that contains it (the 2D owner rule per axis,
// solver.cpp:35-57); Galerkin coarse operators P^T A P (transfer.cpp:81-93).
struct Lv3 {
    int N;
    double h;
    double* v[LZB_V_NFIELDS];
    const double* op;  // class records, kCls3 per cell
    int z0;            // first vertex plane of a z-range launch (blockIdx.z + z0)
};

__device__ __forceinline__ bool vxyz(const Lv3& L, int& ix, int& iy, int& iz, int64_t& vi) {
    ix = blockIdx.x * blockDim.x + threadIdx.x;
    iy = blockIdx.y;
    iz = blockIdx.z + L.z0;
    if (ix > L.N) return false;
    vi = (static_cast<int64_t>(iz) * (L.N + 1) + iy) * (L.N + 1) + ix;
    return true;
}
__device__ __forceinline__ bool bnd3(int N, int ix, int iy, int iz) {
    return ix == 0 || iy == 0 || iz == 0 || ix == N || iy == N || iz == N;
}
__device__ __forceinline__ int64_t vidx3(int N, int x, int y, int z) {
    return (static_cast<int64_t>(z) * (N + 1) + y) * (N + 1) + x;
}
// k / 27 for the integer weight products k = 0..27 (the divisions of the
// trilinear lattice weights, tabulated: the same correctly rounded quotients)
__device__ const double g_w27[28] = {
    0 / 27.0,  1 / 27.0,  2 / 27.0,  3 / 27.0,  4 / 27.0,  5 / 27.0,  6 / 27.0,  7 / 27.0,  8 / 27.0,  9 / 27.0,
    10 / 27.0, 11 / 27.0, 12 / 27.0, 13 / 27.0, 14 / 27.0, 15 / 27.0, 16 / 27.0, 17 / 27.0, 18 / 27.0, 19 / 27.0,
    20 / 27.0, 21 / 27.0, 22 / 27.0, 23 / 27.0, 24 / 27.0, 25 / 27.0, 26 / 27.0, 27 / 27.0};
__device__ __forceinline__ double pw3(int lx, int ly, int lz, int a) {
    return g_w27[((a & 1) ? lx : 3 - lx) * (((a >> 1) & 1) ? ly : 3 - ly) * ((a >> 2) ? lz : 3 - lz)];
}
__device__ __forceinline__ int owner3(int f, int Nc) {
    const int x1 = f / 3;
    const int p = (f - 3 * x1 == 0 && x1 > 0) ? x1 - 1 : x1;
    return p > Nc - 1 ? Nc - 1 : p;
}

// fl = sum over the adjacent leaves of f(v) h^3 / 8, f = scale prod sin(pi x_d)
// (the lumped load of solver.cpp:99-118 in 3D; BASELINE f = 3 pi^2 prod sin)
__global__ void k3_init_rhs(Lv3 F, double scale, double w) {
    lzb_pdl_enter();
    int ix, iy, iz;
    int64_t vi;
    if (!vxyz(F, ix, iy, iz, vi)) return;
    int adj = 0;
    for (int dz = 0; dz < 2; ++dz)
        for (int dy = 0; dy < 2; ++dy)
            for (int dx = 0; dx < 2; ++dx) {
                const int cx = ix - dx, cy = iy - dy, cz = iz - dz;
                adj += (cx >= 0 && cy >= 0 && cz >= 0 && cx < F.N && cy < F.N && cz < F.N);
            }
    const double x = ix * F.h, y = iy * F.h, z = iz * F.h;
    const double term = w * (scale * sin(kPi * x) * sin(kPi * y) * sin(kPi * z));
    double fl = 0.0;
    for (int k = 0; k < adj; ++k) fl += term;
    F.v[LZB_V_FL][vi] = fl;
}

__global__ void k3_noise(Lv3 L, int level, uint64_t seed, double gval) {
    lzb_pdl_enter();
    int ix, iy, iz;
    int64_t vi;
    if (!vxyz(L, ix, iy, iz, vi)) return;
    if (bnd3(L.N, ix, iy, iz)) {
        L.v[LZB_V_U][vi] = gval;
        return;
    }
    auto mix = [](uint64_t z) {
        z += 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    };
    const uint64_t k = mix(seed ^ mix((static_cast<uint64_t>(level) << 48) ^ (static_cast<uint64_t>(ix) << 32) ^
                                      (static_cast<uint64_t>(iy) << 16) ^ static_cast<uint64_t>(iz)));
    L.v[LZB_V_U][vi] = (4.0 / 3.0) * static_cast<double>(k >> 11) * 0x1.0p-53;
}

__global__ void k3_uhat(Lv3 F, Lv3 C, int has_coarse) {
    lzb_pdl_enter();
    int fx, fy, fz;
    int64_t vi;
    if (!vxyz(F, fx, fy, fz, vi)) return;
    const double u = F.v[LZB_V_U][vi];
    if (!has_coarse) {
        F.v[LZB_V_UHAT][vi] = u;
        return;
    }
    const int px = owner3(fx, C.N), py = owner3(fy, C.N), pz = owner3(fz, C.N);
    const int lx = fx - 3 * px, ly = fy - 3 * py, lz = fz - 3 * pz;
    double interp = 0.0;
    for (int a = 0; a < 8; ++a)
        interp += pw3(lx, ly, lz, a) * C.v[LZB_V_U][vidx3(C.N, px + (a & 1), py + ((a >> 1) & 1), pz + (a >> 2))];
    F.v[LZB_V_UHAT][vi] = u - interp;
}

// r, r̂, diag per vertex over the 8 adjacent cells in (z, y, x) order
// (solver.cpp:145-175 restated), cell-centric and z-marching: a block owns a tile of
// 31 x 7 vertex columns and a range of vertex planes; per cell layer every
// thread loads one cell's 27 class values (decoded once, not once per
// adjacent vertex), forms the 8 row products K_a. u and K_a. û of the 8x8
// operator and its diagonal, and stages them in shared memory; the vertex
// threads then subtract them in the gather kernel's order (cells q = dx +
// 2 dy + 4 dz: the 4 cells below a vertex plane while the previous layer is
// staged, the 4 above in this layer) — the per-vertex gather's order. The
// u / û corners of the layer below stay in registers.
constexpr int kRzX = 32, kRzY = 8, kRzChunk = 32;  // chunk: vertex planes per block (at most)
template <class Src>
__global__ void __launch_bounds__(kRzX * kRzY, Src::kMinBlocks) k3_residual_z(Lv3 F, Src S, int zbeg, int zend,
                                                                              int zc) {
    lzb_pdl_enter();
    __shared__ double sy[3][8][kRzX * kRzY];  // [u, û, diag][corner][cell of the tile]
    const int tx = threadIdx.x % kRzX, ty = threadIdx.x / kRzX, t = threadIdx.x;
    const int N = F.N, NV = N + 1;
    const int X0 = blockIdx.x * (kRzX - 1), Y0 = blockIdx.y * (kRzY - 1);
    const int zs = zbeg + blockIdx.z * zc, ze = min(zs + zc, zend);
    if (zs >= ze) return;
    const int cx = X0 - 1 + tx, cy = Y0 - 1 + ty;  // this thread's cell column
    const bool colok = cx >= 0 && cy >= 0 && cx < N && cy < N;
    const int ix = X0 + tx, iy = Y0 + ty;  // this thread's vertex column (tx < 31, ty < 7)
    const bool vthr = tx < kRzX - 1 && ty < kRzY - 1 && ix <= N && iy <= N;
    const double* __restrict__ U = F.v[LZB_V_U];
    const double* __restrict__ UH = F.v[LZB_V_UHAT];
    const double* __restrict__ FL = F.v[LZB_V_FL];
    auto vid = [&](int x, int y, int z) {
        return (static_cast<int64_t>(min(max(z, 0), N)) * NV + min(max(y, 0), N)) * NV + min(max(x, 0), N);
    };
    auto cell = [&](int z) { return (static_cast<int64_t>(z) * N + cy) * N + cx; };
    // software pipeline, one cell layer ahead: the next layer's class values
    // and upper corners and the next vertex plane's load are in flight while
    // the current layer computes (the kernel is latency-bound otherwise)
    double ul[4], uhl[4], un[4], uhn[4];  // corners of the layer's lower / upper plane
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t v0 = vid(cx + (k & 1), cy + (k >> 1), zs - 1), v1 = vid(cx + (k & 1), cy + (k >> 1), zs);
        ul[k] = U[v0];
        uhl[k] = UH[v0];
        un[k] = U[v1];
        uhn[k] = UH[v1];
    }
    typename Src::Raw nxt;
    if (colok && zs - 1 >= 0) S.fetch(cell(zs - 1), nxt);
    double fln = vthr ? FL[vid(ix, iy, zs)] : 0.0;  // plane zs: opened in the first iteration
    double rp = 0.0, rhp = 0.0, dgp = 0.0;  // partial sums of the vertex plane being completed
    for (int cz = zs - 1; cz < ze; ++cz) {
        // 1. this thread's cell of layer cz: row products into shared memory
        double uu[8], uh[8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            uu[k] = ul[k];
            uh[k] = uhl[k];
            uu[4 + k] = un[k];
            uh[4 + k] = uhn[k];
            ul[k] = un[k];
            uhl[k] = uhn[k];
        }
        const typename Src::Raw cur = nxt;
        const bool ok = colok && cz >= 0 && cz < N;
        const double flc = fln;
        if (cz + 1 < ze) {  // the next layer's operands
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t v = vid(cx + (k & 1), cy + (k >> 1), cz + 2);
                un[k] = U[v];
                uhn[k] = UH[v];
            }
            if (colok && cz + 1 < N) S.fetch(cell(cz + 1), nxt);
            if (vthr) fln = FL[vid(ix, iy, cz + 2)];
        }
        if (ok) {
            double K[27];
            S.decode(cur, K);
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                double au = 0.0, auh = 0.0;
#pragma unroll
                for (int col = 0; col < 8; ++col) {  // explicit FMA (the 3D cycle is restated, not pinned bitwise)
                    au = __fma_rn(K[cls3(a, col)], uu[col], au);
                    auh = __fma_rn(K[cls3(a, col)], uh[col], auh);
                }
                sy[0][a][t] = au;
                sy[1][a][t] = auh;
                sy[2][a][t] = K[cls3(a, a)];
            }
        }
        __syncthreads();
        // 2. vertex threads: plane cz (cells above it, q = 4..7) is completed,
        // plane cz + 1 starts (cells below it, q = 0..3)
        if (vthr) {
            auto sub = [&](int q, double& r, double& rh, double& dg) {
                const int dx = q & 1, dy = (q >> 1) & 1, dz = q >> 2;
                const int row = (1 - dx) + 2 * (1 - dy) + 4 * (1 - dz);
                const int ccx = ix - 1 + dx, ccy = iy - 1 + dy;
                if (ccx < 0 || ccy < 0 || ccx >= N || ccy >= N) return;
                const int c = (ty + dy) * kRzX + tx + dx;
                r -= sy[0][row][c];
                rh -= sy[1][row][c];
                dg += sy[2][row][c];
            };
            if (cz >= zs && cz < N) {  // layer cz lies above plane cz
#pragma unroll
                for (int q = 4; q < 8; ++q) sub(q, rp, rhp, dgp);
            }
            if (cz >= zs) {
                double r = rp, rh = rhp;
                if (bnd3(N, ix, iy, cz)) {
                    r = 0.0;
                    rh = 0.0;
                }
                const int64_t vi = (static_cast<int64_t>(cz) * NV + iy) * NV + ix;
                __stcs(F.v[LZB_V_R] + vi, r);
                __stcs(F.v[LZB_V_RHAT] + vi, rh);
                __stcs(F.v[LZB_V_DIAG] + vi, dgp);
            }
            if (cz + 1 < ze) {  // plane cz + 1: fl, then the cells of layer cz below it
                rp = rhp = flc;
                dgp = 0.0;
                if (cz >= 0) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) sub(q, rp, rhp, dgp);
                }
            }
        }
        __syncthreads();
    }
}

// ---- the leaf residual with TMA tile staging (sm_100a: cp.async.bulk.tensor
// + mbarrier). The leaf planes are 4D tensors [class q][z][y][x padded]; per
// cell layer one elected thread issues one tensor copy per plane piece (the
// block's 32 x 8 cells x 27 classes; out-of-range cells are zero-filled by
// the TMA unit) plus, for compressed planes, one of eps(centre), into a
// shared-memory stage armed on an mbarrier; the copy of layer cz + 1 runs
// while the block's threads finish layer cz's vertex sums and open the next
// layer. Each cell thread decodes its own 27 class values from the stage.
// Same products, same sums, same order as k3_residual_z: identical results.
struct TmaMaps {
    CUtensorMap piece[3];  // plane pieces, largest first (FP64: piece 0 = the doubles)
    CUtensorMap ec;        // eps(centre) (compressed planes)
    int z0;                // first stored cell layer (tensor z = cell layer - z0)
};
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
// piece sizes of a plane word of W bytes (W = 0: one piece of FP64 values)
__host__ __device__ constexpr int tma_piece(int W, int k) {
    return W == 0 ? (k == 0 ? 8 : 0)
           : W == 8 ? (k == 0 ? 8 : 0)
                    : (k == 0 ? ((W & 4) ? 4 : (W & 2) ? 2 : 1)
                               : k == 1 ? ((W & 4) ? ((W & 2) ? 2 : (W & 1) ? 1 : 0) : (W & 2) ? ((W & 1) ? 1 : 0) : 0)
                                        : ((W & 4) && (W & 2) && (W & 1)) ? 1 : 0);
}
constexpr int kTmaCells = kRzX * kRzY;  // cells of one layer of a block tile
// A tensor copy's box must start 16-byte aligned in x: the box of a piece of
// e-byte elements starts at the tile's first storage x rounded down to 16 / e
// elements and is 32 + 16 / e elements wide (the tile sits at offset < 16 / e).
__host__ __device__ constexpr int tma_width(int e) { return e ? kRzX + 16 / e : 0; }
__host__ __device__ constexpr int tma_piece_bytes(int e) { return 27 * kRzY * tma_width(e) * e; }
__host__ __device__ constexpr int tma_stage_bytes(int W) {
    return tma_piece_bytes(tma_piece(W, 0)) + tma_piece_bytes(tma_piece(W, 1)) + tma_piece_bytes(tma_piece(W, 2)) +
           (W ? kRzY * tma_width(8) * 8 : 0);
}
__host__ __device__ constexpr int tma_smem_bytes(int W) {
    return 3 * 8 * kTmaCells * 8 + tma_stage_bytes(W) + 16;
}

// The leaf level's Jacobi diagonal (the residual's dg: the 8 adjacent cells'
// diagonal entries, in its order -- the 4 cells below the vertex plane, then
// the 4 above), once per change of the leaf operators: the TMA residual does
// not recompute / rewrite it every cycle.
template <class Src>
__global__ void k3_leaf_diag(Lv3 F, Src S) {
    lzb_pdl_enter();
    int ix, iy, iz;
    int64_t vi;
    if (!vxyz(F, ix, iy, iz, vi)) return;
    const int N = F.N;
    double dg = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int dx = q & 1, dy = (q >> 1) & 1, dz = q >> 2;
        const int row = (1 - dx) + 2 * (1 - dy) + 4 * (1 - dz);
        const int cx = ix - 1 + dx, cy = iy - 1 + dy, cz = iz - 1 + dz;
        if (cx < 0 || cy < 0 || cz < 0 || cx >= N || cy >= N || cz >= N) continue;
        dg += S.at_xyz(cx, cy, cz, N, cls3(row, row));
    }
    F.v[LZB_V_DIAG][vi] = dg;
}

// u / u-hat tiles of a vertex plane (corners of a block's 32 x 8 cells: x from
// the cells' first column rounded down to even, 34 wide; y from the first
// row, 9 rows) and the vertex plane's load tile (32 x 8)
constexpr int kTmaUX = 34, kTmaUY = 9, kTmaFX = 32, kTmaFY = 8;
// tensor-copy destinations start 128-byte aligned: each tile's slot rounded up
constexpr int kTmaUSlot = (kTmaUX * kTmaUY * 8 + 127) / 128 * 128 / 8;  // doubles
__host__ __device__ constexpr int tma_vbytes() { return (2 * kTmaUSlot + kTmaFX * kTmaFY) * 8; }

struct TmaVMaps {
    CUtensorMap u, uh, fl;
};
__host__ __device__ constexpr int tma_stage_total(int W) { return tma_stage_bytes(W) + tma_vbytes(); }
__host__ __device__ constexpr int tma_smem_bytes2(int W, int S) {
    return 2 * 8 * kTmaCells * 8 + S * tma_stage_total(W) + 16 * S;
}

// S stages: the tiles of iteration j land in stage j % S, issued S - 1
// iterations ahead (S = 2 for the small compressed words, whose stages are
// small; the FP64 planes' 66 KB stage leaves room for one per block)
// NORM: the block also sums r^2 of the vertices it writes (r is zero on the
// boundary) into norm_part[block]: the residual norm of step() without the
// 8 B per vertex re-read of k3_norm_partial (fixed order: per thread over its
// planes, then a tree over the block; the blocks' partials are summed by
// k3_sum_wide).
template <int W, int S, bool SYM, bool NORM>
__global__ void __launch_bounds__(kRzX * kRzY, 2) k3_residual_tma(Lv3 F, const __grid_constant__ TmaMaps M,
                                                                 const __grid_constant__ TmaVMaps VM, Planes3 P,
                                                                 int zbeg, int zend, int zc,
                                                                 double* __restrict__ norm_part) {
    lzb_pdl_enter();
    extern __shared__ __align__(128) unsigned char smraw[];
    double(*sy)[8][kTmaCells] = reinterpret_cast<double(*)[8][kTmaCells]>(smraw);  // [u, û][corner][cell]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smraw + tma_smem_bytes2(W, S) - 16 * S);
    unsigned char* stage = smraw + 2 * 8 * kTmaCells * 8;
    constexpr int e0 = tma_piece(W, 0), e1 = tma_piece(W, 1), e2 = tma_piece(W, 2);
    constexpr int w0 = tma_width(e0), w1 = tma_width(e1), w2 = tma_width(e2), we = tma_width(8);
    // the regions of stage st
    auto pc0 = [&](int st) { return stage + st * tma_stage_total(W); };
    auto pc1 = [&](int st) { return pc0(st) + tma_piece_bytes(e0); };
    auto pc2 = [&](int st) { return pc1(st) + tma_piece_bytes(e1); };
    auto sec = [&](int st) { return reinterpret_cast<double*>(pc2(st) + tma_piece_bytes(e2)); };
    auto su = [&](int st) { return reinterpret_cast<double*>(pc0(st) + tma_stage_bytes(W)); };
    auto suh = [&](int st) { return su(st) + kTmaUSlot; };
    auto sfl = [&](int st) { return suh(st) + kTmaUSlot; };
    const int tx = threadIdx.x % kRzX, ty = threadIdx.x / kRzX, t = threadIdx.x;
    const int N = F.N, NV = N + 1;
    const int X0 = blockIdx.x * (kRzX - 1), Y0 = blockIdx.y * (kRzY - 1);
    const int zs = zbeg + blockIdx.z * zc, ze = min(zs + zc, zend);
    if (zs >= ze) {
        if (NORM && t == 0) norm_part[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = 0.0;
        return;
    }
    double nsum = 0.0;
    const int cx = X0 - 1 + tx, cy = Y0 - 1 + ty;  // this thread's cell column
    const bool colok = cx >= 0 && cy >= 0 && cx < N && cy < N;
    const int ix = X0 + tx, iy = Y0 + ty;  // this thread's vertex column (tx < 31, ty < 7)
    const bool vthr = tx < kRzX - 1 && ty < kRzY - 1 && ix <= N && iy <= N;
    // tile origins (tensor coordinates are never negative; boxes start 16-byte aligned in x)
    const int ux0 = max(X0 - 1, 0) & ~1, uy0 = max(Y0 - 1, 0), fx0 = X0 & ~1;
    auto layer_ok = [&](int cz) { return cz >= 0 && cz < N; };
    auto issue = [&](int cz) {  // one elected thread: iteration cz's tiles into its stage
        const bool cells = layer_ok(cz), load = cz + 1 < ze;
        const int st = (cz - zs + 1) % S;
        uint64_t* bar = bars + 2 * st;
        uint32_t bytes = 0;
        if (cells) bytes += tma_stage_bytes(W) + 2 * kTmaUX * kTmaUY * 8;
        if (load) bytes += kTmaFX * kTmaFY * 8;
        if (!bytes) return;
        mbar_expect(bar, bytes);
        if (cells) {
            // storage x / y of cell (X0 - 1, Y0 - 1) are X0 / Y0 (the leading pad)
            const int tz = cz - M.z0;  // the leaf planes' tensors start at the window's first layer
            tma_load_4d(pc0(st), &M.piece[0], X0 & ~(16 / e0 - 1), Y0, tz, 0, bar);
            if (e1) tma_load_4d(pc1(st), &M.piece[1], X0 & ~(16 / (e1 ? e1 : 1) - 1), Y0, tz, 0, bar);
            if (e2) tma_load_4d(pc2(st), &M.piece[2], X0 & ~(16 / (e2 ? e2 : 1) - 1), Y0, tz, 0, bar);
            if (W) tma_load_3d(sec(st), &M.ec, X0 & ~1, Y0, tz, bar);
            tma_load_3d(su(st), &VM.u, ux0, uy0, cz + 1, bar);  // the layer's upper vertex plane
            tma_load_3d(suh(st), &VM.uh, ux0, uy0, cz + 1, bar);
        }
        if (load) tma_load_3d(sfl(st), &VM.fl, fx0, Y0, cz + 1, bar);
    };
    auto needs = [&](int cz) { return layer_ok(cz) || cz + 1 < ze; };
    if (t == 0)
        for (int st = 0; st < S; ++st) mbar_init(bars + 2 * st, 1);
    __syncthreads();
    uint32_t phases = 0;  // bit st: the parity stage st waits for next
    if (t == 0)
        for (int j = 0; j < S && zs - 1 + j < ze; ++j) issue(zs - 1 + j);
    // this thread's corner slots in the u / u-hat tiles (clamped: a corner left
    // of / below the tile only occurs for threads whose cell does not exist)
    int us[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
        us[k] = max(cy + (k >> 1) - uy0, 0) * kTmaUX + max(cx + (k & 1) - ux0, 0);
    const int fs = ty * kTmaFX + ix - fx0;
    double ul[4], uhl[4];  // corners of the current layer's lower plane
    {
        auto vid = [&](int x, int y, int z) {
            return (static_cast<int64_t>(min(max(z, 0), N)) * NV + min(max(y, 0), N)) * NV + min(max(x, 0), N);
        };
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t v = vid(cx + (k & 1), cy + (k >> 1), zs - 1);
            ul[k] = F.v[LZB_V_U][v];
            uhl[k] = F.v[LZB_V_UHAT][v];
        }
    }
    double rp = 0.0, rhp = 0.0;  // partial sums of the vertex plane being completed
    for (int cz = zs - 1; cz < ze; ++cz) {
        const int st = (cz - zs + 1) % S;
        double flc = 0.0;
        if (needs(cz)) {
            mbar_wait(bars + 2 * st, (phases >> st) & 1u);
            phases ^= 1u << st;
        }
        if (vthr && cz + 1 < ze) flc = sfl(st)[fs];
        if (layer_ok(cz)) {
            double uu[8], uh[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uu[k] = ul[k];
                uh[k] = uhl[k];
                uu[4 + k] = su(st)[us[k]];
                uh[4 + k] = suh(st)[us[k]];
                ul[k] = uu[4 + k];
                uhl[k] = uh[4 + k];
            }
            if (colok) {
                double K[27];
                // the cell's slot in each box: row ty, column tx + the box's alignment offset
                const int i0 = ty * w0 + tx + (X0 & (16 / e0 - 1));
                if constexpr (W == 0) {
#pragma unroll
                    for (int q = 0; q < 27; ++q) K[q] = reinterpret_cast<const double*>(pc0(st))[q * kRzY * w0 + i0];
                } else {
                    const int i1 = ty * w1 + tx + (e1 ? (X0 & (16 / (e1 ? e1 : 1) - 1)) : 0);
                    const int i2 = ty * w2 + tx + (e2 ? (X0 & (16 / (e2 ? e2 : 1) - 1)) : 0);
                    // SYM (the n = 1 classes symmetric, s1[0] == s1[2]: the unit interval): the
                    // baseline takes 8 values, class (cx, cy, cz) -> (cx == 1, cy == 1, cz == 1)
                    double b8[8];
                    {
                        const Base3 B(sec(st)[ty * we + tx + (X0 & 1)], P.s1, P.h);
#pragma unroll
                        for (int k = 0; k < 8; ++k) b8[k] = B(k >> 2, (k >> 1) & 1, k & 1);
                    }
#pragma unroll
                    for (int q = 0; q < 27; ++q) {
                        unsigned long long w;
                        if constexpr (e0 == 8) w = reinterpret_cast<const unsigned long long*>(pc0(st))[q * kRzY * w0 + i0];
                        else if constexpr (e0 == 4) w = reinterpret_cast<const uint32_t*>(pc0(st))[q * kRzY * w0 + i0];
                        else if constexpr (e0 == 2) w = reinterpret_cast<const uint16_t*>(pc0(st))[q * kRzY * w0 + i0];
                        else w = pc0(st)[q * kRzY * w0 + i0];
                        if constexpr (e1 == 2) w |= static_cast<unsigned long long>(reinterpret_cast<const uint16_t*>(pc1(st))[q * kRzY * w1 + i1]) << (8 * e0);
                        else if constexpr (e1 == 1) w |= static_cast<unsigned long long>(pc1(st)[q * kRzY * w1 + i1]) << (8 * e0);
                        if constexpr (e2 == 1) w |= static_cast<unsigned long long>(pc2(st)[q * kRzY * w2 + i2]) << (8 * (e0 + e1));
                        const double rt = SrcComp<W>::dec(static_cast<typename SrcComp<W>::Word>(w));
                        if constexpr (SYM) {
                            K[q] = b8[(q / 9 == 1) * 4 + ((q / 3) % 3 == 1) * 2 + (q % 3 == 1)] + rt;
                        } else {
                            const Base3 B(sec(st)[ty * we + tx + (X0 & 1)], P.s1, P.h);
                            K[q] = B(q / 9, (q / 3) % 3, q % 3) + rt;
                        }
                    }
                }
#pragma unroll
                for (int a = 0; a < 8; ++a) {
                    double au = 0.0, auh = 0.0;
#pragma unroll
                    for (int col = 0; col < 8; ++col) {  // explicit FMA (the 3D cycle is restated, not pinned bitwise)
                        au = __fma_rn(K[cls3(a, col)], uu[col], au);
                        auh = __fma_rn(K[cls3(a, col)], uh[col], auh);
                    }
                    sy[0][a][t] = au;
                    sy[1][a][t] = auh;
                }
            }
        }
        __syncthreads();  // the stage is consumed: iteration cz + S's tiles may land in it
        if (t == 0 && cz + S < ze) issue(cz + S);
        if (vthr) {
            auto sub = [&](int q, double& r, double& rh) {
                const int dx = q & 1, dy = (q >> 1) & 1, dz = q >> 2;
                const int row = (1 - dx) + 2 * (1 - dy) + 4 * (1 - dz);
                const int ccx = ix - 1 + dx, ccy = iy - 1 + dy;
                if (ccx < 0 || ccy < 0 || ccx >= N || ccy >= N) return;
                const int c = (ty + dy) * kRzX + tx + dx;
                r -= sy[0][row][c];
                rh -= sy[1][row][c];
            };
            if (cz >= zs && cz < N) {
#pragma unroll
                for (int q = 4; q < 8; ++q) sub(q, rp, rhp);
            }
            if (cz >= zs) {
                double r = rp, rh = rhp;
                if (bnd3(N, ix, iy, cz)) {
                    r = 0.0;
                    rh = 0.0;
                }
                const int64_t vi = (static_cast<int64_t>(cz) * NV + iy) * NV + ix;
                __stcs(F.v[LZB_V_R] + vi, r);
                __stcs(F.v[LZB_V_RHAT] + vi, rh);
                if (NORM) nsum += r * r;
            }
            if (cz + 1 < ze) {
                rp = rhp = flc;
                if (cz >= 0) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) sub(q, rp, rhp);
                }
            }
        }
        __syncthreads();
    }
    if (NORM) {  // the loop ended on a barrier: the row-product stage is free
        double* red = &sy[0][0][0];
        red[t] = nsum;
        __syncthreads();
        for (int w = (kRzX * kRzY) / 2; w > 0; w >>= 1) {
            if (t < w) red[t] += red[t + w];
            __syncthreads();
        }
        if (t == 0) norm_part[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = red[0];
    }
}

// fl_c = P^T r̂ over owned lattice points (adjacent patches in (z, y, x)
// order, lattice points in (z, y, x) order). mode 1: r into aux (unused).
__global__ void k3_restrict(Lv3 F, Lv3 C) {
    lzb_pdl_enter();
    int IX, IY, IZ;
    int64_t vi;
    if (!vxyz(C, IX, IY, IZ, vi)) return;
    const int Nc = C.N;
    double acc = 0.0;
    for (int q = 0; q < 8; ++q) {
        const int dx = q & 1, dy = (q >> 1) & 1, dz = q >> 2;
        const int px = IX - 1 + dx, py = IY - 1 + dy, pz = IZ - 1 + dz;
        if (px < 0 || py < 0 || pz < 0 || px >= Nc || py >= Nc || pz >= Nc) continue;
        const int k = (1 - dx) + 2 * (1 - dy) + 4 * (1 - dz);  // the vertex's corner in the patch
        for (int lz = 0; lz < 4; ++lz) {
            if (lz == 0 && pz != 0) continue;
            for (int ly = 0; ly < 4; ++ly) {
                if (ly == 0 && py != 0) continue;
                for (int lx = 0; lx < 4; ++lx) {
                    if (lx == 0 && px != 0) continue;
                    const double w = pw3(lx, ly, lz, k);
                    if (w == 0.0) continue;
                    acc += w * F.v[LZB_V_RHAT][vidx3(F.N, 3 * px + lx, 3 * py + ly, 3 * pz + lz)];
                }
            }
        }
    }
    C.v[LZB_V_FL][vi] = acc;
}

// The same restriction as a staged z-march (the cycle's kernel; k3_restrict
// above stays as the plain form, LZB_PLAIN_RESTRICT=1). Ownership and the
// lattice weights are per-axis, so P^T is the tensor product of the 1D
// restriction c[I] = (f[3I-2] + 2 f[3I-1] + 3 f[3I] + 2 f[3I+1] + f[3I+2]) / 3
// (fine vertex 3I is owned by patch I - 1 at its lattice index 3, by patch 0
// at index 0 when I = 0: weight 3 either way). A block owns 32 x 8 coarse
// columns and a chunk of coarse planes; per fine plane it stages the 98 x 26
// tile of r-hat with coalesced loads (each fine value is read once, not ~4.6
// times through strided gathers), restricts in x, then y, in shared memory,
// and every thread accumulates its column's value into the one or two coarse
// planes the fine plane belongs to (ascending fine planes: the same order for
// any chunking, so slab-range launches give the same bits). Integer weights,
// one division by 27 per coarse vertex: the sums differ from k3_restrict's
// (one rounded weight product per term) in the last bits only -- the 3D cycle
// is a restatement with a 1e-10 parity bar.
constexpr int kRsX = 32, kRsY = 8, kRsFX = 3 * kRsX + 2, kRsFY = 3 * kRsY + 2;
__global__ void __launch_bounds__(kRsX * kRsY) k3_restrict_zm(Lv3 F, Lv3 C, int Z0, int Z1, int zc) {
    lzb_pdl_enter();
    __shared__ double tile[kRsFY][kRsFX];
    __shared__ double s1[kRsFY][kRsX];
    const int t = threadIdx.x, tx = t % kRsX, ty = t / kRsX;
    const int IX0 = blockIdx.x * kRsX, IY0 = blockIdx.y * kRsY;
    const int za = Z0 + blockIdx.z * zc, zb = min(za + zc, Z1);
    if (za >= zb) return;
    const int Nf = F.N, NVf = Nf + 1, Nc = C.N, NVc = Nc + 1;
    const int IX = IX0 + tx, IY = IY0 + ty;
    const bool own = IX < NVc && IY < NVc;
    const int fx0 = 3 * IX0 - 2, fy0 = 3 * IY0 - 2;
    const double* __restrict__ rh = F.v[LZB_V_RHAT];
    double* __restrict__ out = C.v[LZB_V_FL];
    double cur = 0.0, nxt = 0.0;  // coarse planes I and I + 1
    int I = za;
    const int fbeg = max(3 * za - 2, 0), fend = min(3 * (zb - 1) + 2, Nf);
    // this thread's tile elements (the same for every fine plane): in-plane offset, or -1 outside the grid
    constexpr int kPer = (kRsFY * kRsFX + kRsX * kRsY - 1) / (kRsX * kRsY);
    int off[kPer];
#pragma unroll
    for (int e = 0; e < kPer; ++e) {
        const int k = t + e * kRsX * kRsY;
        const int r = k / kRsFX, c = k - r * kRsFX;
        const int fy = fy0 + r, fx = fx0 + c;
        off[e] = (k < kRsFY * kRsFX && fx >= 0 && fy >= 0 && fx <= Nf && fy <= Nf) ? fy * NVf + fx : -1;
    }
    double* const tflat = &tile[0][0];
    double pre[kPer];  // the next fine plane's values, in flight while this one is restricted
    auto fetch = [&](int fz) {
        const double* pl = rh + static_cast<int64_t>(fz) * NVf * NVf;
#pragma unroll
        for (int e = 0; e < kPer; ++e) pre[e] = off[e] >= 0 ? __ldg(pl + off[e]) : 0.0;
    };
    fetch(fbeg);
    for (int fz = fbeg; fz <= fend; ++fz) {
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const int k = t + e * kRsX * kRsY;
            if (k < kRsFY * kRsFX) tflat[k] = pre[e];
        }
        __syncthreads();
        if (fz < fend) fetch(fz + 1);
        for (int r = ty; r < kRsFY; r += kRsY) {  // x: fine 3 IX + j sits in column 3 tx + j + 2
            const double* p = &tile[r][3 * tx];
            s1[r][tx] = ((p[0] + 2.0 * p[1]) + 3.0 * p[2]) + (2.0 * p[3] + p[4]);
        }
        __syncthreads();
        const int r0 = 3 * ty;  // y: fine 3 IY + j sits in row 3 ty + j + 2
        const double v = ((s1[r0][tx] + 2.0 * s1[r0 + 1][tx]) + 3.0 * s1[r0 + 2][tx]) +
                         (2.0 * s1[r0 + 3][tx] + s1[r0 + 4][tx]);
        // z: fine plane 3 q + m feeds coarse q (weights 3, 2, 1 for m = 0, 1, 2) and q + 1 (0, 1, 2)
        const int q = fz / 3, m = fz - 3 * q;
        const double wq = static_cast<double>(3 - m), wq1 = static_cast<double>(m);
        if (q == I) cur += wq * v;
        else if (q == I + 1) nxt += wq * v;
        if (m != 0) {
            if (q + 1 == I) cur += wq1 * v;
            else if (q + 1 == I + 1) nxt += wq1 * v;
        }
        if (fz == 3 * I + 2 || fz == Nf) {  // coarse plane I is complete
            if (own && I < zb) out[(static_cast<int64_t>(I) * NVc + IY) * NVc + IX] = cur / 27.0;
            cur = nxt;
            nxt = 0.0;
            ++I;
        }
    }
}

// Per-block partial sums of r^2 over the interior vertices of planes
// [max(zlo, 1), min(zhi, N)): block b takes rows b, b + G, ... four rows per
// step (four independent loads in flight per thread), then a fixed-order tree.
__global__ void k3_norm_partial(Lv3 F, double* partial, int zlo, int zhi) {
    lzb_pdl_enter();
    __shared__ double sh[256];
    const int N = F.N;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    const int za = max(zlo, 1), zb = min(zhi, N);
    const int64_t rows = zb > za ? static_cast<int64_t>(N - 1) * (zb - za) : 0;
    const int64_t G = gridDim.x;
    for (int64_t r0 = blockIdx.x; r0 < rows; r0 += 4 * G) {
        int64_t base[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t rz = r0 + k * G;
            base[k] = rz < rows ? vidx3(N, 0, 1 + static_cast<int>(rz % (N - 1)), za + static_cast<int>(rz / (N - 1)))
                                : -1;
        }
        for (int ix = 1 + threadIdx.x; ix < N; ix += blockDim.x) {
            double r[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) r[k] = base[k] >= 0 ? F.v[LZB_V_R][base[k] + ix] : 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) s[k] += r[k] * r[k];
        }
    }
    sh[threadIdx.x] = (s[0] + s[1]) + (s[2] + s[3]);
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

// the slab's sum of r^2 from the norm partials, the host loop's order (step())
__global__ void k3_sum_partials(const double* partial, int n, double* out) {
    lzb_pdl_enter();
    if (threadIdx.x != 0) return;
    double s2 = 0.0;
    for (int i = 0; i < n; ++i) s2 += partial[i];
    *out = s2;
}

// sum of n partials in a fixed order: strided per thread, then a tree
__global__ void __launch_bounds__(1024) k3_sum_wide(const double* __restrict__ partial, int n, double* out) {
    lzb_pdl_enter();
    __shared__ double sh[1024];
    double a = 0.0;
    for (int i = threadIdx.x; i < n; i += 1024) a += partial[i];
    sh[threadIdx.x] = a;
    __syncthreads();
    for (int w = 512; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

__global__ void k3_snap(Lv3 L, int64_t nv) {
    lzb_pdl_enter();
    const int64_t i = gtid();
    if (i >= nv) return;
    L.v[LZB_V_USNAP][i] = L.v[LZB_V_U][i];
    L.v[LZB_V_AUX][i] = 0.0;
}

__global__ void k3_aux_inject(Lv3 F, Lv3 C) {
    lzb_pdl_enter();
    int ix, iy, iz;
    int64_t vi;
    if (!vxyz(C, ix, iy, iz, vi)) return;
    C.v[LZB_V_AUX][vi] = F.v[LZB_V_R][vidx3(F.N, 3 * ix, 3 * iy, 3 * iz)];
}

__global__ void k3_aux_sub(Lv3 F, Lv3 C, double omega) {
    lzb_pdl_enter();
    int fx, fy, fz;
    int64_t vi;
    if (!vxyz(F, fx, fy, fz, vi)) return;
    if (bnd3(F.N, fx, fy, fz)) return;
    const int px = owner3(fx, C.N), py = owner3(fy, C.N), pz = owner3(fz, C.N);
    const int lx = fx - 3 * px, ly = fy - 3 * py, lz = fz - 3 * pz;
    double p = 0.0;
    for (int a = 0; a < 8; ++a) {
        const int cx = px + (a & 1), cy = py + ((a >> 1) & 1), cz = pz + (a >> 2);
        const int64_t ci = vidx3(C.N, cx, cy, cz);
        const double dg = C.v[LZB_V_DIAG][ci];
        const double caux = (!bnd3(C.N, cx, cy, cz) && dg != 0.0) ? omega / dg * C.v[LZB_V_AUX][ci] : 0.0;
        p += pw3(lx, ly, lz, a) * caux;
    }
    F.v[LZB_V_U][vi] -= p;
}

__global__ void k3_jacobi(Lv3 F, double damping) {
    lzb_pdl_enter();
    int ix, iy, iz;
    int64_t vi;
    if (!vxyz(F, ix, iy, iz, vi)) return;
    if (bnd3(F.N, ix, iy, iz)) return;
    const double dg = F.v[LZB_V_DIAG][vi];
    if (dg != 0.0) F.v[LZB_V_U][vi] += damping / dg * F.v[LZB_V_R][vi];
}

__global__ void k3_prolong(Lv3 F, Lv3 C) {
    lzb_pdl_enter();
    int fx, fy, fz;
    int64_t vi;
    if (!vxyz(F, fx, fy, fz, vi)) return;
    if (bnd3(F.N, fx, fy, fz)) return;
    const int px = owner3(fx, C.N), py = owner3(fy, C.N), pz = owner3(fz, C.N);
    const int lx = fx - 3 * px, ly = fy - 3 * py, lz = fz - 3 * pz;
    double d[8];
    bool any = false;
    for (int a = 0; a < 8; ++a) {
        const int64_t ci = vidx3(C.N, px + (a & 1), py + ((a >> 1) & 1), pz + (a >> 2));
        d[a] = C.v[LZB_V_U][ci] - C.v[LZB_V_USNAP][ci];
        any |= d[a] != 0.0;
    }
    if (!any) return;
    double p = 0.0;
    for (int a = 0; a < 8; ++a) p += pw3(lx, ly, lz, a) * d[a];
    F.v[LZB_V_U][vi] += p;
}

// ---- staged leaf-level vertex kernels
// A block is a row segment of 256 fine vertices along x on kStY consecutive
// rows along y of one vertex plane z (rows of one plane are 8 (N+1) bytes
// apart: the block's loads stay within a page or two per array, where a z
// chunk would touch a page per plane). The owner patch's z coordinate and
// lattice offset are uniform over the block, so the coarse values the block
// needs are the x-range of its owner patches (<= 88 coarse x) on the <= 5
// coarse y lines its rows' owners span and 2 coarse z planes; they are staged
// once in shared memory. The trilinear interpolation is then evaluated
// separably: per fine row the block contracts y and z for every staged coarse
// x, and each fine vertex takes the x contraction of two of those -- 2 FMA per
// vertex instead of 8 weights x 8 corners. The 3D cycle is a restatement
// (oracle/port3.py sums the 8 corners with k / 27 weights): the regrouping
// changes the last bits only (tests: 1e-12 on u).
constexpr int kStThreads = 256;  // fine x per block
constexpr int kStX = 96;  // staged coarse x per line (256 / 3 + 3 rounded up)
constexpr int kStY = 8;   // fine rows per block of the u-hat kernel
constexpr int kStYu = 4;  // of the fused update (three arrays per row in registers: 64 registers, twice the
                          // resident warps of the 8-row form; measured 5.2 -> 4.8 ms at 729^3, while the
                          // u-hat kernel is faster with 8: 1.40 vs 1.83 ms)
constexpr int kStCy = 5;  // coarse y lines the rows' owner patches span (<= kStY / 3 + 3)
struct RowStage {
    int px0, nx, pz, lz, py0, ny, fy0, fy1, fz;
};
template <int ROWS>
__device__ __forceinline__ RowStage row_stage(const Lv3& F, const Lv3& C) {
    RowStage r;
    const int fx0 = blockIdx.x * blockDim.x;
    const int fx1 = min(fx0 + static_cast<int>(blockDim.x) - 1, F.N);
    r.px0 = owner3(fx0, C.N);
    r.nx = owner3(fx1, C.N) + 2 - r.px0;  // owner patches' x corners px .. px + 1
    r.fz = blockIdx.z + F.z0;
    r.pz = owner3(r.fz, C.N);
    r.lz = r.fz - 3 * r.pz;
    r.fy0 = blockIdx.y * ROWS;
    r.fy1 = min(r.fy0 + ROWS, F.N + 1);
    r.py0 = owner3(r.fy0, C.N);
    r.ny = owner3(r.fy1 - 1, C.N) + 2 - r.py0;
    return r;
}
// per-axis lattice weights (a ? L : 3 - L) / 3
// (k / 3.0 for k = 0..3 as selects of the compile-time quotients: the same
// correctly rounded values without a double-precision division per call --
// the divisions were 12 % of the fused update's stall samples)
__device__ __forceinline__ double wax(int L, int a) {
    const int k = a ? L : 3 - L;
    return k == 0 ? 0.0 : k == 1 ? 1.0 / 3.0 : k == 2 ? 2.0 / 3.0 : 1.0;
}

// Per coarse vertex of the level below the leaves, once per cycle: the
// adaFAC-PI aux correction factor omega / diag * aux (0 on the boundary and
// where diag = 0) and the prolongated correction u - usnap.
__global__ void k3_coarse_pre(Lv3 C, double omega, int pi, double2* __restrict__ pre) {
    lzb_pdl_enter();
    int cx, cy, cz;
    int64_t ci;
    if (!vxyz(C, cx, cy, cz, ci)) return;
    double caux = 0.0;
    if (pi) {
        const double dg = C.v[LZB_V_DIAG][ci];
        caux = (!bnd3(C.N, cx, cy, cz) && dg != 0.0) ? omega / dg * C.v[LZB_V_AUX][ci] : 0.0;
    }
    pre[ci] = make_double2(caux, C.v[LZB_V_U][ci] - C.v[LZB_V_USNAP][ci]);
}

// The leaf level's three u updates of a cycle in one pass (the adaFAC-PI aux
// correction, damped Jacobi, the prolongated coarse correction -- k3_aux_sub,
// k3_jacobi, k3_prolong in that order; the coarse levels are updated first,
// nothing there reads the leaf u).
__global__ void __launch_bounds__(kStThreads) k3_update_fine_st(Lv3 F, Lv3 C, const double2* __restrict__ pre, int pi,
                                                          double damping) {
    lzb_pdl_enter();
    __shared__ double2 s_pre[kStCy][2][kStX];
    __shared__ double2 s_g[kStYu][kStX];  // per row, per coarse x: (aux, correction) contracted over y, z
    __shared__ unsigned char s_nz[kStYu][kStX];
    const int fx = blockIdx.x * blockDim.x + threadIdx.x;
    const RowStage R = row_stage<kStYu>(F, C);
    const bool act = fx < F.N && fx > 0 && R.fz > 0 && R.fz < F.N;
    // the fine vertices' loads first: they stream from HBM while the block stages
    double u[kStYu], dg[kStYu], r[kStYu];
    const int64_t vi0 = vidx3(F.N, min(fx, F.N), R.fy0, R.fz);
#pragma unroll
    for (int k = 0; k < kStYu; ++k) {
        const int fy = R.fy0 + k;
        if (act && fy < R.fy1 && fy > 0 && fy < F.N) {
            const int64_t vi = vi0 + static_cast<int64_t>(k) * (F.N + 1);
            u[k] = __ldcs(F.v[LZB_V_U] + vi);
            dg[k] = __ldcs(F.v[LZB_V_DIAG] + vi);
            r[k] = __ldcs(F.v[LZB_V_R] + vi);
        }
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    for (int q = warp; q < 2 * R.ny; q += nwarp) {  // a warp per staged coarse line
        const int az = q & 1, iy = q >> 1;
        const int64_t base = vidx3(C.N, 0, min(R.py0 + iy, C.N), R.pz + az);
        for (int j = lane; j < R.nx; j += 32) s_pre[iy][az][j] = pre[base + min(R.px0 + j, C.N)];
    }
    __syncthreads();
    const double wz0 = wax(R.lz, 0), wz1 = wax(R.lz, 1);
    for (int k = warp; k < kStYu; k += nwarp)  // a warp per fine row, lanes over the coarse x
        for (int j = lane; j < R.nx; j += 32) {
            const int fy = min(R.fy0 + k, F.N);
            const int py = owner3(fy, C.N), ly = fy - 3 * py, jy = py - R.py0;
            const double wy0 = wax(ly, 0), wy1 = wax(ly, 1);
            const double2 c00 = s_pre[jy][0][j], c10 = s_pre[jy + 1][0][j], c01 = s_pre[jy][1][j],
                          c11 = s_pre[jy + 1][1][j];
            s_g[k][j] = make_double2(wz0 * (wy0 * c00.x + wy1 * c10.x) + wz1 * (wy0 * c01.x + wy1 * c11.x),
                                     wz0 * (wy0 * c00.y + wy1 * c10.y) + wz1 * (wy0 * c01.y + wy1 * c11.y));
            s_nz[k][j] = (c00.y != 0.0) | (c10.y != 0.0) | (c01.y != 0.0) | (c11.y != 0.0);
        }
    __syncthreads();
    if (!act) return;
    const int px = owner3(fx, C.N), lx = fx - 3 * px, jx = px - R.px0;
    const double wx0 = wax(lx, 0), wx1 = wax(lx, 1);
#pragma unroll
    for (int k = 0; k < kStYu; ++k) {
        const int fy = R.fy0 + k;
        if (!(fy < R.fy1 && fy > 0 && fy < F.N)) continue;
        const double2 g0 = s_g[k][jx], g1 = s_g[k][jx + 1];
        double uu = u[k];
        if (pi) uu -= wx0 * g0.x + wx1 * g1.x;
        if (dg[k] != 0.0) uu += damping / dg[k] * r[k];
        if (s_nz[k][jx] | s_nz[k][jx + 1]) uu += wx0 * g0.y + wx1 * g1.y;
        __stcs(F.v[LZB_V_U] + vi0 + static_cast<int64_t>(k) * (F.N + 1), uu);
    }
}

// The same update as a march along y: a block keeps its 256 fine x and walks
// kMarchPatches owner-patch rows (3 fine rows each) of one vertex plane. The
// coarse lines live in a ring of three slots (a patch row needs lines p and
// p + 1; line p + 2 is fetched into a register during row p), the next patch
// row's u / diag / r are loaded before the current one is computed, so the
// loads of a block are in flight throughout instead of once per block, and
// the staging is paid once per 81 rows instead of once per 4. Per vertex the
// arithmetic is that of k3_update_fine_st, operation for operation (the two
// kernels give identical bits; LZB_UPDATE3_ROWS=1 selects the row kernel).
constexpr int kMarchPatches = 27;  // owner-patch rows per block (LZB_UPDATE3_PG overrides, for sweeps)
__global__ void __launch_bounds__(kStThreads, 3) k3_update_fine_march(Lv3 F, Lv3 C, const double2* __restrict__ pre,
                                                                    int pi, double damping, int pg) {
    lzb_pdl_enter();
    __shared__ double2 s_ring[3][2][kStX];
    __shared__ double2 s_g[3][kStX];
    __shared__ unsigned char s_nz[3][kStX];
    const int fz = blockIdx.z + F.z0;
    if (fz <= 0 || fz >= F.N) return;  // boundary planes (uniform over the block)
    const int tid = threadIdx.x;
    const int fx0 = blockIdx.x * blockDim.x, fx = fx0 + tid;
    const int fx1 = min(fx0 + static_cast<int>(blockDim.x) - 1, F.N);
    const int px0 = owner3(fx0, C.N), nx = owner3(fx1, C.N) + 2 - px0;
    const int pz = owner3(fz, C.N), lz = fz - 3 * pz;
    const int p0 = blockIdx.y * pg, p1 = min(p0 + pg, C.N);
    const bool act = fx < F.N && fx > 0;
    const int NV = F.N + 1, NC1 = C.N + 1;
    // staging role: thread (saz, sj) owns element sj of the coarse line at z plane pz + saz
    const int saz = tid / kStX, sj = tid - saz * kStX;
    const bool stg = saz < 2 && sj < nx;
    const double2* cline = pre + vidx3(C.N, min(px0 + sj, C.N), 0, pz + (saz & 1));
    int s0 = 0, s1 = 1, s2 = 2;  // ring slots of lines p, p + 1, p + 2
    if (stg) {
        s_ring[0][saz][sj] = cline[static_cast<int64_t>(p0) * NC1];
        s_ring[1][saz][sj] = cline[static_cast<int64_t>(p0 + 1) * NC1];
    }
    double u[3], dg[3], r[3];
    const double* __restrict__ gu = F.v[LZB_V_U] + vidx3(F.N, min(fx, F.N), 3 * p0 + 1, fz);
    const double* __restrict__ gd = F.v[LZB_V_DIAG] + vidx3(F.N, min(fx, F.N), 3 * p0 + 1, fz);
    const double* __restrict__ gr = F.v[LZB_V_R] + vidx3(F.N, min(fx, F.N), 3 * p0 + 1, fz);
    double* __restrict__ gw = F.v[LZB_V_U] + vidx3(F.N, min(fx, F.N), 3 * p0 + 1, fz);
#pragma unroll
    for (int k = 0; k < 3; ++k)
        if (act && 3 * p0 + 1 + k < F.N) {
            u[k] = __ldcs(gu + k * NV);
            dg[k] = __ldcs(gd + k * NV);
            r[k] = __ldcs(gr + k * NV);
        }
    const int px = owner3(min(fx, F.N), C.N), lx = min(fx, F.N) - 3 * px, jx = px - px0;
    const double wx0 = wax(lx, 0), wx1 = wax(lx, 1);
    const double wz0 = wax(lz, 0), wz1 = wax(lz, 1);
    __syncthreads();
    for (int p = p0; p < p1; ++p) {
        const bool more = p + 1 < p1;
        double un[3], dgn[3], rn[3];
        double2 ln = make_double2(0.0, 0.0);
        if (more) {  // the next patch row's loads, in flight while this one is computed
            gu += 3 * NV;
            gd += 3 * NV;
            gr += 3 * NV;
#pragma unroll
            for (int k = 0; k < 3; ++k)
                if (act && 3 * p + 4 + k < F.N) {
                    un[k] = __ldcs(gu + k * NV);
                    dgn[k] = __ldcs(gd + k * NV);
                    rn[k] = __ldcs(gr + k * NV);
                }
            if (stg) ln = cline[static_cast<int64_t>(p + 2) * NC1];
        }
        for (int it = tid; it < 3 * kStX; it += kStThreads) {  // y, z contraction per fine row and coarse x
            const int k = it / kStX, j = it - k * kStX;
            if (j >= nx) continue;
            const double wy0 = wax(k + 1, 0), wy1 = wax(k + 1, 1);
            const double2 c00 = s_ring[s0][0][j], c10 = s_ring[s1][0][j], c01 = s_ring[s0][1][j], c11 = s_ring[s1][1][j];
            s_g[k][j] = make_double2(wz0 * (wy0 * c00.x + wy1 * c10.x) + wz1 * (wy0 * c01.x + wy1 * c11.x),
                                     wz0 * (wy0 * c00.y + wy1 * c10.y) + wz1 * (wy0 * c01.y + wy1 * c11.y));
            s_nz[k][j] = (c00.y != 0.0) | (c10.y != 0.0) | (c01.y != 0.0) | (c11.y != 0.0);
        }
        __syncthreads();
        if (act) {
            // the three rows' damping / diag first, branch-free: three independent division chains the
            // scheduler can interleave (the division was 37 % of the stall samples as one chain per row)
            double jq[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) jq[k] = damping / (dg[k] != 0.0 ? dg[k] : 1.0);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                if (!(3 * p + 1 + k < F.N)) continue;
                const double2 g0 = s_g[k][jx], g1 = s_g[k][jx + 1];
                double uu = u[k];
                if (pi) uu -= wx0 * g0.x + wx1 * g1.x;
                if (dg[k] != 0.0) uu += jq[k] * r[k];
                if (s_nz[k][jx] | s_nz[k][jx + 1]) uu += wx0 * g0.y + wx1 * g1.y;
                __stcs(gw + k * NV, uu);
            }
        }
        if (more && stg) s_ring[s2][saz][sj] = ln;
        __syncthreads();
        gw += 3 * NV;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            u[k] = un[k];
            dg[k] = dgn[k];
            r[k] = rn[k];
        }
        const int t = s0;
        s0 = s1;
        s1 = s2;
        s2 = t;
    }
}

// u-hat = u - P u_c on the leaf level (compute_uhat, solver.cpp:120-143 in 3D)
__global__ void __launch_bounds__(kStThreads) k3_uhat_st(Lv3 F, Lv3 C) {
    lzb_pdl_enter();
    __shared__ double s_u[kStCy][2][kStX];
    __shared__ double s_g[kStY][kStX];
    const int fx = blockIdx.x * blockDim.x + threadIdx.x;
    const RowStage R = row_stage<kStY>(F, C);
    double u[kStY];  // the fine loads first (see k3_update_fine_st)
    const int64_t vi0 = vidx3(F.N, min(fx, F.N), R.fy0, R.fz);
#pragma unroll
    for (int k = 0; k < kStY; ++k)
        if (fx <= F.N && R.fy0 + k < R.fy1) u[k] = __ldcs(F.v[LZB_V_U] + vi0 + static_cast<int64_t>(k) * (F.N + 1));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    for (int q = warp; q < 2 * R.ny; q += nwarp) {  // a warp per staged coarse line
        const int az = q & 1, iy = q >> 1;
        const int64_t base = vidx3(C.N, 0, min(R.py0 + iy, C.N), R.pz + az);
        for (int j = lane; j < R.nx; j += 32) s_u[iy][az][j] = C.v[LZB_V_U][base + min(R.px0 + j, C.N)];
    }
    __syncthreads();
    const double wz0 = wax(R.lz, 0), wz1 = wax(R.lz, 1);
    for (int k = warp; k < kStY; k += nwarp)  // a warp per fine row, lanes over the coarse x
        for (int j = lane; j < R.nx; j += 32) {
            const int fy = min(R.fy0 + k, F.N);
            const int py = owner3(fy, C.N), ly = fy - 3 * py, jy = py - R.py0;
            s_g[k][j] = wz0 * (wax(ly, 0) * s_u[jy][0][j] + wax(ly, 1) * s_u[jy + 1][0][j]) +
                        wz1 * (wax(ly, 0) * s_u[jy][1][j] + wax(ly, 1) * s_u[jy + 1][1][j]);
        }
    __syncthreads();
    if (fx > F.N) return;
    const int px = owner3(fx, C.N), lx = fx - 3 * px, jx = px - R.px0;
    const double wx0 = wax(lx, 0), wx1 = wax(lx, 1);
#pragma unroll
    for (int k = 0; k < kStY; ++k) {
        if (R.fy0 + k >= R.fy1) continue;
        __stcs(F.v[LZB_V_UHAT] + vi0 + static_cast<int64_t>(k) * (F.N + 1),
               u[k] - (wx0 * s_g[k][jx] + wx1 * s_g[k][jx + 1]));
    }
}

// u-hat as a march along y (the structure of k3_update_fine_march: ring of
// coarse u lines, next patch row's u in flight while the current one is
// contracted and stored). All vertices take part, boundary planes and rows
// included; row 0 (lattice offset 0 of patch row 0) is the first chunk's
// prologue. Same expression per vertex as k3_uhat_st, same bits.
// Measured and NOT the default (LZB_UHAT3_MARCH=1 selects it): with one array
// to read, three rows per step leave a thread 3 loads in flight against the
// row kernel's 8 -- 729^3 1.67 ms against 1.34 ms, 243^3 0.066 against 0.052.
__global__ void __launch_bounds__(kStThreads, 4) k3_uhat_march(Lv3 F, Lv3 C, int pg) {
    lzb_pdl_enter();
    __shared__ double s_ring[3][2][kStX];
    __shared__ double s_g[3][kStX];
    const int fz = blockIdx.z + F.z0;
    const int tid = threadIdx.x;
    const int fx0 = blockIdx.x * blockDim.x, fx = fx0 + tid;
    const int fx1 = min(fx0 + static_cast<int>(blockDim.x) - 1, F.N);
    const int px0 = owner3(fx0, C.N), nx = owner3(fx1, C.N) + 2 - px0;
    const int pz = owner3(fz, C.N), lz = fz - 3 * pz;
    const int p0 = blockIdx.y * pg, p1 = min(p0 + pg, C.N);
    const bool act = fx <= F.N;
    const int NV = F.N + 1, NC1 = C.N + 1;
    const int saz = tid / kStX, sj = tid - saz * kStX;
    const bool stg = saz < 2 && sj < nx;
    const double* cline = C.v[LZB_V_U] + vidx3(C.N, min(px0 + sj, C.N), 0, pz + (saz & 1));
    int s0 = 0, s1 = 1, s2 = 2;
    if (stg) {
        s_ring[0][saz][sj] = cline[static_cast<int64_t>(p0) * NC1];
        s_ring[1][saz][sj] = cline[static_cast<int64_t>(p0 + 1) * NC1];
    }
    const int64_t v0 = vidx3(F.N, min(fx, F.N), 3 * p0 + 1, fz);
    const double* __restrict__ gu = F.v[LZB_V_U] + v0;
    double* __restrict__ gw = F.v[LZB_V_UHAT] + v0;
    double u[3], u0 = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k)
        if (act) u[k] = __ldcs(gu + k * NV);
    if (p0 == 0 && act) u0 = __ldcs(gu - NV);
    const int px = owner3(min(fx, F.N), C.N), lx = min(fx, F.N) - 3 * px, jx = px - px0;
    const double wx0 = wax(lx, 0), wx1 = wax(lx, 1);
    const double wz0 = wax(lz, 0), wz1 = wax(lz, 1);
    __syncthreads();
    if (p0 == 0) {  // row 0
        for (int j = tid; j < nx; j += kStThreads)
            s_g[0][j] = wz0 * (wax(0, 0) * s_ring[0][0][j] + wax(0, 1) * s_ring[1][0][j]) +
                        wz1 * (wax(0, 0) * s_ring[0][1][j] + wax(0, 1) * s_ring[1][1][j]);
        __syncthreads();
        if (act) __stcs(gw - NV, u0 - (wx0 * s_g[0][jx] + wx1 * s_g[0][jx + 1]));
        __syncthreads();
    }
    for (int p = p0; p < p1; ++p) {
        const bool more = p + 1 < p1;
        double un[3], ln = 0.0;
        if (more) {
            gu += 3 * NV;
#pragma unroll
            for (int k = 0; k < 3; ++k)
                if (act) un[k] = __ldcs(gu + k * NV);
            if (stg) ln = cline[static_cast<int64_t>(p + 2) * NC1];
        }
        for (int it = tid; it < 3 * kStX; it += kStThreads) {
            const int k = it / kStX, j = it - k * kStX;
            if (j >= nx) continue;
            s_g[k][j] = wz0 * (wax(k + 1, 0) * s_ring[s0][0][j] + wax(k + 1, 1) * s_ring[s1][0][j]) +
                        wz1 * (wax(k + 1, 0) * s_ring[s0][1][j] + wax(k + 1, 1) * s_ring[s1][1][j]);
        }
        __syncthreads();
        if (act) {
#pragma unroll
            for (int k = 0; k < 3; ++k) __stcs(gw + k * NV, u[k] - (wx0 * s_g[k][jx] + wx1 * s_g[k][jx + 1]));
        }
        if (more && stg) s_ring[s2][saz][sj] = ln;
        __syncthreads();
        gw += 3 * NV;
#pragma unroll
        for (int k = 0; k < 3; ++k) u[k] = un[k];
        const int t = s0;
        s0 = s1;
        s1 = s2;
        s2 = t;
    }
}

__global__ void k3_inject(Lv3 F, Lv3 C) {
    lzb_pdl_enter();
    int ix, iy, iz;
    int64_t vi;
    if (!vxyz(C, ix, iy, iz, vi)) return;
    C.v[LZB_V_U][vi] = F.v[LZB_V_U][vidx3(F.N, 3 * ix, 3 * iy, 3 * iz)];
}

// Galerkin coarse element (transfer.cpp:81-93 restated): in class form
//   A_c[q] = sum_children sum_k K_child[k] W[child][k][q],
//   W[child][k][q] = sum_{(i,j) in class k} Q_child[i][a_q] Q_child[j][b_q],
// Q_child[i][a] = w(child lattice of corner i, a), (a_q, b_q) the
// representative entry of class q. Q is a tensor product of per-axis
// factors and a class is a per-axis product of pair classes, so W factors:
// W[child][k][q] = prod_d wa[l_d][k_d][q_d], wa[l][kd][qd] = sum over the
// axis pairs (i, j) of class kd of qax(l + i, a(qd)) qax(l + j, b(qd)),
// qax(L, a) = (a ? L : 3 - L) / 3. The product is contracted axis by axis
// (x, then y, then z): 243 FMA per child instead of 729, no weight table in
// shared memory.
__constant__ double c_wa[27];  // wa[l][kd][qd] at l * 9 + kd * 3 + qd

std::vector<double> galerkin_axis_weights() {
    std::vector<double> w(27, 0.0);
    auto qax = [](int L, int a) { return static_cast<double>(a ? L : 3 - L) / 3.0; };
    for (int l = 0; l < 3; ++l)
        for (int kd = 0; kd < 3; ++kd)
            for (int qd = 0; qd < 3; ++qd) {
                const int a = qd == 2, b = qd >= 1;  // class representative (a, b) per axis
                double acc = 0.0;
                for (int i = 0; i < 2; ++i)
                    for (int j = 0; j < 2; ++j) {
                        const int cls = i == j ? 2 * i : 1;
                        if (cls == kd) acc += qax(l + i, a) * qax(l + j, b);
                    }
                w[l * 9 + kd * 3 + qd] = acc;
            }
    return w;
}
void upload_galerkin_weights() {
    static bool done = false;  // per process (one device per process)
    if (done) return;
    const std::vector<double> w = galerkin_axis_weights();
    LZB_CUDA(cudaMemcpyToSymbol(c_wa, w.data(), 27 * sizeof(double)));
    done = true;
}

// out[9 qx + 3 qy + qz] += sum_k K[9 kx + 3 ky + kz] wx[kx][qx] wy[ky][qy] wz[kz][qz]
__device__ __forceinline__ void galerkin_child(const double* K, int lx, int ly, int lz, double* out) {
    const double* wx = c_wa + lx * 9;
    const double* wy = c_wa + ly * 9;
    const double* wz = c_wa + lz * 9;
#pragma unroll
    for (int kz = 0; kz < 3; ++kz) {
        double t1[3][3], t2[3][3];
#pragma unroll
        for (int qx = 0; qx < 3; ++qx)
#pragma unroll
            for (int ky = 0; ky < 3; ++ky) {
                double acc = 0.0;
#pragma unroll
                for (int kx = 0; kx < 3; ++kx) acc = __fma_rn(K[9 * kx + 3 * ky + kz], wx[kx * 3 + qx], acc);
                t1[qx][ky] = acc;
            }
#pragma unroll
        for (int qx = 0; qx < 3; ++qx)
#pragma unroll
            for (int qy = 0; qy < 3; ++qy) {
                double acc = 0.0;
#pragma unroll
                for (int ky = 0; ky < 3; ++ky) acc = __fma_rn(t1[qx][ky], wy[ky * 3 + qy], acc);
                t2[qx][qy] = acc;
            }
#pragma unroll
        for (int qx = 0; qx < 3; ++qx)
#pragma unroll
            for (int qy = 0; qy < 3; ++qy)
#pragma unroll
                for (int qz = 0; qz < 3; ++qz)
                    out[9 * qx + 3 * qy + qz] = __fma_rn(t2[qx][qy], wz[kz * 3 + qz], out[9 * qx + 3 * qy + qz]);
    }
}

template <class Src>
__global__ void __launch_bounds__(256) k3_galerkin(double* __restrict__ cop, Src S, int Nc, int64_t cbeg,
                                                   int64_t cend) {
    lzb_pdl_enter();
    const int64_t c = cbeg + gtid();  // coarse cells [cbeg, cend)
    const int64_t ncc = static_cast<int64_t>(Nc) * Nc * Nc;
    if (c >= cend) return;
    const int px = static_cast<int>(c % Nc), py = static_cast<int>((c / Nc) % Nc), pz = static_cast<int>(c / Nc / Nc);
    const int Nf = 3 * Nc;
    double out[27];
#pragma unroll
    for (int q = 0; q < 27; ++q) out[q] = 0.0;
    for (int ch = 0; ch < 27; ++ch) {  // child (lz, ly, lx) = (ch / 9, (ch / 3) % 3, ch % 3)
        const int lz = ch / 9, ly = (ch / 3) % 3, lx = ch % 3;
        double K27[27];
        S.load27((static_cast<int64_t>(3 * pz + lz) * Nf + 3 * py + ly) * Nf + 3 * px + lx, K27);
        galerkin_child(K27, lx, ly, lz, out);
    }
#pragma unroll
    for (int q = 0; q < 27; ++q) cop[q * ncc + c] = out[q];
}

// ------------------------------------------------------------ host side
uint64_t splitmix64_host(uint64_t& z) {
    z += 0x9e3779b97f4a7c15ull;
    uint64_t r = z;
    r = (r ^ (r >> 30)) * 0xbf58476d1ce4e5b9ull;
    r = (r ^ (r >> 27)) * 0x94d049bb133111ebull;
    return r ^ (r >> 31);
}

// In-place radix-2 complex FFT of length n (power of 2), stride st, sign
// +1 (inverse, unnormalised) or -1.
void fft1(std::complex<double>* a, int n, int st, int sign) {
    for (int i = 1, j = 0; i < n; ++i) {
        int bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(a[i * st], a[j * st]);
    }
    for (int len = 2; len <= n; len <<= 1) {
        const double ang = sign * 2.0 * 3.14159265358979323846 / len;
        const std::complex<double> wl(std::cos(ang), std::sin(ang));
        for (int i = 0; i < n; i += len) {
            std::complex<double> w(1.0, 0.0);
            for (int k = 0; k < len / 2; ++k) {
                const std::complex<double> u = a[(i + k) * st], v = a[(i + k + len / 2) * st] * w;
                a[(i + k) * st] = u + v;
                a[(i + k + len / 2) * st] = u - v;
                w *= wl;
            }
        }
    }
}

// g(x) = sum_k sqrt(S_k / Z) (xi_k cos(2 pi k.x) + eta_k sin(2 pi k.x)) on
// x = (i, j, l) / n, k in [-n/2, n/2)^3, S_k = exp(-(2 pi |k| ell)^2 / 2)
// (the spectrum of sigma2 exp(-r^2 / 2 ell^2)), Z = sum_k S_k / sigma2 so that
// Var g = sigma2; xi, eta ~ N(0,1) from splitmix64 + Box-Muller in k order.
void grf_table(uint64_t seed, int n, double ell, double sigma2, double* out) {
    if (n < 2 || (n & (n - 1))) throw Error(LZB_ERR_INVALID, "GRF table size must be a power of 2");
    const size_t n3 = static_cast<size_t>(n) * n * n;
    std::vector<std::complex<double>> c(n3);
    const double tpi = 2.0 * 3.14159265358979323846;
    double Z = 0.0;
    std::vector<double> S(n3);
    auto freq = [n](int i) { return i < n / 2 ? i : i - n; };
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            for (int l = 0; l < n; ++l) {
                const double k2 = static_cast<double>(freq(i)) * freq(i) + static_cast<double>(freq(j)) * freq(j) +
                                  static_cast<double>(freq(l)) * freq(l);
                const double s = std::exp(-0.5 * tpi * tpi * ell * ell * k2);
                S[(static_cast<size_t>(i) * n + j) * n + l] = s;
                Z += s;
            }
    Z /= sigma2;
    uint64_t st = seed;
    auto uniform = [&st]() { return (static_cast<double>(splitmix64_host(st) >> 11) + 0.5) * 0x1.0p-53; };
    for (size_t q = 0; q < n3; ++q) {
        // Box-Muller: one pair (xi, eta) per mode
        const double u1 = uniform(), u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double xi = r * std::cos(tpi * u2), eta = r * std::sin(tpi * u2);
        const double a = std::sqrt(S[q] / Z);
        c[q] = std::complex<double>(a * xi, -a * eta);  // Re(c e^{i th}) = a (xi cos th + eta sin th)
    }
    for (int j = 0; j < n; ++j)
        for (int l = 0; l < n; ++l) fft1(c.data() + static_cast<size_t>(j) * n + l, n, n * n, +1);
    for (int i = 0; i < n; ++i)
        for (int l = 0; l < n; ++l) fft1(c.data() + static_cast<size_t>(i) * n * n + l, n, n, +1);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) fft1(c.data() + (static_cast<size_t>(i) * n + j) * n, n, 1, +1);
    for (size_t q = 0; q < n3; ++q) out[q] = c[q].real();
}

Field3 to_device(const lzb_field3& f, DevBuf<double>& table) {
    Field3 F{};
    F.kind = f.kind;
    F.n = f.grf_n;
    F.value = f.value;
    F.xy = f.xy;
    F.cx = f.centre[0];
    F.cy = f.centre[1];
    F.cz = f.centre[2];
    F.radius = f.radius;
    F.width = f.width;
    F.eps_in = f.eps_in;
    F.eps_out = f.eps_out;
    if (f.kind == LZB_F3_SPHERE && !(f.width > 0.0)) throw Error(LZB_ERR_INVALID, "sphere interface width must be > 0");
    if (f.kind == LZB_F3_GRF) {
        if (!f.grf || f.grf_n < 2) throw Error(LZB_ERR_INVALID, "GRF field needs a table");
        const size_t n = f.grf_n, n3 = n * n * n, np = n + 1, np3 = np * np * np;
        std::vector<double> host(n3 + np3);
        std::copy(f.grf, f.grf + n3, host.begin());
        for (size_t k = 0; k < np; ++k)
            for (size_t j = 0; j < np; ++j)
                for (size_t i = 0; i < np; ++i)
                    host[n3 + (k * np + j) * np + i] = f.grf[((i % n) * n + j % n) * n + k % n];
        table.alloc(host.size());
        LZB_CUDA(cudaMemcpy(table.p, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice));
        F.grf = table.p;
        F.grf_t = table.p + n3;
    } else if (f.kind != LZB_F3_CONSTANT && f.kind != LZB_F3_EXTRUDED && f.kind != LZB_F3_SPHERE) {
        throw Error(LZB_ERR_INVALID, "unknown 3D field kind");
    }
    return F;
}

}  // namespace

class Grid3 {
public:
    // [cz0, cz1): the leaf cell layers whose operators this grid stores (-1:
    // all). A rank of the z-slab decomposition stores the layers its residual,
    // diagonal and level-(D-1) Galerkin kernels read -- [max(v0 - 1, 0),
    // min(v1, N)) for vertex planes [v0, v1) -- so the leaf operators, 3/4 of
    // the memory of a 729^3 grid, scale as 1/ranks. Such a grid
    // runs the distributed cycle and the plane-range assembly calls only.
    Grid3(lzb_ctx* ctx, int depth, const lzb_field3& f, double delta_max, int fixed_p3, int plane_width = 0,
          int cz0 = -1, int cz1 = -1)
        : ctx_(ctx), D_(depth), fixed_(fixed_p3), W_(plane_width), delta_(delta_max) {
        if (depth < 0 || depth > 6) throw Error(LZB_ERR_INVALID, "3D depth must be in 0..6");
        if (fixed_p3 != 0 && (fixed_p3 < 2 || fixed_p3 > 8)) throw Error(LZB_ERR_INVALID, "fixed_p3 must be 0 or 2..8");
        if (plane_width != 0 && (plane_width < 2 || plane_width > 8))
            throw Error(LZB_ERR_INVALID, "plane_width must be 0 or 2..8");
        if (plane_width != 0 && fixed_p3 > plane_width)
            throw Error(LZB_ERR_INVALID, "fixed_p3 wider than plane_width");
        LZB_CUDA(cudaSetDevice(ctx->device));
        s_ = ctx->solve;
        N_ = 1;
        for (int i = 0; i < depth; ++i) N_ *= 3;
        nc_ = static_cast<int64_t>(N_) * N_ * N_;
        xp_ = (N_ + 1 + 15) / 16 * 16;
        wz0_ = cz0 < 0 ? 0 : cz0;
        wz1_ = cz1 < 0 ? N_ : cz1;
        if (wz0_ < 0 || wz1_ > N_ || wz0_ >= wz1_) throw Error(LZB_ERR_INVALID, "bad leaf layer window");
        ncs_ = static_cast<int64_t>(wz1_ - wz0_) * (N_ + 1) * xp_;
        woff_ = static_cast<int64_t>(wz0_) * (N_ + 1) * xp_;
        h_ = std::pow(1.0 / 3, depth);
        F_ = to_device(f, table_);
        if (W_ == 0) {
            op_.alloc(static_cast<size_t>(ncs_) * kCls3);
        } else {  // compressed class planes + eps(centre); no FP64 leaf operators
            planes_.alloc(static_cast<size_t>(ncs_) * kCls3 * W_);
            ec_.alloc(ncs_);
        }
        wide_.alloc(1);
        LZB_CUDA(cudaMemsetAsync(wide_.p, 0, sizeof(int), s_));
        p3_.alloc(nc_);
        n_.alloc(nc_);
        stats_.alloc(20);
        LZB_CUDA(cudaMemsetAsync(p3_.p, 0, p3_.bytes(), s_));
        LZB_CUDA(cudaMemsetAsync(n_.p, 0, n_.bytes(), s_));
        LZB_CUDA(cudaMemsetAsync(stats_.p, 0, stats_.bytes(), s_));
        LZB_CUDA(cudaStreamSynchronize(s_));
    }

    bool windowed() const { return wz0_ != 0 || wz1_ != N_; }
    void need_whole(const char* what) const {
        if (windowed())
            throw Error(LZB_ERR_INVALID, std::string(what) + ": this grid stores a z-slab window of the leaf operators; "
                                                             "it runs the distributed cycle and plane-range calls");
    }
    void need_layers(int z0, int z1, const char* what) const {
        if (z0 < wz0_ || z1 > wz1_)
            throw Error(LZB_ERR_INVALID, std::string(what) + ": leaf cell layers outside the stored window");
    }
    // resident bytes of the leaf operator storage (the class planes or plane words + eps centre)
    int64_t leaf_storage_bytes() const {
        return W_ == 0 ? static_cast<int64_t>(op_.bytes()) : static_cast<int64_t>(planes_.bytes() + ec_.bytes());
    }
    void leaf_window(int* z0, int* z1) const {
        *z0 = wz0_;
        *z1 = wz1_;
    }

    void assemble_fixed(int n) { assemble_planes(n, wz0_, wz1_); }  // every stored layer

    // Fixed-p assembly of the leaf cells in z planes [cz0, cz1) (a z-slab of
    // the distributed assembly; cells are independent, no exchange).
    void assemble_planes(int n, int cz0, int cz1) {
        if (n < 1 || n > kMaxN3) throw Error(LZB_ERR_INVALID, "3D sub-samples per axis must be in 1..16");
        if (cz0 < 0 || cz1 > N_ || cz0 > cz1) throw Error(LZB_ERR_INVALID, "bad z plane range");
        if (cz1 > cz0) need_layers(cz0, cz1, "assemble_planes");
        ops_dirty_ = true;
        leaf_diag_dirty_ = true;
        const AxisTab3 T = axis_tab3(n);
        const int64_t cb = static_cast<int64_t>(cz0) * N_ * N_, ce = static_cast<int64_t>(cz1) * N_ * N_;
        if (ce > cb)
        {
            const bool small = F_.kind == LZB_F3_GRF && h_ * F_.n < 1.0;  // cells under one table spacing
            auto go = [&](auto kern) {
                LZB_LAUNCH(kern, blocks_for(ce - cb, 128), 128, 0, s_, F_, N_, h_, T, delta_, fixed_, op_.p, planes(),
                           W_, p3_.p, n_.p, stats_.p, ctx_->err.p, wide_.p, cb, ce);
            };
            auto pick = [&](auto comp) {
                constexpr bool C = decltype(comp)::value;
                if (small && n == 1) go(k_assemble3<LZB_F3_GRF, 1, C>);
                else if (small && n == 2) go(k_assemble3<LZB_F3_GRF, 2, C>);
                else if (F_.kind == LZB_F3_GRF) go(k_assemble3<LZB_F3_GRF, 0, C>);
                else go(k_assemble3<-1, 0, C>);
            };
            if (W_ == 0) pick(std::false_type{});
            else pick(std::true_type{});
        }
        n_last_ = n;
    }

    // Galerkin coarse operators of `level` (from level + 1) for the coarse
    // cells in z planes [pz0, pz1).
    void galerkin_planes(int level, int pz0, int pz1) {
        if (L3_.empty()) throw Error(LZB_ERR_INVALID, "call init_cycle first");
        if (level < 0 || level >= D_) throw Error(LZB_ERR_INVALID, "bad coarse level");
        const int N = L3_[level].N;
        if (pz0 < 0 || pz1 > N || pz0 > pz1) throw Error(LZB_ERR_INVALID, "bad z plane range");
        const int64_t cb = static_cast<int64_t>(pz0) * N * N, ce = static_cast<int64_t>(pz1) * N * N;
        if (ce <= cb) return;
        if (level + 1 == D_) {
            need_layers(3 * pz0, 3 * pz1, "galerkin_planes");
            leaf_cls([&](auto S) {
                LZB_LAUNCH(k3_galerkin<decltype(S)>, blocks_for(ce - cb, 256), 256, 0, s_, L3_[level].op.p, S, N,
                           cb, ce);
            });
        } else {
            const Src64 S{L3_[level + 1].op.p,
                          static_cast<int64_t>(L3_[level + 1].N) * L3_[level + 1].N * L3_[level + 1].N};
            LZB_LAUNCH(k3_galerkin<Src64>, blocks_for(ce - cb, 256), 256, 0, s_, L3_[level].op.p, S, N, cb, ce);
        }
    }

    // The coarse operators of levels below `level` from it (Galerkin chain);
    // level D: every coarse level from the leaves. Clears the dirty mark.
    void coarse_below(int level) {
        if (L3_.empty()) throw Error(LZB_ERR_INVALID, "call init_cycle first");
        if (level < 0 || level > D_) throw Error(LZB_ERR_INVALID, "bad level");
        for (int l = level - 1; l >= 0; --l) galerkin_planes(l, 0, L3_[l].N);
        ops_dirty_ = false;
    }

    double* level_ops(int level) const {
        if (L3_.empty() || level < 0 || level > D_) throw Error(LZB_ERR_INVALID, "bad level");
        if (level == D_ && W_) throw Error(LZB_ERR_INVALID, "leaf operators are compressed planes");
        return level == D_ ? op_.p : L3_[level].op.p;
    }

    lzb_compression_stats stats() {
        LZB_CUDA(cudaMemsetAsync(stats_.p + S_HIST, 0, 9 * sizeof(unsigned long long), s_));
        LZB_LAUNCH(k_stats3, 148 * 4, 256, 0, s_, p3_.p, nc_, stats_.p);
        unsigned long long s[20];
        LZB_CUDA(cudaMemcpyAsync(s, stats_.p, sizeof s, cudaMemcpyDeviceToHost, s_));
        sync();
        lzb_compression_stats st;
        std::memset(&st, 0, sizeof st);
        st.fine_cells = static_cast<uint64_t>(nc_);
        double ratio = 0.0;
        for (int p = 0; p <= 8; ++p) {
            st.p3_histogram[p] = s[S_HIST + p];
            st.fine_stored_bytes += s[S_HIST + p] * (p == 0 ? 1ull : 1ull + 64ull * p);
            ratio += static_cast<double>(s[S_HIST + p]) * (512.0 / (p == 0 ? 1.0 : 1.0 + 64.0 * p));
        }
        st.fine_uncompressed_bytes = 512ull * nc_;
        st.fine_factor_totals = static_cast<double>(st.fine_uncompressed_bytes) / st.fine_stored_bytes;
        st.fine_factor_mean = ratio / nc_;
        st.max_n = n_last_;
        st.avg_n = n_last_;
        double md;
        std::memcpy(&md, &s[S_MAXDELTA], sizeof md);
        st.max_delta = md;
        st.total_stored_bytes = st.fine_stored_bytes;
        st.total_uncompressed_bytes = st.fine_uncompressed_bytes;
        st.total_factor = st.fine_factor_totals;
        return st;
    }

    void cells(int64_t first, int64_t count, double* ops, int32_t* p3) {
        if (first < 0 || count < 0 || first + count > nc_) throw Error(LZB_ERR_INVALID, "bad cell range");
        if (ops && count > 0)
            need_layers(static_cast<int>(first / N_ / N_), static_cast<int>((first + count - 1) / N_ / N_) + 1, "cells");
        std::vector<double> cls(static_cast<size_t>(count) * kCls3);
        if (ops && count > 0) {
            DevBuf<double> tmp;
            tmp.alloc(cls.size());
            leaf_cls([&](auto S) {
                LZB_LAUNCH(k3_read_cls<decltype(S)>, blocks_for(count, 128), 128, 0, s_, S, first, count, tmp.p);
            });
            LZB_CUDA(cudaMemcpyAsync(cls.data(), tmp.p, cls.size() * sizeof(double), cudaMemcpyDeviceToHost, s_));
            LZB_CUDA(cudaStreamSynchronize(s_));
        }
        std::vector<int8_t> q(count);
        if (p3) LZB_CUDA(cudaMemcpyAsync(q.data(), p3_.p + first, count, cudaMemcpyDeviceToHost, s_));
        sync();
        if (ops)  // the 64 entries of each class record
            for (int64_t i = 0; i < count; ++i)
                for (int a = 0; a < 8; ++a)
                    for (int b = 0; b < 8; ++b) ops[64 * i + 8 * a + b] = cls[kCls3 * i + cls3(a, b)];
        if (p3)
            for (int64_t i = 0; i < count; ++i) p3[i] = q[i];
    }

    // ------------------------------------------------------- 3D cycle
    void init_cycle(int variant, double omega, double rhs_scale, uint64_t noise_seed, int max_cycles,
                    double target) {
        if (variant == LZB_ADAFAC_JAC) throw Error(LZB_ERR_INVALID, "the 3D cycle runs additive and adafac-pi");
        variant_ = variant;
        omega_ = omega;
        max_cycles_ = max_cycles;
        target_ = target;
        L3_.resize(D_ + 1);
        for (int l = 0; l <= D_; ++l) {
            Lev& L = L3_[l];
            L.N = 1;
            for (int i = 0; i < l; ++i) L.N *= 3;
            L.nv = static_cast<int64_t>(L.N + 1) * (L.N + 1) * (L.N + 1);
            L.h = std::pow(1.0 / 3, l);
            for (int f = 0; f < LZB_V_NFIELDS; ++f) {
                L.v[f].alloc(L.nv);
                LZB_CUDA(cudaMemsetAsync(L.v[f].p, 0, L.v[f].bytes(), s_));
            }
            // the coarse operators survive a re-initialisation of the cycle (a fresh
            // allocation holds nothing: they are then re-formed from the leaves)
            const size_t nop = static_cast<size_t>(L.N) * L.N * L.N * kCls3;
            if (l < D_ && L.op.n != nop) {
                L.op.alloc(nop);
                ops_dirty_ = true;
            }
        }
        partial3_.alloc(kNormBlocks3);
        leaf_diag_dirty_ = true;  // fresh vertex arrays
        vkey_[0] = vkey_[1] = vkey_[2] = nullptr;
        upload_galerkin_weights();
        res3_.alloc(1);
        for (int l = 0; l <= D_; ++l)
            LZB_LAUNCH(k3_noise, vg(l), 128, 0, s_, lv(l), l, noise_seed, 0.0);
        inject3();
        LZB_LAUNCH(k3_init_rhs, vg(D_), 128, 0, s_, lv(D_), rhs_scale, L3_[D_].h * L3_[D_].h * L3_[D_].h / 8.0);
        cycle_ = 0;
        history_.clear();
        sync();
    }

    // Coarse operators from the leaves (after an assembly): Galerkin, finest first.
    void coarse_ops() {
        need_whole("coarse operators from every leaf");
        for (int l = D_ - 1; l >= 0; --l) galerkin_planes(l, 0, L3_[l].N);
    }

    // A multiplicative V(nu, nu) cycle on the same hierarchy (BASELINE
    // configs[1..2] name V(1,1) / V(2,2) cycles; the reference has only the
    // additive cycle, so this is a restated extension, oracle/port3.py
    // Cycle3.vstep): per level from the leaves, nu damped-Jacobi sweeps,
    // the residual restricted (R = P^T, the restriction of the additive
    // cycle) into the next level's right-hand side with a zero start; at the
    // bottom back up, the coarse correction prolongated (P, the additive
    // cycle's interpolation) and nu sweeps. The report's residual is the
    // leaf residual before the cycle.
    lzb_cycle_report vcycle(int nu) {
        if (L3_.empty()) throw Error(LZB_ERR_INVALID, "call init_cycle first");
        if (nu < 0) throw Error(LZB_ERR_INVALID, "nu must be >= 0");
        need_whole("vcycle");
        if (ops_dirty_) {
            coarse_ops();
            ops_dirty_ = false;
        }
        lzb_cycle_report rep;
        std::memset(&rep, 0, sizeof rep);
        rep.cycle = static_cast<int32_t>(++cycle_);
        struct Alias {  // the level views alias u-hat to u for this cycle
            bool& f;
            explicit Alias(bool& x) : f(x) { f = true; }
            ~Alias() { f = false; }
        } alias(uhat_is_u_);
        auto residual_plain = [&](int l) { residual3(l, 0, L3_[l].N + 1); };  // r (and r-hat = r) from fl
        auto smooth = [&](int l, int k) {
            for (int i = 0; i < k; ++i) {
                residual_plain(l);
                LZB_LAUNCH(k3_jacobi, vg(l), 128, 0, s_, lv(l), omega_);
            }
        };
        residual_plain(D_);
        LZB_CUDA(cudaMemsetAsync(partial3_.p, 0, partial3_.bytes(), s_));
        if (L3_[D_].N > 1)
            LZB_LAUNCH(k3_norm_partial, kNormBlocks3, 256, 0, s_, lv(D_), partial3_.p, 0, L3_[D_].N + 1);
        std::vector<double> part(kNormBlocks3);
        LZB_CUDA(cudaMemcpyAsync(part.data(), partial3_.p, kNormBlocks3 * sizeof(double), cudaMemcpyDeviceToHost, s_));
        sync();
        double s2 = 0.0;
        for (double x : part) s2 += x;
        rep.residual = std::sqrt(s2);
        if (history_.empty()) first_ = rep.residual > 0.0 ? rep.residual : 1.0;
        history_.push_back(rep.residual);
        rep.normalized = rep.residual / first_;
        rep.status = rep.normalized <= target_ ? LZB_CONVERGED
                     : rep.normalized >= 1e2 ? LZB_DIVERGED
                     : static_cast<int>(cycle_) >= max_cycles_ ? LZB_TIMEOUT : LZB_CONTINUE;
        if (rep.status == LZB_CONTINUE || rep.status == LZB_TIMEOUT) {
            for (int l = D_; l >= 1; --l) {
                smooth(l, nu);
                residual_plain(l);
                restrict3(l, 0, L3_[l - 1].N + 1);  // fl_{l-1} = P^T r_l
                LZB_CUDA(cudaMemsetAsync(L3_[l - 1].v[LZB_V_U].p, 0, L3_[l - 1].v[LZB_V_U].bytes(), s_));
            }
            for (int l = 1; l <= D_; ++l) {
                // u_l += P u_{l-1}: the additive cycle's prolongation with a zero snapshot
                LZB_CUDA(cudaMemsetAsync(L3_[l - 1].v[LZB_V_USNAP].p, 0, L3_[l - 1].v[LZB_V_USNAP].bytes(), s_));
                LZB_LAUNCH(k3_prolong, vg(l), 128, 0, s_, lv(l), lv(l - 1));
                smooth(l, nu);
            }
            // coarse u held corrections: re-inject the fine solution so that a
            // later additive step() forms u-hat = u - P u_c from the additive
            // cycle's invariant (finish_cycle_sync, solver.cpp:344-347)
            inject3();
            const uint64_t Nf = static_cast<uint64_t>(L3_[D_].N);
            rep.dof_updates = static_cast<uint64_t>(2 * nu) * (Nf - 1) * (Nf - 1) * (Nf - 1);
        }
        rep.levels = D_ + 1;
        rep.cells = static_cast<uint64_t>(nc_);
        sync();
        return rep;
    }

    lzb_cycle_report step() {
        if (L3_.empty()) throw Error(LZB_ERR_INVALID, "call init_cycle first");
        need_whole("step");
        if (ops_dirty_) {
            coarse_ops();
            ops_dirty_ = false;
        }
        lzb_cycle_report rep;
        std::memset(&rep, 0, sizeof rep);
        rep.cycle = static_cast<int32_t>(++cycle_);
        // the leaf residual also sums r^2 (TMA kernel, NORM): no separate pass over r
        const bool fused = use_tma_ && L3_[D_].N > 1 && std::getenv("LZB_PLAIN_NORM") == nullptr;
        for (int l = D_; l >= 0; --l) {
            uhat3(l, 0, L3_[l].N + 1);
            fuse_norm_ = fused && l == D_;
            residual3(l, 0, L3_[l].N + 1);
            fuse_norm_ = false;
            if (l > 0) restrict3(l, 0, L3_[l - 1].N + 1);
        }
        double s2 = 0.0;
        if (fused) {
            LZB_LAUNCH(k3_sum_wide, 1, 1024, 0, s_, static_cast<const double*>(rpartial_.p), norm_blocks_, res3_.p);
            LZB_CUDA(cudaMemcpyAsync(&s2, res3_.p, sizeof(double), cudaMemcpyDeviceToHost, s_));
            sync();
        } else {
            const int ng = L3_[D_].N > 1 ? kNormBlocks3 : 1;
            LZB_CUDA(cudaMemsetAsync(partial3_.p, 0, partial3_.bytes(), s_));
            if (L3_[D_].N > 1) LZB_LAUNCH(k3_norm_partial, ng, 256, 0, s_, lv(D_), partial3_.p, 0, L3_[D_].N + 1);
            std::vector<double> part(kNormBlocks3);
            LZB_CUDA(cudaMemcpyAsync(part.data(), partial3_.p, kNormBlocks3 * sizeof(double), cudaMemcpyDeviceToHost,
                                     s_));
            sync();
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
            // the update pass (solver.cpp:212-313) and the prolongation cascade
            // (solver.cpp:315-342); the leaf level's three updates run last, fused
            for (int l = 0; l < D_; ++l) LZB_LAUNCH(k3_snap, blocks_for(L3_[l].nv, 256), 256, 0, s_, lv(l), L3_[l].nv);
            const bool pi = variant_ == LZB_ADAFAC_PI;
            if (pi && D_ > 0) LZB_LAUNCH(k3_aux_inject, vg(D_ - 1), 128, 0, s_, lv(D_), lv(D_ - 1));
            for (int l = D_ - 1; l >= 0; --l) {
                if (pi && l > 0) {
                    LZB_LAUNCH(k3_aux_inject, vg(l - 1), 128, 0, s_, lv(l), lv(l - 1));
                    LZB_LAUNCH(k3_aux_sub, vg(l), 128, 0, s_, lv(l), lv(l - 1), omega_);
                }
                LZB_LAUNCH(k3_jacobi, vg(l), 128, 0, s_, lv(l), damping3(l));
            }
            for (int l = 1; l < D_; ++l) LZB_LAUNCH(k3_prolong, vg(l), 128, 0, s_, lv(l), lv(l - 1));
            if (D_ > 0)
                update_fine3(0, L3_[D_].N + 1, pi, damping3(D_));
            else
                LZB_LAUNCH(k3_jacobi, vg(0), 128, 0, s_, lv(0), damping3(0));
            inject3();
            const uint64_t Nf = static_cast<uint64_t>(L3_[D_].N);
            rep.dof_updates = (Nf - 1) * (Nf - 1) * (Nf - 1);
        }
        rep.levels = D_ + 1;
        rep.cells = static_cast<uint64_t>(nc_);
        sync();
        return rep;
    }

    // ---------------------------------------- slab-distributed 3D cycle
    // The 2D scheme of Grid::dist_phase on z-slabs of leaf vertex planes
    // [v0, v1) (multiples of 3; the last slab ends at N+1), the coarse levels
    // replicated; phases 0..5 with the host exchanges in between
    // (parallel.dist_cycle3): 0 leaf û (slab +-1 plane), residual, norm^2
    // partial -> r̂ halo (3 planes); 1 restriction into the slab's level-(D-1)
    // planes -> all-gather fl_{D-1}; 2 residual pass of the coarse levels ->
    // all-reduce norm^2, report; 3 snapshots, adaFAC-PI injection of the slab's
    // aux_{D-1} planes -> all-gather; 4 coarse updates, prolongation to D-1,
    // the slab's leaf aux correction / Jacobi / prolongation, injection of its
    // u_{D-1} planes -> all-gather; 5 coarse injections -> u halo (1 plane).
    void set_slab(int v0, int v1) {
        if (L3_.empty()) throw Error(LZB_ERR_INVALID, "call init_cycle first");
        const int NV = L3_[D_].N + 1;
        if (D_ < 1 || v0 < 0 || v1 > NV || v0 >= v1 || v0 % 3 != 0 || (v1 % 3 != 0 && v1 != NV))
            throw Error(LZB_ERR_INVALID, "bad slab planes");
        sv0_ = v0;
        sv1_ = v1;
    }
    Lv3 lvz(int l, int z0) const {
        Lv3 v = lv(l);
        v.z0 = z0;
        return v;
    }
    dim3 vgz(int l, int z0, int z1) const { return dim3(blocks_for(L3_[l].N + 1, 128), L3_[l].N + 1, z1 - z0); }

    void* dist_result_dev() const { return res3_.p; }
    lzb_ctx* context() const { return ctx_; }
    int depth() const { return D_; }
    int variant() const { return variant_; }
    void dist_phase(int phase, int flags = 0) {
        if (L3_.empty()) throw Error(LZB_ERR_INVALID, "call init_cycle first");
        const int N = L3_[D_].N, v0 = sv0_, v1 = sv1_ < 0 ? N + 1 : sv1_;
        const int c0 = v0 / 3, c1 = (v1 + 2) / 3;
        switch (phase) {
            case 0: {
                if (ops_dirty_) {
                    coarse_ops();
                    ops_dirty_ = false;
                }
                ++cycle_;
                const int u0 = std::max(v0 - 1, 0), u1 = std::min(v1 + 1, N + 1);
                uhat3(D_, u0, u1);
                residual3(D_, v0, v1);
                LZB_CUDA(cudaMemsetAsync(partial3_.p, 0, partial3_.bytes(), s_));
                LZB_LAUNCH(k3_norm_partial, kNormBlocks3, 256, 0, s_, lv(D_), partial3_.p, v0, v1);
                break;
            }
            case 1:
                restrict3(D_, c0, c1);
                break;
            case 2: {
                for (int l = D_ - 1; l >= 0; --l) {
                    uhat3(l, 0, L3_[l].N + 1);
                    residual3(l, 0, L3_[l].N + 1);
                    if (l > 0) restrict3(l, 0, L3_[l - 1].N + 1);
                }
                if (flags & 2) {  // the C++ data plane: the slab's norm^2 stays on the device (dist.cpp)
                    LZB_LAUNCH(k3_sum_partials, 1, 32, 0, s_, partial3_.p, kNormBlocks3, res3_.p);
                    break;
                }
                std::vector<double> part(kNormBlocks3);
                LZB_CUDA(cudaMemcpyAsync(part.data(), partial3_.p, kNormBlocks3 * sizeof(double),
                                         cudaMemcpyDeviceToHost, s_));
                sync();
                dist_norm2_ = 0.0;
                for (double x : part) dist_norm2_ += x;
                break;
            }
            case 3:
                for (int l = 0; l < D_; ++l)
                    LZB_LAUNCH(k3_snap, blocks_for(L3_[l].nv, 256), 256, 0, s_, lv(l), L3_[l].nv);
                if (variant_ == LZB_ADAFAC_PI)
                    LZB_LAUNCH(k3_aux_inject, vgz(D_ - 1, c0, c1), 128, 0, s_, lv(D_), lvz(D_ - 1, c0));
                break;
            case 4: {
                for (int l = D_ - 1; l >= 0; --l) {
                    if (variant_ == LZB_ADAFAC_PI && l > 0) {
                        LZB_LAUNCH(k3_aux_inject, vg(l - 1), 128, 0, s_, lv(l), lv(l - 1));
                        LZB_LAUNCH(k3_aux_sub, vg(l), 128, 0, s_, lv(l), lv(l - 1), omega_);
                    }
                    LZB_LAUNCH(k3_jacobi, vg(l), 128, 0, s_, lv(l), damping3(l));
                }
                for (int l = 1; l < D_; ++l) LZB_LAUNCH(k3_prolong, vg(l), 128, 0, s_, lv(l), lv(l - 1));
                // the slab's leaf planes: aux correction, Jacobi, prolongation (fused, the one-GPU kernel)
                update_fine3(v0, v1, variant_ == LZB_ADAFAC_PI, damping3(D_));
                LZB_LAUNCH(k3_inject, vgz(D_ - 1, c0, c1), 128, 0, s_, lv(D_), lvz(D_ - 1, c0));
                break;
            }
            case 5:
                for (int l = D_ - 1; l >= 1; --l) LZB_LAUNCH(k3_inject, vg(l - 1), 128, 0, s_, lv(l), lv(l - 1));
                if (!(flags & 2)) sync();
                break;
            default: throw Error(LZB_ERR_INVALID, "unknown phase");
        }
    }

    double dist_norm2() const { return dist_norm2_; }

    // Average device ms of one leaf-level cycle kernel (LZB_TK_UHAT, _RESIDUAL,
    // _RESTRICT, _JACOBI, _PROLONG) over `reps` back-to-back launches, CUDA
    // events on the solve stream.
    double time_kernel(int what, int reps) {
        if (L3_.empty()) throw Error(LZB_ERR_INVALID, "call init_cycle first");
        if (reps < 1) throw Error(LZB_ERR_INVALID, "reps must be >= 1");
        if (D_ < 1) throw Error(LZB_ERR_INVALID, "needs depth >= 1");
        need_whole("time_kernel");
        if (ops_dirty_) {
            coarse_ops();
            ops_dirty_ = false;
        }
        auto launch = [&] {
            switch (what) {
                case LZB_TK_UHAT: uhat3(D_, 0, L3_[D_].N + 1); break;
                case LZB_TK_RESIDUAL: residual3(D_, 0, L3_[D_].N + 1); break;
                case LZB_TK_RESTRICT: restrict3(D_, 0, L3_[D_ - 1].N + 1); break;
                case LZB_TK_JACOBI: LZB_LAUNCH(k3_jacobi, vg(D_), 128, 0, s_, lv(D_), 0.0); break;
                case LZB_TK_PROLONG: LZB_LAUNCH(k3_prolong, vg(D_), 128, 0, s_, lv(D_), lv(D_ - 1)); break;
                case LZB_TK_BACK:  // the fused leaf update with the cycle's own damping (u drifts by the Jacobi and
                                   // prolongated corrections; a zero damping would send every damping / diag
                                   // through the division's slow path, which no cycle does)
                    update_fine3(0, L3_[D_].N + 1, true, damping3(D_));
                    break;
                default: throw Error(LZB_ERR_INVALID, "unknown kernel id");
            }
        };
        launch();
        cudaEvent_t a, b;
        LZB_CUDA(cudaEventCreate(&a));
        LZB_CUDA(cudaEventCreate(&b));
        LZB_CUDA(cudaEventRecord(a, s_));
        for (int i = 0; i < reps; ++i) launch();
        LZB_CUDA(cudaEventRecord(b, s_));
        LZB_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        LZB_CUDA(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        sync();
        return static_cast<double>(ms) / reps;
    }

    lzb_cycle_report dist_report(double norm2) {
        lzb_cycle_report rep;
        std::memset(&rep, 0, sizeof rep);
        rep.cycle = static_cast<int32_t>(cycle_);
        rep.residual = std::sqrt(norm2);
        if (history_.empty()) first_ = rep.residual > 0.0 ? rep.residual : 1.0;
        history_.push_back(rep.residual);
        rep.normalized = rep.residual / first_;
        rep.status = rep.normalized <= target_ ? LZB_CONVERGED
                     : rep.normalized >= 1e2 ? LZB_DIVERGED
                     : static_cast<int>(cycle_) >= max_cycles_ ? LZB_TIMEOUT : LZB_CONTINUE;
        if (rep.status == LZB_CONTINUE || rep.status == LZB_TIMEOUT) {
            const uint64_t Nf = static_cast<uint64_t>(L3_[D_].N);
            rep.dof_updates = (Nf - 1) * (Nf - 1) * (Nf - 1);
        }
        rep.levels = D_ + 1;
        rep.cells = static_cast<uint64_t>(nc_);
        return rep;
    }

    void* device_field(int level, int field) const {
        if (L3_.empty() || level < 0 || level > D_ || field < 0 || field >= LZB_V_NFIELDS)
            throw Error(LZB_ERR_INVALID, "bad level / field");
        return L3_[level].v[field].p;
    }

    void vertices(int level, int field, double* out) {
        if (L3_.empty() || level < 0 || level > D_ || field < 0 || field >= LZB_V_NFIELDS)
            throw Error(LZB_ERR_INVALID, "bad level / field");
        LZB_CUDA(cudaMemcpyAsync(out, L3_[level].v[field].p, L3_[level].v[field].bytes(), cudaMemcpyDeviceToHost, s_));
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
        if (W_) {
            LZB_CUDA(cudaMemcpy(&flag, wide_.p, sizeof(int), cudaMemcpyDeviceToHost));
            if (flag) {
                LZB_CUDA(cudaMemset(wide_.p, 0, sizeof(int)));
                throw Error(LZB_ERR_RESOURCE, "a record's p3 exceeds plane_width");
            }
        }
    }

private:
    lzb_ctx* ctx_;
    cudaStream_t s_ = nullptr;
    int D_, N_ = 1, n_last_ = 0, fixed_, W_ = 0;
    int64_t nc_ = 1, ncs_ = 1;  // leaf cells, storage elements of one leaf plane
    int wz0_ = 0, wz1_ = 1;     // the stored leaf cell layers (a z window; the whole level by default)
    int64_t woff_ = 0;          // storage index of layer wz0_ (plane_sidx)
    int xp_ = 16;                // padded x extent of the leaf planes
    double h_ = 1.0, delta_;
    Field3 F_{};
    DevBuf<double> table_, op_, ec_;
    DevBuf<uint8_t> planes_;
    DevBuf<int> wide_;
    DevBuf<int8_t> p3_;
    DevBuf<int32_t> n_;
    DevBuf<unsigned long long> stats_;
    // 3D cycle
    struct Lev {
        int N = 1;
        int64_t nv = 8;
        double h = 1.0;
        DevBuf<double> v[LZB_V_NFIELDS];
        DevBuf<double> op;  // coarse levels (the leaves use op_)
    };
    static constexpr int kNormBlocks3 = 148 * 4;
    std::vector<Lev> L3_;
    DevBuf<double> partial3_, res3_;
    int variant_ = LZB_ADDITIVE, max_cycles_ = 100;
    double omega_ = 0.6, target_ = 1e-10, first_ = 1.0;
    uint32_t cycle_ = 0;
    bool ops_dirty_ = true;
    std::vector<double> history_;
    int sv0_ = 0, sv1_ = -1;
    double dist_norm2_ = 0.0;

    Lv3 lv(int l) const {
        Lv3 v{};
        v.N = L3_[l].N;
        v.h = L3_[l].h;
        for (int f = 0; f < LZB_V_NFIELDS; ++f) v.v[f] = L3_[l].v[f].p;
        v.op = l == D_ ? op_.p : L3_[l].op.p;
        if (uhat_is_u_) v.v[LZB_V_UHAT] = v.v[LZB_V_U];  // V-cycle: u-hat = u without a copy
        return v;
    }
    Planes3 planes() const {
        Planes3 P{};
        P.base = planes_.p;
        P.ec = ec_.p;
        P.nc = ncs_;
        P.N = N_;
        P.xp = xp_;
        P.woff = woff_;
        P.h = h_;
        const AxisTab3 T1 = axis_tab3(1);
        for (int c = 0; c < 3; ++c) P.s1[c] = T1.s[0][c];
        return P;
    }
    // fn(source of the leaves' 27 class values) for width w (default: this grid's)
    template <class Fn>
    void leaf_cls(Fn&& fn, int w = -1) const {
        switch (w < 0 ? W_ : w) {
            case 0: fn(Src64{op_.p, ncs_, N_, xp_, woff_}); break;
            case 2: fn(SrcComp<2>{planes()}); break;
            case 3: fn(SrcComp<3>{planes()}); break;
            case 4: fn(SrcComp<4>{planes()}); break;
            case 5: fn(SrcComp<5>{planes()}); break;
            case 6: fn(SrcComp<6>{planes()}); break;
            case 7: fn(SrcComp<7>{planes()}); break;
            default: fn(SrcComp<8>{planes()}); break;
        }
    }
    // the residual kernel of level l on vertex planes [z0, z1) (the leaves
    // read this grid's leaf source): the cell-centric z-marching form
    void residual3(int l, int z0, int z1) {
        const int N = L3_[l].N;
        // planes per block: kRzChunk, halved (down to 2) while the grid is under
        // four waves of the 2 resident blocks per SM -- the coarse levels are
        // latency-bound marches otherwise (81^3: 108 blocks of 32 planes)
        const int bx = (N + kRzX - 1) / (kRzX - 1), by = (N + kRzY - 1) / (kRzY - 1);
        int zc = kRzChunk;
        while (zc > 2 && static_cast<int64_t>(bx) * by * ((z1 - z0 + zc - 1) / zc) < 4 * 2 * ctx_->sms)
            zc /= 2;
        const dim3 grid(bx, by, (z1 - z0 + zc - 1) / zc);
        const Lv3 v = lv(l);
        if (l == D_ && use_tma_) {  // the leaves: TMA-staged tiles (k3_residual_tma)
            if (leaf_diag_dirty_) {  // the Jacobi diagonal, once per change of the leaf operators
                // (a windowed grid: of the vertex planes its residual covers, always its slab's)
                const int d0 = sv1_ < 0 ? z0 : sv0_, d1 = sv1_ < 0 ? z1 : sv1_;  // the slab's planes when set
                const dim3 gd = windowed() ? vgz(D_, d0, d1) : vg(D_);
                const Lv3 vd = windowed() ? lvz(D_, d0) : lv(D_);
                if (W_ == 0) LZB_LAUNCH(k3_leaf_diag<Src64>, gd, 128, 0, s_, vd, Src64{op_.p, ncs_, N_, xp_, woff_});
                else leaf_cls([&](auto S) { LZB_LAUNCH(k3_leaf_diag<decltype(S)>, gd, 128, 0, s_, vd, S); });
                leaf_diag_dirty_ = false;
            }
            const dim3 g2(bx, by, (z1 - z0 + zc2(bx, by, z0, z1) - 1) / zc2(bx, by, z0, z1));
            const int zcl = zc2(bx, by, z0, z1);
            switch (W_) {
                case 0: launch_tma<0>(g2, v, z0, z1, zcl); break;
                case 2: launch_tma<2>(g2, v, z0, z1, zcl); break;
                case 3: launch_tma<3>(g2, v, z0, z1, zcl); break;
                case 4: launch_tma<4>(g2, v, z0, z1, zcl); break;
                case 5: launch_tma<5>(g2, v, z0, z1, zcl); break;
                case 6: launch_tma<6>(g2, v, z0, z1, zcl); break;
                case 7: launch_tma<7>(g2, v, z0, z1, zcl); break;
                default: launch_tma<8>(g2, v, z0, z1, zcl); break;
            }
            return;
        }
        if (l < D_ || W_ == 0) {
            const Src64 S = l < D_ ? Src64{L3_[l].op.p, static_cast<int64_t>(N) * N * N}
                                   : Src64{op_.p, ncs_, N_, xp_, woff_};
            LZB_LAUNCH(k3_residual_z<Src64>, grid, kRzX * kRzY, 0, s_, v, S, z0, z1, zc);
            return;
        }
        leaf_cls([&](auto S) { LZB_LAUNCH(k3_residual_z<decltype(S)>, grid, kRzX * kRzY, 0, s_, v, S, z0, z1, zc); });
    }
    // planes per block of the TMA residual: as residual3's rule with 2 blocks per SM
    int zc2(int bx, int by, int z0, int z1) const {
        int zc = kRzChunk;
        while (zc > 2 && static_cast<int64_t>(bx) * by * ((z1 - z0 + zc - 1) / zc) < 4 * 2 * ctx_->sms) zc /= 2;
        return zc;
    }
    // TMA tensor maps of the leaf planes (built once: the storage never moves)
    bool use_tma_ = std::getenv("LZB_NO_TMA") == nullptr;
    bool maps_ready_ = false;
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Encode encode_fn() {  // the driver's cuTensorMapEncodeTiled (no link-time libcuda dependency)
        static Encode encode = nullptr;
        if (!encode) {
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            LZB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
            if (!fn || q != cudaDriverEntryPointSuccess) throw Error(LZB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
            encode = reinterpret_cast<Encode>(fn);
        }
        return encode;
    }
    TmaMaps maps_{};
    void build_maps() {
        if (maps_ready_) return;
        auto encode = encode_fn();
        auto dtype = [](int e) {
            return e == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : e == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32
                   : e == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_UINT8;
        };
        auto make = [&](CUtensorMap* m, void* base, int e, int rank) {
            const cuuint64_t dims[4] = {static_cast<cuuint64_t>(xp_), static_cast<cuuint64_t>(N_ + 1),
                                        static_cast<cuuint64_t>(wz1_ - wz0_), 27};
            const cuuint64_t strides[3] = {static_cast<cuuint64_t>(xp_) * e,
                                           static_cast<cuuint64_t>(xp_) * (N_ + 1) * e,
                                           static_cast<cuuint64_t>(ncs_) * e};
            const cuuint32_t box[4] = {static_cast<cuuint32_t>(tma_width(e)), kRzY, 1, 27}, es[4] = {1, 1, 1, 1};
            const CUresult r = encode(m, dtype(e), rank, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) throw Error(LZB_ERR_CUDA, "cuTensorMapEncodeTiled failed");
        };
        if (W_ == 0) {
            make(&maps_.piece[0], op_.p, 8, 4);
        } else {
            size_t off = 0;
            for (int k = 0; k < 3; ++k) {
                const int e = tma_piece(W_, k);
                if (!e) break;
                make(&maps_.piece[k], planes_.p + off, e, 4);
                off += static_cast<size_t>(e) * 27 * ncs_;
            }
            make(&maps_.ec, ec_.p, 8, 3);
        }
        maps_.z0 = wz0_;
        maps_ready_ = true;
    }
    template <int W>
    void launch_tma(dim3 g, const Lv3& v, int z0, int z1, int zc) {
        constexpr int S = (W >= 2 && W <= 4) ? 2 : 1;  // stages (k3_residual_tma)
        build_maps();
        vmaps(v);
        const Planes3 pl = planes();
        const bool sym = pl.s1[0] == pl.s1[2];
        double* np = nullptr;
        if (fuse_norm_) {  // step(): the norm partials come from this launch
            norm_blocks_ = static_cast<int>(g.x * g.y * g.z);
            if (rpartial_.n < static_cast<size_t>(norm_blocks_)) rpartial_.alloc(norm_blocks_);
            np = rpartial_.p;
        }
        static bool attr = false;  // per width: the four variants share the launch shape
        if (!attr) {
            const int bytes = tma_smem_bytes2(W, S);
            LZB_CUDA(cudaFuncSetAttribute(k3_residual_tma<W, S, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
            LZB_CUDA(cudaFuncSetAttribute(k3_residual_tma<W, S, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
            LZB_CUDA(cudaFuncSetAttribute(k3_residual_tma<W, S, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
            LZB_CUDA(cudaFuncSetAttribute(k3_residual_tma<W, S, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
            attr = true;
        }
        auto go = [&](auto kern) {
            LZB_LAUNCH(kern, g, kRzX * kRzY, tma_smem_bytes2(W, S), s_, v, maps_, vmaps_, pl, z0, z1, zc, np);
        };
        if (sym && np) go(k3_residual_tma<W, S, true, true>);
        else if (sym) go(k3_residual_tma<W, S, true, false>);
        else if (np) go(k3_residual_tma<W, S, false, true>);
        else go(k3_residual_tma<W, S, false, false>);
    }
    bool fuse_norm_ = false;  // set by step() around the leaf residual
    int norm_blocks_ = 0;
    DevBuf<double> rpartial_;
    // fl_{l-1} = P^T r-hat_l on the coarse vertex planes [c0, c1) of level l - 1
    void restrict3(int l, int c0, int c1) {
        static const bool plain = std::getenv("LZB_PLAIN_RESTRICT") != nullptr;
        if (plain) {
            LZB_LAUNCH(k3_restrict, vgz(l - 1, c0, c1), 128, 0, s_, lv(l), lvz(l - 1, c0));
            return;
        }
        const int NVc = L3_[l - 1].N + 1;
        const int bx = (NVc + kRsX - 1) / kRsX, by = (NVc + kRsY - 1) / kRsY;
        // chunks of coarse planes: one wave of resident blocks (8 per SM: 27 KB of shared
        // memory, 62 registers), no partial second wave; each chunk re-reads 4 fine planes
        int chunks = static_cast<int>(8LL * ctx_->sms / (static_cast<int64_t>(bx) * by));
        chunks = std::max(1, std::min(chunks, (c1 - c0 + 3) / 4));
        const int zc = (c1 - c0 + chunks - 1) / chunks;
        LZB_LAUNCH(k3_restrict_zm, dim3(bx, by, (c1 - c0 + zc - 1) / zc), kRsX * kRsY, 0, s_, lv(l), lv(l - 1), c0,
                   c1, zc);
    }
    bool leaf_diag_dirty_ = true;
    // TMA maps of the leaf vertex fields the residual reads (u, u-hat -- u
    // itself during V-cycles -- and the load), rebuilt when the pointers change
    TmaVMaps vmaps_{};
    const void* vkey_[3] = {nullptr, nullptr, nullptr};
    void vmaps(const Lv3& v) {
        const void* key[3] = {v.v[LZB_V_U], v.v[LZB_V_UHAT], v.v[LZB_V_FL]};
        if (key[0] == vkey_[0] && key[1] == vkey_[1] && key[2] == vkey_[2]) return;
        const cuuint64_t NV = static_cast<cuuint64_t>(N_) + 1;
        const cuuint64_t dims[3] = {NV, NV, NV}, strides[2] = {NV * 8, NV * NV * 8};
        auto make = [&](CUtensorMap* m, const void* base, cuuint32_t bx, cuuint32_t by) {
            const cuuint32_t box[3] = {bx, by, 1}, es[3] = {1, 1, 1};
            const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(base), dims, strides,
                                           box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) throw Error(LZB_ERR_CUDA, "cuTensorMapEncodeTiled failed (vertex tiles)");
        };
        make(&vmaps_.u, key[0], kTmaUX, kTmaUY);
        make(&vmaps_.uh, key[1], kTmaUX, kTmaUY);
        make(&vmaps_.fl, key[2], kTmaFX, kTmaFY);
        for (int i = 0; i < 3; ++i) vkey_[i] = key[i];
    }
    bool uhat_is_u_ = false;
    double damping3(int l) const { return variant_ == LZB_ADDITIVE ? std::pow(omega_, D_ - l + 1) : omega_; }
    dim3 vg(int l) const { return dim3(blocks_for(L3_[l].N + 1, 128), L3_[l].N + 1, L3_[l].N + 1); }
    // u-hat of level l on vertex planes [z0, z1): the leaf level (and any level
    // with a coarse level below) through the staged row kernel
    void uhat3(int l, int z0, int z1) {
        if (l == 0) LZB_LAUNCH(k3_uhat, vgz(0, z0, z1), 128, 0, s_, lvz(0, z0), lv(0), 0);
        else if (L3_[l].N >= 243 && std::getenv("LZB_UHAT3_MARCH") != nullptr) {  // opt-in: measured slower, see the kernel
            const int64_t blocks27 = static_cast<int64_t>(blocks_for(L3_[l].N + 1, kStThreads)) *
                                     ((L3_[l - 1].N + kMarchPatches - 1) / kMarchPatches) * (z1 - z0);
            const int pg = blocks27 >= 24LL * ctx_->sms ? kMarchPatches : kMarchPatches / 3;
            LZB_LAUNCH(k3_uhat_march, dim3(blocks_for(L3_[l].N + 1, kStThreads), (L3_[l - 1].N + pg - 1) / pg, z1 - z0),
                       kStThreads, 0, s_, lvz(l, z0), lv(l - 1), pg);
        } else LZB_LAUNCH(k3_uhat_st, vgst(l, z0, z1), kStThreads, 0, s_, lvz(l, z0), lv(l - 1));
    }
    // the staged row kernels: 128 x, kStY rows, one plane per block
    dim3 vgst(int l, int z0, int z1, int rows = kStY) const {
        return dim3(blocks_for(L3_[l].N + 1, kStThreads), (L3_[l].N + rows) / rows, z1 - z0);
    }
    // the leaf level's fused update on vertex planes [z0, z1): the coarse
    // factors (aux correction, prolongated correction) once per coarse vertex,
    // then the staged row kernel
    void update_fine3(int z0, int z1, bool pi, double damping) {
        if (pre3_.n < static_cast<size_t>(L3_[D_ - 1].nv)) pre3_.alloc(L3_[D_ - 1].nv);
        LZB_LAUNCH(k3_coarse_pre, vg(D_ - 1), 128, 0, s_, lv(D_ - 1), omega_, pi ? 1 : 0, pre3_.p);
        static const bool rows = std::getenv("LZB_UPDATE3_ROWS") != nullptr;  // comparison switch (DESIGN 9b)
        if (rows)
            LZB_LAUNCH(k3_update_fine_st, vgst(D_, z0, z1, kStYu), kStThreads, 0, s_, lvz(D_, z0), lv(D_ - 1), pre3_.p,
                       pi ? 1 : 0, damping);
        else
        {
            // 27 patch rows per block where that still fills the GPU several times over, else 9 (243^3: 726 blocks
            // of 27 are 1.6 waves; measured 0.119 vs 0.109 ms)
            static const int pg_env = std::getenv("LZB_UPDATE3_PG") ? std::max(1, std::atoi(std::getenv("LZB_UPDATE3_PG"))) : 0;
            const int64_t blocks27 = static_cast<int64_t>(blocks_for(L3_[D_].N + 1, kStThreads)) *
                                     ((L3_[D_ - 1].N + kMarchPatches - 1) / kMarchPatches) * (z1 - z0);
            const int pg = pg_env ? pg_env : blocks27 >= 24LL * ctx_->sms ? kMarchPatches : kMarchPatches / 3;
            LZB_LAUNCH(k3_update_fine_march, dim3(blocks_for(L3_[D_].N + 1, kStThreads), (L3_[D_ - 1].N + pg - 1) / pg, z1 - z0),
                       kStThreads, 0, s_, lvz(D_, z0), lv(D_ - 1), pre3_.p, pi ? 1 : 0, damping, pg);
        }
    }
    DevBuf<double2> pre3_;
    void inject3() {
        for (int l = D_; l >= 1; --l) LZB_LAUNCH(k3_inject, vg(l - 1), 128, 0, s_, lv(l), lv(l - 1));
    }
};

}  // namespace lzb

struct lzb_grid3 {
    std::unique_ptr<lzb::Grid3> g;
};

extern "C" {

int lzb_grf_table(uint64_t seed, int n, double ell, double sigma2, double* out) { LZB_RANGE("lzb_grf_table");
    return lzb::guarded([&] { lzb::grf_table(seed, n, ell, sigma2, out); });
}

int lzb_integrate_elements3(lzb_ctx* ctx, const lzb_field3* f, int64_t count, const double* x0, const double* y0,
                            const double* z0, const double* h, const int32_t* n, double* out) { LZB_RANGE("lzb_integrate_elements3");
    return lzb::guarded([&] {
        using namespace lzb;
        if (count <= 0) return;
        LZB_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t s = ctx->solve;
        DevBuf<double> table;
        const Field3 F = to_device(*f, table);
        DevBuf<double> dx, dy, dz, dh, dout;
        DevBuf<int32_t> dn;
        for (auto* b : {&dx, &dy, &dz, &dh}) b->alloc(count);
        dn.alloc(count);
        dout.alloc(static_cast<size_t>(count) * 64);
        LZB_CUDA(cudaMemcpyAsync(dx.p, x0, count * 8, cudaMemcpyHostToDevice, s));
        LZB_CUDA(cudaMemcpyAsync(dy.p, y0, count * 8, cudaMemcpyHostToDevice, s));
        LZB_CUDA(cudaMemcpyAsync(dz.p, z0, count * 8, cudaMemcpyHostToDevice, s));
        LZB_CUDA(cudaMemcpyAsync(dh.p, h, count * 8, cudaMemcpyHostToDevice, s));
        LZB_CUDA(cudaMemcpyAsync(dn.p, n, count * 4, cudaMemcpyHostToDevice, s));
        std::vector<int> seen(kMaxN3 + 1, 0);
        for (int64_t i = 0; i < count; ++i) {
            if (n[i] < 1 || n[i] > kMaxN3) throw Error(LZB_ERR_INVALID, "3D sub-samples per axis must be in 1..16");
            seen[n[i]] = 1;
        }
        for (int q = 1; q <= kMaxN3; ++q)
            if (seen[q])
                LZB_LAUNCH(k_elements3, blocks_for(count, 128), 128, 0, s, F, count, dx.p, dy.p, dz.p, dh.p, dn.p,
                           axis_tab3(q), dout.p);
        LZB_CUDA(cudaMemcpyAsync(out, dout.p, static_cast<size_t>(count) * 64 * 8, cudaMemcpyDeviceToHost, s));
        LZB_CUDA(cudaStreamSynchronize(s));
    });
}

int lzb_grid3_create(lzb_ctx* ctx, int depth, const lzb_field3* f, double delta_max, int fixed_p3, lzb_grid3** out) { LZB_RANGE("lzb_grid3_create");
    return lzb_grid3_create_planes(ctx, depth, f, delta_max, fixed_p3, 0, out);
}
int lzb_grid3_create_planes(lzb_ctx* ctx, int depth, const lzb_field3* f, double delta_max, int fixed_p3,
                            int plane_width, lzb_grid3** out) { LZB_RANGE("lzb_grid3_create_planes");
    return lzb::guarded([&] {
        auto g = std::make_unique<lzb_grid3>();
        g->g = std::make_unique<lzb::Grid3>(ctx, depth, *f, delta_max, fixed_p3, plane_width);
        *out = g.release();
    });
}
int lzb_grid3_create_window(lzb_ctx* ctx, int depth, const lzb_field3* f, double delta_max, int fixed_p3,
                            int plane_width, int cz0, int cz1, lzb_grid3** out) { LZB_RANGE("lzb_grid3_create_window");
    return lzb::guarded([&] {
        auto g = std::make_unique<lzb_grid3>();
        g->g = std::make_unique<lzb::Grid3>(ctx, depth, *f, delta_max, fixed_p3, plane_width, cz0, cz1);
        *out = g.release();
    });
}
int lzb_grid3_leaf_storage(lzb_grid3* g, int64_t* bytes, int* cz0, int* cz1) { LZB_RANGE("lzb_grid3_leaf_storage");
    return lzb::guarded([&] {
        if (bytes) *bytes = g->g->leaf_storage_bytes();
        int a, b;
        g->g->leaf_window(&a, &b);
        if (cz0) *cz0 = a;
        if (cz1) *cz1 = b;
    });
}
int lzb_grid3_destroy(lzb_grid3* g) {
    return lzb::guarded([&] { delete g; });
}
int lzb_grid3_assemble_fixed(lzb_grid3* g, int n) { LZB_RANGE("lzb_grid3_assemble_fixed");
    return lzb::guarded([&] {
        g->g->assemble_fixed(n);
        g->g->sync();
    });
}
int lzb_grid3_stats(lzb_grid3* g, lzb_compression_stats* out) { LZB_RANGE("lzb_grid3_stats");
    return lzb::guarded([&] { *out = g->g->stats(); });
}
int lzb_grid3_cells(lzb_grid3* g, int64_t first, int64_t count, double* ops, int32_t* p3) { LZB_RANGE("lzb_grid3_cells");
    return lzb::guarded([&] { g->g->cells(first, count, ops, p3); });
}
int lzb_grid3_init_cycle(lzb_grid3* g, int variant, double omega, double rhs_scale, uint64_t noise_seed,
                         int max_cycles, double target) {
    return lzb::guarded([&] { g->g->init_cycle(variant, omega, rhs_scale, noise_seed, max_cycles, target); });
}
int lzb_grid3_step(lzb_grid3* g, lzb_cycle_report* out) { LZB_RANGE("lzb_grid3_step");
    return lzb::guarded([&] { *out = g->g->step(); });
}
int lzb_grid3_vcycle(lzb_grid3* g, int nu, lzb_cycle_report* out) { LZB_RANGE("lzb_grid3_vcycle");
    return lzb::guarded([&] { *out = g->g->vcycle(nu); });
}
int lzb_grid3_vertices(lzb_grid3* g, int level, int field, double* out) { LZB_RANGE("lzb_grid3_vertices");
    return lzb::guarded([&] { g->g->vertices(level, field, out); });
}
int lzb_grid3_set_slab(lzb_grid3* g, int v0, int v1) { LZB_RANGE("lzb_grid3_set_slab");
    return lzb::guarded([&] { g->g->set_slab(v0, v1); });
}
int lzb_grid3_dist_phase(lzb_grid3* g, int phase) { LZB_RANGE("lzb_grid3_dist_phase");
    return lzb::guarded([&] { g->g->dist_phase(phase); });
}
int lzb_grid3_dist_phase_flags(lzb_grid3* g, int phase, int flags) { LZB_RANGE("lzb_grid3_dist_phase_flags");
    return lzb::guarded([&] { g->g->dist_phase(phase, flags); });
}
int lzb_grid3_dist_result_dev(lzb_grid3* g, void** norm2) {
    return lzb::guarded([&] { *norm2 = g->g->dist_result_dev(); });
}
int lzb_grid3_dist_result(lzb_grid3* g, double* norm2) {
    return lzb::guarded([&] { *norm2 = g->g->dist_norm2(); });
}
int lzb_grid3_dist_report(lzb_grid3* g, double norm2, lzb_cycle_report* out) { LZB_RANGE("lzb_grid3_dist_report");
    return lzb::guarded([&] { *out = g->g->dist_report(norm2); });
}
int lzb_grid3_assemble_planes(lzb_grid3* g, int n, int cz0, int cz1) { LZB_RANGE("lzb_grid3_assemble_planes");
    return lzb::guarded([&] {
        g->g->assemble_planes(n, cz0, cz1);
        g->g->sync();
    });
}
int lzb_grid3_galerkin_planes(lzb_grid3* g, int level, int pz0, int pz1) { LZB_RANGE("lzb_grid3_galerkin_planes");
    return lzb::guarded([&] {
        g->g->galerkin_planes(level, pz0, pz1);
        g->g->sync();
    });
}
int lzb_grid3_coarse_below(lzb_grid3* g, int level) { LZB_RANGE("lzb_grid3_coarse_below");
    return lzb::guarded([&] {
        g->g->coarse_below(level);
        g->g->sync();
    });
}
int lzb_grid3_variant(lzb_grid3* g) { LZB_RANGE("lzb_grid3_variant"); return g->g->variant(); }
int lzb_grid3_info(lzb_grid3* g, lzb_ctx** ctx, int* depth) {
    return lzb::guarded([&] {
        if (ctx) *ctx = g->g->context();
        if (depth) *depth = g->g->depth();
    });
}
int lzb_grid3_level_ops(lzb_grid3* g, int level, void** ptr) { LZB_RANGE("lzb_grid3_level_ops");
    return lzb::guarded([&] { *ptr = g->g->level_ops(level); });
}
int lzb_grid3_time_kernel(lzb_grid3* g, int what, int reps, double* avg_ms) { LZB_RANGE("lzb_grid3_time_kernel");
    return lzb::guarded([&] { *avg_ms = g->g->time_kernel(what, reps); });
}
int lzb_grid3_device_view(lzb_grid3* g, int level, int field, void** ptr) {
    return lzb::guarded([&] { *ptr = g->g->device_field(level, field); });
}

}  // extern "C"

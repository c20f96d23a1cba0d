// integrate.cuh — K1: per-cell element-matrix integration with n x n eps
// sub-samples (integrate_element, element.hpp:36-49), FP64.
//
// What depends on the cell and what does not:
//   * K_sub(i,j) = reference_subcell_stiffness(i/n,(i+1)/n,j/n,(j+1)/n) depends
//     on (n,i,j) only: tabulated ONCE per n (ktab, 9 distinct values per (i,j)
//     + 1 pad double, element.cpp:19-32 arithmetic) and staged tile by tile in
//     shared memory, read as broadcast LDS.128 by every thread of the block;
//   * the per-axis seg values (len, S0, S1, S2) of sub-interval i: per n (seg);
//   * the eps field parts: x part per (cell column, i), y part per (cell row, j)
//     (fx, fy), computed with the reference's sample-coordinate expression
//     x0 + ((i+0.5)*inv)*h (element.hpp:44) and the field's expression tree.
// A table lookup returns the very bits the reference recomputes per sample.
//
// EXACT: i-major, j-minor sequential accumulation of fl(K*e) into the 9
//        distinct accumulators (out.m += e*K, element.hpp:45): 2 + 9 + 9 DP
//        ops per sub-sample, no FMA — bit-identical to the reference.
// FAST:  separable form with explicit FMAs: per row i, s_k = sum_j e_ij S_k(j),
//        t = sum_j e_ij len_j; then U_k += len_i s_k, V_k += S_k(i) t; entries
//        are +-U +-V. 5 FMA per sub-sample; within 1e-12 relative of EXACT.
#pragma once

#include "device.cuh"

namespace lzb {

constexpr int kKs = 10;          // doubles per K_sub(i,j) table entry (9 + pad, 16 B aligned)
constexpr int kSeg = 4;          // len, S0, S1, S2
constexpr int kIntThreads = 256; // block size of the table-driven integration kernels
constexpr int kCPT = 2;          // cells per thread (share K_sub loads, 2x independent chains)
constexpr int kKTileBytes = 40 * 1024;

struct IntTables {
    const double* fx;    // [N][n] x field parts
    const double* fy;    // [N][n] y field parts
    const double* seg;   // [n][4]
    const double* ktab;  // [n][n][10]
    const double* cxp;   // [N] x field part at the cell centre (the n = 1 sample)
    const double* cyp;   // [N] y field part at the cell centre
    int n;
};

template <int KIND>
__device__ __forceinline__ double combine_k(double xp, double yp, double value, double eps_low,
                                            int blocks, const double* table) {
    if constexpr (KIND == LZB_FIELD_THETA || KIND == LZB_FIELD_SINUSOID) {
        return 1.0 + xp * yp;
    } else if constexpr (KIND == LZB_FIELD_QUADRANT) {
        return xp == yp ? 1.0 : eps_low;
    } else if constexpr (KIND == LZB_FIELD_CHECKER) {
        return table[static_cast<int>(xp) * blocks + static_cast<int>(yp)];
    } else {
        return value;
    }
}

// Shared-memory layout used by the table-driven kernels (dynamic smem):
//   [0, 64)                checker table
//   [64, 64 + 4n)          seg table
//   [64 + 4n, ...)         K_sub tile: rows i0..i0+TI-1, n*10 doubles per row
__host__ __device__ inline int ktile_rows(int n) {
    int r = kKTileBytes / (n * kKs * 8);
    return r < 1 ? 1 : (r > n ? n : r);
}
//   [.., + kFyRows*n)      y field parts of the (<= kFyRows) cell rows the block touches
constexpr int kFyRows = 8;  // rows a block of kIntThreads*kCPT cells may span before falling back to global
__host__ inline size_t int_smem_bytes(int n) {
    return (64 + static_cast<size_t>(kSeg) * n + static_cast<size_t>(ktile_rows(n)) * n * kKs +
            static_cast<size_t>(kFyRows) * n) * 8;
}
__device__ inline double* fy_region(double* sm, int n) {
    return sm + 64 + kSeg * n + static_cast<size_t>(ktile_rows(n)) * n * kKs;
}

__device__ inline void stage_common(double* sm, const lzb_field& f, const IntTables& T) {
    for (int i = threadIdx.x; i < 64; i += blockDim.x) sm[i] = f.table[i];
    for (int i = threadIdx.x; i < kSeg * T.n; i += blockDim.x) sm[64 + i] = T.seg[i];
}

// Stage the y field parts of cell rows [row_lo, row_lo+rows) when they fit;
// returns the base the caller indexes by (cy - row_lo) * n, or nullptr (read
// the global table instead). Visible after integrate_block's first barrier.
__device__ inline const double* stage_rows(double* sm, const IntTables& T, int row_lo, int rows) {
    if (rows > kFyRows) return nullptr;
    double* dst = fy_region(sm, T.n);
    const double* src = T.fy + static_cast<size_t>(row_lo) * T.n;
    for (int i = threadIdx.x; i < rows * T.n; i += blockDim.x) dst[i] = src[i];
    return dst;
}

// Block-cooperative integration of CPT cells per thread: every thread of the
// block must call it (the K_sub tiles are staged with __syncthreads). Cell q
// of the thread is active if act[q]; its field parts are fxc[q][0..n) (its
// column) and fyc[q][0..n) (its row); inactive cells must still point at
// readable tables (their results are discarded). The CPT cells share every
// K_sub / seg load and give the DP pipe CPT x 9 independent chains.
template <int KIND, bool FAST, int CPT, bool RESIDENT = false>
__device__ __forceinline__ void integrate_block(const bool* act, const lzb_field& f, const IntTables& T,
                                                const double* const* fxc, const double* const* fyc,
                                                double* sm, double (*out16)[16]) {
    const int n = T.n;
    const double* s_tab = sm;
    const double* s_seg = sm + 64;
    double* s_k = sm + 64 + kSeg * n;
    const double value = f.value, eps_low = f.eps_low;
    const int blocks = f.blocks;
    bool any = false;
#pragma unroll
    for (int q = 0; q < CPT; ++q) any = any || act[q];
    double a[CPT][9];
#pragma unroll
    for (int q = 0; q < CPT; ++q)
#pragma unroll
        for (int r = 0; r < 9; ++r) a[q][r] = 0.0;
    if (FAST) {
        double U[CPT][3], V[CPT][3];
#pragma unroll
        for (int q = 0; q < CPT; ++q)
#pragma unroll
            for (int r = 0; r < 3; ++r) U[q][r] = V[q][r] = 0.0;
        if (!RESIDENT) __syncthreads();  // seg / rows staged by the caller
        if (any) {
            for (int i = 0; i < n; ++i) {
                double xp[CPT], s0[CPT], s1[CPT], s2[CPT], t[CPT];
#pragma unroll
                for (int q = 0; q < CPT; ++q) {
                    xp[q] = fxc[q][i];
                    s0[q] = s1[q] = s2[q] = t[q] = 0.0;
                }
#pragma unroll 2
                for (int j = 0; j < n; ++j) {
                    const double2 q0 = reinterpret_cast<const double2*>(s_seg)[2 * j];
                    const double2 q1 = reinterpret_cast<const double2*>(s_seg)[2 * j + 1];
#pragma unroll
                    for (int q = 0; q < CPT; ++q) {
                        double e;
                        if constexpr (KIND == LZB_FIELD_THETA || KIND == LZB_FIELD_SINUSOID)
                            e = __fma_rn(xp[q], fyc[q][j], 1.0);
                        else
                            e = combine_k<KIND>(xp[q], fyc[q][j], value, eps_low, blocks, s_tab);
                        t[q] = __fma_rn(e, q0.x, t[q]);
                        s0[q] = __fma_rn(e, q0.y, s0[q]);
                        s1[q] = __fma_rn(e, q1.x, s1[q]);
                        s2[q] = __fma_rn(e, q1.y, s2[q]);
                    }
                }
                const double2 p0 = reinterpret_cast<const double2*>(s_seg)[2 * i];
                const double2 p1 = reinterpret_cast<const double2*>(s_seg)[2 * i + 1];
#pragma unroll
                for (int q = 0; q < CPT; ++q) {
                    U[q][0] = __fma_rn(p0.x, s0[q], U[q][0]);
                    U[q][1] = __fma_rn(p0.x, s1[q], U[q][1]);
                    U[q][2] = __fma_rn(p0.x, s2[q], U[q][2]);
                    V[q][0] = __fma_rn(p0.y, t[q], V[q][0]);
                    V[q][1] = __fma_rn(p1.x, t[q], V[q][1]);
                    V[q][2] = __fma_rn(p1.y, t[q], V[q][2]);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            a[q][0] = U[q][0] + V[q][0];
            a[q][1] = U[q][0] + V[q][2];
            a[q][2] = U[q][2] + V[q][0];
            a[q][3] = U[q][2] + V[q][2];
            a[q][4] = V[q][1] - U[q][0];
            a[q][5] = V[q][1] - U[q][2];
            a[q][6] = U[q][1] - V[q][0];
            a[q][7] = U[q][1] - V[q][2];
            a[q][8] = -(U[q][1] + V[q][1]);
        }
    } else {
        // RESIDENT: the caller staged the whole K_sub table once (persistent kernels)
        const int TI = RESIDENT ? n : ktile_rows(n);
        for (int i0 = 0; i0 < n; i0 += TI) {
            const int rows = (n - i0) < TI ? (n - i0) : TI;
            if (!RESIDENT) {
                __syncthreads();
                {   // stage K_sub rows [i0, i0+rows) (contiguous in ktab), 16-byte vectors
                    const double2* src = reinterpret_cast<const double2*>(T.ktab + static_cast<size_t>(i0) * n * kKs);
                    double2* dst = reinterpret_cast<double2*>(s_k);
                    const int nvec = rows * n * kKs / 2;
                    for (int v = threadIdx.x; v < nvec; v += blockDim.x) dst[v] = src[v];
                }
                __syncthreads();
            }
            if (any) {
                for (int ii = 0; ii < rows; ++ii) {
                    double xp[CPT];
#pragma unroll
                    for (int q = 0; q < CPT; ++q) xp[q] = fxc[q][i0 + ii];
                    const double2* kp = reinterpret_cast<const double2*>(s_k + static_cast<size_t>(ii) * n * kKs);
#pragma unroll 2
                    for (int j = 0; j < n; ++j, kp += kKs / 2) {
                        const double2 k0 = kp[0], k1 = kp[1], k2 = kp[2], k3 = kp[3], k4 = kp[4];
#pragma unroll
                        for (int q = 0; q < CPT; ++q) {
                            const double e = combine_k<KIND>(xp[q], fyc[q][j], value, eps_low, blocks, s_tab);
                            // out.m += e * K   (Mat4 operator* rounds K*e, then +=)
                            a[q][0] = a[q][0] + k0.x * e;
                            a[q][1] = a[q][1] + k0.y * e;
                            a[q][2] = a[q][2] + k1.x * e;
                            a[q][3] = a[q][3] + k1.y * e;
                            a[q][4] = a[q][4] + k2.x * e;
                            a[q][5] = a[q][5] + k2.y * e;
                            a[q][6] = a[q][6] + k3.x * e;
                            a[q][7] = a[q][7] + k3.y * e;
                            a[q][8] = a[q][8] + k4.x * e;
                        }
                    }
                }
            }
        }
    }
#pragma unroll
    for (int q = 0; q < CPT; ++q) k9_expand(a[q], out16[q]);
}

// Persistent ("resident") layout: [64 table][4n seg][n*n*10 K_sub][kFyRows*n fy].
constexpr size_t kResidentSmemMax = 100 * 1024;  // 2 blocks per SM
__host__ __device__ inline size_t res_smem_bytes(int n) {
    return (64 + static_cast<size_t>(kSeg) * n + static_cast<size_t>(n) * n * kKs +
            static_cast<size_t>(kFyRows) * n) * 8;
}
__device__ inline double* res_fy_region(double* sm, int n) {
    return sm + 64 + kSeg * n + static_cast<size_t>(n) * n * kKs;
}

// Table builders (runtime.cu).
__global__ void k_field_parts(lzb_field f, int N, double h, int n, int axis, double* out);
__global__ void k_seg_table(int n, double* seg);
__global__ void k_ksub_table(int n, double* ktab);

// Arbitrary CellBox (x0, y0, h) at n: axis parts recomputed per sample with
// the reference arithmetic (per-cell compatibility path, no tables).
__device__ inline void integrate_cell(const lzb_field& f, double x0, double y0, double h, int n,
                                      int fast, double* out16) {
    const double inv = 1.0 / n;
    double a[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    double U[3] = {0, 0, 0}, V[3] = {0, 0, 0};
    for (int i = 0; i < n; ++i) {
        double xp = field_xpart(f, x0 + (i + 0.5) * inv * h);
        AxisSeg X = axis_seg(i, inv);
        double s[3] = {0, 0, 0}, t = 0;
        for (int j = 0; j < n; ++j) {
            double yp = field_ypart(f, y0 + (j + 0.5) * inv * h);
            double e = field_combine(f, xp, yp);
            AxisSeg Y = axis_seg(j, inv);
            if (fast) {
                t = __fma_rn(e, Y.len, t);
                s[0] = __fma_rn(e, Y.s0, s[0]);
                s[1] = __fma_rn(e, Y.s1, s[1]);
                s[2] = __fma_rn(e, Y.s2, s[2]);
            } else {
                K9 k = ksub(X, Y);
                a[0] = a[0] + k.k00 * e; a[1] = a[1] + k.k11 * e; a[2] = a[2] + k.k22 * e;
                a[3] = a[3] + k.k33 * e; a[4] = a[4] + k.k01 * e; a[5] = a[5] + k.k23 * e;
                a[6] = a[6] + k.k02 * e; a[7] = a[7] + k.k13 * e; a[8] = a[8] + k.k03 * e;
            }
        }
        if (fast) {
            for (int q = 0; q < 3; ++q) U[q] = __fma_rn(X.len, s[q], U[q]);
            V[0] = __fma_rn(X.s0, t, V[0]);
            V[1] = __fma_rn(X.s1, t, V[1]);
            V[2] = __fma_rn(X.s2, t, V[2]);
        }
    }
    if (fast) {
        a[0] = U[0] + V[0]; a[1] = U[0] + V[2]; a[2] = U[2] + V[0]; a[3] = U[2] + V[2];
        a[4] = V[1] - U[0]; a[5] = V[1] - U[2]; a[6] = U[1] - V[0]; a[7] = U[1] - V[2];
        a[8] = -(U[1] + V[1]);
    }
    k9_expand(a, out16);
}

}  // namespace lzb

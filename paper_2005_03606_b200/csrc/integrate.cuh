// integrate.cuh — K1: per-cell element-matrix integration with n x n eps
// sub-samples (integrate_element, element.hpp:36-49), FP64.
//
// Per-axis tables: for a regular level (N cells per axis, width h) and a
// sampling n, everything the inner loop needs that depends on one axis only
// is tabulated once per (cell column/row, sub-index):
//   tab[(c*n + i)*kTab + 0] = field part of eps at x_i = c*h + ((i+0.5)/n)*h
//   tab[... + 1..4]         = len_i, S0_i, S1_i, S2_i (element.cpp:8-32 on [i/n,(i+1)/n])
// The sample coordinate and every tabulated value are computed with the
// reference expression (no FMA in this TU), so a table lookup returns the same
// bits the reference recomputes per sample.
//
// EXACT: i-major, j-minor sequential accumulation of fl(e*K) into 9 distinct
//        accumulators (the 16 entries of K_sub take 9 values) — bit-identical
//        to the reference.
// FAST:  separable form with explicit FMAs: per row i, s_k = sum_j e_ij S_k(j)
//        and t = sum_j e_ij len_j, then U_k += len_i s_k, V_k += S_k(i) t;
//        entries are +-U +-V. 4 FMA per sub-sample instead of 9 mul + 9 add
//        + 9 add + 6 mul; within 1e-12 relative of EXACT (tests).
#pragma once

#include "device.cuh"

namespace lzb {

constexpr int kTab = 5;

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

// One axis table: thread per (c, i); axis 0 = x part, 1 = y part.
__global__ void k_axis_table(lzb_field f, int N, double h, int n, int axis, double* tab);

template <int KIND>
__device__ __forceinline__ void integrate_exact_tab(const double* __restrict__ tx,
                                                    const double* __restrict__ ty, int n,
                                                    double value, double eps_low, int blocks,
                                                    const double* table, double* out16) {
    double a[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < n; ++i) {
        const double* xi = tx + i * kTab;
        const double xp = xi[0];
        const AxisSeg X{xi[1], xi[2], xi[3], xi[4]};
        for (int j = 0; j < n; ++j) {
            const double* yj = ty + j * kTab;
            const double e = combine_k<KIND>(xp, yj[0], value, eps_low, blocks, table);
            const AxisSeg Y{yj[1], yj[2], yj[3], yj[4]};
            const K9 k = ksub(X, Y);
            // out.m += e * K  (element.hpp:45; Mat4 operator* computes K*e)
            a[0] = a[0] + k.k00 * e;
            a[1] = a[1] + k.k11 * e;
            a[2] = a[2] + k.k22 * e;
            a[3] = a[3] + k.k33 * e;
            a[4] = a[4] + k.k01 * e;
            a[5] = a[5] + k.k23 * e;
            a[6] = a[6] + k.k02 * e;
            a[7] = a[7] + k.k13 * e;
            a[8] = a[8] + k.k03 * e;
        }
    }
    k9_expand(a, out16);
}

template <int KIND>
__device__ __forceinline__ void integrate_fast_tab(const double* __restrict__ tx,
                                                   const double* __restrict__ ty, int n,
                                                   double value, double eps_low, int blocks,
                                                   const double* table, double* out16) {
    double U0 = 0, U1 = 0, U2 = 0, V0 = 0, V1 = 0, V2 = 0;
    for (int i = 0; i < n; ++i) {
        const double* xi = tx + i * kTab;
        const double xp = xi[0];
        double s0 = 0, s1 = 0, s2 = 0, t = 0;
        for (int j = 0; j < n; ++j) {
            const double* yj = ty + j * kTab;
            double e;
            if constexpr (KIND == LZB_FIELD_THETA || KIND == LZB_FIELD_SINUSOID)
                e = __fma_rn(xp, yj[0], 1.0);
            else
                e = combine_k<KIND>(xp, yj[0], value, eps_low, blocks, table);
            t = __fma_rn(e, yj[1], t);
            s0 = __fma_rn(e, yj[2], s0);
            s1 = __fma_rn(e, yj[3], s1);
            s2 = __fma_rn(e, yj[4], s2);
        }
        U0 = __fma_rn(xi[1], s0, U0);
        U1 = __fma_rn(xi[1], s1, U1);
        U2 = __fma_rn(xi[1], s2, U2);
        V0 = __fma_rn(xi[2], t, V0);
        V1 = __fma_rn(xi[3], t, V1);
        V2 = __fma_rn(xi[4], t, V2);
    }
    // same sign pattern as ksub with A_k = U_k, B_k = V_k
    double a[9];
    a[0] = U0 + V0;
    a[1] = U0 + V2;
    a[2] = U2 + V0;
    a[3] = U2 + V2;
    a[4] = V1 - U0;
    a[5] = V1 - U2;
    a[6] = U1 - V0;
    a[7] = U1 - V2;
    a[8] = -(U1 + V1);
    k9_expand(a, out16);
}

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

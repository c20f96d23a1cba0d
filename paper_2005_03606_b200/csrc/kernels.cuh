// kernels.cuh — declarations shared between the .cu translation units.
#pragma once

#include <future>
#include <vector>

#include "device.cuh"
#include "engine.hpp"
#include "integrate.cuh"

namespace lzb {

// First statement of EVERY kernel of liblzb.so (tests/test_abi_host.py checks
// it): LZB_LAUNCH may launch any kernel with programmatic dependent launch
// while a cycle body is captured, and griddepcontrol.wait is what makes the
// kernel wait for its predecessor's completion and memory (a no-op without a
// programmatic predecessor).
__device__ __forceinline__ void lzb_pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Constant tables uploaded once per device (make_ctx): K_unit = the reference
// reference_subcell_stiffness(0,1,0,1) and the geometric transfer block.
// (liblzb.so has a single device translation unit, lzb_unity.cu.)
__constant__ double c_kunit[16];
__constant__ double c_geo[64];

void upload_constants();

// Per-n integration tables (integrate.cuh), rebuilt on demand.
struct HostParts {  // host-libm field parts of one (level, n): x and y tables
    int n = 0, N = 0;
    std::vector<double> x, y;
};
struct TableSet {
    DevBuf<double> fx, fy, seg, ktab, cxp, cyp;
    int n = 0, N = 0;
    int reserve_n = 64;  // capacity (samples per axis) allocated at the first build
    int centre_N = 0;    // level whose centre parts are uploaded
    // the next rung's host tables, computed on a host thread while the GPU
    // integrates the current rung (a p ladder knows its next n)
    std::future<HostParts> ahead;
    void build(const lzb_field& f, int N, double h, int n, cudaStream_t s);
    void prefetch(const lzb_field& f, int N, double h, int n);
    IntTables view() const { return IntTables{fx.p, fy.p, seg.p, ktab.p, cxp.p, cyp.p, n}; }
};
// Host-libm field parts of the N cells' n samples per axis (k_field_parts
// arithmetic) and their upload to device arrays on stream s.
void host_field_parts(const lzb_field& f, int N, double h, int n, int axis, double* out);
void upload_field_parts(const lzb_field& f, int N, double h, int n, double* dx, double* dy, cudaStream_t s);
template <typename K>
void set_smem(K kernel, size_t bytes);
void host_kunit(double* out16);
void host_geo(double* out64);

// Galerkin RAP in the reference loop order (transfer.cpp:81-93,182-200).
__device__ inline void patch_operator_dev(const double* ch, double* A) {
    for (int i = 0; i < 256; ++i) A[i] = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            const double* K = ch + 16 * (i * 3 + j);
            int ids[4];
            for (int c = 0; c < 4; ++c) ids[c] = (j + cdy(c)) * 4 + (i + cdx(c));
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b) A[ids[a] * 16 + ids[b]] += K[a * 4 + b];
        }
}

__device__ inline void galerkin_from_A(const double* A, const double* P, double* out) {
    double T[64];
    for (int i = 0; i < 64; ++i) T[i] = 0.0;
    for (int r = 0; r < 16; ++r)
        for (int k = 0; k < 16; ++k) {
            double a = A[r * 16 + k];
            if (a == 0.0) continue;
            for (int c = 0; c < 4; ++c) T[r * 4 + c] += a * P[k * 4 + c];
        }
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) {
            double v = 0.0;
            for (int k = 0; k < 16; ++k) v += P[k * 4 + r] * T[k * 4 + c];
            out[r * 4 + c] = v;
        }
}

// BoxMG operator-dependent prolongation (transfer.cpp:95-180). Returns
// fallback rows.
__device__ int boxmg_from_A(const double* A, double* P);

}  // namespace lzb

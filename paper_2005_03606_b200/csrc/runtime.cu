// runtime.cu — context, error state, constants and the batched primitive
// entry points (element / codec / transfer) of the C-ABI.
//
// Compiled as part of lzb_unity.cu (one device translation unit, -fmad=false).
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <cmath>
#include <mutex>
#include <thread>
#include <vector>

#include "engine.hpp"
#include "kernels.cuh"

namespace lzb {

std::atomic<uint64_t> g_launches{0};
thread_local bool g_pdl = false;
static thread_local std::string t_last_error;

void set_last_error(const std::string& msg) { t_last_error = msg; }

void host_kunit(double* out) {
    // reference_subcell_stiffness(0,1,0,1) (element.cpp:34-37), same operand order
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            double dXi = cdx(i) ? 1.0 : -1.0, dXj = cdx(j) ? 1.0 : -1.0;
            double dYi = cdy(i) ? 1.0 : -1.0, dYj = cdy(j) ? 1.0 : -1.0;
            out[i * 4 + j] = dXi * dXj * (1.0 - 0.0) * seg_int(cdy(i), cdy(j), 0.0, 1.0) +
                             dYi * dYj * (1.0 - 0.0) * seg_int(cdx(i), cdx(j), 0.0, 1.0);
        }
}

void host_geo(double* out) {
    for (int L = 0; L < 16; ++L)
        for (int c = 0; c < 4; ++c) out[L * 4 + c] = geo_weight(L, c);
}

void upload_constants() {
    double k[16], g[64];
    host_kunit(k);
    host_geo(g);
    LZB_CUDA(cudaMemcpyToSymbol(c_kunit, k, sizeof k));
    LZB_CUDA(cudaMemcpyToSymbol(c_geo, g, sizeof g));
}

lzb_ctx* make_ctx(int device) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        throw Error(LZB_ERR_CUDA, "no CUDA device available (this library has no CPU fallback)");
    if (device < 0 || device >= count) throw Error(LZB_ERR_INVALID, "device index out of range");
    LZB_CUDA(cudaSetDevice(device));
    auto* c = new lzb_ctx;
    c->device = device;
    LZB_CUDA(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device));
    int lo = 0, hi = 0;
    LZB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    // solve stream high priority, assembly stream low priority
    LZB_CUDA(cudaStreamCreateWithPriority(&c->solve, cudaStreamNonBlocking, hi));
    LZB_CUDA(cudaStreamCreateWithPriority(&c->assembly, cudaStreamNonBlocking, lo));
    c->err.alloc(1);
    LZB_CUDA(cudaMemset(c->err.p, 0, sizeof(int)));
    upload_constants();
    return c;
}

void destroy_ctx(lzb_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    release_comm(c);
    if (c->solve) cudaStreamDestroy(c->solve);
    if (c->assembly) cudaStreamDestroy(c->assembly);
    delete c;
}

void check_device_flag(lzb_ctx* c, cudaStream_t s) {
    int flag = 0;
    LZB_CUDA(cudaMemcpyAsync(&flag, c->err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    LZB_CUDA(cudaStreamSynchronize(s));
    if (flag) {
        LZB_CUDA(cudaMemsetAsync(c->err.p, 0, sizeof(int), s));
        LZB_CUDA(cudaStreamSynchronize(s));
        throw Error(LZB_ERR_PROTOCOL, "cannot encode non-finite operator entry");
    }
}

// ------------------------------------------------------------ tables
__global__ void k_field_parts(lzb_field f, int N, double h, int n, int axis, double* out) {
    lzb_pdl_enter();
    int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= static_cast<int64_t>(N) * n) return;
    int c = static_cast<int>(t / n), i = static_cast<int>(t % n);
    double inv = 1.0 / n;
    double x0 = c * h;                       // cell_box, element.hpp:29-32
    double x = x0 + (i + 0.5) * inv * h;     // element.hpp:44
    out[t] = axis == 0 ? field_xpart(f, x) : field_ypart(f, x);
}

__global__ void k_seg_table(int n, double* seg) {
    lzb_pdl_enter();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    AxisSeg s = axis_seg(i, 1.0 / n);
    seg[4 * i + 0] = s.len;
    seg[4 * i + 1] = s.s0;
    seg[4 * i + 2] = s.s1;
    seg[4 * i + 3] = s.s2;
}

__global__ void k_ksub_table(int n, double* ktab) {
    lzb_pdl_enter();
    int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= static_cast<int64_t>(n) * n) return;
    int i = static_cast<int>(t / n), j = static_cast<int>(t % n);
    double inv = 1.0 / n;
    K9 k = ksub(axis_seg(i, inv), axis_seg(j, inv));  // element.cpp:19-32, reference order
    double* o = ktab + t * kKs;
    o[0] = k.k00; o[1] = k.k11; o[2] = k.k22; o[3] = k.k33; o[4] = k.k01;
    o[5] = k.k23; o[6] = k.k02; o[7] = k.k13; o[8] = k.k03; o[9] = 0.0;
}

void host_field_parts(const lzb_field& f, int N, double h, int n, int axis, double* out) {
    // the same arithmetic as k_field_parts (cell_box element.hpp:29-32, the
    // sample element.hpp:44), the transcendentals from the host libm; large
    // tables (the upper rungs of the p ladder) are cut over a few host threads
    const double inv = 1.0 / n;
    auto rows = [&](int c0, int c1) {
        for (int c = c0; c < c1; ++c) {
            const double x0 = c * h;
            for (int i = 0; i < n; ++i) {
                const double x = x0 + (i + 0.5) * inv * h;
                out[static_cast<int64_t>(c) * n + i] = axis == 0 ? field_xpart(f, x) : field_ypart(f, x);
            }
        }
    };
    const int64_t total = static_cast<int64_t>(N) * n;
    const unsigned hw = std::thread::hardware_concurrency();
    const int nt = static_cast<int>(std::min<int64_t>({8, hw ? hw : 1, total / 2048}));
    if (nt <= 1) {
        rows(0, N);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
        th.emplace_back(rows, static_cast<int>(static_cast<int64_t>(N) * t / nt),
                        static_cast<int>(static_cast<int64_t>(N) * (t + 1) / nt));
    for (auto& t : th) t.join();
}

void upload_field_parts(const lzb_field& f, int N, double h, int n, double* dx, double* dy, cudaStream_t s) {
    std::vector<double> hx(static_cast<size_t>(N) * n), hy(static_cast<size_t>(N) * n);
    host_field_parts(f, N, h, n, 0, hx.data());
    host_field_parts(f, N, h, n, 1, hy.data());
    // pageable source: the call returns once the bytes are staged
    LZB_CUDA(cudaMemcpyAsync(dx, hx.data(), hx.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    LZB_CUDA(cudaMemcpyAsync(dy, hy.data(), hy.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    LZB_CUDA(cudaStreamSynchronize(s));
}

void TableSet::build(const lzb_field& f, int N_, double h, int n_, cudaStream_t s) {
    // capacity for the whole ladder at once (reserve_n: the grid's n_max, at
    // least 64): a p doubling run rebuilds the tables at every rung, and each
    // regrowth would cost a stream synchronisation and a cudaMalloc / cudaFree
    const int ncap = std::max(n_, reserve_n);
    const size_t nf = static_cast<size_t>(N_) * ncap;
    if (fx.n < nf) {
        LZB_CUDA(cudaStreamSynchronize(s));
        fx.alloc(nf);
        fy.alloc(nf);
    }
    if (seg.n < static_cast<size_t>(kSeg) * ncap) {
        LZB_CUDA(cudaStreamSynchronize(s));
        seg.alloc(static_cast<size_t>(kSeg) * ncap);
    }
    if (ktab.n < static_cast<size_t>(ncap) * ncap * kKs) {
        LZB_CUDA(cudaStreamSynchronize(s));
        ktab.alloc(static_cast<size_t>(ncap) * ncap * kKs);
    }
    if (cxp.n < static_cast<size_t>(N_)) {
        LZB_CUDA(cudaStreamSynchronize(s));
        cxp.alloc(N_);
        cyp.alloc(N_);
        centre_N = 0;
    }
    // cell-centre parts: the n = 1 sample, x0 + ((0+0.5)*1.0)*h (element.hpp:44),
    // once per level (field and level are fixed per TableSet owner);
    // sample parts at n -- host libm (see field_xpart)
    if (centre_N != N_) {
        upload_field_parts(f, N_, h, 1, cxp.p, cyp.p, s);
        centre_N = N_;
    }
    HostParts hp;
    if (ahead.valid()) hp = ahead.get();
    if (hp.n != n_ || hp.N != N_) {
        hp.x.resize(static_cast<size_t>(N_) * n_);
        hp.y.resize(static_cast<size_t>(N_) * n_);
        host_field_parts(f, N_, h, n_, 0, hp.x.data());
        host_field_parts(f, N_, h, n_, 1, hp.y.data());
    }
    // pageable source: the calls return once the bytes are staged
    LZB_CUDA(cudaMemcpyAsync(fx.p, hp.x.data(), hp.x.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    LZB_CUDA(cudaMemcpyAsync(fy.p, hp.y.data(), hp.y.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    LZB_CUDA(cudaStreamSynchronize(s));
    LZB_LAUNCH(k_seg_table, blocks_for(n_, 128), 128, 0, s, n_, seg.p);
    LZB_LAUNCH(k_ksub_table, blocks_for(static_cast<int64_t>(n_) * n_, 256), 256, 0, s, n_, ktab.p);
    n = n_;
    N = N_;
}

void TableSet::prefetch(const lzb_field& f, int N_, double h, int n_) {
    if (ahead.valid()) ahead.get();  // a stale request (never more than one in flight)
    const lzb_field fc = f;
    ahead = std::async(std::launch::async, [fc, N_, h, n_] {
        HostParts hp;
        hp.n = n_;
        hp.N = N_;
        hp.x.resize(static_cast<size_t>(N_) * n_);
        hp.y.resize(static_cast<size_t>(N_) * n_);
        host_field_parts(fc, N_, h, n_, 0, hp.x.data());
        host_field_parts(fc, N_, h, n_, 1, hp.y.data());
        return hp;
    });
}

// Arbitrary CellBox per cell: axis parts recomputed per sample (the
// reference's exact arithmetic); the per-cell compatibility API.
__global__ void k_integrate_boxes(lzb_field f, int64_t ncells, const double* __restrict__ x0,
                                  const double* __restrict__ y0, const double* __restrict__ hh,
                                  const int32_t* __restrict__ nn, double* __restrict__ out,
                                  int fast) {
    lzb_pdl_enter();
    int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (c >= ncells) return;
    integrate_cell(f, x0[c], y0[c], hh[c], nn[c], fast, out + 16 * c);
}

// Whole regular level at one n.
template <int KIND, bool FAST>
__global__ void __launch_bounds__(kIntThreads, 2) k_integrate_level(lzb_field f, int N, IntTables T,
                                                                    double* __restrict__ out) {
    lzb_pdl_enter();
    extern __shared__ double sm[];
    stage_common(sm, f, T);
    const int64_t ncell = static_cast<int64_t>(N) * N;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * blockDim.x * kCPT;
    const int64_t c1 = (c0 + static_cast<int64_t>(blockDim.x) * kCPT < ncell
                            ? c0 + static_cast<int64_t>(blockDim.x) * kCPT : ncell) - 1;
    const int row_lo = static_cast<int>(c0 / N), rows = static_cast<int>(c1 / N) - row_lo + 1;
    const double* s_fy = stage_rows(sm, T, row_lo, rows);
    bool act[kCPT];
    int64_t cc[kCPT];
    const double* fxc[kCPT];
    const double* fyc[kCPT];
#pragma unroll
    for (int q = 0; q < kCPT; ++q) {
        const int64_t c = c0 + threadIdx.x + q * blockDim.x;
        act[q] = c < ncell;
        cc[q] = act[q] ? c : c0;
        const int cx = static_cast<int>(cc[q] % N), cy = static_cast<int>(cc[q] / N);
        fxc[q] = T.fx + static_cast<int64_t>(cx) * T.n;
        fyc[q] = s_fy ? s_fy + static_cast<int64_t>(cy - row_lo) * T.n : T.fy + static_cast<int64_t>(cy) * T.n;
    }
    double m[kCPT][16];
    integrate_block<KIND, FAST, kCPT>(act, f, T, fxc, fyc, sm, m);
#pragma unroll
    for (int q = 0; q < kCPT; ++q) {
        if (!act[q]) continue;
        double2* o = reinterpret_cast<double2*>(out + 16 * cc[q]);
        for (int k = 0; k < 8; ++k) o[k] = make_double2(m[q][2 * k], m[q][2 * k + 1]);
    }
}

template <typename K>
void set_smem(K kernel, size_t bytes) {
    if (bytes > 48 * 1024)
        LZB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(bytes)));
}

template <int KIND, bool FAST>
void launch_level_k(const lzb_field& f, int N, const IntTables& T, double* out, cudaStream_t s) {
    size_t smem = int_smem_bytes(T.n);
    set_smem(k_integrate_level<KIND, FAST>, smem);
    LZB_LAUNCH((k_integrate_level<KIND, FAST>), blocks_for(static_cast<int64_t>(N) * N, kIntThreads * kCPT),
               kIntThreads, smem, s, f, N, T, out);
}

template <bool FAST>
void launch_integrate_level(const lzb_field& f, int N, const IntTables& T, double* out,
                            cudaStream_t s) {
    switch (f.kind) {
        case LZB_FIELD_THETA: launch_level_k<LZB_FIELD_THETA, FAST>(f, N, T, out, s); break;
        case LZB_FIELD_QUADRANT: launch_level_k<LZB_FIELD_QUADRANT, FAST>(f, N, T, out, s); break;
        case LZB_FIELD_CHECKER: launch_level_k<LZB_FIELD_CHECKER, FAST>(f, N, T, out, s); break;
        case LZB_FIELD_SINUSOID: launch_level_k<LZB_FIELD_SINUSOID, FAST>(f, N, T, out, s); break;
        default: launch_level_k<LZB_FIELD_CONSTANT, FAST>(f, N, T, out, s); break;
    }
}

// FP64 peak probe: 8 independent DFMA chains per thread, one CTA per SM slot.
__global__ void k_fp64_probe(int iters, double seed, double* sink) {
    lzb_pdl_enter();
    double a[8];
    for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x * 1e-9 + k;
    const double m = 0.999999999, c = 1e-9;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = __fma_rn(a[k], m, c);
    double s = 0;
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.678) sink[0] = s;  // keep the chains alive
}

// ------------------------------------------------------------------ codec
__global__ void k_encode(int64_t count, const double* __restrict__ x, int p3, uint8_t* out,
                         int* err) {
    lzb_pdl_enter();
    int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= count) return;
    if (!encode_value(x[i], p3, out + i * p3)) atomicExch(err, 1);
}
__global__ void k_decode(int64_t count, const uint8_t* in, int p3, double* out) {
    lzb_pdl_enter();
    int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= count) return;
    out[i] = decode_value(in + i * p3, p3);
}
__global__ void k_choose(int64_t nrec, int entries, const double* __restrict__ v, double delta,
                         int32_t* out, int* err) {
    lzb_pdl_enter();
    int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (r >= nrec) return;
    int p = choose_precision(v + r * entries, entries, delta);
    if (p < 0) {
        atomicExch(err, 1);
        p = 8;
    }
    out[r] = p;
}

// --------------------------------------------------------------- transfer
__device__ int boxmg_from_A(const double* A, double* P) {
    int fallback = 0;
    for (int i = 0; i < 64; ++i) P[i] = 0.0;
    const int corner_lattice[4] = {0, 3, 12, 15};
    for (int c = 0; c < 4; ++c) P[corner_lattice[c] * 4 + c] = 1.0;
    const int e_ids[4][2] = {{1, 2}, {13, 14}, {4, 8}, {7, 11}};
    const int e_a[4] = {0, 2, 0, 1}, e_b[4] = {1, 3, 2, 3};
    const bool e_x[4] = {true, true, false, false};
    for (int e = 0; e < 4; ++e) {
        double w[2], c[2], s[2];
        bool ok = true;
        for (int k = 0; k < 2; ++k) {
            int L = e_ids[e][k], lx = L % 4, ly = L / 4;
            double S[3][3];
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    int nx = lx + dx, ny = ly + dy;
                    S[dy + 1][dx + 1] = (nx >= 0 && nx < 4 && ny >= 0 && ny < 4)
                                            ? A[L * 16 + ny * 4 + nx] : 0.0;
                }
            if (e_x[e]) {
                w[k] = S[0][0] + S[1][0] + S[2][0];
                c[k] = S[0][1] + S[1][1] + S[2][1];
                s[k] = S[0][2] + S[1][2] + S[2][2];
            } else {
                w[k] = S[0][0] + S[0][1] + S[0][2];
                c[k] = S[1][0] + S[1][1] + S[1][2];
                s[k] = S[2][0] + S[2][1] + S[2][2];
            }
            if (!(c[k] > 0.0)) ok = false;
        }
        double det = c[0] * c[1] - s[0] * w[1];
        if (!ok || fabs(det) < 1e-300) {
            for (int k = 0; k < 2; ++k) {
                for (int cc = 0; cc < 4; ++cc) P[e_ids[e][k] * 4 + cc] = c_geo[e_ids[e][k] * 4 + cc];
                ++fallback;
            }
            continue;
        }
        P[e_ids[e][0] * 4 + e_a[e]] = (-w[0] * c[1]) / det;
        P[e_ids[e][1] * 4 + e_a[e]] = (w[0] * w[1]) / det;
        P[e_ids[e][0] * 4 + e_b[e]] = (s[0] * s[1]) / det;
        P[e_ids[e][1] * 4 + e_b[e]] = (-c[0] * s[1]) / det;
    }
    const int interior[4] = {5, 6, 9, 10};
    double M[4][4], rhs[4][4];
    for (int r = 0; r < 4; ++r)
        for (int q = 0; q < 4; ++q) {
            M[r][q] = A[interior[r] * 16 + interior[q]];
            rhs[r][q] = 0.0;
        }
    for (int r = 0; r < 4; ++r)
        for (int L = 0; L < 16; ++L) {
            if (L == 5 || L == 6 || L == 9 || L == 10) continue;
            double a = A[interior[r] * 16 + L];
            if (a == 0.0) continue;
            for (int cc = 0; cc < 4; ++cc) rhs[r][cc] -= a * P[L * 4 + cc];
        }
    // solve4 (transfer.cpp:41-72)
    int perm[4] = {0, 1, 2, 3};
    bool solved = true;
    for (int k = 0; k < 4 && solved; ++k) {
        int p = k;
        for (int r = k + 1; r < 4; ++r)
            if (fabs(M[perm[r]][k]) > fabs(M[perm[p]][k])) p = r;
        int t = perm[k]; perm[k] = perm[p]; perm[p] = t;
        double piv = M[perm[k]][k];
        if (fabs(piv) < 1e-14) { solved = false; break; }
        for (int r = k + 1; r < 4; ++r) {
            double f = M[perm[r]][k] / piv;
            if (f == 0.0) continue;
            for (int c = k; c < 4; ++c) M[perm[r]][c] -= f * M[perm[k]][c];
            for (int c = 0; c < 4; ++c) rhs[perm[r]][c] -= f * rhs[perm[k]][c];
        }
    }
    if (solved) {
        for (int k = 3; k >= 0; --k)
            for (int c = 0; c < 4; ++c) {
                double v = rhs[perm[k]][c];
                for (int j = k + 1; j < 4; ++j) v -= M[perm[k]][j] * rhs[perm[j]][c];
                rhs[perm[k]][c] = v / M[perm[k]][k];
            }
        for (int r = 0; r < 4; ++r)
            for (int cc = 0; cc < 4; ++cc) P[interior[r] * 4 + cc] = rhs[perm[r]][cc];
    } else {
        for (int r = 0; r < 4; ++r) {
            for (int cc = 0; cc < 4; ++cc) P[interior[r] * 4 + cc] = c_geo[interior[r] * 4 + cc];
            ++fallback;
        }
    }
    return fallback;
}

__global__ void k_galerkin_batch(int64_t np, const double* __restrict__ ch,
                                 const double* __restrict__ P, double* __restrict__ out) {
    lzb_pdl_enter();
    int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= np) return;
    double A[256], Pl[64];
    patch_operator_dev(ch + 144 * i, A);
    for (int k = 0; k < 64; ++k) Pl[k] = P ? P[64 * i + k] : c_geo[k];
    galerkin_from_A(A, Pl, out + 16 * i);
}

__global__ void k_boxmg_batch(int64_t np, const double* __restrict__ ch, double* __restrict__ P,
                              int32_t* fb) {
    lzb_pdl_enter();
    int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= np) return;
    double A[256];
    patch_operator_dev(ch + 144 * i, A);
    int f = boxmg_from_A(A, P + 64 * i);
    if (fb) fb[i] = f;
}

}  // namespace lzb

// ======================================================================= C-ABI
using namespace lzb;

namespace {
template <typename T>
DevBuf<T> upload(const T* host, size_t n, cudaStream_t s) {
    DevBuf<T> d(n);
    if (n) LZB_CUDA(cudaMemcpyAsync(d.p, host, n * sizeof(T), cudaMemcpyHostToDevice, s));
    return d;
}
template <typename T>
void download(T* host, const DevBuf<T>& d, size_t n, cudaStream_t s) {
    if (n) LZB_CUDA(cudaMemcpyAsync(host, d.p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
}
}  // namespace

extern "C" {

const char* lzb_last_error(void) { return lzb::t_last_error.c_str(); }
int lzb_version(void) { return 1; }
uint64_t lzb_launch_count(void) { return lzb::g_launches.load(); }

int lzb_ctx_create(int device, lzb_ctx** out) {
    return guarded([&] { *out = make_ctx(device); });
}
void lzb_ctx_destroy(lzb_ctx* ctx) { destroy_ctx(ctx); }
int lzb_ctx_synchronize(lzb_ctx* ctx) {
    return guarded([&] {
        LZB_CUDA(cudaStreamSynchronize(ctx->solve));
        LZB_CUDA(cudaStreamSynchronize(ctx->assembly));
    });
}
void* lzb_ctx_solve_stream(lzb_ctx* ctx) { return ctx->solve; }
void* lzb_ctx_assembly_stream(lzb_ctx* ctx) { return ctx->assembly; }

void lzb_field_checkerboard(lzb_field* f, uint64_t seed, int blocks) {
    std::memset(f, 0, sizeof *f);
    f->kind = LZB_FIELD_CHECKER;
    f->blocks = blocks;
    f->value = 1.0;
    auto mix = [](uint64_t z) {  // splitmix64, problem.cpp:43-48
        z += 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    };
    for (int i = 0; i < blocks; ++i)
        for (int j = 0; j < blocks; ++j) {
            double u = static_cast<double>(mix(seed ^ static_cast<uint64_t>(blocks * i + j)) >> 11) *
                       0x1.0p-53;
            f->table[i * blocks + j] = std::pow(10.0, -2.0 + 4.0 * u);
        }
}

double lzb_field_eval_host(const lzb_field* f, double x, double y) {
    switch (f->kind) {
        case LZB_FIELD_THETA: {
            const double amplitude = 0.3 / 2.0;
            double px = std::exp(-f->theta * x) * std::cos(kPi * f->theta * x);
            double py = std::exp(-f->theta * y) * std::cos(kPi * f->theta * y);
            return 1.0 + amplitude * px * py;
        }
        case LZB_FIELD_QUADRANT: return (x >= kQuadCentre) == (y >= kQuadCentre) ? 1.0 : f->eps_low;
        case LZB_FIELD_CHECKER: {
            int b = f->blocks, bx = static_cast<int>(b * x), by = static_cast<int>(b * y);
            if (bx > b - 1) bx = b - 1;
            if (by > b - 1) by = b - 1;
            return f->table[bx * b + by];
        }
        case LZB_FIELD_SINUSOID:
            return 1.0 + f->amp * std::sin(f->freq * kPi * x) * std::sin(f->freq * kPi * y);
        default: return f->value;
    }
}

int lzb_integrate_elements_dev(lzb_ctx* ctx, const lzb_field* eps, int64_t ncells,
                               const double* x0, const double* y0, const double* h,
                               const int32_t* n, double* out, int integration, void* stream) {
    return guarded([&] {
        (void)ctx;
        if (ncells <= 0) return;
        LZB_LAUNCH(k_integrate_boxes, blocks_for(ncells, 128), 128, 0,
                   static_cast<cudaStream_t>(stream), *eps, ncells, x0, y0, h, n, out,
                   integration == LZB_INTEGRATE_FAST ? 1 : 0);
    });
}

int lzb_integrate_elements(lzb_ctx* ctx, const lzb_field* eps, int64_t ncells, const double* x0,
                           const double* y0, const double* h, const int32_t* n, double* out,
                           int integration) {
    return guarded([&] {
        if (ncells <= 0) return;
        for (int64_t i = 0; i < ncells; ++i)
            if (n[i] < 1) throw Error(LZB_ERR_INVALID, "sub-sample count must be >= 1");
        cudaStream_t s = ctx->solve;
        auto dx = upload(x0, ncells, s), dy = upload(y0, ncells, s), dh = upload(h, ncells, s);
        auto dn = upload(n, ncells, s);
        DevBuf<double> dout(16 * ncells);
        LZB_LAUNCH(k_integrate_boxes, blocks_for(ncells, 128), 128, 0, s, *eps, ncells, dx.p,
                   dy.p, dh.p, dn.p, dout.p, integration == LZB_INTEGRATE_FAST ? 1 : 0);
        download(out, dout, 16 * ncells, s);
        LZB_CUDA(cudaStreamSynchronize(s));
    });
}

int lzb_integrate_level_dev(lzb_ctx* ctx, const lzb_field* eps, int level, int n, double* out,
                            int integration, void* stream) {
    return guarded([&] {
        (void)ctx;
        if (level < 0 || level > 9 || n < 1) throw Error(LZB_ERR_INVALID, "bad level or n");
        int N = 1;
        for (int i = 0; i < level; ++i) N *= 3;
        double h = std::pow(1.0 / 3, level);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        TableSet T;
        T.build(*eps, N, h, n, s);
        if (integration == LZB_INTEGRATE_FAST)
            launch_integrate_level<true>(*eps, N, T.view(), out, s);
        else
            launch_integrate_level<false>(*eps, N, T.view(), out, s);
        LZB_CUDA(cudaStreamSynchronize(s));  // tables are freed on return
    });
}

int lzb_integrate_level(lzb_ctx* ctx, const lzb_field* eps, int level, int n, double* host_out,
                        int integration) {
    return guarded([&] {
        if (level < 0 || level > 9 || n < 1) throw Error(LZB_ERR_INVALID, "bad level or n");
        int N = 1;
        for (int i = 0; i < level; ++i) N *= 3;
        double h = std::pow(1.0 / 3, level);
        cudaStream_t s = ctx->solve;
        DevBuf<double> out(static_cast<size_t>(N) * N * 16);
        TableSet T;
        T.build(*eps, N, h, n, s);
        if (integration == LZB_INTEGRATE_FAST)
            launch_integrate_level<true>(*eps, N, T.view(), out.p, s);
        else
            launch_integrate_level<false>(*eps, N, T.view(), out.p, s);
        LZB_CUDA(cudaMemcpyAsync(host_out, out.p, out.bytes(), cudaMemcpyDeviceToHost, s));
        LZB_CUDA(cudaStreamSynchronize(s));
    });
}

int lzb_probe_fp64_tflops(int device, double* tflops) {
    return guarded([&] {
        LZB_CUDA(cudaSetDevice(device));
        int sms = 0;
        LZB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        DevBuf<double> sink(1);
        const int threads = 512, blocks = sms * 4, iters = 4096;
        cudaEvent_t a, b;
        LZB_CUDA(cudaEventCreate(&a));
        LZB_CUDA(cudaEventCreate(&b));
        LZB_LAUNCH(k_fp64_probe, blocks, threads, 0, 0, iters, 1.0, sink.p);  // warm-up
        double best = 0.0;
        for (int rep = 0; rep < 5; ++rep) {
            LZB_CUDA(cudaEventRecord(a, 0));
            LZB_LAUNCH(k_fp64_probe, blocks, threads, 0, 0, iters, 1.0 + rep, sink.p);
            LZB_CUDA(cudaEventRecord(b, 0));
            LZB_CUDA(cudaEventSynchronize(b));
            float ms = 0;
            LZB_CUDA(cudaEventElapsedTime(&ms, a, b));
            double flops = 2.0 * 8.0 * iters * static_cast<double>(threads) * blocks;
            best = std::max(best, flops / (ms * 1e-3) / 1e12);
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        *tflops = best;
    });
}

int lzb_subcell_stiffness(lzb_ctx* ctx, double a, double b, double c, double d, double* out16) {
    return guarded([&] {
        (void)ctx;
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) {
                double dXi = cdx(i) ? 1.0 : -1.0, dXj = cdx(j) ? 1.0 : -1.0;
                double dYi = cdy(i) ? 1.0 : -1.0, dYj = cdy(j) ? 1.0 : -1.0;
                out16[i * 4 + j] = dXi * dXj * (b - a) * seg_int(cdy(i), cdy(j), c, d) +
                                   dYi * dYj * (d - c) * seg_int(cdx(i), cdx(j), a, b);
            }
    });
}

int lzb_codec_encode(lzb_ctx* ctx, int64_t count, const double* x, int p3, uint8_t* out) {
    return guarded([&] {
        if (p3 < 0 || p3 == 1 || p3 > 8) throw Error(LZB_ERR_INVALID, "p3 must be 0 or 2..8");
        if (count <= 0 || p3 == 0) return;
        cudaStream_t s = ctx->solve;
        auto dx = upload(x, count, s);
        DevBuf<uint8_t> dout(count * p3);
        LZB_LAUNCH(k_encode, blocks_for(count, 256), 256, 0, s, count, dx.p, p3, dout.p, ctx->err.p);
        download(out, dout, count * p3, s);
        check_device_flag(ctx, s);
    });
}

int lzb_codec_decode(lzb_ctx* ctx, int64_t count, const uint8_t* in, int p3, double* out) {
    return guarded([&] {
        if (p3 < 2 || p3 > 8) throw Error(LZB_ERR_INVALID, "p3 must be 2..8");
        if (count <= 0) return;
        cudaStream_t s = ctx->solve;
        auto din = upload(in, count * p3, s);
        DevBuf<double> dout(count);
        LZB_LAUNCH(k_decode, blocks_for(count, 256), 256, 0, s, count, din.p, p3, dout.p);
        download(out, dout, count, s);
        LZB_CUDA(cudaStreamSynchronize(s));
    });
}

int lzb_codec_choose_precision_dev(lzb_ctx* ctx, int64_t nrec, int32_t entries,
                                   const double* values, double delta_max, int32_t* out_p3,
                                   void* stream) {
    return guarded([&] {
        if (nrec <= 0) return;
        LZB_LAUNCH(k_choose, blocks_for(nrec, 128), 128, 0, static_cast<cudaStream_t>(stream),
                   nrec, entries, values, delta_max, out_p3, ctx->err.p);
    });
}

int lzb_codec_choose_precision(lzb_ctx* ctx, int64_t nrec, int32_t entries, const double* values,
                               double delta_max, int32_t* out_p3) {
    return guarded([&] {
        if (nrec <= 0) return;
        cudaStream_t s = ctx->solve;
        auto dv = upload(values, nrec * entries, s);
        DevBuf<int32_t> dout(nrec);
        LZB_LAUNCH(k_choose, blocks_for(nrec, 128), 128, 0, s, nrec, entries, dv.p, delta_max,
                   dout.p, ctx->err.p);
        download(out_p3, dout, nrec, s);
        check_device_flag(ctx, s);
    });
}

uint8_t lzb_pack_header(int32_t p1, int p2, int p3) { return pack_header(p1, p2, p3); }

int lzb_unpack_header(uint8_t h, int* cls, int* p2, int* p3) {
    *cls = (h >> 6) & 0x3;
    *p2 = (h & 0x20) != 0;
    *p3 = h & 0x0f;
    if (*cls == 3 || *p3 == 1 || *p3 > 8) {
        set_last_error("invalid record header byte");
        return LZB_ERR_CORRUPT;
    }
    return LZB_OK;
}

void lzb_geometric_prolongation(double* out64) { host_geo(out64); }

int lzb_galerkin(lzb_ctx* ctx, int64_t np, const double* children, const double* P, double* out) {
    return guarded([&] {
        if (np <= 0) return;
        cudaStream_t s = ctx->solve;
        auto dch = upload(children, np * 144, s);
        DevBuf<double> dP;
        if (P) dP = upload(P, np * 64, s);
        DevBuf<double> dout(np * 16);
        LZB_LAUNCH(k_galerkin_batch, blocks_for(np, 64), 64, 0, s, np, dch.p, P ? dP.p : nullptr,
                   dout.p);
        download(out, dout, np * 16, s);
        LZB_CUDA(cudaStreamSynchronize(s));
    });
}

int lzb_boxmg(lzb_ctx* ctx, int64_t np, const double* children, double* P, int32_t* fallback) {
    return guarded([&] {
        if (np <= 0) return;
        cudaStream_t s = ctx->solve;
        auto dch = upload(children, np * 144, s);
        DevBuf<double> dP(np * 64);
        DevBuf<int32_t> dfb(np);
        LZB_LAUNCH(k_boxmg_batch, blocks_for(np, 64), 64, 0, s, np, dch.p, dP.p, dfb.p);
        download(P, dP, np * 64, s);
        if (fallback) download(fallback, dfb, np, s);
        LZB_CUDA(cudaStreamSynchronize(s));
    });
}

}  // extern "C"

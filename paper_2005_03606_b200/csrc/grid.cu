// grid.cu — the regular-grid engine: Mesh + CellStream + Assembler +
// AdditiveSolver of the reference, resident in HBM, driven by sm_100a kernels.
//
// Layout in HBM (per level l, N = 3^l):
//   vertex fields u, fl, r, rhat, uhat, diag, aux, usnap: (N+1)^2 doubles each,
//     index iy*(N+1)+ix (SoA: one coalesced stream per field);
//   cell operators: 16 doubles per cell (AoS, 128 B = one cache line pair),
//     index cy*N+cx; markers p1 (int32), p2 (u8), p3 (i8), n, epoch;
//   transfer blocks: 64 doubles per refined cell, only for transfer = boxmg
//     (geometric blocks are implicit: decoded P == geometric, stream.cpp:134-151).
//
// Every floating-point accumulation that the reference performs in a fixed
// order (cell-wise scatter over level_cells, patch-wise restriction over owned
// lattice vertices) is re-expressed as a per-vertex gather that visits the
// contributing cells in the reference's creation-rank order, so the solver
// state is bit-identical to the reference (tests/test_gpu_parity.py).
#include <algorithm>
#include <array>
#include <deque>
#include <unordered_map>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>

#include <cub/device/device_scan.cuh>

#include "engine.hpp"
#include "kernels.cuh"

namespace lzb {


namespace {

constexpr int kThreads = 256;
constexpr int kNHist = 4097;      // p1 histogram bins (n < 4096)

// Result block copied to the host once per cycle.
struct Result {
    double norm;
    unsigned long long s[20];
};
enum StatSlot {
    S_HIST = 0,         // 0..8 p3 histogram over leaves
    S_FINE_BYTES = 9,
    S_NSUM = 10,
    S_MAXN = 11,
    S_TOTAL_BYTES = 12,
    S_ZERO_NORM = 13,   // cumulative
    S_MAXDELTA = 14,    // cumulative, bits of a non-negative double
    S_MAXSAMPLES = 15,  // cumulative
    S_PENDING = 16,     // leaves with a task in flight (p2), per cycle
    S_COARSE_ACTIVE = 17,  // the last cycle in which a coarse cell passed its change gate
};

__device__ inline int64_t gtid() { return blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; }

__device__ inline double baseline_entry(int k, double e) { return 0.0 + c_kunit[k] * e; }

__device__ inline double centre_eps(const lzb_field& f, const LevelView& L, int cx, int cy) {
    // integrate_element(box, eps, 1): the sample at x0 + ((0+0.5)*1.0)*h
    // (element.hpp:44), its axis parts evaluated on the host (Level::cex/cey)
    return field_combine(f, L.cex[cx], L.cey[cy]);
}

__device__ inline const double* transfer_of(const LevelView& C, int c) {
    return (C.P && C.has_P[c]) ? C.P + 64 * static_cast<int64_t>(c) : c_geo;
}

__device__ inline void element_or_baseline(const lzb_field& f, const LevelView& L, int cx, int cy,
                                           double* K) {
    int c = cy * L.N + cx;
    if (L.p1[c] != LZB_P1_BOTTOM) {
        const double2* src = reinterpret_cast<const double2*>(L.op + 16 * static_cast<int64_t>(c));
        for (int k = 0; k < 8; ++k) {
            double2 t = src[k];
            K[2 * k] = t.x;
            K[2 * k + 1] = t.y;
        }
    } else {
        double e = L.geo0 ? 1.0 : centre_eps(f, L, cx, cy);
        for (int k = 0; k < 16; ++k) K[k] = baseline_entry(k, e);
    }
}

// Running maxima shared by every publishing thread: read first, and only
// contend for the atomic when the value would raise the maximum (after the
// first few cells almost none do), instead of one serialised atomic per cell.
__device__ inline void atomic_max_u64(unsigned long long* a, unsigned long long v) {
    if (v > *reinterpret_cast<volatile unsigned long long*>(a)) atomicMax(a, v);
}
__device__ inline void atomic_max_double_bits(unsigned long long* a, double v) {  // v >= 0
    atomic_max_u64(a, static_cast<unsigned long long>(__double_as_longlong(v)));
}

// The compressed copy of a published leaf record for the residual
// (plane_width > 0). A slot holds the p3-byte little-endian word of the
// roundtrip value rt = codec::roundtrip(surplus, p3) in a register-friendly
// order (sign | e_hat+128 | top m fraction bits; raw IEEE at p3 = 8; 0 <-> +0):
// the same information as the LZMG bytes (stream.cpp:311-337), rebuilt into
// the double with shifts and masks only.
__device__ __forceinline__ unsigned long long plane_word(double rt, int p3) {
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(rt));
    if (p3 == 8) return u;
    if (rt == 0.0) return 0;
    const int m = 8 * (p3 - 1) - 1;
    const unsigned long long e8 = ((u >> 52) & 0x7ff) - 895;  // e_hat + 128 in [0, 255]
    return ((u >> 63) << (8 * p3 - 1)) | (e8 << m) | ((u & 0xFFFFFFFFFFFFFull) >> (52 - m));
}
__device__ __forceinline__ void store_planes_rt(const LevelView& F, int c, const double* rt, int p3) {
    if (!F.cplanes) return;
    if (p3 > F.cw) {
        F.cp3[c] = 9;  // wider than a slot: the residual reads the FP64 operator
        return;
    }
    uint8_t* base = F.cplanes + static_cast<int64_t>(c) * 16 * F.cw;
    for (int k = 0; k < 16; ++k) put_bytes(base + k * F.cw, plane_word(rt[k], p3), p3);
    F.cp3[c] = static_cast<int8_t>(p3);
}

// CellStream::mark_parent_dirty (stream.cpp:240-245) under ripple: the
// parent's flag of parity (cycle + 1) & 1, taken by the next cycle's walk.
__device__ __forceinline__ void mark_parent(const LevelView& L, int64_t c, uint32_t cycle) {
    if (!L.pdirty) return;
    const int cx = static_cast<int>(c % L.N), cy = static_cast<int>(c / L.N);
    atomicOr(L.pdirty + static_cast<int64_t>(cy / 3) * (L.N / 3) + cx / 3, 1u << ((cycle + 1) & 1u));
}

// CellStream::publish_element (stream.cpp:100-132); caller stores p1.
__device__ inline bool publish_leaf(const LevelView& F, int c, const double* m, int n, double e_c,
                                    double delta_max, uint32_t cycle, unsigned long long* stats) {
    double base[16], sur[16];
    for (int k = 0; k < 16; ++k) {
        base[k] = baseline_entry(k, e_c);
        sur[k] = m[k] - base[k];
    }
    int p3 = F.fixed_p3 ? F.fixed_p3 : choose_precision(sur, 16, delta_max);
    if (p3 < 0) return false;
    double delta = 0.0, rts[16];
    double* op = F.op + 16 * static_cast<int64_t>(c);
    for (int k = 0; k < 16; ++k) {
        double rt;
        if (!roundtrip_fast(sur[k], p3, rt)) return false;
        double err = fabs(rt - sur[k]);
        delta = delta < err ? err : delta;
        op[k] = base[k] + rt;
        rts[k] = rt;
    }
    store_planes_rt(F, c, rts, p3);
    mark_parent(F, c, cycle);
    atomic_max_double_bits(&stats[S_MAXDELTA], delta);
    atomic_max_u64(&stats[S_MAXSAMPLES], static_cast<unsigned long long>(n));
    F.n[c] = n;
    F.epoch[c] = cycle;
    F.chg[c] = cycle + 1;
    F.p3[c] = static_cast<int8_t>(p3);
    return true;
}

// publish_element for a matrix produced by the integration kernels, whose 16
// entries are the 9 k9 values by construction (k9_expand), as are the
// baseline's (0 + K_unit*e): surplus, width choice and roundtrip run on the 9
// distinct values; the stored 16 are their bitwise copies.
// (positions of the 9 distinct values in the 16 entries: compile-time, so m16 stays in registers)

__device__ inline bool publish_leaf_k9(const LevelView& F, int c, const double* m16, int n, double e_c,
                                       double delta_max, uint32_t cycle, unsigned long long* stats) {
    double base9[9], sur9[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        constexpr int kpos[9] = {0, 5, 10, 15, 1, 11, 2, 7, 3};
        const int k = kpos[i];
        base9[i] = baseline_entry(k, e_c);
        sur9[i] = m16[k] - base9[i];
    }
    const int p3 = F.fixed_p3 ? F.fixed_p3 : choose_precision_k9(sur9, delta_max);
    if (p3 < 0) return false;
    double delta = 0.0, dec9[9], rt9[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        double rt;
        if (!roundtrip_fast(sur9[i], p3, rt)) return false;
        const double err = fabs(rt - sur9[i]);
        delta = delta < err ? err : delta;
        dec9[i] = base9[i] + rt;
        rt9[i] = rt;
    }
    double dec[16];
    k9_expand(dec9, dec);
    double2* op = reinterpret_cast<double2*>(F.op + 16 * static_cast<int64_t>(c));
#pragma unroll
    for (int q = 0; q < 8; ++q) op[q] = make_double2(dec[2 * q], dec[2 * q + 1]);
    if (F.cplanes) {
        double rt16[16];
        k9_expand(rt9, rt16);
        store_planes_rt(F, c, rt16, p3);
    }
    mark_parent(F, c, cycle);
    atomic_max_double_bits(&stats[S_MAXDELTA], delta);
    atomic_max_u64(&stats[S_MAXSAMPLES], static_cast<unsigned long long>(n));
    F.n[c] = n;
    F.epoch[c] = cycle;
    F.chg[c] = cycle + 1;
    F.p3[c] = static_cast<int8_t>(p3);
    return true;
}

// -------------------------------------------------------------- assembly
// Order-preserving compaction of the selected leaves (ascending cell index,
// so a block of list entries covers few cell rows): count per block, scan,
// scatter. selector: 0 unconverged, 1 tasks (p2 set, FIFO key <= limit), 2 bottom.
// p2 = 1: a step task (spawn_step_task); p2 = 2: a forced task (spawn_forced),
// listed with snap = kForcedSnap so that no step kernel takes it.
constexpr int32_t kForcedSnap = INT32_MIN;
__device__ inline bool selected(const LevelView& F, int64_t c, int selector, const long long* keys,
                                long long key_limit, int32_t& p1) {
    p1 = F.p1[c];
    if (selector == 0) return p1 != LZB_P1_TOP;
    if (selector == 1) {
        const uint8_t t = F.p2[c];
        if (t == 2) p1 = kForcedSnap;
        return t != 0 && (!keys || keys[c] <= key_limit);  // a task on a top cell still completes
    }
    return p1 == LZB_P1_BOTTOM;
}

constexpr int kCompactThreads = 256;

__global__ void k_compact_count(LevelView F, int selector, const long long* keys, long long key_limit,
                                int* block_counts) {
    lzb_pdl_enter();
    __shared__ int warp_n[kCompactThreads / 32];
    int64_t c = gtid();
    int32_t p1;
    bool take = c < static_cast<int64_t>(F.N) * F.N && selected(F, c, selector, keys, key_limit, p1);
    unsigned mask = __ballot_sync(0xffffffffu, take);
    if ((threadIdx.x & 31) == 0) warp_n[threadIdx.x >> 5] = __popc(mask);
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int w = 0; w < kCompactThreads / 32; ++w) s += warp_n[w];
        block_counts[blockIdx.x] = s;
    }
}

// Exclusive scan of the block counts in one CTA; total into *count.
__global__ void k_compact_scan(int* block_counts, int nblocks, int* count) {
    lzb_pdl_enter();
    __shared__ int carry;
    __shared__ int warp_sum[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nblocks; base += blockDim.x) {
        int i = base + threadIdx.x;
        int v = i < nblocks ? block_counts[i] : 0;
        int x = v;  // inclusive warp scan
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, x, o);
            if ((threadIdx.x & 31) >= o) x += y;
        }
        if ((threadIdx.x & 31) == 31) warp_sum[threadIdx.x >> 5] = x;
        __syncthreads();
        if (threadIdx.x < 32) {
            int w = threadIdx.x < (blockDim.x >> 5) ? warp_sum[threadIdx.x] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, w, o);
                if (threadIdx.x >= o) w += y;
            }
            warp_sum[threadIdx.x] = w;  // inclusive over warps
        }
        __syncthreads();
        int before = (threadIdx.x >> 5) ? warp_sum[(threadIdx.x >> 5) - 1] : 0;
        if (i < nblocks) block_counts[i] = carry + before + x - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += before + x;
        __syncthreads();
    }
    if (threadIdx.x == 0) *count = carry;
}

__global__ void k_compact_scatter(LevelView F, int selector, const long long* keys, long long key_limit,
                                  const int* block_offsets, int32_t* list, int32_t* snap, unsigned* hist) {
    lzb_pdl_enter();
    __shared__ int warp_off[kCompactThreads / 32];
    int64_t c = gtid();
    int32_t p1 = 0;
    bool take = c < static_cast<int64_t>(F.N) * F.N && selected(F, c, selector, keys, key_limit, p1);
    unsigned mask = __ballot_sync(0xffffffffu, take);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) warp_off[w] = __popc(mask);
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = block_offsets[blockIdx.x];
        for (int k = 0; k < kCompactThreads / 32; ++k) {
            int t = warp_off[k];
            warp_off[k] = s;
            s += t;
        }
    }
    __syncthreads();
    int bin = -1;
    if (take) {
        int pos = warp_off[w] + __popc(mask & ((1u << lane) - 1));
        list[pos] = static_cast<int32_t>(c);
        snap[pos] = p1;
        if (p1 != kForcedSnap) bin = p1 == LZB_P1_TOP ? kNHist - 1 : (p1 < kNHist - 1 ? p1 : kNHist - 1);
    }
    // the p1 histogram, one atomic per distinct bin of a warp (on a ladder the
    // whole level sits at one n: per-leaf atomics on one address serialise,
    // 0.35 ms for the 531 k leaves of 729^2)
    const unsigned peers = __match_any_sync(0xffffffffu, bin);
    if (bin >= 0 && lane == __ffs(peers) - 1) atomicAdd(&hist[bin], static_cast<unsigned>(__popc(peers)));
}

// p1 = bottom -> integrate with n = 1, publish, p1 = 1 (assembly.cpp:26-34).
// count_ptr: the count on the device (concurrent batches), else `count`.
__global__ void k_bottom(LevelView F, lzb_field f, const int32_t* list, const int32_t* snap,
                         int count, const int* count_ptr, double delta_max, uint32_t cycle, int clear_p2,
                         unsigned long long* stats, int* err) {
    lzb_pdl_enter();
    int64_t t = gtid();
    if (t >= (count_ptr ? *count_ptr : count) || snap[t] != LZB_P1_BOTTOM) return;
    int c = list[t], cx = c % F.N, cy = c / F.N;
    double e = centre_eps(f, F, cx, cy), m[16];
    for (int k = 0; k < 16; ++k) m[k] = baseline_entry(k, e);
    if (!publish_leaf_k9(F, c, m, 1, e, delta_max, cycle, stats)) atomicExch(err, 1);
    F.p1[c] = 1;
    if (clear_p2) F.p2[c] = 0;
}

// p1 = n -> (n+1)^2 (or (2n)^2) integration, max-norm comparison, keep or
// publish (assembly.cpp:36-59). Fused K1 + K3: integrate, surplus,
// choose_precision, roundtrip, store.
template <int KIND, bool FAST>
// F = live state (old matrix, markers); D = destination of the outcome (== F in
// the deterministic modes; the staging copy for concurrent assembly batches,
// swapped in by k_commit). count is read on the device (no host round trip).
__global__ void __launch_bounds__(kIntThreads, 2) k_step(LevelView F, LevelView D, lzb_field f,
                                                         const int32_t* list, const int32_t* snap,
                                                         const int* count_ptr, int n, int nn,
                                                         int n_cap_top, IntTables T, double term_c,
                                                         double delta_max, uint32_t cycle, int clear_p2,
                                                         unsigned long long* stats, int* err) {
    lzb_pdl_enter();
    extern __shared__ double sm[];
    const int count = *count_ptr;
    const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x * kCPT;
    if (t0 >= count) return;  // uniform per block: no barrier is skipped by part of a block
    bool mine[kCPT];
    int cc[kCPT];
#pragma unroll
    for (int q = 0; q < kCPT; ++q) {
        const int64_t t = t0 + threadIdx.x + q * blockDim.x;
        mine[q] = t < count && snap[t] == n;
        cc[q] = mine[q] ? list[t] : list[t0];
    }
    if (n_cap_top) {  // sampling cap reached: the marker becomes top, nothing integrated
#pragma unroll
        for (int q = 0; q < kCPT; ++q)
            if (mine[q]) {
                D.p1[cc[q]] = LZB_P1_TOP;
                if (clear_p2) F.p2[cc[q]] = 0;
            }
        return;
    }
    stage_common(sm, f, T);
    // the list is in ascending cell order: the block's rows span first..last entry
    const int64_t t1 = (t0 + static_cast<int64_t>(blockDim.x) * kCPT < count
                            ? t0 + static_cast<int64_t>(blockDim.x) * kCPT : count) - 1;
    const int row_lo = list[t0] / F.N, rows = list[t1] / F.N - row_lo + 1;
    const double* s_fy = stage_rows(sm, T, row_lo, rows);
    const double* fxc[kCPT];
    const double* fyc[kCPT];
#pragma unroll
    for (int q = 0; q < kCPT; ++q) {
        const int cx = cc[q] % F.N, cy = cc[q] / F.N;
        fxc[q] = T.fx + static_cast<int64_t>(cx) * nn;
        fyc[q] = s_fy ? s_fy + static_cast<int64_t>(cy - row_lo) * nn : T.fy + static_cast<int64_t>(cy) * nn;
    }
    double fresh[kCPT][16];
    integrate_block<KIND, FAST, kCPT>(mine, f, T, fxc, fyc, sm, fresh);
#pragma unroll
    for (int q = 0; q < kCPT; ++q) {
        if (!mine[q]) continue;
        const int c = cc[q], cx = c % F.N, cy = c / F.N;
        const double* old = F.op + 16 * static_cast<int64_t>(c);
        double denom = 0.0, dmax = 0.0;
        for (int k = 0; k < 16; ++k) {
            double a = fabs(old[k]);
            denom = denom < a ? a : denom;
            double d = fabs(fresh[q][k] - old[k]);
            dmax = dmax < d ? d : dmax;
        }
        double ratio = 0.0;
        if (denom == 0.0) atomicAdd(&stats[S_ZERO_NORM], 1ull);
        else ratio = dmax / denom;
        if (ratio < term_c) {
            D.p1[c] = LZB_P1_TOP;  // keep the old matrix (assembly.cpp:47-53)
        } else {
            const double e_c = combine_k<KIND>(T.cxp[cx], T.cyp[cy], f.value, f.eps_low, f.blocks, sm);
            if (!publish_leaf_k9(D, c, fresh[q], nn, e_c, delta_max, cycle, stats)) atomicExch(err, 1);
            D.p1[c] = nn;
        }
        if (clear_p2) F.p2[c] = 0;
    }
}

// Anarchic request_stencil for non-bottom leaves: spawn if not top and not in
// flight (assembly.cpp:95-106); key = FIFO position (spawn cycle, pre-order).
// Keys: cycle k's forced tasks (spawned at cycle start) precede its step tasks
// (spawned by the assembly pass): 2k and 2k + 1 blocks of leaf_count.
__global__ void k_spawn(LevelView F, uint32_t cycle, long long leaf_count, long long* keys) {
    lzb_pdl_enter();
    int64_t c = gtid();
    if (c >= static_cast<int64_t>(F.N) * F.N) return;
    if (F.p1[c] == LZB_P1_TOP || F.p2[c]) return;
    F.p2[c] = 1;
    if (keys) keys[c] = (2ll * cycle + 1) * leaf_count + crank(F, c % F.N, c / F.N);
}

// run_experiment's on_cycle_start (experiment.cpp:260-270): a forced task for
// every leaf whose roll splitmix64(0x6f4ce1a3 ^ id) * 2^-53 is below the
// fraction, unless a task of the cell is in flight (Assembler::spawn_forced,
// assembly.cpp:138-154). Cell ids are level by level in creation order, so a
// leaf's id is id0 + its creation rank.
__global__ void k_spawn_forced(LevelView F, uint32_t cycle, long long leaf_count, long long* keys,
                               long long id0, double fraction) {
    lzb_pdl_enter();
    int64_t c = gtid();
    if (c >= static_cast<int64_t>(F.N) * F.N) return;
    const long long rank = crank(F, static_cast<int>(c % F.N), static_cast<int>(c / F.N));
    const double roll = static_cast<double>(splitmix64(0x6f4ce1a3ull ^ static_cast<uint64_t>(id0 + rank)) >> 11) *
                        0x1.0p-53;
    if (!(roll < fraction) || F.p2[c]) return;
    F.p2[c] = 2;
    keys[c] = 2ll * cycle * leaf_count + rank;
}

// A forced task's body: integrate_element(box, eps, fixed_n) whose result only
// feeds a sink (workload emulation; the markers are untouched).
__global__ void k_forced_work(LevelView F, lzb_field f, const int32_t* list, const int32_t* snap, int count,
                              int n, double* sink) {
    lzb_pdl_enter();
    int64_t t = gtid();
    if (t >= count || snap[t] != kForcedSnap) return;
    const int c = list[t];
    double m[16];
    integrate_cell(f, (c % F.N) * F.h, (c / F.N) * F.h, F.h, n, 0, m);
    double mx = 0.0;
    for (int k = 0; k < 16; ++k) mx = fmax(mx, fabs(m[k]));
    if (mx == -1.0) sink[0] = mx;  // never taken; keeps the integration live
}

// A rectangle of leaf cells [x0, x0 + w) x [y0, ...): the fixed-p kernels
// walk a linear range of its cells (rect-local index cy' * w + cx'); the
// whole level is {0, N, 0}.
struct CellRect {
    int x0, w, y0;
    __device__ __forceinline__ int cx(int64_t cl) const { return x0 + static_cast<int>(cl % w); }
    __device__ __forceinline__ int cy(int64_t cl) const { return y0 + static_cast<int>(cl / w); }
};

// The integrated (pre-compression) element matrix of a cell, for the parity
// tests of the fused assembly kernels (lzb_grid_assemble_fixed_raw); raw is
// null on every other path.
__device__ __forceinline__ void store_raw(double* out, const double* m) {
#pragma unroll
    for (int k = 0; k < 16; ++k) out[k] = m[k];
}

// Fixed-p assembly: every leaf integrated at n, published, p1 = top.
template <int KIND, bool FAST>
__global__ void __launch_bounds__(kIntThreads, 2) k_fixed(LevelView F, lzb_field f, int n, IntTables T,
                                                          double delta_max, uint32_t cycle,
                                                          unsigned long long* stats, int* err,
                                                          int64_t cbeg, int64_t cend, CellRect R, double* __restrict__ raw) {
    lzb_pdl_enter();
    extern __shared__ double sm[];
    stage_common(sm, f, T);
    const int64_t ncell = cend;  // rect-local cells [cbeg, cend)
    const int64_t c0 = cbeg + static_cast<int64_t>(blockIdx.x) * blockDim.x * kCPT;
    const int64_t c1 = (c0 + static_cast<int64_t>(blockDim.x) * kCPT < ncell
                            ? c0 + static_cast<int64_t>(blockDim.x) * kCPT : ncell) - 1;
    const int row_lo = R.cy(c0), rows = R.cy(c1) - row_lo + 1;
    const double* s_fy = stage_rows(sm, T, row_lo, rows);
    bool mine[kCPT];
    int64_t cc[kCPT];
    const double* fxc[kCPT];
    const double* fyc[kCPT];
#pragma unroll
    for (int q = 0; q < kCPT; ++q) {
        const int64_t c = c0 + threadIdx.x + q * blockDim.x;
        mine[q] = c < ncell;
        const int64_t cl = mine[q] ? c : c0;
        const int cx = R.cx(cl), cy = R.cy(cl);
        cc[q] = static_cast<int64_t>(cy) * F.N + cx;
        fxc[q] = T.fx + static_cast<int64_t>(cx) * n;
        fyc[q] = s_fy ? s_fy + static_cast<int64_t>(cy - row_lo) * n : T.fy + static_cast<int64_t>(cy) * n;
    }
    double m[kCPT][16];
    integrate_block<KIND, FAST, kCPT>(mine, f, T, fxc, fyc, sm, m);
#pragma unroll
    for (int q = 0; q < kCPT; ++q) {
        if (!mine[q]) continue;
        const int cx = static_cast<int>(cc[q] % F.N), cy = static_cast<int>(cc[q] / F.N);
        const double e_c = combine_k<KIND>(T.cxp[cx], T.cyp[cy], f.value, f.eps_low, f.blocks, sm);
        if (raw) store_raw(raw + 16 * cc[q], m[q]);
        if (!publish_leaf_k9(F, static_cast<int>(cc[q]), m[q], n, e_c, delta_max, cycle, stats))
            atomicExch(err, 1);
        F.p1[cc[q]] = LZB_P1_TOP;
    }
}

// Persistent fixed-p assembly: one contiguous cell range per resident block,
// the whole K_sub table and the range's eps rows staged once, then every
// thread strides through its cells kCPT at a time with no barrier.
template <int KIND, bool FAST>
__global__ void __launch_bounds__(kIntThreads, 2) k_fixed_res(LevelView F, lzb_field f, int n, IntTables T,
                                                              double delta_max, uint32_t cycle,
                                                              unsigned long long* stats, int* err,
                                                              int64_t cbeg, int64_t cend, CellRect R, double* __restrict__ raw) {
    lzb_pdl_enter();
    extern __shared__ double sm[];
    stage_common(sm, f, T);
    if (!FAST) {
        const double2* src = reinterpret_cast<const double2*>(T.ktab);
        double2* dst = reinterpret_cast<double2*>(sm + 64 + kSeg * n);
        for (int v = threadIdx.x; v < n * n * kKs / 2; v += blockDim.x) dst[v] = src[v];
    }
    const int64_t total = cend - cbeg;
    const int64_t b0 = cbeg + blockIdx.x * total / gridDim.x;
    const int64_t b1 = cbeg + (blockIdx.x + 1) * total / gridDim.x;
    const int row_lo = R.cy(b0);
    const int rows = b1 > b0 ? R.cy(b1 - 1) - row_lo + 1 : 0;
    double* s_fy = nullptr;
    if (rows > 0 && rows <= kFyRows) {
        s_fy = res_fy_region(sm, n);
        const double* src = T.fy + static_cast<size_t>(row_lo) * n;
        for (int i = threadIdx.x; i < rows * n; i += blockDim.x) s_fy[i] = src[i];
    }
    __syncthreads();
    for (int64_t base = b0 + threadIdx.x; base < b1; base += static_cast<int64_t>(kCPT) * blockDim.x) {
        bool mine[kCPT];
        int64_t cc[kCPT];
        const double* fxc[kCPT];
        const double* fyc[kCPT];
#pragma unroll
        for (int q = 0; q < kCPT; ++q) {
            const int64_t c = base + static_cast<int64_t>(q) * blockDim.x;
            mine[q] = c < b1;
            const int64_t cl = mine[q] ? c : base;
            const int cx = R.cx(cl), cy = R.cy(cl);
            cc[q] = static_cast<int64_t>(cy) * F.N + cx;
            fxc[q] = T.fx + static_cast<int64_t>(cx) * n;
            fyc[q] = s_fy ? s_fy + static_cast<int64_t>(cy - row_lo) * n : T.fy + static_cast<int64_t>(cy) * n;
        }
        double m[kCPT][16];
        integrate_block<KIND, FAST, kCPT, true>(mine, f, T, fxc, fyc, sm, m);
#pragma unroll
        for (int q = 0; q < kCPT; ++q) {
            if (!mine[q]) continue;
            const int cx = static_cast<int>(cc[q] % F.N), cy = static_cast<int>(cc[q] / F.N);
            const double e_c = combine_k<KIND>(T.cxp[cx], T.cyp[cy], f.value, f.eps_low, f.blocks, sm);
            if (raw) store_raw(raw + 16 * cc[q], m[q]);
            if (!publish_leaf_k9(F, static_cast<int>(cc[q]), m[q], n, e_c, delta_max, cycle, stats))
                atomicExch(err, 1);
            F.p1[cc[q]] = LZB_P1_TOP;
        }
    }
}

// recompute_coarse + publish_coarse for the geometric transfer (solver.cpp:59-77,
// transfer.cpp:81-93,182-200, stream.cpp:134-184), register-streaming form:
// T is produced one lattice row k at a time (A[k][m] summed over the children
// that contain both lattice vertices, in the reference's child order, zero
// entries skipped) and out += P[k][.] * T[k][.] accumulates in ascending k,
// which is exactly the reference's summation order — without the 16x16 A.
// Each child entry feeds exactly one A entry, so the 144 child values are read
// once each, straight from the (L1/L2-resident) fine operator array.
constexpr int kCoarseThreads = 128;
// only != null: the coarse_recompute tasks of a throttled ripple batch (cells
// of this level, one launch per dependency generation), run unconditionally
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_geo(LevelView C, LevelView F, lzb_field f,
                                                               double delta_max, const uint32_t* cycle_ptr,
                                                               unsigned long long* stats, int* err,
                                                               const int32_t* only, int nonly) {
    lzb_pdl_enter();
    const uint32_t cycle = *cycle_ptr;  // device-resident: the cycle is replayed as a CUDA graph
    int64_t c = gtid();
    if (only) {
        if (c >= nonly) return;
        c = only[c];
    }
    if (c >= static_cast<int64_t>(C.N) * C.N) return;
    const int cx = static_cast<int>(c % C.N), cy = static_cast<int>(c / C.N);

    // ripple: only the pending coarse_recompute tasks, each consumed
    // (solver.cpp:86-90); policy `always` recomputes every refined cell each
    // cycle (solver.cpp:83-85): recomputing a patch none of whose children
    // changed since the last attempt reproduces the stored result bit for bit
    // and publish_coarse would be a no-op (stream.cpp:153-158), so those
    // patches are skipped
    if (only) {
    } else if (C.pend) {
        if (!C.pend[c]) return;
        C.pend[c] = 0;
    } else {
        const uint32_t seen = C.seen[c];
        if (seen != 0) {
            uint32_t mx = 0;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    const uint32_t v = F.chg[static_cast<int64_t>(3 * cy + j) * F.N + 3 * cx + i];
                    mx = v > mx ? v : mx;
                }
            if (mx < seen) return;
        }
        C.seen[c] = cycle + 1;
        stats[S_COARSE_ACTIVE] = cycle;  // benign race: every writer stores the cycle
    }
    const double* ch[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            int64_t fc = static_cast<int64_t>(3 * cy + j) * F.N + 3 * cx + i;
            if (F.p1[fc] == LZB_P1_BOTTOM) return;  // delayed semantics (solver.cpp:65)
            ch[i * 3 + j] = F.op + 16 * fc;
        }
    double o[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) o[q] = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const int kx = k & 3, ky = k >> 2;
        double T0 = 0.0, T1 = 0.0, T2 = 0.0, T3 = 0.0;
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            const int mx = m & 3, my = m >> 2;
            if (mx - kx > 1 || kx - mx > 1 || my - ky > 1 || ky - my > 1) continue;  // A[k][m] == 0
            double a = 0.0;
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    const int ak = (kx - i) + 2 * (ky - j), am = (mx - i) + 2 * (my - j);
                    if (kx - i < 0 || kx - i > 1 || ky - j < 0 || ky - j > 1) continue;
                    if (mx - i < 0 || mx - i > 1 || my - j < 0 || my - j > 1) continue;
                    a += __ldg(ch[i * 3 + j] + ak * 4 + am);
                }
            if (a == 0.0) continue;  // transfer.cpp:189
            T0 += a * c_geo[m * 4 + 0];
            T1 += a * c_geo[m * 4 + 1];
            T2 += a * c_geo[m * 4 + 2];
            T3 += a * c_geo[m * 4 + 3];
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const double p = c_geo[k * 4 + r];
            o[r * 4 + 0] += p * T0;
            o[r * 4 + 1] += p * T1;
            o[r * 4 + 2] += p * T2;
            o[r * 4 + 3] += p * T3;
        }
    }
    // publish_coarse: one p3 across A-hat and P-hat; P-hat = P - geo = 0 here, so the
    // joint width equals the width of A-hat alone whenever delta_max >= 0.
    const double e_c = centre_eps(f, C, cx, cy);
    double sur[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) sur[k] = o[k] - baseline_entry(k, e_c);
    int p3;
    if (delta_max >= 0.0) {
        p3 = choose_precision(sur, 16, delta_max);
    } else {  // a negative threshold fails the zero P-hat entries at every width 2..7
        bool fin = true;
        for (int k = 0; k < 16; ++k) fin = fin && dev_isfinite(sur[k]);
        p3 = fin ? 8 : -1;
    }
    if (p3 < 0) {
        atomicExch(err, 1);
        return;
    }
    double delta = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        double rt;
        if (!roundtrip_fast(sur[k], p3, rt)) {
            atomicExch(err, 1);
            return;
        }
        double e = fabs(rt - sur[k]);
        delta = delta < e ? e : delta;
        o[k] = baseline_entry(k, e_c) + rt;
    }
    double* op = C.op + 16 * c;
    if (C.p1[c] == LZB_P1_TOP && C.has_P[c]) {
        bool same = true;
#pragma unroll
        for (int k = 0; k < 16; ++k) same = same && (o[k] == op[k]);
        if (same) return;  // epoch stamps track real information flow (stream.cpp:153-158)
    }
    atomic_max_double_bits(&stats[S_MAXDELTA], delta);
    double2* dst = reinterpret_cast<double2*>(op);
#pragma unroll
    for (int q = 0; q < 8; ++q) dst[q] = make_double2(o[2 * q], o[2 * q + 1]);
    C.has_P[c] = 1;
    C.n[c] = 1;
    C.epoch[c] = cycle;
    C.chg[c] = cycle + 1;
    C.p3[c] = static_cast<int8_t>(p3);
    C.p1[c] = LZB_P1_TOP;
    mark_parent(C, c, cycle);
}

// recompute_coarse + publish_coarse with BoxMG transfer (needs the full patch
// operator A for the operator-dependent prolongation, transfer.cpp:95-180).
__global__ void __launch_bounds__(64) k_coarse(LevelView C, LevelView F, lzb_field f, int boxmg,
                                               double delta_max, const uint32_t* cycle_ptr,
                                               unsigned long long* stats, int* err, const int32_t* only,
                                               int nonly) {
    lzb_pdl_enter();
    const uint32_t cycle = *cycle_ptr;
    int64_t c = gtid();
    if (only) {
        if (c >= nonly) return;
        c = only[c];
    }
    if (c >= static_cast<int64_t>(C.N) * C.N) return;
    int cx = static_cast<int>(c % C.N), cy = static_cast<int>(c / C.N);

    // ripple: only the pending coarse_recompute tasks, each consumed
    // (solver.cpp:86-90); policy `always` recomputes every refined cell each
    // cycle (solver.cpp:83-85): recomputing a patch none of whose children
    // changed since the last attempt reproduces the stored result bit for bit
    // and publish_coarse would be a no-op (stream.cpp:153-158), so those
    // patches are skipped
    if (only) {
    } else if (C.pend) {
        if (!C.pend[c]) return;
        C.pend[c] = 0;
    } else {
        const uint32_t seen = C.seen[c];
        if (seen != 0) {
            uint32_t mx = 0;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    const uint32_t v = F.chg[static_cast<int64_t>(3 * cy + j) * F.N + 3 * cx + i];
                    mx = v > mx ? v : mx;
                }
            if (mx < seen) return;
        }
        C.seen[c] = cycle + 1;
        stats[S_COARSE_ACTIVE] = cycle;  // benign race: every writer stores the cycle
    }
    double ch[144];
    for (int lx = 0; lx < 3; ++lx)
        for (int ly = 0; ly < 3; ++ly) {
            int64_t fc = static_cast<int64_t>(3 * cy + ly) * F.N + 3 * cx + lx;
            if (F.p1[fc] == LZB_P1_BOTTOM) return;  // delayed semantics (solver.cpp:65)
            const double* src = F.op + 16 * fc;
            for (int k = 0; k < 16; ++k) ch[(lx * 3 + ly) * 16 + k] = src[k];
        }
    double A[256], P[64], m[16];
    patch_operator_dev(ch, A);
    if (boxmg) boxmg_from_A(A, P);
    else
        for (int k = 0; k < 64; ++k) P[k] = c_geo[k];
    galerkin_from_A(A, P, m);
    // publish_coarse: one p3 across A-hat and P-hat
    double e_c = centre_eps(f, C, cx, cy);
    double joint[80];
    for (int k = 0; k < 16; ++k) joint[k] = m[k] - baseline_entry(k, e_c);
    for (int k = 0; k < 64; ++k) joint[16 + k] = P[k] - c_geo[k];
    int p3 = choose_precision(joint, 80, delta_max);
    if (p3 < 0) {
        atomicExch(err, 1);
        return;
    }
    double delta = 0.0;
    for (int k = 0; k < 80; ++k) {
        double rt;
        if (!roundtrip_fast(joint[k], p3, rt)) { atomicExch(err, 1); return; }
        double e = fabs(rt - joint[k]);
        delta = delta < e ? e : delta;
        if (k < 16) m[k] = baseline_entry(k, e_c) + rt;
        else P[k - 16] = c_geo[k - 16] + rt;
    }
    double* op = C.op + 16 * c;
    if (C.p1[c] == LZB_P1_TOP && C.has_P[c]) {
        bool same = true;
        for (int k = 0; k < 16; ++k) same = same && (m[k] == op[k]);
        const double* cur = C.P ? C.P + 64 * c : c_geo;
        for (int k = 0; k < 64; ++k) same = same && (P[k] == cur[k]);
        if (same) return;  // epoch stamps track real information flow (stream.cpp:153-158)
    }
    atomic_max_double_bits(&stats[S_MAXDELTA], delta);
    for (int k = 0; k < 16; ++k) op[k] = m[k];
    if (C.P)
        for (int k = 0; k < 64; ++k) C.P[64 * c + k] = P[k];
    C.has_P[c] = 1;
    C.n[c] = 1;
    C.epoch[c] = cycle;
    C.chg[c] = cycle + 1;
    C.p3[c] = static_cast<int8_t>(p3);
    C.p1[c] = LZB_P1_TOP;
    mark_parent(C, c, cycle);
}

// ------------------------------------------------------------------ cycle
// Vertex kernels run on a 2D grid: x = column block, y = vertex row (no
// integer division for coordinates).
__device__ inline bool vertex_xy(const LevelView& L, int& ix, int& iy, int64_t& vi) {
    ix = blockIdx.x * blockDim.x + threadIdx.x;
    iy = blockIdx.y + L.row0;
    if (ix > L.N) return false;
    vi = static_cast<int64_t>(iy) * (L.N + 1) + ix;
    return true;
}
// The same for a linear vertex index of a whole level (the fused small-level
// kernels: one block walks every vertex of a level).
template <bool LIN>
__device__ __forceinline__ bool vertex_at(int64_t lin, const LevelView& L, int& ix, int& iy, int64_t& vi) {
    if (!LIN) return vertex_xy(L, ix, iy, vi);
    const int NV = L.N + 1;
    if (lin >= static_cast<int64_t>(NV) * NV) return false;
    iy = static_cast<int>(lin / NV);
    ix = static_cast<int>(lin - static_cast<int64_t>(iy) * NV);
    vi = lin;
    return true;
}
__device__ inline bool boundary(int N, int ix, int iy) {
    return ix == 0 || iy == 0 || ix == N || iy == N;
}

// Cells adjacent to vertex (ix,iy) sorted by creation rank; row = the
// vertex's corner index in that cell.
struct Adj {
    int n;
    int cx[4], cy[4], row[4];
};
// Creation rank is strictly increasing in cx (fixed cy) and in cy (fixed cx),
// so the lower-left cell comes first and the upper-right last; only the
// lower-right / upper-left pair needs a rank comparison.
__device__ inline Adj adjacent_cells(const LevelView& L, int ix, int iy) {
    Adj a;
    a.n = 0;
    auto add = [&](int cx, int cy, int row) {
        if (cx < 0 || cy < 0 || cx >= L.N || cy >= L.N) return;
        a.cx[a.n] = cx;
        a.cy[a.n] = cy;
        a.row[a.n] = row;
        ++a.n;
    };
    add(ix - 1, iy - 1, 3);  // the vertex is that cell's NE corner
    const bool both = ix >= 1 && ix < L.N && iy >= 1 && iy < L.N;
    if (!both || crank(L, ix, iy - 1) < crank(L, ix - 1, iy)) {
        add(ix, iy - 1, 2);
        add(ix - 1, iy, 1);
    } else {
        add(ix - 1, iy, 1);
        add(ix, iy - 1, 2);
    }
    add(ix, iy, 0);
    return a;
}

// init_level_rhs on the leaf level (solver.cpp:99-118): fl = sum over
// adjacent leaves of w * f(v) (identical terms, so order-free).
__global__ void k_init_rhs(LevelView F, lzb_rhs rhs, double w) {
    lzb_pdl_enter();
    int ix, iy;
    int64_t vi;
    if (!vertex_xy(F, ix, iy, vi)) return;
    int adj = 0;
    for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
            int cx = ix - dx, cy = iy - dy;
            adj += (cx >= 0 && cy >= 0 && cx < F.N && cy < F.N);
        }
    // rsin[i] = sin(pi * (i / 3^l)) from the host libm (Grid constructor)
    double fv = rhs.kind == LZB_RHS_SINPROD ? rhs.value * F.rsin[ix] * F.rsin[iy] : rhs.value;
    double term = w * fv, fl = 0.0;
    for (int k = 0; k < adj; ++k) fl += term;
    F.v[LZB_V_FL][vi] = fl;
}

// compute_uhat (solver.cpp:120-143): P u_c at fine vertex (fx, fy).
__device__ __forceinline__ double uhat_interp(const LevelView& C, int fx, int fy) {
    int px, py;
    owner_patch(C, fx, fy, px, py);
    const double* P = transfer_of(C, py * C.N + px);
    int L = (fy - 3 * py) * 4 + (fx - 3 * px);
    double interp = 0.0;
    for (int k = 0; k < 4; ++k)
        interp += P[L * 4 + k] * C.v[LZB_V_U][(py + cdy(k)) * (C.N + 1) + px + cdx(k)];
    return interp;
}
template <bool LIN>
__device__ __forceinline__ void k_uhat_body(int64_t lin, LevelView F, LevelView C, int has_coarse) {
    int fx, fy;
    int64_t vi;
    if (!vertex_at<LIN>(lin, F, fx, fy, vi)) return;
    double u = F.v[LZB_V_U][vi];
    if (!has_coarse) {
        F.v[LZB_V_UHAT][vi] = u;
        return;
    }
    F.v[LZB_V_UHAT][vi] = u - uhat_interp(C, fx, fy);
}
// The grid kernel takes two adjacent vertices per thread: N = 3^l is odd, so
// a row holds an even number of vertices, (2t, 2t+1) never straddles a row
// and is 16-byte aligned (the planes are cudaMalloc'd), so u is read and u-hat
// written as one 128-bit access each. Per vertex the arithmetic is the body's.
__global__ void k_uhat(LevelView F, LevelView C, int has_coarse) {
    lzb_pdl_enter();
    const int fx = 2 * static_cast<int>(blockIdx.x * blockDim.x + threadIdx.x);
    const int fy = blockIdx.y + F.row0;
    if (fx > F.N) return;
    const int64_t vi = static_cast<int64_t>(fy) * (F.N + 1) + fx;
    const double2 u = *reinterpret_cast<const double2*>(F.v[LZB_V_U] + vi);
    double2 out = u;
    if (has_coarse) {
        out.x = u.x - uhat_interp(C, fx, fy);
        out.y = u.y - uhat_interp(C, fx + 1, fy);
    }
    *reinterpret_cast<double2*>(F.v[LZB_V_UHAT] + vi) = out;
}

// residual_pass cell mat-vec, as a gather (solver.cpp:149-175).
//
// The four adjacent cells sit at fixed positions q = b*2 + a, cell
// (ix-1+a, iy-1+b), the vertex being its corner row (1-a) + 2(1-b). Every
// load (four 32-B operator rows, p1, the 3x3 u / uhat neighbourhood) is
// issued up front, independent of the creation-rank order, which only picks
// the accumulation order of positions 1 and 2 afterwards.
template <bool LIN>
__device__ __forceinline__ void k_residual_body(int64_t lin, LevelView F, lzb_field f) {
    int ix, iy;
    int64_t vi;
    if (!vertex_at<LIN>(lin, F, ix, iy, vi)) return;
    const int N = F.N, NV = N + 1;
    bool has[4];
    has[0] = ix >= 1 && iy >= 1;
    has[1] = ix < N && iy >= 1;
    has[2] = ix >= 1 && iy < N;
    has[3] = ix < N && iy < N;
    double2 k01[4], k23[4];
    int32_t p1[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int a = q & 1, b = q >> 1, row = (1 - a) + 2 * (1 - b);
        const int cx = has[q] ? ix - 1 + a : 0, cy = has[q] ? iy - 1 + b : 0;
        const int64_t c = static_cast<int64_t>(cy) * N + cx;
        const double2* src = reinterpret_cast<const double2*>(F.op + 16 * c + 4 * row);
        k01[q] = __ldcs(src);
        k23[q] = __ldcs(src + 1);
        p1[q] = F.p1[c];
    }
    double uu[3][3], uh[3][3];
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
            const int x = min(max(ix - 1 + dx, 0), N), y = min(max(iy - 1 + dy, 0), N);
            const int64_t cv = static_cast<int64_t>(y) * NV + x;
            uu[dy][dx] = F.v[LZB_V_U][cv];
            uh[dy][dx] = F.v[LZB_V_UHAT][cv];
        }
    const double fl = F.v[LZB_V_FL][vi];
    // creation-rank order: position 0 first, 3 last; 1 before 2 unless the rank says otherwise
    const bool both = has[0] && has[3];
    const bool swap12 = both && !(crank(F, ix, iy - 1) < crank(F, ix - 1, iy));
    double au[4], auh[4], kd[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int a = q & 1, b = q >> 1, row = (1 - a) + 2 * (1 - b);
        double Kr[4] = {k01[q].x, k01[q].y, k23[q].x, k23[q].y};
        if (has[q] && p1[q] == LZB_P1_BOTTOM) {
            const double e = F.geo0 ? 1.0 : centre_eps(f, F, ix - 1 + a, iy - 1 + b);
            for (int col = 0; col < 4; ++col) Kr[col] = baseline_entry(row * 4 + col, e);
        }
        double s = 0.0, sh = 0.0;
#pragma unroll
        for (int col = 0; col < 4; ++col) {
            const int dy = b + cdy(col), dx = a + cdx(col);
            s += Kr[col] * uu[dy][dx];
            sh += Kr[col] * uh[dy][dx];
        }
        au[q] = s;
        auh[q] = sh;
        kd[q] = Kr[row];
    }
    // accumulate in creation-rank order (positions 1 and 2 possibly swapped)
    const double a1 = swap12 ? au[2] : au[1], a2 = swap12 ? au[1] : au[2];
    const double h1 = swap12 ? auh[2] : auh[1], h2 = swap12 ? auh[1] : auh[2];
    const double d1 = swap12 ? kd[2] : kd[1], d2 = swap12 ? kd[1] : kd[2];
    const bool e1 = swap12 ? has[2] : has[1], e2 = swap12 ? has[1] : has[2];
    double r = fl, rh = fl, dg = 0.0;
    if (has[0]) { r -= au[0]; rh -= auh[0]; dg += kd[0]; }
    if (e1) { r -= a1; rh -= h1; dg += d1; }
    if (e2) { r -= a2; rh -= h2; dg += d2; }
    if (has[3]) { r -= au[3]; rh -= auh[3]; dg += kd[3]; }
    if (boundary(N, ix, iy)) {
        r = 0.0;
        rh = 0.0;
    }
    F.v[LZB_V_R][vi] = r;
    F.v[LZB_V_RHAT][vi] = rh;
    F.v[LZB_V_DIAG][vi] = dg;
}
__global__ void __launch_bounds__(kThreads) k_residual(LevelView F, lzb_field f) {
    lzb_pdl_enter();
    k_residual_body<false>(0, F, f);
}

// ---- residual on the compressed leaf records (plane_width = W > 0)
// Bytes [k*W, k*W + W) of a 4W-byte slot row held as W little-endian words.
template <int W>
__device__ __forceinline__ unsigned long long slot_bytes(const uint32_t* w, int k) {
    unsigned long long r = 0;
#pragma unroll
    for (int j = 0; j < W; ++j) {
        const int b = k * W + j;
        r |= static_cast<unsigned long long>((w[b >> 2] >> (8 * (b & 3))) & 0xffu) << (8 * j);
    }
    return r;
}

// The roundtrip value from a plane word (the inverse of plane_word), with
// the per-row constants of width p3 precomputed.
struct PlaneDec {
    int p3, m, sh_sign;
    unsigned long long fmask;
    __device__ __forceinline__ explicit PlaneDec(int p) : p3(p) {
        m = 8 * (p - 1) - 1;
        sh_sign = 8 * p - 1;
        fmask = (1ull << (m > 0 ? m : 0)) - 1;
    }
    __device__ __forceinline__ double operator()(unsigned long long w) const {
        if (p3 == 8) return __longlong_as_double(static_cast<long long>(w));
        if (p3 == 0 || w == 0) return 0.0;
        const unsigned long long sign = (w >> sh_sign) & 1, e8 = (w >> m) & 0xff;
        return __longlong_as_double(static_cast<long long>((sign << 63) | ((e8 + 895) << 52) |
                                                           ((w & fmask) << (52 - m))));
    }
};

// k_residual reading, per adjacent cell, the vertex's row of the compressed
// record (4 slots of W bytes) instead of the 32-B FP64 row: the entry is
// rebuilt as baseline(ε centre) + roundtrip value, which is the stored
// operator bit for bit (publish stores baseline + roundtrip(surplus),
// stream.cpp:100-111).
template <int W>
__global__ void __launch_bounds__(kThreads, 3) k_residual_comp(LevelView F, lzb_field f, const double* __restrict__ cxp,
                                                            const double* __restrict__ cyp) {
    lzb_pdl_enter();
    int ix, iy;
    int64_t vi;
    if (!vertex_xy(F, ix, iy, vi)) return;
    const int N = F.N, NV = N + 1;
    bool has[4];
    has[0] = ix >= 1 && iy >= 1;
    has[1] = ix < N && iy >= 1;
    has[2] = ix >= 1 && iy < N;
    has[3] = ix < N && iy < N;
    uint32_t rw[4][W];
    int cp[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int a = q & 1, b = q >> 1, row = (1 - a) + 2 * (1 - b);
        const int cx = has[q] ? ix - 1 + a : 0, cy = has[q] ? iy - 1 + b : 0;
        const int64_t c = static_cast<int64_t>(cy) * N + cx;
        const uint32_t* src = reinterpret_cast<const uint32_t*>(F.cplanes + (c * 16 + row * 4) * W);
#pragma unroll
        for (int j = 0; j < W; ++j) rw[q][j] = __ldcs(src + j);
        cp[q] = F.cp3[c];  // -1: bottom (baseline), 0..W: slots, > W: FP64 row
    }
    // centre field parts of the two cell columns / rows around the vertex
    const double ex0 = cxp[max(ix - 1, 0)], ex1 = cxp[min(ix, N - 1)];
    const double ey0 = cyp[max(iy - 1, 0)], ey1 = cyp[min(iy, N - 1)];
    double uu[3][3], uh[3][3];
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
            const int x = min(max(ix - 1 + dx, 0), N), y = min(max(iy - 1 + dy, 0), N);
            const int64_t cv = static_cast<int64_t>(y) * NV + x;
            uu[dy][dx] = F.v[LZB_V_U][cv];
            uh[dy][dx] = F.v[LZB_V_UHAT][cv];
        }
    const double fl = F.v[LZB_V_FL][vi];
    const bool both = has[0] && has[3];
    const bool swap12 = both && !(crank(F, ix, iy - 1) < crank(F, ix - 1, iy));
    double au[4], auh[4], kd[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int a = q & 1, b = q >> 1, row = (1 - a) + 2 * (1 - b);
        const double e = field_combine(f, a ? ex1 : ex0, b ? ey1 : ey0);  // ε(centre), the n = 1 sample
        double Kr[4];
        if (cp[q] < 0) {
            for (int col = 0; col < 4; ++col) Kr[col] = baseline_entry(row * 4 + col, F.geo0 ? 1.0 : e);
        } else if (cp[q] <= W) {
            const PlaneDec dec(cp[q]);
#pragma unroll
            for (int col = 0; col < 4; ++col)
                Kr[col] = baseline_entry(row * 4 + col, e) + dec(slot_bytes<W>(rw[q], col));
        } else {  // record wider than a slot: the FP64 row
            const int cx = has[q] ? ix - 1 + a : 0, cy = has[q] ? iy - 1 + b : 0;
            const double* src = F.op + 16 * (static_cast<int64_t>(cy) * N + cx) + 4 * row;
            for (int col = 0; col < 4; ++col) Kr[col] = src[col];
        }
        double s = 0.0, sh = 0.0;
#pragma unroll
        for (int col = 0; col < 4; ++col) {
            const int dy = b + cdy(col), dx = a + cdx(col);
            s += Kr[col] * uu[dy][dx];
            sh += Kr[col] * uh[dy][dx];
        }
        au[q] = s;
        auh[q] = sh;
        kd[q] = Kr[row];
    }
    const double a1 = swap12 ? au[2] : au[1], a2 = swap12 ? au[1] : au[2];
    const double h1 = swap12 ? auh[2] : auh[1], h2 = swap12 ? auh[1] : auh[2];
    const double d1 = swap12 ? kd[2] : kd[1], d2 = swap12 ? kd[1] : kd[2];
    const bool e1 = swap12 ? has[2] : has[1], e2 = swap12 ? has[1] : has[2];
    double r = fl, rh = fl, dg = 0.0;
    if (has[0]) { r -= au[0]; rh -= auh[0]; dg += kd[0]; }
    if (e1) { r -= a1; rh -= h1; dg += d1; }
    if (e2) { r -= a2; rh -= h2; dg += d2; }
    if (has[3]) { r -= au[3]; rh -= auh[3]; dg += kd[3]; }
    if (boundary(N, ix, iy)) {
        r = 0.0;
        rh = 0.0;
    }
    F.v[LZB_V_R][vi] = r;
    F.v[LZB_V_RHAT][vi] = rh;
    F.v[LZB_V_DIAG][vi] = dg;
}

// The same residual, cell-centric and staged (the leaf level's kernel; the
// per-vertex gather above stays as LZB_PLAIN_COMP=1). The gather read each
// cell's record four times, a slot row per adjacent vertex, with ~36 global
// load instructions per vertex: it ran at 94 % of the L1 / LSU throughput and
// no faster than the FP64 rows it replaces. Here a block owns a tile of
// 32 x 8 cells (31 x 7 vertices, the 3D residual's tiling): each cell thread
// reads its own record once (16 W contiguous bytes, coalesced across the
// warp), rebuilds the 16 entries as baseline + roundtrip, forms its four row
// products K_row . u and K_row . u-hat from the staged vertex tile -- the
// per-vertex kernel's products, entry by entry in its order -- and stages them
// with the diagonal entries; the vertex threads then subtract them in the
// creation-rank order. Same bits (tests/test_gpu_grid.py
// test_compressed_residual_bit_identical).
// PlaneDec(W) with the width at compile time (a record coded at the planes'
// own width, the common case: every record of a fixed-width sweep): for words
// of at most 4 bytes the exponent | fraction bits are contiguous, one shift
// puts them at bit 20 of the high half and one add rebiases the exponent
// (grid3.cu's SrcComp<W>::dec).
template <int W>
__device__ __forceinline__ double plane_dec_fixed(unsigned long long w64) {
    if constexpr (W == 8) {
        return __longlong_as_double(static_cast<long long>(w64));
    } else if constexpr (W <= 4) {
        const uint32_t w = static_cast<uint32_t>(w64);
        constexpr int m = 8 * (W - 1) - 1;
        constexpr uint32_t body = (1u << (8 * W - 1)) - 1u;
        const uint32_t mag = w & body;
        const uint32_t hi = (m > 20 ? mag >> (m - 20) : mag << (20 - m)) + (895u << 20);
        const uint32_t sg = (w >> (8 * W - 1)) << 31;
        const uint32_t lo = m > 20 ? w << (52 - m) : 0u;
        return w == 0 ? 0.0 : __hiloint2double(static_cast<int>(hi | sg), static_cast<int>(lo));
    } else {
        return PlaneDec(W)(w64);
    }
}
constexpr int kCsX = 32, kCsY = 8;
template <int W>
__global__ void __launch_bounds__(kCsX * kCsY) k_residual_comp_st(LevelView F, lzb_field f,
                                                                  const double* __restrict__ cxp,
                                                                  const double* __restrict__ cyp, int r0, int r1) {
    lzb_pdl_enter();
    __shared__ double s_u[2][kCsY + 1][kCsX + 1];
    __shared__ double s_a[3][4][kCsX * kCsY];  // K_row . u, K_row . u-hat, K[row][row] per cell
    const int t = threadIdx.x, tx = t % kCsX, ty = t / kCsX;
    const int N = F.N, NV = N + 1;
    const int X0 = blockIdx.x * (kCsX - 1), Y0 = r0 + blockIdx.y * (kCsY - 1);  // the tile's first vertex
    for (int k = t; k < (kCsY + 1) * (kCsX + 1); k += kCsX * kCsY) {
        const int j = k / (kCsX + 1), i = k - j * (kCsX + 1);
        const int x = min(max(X0 - 1 + i, 0), N), y = min(max(Y0 - 1 + j, 0), N);
        const int64_t cv = static_cast<int64_t>(y) * NV + x;
        s_u[0][j][i] = F.v[LZB_V_U][cv];
        s_u[1][j][i] = F.v[LZB_V_UHAT][cv];
    }
    const int cx = X0 - 1 + tx, cy = Y0 - 1 + ty;
    const bool cell = cx >= 0 && cy >= 0 && cx < N && cy < N;
    uint32_t rw[4 * W];  // the record: 16 slots of W bytes
    int cp = -1;
    double e = 0.0;
    if (cell) {
        const int64_t c = static_cast<int64_t>(cy) * N + cx;
        const uint4* src = reinterpret_cast<const uint4*>(F.cplanes + c * 16 * W);
#pragma unroll
        for (int j = 0; j < W; ++j) {
            const uint4 v = __ldcs(src + j);
            rw[4 * j] = v.x;
            rw[4 * j + 1] = v.y;
            rw[4 * j + 2] = v.z;
            rw[4 * j + 3] = v.w;
        }
        cp = F.cp3[c];  // -1: bottom (baseline), 0..W: slots, > W: FP64 row
        e = field_combine(f, cxp[cx], cyp[cy]);  // eps(centre), the n = 1 sample
    }
    __syncthreads();
    if (cell) {
#pragma unroll
        for (int row = 0; row < 4; ++row) {
            double Kr[4];
            if (cp < 0) {
                for (int col = 0; col < 4; ++col) Kr[col] = baseline_entry(row * 4 + col, F.geo0 ? 1.0 : e);
            } else if (cp == W) {  // coded at the planes' width: compile-time decode
#pragma unroll
                for (int col = 0; col < 4; ++col)
                    Kr[col] = baseline_entry(row * 4 + col, e) + plane_dec_fixed<W>(slot_bytes<W>(rw + row * W, col));
            } else if (cp <= W) {
                const PlaneDec dec(cp);
#pragma unroll
                for (int col = 0; col < 4; ++col)
                    Kr[col] = baseline_entry(row * 4 + col, e) + dec(slot_bytes<W>(rw + row * W, col));
            } else {  // record wider than a slot: the FP64 row
                const double* src = F.op + 16 * (static_cast<int64_t>(cy) * N + cx) + 4 * row;
                for (int col = 0; col < 4; ++col) Kr[col] = src[col];
            }
            double su = 0.0, sh = 0.0;
#pragma unroll
            for (int col = 0; col < 4; ++col) {
                su += Kr[col] * s_u[0][ty + cdy(col)][tx + cdx(col)];
                sh += Kr[col] * s_u[1][ty + cdy(col)][tx + cdx(col)];
            }
            s_a[0][row][t] = su;
            s_a[1][row][t] = sh;
            s_a[2][row][t] = Kr[row];
        }
    }
    __syncthreads();
    const int ix = X0 + tx, iy = Y0 + ty;
    if (tx >= kCsX - 1 || ty >= kCsY - 1 || ix > N || iy >= r1 || iy > N) return;
    const int64_t vi = static_cast<int64_t>(iy) * NV + ix;
    bool has[4];
    has[0] = ix >= 1 && iy >= 1;
    has[1] = ix < N && iy >= 1;
    has[2] = ix >= 1 && iy < N;
    has[3] = ix < N && iy < N;
    double au[4], auh[4], kd[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int a = q & 1, b = q >> 1, row = (1 - a) + 2 * (1 - b);
        const int ci = (ty + b) * kCsX + tx + a;  // the cell (ix - 1 + a, iy - 1 + b) in the tile
        au[q] = s_a[0][row][ci];
        auh[q] = s_a[1][row][ci];
        kd[q] = s_a[2][row][ci];
    }
    const double fl = F.v[LZB_V_FL][vi];
    const bool both = has[0] && has[3];
    const bool swap12 = both && !(crank(F, ix, iy - 1) < crank(F, ix - 1, iy));
    const double a1 = swap12 ? au[2] : au[1], a2 = swap12 ? au[1] : au[2];
    const double h1 = swap12 ? auh[2] : auh[1], h2 = swap12 ? auh[1] : auh[2];
    const double d1 = swap12 ? kd[2] : kd[1], d2 = swap12 ? kd[1] : kd[2];
    const bool e1 = swap12 ? has[2] : has[1], e2 = swap12 ? has[1] : has[2];
    double r = fl, rh = fl, dg = 0.0;
    if (has[0]) { r -= au[0]; rh -= auh[0]; dg += kd[0]; }
    if (e1) { r -= a1; rh -= h1; dg += d1; }
    if (e2) { r -= a2; rh -= h2; dg += d2; }
    if (has[3]) { r -= au[3]; rh -= auh[3]; dg += kd[3]; }
    if (boundary(N, ix, iy)) {
        r = 0.0;
        rh = 0.0;
    }
    F.v[LZB_V_R][vi] = r;
    F.v[LZB_V_RHAT][vi] = rh;
    F.v[LZB_V_DIAG][vi] = dg;
}

// Restriction fl_{l-1} += P^T rhat_l over owned lattice vertices
// (solver.cpp:177-200), gathered per coarse vertex in (cell rank, L) order.
// mode 0: rhs restriction of rhat into fl; mode 1: adaFAC-Jac smoothed
// residual into aux (solver.cpp:250-268).
template <bool LIN>
__device__ __forceinline__ void k_restrict_body(int64_t lin, LevelView F, LevelView C, int mode, double omega) {
    int IX, IY;
    int64_t vi;
    if (!vertex_at<LIN>(lin, C, IX, IY, vi)) return;
    const int NV = F.N + 1;
    Adj a = adjacent_cells(C, IX, IY);
    double acc_v = 0.0;
    for (int q = 0; q < a.n; ++q) {
        int cx = a.cx[q], cy = a.cy[q], k = a.row[q];
        const double* P = transfer_of(C, cy * C.N + cx);
        double acc = 0.0;
        for (int L = 0; L < 16; ++L) {
            int lx = L & 3, ly = L >> 2;
            int fx = 3 * cx + lx, fy = 3 * cy + ly;
            if (!owns_lattice(cx, cy, lx, ly)) continue;
            int64_t fi = static_cast<int64_t>(fy) * NV + fx;
            if (mode == 0) {
                double rh = F.v[LZB_V_RHAT][fi];
                if (rh == 0.0) continue;
                acc_v += P[L * 4 + k] * rh;
            } else {
                if (boundary(F.N, fx, fy)) continue;
                double dg = F.v[LZB_V_DIAG][fi];
                double sres = F.v[LZB_V_R][fi] - (dg != 0.0 ? omega / dg * F.v[LZB_V_AUX][fi] : 0.0);
                acc += P[L * 4 + k] * sres;
            }
        }
        if (mode == 1) acc_v += acc;
    }
    if (mode == 0) C.v[LZB_V_FL][vi] = acc_v;
    else C.v[LZB_V_AUX][vi] = acc_v;
}
__global__ void k_restrict(LevelView F, LevelView C, int mode, double omega) {
    lzb_pdl_enter();
    k_restrict_body<false>(0, F, C, mode, omega);
}

// Residual norm partials (solver.cpp:202-209): fine interior vertices. Block
// b sums rows 1+b, 1+b+G, ... four rows per step (independent loads in
// flight), then a fixed-order tree; k_norm_final adds the kNormBlocks partials.
constexpr int kNormBlocks = 148 * 4;
__global__ void __launch_bounds__(kThreads) k_norm_partial(LevelView F, int y0, int y1, double* partial) {
    lzb_pdl_enter();
    __shared__ double sh[kThreads];
    const int N = F.N;
    const double* r = F.v[LZB_V_R];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    const int G = gridDim.x;
    // interior rows [max(y0,1), min(y1,N))
    const int ylo = max(y0, 1), yhi = min(y1, N);
    for (int iy = ylo + blockIdx.x; iy < yhi; iy += 4 * G) {
        const int64_t b0 = static_cast<int64_t>(iy) * (N + 1);
        const bool h1 = iy + G < yhi, h2 = iy + 2 * G < yhi, h3 = iy + 3 * G < yhi;
        for (int ix = 1 + threadIdx.x; ix < N; ix += blockDim.x) {
            const double a0 = r[b0 + ix];
            const double a1 = h1 ? r[b0 + static_cast<int64_t>(G) * (N + 1) + ix] : 0.0;
            const double a2 = h2 ? r[b0 + static_cast<int64_t>(2 * G) * (N + 1) + ix] : 0.0;
            const double a3 = h3 ? r[b0 + static_cast<int64_t>(3 * G) * (N + 1) + ix] : 0.0;
            s0 += a0 * a0;
            s1 += a1 * a1;
            s2 += a2 * a2;
            s3 += a3 * a3;
        }
    }
    sh[threadIdx.x] = (s0 + s1) + (s2 + s3);
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

constexpr int kNormFinalThreads = 1024;
__global__ void __launch_bounds__(kNormFinalThreads) k_norm_final(const double* partial, int n, Result* res,
                                                                   int squared = 0) {
    lzb_pdl_enter();
    __shared__ double sh[kNormFinalThreads];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += partial[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) res->norm = squared ? sh[0] : sqrt(sh[0]);
}

// compression_stats over leaves + record bytes of refined cells (stream.cpp:268-301).
// Grid-stride: per-thread counters over the cells, then warp reductions and
// one atomic per counter per block.
constexpr int kStatsBlocks = 148 * 4;
__global__ void __launch_bounds__(kThreads) k_stats(LevelView L, int leaf, unsigned long long* s,
                                                    int64_t cbeg = 0, int64_t cend = -1) {
    lzb_pdl_enter();
    __shared__ unsigned long long sh[20];
    if (threadIdx.x < 20) sh[threadIdx.x] = 0;
    __syncthreads();
    const int64_t nc = cend < 0 ? static_cast<int64_t>(L.N) * L.N : cend;
    unsigned long long bytes = 0, nsum = 0;
    unsigned nmax = 0, pend = 0, h[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t c = cbeg + gtid(); c < nc; c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t p1 = L.p1[c];
        const int p3raw = L.p3[c];
        const int p3 = p1 != LZB_P1_BOTTOM ? p3raw : 0;
        bytes += p1 == LZB_P1_BOTTOM ? 1u : 1u + p3 * (leaf ? 16u : 144u);
        if (!leaf && L.pend) pend += L.pend[c] ? 1u : 0u;  // pending coarse_recompute tasks
        if (leaf) {
            const unsigned n = p1 != LZB_P1_BOTTOM ? static_cast<unsigned>(L.n[c]) : 0u;
            nsum += n;
            nmax = max(nmax, n);
            pend += L.p2[c] ? 1u : 0u;
#pragma unroll
            for (int b = 0; b <= 8; ++b) h[b] += p3 == b ? 1u : 0u;
        }
    }
    const unsigned full = 0xffffffffu;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        bytes += __shfl_down_sync(full, bytes, o);
        nsum += __shfl_down_sync(full, nsum, o);
    }
    const bool lead = (threadIdx.x & 31) == 0;
    if (lead && bytes) atomicAdd(&sh[S_TOTAL_BYTES], bytes);
    if (leaf) {
#pragma unroll
        for (int b = 0; b <= 8; ++b) {
            const unsigned cnt = __reduce_add_sync(full, h[b]);
            if (lead && cnt) atomicAdd(&sh[S_HIST + b], static_cast<unsigned long long>(cnt));
        }
        const unsigned wmax = __reduce_max_sync(full, nmax);
        if (lead) {
            if (bytes) atomicAdd(&sh[S_FINE_BYTES], bytes);
            if (nsum) atomicAdd(&sh[S_NSUM], nsum);
            if (wmax) atomicMax(&sh[S_MAXN], static_cast<unsigned long long>(wmax));
        }
    }
    {
        const unsigned wp = __reduce_add_sync(full, pend);
        if (lead && wp) atomicAdd(&sh[S_PENDING], static_cast<unsigned long long>(wp));
    }
    __syncthreads();
    if ((threadIdx.x < 13 || threadIdx.x == S_PENDING) && sh[threadIdx.x]) {
        if (threadIdx.x == S_MAXN) atomic_max_u64(&s[S_MAXN], sh[S_MAXN]);
        else atomicAdd(&s[threadIdx.x], sh[threadIdx.x]);
    }
}

// The walk's take_dirty (stream.cpp:247-250) for every refined cell of a
// level: the flag of the current parity spawns a coarse_recompute task.
__global__ void k_take_dirty(LevelView L, uint32_t cycle) {
    lzb_pdl_enter();
    const int64_t c = gtid();
    if (c >= static_cast<int64_t>(L.N) * L.N) return;
    const uint32_t bit = 1u << (cycle & 1u), d = L.dirty[c];
    if (d & bit) {
        L.dirty[c] = d & ~bit;
        L.pend[c] = 1;
    }
}

__global__ void k_count_p2(LevelView L, unsigned long long* out) {
    lzb_pdl_enter();
    int64_t c = gtid();
    bool on = c < static_cast<int64_t>(L.N) * L.N && L.p2[c];
    unsigned m = __ballot_sync(0xffffffffu, on);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(out, static_cast<unsigned long long>(__popc(m)));
}

// update_pass pieces (solver.cpp:212-313)
template <bool LIN>
__device__ __forceinline__ void k_snap_body(int64_t lin, LevelView L) {
    int64_t vi = (LIN ? lin : gtid());
    if (vi >= static_cast<int64_t>(L.N + 1) * (L.N + 1)) return;
    L.v[LZB_V_USNAP][vi] = L.v[LZB_V_U][vi];
    L.v[LZB_V_AUX][vi] = 0.0;
}
__global__ void k_snap(LevelView L) {
    lzb_pdl_enter();
    k_snap_body<false>(0, L);
}
template <bool LIN>
__device__ __forceinline__ void k_aux_inject_body(int64_t lin, LevelView F, LevelView C) {  // adaFAC-PI: R~ = injection
    int ix, iy;
    int64_t vi;
    if (!vertex_at<LIN>(lin, C, ix, iy, vi)) return;
    C.v[LZB_V_AUX][vi] = F.v[LZB_V_R][static_cast<int64_t>(3 * iy) * (F.N + 1) + 3 * ix];
}
__global__ void k_aux_inject(LevelView F, LevelView C) {
    lzb_pdl_enter();
    k_aux_inject_body<false>(0, F, C);
}
template <bool LIN>
__device__ __forceinline__ void k_aux_Ar_body(int64_t lin, LevelView F, lzb_field f) {  // adaFAC-Jac: aux = A r on level l
    int ix, iy;
    int64_t vi;
    if (!vertex_at<LIN>(lin, F, ix, iy, vi)) return;
    const int NV = F.N + 1;
    Adj a = adjacent_cells(F, ix, iy);
    double aux = 0.0;
    for (int q = 0; q < a.n; ++q) {
        double K[16];
        element_or_baseline(f, F, a.cx[q], a.cy[q], K);
        double ar = 0.0;
        for (int col = 0; col < 4; ++col)
            ar += K[a.row[q] * 4 + col] *
                  F.v[LZB_V_R][static_cast<int64_t>(a.cy[q] + cdy(col)) * NV + a.cx[q] + cdx(col)];
        aux += ar;
    }
    F.v[LZB_V_AUX][vi] = aux;
}
__global__ void k_aux_Ar(LevelView F, lzb_field f) {
    lzb_pdl_enter();
    k_aux_Ar_body<false>(0, F, f);
}
// u_l -= P (omega/diag_c aux_c) on interior fine vertices (solver.cpp:271-297)
template <bool LIN>
__device__ __forceinline__ void k_aux_sub_body(int64_t lin, LevelView F, LevelView C, double omega) {
    int fx, fy, px, py;
    int64_t vi;
    if (!vertex_at<LIN>(lin, F, fx, fy, vi)) return;
    if (boundary(F.N, fx, fy)) return;
    owner_patch(C, fx, fy, px, py);
    const double* P = transfer_of(C, py * C.N + px);
    int L = (fy - 3 * py) * 4 + (fx - 3 * px);
    double p = 0.0;
    for (int k = 0; k < 4; ++k) {
        int cx = px + cdx(k), cy = py + cdy(k);
        int64_t ci = static_cast<int64_t>(cy) * (C.N + 1) + cx;
        double dg = C.v[LZB_V_DIAG][ci];
        double caux = (!boundary(C.N, cx, cy) && dg != 0.0) ? omega / dg * C.v[LZB_V_AUX][ci] : 0.0;
        p += P[L * 4 + k] * caux;
    }
    F.v[LZB_V_U][vi] -= p;
}
__global__ void k_aux_sub(LevelView F, LevelView C, double omega) {
    lzb_pdl_enter();
    k_aux_sub_body<false>(0, F, C, omega);
}
template <bool LIN>
__device__ __forceinline__ void k_jacobi_body(int64_t lin, LevelView F, double damping) {
    int ix, iy;
    int64_t vi;
    if (!vertex_at<LIN>(lin, F, ix, iy, vi)) return;
    if (boundary(F.N, ix, iy)) return;
    double dg = F.v[LZB_V_DIAG][vi];
    if (dg != 0.0) F.v[LZB_V_U][vi] += damping / dg * F.v[LZB_V_R][vi];
}
__global__ void k_jacobi(LevelView F, double damping) {
    lzb_pdl_enter();
    k_jacobi_body<false>(0, F, damping);
}
// prolong_corrections (solver.cpp:315-342)
template <bool LIN>
__device__ __forceinline__ void k_prolong_body(int64_t lin, LevelView F, LevelView C) {
    int fx, fy, px, py;
    int64_t vi;
    if (!vertex_at<LIN>(lin, F, fx, fy, vi)) return;
    if (boundary(F.N, fx, fy)) return;
    owner_patch(C, fx, fy, px, py);
    double delta[4];
    bool any = false;
    for (int k = 0; k < 4; ++k) {
        int64_t ci = static_cast<int64_t>(py + cdy(k)) * (C.N + 1) + px + cdx(k);
        delta[k] = C.v[LZB_V_U][ci] - C.v[LZB_V_USNAP][ci];
        any |= delta[k] != 0.0;
    }
    if (!any) return;
    const double* P = transfer_of(C, py * C.N + px);
    int L = (fy - 3 * py) * 4 + (fx - 3 * px);
    double p = 0.0;
    for (int k = 0; k < 4; ++k) p += P[L * 4 + k] * delta[k];
    F.v[LZB_V_U][vi] += p;
}
// P u_c - P u_c,snap at an interior fine vertex (the body's arithmetic).
__device__ __forceinline__ bool prolong_delta(const LevelView& F, const LevelView& C, int fx, int fy, double& p) {
    if (boundary(F.N, fx, fy)) return false;
    int px, py;
    owner_patch(C, fx, fy, px, py);
    double delta[4];
    bool any = false;
    for (int k = 0; k < 4; ++k) {
        int64_t ci = static_cast<int64_t>(py + cdy(k)) * (C.N + 1) + px + cdx(k);
        delta[k] = C.v[LZB_V_U][ci] - C.v[LZB_V_USNAP][ci];
        any |= delta[k] != 0.0;
    }
    if (!any) return false;
    const double* P = transfer_of(C, py * C.N + px);
    int L = (fy - 3 * py) * 4 + (fx - 3 * px);
    p = 0.0;
    for (int k = 0; k < 4; ++k) p += P[L * 4 + k] * delta[k];
    return true;
}
// Vertex pairs per thread as in k_uhat. u is only written when a correction
// applies, exactly where the body adds (its += stays even when p == 0).
__global__ void k_prolong(LevelView F, LevelView C) {
    lzb_pdl_enter();
    const int fx = 2 * static_cast<int>(blockIdx.x * blockDim.x + threadIdx.x);
    const int fy = blockIdx.y + F.row0;
    if (fx > F.N) return;
    const int64_t vi = static_cast<int64_t>(fy) * (F.N + 1) + fx;
    double px = 0.0, py = 0.0;
    const bool ax = prolong_delta(F, C, fx, fy, px), ay = prolong_delta(F, C, fx + 1, fy, py);
    double2* up = reinterpret_cast<double2*>(F.v[LZB_V_U] + vi);
    if (ax || ay) {
        double2 u = *up;
        if (ax) u.x += px;
        if (ay) u.y += py;
        *up = u;
    }
}
// The leaf level's three updates of one cycle in one pass over u (u is
// touched by nothing else in between): the adaFAC-PI aux correction
// (k_aux_sub, when caux_c is given), the damped Jacobi step (k_jacobi) and the
// prolongated coarse correction (k_prolong), in that order per vertex, so the
// result is bit-identical to the three kernels. Runs after the coarse levels
// are final (prolongation cascade down to level D-1).
// The coarse factor of k_aux_sub, omega/diag_c * aux_c (0 on the boundary
// and where diag_c = 0), once per coarse vertex instead of four times per
// fine vertex; same expression, same bits.
__global__ void k_scale_aux(LevelView C, double omega, double* __restrict__ out) {
    lzb_pdl_enter();
    int cx, cy;
    int64_t ci;
    if (!vertex_xy(C, cx, cy, ci)) return;
    const double cdg = C.v[LZB_V_DIAG][ci];
    out[ci] = (!boundary(C.N, cx, cy) && cdg != 0.0) ? omega / cdg * C.v[LZB_V_AUX][ci] : 0.0;
}

__global__ void k_update_fine(LevelView F, LevelView C, const double* __restrict__ caux_c, double damping) {
    lzb_pdl_enter();
    int fx, fy, px, py;
    int64_t vi;
    if (!vertex_xy(F, fx, fy, vi)) return;
    if (boundary(F.N, fx, fy)) return;
    owner_patch(C, fx, fy, px, py);
    const double* P = transfer_of(C, py * C.N + px);
    const int L = (fy - 3 * py) * 4 + (fx - 3 * px);
    const double dg = F.v[LZB_V_DIAG][vi], r = F.v[LZB_V_R][vi];
    double u = F.v[LZB_V_U][vi];
    double cu[4], cs[4], caux[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t ci = static_cast<int64_t>(py + cdy(k)) * (C.N + 1) + px + cdx(k);
        cu[k] = C.v[LZB_V_U][ci];
        cs[k] = C.v[LZB_V_USNAP][ci];
        caux[k] = caux_c ? caux_c[ci] : 0.0;
    }
    if (caux_c) {  // k_aux_sub
        double p = 0.0;
        for (int k = 0; k < 4; ++k) p += P[L * 4 + k] * caux[k];
        u -= p;
    }
    if (dg != 0.0) u += damping / dg * r;  // k_jacobi
    double delta[4];  // k_prolong
    bool any = false;
    for (int k = 0; k < 4; ++k) {
        delta[k] = cu[k] - cs[k];
        any |= delta[k] != 0.0;
    }
    if (any) {
        double p = 0.0;
        for (int k = 0; k < 4; ++k) p += P[L * 4 + k] * delta[k];
        u += p;
    }
    F.v[LZB_V_U][vi] = u;
}
// inject_solution (mesh.cpp:226-234)
template <bool LIN>
__device__ __forceinline__ void k_inject_body(int64_t lin, LevelView F, LevelView C) {
    int ix, iy;
    int64_t vi;
    if (!vertex_at<LIN>(lin, C, ix, iy, vi)) return;
    C.v[LZB_V_U][vi] = F.v[LZB_V_U][static_cast<int64_t>(3 * iy) * (F.N + 1) + 3 * ix];
}
__global__ void k_inject(LevelView F, LevelView C) {
    lzb_pdl_enter();
    k_inject_body<false>(0, F, C);
}
// init_noise (problem.cpp:50-68), before the injection.
__global__ void k_noise(LevelView L, int level, uint64_t seed, double gval) {
    lzb_pdl_enter();
    int ix, iy;
    int64_t vi;
    if (!vertex_xy(L, ix, iy, vi)) return;
    if (boundary(L.N, ix, iy)) {
        L.v[LZB_V_U][vi] = gval;
        return;
    }
    auto mix = [](uint64_t z) {
        z += 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    };
    uint64_t k = mix(seed ^ mix((static_cast<uint64_t>(level) << 48) ^
                                (static_cast<uint64_t>(static_cast<uint32_t>(ix)) << 24) ^
                                static_cast<uint64_t>(static_cast<uint32_t>(iy))));
    L.v[LZB_V_U][vi] = (4.0 / 3.0) * static_cast<double>(k >> 11) * 0x1.0p-53;
}

// ------------------------------------------------------- stream image (save)
// Pre-order slot of a cell on a regular tree of depth D: slot(child ci of a
// level-(k-1) cell with slot s) = s + 1 + ci * S_k, S_k = sum_{j<=D-k} 9^j,
// ci = lx*3 + ly (mesh.cpp:152-167).
struct SlotTable {
    int64_t subtree[16];
    // slot(l, cx, cy) = l + sx[l][cx] + sy[l][cy]: the base-3 digit sums
    // sum_k 3*dx_k*S_k and sum_k dy_k*S_k of the pre-order slot
    const int64_t* sx[16];
    const int64_t* sy[16];
};

__device__ __forceinline__ int64_t slot_at(const SlotTable& st, int l, int cx, int cy) {
    return l + st.sx[l][cx] + st.sy[l][cy];
}

// -------------------------------------------- slot-ordered stream packing
// The LZMG image lists records in pre-order (stream.cpp:311-337): record
// sizes -> device exclusive scan -> offsets, then k_pack_patches / k_pack_upper fill
// the image.
constexpr int kMaxLevels = 10;
struct AllLevels {
    LevelView L[kMaxLevels];
    SlotTable st;
    int D;
};

__device__ __forceinline__ int record_size(int p1, int p3, bool leaf) {  // stream.cpp:227-237
    return (p1 == LZB_P1_BOTTOM || p3 == 0) ? 1 : 1 + p3 * (leaf ? 16 : 144);
}

// ---- leaf record payload at a compile-time width
// encode_word for normal values with exponent in [-128,127] at width P3 < 8
// (constants folded); other values take the general path.
template <int P3>
__device__ __forceinline__ unsigned long long encode_word_w(double x) {
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(x));
    if (P3 == 8) return u;
    const int e = static_cast<int>((u >> 52) & 0x7ff) - 1023;
    if (e < -128 || e > 127) return encode_word(x, P3);  // zero, subnormal, clamped exponent
    const unsigned long long w = (u & 0x8000000000000000ull) | ((u << 11) & 0x7FFFFFFFFFFFF800ull);
    const unsigned lo = static_cast<unsigned>(w), hi = static_cast<unsigned>(w >> 32);
    const unsigned long long sw = (static_cast<unsigned long long>(__byte_perm(lo, 0, 0x0123)) << 32) |
                                  __byte_perm(hi, 0, 0x0123);
    constexpr int nb = 8 * (P3 - 1);
    return (sw & ((1ull << nb) - 1)) | (static_cast<unsigned long long>(static_cast<uint8_t>(e)) << nb);
}

// The 16 encoded values of a leaf record (value k at bytes [k*P3, (k+1)*P3))
// packed into 4*P3 little-endian words, then written at byte address dst of a
// zeroed shared-memory window: aligned words, the two boundary words merged
// with atomicOr (they may hold a neighbour's bytes).
template <int P3>
__device__ __forceinline__ void put_leaf_payload(uint8_t* dst, const unsigned long long* w16) {
    constexpr int NW = 4 * P3;
    uint32_t out[NW];
#pragma unroll
    for (int j = 0; j < NW; ++j) {
        uint32_t word = 0;
        constexpr int VB = 8 * P3;  // bits per value
#pragma unroll
        for (int k = (32 * j) / VB; k <= (32 * j + 31) / VB && k < 16; ++k) {
            const int sh = VB * k - 32 * j;
            word |= sh >= 0 ? static_cast<uint32_t>(w16[k] << sh) : static_cast<uint32_t>(w16[k] >> (-sh));
        }
        out[j] = word;
    }
    const uintptr_t a = reinterpret_cast<uintptr_t>(dst);
    uint32_t* wp = reinterpret_cast<uint32_t*>(a & ~uintptr_t{3});
    const int s8 = 8 * static_cast<int>(a & 3);
    if (s8 == 0) {
        atomicOr(wp, out[0]);
#pragma unroll
        for (int j = 1; j < NW - 1; ++j) wp[j] = out[j];
        atomicOr(wp + NW - 1, out[NW - 1]);
    } else {
        atomicOr(wp, out[0] << s8);
#pragma unroll
        for (int j = 1; j < NW; ++j) wp[j] = __funnelshift_l(out[j - 1], out[j], s8);
        atomicOr(wp + NW, out[NW - 1] >> (32 - s8));
    }
}

// Encode the 16 surplus values of a leaf at width P3 (9 encodes when the
// record has the k9 symmetry of the integrated operators, else 16).
template <int P3>
__device__ __forceinline__ void leaf_payload(uint8_t* dst, const double* x, bool sym) {
    unsigned long long w[16];
    if (sym) {
        constexpr int kpos[9] = {0, 5, 10, 15, 1, 11, 2, 7, 3};
        unsigned long long w9[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) w9[i] = encode_word_w<P3>(x[kpos[i]]);
        // k9_expand: 0,5,10,15 diagonal; 1=4; 11=14; 2=8; 7=13; 3=12=6=9
        w[0] = w9[0]; w[5] = w9[1]; w[10] = w9[2]; w[15] = w9[3];
        w[1] = w[4] = w9[4];
        w[11] = w[14] = w9[5];
        w[2] = w[8] = w9[6];
        w[7] = w[13] = w9[7];
        w[3] = w[12] = w[6] = w[9] = w9[8];
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) w[k] = encode_word_w<P3>(x[k]);
    }
    put_leaf_payload<P3>(dst, w);
}

// CellStream::save records of level-(D-1) patches with their 9 leaves. In
// pre-order a patch and its leaves are 10 consecutive records (slot sP, then
// sP+1+ci, ci = lx*3+ly), and sibling patches (px, 3q+j), j = 0..2, follow
// one another: one warp packs such a triple, 30 records, one contiguous byte
// range of the image. Lane = record: a leaf lane encodes its own 16 values
// (one encode_word each) into the warp's shared-memory window; the refined
// records (144 values: Â, P̂ and the R̂ copy) are then encoded by the whole
// warp, lane = value; the window leaves in 16-B aligned vector stores. No
// block barriers.
constexpr int kPackWarps = 4;
constexpr int kPatchBytes = 1153 + 9 * 129;  // refined record + 9 leaf records at p3 = 8
constexpr int kPackWindow = (3 * kPatchBytes + 16 + 15) & ~15;

struct PackArgs {
    const double *cxF, *cyF, *cxC, *cyC;  // centre field parts, leaf and patch level
};

__global__ void __launch_bounds__(kPackWarps * 32) k_pack_patches(AllLevels A, lzb_field f, PackArgs T, int per,
                                                                  const int64_t* __restrict__ offsets,
                                                                  uint8_t* __restrict__ out, int* err, int px0,
                                                                  int pxn, int py_base,
                                                                  const int64_t* __restrict__ basep) {
    lzb_pdl_enter();
    __shared__ __align__(16) uint8_t wbuf[kPackWarps][kPackWindow];
    __shared__ double s_geo[64], s_kunit[16];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < 64) s_geo[threadIdx.x] = c_geo[threadIdx.x];
    if (threadIdx.x < 16) s_kunit[threadIdx.x] = c_kunit[threadIdx.x];
    __syncthreads();
    const int D = A.D;
    const LevelView C = A.L[D - 1];
    const LevelView F = A.L[D];
    // 2D grid: x = patch columns (kPackWarps per block), y = groups of `per` sibling patches;
    // patches [px0, px0 + pxn) x [py_base, ...) (a band of level-1 subtrees, or the whole
    // level), offsets relative to *basep when given
    const int px = px0 + blockIdx.x * kPackWarps + warp, py0 = py_base + blockIdx.y * per;
    if (px >= px0 + pxn) return;
    const int64_t obase = basep ? *basep : 0;
    const unsigned full = 0xffffffffu;
    // pre-order slot of patch (px, py0)
    const int64_t s0 = slot_at(A.st, D - 1, px, py0);  // digit tables (L1/L2-resident)
    const int nrec = 10 * per;
    // the patch records' Â entries (lane < 16), loaded with everything else
    double ra[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < 3; ++j)
        if (lane < 16 && j < per) ra[j] = __ldcs(C.op + 16 * (static_cast<int64_t>(py0 + j) * C.N + px) + lane);
    // lane r < nrec: record r of the range = patch r/10, then leaf (r%10)-1
    const int pj = lane / 10, k = lane % 10;
    const bool have = lane < nrec, leaf = have && k > 0;
    int p3 = 0, size = 0, cell = 0;
    int64_t off = 0;
    double e = 0.0;
    uint8_t hdr = 0;
    if (have) {
        int cx = px, cy = py0 + pj, N = C.N;
        const int32_t* p1a = C.p1;
        const int8_t* p3a = C.p3;
        const uint8_t* p2a = C.p2;
        if (leaf) {
            cx = 3 * px + (k - 1) / 3;
            cy = 3 * (py0 + pj) + (k - 1) % 3;
            N = F.N;
            p1a = F.p1;
            p3a = F.p3;
            p2a = F.p2;
        }
        cell = cy * N + cx;
        // independent loads first
        const int32_t p1 = p1a[cell];
        const int p3raw = p3a[cell];
        const uint8_t p2 = p2a[cell];
        off = offsets[s0 + lane] + obase;
        const double ex = leaf ? T.cxF[cx] : T.cxC[cx], ey = leaf ? T.cyF[cy] : T.cyC[cy];
        p3 = p1 != LZB_P1_BOTTOM ? p3raw : 0;
        hdr = pack_header(p1, p2, p3);
        size = record_size(p1, p3, leaf);
        // centre eps = field at the n = 1 sample (tabulated parts; element.hpp:44)
        if (size > 1) e = field_combine(f, ex, ey);
    }
    const int64_t off0 = __shfl_sync(full, off, 0);
    const int rel = static_cast<int>(off - off0);
    const int64_t g0 = 12 + off0;
    const int shift = static_cast<int>(g0 & 15);
    const int bytes = __shfl_sync(full, rel + size, nrec - 1);
    uint8_t* buf = wbuf[warp];
    // zero the window (payload words are OR-merged at record boundaries)
    {
        uint4* z = reinterpret_cast<uint4*>(buf);
        const int nz = (shift + bytes + 15) >> 4;
        for (int q = lane; q < nz; q += 32) z[q] = make_uint4(0, 0, 0, 0);
    }
    __syncwarp();
    if (have) buf[shift + rel] = hdr;
    __syncwarp();
    bool ok = true;
    // leaves: one lane per record, 16 values, aligned word stores
    if (leaf && size > 1) {
        const double2* src = reinterpret_cast<const double2*>(F.op + 16 * static_cast<int64_t>(cell));
        double2 v[8];  // the whole operator in flight before any use
#pragma unroll
        for (int h = 0; h < 8; ++h) v[h] = __ldcs(src + h);
        double x[16];
#pragma unroll
        for (int h = 0; h < 8; ++h) {
            x[2 * h] = v[h].x - (0.0 + c_kunit[2 * h] * e);
            x[2 * h + 1] = v[h].y - (0.0 + c_kunit[2 * h + 1] * e);
            ok &= dev_isfinite(x[2 * h]) & dev_isfinite(x[2 * h + 1]);  // no short-circuit branches
        }
        // the integrated operators repeat 9 values (k9_expand), and so does the baseline
        const bool sym = x[1] == x[4] && x[11] == x[14] && x[2] == x[8] && x[7] == x[13] && x[3] == x[12] &&
                         x[3] == x[6] && x[3] == x[9];
        uint8_t* dst = buf + shift + rel + 1;
        switch (p3) {
            case 2: leaf_payload<2>(dst, x, sym); break;
            case 3: leaf_payload<3>(dst, x, sym); break;
            case 4: leaf_payload<4>(dst, x, sym); break;
            case 5: leaf_payload<5>(dst, x, sym); break;
            case 6: leaf_payload<6>(dst, x, sym); break;
            case 7: leaf_payload<7>(dst, x, sym); break;
            default: leaf_payload<8>(dst, x, sym); break;
        }
    }
    __syncwarp();
    // refined records with a payload: the whole warp, lane = value
    unsigned todo = __ballot_sync(full, have && !leaf && size > 1);
    while (todo) {
        const int r = __ffs(todo) - 1;
        todo &= todo - 1;
        const int rp3 = __shfl_sync(full, p3, r), rrel = __shfl_sync(full, rel, r);
        const int rcell = __shfl_sync(full, cell, r);
        const double re = __shfl_sync(full, e, r);
        const double* P = (C.P && C.has_P[rcell]) ? C.P + 64 * static_cast<int64_t>(rcell) : nullptr;
        uint8_t* dst = buf + shift + rrel + 1;
        if (!P) {
            // geometric transfer: Â, then P̂ = R̂ = geo - geo = +0 -> (0, 0, -128),
            // whose only non-zero byte is the exponent (raw +0 at p3 = 8)
            if (lane < 16) {
                const int j = r / 10;  // the patch of record lane r
                const double xa = j == 0 ? ra[0] : (j == 1 ? ra[1] : ra[2]);
                const double x = xa - (0.0 + s_kunit[lane] * re);
                ok = ok && dev_isfinite(x);
                put_bytes(dst + lane * rp3, encode_word(x, rp3), rp3);
            }
            if (rp3 < 8)
                for (int q = lane; q < 128; q += 32) dst[(16 + q) * rp3 + rp3 - 1] = 0x80;
            continue;
        }
        for (int i = lane; i < 144; i += 32) {
            double x;
            if (i < 16) {
                x = C.op[16 * static_cast<int64_t>(rcell) + i] - (0.0 + s_kunit[i] * re);
            } else {
                const int kk = (i - 16) & 63;  // P-hat, then the R-hat copy (stream.cpp:326-335)
                x = P ? P[kk] - s_geo[kk] : s_geo[kk] - s_geo[kk];
            }
            ok = ok && dev_isfinite(x);
            put_bytes(dst + i * rp3, encode_word(x, rp3), rp3);
        }
    }
    __syncwarp();
    // write-out of [g0, g0 + bytes)
    const int64_t a0 = (g0 + 15) & ~int64_t{15}, end = g0 + bytes;
    const int64_t a1 = max(a0, end & ~int64_t{15});
    const int head = static_cast<int>(min(a0, end) - g0);
    if (lane < head) out[g0 + lane] = buf[shift + lane];
    const int nvec = static_cast<int>((a1 - a0) >> 4);
    const uint4* src = reinterpret_cast<const uint4*>(buf + (a0 - g0) + shift);
    uint4* dst = reinterpret_cast<uint4*>(out + a0);
    for (int q = lane; q < nvec; q += 32) __stcs(dst + q, src[q]);
    if (a0 < end && lane < end - a1) out[a1 + lane] = buf[shift + (a1 - g0) + lane];
    if (!__all_sync(full, ok) && lane == 0) atomicExch(err, 1);
}

// Records of levels 0..D-2 (1/80 of the image): one warp per record, lane =
// value, bytes straight to global memory.
// Cell t of the upper levels in the walk order of k_pack_upper /
// k_record_sizes_upper: levels 0..D-2 (ca < 0), or levels 1..D-2 of the
// level-1 subtree (ca, cb) (9^(l-1) cells at level l).
__device__ __forceinline__ void upper_cell(const AllLevels& A, int64_t t, int ca, int cb, int& l, int& cx, int& cy) {
    l = ca < 0 ? 0 : 1;
    int64_t n = 1;
    while (t >= n) {
        t -= n;
        ++l;
        n *= 9;
    }
    const int w = ca < 0 ? A.L[l].N : A.L[l].N / 3;
    cx = (ca < 0 ? 0 : ca * w) + static_cast<int>(t % w);
    cy = (cb < 0 ? 0 : cb * w) + static_cast<int>(t / w);
}

__global__ void k_pack_upper(AllLevels A, lzb_field f, int64_t ncells, const int64_t* __restrict__ offsets,
                             uint8_t* __restrict__ out, int* err, int ca, int cb,
                             const int64_t* __restrict__ basep) {
    lzb_pdl_enter();
    const int lane = threadIdx.x & 31;
    int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (t >= ncells) return;
    int l, cx, cy;
    upper_cell(A, t, ca, cb, l, cx, cy);
    const LevelView& L = A.L[l];
    const int c = cy * L.N + cx;
    const int32_t p1 = L.p1[c];
    const int p3 = p1 != LZB_P1_BOTTOM ? L.p3[c] : 0;
    const int size = record_size(p1, p3, false);
    uint8_t* rec = out + 12 + offsets[slot_at(A.st, l, cx, cy)] + (basep ? *basep : 0);
    if (lane == 0) rec[0] = pack_header(p1, L.p2[c], p3);
    if (size == 1) return;
    const double e = centre_eps(f, L, cx, cy);
    const double* P = (L.P && L.has_P[c]) ? L.P + 64 * static_cast<int64_t>(c) : nullptr;
    uint8_t* dst = rec + 1;
    const unsigned long long zero = encode_word(0.0, p3);  // geometric P-hat / R-hat: geo - geo = +0
    bool ok = true;
    for (int i = lane; i < 144; i += 32) {
        if (i >= 16 && !P) {
            put_bytes(dst + i * p3, zero, p3);
            continue;
        }
        const double x = i < 16 ? L.op[16 * static_cast<int64_t>(c) + i] - baseline_entry(i, e)
                                : P[(i - 16) & 63] - c_geo[(i - 16) & 63];
        ok = ok && dev_isfinite(x);
        put_bytes(dst + i * p3, encode_word(x, p3), p3);
    }
    if (!__all_sync(0xffffffffu, ok) && lane == 0) atomicExch(err, 1);
}

// Record sizes in slot order (stream.cpp:227-237): one thread per
// level-(D-1) patch writes its record and its 9 leaves' (10 consecutive
// slots); one thread per cell of the levels above.
__global__ void k_record_sizes_patches(AllLevels A, int64_t* __restrict__ sizes, int px0, int pxn, int py_base) {
    lzb_pdl_enter();
    const int D = A.D;
    const LevelView& C = A.L[D - 1];
    const LevelView& F = A.L[D];
    const int px = px0 + blockIdx.x * blockDim.x + threadIdx.x, py = py_base + blockIdx.y;
    if (px >= px0 + pxn) return;
    const int64_t sP = slot_at(A.st, D - 1, px, py);
    int c = py * C.N + px;
    int32_t p1 = C.p1[c];
    sizes[sP] = record_size(p1, p1 != LZB_P1_BOTTOM ? C.p3[c] : 0, false);
#pragma unroll
    for (int ci = 0; ci < 9; ++ci) {
        c = (3 * py + ci % 3) * F.N + 3 * px + ci / 3;
        p1 = F.p1[c];
        sizes[sP + 1 + ci] = record_size(p1, p1 != LZB_P1_BOTTOM ? F.p3[c] : 0, true);
    }
}
__global__ void k_record_sizes_upper(AllLevels A, int64_t ncells, int64_t* __restrict__ sizes, int ca, int cb) {
    lzb_pdl_enter();
    int64_t t = gtid();
    if (t >= ncells) return;
    int l, cx, cy;
    upper_cell(A, t, ca, cb, l, cx, cy);
    const LevelView& L = A.L[l];
    const int c = cy * L.N + cx;
    const int32_t p1 = L.p1[c];
    sizes[slot_at(A.st, l, cx, cy)] = record_size(p1, p1 != LZB_P1_BOTTOM ? L.p3[c] : 0, false);
}

// ---- the small levels of the cycle in one block: levels 0..lc ((N+1)^2 <=
// 100 vertices each) run the per-vertex bodies of the per-level kernels in
// the same order, a block barrier between passes (global writes of the block
// are visible to it after __syncthreads). Bit-identical to the per-level
// launches. (Measured, round 2: the same fusion over an 8-block cluster with
// cluster barriers, extended to the 27^2 and 81^2 levels, cut the 729^2 settled
// cycle from 40 to 22 launches but ran 183 us against 166 us: a handful of SMs
// doing the latency-bound per-vertex gathers of 6.7 k vertices per pass loses
// to separate launches spread over the GPU with programmatic dependent launch.)
constexpr int kSmallThreads = 1024;
constexpr int kSmallMaxN = 9;
struct Damp {
    double d[kMaxLevels];
};
#define LZB_FOR_VERTS(L, i) for (int64_t i = threadIdx.x; i < static_cast<int64_t>((L).N + 1) * ((L).N + 1); i += blockDim.x)

// residual_pass of levels lc..0 (uhat, residual, restriction per level)
__global__ void __launch_bounds__(kSmallThreads) k_small_front(AllLevels A, int lc, lzb_field f) {
    lzb_pdl_enter();
    for (int l = lc; l >= 0; --l) {
        const LevelView F = A.L[l], C = A.L[l > 0 ? l - 1 : 0];
        LZB_FOR_VERTS(F, i) k_uhat_body<true>(i, F, C, l > 0 ? 1 : 0);
        __syncthreads();
        LZB_FOR_VERTS(F, i) k_residual_body<true>(i, F, f);
        __syncthreads();
        if (l > 0) {
            LZB_FOR_VERTS(C, i) k_restrict_body<true>(i, F, C, 0, 0.0);
            __syncthreads();
        }
    }
}
// snapshots of levels 0..lc (update_pass prologue)
__global__ void __launch_bounds__(kSmallThreads) k_small_snap(AllLevels A, int lc) {
    lzb_pdl_enter();
    for (int l = 0; l <= lc; ++l) LZB_FOR_VERTS(A.L[l], i) k_snap_body<true>(i, A.L[l]);
}
// update_pass of levels lc..0, then the prolongation of levels 1..lc
__global__ void __launch_bounds__(kSmallThreads) k_small_back(AllLevels A, int lc, int variant, double omega,
                                                               Damp dm, lzb_field f) {
    lzb_pdl_enter();
    for (int l = lc; l >= 0; --l) {
        const LevelView F = A.L[l];
        if (variant != LZB_ADDITIVE && l > 0) {
            const LevelView C = A.L[l - 1];
            if (variant == LZB_ADAFAC_PI) {
                LZB_FOR_VERTS(C, i) k_aux_inject_body<true>(i, F, C);
                __syncthreads();
            } else {
                LZB_FOR_VERTS(F, i) k_aux_Ar_body<true>(i, F, f);
                __syncthreads();
                LZB_FOR_VERTS(C, i) k_restrict_body<true>(i, F, C, 1, omega);
                __syncthreads();
            }
            LZB_FOR_VERTS(F, i) k_aux_sub_body<true>(i, F, C, omega);
            __syncthreads();
        }
        LZB_FOR_VERTS(F, i) k_jacobi_body<true>(i, F, dm.d[l]);
        __syncthreads();
    }
    for (int l = 1; l <= lc; ++l) {
        LZB_FOR_VERTS(A.L[l], i) k_prolong_body<true>(i, A.L[l], A.L[l - 1]);
        __syncthreads();
    }
}
// injection of levels lc..1 into lc-1..0
__global__ void __launch_bounds__(kSmallThreads) k_small_inject(AllLevels A, int lc) {
    lzb_pdl_enter();
    for (int l = lc; l >= 1; --l) {
        LZB_FOR_VERTS(A.L[l - 1], i) k_inject_body<true>(i, A.L[l], A.L[l - 1]);
        __syncthreads();
    }
}
// the bottom of a V(nu, nu) cycle (Grid::vback_body) on the small levels lc..0
// in one block: down (nu sweeps, residual, restriction into a zero-start
// coarse problem), then up (prolongation against a zero snapshot, nu sweeps)
// -- the per-level launches' bodies in their order, a block barrier between
// passes. Level 0 has no interior vertex: nothing is smoothed there.
__global__ void __launch_bounds__(kSmallThreads) k_small_v(AllLevels A, int lc, int nu, double omega, lzb_field f) {
    lzb_pdl_enter();
    for (int l = lc; l >= 1; --l) {
        const LevelView F = A.L[l], C = A.L[l - 1];
        for (int k = 0; k <= nu; ++k) {  // nu sweeps, then the residual that is restricted
            LZB_FOR_VERTS(F, i) k_residual_body<true>(i, F, f);
            __syncthreads();
            if (k == nu) break;
            LZB_FOR_VERTS(F, i) k_jacobi_body<true>(i, F, omega);
            __syncthreads();
        }
        LZB_FOR_VERTS(C, i) {
            k_restrict_body<true>(i, F, C, 0, 0.0);
            C.v[LZB_V_U][i] = 0.0;
        }
        __syncthreads();
    }
    for (int l = 1; l <= lc; ++l) {
        const LevelView F = A.L[l], C = A.L[l - 1];
        LZB_FOR_VERTS(C, i) C.v[LZB_V_USNAP][i] = 0.0;
        __syncthreads();
        LZB_FOR_VERTS(F, i) k_prolong_body<true>(i, F, C);
        __syncthreads();
        for (int k = 0; k < nu; ++k) {
            LZB_FOR_VERTS(F, i) k_residual_body<true>(i, F, f);
            __syncthreads();
            LZB_FOR_VERTS(F, i) k_jacobi_body<true>(i, F, omega);
            __syncthreads();
        }
    }
}
#undef LZB_FOR_VERTS

// ---- the middle levels of the update pass in three launches. Between the
// small levels (one block) and the leaf level (k_update_fine) the update pass
// ran, per level, a snapshot, the adaFAC-PI injection, the aux correction and
// the Jacobi step, and after the prolongation one injection per level: 16
// launches of a few microseconds of work at 729^2, a third of the cycle's
// latency. None of them depends on another level's result (the injections
// read r, which the update pass never writes; the aux correction reads the
// level below's aux and diagonal only; a level's injected u is the leaf
// level's u at the same point), so each group runs as one launch over the
// concatenated vertices of levels l0..l1, every vertex through the per-level
// bodies in the per-level order: the same bits.
struct MidRange {
    int l0, l1;                 // levels l0..l1
    int64_t start[kMaxLevels];  // first concatenated index of level l (start[l1 + 1] = total)
};
__device__ __forceinline__ bool mid_locate(const MidRange& R, int64_t t, int& l, int64_t& i) {
    if (t >= R.start[R.l1 + 1]) return false;
    l = R.l0;
    while (l < R.l1 && t >= R.start[l + 1]) ++l;
    i = t - R.start[l];
    return true;
}
// usnap = u; aux = the injected residual of the level above (adaFAC-PI), else 0.
// lc_aux >= 0: also the injection into level lc_aux (the top small level,
// snapshot already taken by k_small_snap) -- its indices follow level l1's.
// R covers levels 0..l1 here: the small levels' snapshot (k_small_snap) rides
// along; their injections (levels below lc_aux) stay in k_small_back, which
// runs them in the per-level order after this kernel.
__global__ void k_mid_snap(AllLevels A, MidRange R, int pi, int lc_aux) {
    lzb_pdl_enter();
    int l;
    int64_t i;
    if (!mid_locate(R, gtid(), l, i)) return;
    k_snap_body<true>(i, A.L[l]);
    if (pi && l >= lc_aux && l >= 0) k_aux_inject_body<true>(i, A.L[l + 1], A.L[l]);
}
// the aux correction (adaFAC-PI) and the Jacobi step of levels l0..l1
// (and, adaFAC-PI, k_scale_aux of level l1 = D - 1 for the leaf update: it
// reads that level's aux and diagonal, which nothing here writes)
__global__ void k_mid_update(AllLevels A, MidRange R, int pi, double omega, Damp dm, double* __restrict__ caux) {
    lzb_pdl_enter();
    int l;
    int64_t i;
    if (!mid_locate(R, gtid(), l, i)) return;
    if (pi && l == R.l1) {
        const LevelView C = A.L[l];
        const int NV = C.N + 1;
        const int cy = static_cast<int>(i / NV), cx = static_cast<int>(i - static_cast<int64_t>(cy) * NV);
        const double cdg = C.v[LZB_V_DIAG][i];
        caux[i] = (!boundary(C.N, cx, cy) && cdg != 0.0) ? omega / cdg * C.v[LZB_V_AUX][i] : 0.0;
    }
    if (pi && l > 0) k_aux_sub_body<true>(i, A.L[l], A.L[l - 1], omega);
    k_jacobi_body<true>(i, A.L[l], dm.d[l]);
}
// u-hat of levels l0..l1 (compute_uhat, solver.cpp:120-143): u of every level
// is fixed during the residual pass, so the middle levels' u-hat do not wait
// for the restriction chain
__global__ void k_mid_uhat(AllLevels A, MidRange R) {
    lzb_pdl_enter();
    int l;
    int64_t i;
    if (!mid_locate(R, gtid(), l, i)) return;
    k_uhat_body<true>(i, A.L[l], A.L[l > 0 ? l - 1 : 0], l > 0 ? 1 : 0);
}
// inject_solution of levels l0..l1 from the leaf level (level l's vertex v is
// leaf vertex 3^(D-l) v; the per-level chain copies the same value down)
__global__ void k_mid_inject(AllLevels A, MidRange R) {
    lzb_pdl_enter();
    int l;
    int64_t i;
    if (!mid_locate(R, gtid(), l, i)) return;
    const LevelView C = A.L[l], F = A.L[A.D];
    const int NV = C.N + 1;
    const int iy = static_cast<int>(i / NV), ix = static_cast<int>(i - static_cast<int64_t>(iy) * NV);
    const int s3 = F.N / C.N;
    C.v[LZB_V_U][i] = F.v[LZB_V_U][static_cast<int64_t>(s3 * iy) * (F.N + 1) + s3 * ix];
}

// Running image offset of the bands of level-1 subtrees (assemble_stream):
// base[1] = base[0] + the band's bytes (its last local offset plus its last record).
__global__ void k_chunk_base(const int64_t* __restrict__ sizes, const int64_t* __restrict__ offs, int64_t n,
                             int64_t* base) {
    lzb_pdl_enter();
    base[1] = base[0] + offs[n - 1] + sizes[n - 1];
}
__global__ void k_root_base(const int64_t* __restrict__ sizes, int64_t* __restrict__ offs, int64_t* base) {
    lzb_pdl_enter();
    offs[0] = 0;
    base[0] = sizes[0];
}

// CellStream::load record (stream.cpp:355-392); offsets from the host parse.
__global__ void k_unpack(LevelView L, lzb_field f, int level, int leaf, SlotTable st,
                         const int64_t* __restrict__ offsets, const uint8_t* __restrict__ in,
                         double delta_max, uint32_t cycle, unsigned long long* stats, int* err) {
    lzb_pdl_enter();
    int64_t c = gtid();
    if (c >= static_cast<int64_t>(L.N) * L.N) return;
    int cx = static_cast<int>(c % L.N), cy = static_cast<int>(c / L.N);
    const uint8_t* rec = in + offsets[slot_at(st, level, cx, cy)];
    uint8_t h = rec[0];
    int cls = (h >> 6) & 3, p2 = (h & 0x20) != 0, p3 = h & 0x0f;
    L.p2[c] = static_cast<uint8_t>(p2);
    if (cls == 0) {
        L.p1[c] = LZB_P1_BOTTOM;
        if (L.cp3) L.cp3[c] = -1;
        L.chg[c] = cycle + 1;  // the payload disappears: parents must see it
        return;
    }
    double e = centre_eps(f, L, cx, cy);
    double m[16], P[64];
    for (int k = 0; k < 16; ++k) m[k] = baseline_entry(k, e);
    for (int k = 0; k < 64; ++k) P[k] = c_geo[k];
    if (p3 != 0) {
        const uint8_t* cur = rec + 1;
        for (int k = 0; k < 16; ++k, cur += p3) m[k] += decode_value(cur, p3);
        if (!leaf)
            for (int k = 0; k < 64; ++k, cur += p3) P[k] += decode_value(cur, p3);
    }
    if (leaf) {
        if (!publish_leaf(L, static_cast<int>(c), m, 1, e, delta_max, cycle, stats)) atomicExch(err, 1);
    } else {
        // publish_coarse (stream.cpp:134-184)
        double joint[80];
        for (int k = 0; k < 16; ++k) joint[k] = m[k] - baseline_entry(k, e);
        for (int k = 0; k < 64; ++k) joint[16 + k] = P[k] - c_geo[k];
        int q3 = choose_precision(joint, 80, delta_max);
        if (q3 < 0) {
            atomicExch(err, 1);
            return;
        }
        double delta = 0.0;
        for (int k = 0; k < 80; ++k) {
            double rt;
            if (!roundtrip_fast(joint[k], q3, rt)) { atomicExch(err, 1); return; }
            double d = fabs(rt - joint[k]);
            delta = delta < d ? d : delta;
            if (k < 16) m[k] = baseline_entry(k, e) + rt;
            else P[k - 16] = c_geo[k - 16] + rt;
        }
        double* op = L.op + 16 * c;
        bool same = L.p1[c] == LZB_P1_TOP && L.has_P[c];
        if (same) {
            const double* cur = L.P ? L.P + 64 * c : c_geo;
            for (int k = 0; k < 16; ++k) same = same && m[k] == op[k];
            for (int k = 0; k < 64; ++k) same = same && P[k] == cur[k];
        }
        if (!same) {
            atomic_max_double_bits(&stats[S_MAXDELTA], delta);
            for (int k = 0; k < 16; ++k) op[k] = m[k];
            if (L.P)
                for (int k = 0; k < 64; ++k) L.P[64 * c + k] = P[k];
            L.has_P[c] = 1;
            L.n[c] = 1;
            L.epoch[c] = cycle;
            L.chg[c] = cycle + 1;
            L.p3[c] = static_cast<int8_t>(q3);
        }
    }
    L.p1[c] = cls == 2 ? LZB_P1_TOP : 1;
    L.p3[c] = static_cast<int8_t>(p3);
}

// assemble_vertex_stencil (assembly.cpp:120-136) for every vertex of a level:
// the adjacent cells (stepping c = SW, SE, NW, NE) contribute, through
// scatter_row (element.cpp:39-45), the row of the corner diagonally opposite
// to the step; missing cells contribute zero. out: 9 per vertex, index
// (dy+1)*3 + (dx+1) (Stencil9, types.hpp:53-58). require_payload: a bottom
// neighbour raises *err (protocol_error).
__global__ void k_vertex_stencils(LevelView F, lzb_field f, double* __restrict__ out, int require_payload,
                                  int* err) {
    lzb_pdl_enter();
    int ix, iy;
    int64_t vi;
    if (!vertex_xy(F, ix, iy, vi)) return;
    double st[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int c = 0; c < 4; ++c) {
        const int cx = ix - 1 + cdx(c), cy = iy - 1 + cdy(c);
        if (cx < 0 || cy < 0 || cx >= F.N || cy >= F.N) continue;
        if (require_payload && F.p1[static_cast<int64_t>(cy) * F.N + cx] == LZB_P1_BOTTOM) atomicExch(err, 1);
        const int corner = (1 - cdx(c)) | ((1 - cdy(c)) << 1);
        double K[16];
        element_or_baseline(f, F, cx, cy, K);
        for (int k = 0; k < 4; ++k) {
            const int dx = cdx(k) - cdx(corner), dy = cdy(k) - cdy(corner);
            st[(dy + 1) * 3 + (dx + 1)] += K[corner * 4 + k];
        }
    }
    for (int k = 0; k < 9; ++k) out[9 * vi + k] = st[k];
}

// Single-cell protocol ops for the per-cell compatibility API.
__global__ void k_publish_one(LevelView F, lzb_field f, int c, const double* m, int n, int32_t p1,
                              double delta_max, uint32_t cycle, unsigned long long* stats, int* err) {
    lzb_pdl_enter();
    if (gtid() != 0) return;
    double e = centre_eps(f, F, c % F.N, c / F.N);
    if (!publish_leaf(F, c, m, n, e, delta_max, cycle, stats)) atomicExch(err, 1);
    F.p1[c] = p1;
    if (F.cp3 && p1 == LZB_P1_BOTTOM) F.cp3[c] = -1;
}

// CellStream::publish_element + marker store for every leaf cell (the batched
// form of k_publish_one; mats: 16 doubles per cell, n per cell).
__global__ void k_publish_level(LevelView F, lzb_field f, const double* __restrict__ mats,
                                const int32_t* __restrict__ nn, int32_t p1, double delta_max, uint32_t cycle,
                                unsigned long long* stats, int* err) {
    lzb_pdl_enter();
    const int64_t c = gtid();
    if (c >= static_cast<int64_t>(F.N) * F.N) return;
    double m[16];
    for (int k = 0; k < 16; ++k) m[k] = mats[16 * c + k];
    const double e = centre_eps(f, F, static_cast<int>(c % F.N), static_cast<int>(c / F.N));
    if (!publish_leaf(F, static_cast<int>(c), m, nn[c], e, delta_max, cycle, stats)) atomicExch(err, 1);
    F.p1[c] = p1;
    if (F.cp3 && p1 == LZB_P1_BOTTOM) F.cp3[c] = -1;
}

__global__ void k_step_one(LevelView F, lzb_field f, int c, int schedule, int n_max, double term_c,
                           double delta_max, uint32_t cycle, int fast, unsigned long long* stats,
                           int* err) {
    lzb_pdl_enter();
    if (gtid() != 0) return;
    int cx = c % F.N, cy = c / F.N;
    int32_t p1 = F.p1[c];
    if (p1 == LZB_P1_TOP) return;
    double e = centre_eps(f, F, cx, cy);
    if (p1 == LZB_P1_BOTTOM) {
        double m[16];
        for (int k = 0; k < 16; ++k) m[k] = baseline_entry(k, e);
        if (!publish_leaf_k9(F, c, m, 1, e, delta_max, cycle, stats)) atomicExch(err, 1);
        F.p1[c] = 1;
        return;
    }
    int n = p1;
    if (n_max > 0 && n >= n_max) {
        F.p1[c] = LZB_P1_TOP;
        return;
    }
    int nn = schedule == LZB_SCHEDULE_DOUBLE ? 2 * n : n + 1;
    if (n_max > 0 && nn > n_max) nn = n_max;
    double fresh[16];
    integrate_cell(f, cx * F.h, cy * F.h, F.h, nn, fast, fresh);
    const double* old = F.op + 16 * static_cast<int64_t>(c);
    double denom = 0.0, dmax = 0.0;
    for (int k = 0; k < 16; ++k) {
        double a = fabs(old[k]);
        denom = denom < a ? a : denom;
        double d = fabs(fresh[k] - old[k]);
        dmax = dmax < d ? d : dmax;
    }
    double ratio = 0.0;
    if (denom == 0.0) atomicAdd(&stats[S_ZERO_NORM], 1ull);
    else ratio = dmax / denom;
    if (ratio < term_c) {
        F.p1[c] = LZB_P1_TOP;
        return;
    }
    if (!publish_leaf(F, c, fresh, nn, e, delta_max, cycle, stats)) atomicExch(err, 1);
    F.p1[c] = nn;
}

__global__ void k_clear_p2(LevelView F, const int32_t* list, int count) {
    lzb_pdl_enter();
    int64_t t = gtid();
    if (t < count) F.p2[list[t]] = 0;
}

// Concurrent assembly, fallback for batch entries off the lockstep n: the
// adaptive step with on-the-fly axis parts (same arithmetic), outcome to D.
__global__ void k_step_generic(LevelView F, LevelView D, lzb_field f, const int32_t* list,
                               const int32_t* snap, const int* count_ptr, int n_main, int schedule,
                               int n_max, int fast, double term_c, double delta_max, uint32_t cycle,
                               unsigned long long* stats, int* err) {
    lzb_pdl_enter();
    int64_t t = gtid();
    if (t >= *count_ptr) return;
    const int32_t p1 = snap[t];
    if (p1 == n_main || p1 == LZB_P1_BOTTOM || p1 == kForcedSnap) return;  // main kernel / bottoms / forced
    const int c = list[t], cx = c % F.N, cy = c / F.N;
    if (p1 == LZB_P1_TOP || (n_max > 0 && p1 >= n_max)) {
        D.p1[c] = LZB_P1_TOP;
        return;
    }
    int nn = schedule == LZB_SCHEDULE_DOUBLE ? 2 * p1 : p1 + 1;
    if (n_max > 0 && nn > n_max) nn = n_max;
    double fresh[16];
    integrate_cell(f, cx * F.h, cy * F.h, F.h, nn, fast, fresh);
    const double* old = F.op + 16 * static_cast<int64_t>(c);
    double denom = 0.0, dmax = 0.0;
    for (int k = 0; k < 16; ++k) {
        double a = fabs(old[k]);
        denom = denom < a ? a : denom;
        double d = fabs(fresh[k] - old[k]);
        dmax = dmax < d ? d : dmax;
    }
    double ratio = 0.0;
    if (denom == 0.0) atomicAdd(&stats[S_ZERO_NORM], 1ull);
    else ratio = dmax / denom;
    if (ratio < term_c) {
        D.p1[c] = LZB_P1_TOP;
        return;
    }
    if (!publish_leaf_k9(D, c, fresh, nn, centre_eps(f, F, cx, cy), delta_max, cycle, stats))
        atomicExch(err, 1);
    D.p1[c] = nn;
}

// Swap-in of a completed concurrent batch, on the solve stream: the outcome of
// every task in the batch becomes the live operator / marker, and the task
// completes (p2 cleared, assembly.cpp:66-68).
__global__ void k_commit(LevelView F, LevelView S, const int32_t* list, const int* count_ptr,
                         uint32_t cycle) {
    lzb_pdl_enter();
    int64_t t = gtid();
    if (t >= *count_ptr) return;
    const int c = list[t];
    const int32_t p1 = S.p1[c];
    if (p1 != LZB_P1_TOP) {
        const double2* src = reinterpret_cast<const double2*>(S.op + 16 * static_cast<int64_t>(c));
        double2* dst = reinterpret_cast<double2*>(F.op + 16 * static_cast<int64_t>(c));
        for (int q = 0; q < 8; ++q) dst[q] = src[q];
        F.n[c] = S.n[c];
        F.p3[c] = S.p3[c];
        if (F.cp3) F.cp3[c] = 9;  // no compressed copy staged: FP64 operator
        F.epoch[c] = S.epoch[c];
        F.chg[c] = cycle + 1;  // swapped in at this cycle's start: the walk sees it
    }
    F.p1[c] = p1;
    F.p2[c] = 0;
}

__global__ void k_reset_stats(Result* r) {
    lzb_pdl_enter();
    // per-cycle slots; the norm is written by k_norm_final
    if (threadIdx.x < 13 || threadIdx.x == S_PENDING) r->s[threadIdx.x] = 0;
}

// ---- device-side cycle loop (Grid::run_device_loop): the termination test of
// solver.cpp:8-16 on the device, steering a conditional WHILE graph node whose
// body is one whole cycle, so a quiescent solve (no assembly work pending)
// runs cycle after cycle without a host round trip per residual norm.
struct LoopState {
    double front;        // history.front(): the first residual of the solve
    double target, divergence;
    int32_t max_cycles;
    uint32_t count, cap;  // cycles recorded by this launch / room in the history
    int32_t status, err;
    int32_t settled;  // out (full body): a whole coarse pass found nothing to recompute
};
// ++cycle (the epoch the coarse pass stamps)
__global__ void k_loop_begin(uint32_t* cycle) {
    lzb_pdl_enter();
    if (threadIdx.x == 0) *cycle += 1;
}
// After a cycle's residual pass and stats: record the result, decide
// (check_termination), and set the two conditions -- `update` (the IF node
// around update + prolongation + injection: solver.cpp:359-370 runs them on
// CONTINUE and on TIMEOUT) and `again` (the WHILE node).
__global__ void k_loop_check(Result* res, Result* hist, LoopState* st, const uint32_t* cycle, const int* err,
                             cudaGraphConditionalHandle h_again, cudaGraphConditionalHandle h_update, int full) {
    lzb_pdl_enter();
    if (threadIdx.x != 0) return;
    const uint32_t i = st->count;
    // full body: did this cycle's coarse pass recompute anything? When it did
    // not, no operator, marker or epoch changed, so the next pass cannot
    // either (its gates read only those): the hierarchy has settled, and the
    // coarse pass and the stats are no-ops from here on (the settled body).
    bool settled = false;
    if (full) settled = res->s[S_COARSE_ACTIVE] != *cycle;
    hist[i] = *res;
    st->count = i + 1;
    const double normalized = res->norm / st->front;
    int status = LZB_CONTINUE;
    if (normalized <= st->target) status = LZB_CONVERGED;
    else if (normalized >= st->divergence) status = LZB_DIVERGED;
    else if (static_cast<int>(*cycle) >= st->max_cycles) status = LZB_TIMEOUT;
    const bool bad = *err != 0;  // a non-finite encode: the host throws, nothing more runs
    st->status = status;
    st->err = bad ? 1 : 0;
    st->settled = settled ? 1 : 0;
    const bool update = !bad && (status == LZB_CONTINUE || status == LZB_TIMEOUT);
    cudaGraphSetConditional(h_update, update ? 1u : 0u);
    cudaGraphSetConditional(h_again, (!bad && !settled && status == LZB_CONTINUE && i + 1 < st->cap) ? 1u : 0u);
}

template <int KIND, bool FAST>
void launch_step_k(cudaStream_t s, const LevelView& F, const LevelView& D, const lzb_field& f,
                   const int32_t* list, const int32_t* snap, const int* count_ptr, int64_t max_count,
                   int n, int nn, int cap, const IntTables& T, double term_c, double dmax, uint32_t cycle,
                   unsigned long long* stats, int* err) {
    size_t smem = cap ? 0 : int_smem_bytes(nn);
    set_smem(k_step<KIND, FAST>, smem);
    LZB_LAUNCH((k_step<KIND, FAST>), blocks_for(max_count, kIntThreads * kCPT), kIntThreads, smem, s, F, D,
               f, list, snap, count_ptr, n, nn, cap, T, term_c, dmax, cycle, 0, stats, err);
}

template <int KIND>
void launch_step(bool fast, cudaStream_t s, const LevelView& F, const LevelView& D, const lzb_field& f,
                 const int32_t* list, const int32_t* snap, const int* count_ptr, int64_t max_count,
                 int n, int nn, int cap, const IntTables& T, double term_c, double dmax, uint32_t cycle,
                 unsigned long long* stats, int* err) {
    if (fast)
        launch_step_k<KIND, true>(s, F, D, f, list, snap, count_ptr, max_count, n, nn, cap, T, term_c, dmax,
                                  cycle, stats, err);
    else
        launch_step_k<KIND, false>(s, F, D, f, list, snap, count_ptr, max_count, n, nn, cap, T, term_c, dmax,
                                   cycle, stats, err);
}

// Dispatch on the field kind (one instantiation per kind).
inline void dispatch_step(bool fast, cudaStream_t s, const LevelView& F, const LevelView& D,
                          const lzb_field& f, const int32_t* list, const int32_t* snap,
                          const int* count_ptr, int64_t max_count, int n, int nn, int cap,
                          const IntTables& T, double term_c, double dmax, uint32_t cycle,
                          unsigned long long* stats, int* err) {
    switch (f.kind) {
        case LZB_FIELD_THETA: launch_step<LZB_FIELD_THETA>(fast, s, F, D, f, list, snap, count_ptr, max_count, n, nn, cap, T, term_c, dmax, cycle, stats, err); break;
        case LZB_FIELD_QUADRANT: launch_step<LZB_FIELD_QUADRANT>(fast, s, F, D, f, list, snap, count_ptr, max_count, n, nn, cap, T, term_c, dmax, cycle, stats, err); break;
        case LZB_FIELD_CHECKER: launch_step<LZB_FIELD_CHECKER>(fast, s, F, D, f, list, snap, count_ptr, max_count, n, nn, cap, T, term_c, dmax, cycle, stats, err); break;
        case LZB_FIELD_SINUSOID: launch_step<LZB_FIELD_SINUSOID>(fast, s, F, D, f, list, snap, count_ptr, max_count, n, nn, cap, T, term_c, dmax, cycle, stats, err); break;
        default: launch_step<LZB_FIELD_CONSTANT>(fast, s, F, D, f, list, snap, count_ptr, max_count, n, nn, cap, T, term_c, dmax, cycle, stats, err); break;
    }
}

template <int KIND, bool FAST>
void launch_fixed_k(cudaStream_t s, const LevelView& F, const lzb_field& f, int n, const IntTables& T,
                    double dmax, uint32_t cycle, unsigned long long* stats, int* err, int64_t cbeg,
                    int64_t cend, CellRect R, double* raw) {
    const size_t rsmem = res_smem_bytes(n);
    if (rsmem <= kResidentSmemMax) {  // persistent: K_sub table resident, one range per block
        static int grid = 0;          // per instantiation: resident blocks x SMs
        set_smem(k_fixed_res<KIND, FAST>, rsmem);
        if (!grid) {
            int dev = 0, sms = 0, per = 0;
            LZB_CUDA(cudaGetDevice(&dev));
            LZB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            LZB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_fixed_res<KIND, FAST>, kIntThreads,
                                                                   rsmem));
            grid = (per > 0 ? per : 1) * sms;
        }
        // never more blocks than cell pairs
        const int64_t want = (cend - cbeg + kCPT - 1) / kCPT;
        const unsigned g = static_cast<unsigned>(want < grid ? (want > 0 ? want : 1) : grid);
        LZB_LAUNCH((k_fixed_res<KIND, FAST>), g, kIntThreads, rsmem, s, F, f, n, T, dmax, cycle, stats, err,
                   cbeg, cend, R, raw);
        return;
    }
    size_t smem = int_smem_bytes(n);
    set_smem(k_fixed<KIND, FAST>, smem);
    LZB_LAUNCH((k_fixed<KIND, FAST>), blocks_for(cend - cbeg, kIntThreads * kCPT), kIntThreads, smem, s, F,
               f, n, T, dmax, cycle, stats, err, cbeg, cend, R, raw);
}

template <int KIND>
void launch_fixed(bool fast, cudaStream_t s, const LevelView& F, const lzb_field& f, int n,
                  const IntTables& T, double dmax, uint32_t cycle, unsigned long long* stats, int* err,
                  int64_t cbeg, int64_t cend, CellRect R, double* raw) {
    if (fast) launch_fixed_k<KIND, true>(s, F, f, n, T, dmax, cycle, stats, err, cbeg, cend, R, raw);
    else launch_fixed_k<KIND, false>(s, F, f, n, T, dmax, cycle, stats, err, cbeg, cend, R, raw);
}

}  // namespace

// ==================================================================== host
struct Level {
    int N = 1;
    int64_t nc = 1, nv = 4;
    double h = 1.0, pow3l = 1.0;
    DevBuf<int32_t> rx, ry;
    DevBuf<double> v[LZB_V_NFIELDS];
    DevBuf<double> op, P;
    DevBuf<int32_t> p1, n;
    DevBuf<uint8_t> p2, has_P;
    DevBuf<int8_t> p3;
    DevBuf<uint32_t> epoch, chg, seen;
    DevBuf<uint8_t> cplanes;  // leaf level, plane_width > 0
    DevBuf<int8_t> cp3;
    DevBuf<uint32_t> dirty;  // refined levels, coarse-recompute = ripple
    DevBuf<uint8_t> pend;
    DevBuf<double> cex, cey, rsin;  // host-libm centre parts; leaf-level load sines
    LevelView view(int depth) const {
        LevelView L{};
        L.N = N;
        L.depth_of_grid = depth;
        L.h = h;
        L.pow3l = pow3l;
        L.rx = rx.p;
        L.ry = ry.p;
        for (int f = 0; f < LZB_V_NFIELDS; ++f) L.v[f] = v[f].p;
        L.op = op.p;
        L.P = P.p;
        L.p1 = p1.p;
        L.p2 = p2.p;
        L.p3 = p3.p;
        L.n = n.p;
        L.epoch = epoch.p;
        L.chg = chg.p;
        L.seen = seen.p;
        L.has_P = has_P.p;
        L.cplanes = cplanes.p;
        L.cp3 = cp3.p;
        L.dirty = dirty.p;
        L.pend = pend.p;
        L.cex = cex.p;
        L.cey = cey.p;
        L.rsin = rsin.p;
        return L;
    }
};

class Grid {
public:
    Grid(lzb_ctx* ctx, const lzb_grid_desc& d) : ctx_(ctx), d_(d), D_(d.depth) {
        if (d.dim != 2) throw Error(LZB_ERR_INVALID, "only dim = 2 is implemented in this round");
        if (d.depth < 1) throw Error(LZB_ERR_INVALID, "mesh depth must be >= 1");
        if (d.depth > kMaxLevels - 1) throw Error(LZB_ERR_RESOURCE, "initial mesh depth exceeds the cell limit");
        if (d.field.kind == LZB_FIELD_CHECKER && (d.field.blocks < 1 || d.field.blocks > 8))
            throw Error(LZB_ERR_INVALID, "checkerboard blocks must be in 1..8");
        LZB_CUDA(cudaSetDevice(ctx->device));
        s_ = ctx->solve;
        L_.resize(D_ + 1);
        std::vector<int32_t> prx{0}, pry{0};
        for (int l = 0; l <= D_; ++l) {
            Level& L = L_[l];
            L.N = 1;
            for (int i = 0; i < l; ++i) L.N *= 3;
            L.nc = static_cast<int64_t>(L.N) * L.N;
            L.nv = static_cast<int64_t>(L.N + 1) * (L.N + 1);
            L.h = std::pow(1.0 / 3, l);
            L.pow3l = std::pow(3.0, l);
            std::vector<int32_t> rx(L.N), ry(L.N);
            for (int c = 0; c < L.N; ++c) {
                rx[c] = l == 0 ? 0 : 9 * prx[c / 3] + 3 * (c % 3);
                ry[c] = l == 0 ? 0 : 9 * pry[c / 3] + (c % 3);
            }
            L.rx.alloc(L.N);
            L.ry.alloc(L.N);
            LZB_CUDA(cudaMemcpy(L.rx.p, rx.data(), L.N * sizeof(int32_t), cudaMemcpyHostToDevice));
            LZB_CUDA(cudaMemcpy(L.ry.p, ry.data(), L.N * sizeof(int32_t), cudaMemcpyHostToDevice));
            prx.swap(rx);
            pry.swap(ry);
            for (int f = 0; f < LZB_V_NFIELDS; ++f) {
                L.v[f].alloc(L.nv);
                LZB_CUDA(cudaMemsetAsync(L.v[f].p, 0, L.v[f].bytes(), s_));
            }
            L.op.alloc(16 * L.nc);
            L.p1.alloc(L.nc);
            L.n.alloc(L.nc);
            L.p2.alloc(L.nc);
            L.p3.alloc(L.nc);
            L.epoch.alloc(L.nc);
            L.chg.alloc(L.nc);
            L.seen.alloc(L.nc);
            LZB_CUDA(cudaMemsetAsync(L.chg.p, 0, L.chg.bytes(), s_));
            LZB_CUDA(cudaMemsetAsync(L.seen.p, 0, L.seen.bytes(), s_));
            L.has_P.alloc(L.nc);
            LZB_CUDA(cudaMemsetAsync(L.op.p, 0, L.op.bytes(), s_));
            LZB_CUDA(cudaMemsetAsync(L.p1.p, 0, L.p1.bytes(), s_));
            LZB_CUDA(cudaMemsetAsync(L.n.p, 0, L.n.bytes(), s_));
            LZB_CUDA(cudaMemsetAsync(L.p2.p, 0, L.p2.bytes(), s_));
            LZB_CUDA(cudaMemsetAsync(L.p3.p, 0, L.p3.bytes(), s_));
            LZB_CUDA(cudaMemsetAsync(L.epoch.p, 0, L.epoch.bytes(), s_));
            LZB_CUDA(cudaMemsetAsync(L.has_P.p, 0, L.has_P.bytes(), s_));
            if (l < D_ && d.transfer == LZB_BOXMG) {
                L.P.alloc(64 * L.nc);
                LZB_CUDA(cudaMemsetAsync(L.P.p, 0, L.P.bytes(), s_));
            }
        }
        // centre field parts (the n = 1 sample) of every level, host libm; the
        // patch and leaf levels' also as centre_ (read by the pack / residual kernels)
        for (int l = 0; l <= D_; ++l) {
            Level& L = L_[l];
            L.cex.alloc(L.N);
            L.cey.alloc(L.N);
            upload_field_parts(d.field, L.N, L.h, 1, L.cex.p, L.cey.p, s_);
        }
        for (int k = 0; k < 2; ++k) {
            const Level& L = L_[D_ - 1 + k];
            centre_[k].x.alloc(L.N);
            centre_[k].y.alloc(L.N);
            LZB_CUDA(cudaMemcpyAsync(centre_[k].x.p, L.cex.p, L.cex.bytes(), cudaMemcpyDeviceToDevice, s_));
            LZB_CUDA(cudaMemcpyAsync(centre_[k].y.p, L.cey.p, L.cey.bytes(), cudaMemcpyDeviceToDevice, s_));
        }
        {  // sin(pi x) of the leaf vertices for the BASELINE load (k_init_rhs)
            Level& L = L_[D_];
            std::vector<double> sv(static_cast<size_t>(L.N) + 1);
            for (int i = 0; i <= L.N; ++i) sv[i] = std::sin(kPi * (i / L.pow3l));
            L.rsin.alloc(sv.size());
            LZB_CUDA(cudaMemcpyAsync(L.rsin.p, sv.data(), sv.size() * sizeof(double), cudaMemcpyHostToDevice, s_));
            LZB_CUDA(cudaStreamSynchronize(s_));
        }
        leaves_ = L_[D_].nc;
        list_.alloc(leaves_);
        snap_.alloc(leaves_);
        counter_.alloc(1);
        blockcnt_.alloc(blocks_for(leaves_, kCompactThreads));
        hist_.alloc(kNHist);
        partial_.alloc(kNormBlocks);
        if (d.variant == LZB_ADAFAC_PI && D_ >= 1) caux_.alloc(L_[D_ - 1].nv);
        if (d.policy == LZB_RIPPLE) {
            if (d.concurrent) throw Error(LZB_ERR_INVALID, "coarse-recompute = ripple needs the deterministic modes");
            for (int l = 0; l < D_; ++l) {
                L_[l].dirty.alloc(L_[l].nc);
                L_[l].pend.alloc(L_[l].nc);
                LZB_CUDA(cudaMemsetAsync(L_[l].dirty.p, 0, L_[l].dirty.bytes(), s_));
                LZB_CUDA(cudaMemsetAsync(L_[l].pend.p, 0, L_[l].pend.bytes(), s_));
            }
        }
        if (d.fixed_p3 != 0 && (d.fixed_p3 < 2 || d.fixed_p3 > 8))
            throw Error(LZB_ERR_INVALID, "fixed_p3 must be 0 or 2..8");
        if (d.plane_width != 0) {
            if (d.plane_width < 2 || d.plane_width > 8) throw Error(LZB_ERR_INVALID, "plane_width must be 0 or 2..8");
            if (d.concurrent) throw Error(LZB_ERR_INVALID, "plane_width needs the deterministic modes");
            Level& F = L_[D_];
            F.cplanes.alloc(static_cast<size_t>(F.nc) * 16 * d.plane_width);
            F.cp3.alloc(F.nc);
            LZB_CUDA(cudaMemsetAsync(F.cp3.p, 0xff, F.cp3.bytes(), s_));  // -1: every leaf starts bottom
        }
        res_.alloc(1);
        LZB_CUDA(cudaMemsetAsync(res_.p, 0, sizeof(Result), s_));
        if (d.forced_fraction > 0.0) {
            if (d.concurrent) throw Error(LZB_ERR_INVALID, "forced tasks need the deterministic modes (workers = 1)");
            if (d.mode == LZB_ADAPTIVE && d.policy == LZB_RIPPLE)
                throw Error(LZB_ERR_INVALID, "forced tasks with assembly = adaptive need coarse-recompute = always");
            if (d.forced_n < 1) throw Error(LZB_ERR_INVALID, "forced-task-n must be >= 1");
            sink_.alloc(1);
        }
        if (d.throttle || d.forced_fraction > 0.0) keys_.alloc(leaves_);
        if (d.concurrent) {
            if (d.mode != LZB_ANARCHIC)
                throw Error(LZB_ERR_INVALID, "concurrent assembly needs assembly = anarchic");
            if (d.throttle)
                throw Error(LZB_ERR_INVALID, "concurrent assembly runs every pending task (throttle = 0)");
            a_ = ctx->assembly;
            alist_.alloc(leaves_);
            asnap_.alloc(leaves_);
            acounter_.alloc(1);
            ablockcnt_.alloc(blocks_for(leaves_, kCompactThreads));
            ahist_.alloc(kNHist);
            sop_.alloc(16 * leaves_);
            sp1_.alloc(leaves_);
            sn_.alloc(leaves_);
            sp3_.alloc(leaves_);
            sepoch_.alloc(leaves_);
            schg_.alloc(leaves_);
            LZB_CUDA(cudaEventCreateWithFlags(&ev_batch_, cudaEventDisableTiming));
            LZB_CUDA(cudaEventCreateWithFlags(&ev_spawn_, cudaEventDisableTiming));
        }
        LZB_CUDA(cudaMallocHost(&hres_, sizeof(Result)));
        LZB_CUDA(cudaMallocHost(&hhist_, kNHist * sizeof(unsigned) + sizeof(int)));
        LZB_CUDA(cudaMallocHost(&hcycle_, sizeof(uint32_t)));
        LZB_CUDA(cudaMallocHost(&herr_, sizeof(int)));
        *hcycle_ = 0;
        *herr_ = 0;
        dcycle_.alloc(1);
        use_graphs_ = std::getenv("LZB_NO_GRAPHS") == nullptr;
        tables_.reserve_n = atables_.reserve_n = d_.n_max > 0 ? std::min(d_.n_max, 128) : 64;
        // subtree sizes for pre-order slots
        for (int k = 0; k <= D_; ++k) {
            int64_t s = 0, p = 1;
            for (int j = 0; j <= D_ - k; ++j, p *= 9) s += p;
            slots_.subtree[k] = s;
        }
        for (int l = 0; l <= D_; ++l) {
            const int N = L_[l].N;
            std::vector<int64_t> sx(N), sy(N);
            for (int c = 0; c < N; ++c) {
                int64_t ax = 0, ay = 0, p = N / 3;
                for (int k = 1; k <= l; ++k, p /= 3) {
                    const int64_t d = (c / p) % 3;
                    ax += 3 * d * slots_.subtree[k];
                    ay += d * slots_.subtree[k];
                }
                sx[c] = ax;
                sy[c] = ay;
            }
            slot_x_[l].alloc(N);
            slot_y_[l].alloc(N);
            LZB_CUDA(cudaMemcpy(slot_x_[l].p, sx.data(), N * sizeof(int64_t), cudaMemcpyHostToDevice));
            LZB_CUDA(cudaMemcpy(slot_y_[l].p, sy.data(), N * sizeof(int64_t), cudaMemcpyHostToDevice));
            slots_.sx[l] = slot_x_[l].p;
            slots_.sy[l] = slot_y_[l].p;
        }
        for (int l = 0; l <= D_; ++l) total_cells_ += L_[l].nc;
        for (int l = 0; l <= D_; ++l) total_vertices_ += L_[l].nv;
        LZB_CUDA(cudaStreamSynchronize(s_));
    }

    ~Grid() {
        cudaStreamSynchronize(s_);
        if (a_) cudaStreamSynchronize(a_);
        if (ev_batch_) cudaEventDestroy(ev_batch_);
        if (ev_spawn_) cudaEventDestroy(ev_spawn_);
        if (hres_) cudaFreeHost(hres_);
        if (hhist_) cudaFreeHost(hhist_);
        if (hcycle_) cudaFreeHost(hcycle_);
        if (herr_) cudaFreeHost(herr_);
        for (cudaGraphExec_t* e : {&g_coarse_, &g_front_, &g_back_, &g_front_quiet_, &g_vfront_, &g_vback_, &g_loop_[0], &g_loop_[1]})
            if (*e) cudaGraphExecDestroy(*e);
        if (hloop_) cudaFreeHost(hloop_);
        if (st_ready_) {
            cudaStreamSynchronize(cp_);
            cudaStreamDestroy(cp_);
            cudaFreeHost(hbase_);
            for (int k = 0; k < kBands; ++k) {
                cudaEventDestroy(ev_asm_[k]);
                cudaEventDestroy(ev_pack_[k]);
                cudaEventDestroy(ev_copy_[k]);
            }
            cudaEventDestroy(ev_root_);
            cudaEventDestroy(ev_start_);
        }
    }

    LevelView V(int l) const {
        LevelView v = L_[l].view(D_);
        if (l == D_) {
            v.cw = d_.plane_width;
            v.fixed_p3 = d_.fixed_p3;
        }
        v.geo0 = d_.start_geometric;  // every level: unassembled cells read the eps = 1 stencil
        if (l > 0) v.pdirty = L_[l - 1].dirty.p;  // nullptr unless ripple
        if (uhat_is_u_) v.v[LZB_V_UHAT] = v.v[LZB_V_U];  // V-cycle: u-hat = u without a copy
        return v;
    }
    // 2D launch geometry of the vertex kernels: x = column blocks, y = rows
    dim3 vgrid(int l) const { return dim3(blocks_for(L_[l].N + 1, kThreads), L_[l].N + 1); }
    // k_uhat: one thread per vertex pair of a row
    dim3 ugrid(int l) const { return dim3(blocks_for((L_[l].N + 1) / 2, kThreads), L_[l].N + 1); }
    dim3 ugrid_rows(int l, int r0, int r1) const { return dim3(blocks_for((L_[l].N + 1) / 2, kThreads), r1 - r0); }
    const lzb_grid_desc& desc() const { return d_; }
    lzb_ctx* context() const { return ctx_; }
    int depth() const { return D_; }
    uint32_t cycle() const { return cycle_; }

    void init_noise(uint64_t seed) {
        for (int l = 0; l <= D_; ++l)
            LZB_LAUNCH(k_noise, vgrid(l), kThreads, 0, s_, V(l), l, seed,
                       d_.boundary_value);
        inject();
        sync_check();
    }

    // ------------------------------------------------------ assembly protocol
    int next_n(int n) const {
        int nn = d_.schedule == LZB_SCHEDULE_DOUBLE ? 2 * n : n + 1;
        if (d_.n_max > 0 && nn > d_.n_max) nn = d_.n_max;
        return nn;
    }

    void ensure_tables(int nn) {  // per-n tables; the field and level are fixed per grid
        if (tables_.n == nn && tables_.N == L_[D_].N) return;
        tables_.build(d_.field, L_[D_].N, L_[D_].h, nn, s_);
        if (next_n(nn) != nn && next_n(nn) <= 512) tables_.prefetch(d_.field, L_[D_].N, L_[D_].h, next_n(nn));
    }

    // One batched round of adaptive steps over the selected leaves; returns
    // the number of selected leaves. selector: 0 unconverged, 1 tasks, 2 bottom.
    // Order-preserving compaction of the selected leaves into (list, snap),
    // count and p1 histogram left on the device.
    void compact(cudaStream_t st, int selector, long long key_limit, int32_t* list, int32_t* snap,
                 int* counter, int* blockcnt, unsigned* hist) {
        LevelView F = V(D_);
        LZB_CUDA(cudaMemsetAsync(hist, 0, kNHist * sizeof(unsigned), st));
        const long long* keys = key_limit >= 0 ? keys_.p : nullptr;
        const unsigned nb = blocks_for(leaves_, kCompactThreads);
        LZB_LAUNCH(k_compact_count, nb, kCompactThreads, 0, st, F, selector, keys, key_limit, blockcnt);
        LZB_LAUNCH(k_compact_scan, 1, 1024, 0, st, blockcnt, static_cast<int>(nb), counter);
        LZB_LAUNCH(k_compact_scatter, nb, kCompactThreads, 0, st, F, selector, keys, key_limit, blockcnt, list,
                   snap, hist);
    }

    // ------------------------------------------- concurrent (anarchic) assembly
    // A batch = one adaptive step for every task pending when it starts, on the
    // low-priority assembly stream, outcomes into the staging copy S; it is
    // swapped in (k_commit) by the first cycle that finds its event complete.
    LevelView staging() const {
        LevelView S = V(D_);
        S.op = sop_.p;
        S.p1 = sp1_.p;
        S.n = sn_.p;
        S.p3 = sp3_.p;
        S.epoch = sepoch_.p;
        S.chg = schg_.p;  // publish into staging must not signal the live parents
        return S;
    }

    void launch_batch() {
        LZB_CUDA(cudaEventRecord(ev_spawn_, s_));
        LZB_CUDA(cudaStreamWaitEvent(a_, ev_spawn_, 0));
        compact(a_, 1, -1, alist_.p, asnap_.p, acounter_.p, ablockcnt_.p, ahist_.p);
        // tasks advance in lockstep (all cells start at n = 1, every pending task
        // runs in every batch): the main kernel takes n = batch_n_, the generic
        // kernel any entry that is off the lockstep
        const int n = batch_n_;
        const bool cap = d_.n_max > 0 && n >= d_.n_max;
        const int nn = next_n(n);
        if (!cap && !(atables_.n == nn && atables_.N == L_[D_].N))
        {
            atables_.build(d_.field, L_[D_].N, L_[D_].h, nn, a_);
            if (next_n(nn) != nn && next_n(nn) <= 512) atables_.prefetch(d_.field, L_[D_].N, L_[D_].h, next_n(nn));
        }
        const bool fast = d_.integration == LZB_INTEGRATE_FAST;
        unsigned long long* stats = res_.p->s;
        // geometric start: the first batch holds the deferred bottom -> 1 steps
        const bool bottoms = d_.start_geometric && batches_launched_ == 0;
        if (bottoms)
            LZB_LAUNCH(k_bottom, blocks_for(leaves_, kThreads), kThreads, 0, a_, staging(), d_.field, alist_.p,
                       asnap_.p, static_cast<int>(leaves_), static_cast<const int*>(acounter_.p), d_.delta_max,
                       cycle_, 0, stats, ctx_->err.p);
        dispatch_step(fast, a_, V(D_), staging(), d_.field, alist_.p, asnap_.p, acounter_.p, leaves_, n, nn,
                      cap, atables_.view(), d_.termination_c, d_.delta_max, cycle_, stats, ctx_->err.p);
        LZB_LAUNCH(k_step_generic, blocks_for(leaves_, kThreads), kThreads, 0, a_, V(D_), staging(), d_.field,
                   alist_.p, asnap_.p, acounter_.p, n, d_.schedule, d_.n_max, fast ? 1 : 0, d_.termination_c,
                   d_.delta_max, cycle_, stats, ctx_->err.p);
        LZB_CUDA(cudaEventRecord(ev_batch_, a_));
        batch_inflight_ = true;
        if (!bottoms) batch_n_ = cap ? n : nn;
        ++batches_launched_;
    }

    // Swap in the in-flight batch if it has finished (wait = block until it has).
    bool try_commit(bool wait) {
        if (!batch_inflight_) return false;
        if (!wait) {
            cudaError_t q = cudaEventQuery(ev_batch_);
            if (q == cudaErrorNotReady) return false;
            LZB_CUDA(q);
        }
        LZB_CUDA(cudaStreamWaitEvent(s_, ev_batch_, 0));
        LZB_LAUNCH(k_commit, blocks_for(leaves_, kThreads), kThreads, 0, s_, V(D_), staging(), alist_.p,
                   acounter_.p, cycle_);
        all_top_ = false;
        settled_ = false;
        batch_inflight_ = false;
        ++batches_committed_;
        return true;
    }

    // TaskPool::drain_all (scheduler.cpp:125-141): finish every pending task.
    void drain() {
        if (d_.concurrent) try_commit(true);
        if (ripple_fifo()) ripple_run_fifo(-1);  // the high class first (scheduler.cpp:125-141)
        else if (ripple()) ripple_tasks();
        if (d_.mode == LZB_ANARCHIC || d_.forced_fraction > 0.0) {
            while (count_pending() > 0) round(1, true);
        }
        pending_ = count_pending();
    }

    int64_t round(int selector, bool complete_tasks, long long key_limit = -1) {
        LevelView F = V(D_);
        const double t_round = trace() ? now_ms() : 0.0;
        compact(s_, selector, key_limit, list_.p, snap_.p, counter_.p, blockcnt_.p, hist_.p);
        LZB_CUDA(cudaMemcpyAsync(hhist_, hist_.p, kNHist * sizeof(unsigned), cudaMemcpyDeviceToHost, s_));
        LZB_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(hhist_) + kNHist * sizeof(unsigned),
                                 counter_.p, sizeof(int), cudaMemcpyDeviceToHost, s_));
        sync_check();
        int count = *reinterpret_cast<int*>(reinterpret_cast<char*>(hhist_) + kNHist * sizeof(unsigned));
        if (trace()) std::fprintf(stderr, "[lzb] round: compact + readback %.3f ms, %d leaves\n", now_ms() - t_round, count);
        if (count == 0) return 0;
        if (hhist_[kNHist - 1] && selector != 1)
            throw Error(LZB_ERR_RESOURCE, "sub-sample count beyond 4095 per axis");
        unsigned long long* stats = res_.p->s;
        if (hhist_[0])
            LZB_LAUNCH(k_bottom, blocks_for(count, kThreads), kThreads, 0, s_, F, d_.field, list_.p,
                       snap_.p, count, static_cast<const int*>(nullptr), d_.delta_max, cycle_, 0, stats,
                       ctx_->err.p);
        if (d_.forced_fraction > 0.0 && selector == 1)  // forced tasks: the integration, discarded
            LZB_LAUNCH(k_forced_work, blocks_for(count, 128), 128, 0, s_, F, d_.field, list_.p, snap_.p, count,
                       d_.forced_n, sink_.p);
        for (int n = 1; n < kNHist - 1; ++n) {
            if (!hhist_[n]) continue;
            bool cap = d_.n_max > 0 && n >= d_.n_max;
            int nn = next_n(n);
            const double t_tab = trace() ? now_ms() : 0.0;
            if (!cap) ensure_tables(nn);
            const double t_step = trace() ? now_ms() : 0.0;
            bool fast = d_.integration == LZB_INTEGRATE_FAST;
            const IntTables T = tables_.view();
            dispatch_step(fast, s_, F, F, d_.field, list_.p, snap_.p, counter_.p, count, n, nn, cap, T,
                          d_.termination_c, d_.delta_max, cycle_, stats, ctx_->err.p);
            if (trace()) {
                LZB_CUDA(cudaStreamSynchronize(s_));
                std::fprintf(stderr, "[lzb] round: n %d -> %d: tables %.3f ms, step kernels %.3f ms\n", n, nn,
                             t_step - t_tab, now_ms() - t_step);
            }
        }
        if (complete_tasks)
            LZB_LAUNCH(k_clear_p2, blocks_for(count, kThreads), kThreads, 0, s_, F, list_.p, count);
        return count;
    }

    void eager_setup() {  // assembly.cpp:111-118, batched by rounds
        while (round(0, false) > 0) {
        }
    }

    void assemble_fixed(int n) { assemble_fixed_rows(n, 0, L_[D_].N); }

    // Fixed-p assembly of the leaf cell rows [row0, row1) (a slab of a
    // multi-GPU decomposition: cells are independent, no exchange needed).
    void assemble_fixed_rows(int n, int row0, int row1) {
        if (n < 1) throw Error(LZB_ERR_INVALID, "n must be >= 1");
        if (row0 < 0 || row1 > L_[D_].N || row0 >= row1) throw Error(LZB_ERR_INVALID, "bad row range");
        // the whole level ends at p1 = top only when every row is assembled here
        all_top_ = row0 == 0 && row1 == L_[D_].N;
        ensure_tables(n);
        assemble_rect(n, CellRect{0, L_[D_].N, row0}, static_cast<int64_t>(row1 - row0) * L_[D_].N, s_);
    }

    // Fixed-p assembly launch over the leaf cells of rectangle R (count cells) on stream st (tables ready).
    void assemble_rect(int n, CellRect R, int64_t count, cudaStream_t st) {
        LevelView F = V(D_);
        bool fast = d_.integration == LZB_INTEGRATE_FAST;
        unsigned long long* stats = res_.p->s;
        const IntTables T = tables_.view();
        int* err = ctx_->err.p;
        const double dm = d_.delta_max;
        switch (d_.field.kind) {
            case LZB_FIELD_THETA: launch_fixed<LZB_FIELD_THETA>(fast, st, F, d_.field, n, T, dm, cycle_, stats, err, 0, count, R, raw_); break;
            case LZB_FIELD_QUADRANT: launch_fixed<LZB_FIELD_QUADRANT>(fast, st, F, d_.field, n, T, dm, cycle_, stats, err, 0, count, R, raw_); break;
            case LZB_FIELD_CHECKER: launch_fixed<LZB_FIELD_CHECKER>(fast, st, F, d_.field, n, T, dm, cycle_, stats, err, 0, count, R, raw_); break;
            case LZB_FIELD_SINUSOID: launch_fixed<LZB_FIELD_SINUSOID>(fast, st, F, d_.field, n, T, dm, cycle_, stats, err, 0, count, R, raw_); break;
            default: launch_fixed<LZB_FIELD_CONSTANT>(fast, st, F, d_.field, n, T, dm, cycle_, stats, err, 0, count, R, raw_); break;
        }
    }

    // pre-order semantics: coarse levels first, each reads l+1 (post_order:
    // finest first, each level reads the l+1 written in the same pass -- the
    // V-cycle's consistent Galerkin hierarchy)
    void coarse_pass_order(bool post_order) {
        // the epoch comes from pinned host memory at execution time (graph-replayable)
        // (the device loop's body counts the epoch on the device: k_loop_begin)
        if (!loop_capture_)
            LZB_CUDA(cudaMemcpyAsync(dcycle_.p, hcycle_, sizeof(uint32_t), cudaMemcpyHostToDevice, s_));
        for (int i = 0; i < D_; ++i) {
            const int l = post_order ? D_ - 1 - i : i;
            if (d_.transfer == LZB_BOXMG)
                LZB_LAUNCH(k_coarse, blocks_for(L_[l].nc, 64), 64, 0, s_, V(l), V(l + 1), d_.field, 1,
                           d_.delta_max, dcycle_.p, res_.p->s, ctx_->err.p, static_cast<const int32_t*>(nullptr), 0);
            else
                LZB_LAUNCH(k_coarse_geo, blocks_for(L_[l].nc, kCoarseThreads), kCoarseThreads, 0, s_,
                           V(l), V(l + 1), d_.field, d_.delta_max, dcycle_.p, res_.p->s, ctx_->err.p,
                           static_cast<const int32_t*>(nullptr), 0);
        }
    }
    void coarse_pass() { coarse_pass_order(false); }
    void coarse_pass_post() { coarse_pass_order(true); }

    // ------------------------------------------------------------ CUDA graphs
    // The fixed part of a cycle is replayed as two graphs: (coarse recompute +
    // residual pass + stats + result copy) and (update + prolongation +
    // injection). All kernel arguments are stable per grid; the epoch and the
    // result travel through pinned host memory read/written at replay time.
    struct PdlScope {  // programmatic dependent launches for the cycle bodies
        bool prev;
        PdlScope() : prev(g_pdl) { g_pdl = std::getenv("LZB_NO_PDL") == nullptr; }
        ~PdlScope() { g_pdl = prev; }
    };
    static bool trace() {
        static const bool on = std::getenv("LZB_TRACE") != nullptr;
        return on;
    }
    static double now_ms() {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    }
    void run_graph(cudaGraphExec_t& exec, void (Grid::*body)()) {
        if (!use_graphs_) {
            PdlScope pdl;
            (this->*body)();
            return;
        }
        const int slot = &exec == &g_coarse_ ? 0 : &exec == &g_front_ ? 1 : &exec == &g_back_ ? 2 : &exec == &g_vfront_ ? 3 : &exec == &g_vback_ ? 4 : 5;
        static const char* const kSlotName[6] = {"cycle:coarse", "cycle:front", "cycle:back", "vcycle:down", "vcycle:up", "cycle:graph"};
        LZB_RANGE(kSlotName[slot]);
        if (!exec) {
            cudaGraph_t g = nullptr;
            const uint64_t l0 = g_launches.load();
            const double tb = trace() ? now_ms() : 0.0;
            LZB_CUDA(cudaStreamBeginCapture(s_, cudaStreamCaptureModeThreadLocal));
            try {
                PdlScope pdl;
                (this->*body)();
            } catch (...) {
                cudaStreamEndCapture(s_, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            LZB_CUDA(cudaStreamEndCapture(s_, &g));
            graph_kernels_[slot] = g_launches.load() - l0;  // kernels per replay
            g_launches.fetch_sub(graph_kernels_[slot]);      // counted when they run
            LZB_CUDA(cudaGraphInstantiate(&exec, g, 0));
            LZB_CUDA(cudaGraphDestroy(g));
            if (trace())
                std::fprintf(stderr, "[lzb] graph slot %d: %llu kernels, capture + instantiate %.3f ms\n", slot,
                             static_cast<unsigned long long>(graph_kernels_[slot]), now_ms() - tb);
        }
        LZB_CUDA(cudaGraphLaunch(exec, s_));
        g_launches.fetch_add(graph_kernels_[slot], std::memory_order_relaxed);
    }
    void front_body() {  // residual pass + stats + result / error flag D2H
        residual_launches();
        stats_launches();
        LZB_CUDA(cudaMemcpyAsync(hres_, res_.p, sizeof(Result), cudaMemcpyDeviceToHost, s_));
        LZB_CUDA(cudaMemcpyAsync(herr_, ctx_->err.p, sizeof(int), cudaMemcpyDeviceToHost, s_));
    }
    void front_body_quiet() {  // a settled cycle: the residual pass + result / error flag D2H
        residual_launches();
        LZB_CUDA(cudaMemcpyAsync(hres_, res_.p, sizeof(Result), cudaMemcpyDeviceToHost, s_));
        LZB_CUDA(cudaMemcpyAsync(herr_, ctx_->err.p, sizeof(int), cudaMemcpyDeviceToHost, s_));
    }
    MidRange mid_range(int l0, int l1) const {
        MidRange R{};
        R.l0 = l0;
        R.l1 = l1;
        int64_t at = 0;
        for (int l = l0; l <= l1 + 1 && l < kMaxLevels; ++l) {
            R.start[l] = at;
            if (l <= l1) at += L_[l].nv;
        }
        return R;
    }
    // the fused middle levels (k_mid_*): additive and adaFAC-PI, at least one level
    // between the small levels and the leaves; LZB_PLAIN_BACK=1 keeps the per-level launches
    bool fused_back_ok() const {
        static const bool plain = std::getenv("LZB_PLAIN_BACK") != nullptr;
        return !plain && d_.variant != LZB_ADAFAC_JAC && small_lc() + 1 <= D_ - 1 && D_ + 1 < kMaxLevels;
    }
    void back_body_fused() {
        const int lc = small_lc(), l0 = lc + 1, l1 = D_ - 1;
        const bool pi = d_.variant == LZB_ADAFAC_PI;
        const MidRange R = mid_range(l0, l1);
        const int64_t nmid = R.start[l1 + 1];
        Damp dm{};
        for (int l = 0; l <= D_; ++l) dm.d[l] = damping(l);
        // snapshots of every level below the leaves, the injected residuals of levels lc..D-1
        const MidRange Rs = mid_range(0, l1);
        LZB_LAUNCH(k_mid_snap, blocks_for(Rs.start[l1 + 1], kThreads), kThreads, 0, s_, all_levels(), Rs, pi ? 1 : 0,
                   std::max(lc, 0));
        LZB_LAUNCH(k_mid_update, blocks_for(nmid, kThreads), kThreads, 0, s_, all_levels(), R, pi ? 1 : 0, d_.omega,
                   dm, caux_.p);
        if (lc >= 0)
            LZB_LAUNCH(k_small_back, 1, kSmallThreads, 0, s_, all_levels(), lc, static_cast<int>(d_.variant),
                       d_.omega, dm, d_.field);
        for (int l = std::max(lc, 0) + 1; l <= D_ - 1; ++l)
            LZB_LAUNCH(k_prolong, ugrid(l), kThreads, 0, s_, V(l), V(l - 1));
        LZB_LAUNCH(k_update_fine, vgrid(D_), kThreads, 0, s_, V(D_), V(D_ - 1), pi ? caux_.p : nullptr,
                   damping(D_));
        // injection: levels D-1 .. max(lc, 0) straight from the leaves, then the small levels' chain
        const MidRange Ri = mid_range(std::max(lc, 0), D_ - 1);
        LZB_LAUNCH(k_mid_inject, blocks_for(Ri.start[D_], kThreads), kThreads, 0, s_, all_levels(), Ri);
        if (lc >= 1) LZB_LAUNCH(k_small_inject, 1, kSmallThreads, 0, s_, all_levels(), lc);
    }
    void back_body() {  // update + prolongation + injection
        if (fused_back_ok()) {
            back_body_fused();
            return;
        }
        update_launches(true, true);
        for (int l = std::max(small_lc(), 0) + 1; l <= D_ - 1; ++l)
            LZB_LAUNCH(k_prolong, ugrid(l), kThreads, 0, s_, V(l), V(l - 1));
        const bool pi = d_.variant == LZB_ADAFAC_PI;
        if (pi) LZB_LAUNCH(k_scale_aux, vgrid(D_ - 1), kThreads, 0, s_, V(D_ - 1), d_.omega, caux_.p);
        LZB_LAUNCH(k_update_fine, vgrid(D_), kThreads, 0, s_, V(D_), V(D_ - 1), pi ? caux_.p : nullptr,
                   damping(D_));
        inject();
    }

    // budget: the leaf tasks this begin_cycle may run (the cycle's throttle
    // minus the high-class tasks already run; -1 = unlimited)
    void pool_begin_cycle(int64_t budget = -2) {  // TaskPool::begin_cycle, workers = 1 (scheduler.cpp:88-111)
        if (budget == -2) budget = d_.throttle ? static_cast<int64_t>(d_.throttle) : -1;
        // step tasks (anarchic) and forced tasks (any mode) are the leaf tasks
        const int64_t leaf_pending = pending_ - static_cast<int64_t>(hq_pending_at_report_);
        if (leaf_pending <= 0 || budget == 0 || (d_.mode != LZB_ANARCHIC && d_.forced_fraction <= 0.0)) return;
        long long limit = -1;
        if (budget > 0 && leaf_pending > budget) {
            // FIFO: only the `budget` oldest spawns run this cycle
            std::vector<long long> k(leaves_);
            std::vector<uint8_t> p2(leaves_);
            LZB_CUDA(cudaMemcpyAsync(k.data(), keys_.p, leaves_ * sizeof(long long), cudaMemcpyDeviceToHost, s_));
            LZB_CUDA(cudaMemcpyAsync(p2.data(), L_[D_].p2.p, leaves_, cudaMemcpyDeviceToHost, s_));
            sync_check();
            std::vector<long long> pend;
            for (int64_t c = 0; c < leaves_; ++c)
                if (p2[c]) pend.push_back(k[c]);
            std::nth_element(pend.begin(), pend.begin() + (budget - 1), pend.end());
            limit = pend[budget - 1];
        }
        round(1, true, limit);
    }

    // ---- coarse-recompute = ripple with a throttle: the high class as a real
    // FIFO (TaskPool high_, scheduler.cpp:95-111) on the host -- spawns in
    // pre-order per walk, duplicates allowed, at most `throttle` tasks (high
    // class first) per begin_cycle. A batch runs in dependency generations
    // (a task waits for an earlier one on the same cell, its parent or a
    // child: it reads the children's operators), one launch per generation
    // and level over the listed cells.
    static int32_t task_code(int l, int64_t c) { return static_cast<int32_t>((l << 27) | c); }
    void build_preorder() {  // the walk order of the refined cells (solver.cpp:79-97, mesh.cpp:140-157)
        preorder_.clear();
        std::vector<std::array<int, 3>> st{{0, 0, 0}};
        while (!st.empty()) {
            auto [l, cx, cy] = st.back();
            st.pop_back();
            if (l >= D_) continue;
            preorder_.push_back(task_code(l, static_cast<int64_t>(cy) * L_[l].N + cx));
            for (int k = 8; k >= 0; --k)  // child lx * 3 + ly, pushed in reverse
                st.push_back({l + 1, 3 * cx + k / 3, 3 * cy + k % 3});
        }
    }
    // after the walk's take_dirty launches: the flagged cells, in pre-order, join the FIFO
    void ripple_spawn_fifo() {
        if (preorder_.empty()) build_preorder();
        std::vector<std::vector<uint8_t>> fl(D_);
        for (int l = 0; l < D_; ++l) {
            fl[l].resize(L_[l].nc);
            LZB_CUDA(cudaMemcpyAsync(fl[l].data(), L_[l].pend.p, L_[l].nc, cudaMemcpyDeviceToHost, s_));
        }
        sync_check();
        for (int32_t code : preorder_) {
            const int l = code >> 27;
            if (fl[l][code & ((1 << 27) - 1)]) hq_.push_back(code);
        }
        for (int l = 0; l < D_; ++l) LZB_CUDA(cudaMemsetAsync(L_[l].pend.p, 0, L_[l].nc, s_));
    }
    // the first `budget` FIFO tasks (-1: all); returns how many ran
    int64_t ripple_run_fifo(int64_t budget) {
        const int64_t k = budget < 0 ? static_cast<int64_t>(hq_.size())
                                     : std::min<int64_t>(budget, static_cast<int64_t>(hq_.size()));
        if (k == 0) return 0;
        std::vector<int32_t> batch(hq_.begin(), hq_.begin() + k);
        hq_.erase(hq_.begin(), hq_.begin() + k);
        std::unordered_map<int32_t, int> gen_of;
        std::vector<int> gen(k);
        int ngen = 0;
        for (int64_t i = 0; i < k; ++i) {
            const int l = batch[i] >> 27;
            const int64_t c = batch[i] & ((1 << 27) - 1);
            const int cx = static_cast<int>(c % L_[l].N), cy = static_cast<int>(c / L_[l].N);
            int g = 0;
            auto dep = [&](int32_t code) {
                auto it = gen_of.find(code);
                if (it != gen_of.end()) g = std::max(g, it->second + 1);
            };
            dep(batch[i]);
            if (l > 0) dep(task_code(l - 1, static_cast<int64_t>(cy / 3) * L_[l - 1].N + cx / 3));
            if (l + 1 < D_)
                for (int k9 = 0; k9 < 9; ++k9)
                    dep(task_code(l + 1, static_cast<int64_t>(3 * cy + k9 % 3) * L_[l + 1].N + 3 * cx + k9 / 3));
            gen[i] = g;
            gen_of[batch[i]] = g;
            ngen = std::max(ngen, g + 1);
        }
        *hcycle_ = cycle_;
        LZB_CUDA(cudaMemcpyAsync(dcycle_.p, hcycle_, sizeof(uint32_t), cudaMemcpyHostToDevice, s_));
        std::vector<int32_t> cells;
        DevBuf<int32_t> dcells(static_cast<size_t>(k));
        for (int g = 0; g < ngen; ++g)
            for (int l = 0; l < D_; ++l) {
                cells.clear();
                for (int64_t i = 0; i < k; ++i)
                    if (gen[i] == g && (batch[i] >> 27) == l) cells.push_back(batch[i] & ((1 << 27) - 1));
                if (cells.empty()) continue;
                LZB_CUDA(cudaMemcpyAsync(dcells.p, cells.data(), cells.size() * sizeof(int32_t),
                                         cudaMemcpyHostToDevice, s_));
                const int n = static_cast<int>(cells.size());
                if (d_.transfer == LZB_BOXMG)
                    LZB_LAUNCH(k_coarse, blocks_for(n, 64), 64, 0, s_, V(l), V(l + 1), d_.field, 1, d_.delta_max,
                               dcycle_.p, res_.p->s, ctx_->err.p, static_cast<const int32_t*>(dcells.p), n);
                else
                    LZB_LAUNCH(k_coarse_geo, blocks_for(n, kCoarseThreads), kCoarseThreads, 0, s_, V(l), V(l + 1),
                               d_.field, d_.delta_max, dcycle_.p, res_.p->s, ctx_->err.p,
                               static_cast<const int32_t*>(dcells.p), n);
                LZB_CUDA(cudaStreamSynchronize(s_));  // dcells is reused by the next launch
            }
        return k;
    }
    bool ripple_fifo() const { return d_.policy == LZB_RIPPLE && d_.throttle > 0; }
    std::deque<int32_t> hq_;        // pending coarse_recompute tasks (throttled ripple)
    std::vector<int32_t> preorder_;  // refined cells in walk order
    uint64_t hq_pending_at_report_ = 0;

    bool ripple() const { return d_.policy == LZB_RIPPLE; }

    // The high-priority class of TaskPool::begin_cycle (scheduler.cpp:95-111):
    // every pending coarse_recompute task, in pre-order = level by level from
    // the root (siblings are independent; a task reads its children before
    // their own pending recompute, as the pre-order FIFO does).
    void ripple_tasks() {
        *hcycle_ = cycle_;
        LZB_CUDA(cudaMemcpyAsync(dcycle_.p, hcycle_, sizeof(uint32_t), cudaMemcpyHostToDevice, s_));
        for (int l = 0; l < D_; ++l) {
            if (d_.transfer == LZB_BOXMG)
                LZB_LAUNCH(k_coarse, blocks_for(L_[l].nc, 64), 64, 0, s_, V(l), V(l + 1), d_.field, 1, d_.delta_max,
                           dcycle_.p, res_.p->s, ctx_->err.p, static_cast<const int32_t*>(nullptr), 0);
            else
                LZB_LAUNCH(k_coarse_geo, blocks_for(L_[l].nc, kCoarseThreads), kCoarseThreads, 0, s_, V(l), V(l + 1),
                           d_.field, d_.delta_max, dcycle_.p, res_.p->s, ctx_->err.p,
                           static_cast<const int32_t*>(nullptr), 0);
        }
    }
    // The walk's refined cells under ripple: take_dirty -> spawn (solver.cpp:86-90).
    void ripple_walk() {
        for (int l = 0; l < D_; ++l)
            LZB_LAUNCH(k_take_dirty, blocks_for(L_[l].nc, kThreads), kThreads, 0, s_, V(l), cycle_);
    }
    void begin_cycle_tasks() {
        if (ripple_fifo()) {
            const int64_t ran = ripple_run_fifo(static_cast<int64_t>(d_.throttle));
            pool_begin_cycle(static_cast<int64_t>(d_.throttle) - ran);
            return;
        }
        if (ripple()) ripple_tasks();
        pool_begin_cycle();
    }

    void assembly_pass() {  // solver.cpp:79-97
        *hcycle_ = cycle_;
        if (ripple()) {
            ripple_walk();
            if (ripple_fifo()) ripple_spawn_fifo();
        } else {
            coarse_pass();
        }
        leaves_pass();
    }

    // request_stencil over every leaf, mode by mode (assembly.cpp:76-109). Once a
    // round has found every leaf converged (p1 = top) nothing can change until a
    // publish / load / adaptive_step, so the compaction is skipped.
    void leaves_pass() {
        // adaptive_sync request_stencil runs queued work while the cell's task is
        // in flight (assembly.cpp:86-93): every queued task (only forced tasks
        // exist in this mode) has run by the end of the pass, and none changes a
        // marker, so they run first
        if (d_.mode == LZB_ADAPTIVE && d_.forced_fraction > 0.0) round(1, true);
        if (all_top_) return;
        switch (d_.mode) {
            case LZB_EAGER:
            case LZB_LAZY:
                while (round(0, false) > 0) {
                }
                all_top_ = true;
                break;
            case LZB_ADAPTIVE:
                if (round(0, false) == 0) all_top_ = true;
                break;
            case LZB_ANARCHIC:
                // the initial stencil computation is not deferred (assembly.cpp:98-103),
                // unless the grid starts from the geometric stencil
                if (!d_.start_geometric) round(2, false);
                LZB_LAUNCH(k_spawn, blocks_for(leaves_, kThreads), kThreads, 0, s_, V(D_), cycle_,
                           static_cast<long long>(leaves_), keys_.p);
                break;
        }
    }

    // init_level_rhs on the leaf level (solver.cpp:99-118). The lumped load is
    // a fixed vector (the restriction only writes coarser levels), so it is
    // computed once, outside the replayed cycle graphs; writing the leaf fl
    // through lzb_grid_vertices invalidates it.
    void ensure_rhs() {
        if (rhs_ready_) return;
        const bool rhs_on = d_.rhs.kind == LZB_RHS_SINPROD || d_.rhs.value != 0.0;
        if (rhs_on)
            LZB_LAUNCH(k_init_rhs, vgrid(D_), kThreads, 0, s_, V(D_), d_.rhs, L_[D_].h * L_[D_].h / 4.0);
        else
            LZB_CUDA(cudaMemsetAsync(L_[D_].v[LZB_V_FL].p, 0, L_[D_].v[LZB_V_FL].bytes(), s_));
        rhs_ready_ = true;
    }

    // The leaf level's residual on rows [r0, r1): FP64 operators, or the
    // compressed records when plane_width > 0.
    void leaf_residual(int r0, int r1) {
        const dim3 g = vgrid_rows(D_, r0, r1);
        const LevelView F = Vrow(D_, r0);
        const double *cx = centre_[1].x.p, *cy = centre_[1].y.p;
        static const bool plain = std::getenv("LZB_PLAIN_COMP") != nullptr;
        // staged cell-centric kernel: tiles of 31 x 7 vertices over rows [r0, r1)
        const dim3 gs((L_[D_].N + 1 + kCsX - 2) / (kCsX - 1), (r1 - r0 + kCsY - 2) / (kCsY - 1));
        const LevelView Fw = V(D_);
        auto comp = [&](auto gather, auto staged) {
            if (plain) LZB_LAUNCH(gather, g, kThreads, 0, s_, F, d_.field, cx, cy);
            else LZB_LAUNCH(staged, gs, kCsX * kCsY, 0, s_, Fw, d_.field, cx, cy, r0, r1);
        };
        switch (d_.plane_width) {
            case 0: LZB_LAUNCH(k_residual, g, kThreads, 0, s_, F, d_.field); break;
            case 2: comp(k_residual_comp<2>, k_residual_comp_st<2>); break;
            case 3: comp(k_residual_comp<3>, k_residual_comp_st<3>); break;
            case 4: comp(k_residual_comp<4>, k_residual_comp_st<4>); break;
            case 5: comp(k_residual_comp<5>, k_residual_comp_st<5>); break;
            case 6: comp(k_residual_comp<6>, k_residual_comp_st<6>); break;
            case 7: comp(k_residual_comp<7>, k_residual_comp_st<7>); break;
            case 8:
            // W = 8: a slot row is as wide as the FP64 row, which the residual reads
            default: LZB_LAUNCH(k_residual, g, kThreads, 0, s_, F, d_.field); break;
        }
    }

    // levels 0..small_lc() run fused in one block (k_small_*); -1: none
    int small_lc() const {
        static const int maxn = std::getenv("LZB_SMALL_MAXN") ? std::atoi(std::getenv("LZB_SMALL_MAXN")) : kSmallMaxN;
        int lc = -1;
        while (lc + 1 <= D_ - 1 && L_[lc + 1].N <= maxn) ++lc;
        return lc;
    }

    void residual_launches() {  // solver.cpp:145-210
        const int lc = small_lc();
        static const bool plain = std::getenv("LZB_PLAIN_BACK") != nullptr;
        const bool mid = !plain && lc + 1 <= D_ - 1 && D_ + 1 < kMaxLevels;  // one launch for the middle levels' u-hat
        if (mid) {
            const MidRange R = mid_range(lc + 1, D_ - 1);
            LZB_LAUNCH(k_mid_uhat, blocks_for(R.start[D_], kThreads), kThreads, 0, s_, all_levels(), R);
        }
        for (int l = D_; l > lc; --l) {
            const dim3 g = vgrid(l);
            if (!mid || l == D_)
                LZB_LAUNCH(k_uhat, ugrid(l), kThreads, 0, s_, V(l), l > 0 ? V(l - 1) : V(l), l > 0 ? 1 : 0);
            if (l == D_) leaf_residual(0, L_[D_].N + 1);
            else LZB_LAUNCH(k_residual, g, kThreads, 0, s_, V(l), d_.field);
            if (l > 0)
                LZB_LAUNCH(k_restrict, vgrid(l - 1), kThreads, 0, s_, V(l),
                           V(l - 1), 0, 0.0);
        }
        if (lc >= 0) LZB_LAUNCH(k_small_front, 1, kSmallThreads, 0, s_, all_levels(), lc, d_.field);
        LZB_LAUNCH(k_norm_partial, kNormBlocks, kThreads, 0, s_, V(D_), 0, L_[D_].N + 1, partial_.p);
        LZB_LAUNCH(k_norm_final, 1, kNormFinalThreads, 0, s_, partial_.p, kNormBlocks, res_.p);
    }

    void stats_launches() {
        LZB_LAUNCH(k_reset_stats, 1, 32, 0, s_, res_.p);
        for (int l = 0; l <= D_; ++l)
            LZB_LAUNCH(k_stats, static_cast<unsigned>(std::min<int64_t>(blocks_for(L_[l].nc, kThreads), kStatsBlocks)),
                       kThreads, 0, s_, V(l), l == D_ ? 1 : 0, res_.p->s);
    }

    double damping(int l) const {
        return d_.variant == LZB_ADDITIVE ? std::pow(d_.omega, D_ - l + 1) : d_.omega;
    }

    // fuse_fine: the leaf level's Jacobi step (and, for adaFAC-PI, its aux
    // correction) is left to k_update_fine at the end of the back graph.
    // small: levels 0..small_lc() in k_small_snap / k_small_back, which also
    // prolongates levels 1..small_lc() (the caller prolongates the rest).
    void update_launches(bool fuse_fine = false, bool small = false) {  // solver.cpp:212-313
        const double omega = d_.omega;
        const int lc = small ? small_lc() : -1;
        // usnap / aux of the leaf level are never read (prolongation reads the
        // coarse snapshots; adaFAC-Jac rewrites the leaf aux before use)
        if (lc >= 0) LZB_LAUNCH(k_small_snap, 1, kSmallThreads, 0, s_, all_levels(), lc);
        for (int l = lc + 1; l < D_; ++l)
            LZB_LAUNCH(k_snap, blocks_for(L_[l].nv, kThreads), kThreads, 0, s_, V(l));
        for (int l = D_; l > lc; --l) {
            bool aux = d_.variant != LZB_ADDITIVE && l > 0;
            const dim3 g = vgrid(l);
            if (aux) {
                const dim3 gc = vgrid(l - 1);
                if (d_.variant == LZB_ADAFAC_PI) {
                    LZB_LAUNCH(k_aux_inject, gc, kThreads, 0, s_, V(l), V(l - 1));
                } else {
                    LZB_LAUNCH(k_aux_Ar, g, kThreads, 0, s_, V(l), d_.field);
                    LZB_LAUNCH(k_restrict, gc, kThreads, 0, s_, V(l), V(l - 1), 1, omega);
                }
                if (!(fuse_fine && l == D_ && d_.variant == LZB_ADAFAC_PI))
                    LZB_LAUNCH(k_aux_sub, g, kThreads, 0, s_, V(l), V(l - 1), omega);
            }
            if (!(fuse_fine && l == D_)) LZB_LAUNCH(k_jacobi, g, kThreads, 0, s_, V(l), damping(l));
        }
        if (lc >= 0) {
            Damp dm{};
            for (int l = 0; l <= lc; ++l) dm.d[l] = damping(l);
            LZB_LAUNCH(k_small_back, 1, kSmallThreads, 0, s_, all_levels(), lc, static_cast<int>(d_.variant), omega,
                       dm, d_.field);
        }
    }

    void prolong_launches(int lmax = -1) {
        if (lmax < 0) lmax = D_;
        for (int l = 1; l <= lmax; ++l)
            LZB_LAUNCH(k_prolong, ugrid(l), kThreads, 0, s_, V(l), V(l - 1));
    }

    void inject() {
        const int lc = small_lc();
        for (int l = D_; l >= std::max(lc, 0) + 1; --l)
            LZB_LAUNCH(k_inject, vgrid(l - 1), kThreads, 0, s_, V(l), V(l - 1));
        if (lc >= 1) LZB_LAUNCH(k_small_inject, 1, kSmallThreads, 0, s_, all_levels(), lc);
    }

    void fetch_result() {
        LZB_CUDA(cudaMemcpyAsync(hres_, res_.p, sizeof(Result), cudaMemcpyDeviceToHost, s_));
        sync_check();
    }

    void sync_check() {
        LZB_CUDA(cudaStreamSynchronize(s_));
        int flag = 0;
        LZB_CUDA(cudaMemcpy(&flag, ctx_->err.p, sizeof(int), cudaMemcpyDeviceToHost));
        if (flag) {
            LZB_CUDA(cudaMemset(ctx_->err.p, 0, sizeof(int)));
            throw Error(LZB_ERR_PROTOCOL, "cannot encode non-finite operator entry");
        }
    }

    int64_t count_pending() {
        LZB_CUDA(cudaMemsetAsync(counter_.p, 0, sizeof(int), s_));
        // reuse hist_ slot 0 as a 64-bit counter area
        LZB_CUDA(cudaMemsetAsync(hist_.p, 0, 2 * sizeof(unsigned), s_));
        LZB_LAUNCH(k_count_p2, blocks_for(leaves_, kThreads), kThreads, 0, s_, V(D_),
                   reinterpret_cast<unsigned long long*>(hist_.p));
        unsigned long long v = 0;
        LZB_CUDA(cudaMemcpyAsync(&v, hist_.p, sizeof v, cudaMemcpyDeviceToHost, s_));
        sync_check();
        return static_cast<int64_t>(v);
    }

    void fill_stats(const Result& r, lzb_compression_stats& st) const {
        std::memset(&st, 0, sizeof st);
        st.fine_cells = static_cast<uint64_t>(leaves_);
        st.fine_stored_bytes = r.s[S_FINE_BYTES];
        st.fine_uncompressed_bytes = 128ull * leaves_;
        double ratio_sum = 0.0;
        for (int p = 0; p <= 8; ++p) {
            st.p3_histogram[p] = r.s[S_HIST + p];
            ratio_sum += static_cast<double>(r.s[S_HIST + p]) * (128.0 / (p == 0 ? 1.0 : 1.0 + 16.0 * p));
        }
        st.max_n = static_cast<int32_t>(r.s[S_MAXN]);
        if (st.fine_cells) {
            st.fine_factor_totals = static_cast<double>(st.fine_uncompressed_bytes) /
                                    static_cast<double>(st.fine_stored_bytes);
            st.fine_factor_mean = ratio_sum / static_cast<double>(st.fine_cells);
            long double nsum = static_cast<long double>(r.s[S_NSUM]);
            st.avg_n = static_cast<double>(nsum / st.fine_cells);
        }
        st.total_stored_bytes = r.s[S_TOTAL_BYTES];
        uint64_t unc = 0;
        for (int l = 0; l <= D_; ++l) unc += 8ull * (l == D_ ? 16 : 144) * L_[l].nc;
        st.total_uncompressed_bytes = unc;
        if (st.total_stored_bytes)
            st.total_factor = static_cast<double>(unc) / static_cast<double>(st.total_stored_bytes);
        double md;
        std::memcpy(&md, &r.s[S_MAXDELTA], sizeof md);
        st.max_delta = md;
        st.max_sample_count = static_cast<int32_t>(r.s[S_MAXSAMPLES]);
    }

    lzb_compression_stats stats() {
        stats_launches();
        fetch_result();
        lzb_compression_stats st;
        fill_stats(*hres_, st);
        return st;
    }

    int check_termination() const {  // solver.cpp:8-16
        if (history_.empty()) return LZB_CONTINUE;
        double normalized = history_.back() / history_.front();
        if (normalized <= d_.target) return LZB_CONVERGED;
        if (normalized >= d_.divergence) return LZB_DIVERGED;
        if (static_cast<int>(cycle_) >= d_.max_cycles) return LZB_TIMEOUT;
        return LZB_CONTINUE;
    }

    lzb_cycle_report step() {  // solver.cpp:349-400
        auto t0 = std::chrono::steady_clock::now();
        lzb_cycle_report rep;
        std::memset(&rep, 0, sizeof rep);
        ++cycle_;
        *hcycle_ = cycle_;
        // calm: nothing of the assembly side can act in this cycle (every leaf
        // at its top, no task pending or in flight). A calm cycle whose coarse
        // pass recomputed nothing leaves every operator, marker and epoch as it
        // found them, so the next calm cycle's coarse pass and stats are no-ops
        // with the same outcome: settled_ cycles skip both (the stats slots of
        // the device result keep their values).
        const bool calm = quiescent();
        const bool quiet = calm && settled_ && use_graphs_;
        if (!quiet) {
            if (d_.concurrent) try_commit(false);  // swap in a finished batch before the walk
            else begin_cycle_tasks();
        }
        rep.cycle = static_cast<int32_t>(cycle_);
        if (d_.forced_fraction > 0.0) {  // on_cycle_start (experiment.cpp:260-270)
            long long id0 = 0;
            for (int l = 0; l < D_; ++l) id0 += L_[l].nc;
            LZB_LAUNCH(k_spawn_forced, blocks_for(leaves_, kThreads), kThreads, 0, s_, V(D_), cycle_,
                       static_cast<long long>(leaves_), keys_.p, id0, d_.forced_fraction);
        }
        if (quiet) {
            ensure_rhs();
            run_graph(g_front_quiet_, &Grid::front_body_quiet);  // residual + result/error copy-out
        } else {
            if (ripple()) {
                ripple_walk();
                if (ripple_fifo()) ripple_spawn_fifo();
            } else {
                run_graph(g_coarse_, &Grid::coarse_pass);
            }
            leaves_pass();
            if (d_.concurrent && !batch_inflight_ && (cycle_ == 1 || pending_ > 0)) launch_batch();
            ensure_rhs();
            run_graph(g_front_, &Grid::front_body);  // residual + stats + result/error copy-out
        }
        LZB_CUDA(cudaStreamSynchronize(s_));
        if (*herr_) {
            LZB_CUDA(cudaMemset(ctx_->err.p, 0, sizeof(int)));
            *herr_ = 0;
            throw Error(LZB_ERR_PROTOCOL, "cannot encode non-finite operator entry");
        }
        Result r = *hres_;
        if (front_report(rep, r)) run_graph(g_back_, &Grid::back_body);  // update + prolongation + injection
        finish_report(rep, r);
        settled_ = calm && quiescent() && (quiet || r.s[S_COARSE_ACTIVE] != cycle_);
        LZB_CUDA(cudaStreamSynchronize(s_));
        rep.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return rep;
    }

    // A multiplicative V(nu, nu) cycle on the same levels (BASELINE configs[1]
    // names V(1,1); the reference has only the additive cycle, so this is a
    // restated extension, oracle/port2v.py): the coarse operators are brought
    // up to date (the coarse pass finest level first, so every level is the
    // Galerkin product of the current level below it -- the additive cycle's
    // pre-order pass lags one level per cycle, which a multiplicative cycle
    // does not tolerate; ripple mode: the ripple walk; no leaf assembly
    // tasks), then per level from the leaves nu damped-Jacobi sweeps (omega),
    // the residual restricted into the next level's rhs (k_restrict mode 0,
    // the owned-lattice P^T of the additive cycle) with a zero start; at the
    // bottom back up, u_l += P u_{l-1} (k_prolong against a zero snapshot)
    // and nu sweeps. The report's residual is the leaf residual before the cycle.
    lzb_cycle_report vcycle(int nu) {
        if (nu < 0) throw Error(LZB_ERR_INVALID, "nu must be >= 0");
        if (d_.concurrent) throw Error(LZB_ERR_INVALID, "vcycle is not available with concurrent assembly");
        auto t0 = std::chrono::steady_clock::now();
        lzb_cycle_report rep;
        std::memset(&rep, 0, sizeof rep);
        ++cycle_;
        *hcycle_ = cycle_;
        rep.cycle = static_cast<int32_t>(cycle_);
        if (ripple()) {
            ripple_walk();
            if (ripple_fifo()) ripple_spawn_fifo();
        }
        ensure_rhs();
        run_graph(g_vfront_, &Grid::vfront_body);  // (coarse pass) + leaf residual + norm -> host
        LZB_CUDA(cudaStreamSynchronize(s_));
        rep.residual = hres_->norm;
        if (first_residual_ < 0.0) first_residual_ = rep.residual > 0.0 ? rep.residual : 1.0;
        rep.normalized = rep.residual / first_residual_;
        history_.push_back(rep.residual);
        rep.status = check_termination();
        if (rep.status == LZB_CONTINUE || rep.status == LZB_TIMEOUT) {
            if (nu != vnu_ && g_vback_) {  // the sweep counts are baked into the graph
                LZB_CUDA(cudaGraphExecDestroy(g_vback_));
                g_vback_ = nullptr;
            }
            vnu_ = nu;
            run_graph(g_vback_, &Grid::vback_body);
            const uint64_t Nf = static_cast<uint64_t>(L_[D_].N);
            rep.dof_updates = static_cast<uint64_t>(2 * nu) * (Nf - 1) * (Nf - 1);
            for (int l = 0; l < D_; ++l) {
                const uint64_t N = static_cast<uint64_t>(L_[l].N);
                rep.coarse_updates += N > 1 ? static_cast<uint64_t>(2 * nu) * (N - 1) * (N - 1) : 0;
            }
        }
        dof_total_ += rep.dof_updates;
        rep.dof_updates_total = dof_total_;
        rep.levels = D_ + 1;
        rep.cells = static_cast<uint64_t>(total_cells_);
        for (int l = 0; l <= D_ && l < 32; ++l) rep.enabled_mask |= 1u << l;
        const uint64_t Nf = static_cast<uint64_t>(L_[D_].N);
        rep.dofs_fine_interior = (Nf - 1) * (Nf - 1);
        rep.grid_points_total = static_cast<uint64_t>(total_vertices_);
        sync_check();
        rep.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return rep;
    }
    // r, r-hat (= r: the views alias u-hat to u) and the diagonal of level l
    void vresidual(int l) {
        if (l == D_) leaf_residual(0, L_[D_].N + 1);
        else LZB_LAUNCH(k_residual, vgrid(l), kThreads, 0, s_, V(l), d_.field);
    }
    void vsmooth(int l, int k) {
        for (int i = 0; i < k; ++i) {
            vresidual(l);
            LZB_LAUNCH(k_jacobi, vgrid(l), kThreads, 0, s_, V(l), d_.omega);
        }
    }
    void vfront_body() {
        if (!ripple()) coarse_pass_post();
        {
            UhatAlias alias(uhat_is_u_);
            vresidual(D_);
        }
        LZB_LAUNCH(k_norm_partial, kNormBlocks, kThreads, 0, s_, V(D_), 0, L_[D_].N + 1, partial_.p);
        LZB_LAUNCH(k_norm_final, 1, kNormFinalThreads, 0, s_, partial_.p, kNormBlocks, res_.p);
        LZB_CUDA(cudaMemcpyAsync(hres_, res_.p, sizeof(Result), cudaMemcpyDeviceToHost, s_));
    }
    struct UhatAlias {  // scoped: V(l) views alias u-hat to u
        bool& f;
        explicit UhatAlias(bool& x) : f(x) { f = true; }
        ~UhatAlias() { f = false; }
    };
    void vback_body() {
        UhatAlias alias(uhat_is_u_);
        // levels lc..0 (at most 10^2 vertices each) run the bottom of the V in one block
        static const bool plain = std::getenv("LZB_PLAIN_VSMALL") != nullptr;
        const int lc = plain ? 0 : std::max(small_lc(), 0);
        for (int l = D_; l > lc; --l) {
            vsmooth(l, vnu_);
            vresidual(l);
            LZB_LAUNCH(k_restrict, vgrid(l - 1), kThreads, 0, s_, V(l), V(l - 1), 0, 0.0);  // fl = P^T r
            LZB_CUDA(cudaMemsetAsync(L_[l - 1].v[LZB_V_U].p, 0, L_[l - 1].v[LZB_V_U].bytes(), s_));
        }
        if (lc >= 1) LZB_LAUNCH(k_small_v, 1, kSmallThreads, 0, s_, all_levels(), lc, vnu_, d_.omega, d_.field);
        for (int l = lc + 1; l <= D_; ++l) {
            LZB_CUDA(cudaMemsetAsync(L_[l - 1].v[LZB_V_USNAP].p, 0, L_[l - 1].v[LZB_V_USNAP].bytes(), s_));
            LZB_LAUNCH(k_prolong, ugrid(l), kThreads, 0, s_, V(l), V(l - 1));
            vsmooth(l, vnu_);
        }
        // the coarse u held corrections: restore the additive cycle's invariant
        // (coarse u = injected fine u, finish_cycle_sync solver.cpp:344-347) so a
        // later step() forms u-hat = u - P u_c from the solution, not from them
        inject();
    }

    // step() bookkeeping after the residual pass (solver.cpp:359-370): history,
    // normalisation, termination; true when the update passes run.
    bool front_report(lzb_cycle_report& rep, const Result& r) {
        rep.residual = r.norm;
        if (first_residual_ < 0.0) first_residual_ = rep.residual > 0.0 ? rep.residual : 1.0;
        rep.normalized = rep.residual / first_residual_;
        history_.push_back(rep.residual);
        rep.status = check_termination();
        const bool update = rep.status == LZB_CONTINUE || rep.status == LZB_TIMEOUT;
        if (update) {
            uint64_t Nf = static_cast<uint64_t>(L_[D_].N);
            rep.dof_updates = (Nf - 1) * (Nf - 1);
            for (int l = 0; l < D_; ++l) {
                uint64_t N = static_cast<uint64_t>(L_[l].N);
                rep.coarse_updates += N > 1 ? (N - 1) * (N - 1) : 0;
            }
        }
        return update;
    }

    // step() telemetry after the cycle (solver.cpp:371-400).
    void finish_report(lzb_cycle_report& rep, const Result& r) {
        dof_total_ += rep.dof_updates;
        rep.dof_updates_total = dof_total_;
        // leaf tasks (anarchic p2) + pending coarse_recompute tasks (ripple)
        pending_ = static_cast<int64_t>(r.s[S_PENDING]) + static_cast<int64_t>(hq_.size());
        hq_pending_at_report_ = hq_.size();
        // anarchic: no task pending and nothing bottom means every leaf is top
        // (request_stencil spawns a task for every other leaf)
        if (d_.mode == LZB_ANARCHIC && pending_ == 0 && !batch_inflight_) all_top_ = true;
        rep.pending_tasks = static_cast<uint64_t>(pending_);
        lzb_compression_stats st;
        fill_stats(r, st);
        rep.max_n = st.max_n;
        rep.avg_n = st.avg_n;
        rep.max_samples = st.max_sample_count;
        rep.factor_totals = st.fine_factor_totals;
        rep.factor_mean = st.fine_factor_mean;
        rep.levels = D_ + 1;
        rep.cells = static_cast<uint64_t>(total_cells_);
        for (int l = 0; l <= D_ && l < 32; ++l) rep.enabled_mask |= 1u << l;
        uint64_t Nf = static_cast<uint64_t>(L_[D_].N);
        rep.dofs_fine_interior = (Nf - 1) * (Nf - 1);
        rep.grid_points_total = static_cast<uint64_t>(total_vertices_);
    }

    // ------------------------------------------------ slab-distributed cycle
    // SURVEY.md §8e. The leaf level is cut into slabs of vertex rows [v0, v1)
    // (multiples of 3, so every level-(D-1) vertex row 3*IY belongs to one
    // slab); the coarse levels are small (1/8 of the leaf work together) and
    // run replicated. One cycle = phases 0..5 with exchanges in between, done
    // by the host layer (paper_2005_03606_b200/parallel.py, NCCL):
    //   0  cycle start, coarse recompute, leaf û (slab +-1 row), residual,
    //      norm^2 partial, leaf stats of the slab     -> r̂ halo (3 rows)
    //   1  restriction into level D-1, owned rows       -> all-gather fl_{D-1}
    //   2  residual pass of levels D-1..0, result to host -> all-reduce, report
    //   3  snapshots, adaFAC-PI injection into aux_{D-1} -> all-gather aux_{D-1}
    //   4  coarse updates, prolongation to D-1, fused leaf update of the slab,
    //      injection into u_{D-1}                      -> all-gather u_{D-1}
    //   5  injections D-1..1                           -> u halo (1 row)
    // Every vertex value is computed by the same kernel in the same order as
    // on one GPU, so u, r, fl are bit-identical; only the norm sum is regrouped.
    void set_slab(int v0, int v1) {
        const int NV = L_[D_].N + 1;
        if (D_ < 1) throw Error(LZB_ERR_INVALID, "slabs need depth >= 1");
        if (v0 < 0 || v1 > NV || v0 >= v1) throw Error(LZB_ERR_INVALID, "bad slab rows");
        if (v0 % 3 != 0 || (v1 % 3 != 0 && v1 != NV)) throw Error(LZB_ERR_INVALID, "slab rows must be multiples of 3");
        if (d_.variant == LZB_ADAFAC_JAC)
            throw Error(LZB_ERR_INVALID, "the distributed cycle supports additive and adafac-pi");
        if (d_.concurrent) throw Error(LZB_ERR_INVALID, "the distributed cycle runs the deterministic modes");
        slab_v0_ = v0;
        slab_v1_ = v1;
    }
    LevelView Vrow(int l, int r0) const {
        LevelView v = V(l);
        v.row0 = r0;
        return v;
    }
    dim3 vgrid_rows(int l, int r0, int r1) const { return dim3(blocks_for(L_[l].N + 1, kThreads), r1 - r0); }

    void dist_phase(int phase, int flags) {
        const int N = L_[D_].N, v0 = slab_v0_, v1 = slab_v1_ < 0 ? N + 1 : slab_v1_;
        const int c0 = v0 / 3, c1 = (v1 + 2) / 3;
        switch (phase) {
            case 0: {
                dist_t0_ = std::chrono::steady_clock::now();
                ++cycle_;
                *hcycle_ = cycle_;
                pool_begin_cycle();
                run_graph(g_coarse_, &Grid::coarse_pass);
                leaves_pass();
                ensure_rhs();
                const int u0 = std::max(v0 - 1, 0), u1 = std::min(v1 + 1, N + 1);
                LZB_LAUNCH(k_uhat, ugrid_rows(D_, u0, u1), kThreads, 0, s_, Vrow(D_, u0), V(D_ - 1), 1);
                leaf_residual(v0, v1);
                LZB_LAUNCH(k_reset_stats, 1, 32, 0, s_, res_.p);
                const int cr1 = std::min(v1, N);
                if (cr1 > v0)
                    LZB_LAUNCH(k_stats, static_cast<unsigned>(kStatsBlocks), kThreads, 0, s_, V(D_), 1, res_.p->s,
                               static_cast<int64_t>(v0) * N, static_cast<int64_t>(cr1) * N);
                if (flags & 1)  // the replicated coarse levels are counted by one rank
                    for (int l = 0; l < D_; ++l)
                        LZB_LAUNCH(k_stats, static_cast<unsigned>(std::min<int64_t>(blocks_for(L_[l].nc, kThreads),
                                                                                    kStatsBlocks)),
                                   kThreads, 0, s_, V(l), 0, res_.p->s);
                LZB_LAUNCH(k_norm_partial, kNormBlocks, kThreads, 0, s_, V(D_), v0, v1, partial_.p);
                LZB_LAUNCH(k_norm_final, 1, kNormFinalThreads, 0, s_, partial_.p, kNormBlocks, res_.p, 1);
                break;
            }
            case 1:
                LZB_LAUNCH(k_restrict, vgrid_rows(D_ - 1, c0, c1), kThreads, 0, s_, V(D_), Vrow(D_ - 1, c0), 0, 0.0);
                break;
            case 2:
                for (int l = D_ - 1; l >= 0; --l) {
                    const dim3 g = vgrid(l);
                    LZB_LAUNCH(k_uhat, ugrid(l), kThreads, 0, s_, V(l), l > 0 ? V(l - 1) : V(l), l > 0 ? 1 : 0);
                    LZB_LAUNCH(k_residual, g, kThreads, 0, s_, V(l), d_.field);
                    if (l > 0) LZB_LAUNCH(k_restrict, vgrid(l - 1), kThreads, 0, s_, V(l), V(l - 1), 0, 0.0);
                }
                if (!(flags & 2)) {  // flags bit 1: the C++ data plane reduces on the device (dist.cpp)
                    LZB_CUDA(cudaMemcpyAsync(hres_, res_.p, sizeof(Result), cudaMemcpyDeviceToHost, s_));
                    sync_check();
                }
                break;
            case 3:
                for (int l = 0; l < D_; ++l)
                    LZB_LAUNCH(k_snap, blocks_for(L_[l].nv, kThreads), kThreads, 0, s_, V(l));
                if (d_.variant == LZB_ADAFAC_PI)
                    LZB_LAUNCH(k_aux_inject, vgrid_rows(D_ - 1, c0, c1), kThreads, 0, s_, V(D_), Vrow(D_ - 1, c0));
                break;
            case 4: {
                const double omega = d_.omega;
                const bool pi = d_.variant == LZB_ADAFAC_PI;
                for (int l = D_ - 1; l >= 0; --l) {
                    const dim3 g = vgrid(l);
                    if (pi && l > 0) {
                        LZB_LAUNCH(k_aux_inject, vgrid(l - 1), kThreads, 0, s_, V(l), V(l - 1));
                        LZB_LAUNCH(k_aux_sub, g, kThreads, 0, s_, V(l), V(l - 1), omega);
                    }
                    LZB_LAUNCH(k_jacobi, g, kThreads, 0, s_, V(l), damping(l));
                }
                prolong_launches(D_ - 1);
                if (pi) LZB_LAUNCH(k_scale_aux, vgrid(D_ - 1), kThreads, 0, s_, V(D_ - 1), omega, caux_.p);
                LZB_LAUNCH(k_update_fine, vgrid_rows(D_, v0, v1), kThreads, 0, s_, Vrow(D_, v0), V(D_ - 1),
                           pi ? caux_.p : nullptr, damping(D_));
                LZB_LAUNCH(k_inject, vgrid_rows(D_ - 1, c0, c1), kThreads, 0, s_, V(D_), Vrow(D_ - 1, c0));
                break;
            }
            case 5:
                for (int l = D_ - 1; l >= 1; --l)
                    LZB_LAUNCH(k_inject, vgrid(l - 1), kThreads, 0, s_, V(l), V(l - 1));
                if (!(flags & 2)) sync_check();
                break;
            default: throw Error(LZB_ERR_INVALID, "unknown phase");
        }
    }

    // Device address of the phase-2 result (sum of r^2, then the 20 counter
    // slots as u64) for an on-device reduction (dist.cpp)
    void* dist_result_dev() const { return res_.p; }
    // Result of phase 2 for the host reduction: the slab's sum of r^2 and the
    // 20 counter slots.
    void dist_result(double* norm2, uint64_t* slots) const {
        *norm2 = hres_->norm;
        for (int k = 0; k < 20; ++k) slots[k] = hres_->s[k];
    }

    // The cycle report from the reduced norm^2 and counters (every rank gets
    // the same); report.status tells whether phases 3-5 run.
    lzb_cycle_report dist_report(double norm2, const uint64_t* slots) {
        lzb_cycle_report rep;
        std::memset(&rep, 0, sizeof rep);
        rep.cycle = static_cast<int32_t>(cycle_);
        Result r;
        r.norm = std::sqrt(norm2);
        for (int k = 0; k < 20; ++k) r.s[k] = slots[k];
        front_report(rep, r);
        finish_report(rep, r);
        rep.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - dist_t0_).count();
        return rep;
    }

    std::vector<lzb_cycle_report> run() {  // solver.cpp:421-444 (no AMR on regular grids)
        std::vector<lzb_cycle_report> out;
        const double t_run = trace() ? now_ms() : 0.0;
        if (d_.mode == LZB_EAGER) eager_setup();
        if (trace()) {
            LZB_CUDA(cudaStreamSynchronize(s_));
            std::fprintf(stderr, "[lzb] run: eager_setup %.3f ms\n", now_ms() - t_run);
        }
        for (;;) {
            if (device_loop_ok()) {
                run_device_loop(out);
            } else {
                const double ts = trace() ? now_ms() : 0.0;
                out.push_back(step());
                if (trace())
                    std::fprintf(stderr, "[lzb] host step %u: %.3f ms (pending %lld)\n", cycle_, now_ms() - ts,
                                 static_cast<long long>(pending_));
            }
            if (!out.empty() && out.back().status != LZB_CONTINUE) break;
        }
        return out;
    }

    // ---- the quiescent cycles of run() as ONE graph launch (solver.cpp:421-444
    // + 8-16 with the termination test on the device). Once no assembly work
    // is left (every leaf top, no task pending or in flight) a cycle needs
    // nothing from the host: coarse pass (change-gated, it still drains the
    // one-level-per-cycle lag of the Galerkin hierarchy), residual pass, stats,
    // termination, update. The graph is a conditional WHILE node; its body is
    // that cycle, with the update passes inside a conditional IF node
    // (k_loop_check sets both conditions). Each cycle's Result goes to a
    // device history; the host reads it once after the loop and builds the
    // same CycleReports step() would have. LZB_NO_DEVLOOP=1 keeps step().
    static constexpr uint32_t kLoopCap = 4096;
    bool quiescent() const {
        return all_top_ && pending_ == 0 && !batch_inflight_ && hq_.empty() && !ripple() &&
               d_.forced_fraction <= 0.0 && slab_v1_ < 0;
    }
    void unsettle() { settled_ = false; }
    bool device_loop_ok() const {
        const bool on = std::getenv("LZB_DEVLOOP") != nullptr;  // read per call: tests toggle it
        return on && use_graphs_ && cycle_ >= 1 && !history_.empty() && quiescent() &&
               static_cast<int>(cycle_) < d_.max_cycles;
    }
    void build_loop_graph(int full) {
        if (!hloop_) {
            loop_hist_.alloc(kLoopCap);
            loop_state_.alloc(1);
            LZB_CUDA(cudaMallocHost(&hloop_, sizeof(LoopState) + kLoopCap * sizeof(Result)));
        }
        cudaGraph_t g = nullptr;
        LZB_CUDA(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle h_again, h_update;
        LZB_CUDA(cudaGraphConditionalHandleCreate(&h_again, g, 1, cudaGraphCondAssignDefault));
        LZB_CUDA(cudaGraphConditionalHandleCreate(&h_update, g, 0, cudaGraphCondAssignDefault));
        cudaGraphNodeParams wp = {};
        wp.type = cudaGraphNodeTypeConditional;
        wp.conditional.handle = h_again;
        wp.conditional.type = cudaGraphCondTypeWhile;
        wp.conditional.size = 1;
        cudaGraphNode_t wnode;
        LZB_CUDA(cudaGraphAddNode(&wnode, g, nullptr, 0, &wp));
        cudaGraph_t body = wp.conditional.phGraph_out[0], ifbody = nullptr, tmp = nullptr;
        struct Flag {
            bool& f;
            explicit Flag(bool& x) : f(x) { f = true; }
            ~Flag() { f = false; }
        };
        uint64_t* kern = loop_kernels_[full];
        try {
            const uint64_t l0 = g_launches.load();
            LZB_CUDA(cudaStreamBeginCaptureToGraph(s_, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
            try {
                {
                    PdlScope pdl;
                    Flag in_loop(loop_capture_);
                    LZB_LAUNCH(k_loop_begin, 1, 32, 0, s_, dcycle_.p);
                    if (full) coarse_pass();
                    residual_launches();
                    if (full) stats_launches();
                }
                // plain launch and full edges around the decision kernel
                LZB_LAUNCH(k_loop_check, 1, 32, 0, s_, res_.p, loop_hist_.p, loop_state_.p,
                           static_cast<const uint32_t*>(dcycle_.p), static_cast<const int*>(ctx_->err.p), h_again,
                           h_update, full);
                cudaStreamCaptureStatus cst;
                const cudaGraphNode_t* deps = nullptr;
                size_t ndeps = 0;
                LZB_CUDA(cudaStreamGetCaptureInfo(s_, &cst, nullptr, nullptr, &deps, &ndeps));
                cudaGraphNodeParams ip = {};
                ip.type = cudaGraphNodeTypeConditional;
                ip.conditional.handle = h_update;
                ip.conditional.type = cudaGraphCondTypeIf;
                ip.conditional.size = 1;
                cudaGraphNode_t inode;
                LZB_CUDA(cudaGraphAddNode(&inode, body, deps, ndeps, &ip));
                LZB_CUDA(cudaStreamUpdateCaptureDependencies(s_, &inode, 1, cudaStreamSetCaptureDependencies));
                ifbody = ip.conditional.phGraph_out[0];
            } catch (...) {
                cudaStreamEndCapture(s_, &tmp);
                throw;
            }
            LZB_CUDA(cudaStreamEndCapture(s_, &tmp));
            kern[0] = g_launches.load() - l0;
            LZB_CUDA(cudaStreamBeginCaptureToGraph(s_, ifbody, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
            try {
                PdlScope pdl;
                back_body();
            } catch (...) {
                cudaStreamEndCapture(s_, &tmp);
                throw;
            }
            LZB_CUDA(cudaStreamEndCapture(s_, &tmp));
            kern[1] = g_launches.load() - l0 - kern[0];
            g_launches.fetch_sub(kern[0] + kern[1]);  // counted when they run
            LZB_CUDA(cudaGraphInstantiate(&g_loop_[full], g, 0));
        } catch (...) {
            cudaGraphDestroy(g);
            throw;
        }
        LZB_CUDA(cudaGraphDestroy(g));
    }
    // One launch of the loop graph: the full body until the hierarchy has
    // settled (or the run ends), the settled body (no coarse pass, no stats:
    // both are no-ops once nothing changes) after that. settled_ is dropped by
    // everything that can change an operator or a marker.
    void run_device_loop(std::vector<lzb_cycle_report>& out) {
        auto t0 = std::chrono::steady_clock::now();
        ensure_rhs();
        const int full = settled_ ? 0 : 1;
        if (!g_loop_[full]) {
            const double tb = trace() ? now_ms() : 0.0;
            build_loop_graph(full);
            if (trace())
                std::fprintf(stderr, "[lzb] loop graph (full = %d): %llu + %llu kernels, build %.3f ms\n", full,
                             static_cast<unsigned long long>(loop_kernels_[full][0]),
                             static_cast<unsigned long long>(loop_kernels_[full][1]), now_ms() - tb);
        }
        const double tl = trace() ? now_ms() : 0.0;
        LoopState* hs = reinterpret_cast<LoopState*>(hloop_);
        const Result* hh = reinterpret_cast<const Result*>(hloop_ + sizeof(LoopState));
        std::memset(hs, 0, sizeof *hs);
        hs->front = history_.front();
        hs->target = d_.target;
        hs->divergence = d_.divergence;
        hs->max_cycles = d_.max_cycles;
        hs->cap = kLoopCap;
        *hcycle_ = cycle_;
        LZB_CUDA(cudaMemcpyAsync(dcycle_.p, hcycle_, sizeof(uint32_t), cudaMemcpyHostToDevice, s_));
        LZB_CUDA(cudaMemcpyAsync(loop_state_.p, hs, sizeof *hs, cudaMemcpyHostToDevice, s_));
        LZB_CUDA(cudaGraphLaunch(g_loop_[full], s_));
        LZB_CUDA(cudaMemcpyAsync(hs, loop_state_.p, sizeof *hs, cudaMemcpyDeviceToHost, s_));
        LZB_CUDA(cudaStreamSynchronize(s_));
        const uint32_t n = hs->count;
        const int dev_status = hs->status;
        const bool bad = hs->err != 0;
        if (full && hs->settled) settled_ = true;
        if (trace())
            std::fprintf(stderr, "[lzb] device loop (full = %d): %u cycles in %.3f ms (%.1f us per cycle)\n", full, n,
                         now_ms() - tl, 1e3 * (now_ms() - tl) / (n ? n : 1));
        LZB_CUDA(cudaMemcpyAsync(hloop_ + sizeof(LoopState), loop_hist_.p, n * sizeof(Result), cudaMemcpyDeviceToHost,
                                 s_));
        LZB_CUDA(cudaStreamSynchronize(s_));
        if (n == 0) throw Error(LZB_ERR_CUDA, "device cycle loop recorded no cycle");
        const uint32_t good = bad ? n - 1 : n;  // the cycle that raised the flag is not reported (step() throws)
        uint64_t updates = 0;
        const size_t first = out.size();
        for (uint32_t i = 0; i < good; ++i) {
            lzb_cycle_report rep;
            std::memset(&rep, 0, sizeof rep);
            ++cycle_;
            rep.cycle = static_cast<int32_t>(cycle_);
            if (front_report(rep, hh[i])) ++updates;
            finish_report(rep, hh[i]);
            out.push_back(rep);
        }
        if (bad) ++cycle_;
        *hcycle_ = cycle_;
        g_launches.fetch_add(static_cast<uint64_t>(n) * loop_kernels_[full][0] + updates * loop_kernels_[full][1],
                             std::memory_order_relaxed);
        if (bad) {
            LZB_CUDA(cudaMemset(ctx_->err.p, 0, sizeof(int)));
            throw Error(LZB_ERR_PROTOCOL, "cannot encode non-finite operator entry");
        }
        if (good == 0) return;
        if (out.back().status != dev_status)
            throw Error(LZB_ERR_CUDA, "device cycle loop: host and device termination decisions differ");
        const double w = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / good;
        for (size_t i = first; i < out.size(); ++i) out[i].wall_seconds = w;
    }

    double pass(int which) {
        switch (which) {
            case 0: assembly_pass(); sync_check(); return 0.0;
            case 1: ensure_rhs(); residual_launches(); fetch_result(); return hres_->norm;
            case 2: update_launches(); sync_check(); return 0.0;
            case 3: prolong_launches(); sync_check(); return 0.0;
            case 4: inject(); sync_check(); return 0.0;
            case 5: return 0.0;
            case 6: begin_cycle_tasks(); sync_check(); pending_ = count_pending(); return 0.0;
            case 7: drain(); sync_check(); return static_cast<double>(pending_);
            default: throw Error(LZB_ERR_INVALID, "unknown pass");
        }
    }

    void vertices(int level, int field, double* buf, bool write) {
        check_level(level);
        if (field < 0 || field >= LZB_V_NFIELDS) throw Error(LZB_ERR_INVALID, "bad vertex field");
        auto& b = L_[level].v[field];
        if (write && level == D_ && field == LZB_V_FL) rhs_ready_ = false;
        if (write) LZB_CUDA(cudaMemcpyAsync(b.p, buf, b.bytes(), cudaMemcpyHostToDevice, s_));
        else LZB_CUDA(cudaMemcpyAsync(buf, b.p, b.bytes(), cudaMemcpyDeviceToHost, s_));
        sync_check();
    }

    void cells(int level, double* ops, int32_t* p1, int32_t* n, int32_t* p3, uint32_t* epoch) {
        check_level(level);
        const Level& L = L_[level];
        std::vector<int32_t> hp1(L.nc), hn(L.nc);
        std::vector<int8_t> hp3(L.nc);
        std::vector<uint32_t> hep(L.nc);
        std::vector<double> hop(16 * L.nc);
        LZB_CUDA(cudaMemcpyAsync(hp1.data(), L.p1.p, L.p1.bytes(), cudaMemcpyDeviceToHost, s_));
        LZB_CUDA(cudaMemcpyAsync(hn.data(), L.n.p, L.n.bytes(), cudaMemcpyDeviceToHost, s_));
        LZB_CUDA(cudaMemcpyAsync(hp3.data(), L.p3.p, L.p3.bytes(), cudaMemcpyDeviceToHost, s_));
        LZB_CUDA(cudaMemcpyAsync(hep.data(), L.epoch.p, L.epoch.bytes(), cudaMemcpyDeviceToHost, s_));
        LZB_CUDA(cudaMemcpyAsync(hop.data(), L.op.p, L.op.bytes(), cudaMemcpyDeviceToHost, s_));
        sync_check();
        double kunit[16];
        host_kunit(kunit);
        for (int64_t c = 0; c < L.nc; ++c) {
            bool valid = hp1[c] != LZB_P1_BOTTOM;
            if (p1) p1[c] = hp1[c];
            if (n) n[c] = valid ? hn[c] : 0;
            if (p3) p3[c] = hp3[c];
            if (epoch) epoch[c] = valid ? hep[c] : 0;
            if (ops) {
                if (valid) {
                    std::memcpy(ops + 16 * c, hop.data() + 16 * c, 128);
                } else {  // baseline, evaluated on the host only for this debug view
                    int cx = static_cast<int>(c % L.N), cy = static_cast<int>(c / L.N);
                    double x0 = cx * L.h, y0 = cy * L.h;
                    double e = d_.start_geometric ? 1.0  // the geometric stencil (eps = 1)
                                                  : lzb_field_eval_host(&d_.field, x0 + (0 + 0.5) * 1.0 * L.h,
                                                                        y0 + (0 + 0.5) * 1.0 * L.h);
                    for (int k = 0; k < 16; ++k) ops[16 * c + k] = 0.0 + kunit[k] * e;
                }
            }
        }
    }

    void transfer(int level, int cx, int cy, double* out) {
        check_level(level);
        if (level >= D_) throw Error(LZB_ERR_INVALID, "leaf cells have no transfer block");
        int64_t c = static_cast<int64_t>(cy) * L_[level].N + cx;
        uint8_t has = 0;
        LZB_CUDA(cudaMemcpy(&has, L_[level].has_P.p + c, 1, cudaMemcpyDeviceToHost));
        if (has && L_[level].P.p)
            LZB_CUDA(cudaMemcpy(out, L_[level].P.p + 64 * c, 512, cudaMemcpyDeviceToHost));
        else
            host_geo(out);
    }

    void publish_element(int level, int cx, int cy, const double* m, int n, int32_t p1) {
        check_cell(level, cx, cy);
        all_top_ = false;
        settled_ = false;
        if (level != D_) throw Error(LZB_ERR_INVALID, "publish_element is for leaf cells");
        DevBuf<double> dm(16);
        LZB_CUDA(cudaMemcpyAsync(dm.p, m, 128, cudaMemcpyHostToDevice, s_));
        LZB_LAUNCH(k_publish_one, 1, 32, 0, s_, V(D_), d_.field, cy * L_[D_].N + cx, dm.p, n, p1,
                   d_.delta_max, cycle_, res_.p->s, ctx_->err.p);
        sync_check();
    }

    // lzb_grid_vertex_stencils: assemble_vertex_stencil of every vertex of a level
    void vertex_stencils(int level, int require_payload, double* host_out) {
        check_level(level);
        const Level& L = L_[level];
        DevBuf<double> out(static_cast<size_t>(L.nv) * 9);
        DevBuf<int> flag(1);
        LZB_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), s_));
        LZB_LAUNCH(k_vertex_stencils, vgrid(level), kThreads, 0, s_, V(level), d_.field, out.p, require_payload,
                   flag.p);
        int hflag = 0;
        LZB_CUDA(cudaMemcpyAsync(host_out, out.p, out.bytes(), cudaMemcpyDeviceToHost, s_));
        LZB_CUDA(cudaMemcpyAsync(&hflag, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s_));
        sync_check();
        if (hflag) throw Error(LZB_ERR_PROTOCOL, "adjacent cell has no assembled operator (p1 = bottom)");
    }

    // lzb_grid_publish_level: every leaf published from host matrices
    void publish_level(int level, const double* mats, const int32_t* n, int32_t p1) {
        if (level != D_) throw Error(LZB_ERR_INVALID, "publish_level is for the leaf level");
        all_top_ = false;
        settled_ = false;
        const int64_t nc = L_[D_].nc;
        DevBuf<double> dm(static_cast<size_t>(nc) * 16);
        DevBuf<int32_t> dn(static_cast<size_t>(nc));
        LZB_CUDA(cudaMemcpyAsync(dm.p, mats, dm.bytes(), cudaMemcpyHostToDevice, s_));
        LZB_CUDA(cudaMemcpyAsync(dn.p, n, dn.bytes(), cudaMemcpyHostToDevice, s_));
        LZB_LAUNCH(k_publish_level, blocks_for(nc, kThreads), kThreads, 0, s_, V(D_), d_.field, dm.p, dn.p, p1,
                   d_.delta_max, cycle_, res_.p->s, ctx_->err.p);
        sync_check();
    }

    // assemble_fixed through the same fused kernel, also writing each cell's
    // integrated matrix (before compression) to host_raw (nc x 16)
    void assemble_fixed_raw(int n, double* host_raw) {
        DevBuf<double> raw(static_cast<size_t>(L_[D_].nc) * 16);
        raw_ = raw.p;
        try {
            assemble_fixed(n);
        } catch (...) {
            raw_ = nullptr;
            throw;
        }
        raw_ = nullptr;
        LZB_CUDA(cudaMemcpyAsync(host_raw, raw.p, raw.bytes(), cudaMemcpyDeviceToHost, s_));
        sync_check();
    }

    void adaptive_step(int level, int cx, int cy) {
        check_cell(level, cx, cy);
        all_top_ = false;
        settled_ = false;
        if (level != D_) throw Error(LZB_ERR_INVALID, "adaptive steps are for leaf cells");
        LZB_LAUNCH(k_step_one, 1, 32, 0, s_, V(D_), d_.field, cy * L_[D_].N + cx, d_.schedule,
                   d_.n_max, d_.termination_c, d_.delta_max, cycle_,
                   d_.integration == LZB_INTEGRATE_FAST ? 1 : 0, res_.p->s, ctx_->err.p);
        sync_check();
    }

    // ------------------------------------------------------------ stream I/O
    AllLevels all_levels() const {
        AllLevels A{};
        for (int l = 0; l <= D_; ++l) A.L[l] = V(l);
        A.st = slots_;
        A.D = D_;
        return A;
    }

    void record_sizes(int64_t* sizes) {
        const dim3 grid(blocks_for(L_[D_ - 1].N, 64), L_[D_ - 1].N);
        LZB_LAUNCH(k_record_sizes_patches, grid, 64, 0, s_, all_levels(), sizes, 0, L_[D_ - 1].N, 0);
        const int64_t upper = total_cells_ - L_[D_].nc - L_[D_ - 1].nc;
        if (upper > 0)
            LZB_LAUNCH(k_record_sizes_upper, blocks_for(upper, kThreads), kThreads, 0, s_, all_levels(), upper,
                       sizes, -1, -1);
    }

    // Record sizes -> device exclusive scan (cub) -> total. Returns the image size.
    int64_t scan_records() {
        if (rec_sizes_.n < static_cast<size_t>(total_cells_)) {
            rec_sizes_.alloc(total_cells_);
            rec_offs_.alloc(total_cells_ + 1);
            size_t tb = 0;
            LZB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, rec_sizes_.p, rec_offs_.p,
                                                  static_cast<int>(total_cells_ + 1), s_));
            scan_tmp_.alloc(tb);
        }
        record_sizes(rec_sizes_.p);
        size_t tb = scan_tmp_.n;
        // exclusive offsets; the image size is the last offset plus the last record
        LZB_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp_.p, tb, rec_sizes_.p, rec_offs_.p,
                                              static_cast<int>(total_cells_), s_));
        int64_t last[2];
        LZB_CUDA(cudaMemcpyAsync(&last[0], rec_offs_.p + total_cells_ - 1, 8, cudaMemcpyDeviceToHost, s_));
        LZB_CUDA(cudaMemcpyAsync(&last[1], rec_sizes_.p + total_cells_ - 1, 8, cudaMemcpyDeviceToHost, s_));
        sync_check();
        return 12 + last[0] + last[1];
    }

    int64_t image_size() { return scan_records(); }

    // Stream records into img (offsets from scan_records): the level-(D-1)
    // patches with their leaves, then the levels above.
    void pack_launches(uint8_t* img) {
        const PackArgs T{centre_[1].x.p, centre_[1].y.p, centre_[0].x.p, centre_[0].y.p};
        const int per = L_[D_ - 1].N >= 3 ? 3 : 1;  // sibling patches per warp
        const dim3 grid(blocks_for(L_[D_ - 1].N, kPackWarps), L_[D_ - 1].N / per);
        LZB_LAUNCH(k_pack_patches, grid, kPackWarps * 32, 0, s_, all_levels(), d_.field, T, per, rec_offs_.p, img,
                   ctx_->err.p, 0, L_[D_ - 1].N, 0, nullptr);
        const int64_t upper = total_cells_ - L_[D_].nc - L_[D_ - 1].nc;
        if (upper > 0)
            LZB_LAUNCH(k_pack_upper, blocks_for(upper, kThreads / 32), kThreads, 0, s_, all_levels(), d_.field,
                       upper, rec_offs_.p, img, ctx_->err.p, -1, -1, nullptr);
    }

    // assemble_fixed(n) followed by image_into(out, cap), pipelined: the LZMG
    // image is a root record followed by the 9 level-1 subtrees in child
    // order lx * 3 + ly (pre-order, mesh.cpp:152-157), so each x band of 3
    // subtrees is one contiguous byte range, and so is any run of subtrees
    // inside one column. Band by band (the three columns: smaller bands,
    // e.g. {1, 2, 3, 2, 1} subtrees, measured 1.96 ms against 1.90: a band
    // under ~600 cells per resident block slows the persistent assembly
    // kernel more than the earlier copy start saves) the solve stream
    // assembles the leaves, then sizes, scans and packs the band's records
    // (offsets chained through a device running base), and the copy stream
    // moves its bytes to the host while the next band assembles. Same bytes
    // as the sequential calls. timeline: NULL or 3 x kBands floats, device
    // ms of each band's assembly, pack and copy end.
    int64_t assemble_stream(int n, uint8_t* out, int64_t cap, float* timeline) {
        if (n < 1) throw Error(LZB_ERR_INVALID, "n must be >= 1");
        if (D_ < 2) {
            assemble_fixed(n);
            return image_into(out, cap);
        }
        if (cap < 12) throw Error(LZB_ERR_INVALID, "stream image buffer too small");
        all_top_ = true;
        ensure_tables(n);
        if (rec_sizes_.n < static_cast<size_t>(total_cells_)) scan_records();  // allocates the scan buffers
        const int64_t leaves = L_[D_].nc, refined = total_cells_ - leaves;
        const size_t cap_dev = static_cast<size_t>(12 + total_cells_ + leaves * 128 + refined * 1152);
        if (img_.n < cap_dev) img_.alloc(cap_dev);
        if (!st_ready_) {
            stream_base_.alloc(kBands + 1);
            LZB_CUDA(cudaMallocHost(&hbase_, (kBands + 1) * sizeof(int64_t)));
            LZB_CUDA(cudaStreamCreateWithFlags(&cp_, cudaStreamNonBlocking));
            for (int k = 0; k < kBands; ++k) {
                LZB_CUDA(cudaEventCreate(&ev_asm_[k]));
                LZB_CUDA(cudaEventCreate(&ev_pack_[k]));
                LZB_CUDA(cudaEventCreate(&ev_copy_[k]));
            }
            LZB_CUDA(cudaEventCreate(&ev_root_));
            LZB_CUDA(cudaEventCreate(&ev_start_));
            st_ready_ = true;
        }
        const int N = L_[D_].N, Nc = L_[D_ - 1].N, w = N / 3, pw = Nc / 3;
        const int64_t S1 = slots_.subtree[1];
        int64_t nup = 0;  // cells of levels 1..D-2 in one subtree
        for (int l = 1, q = 1; l <= D_ - 2; ++l, q *= 9) nup += q;
        const AllLevels AL = all_levels();
        const PackArgs T{centre_[1].x.p, centre_[1].y.p, centre_[0].x.p, centre_[0].y.p};
        LZB_CUDA(cudaEventRecord(ev_start_, s_));
        // the root record (slot 0, offset 0): its size starts the running base
        LZB_LAUNCH(k_record_sizes_upper, 1, 32, 0, s_, AL, 1, rec_sizes_.p, -1, -1);
        LZB_LAUNCH(k_root_base, 1, 1, 0, s_, rec_sizes_.p, rec_offs_.p, stream_base_.p);
        LZB_LAUNCH(k_pack_upper, 1, 32, 0, s_, AL, d_.field, 1, rec_offs_.p, img_.p, ctx_->err.p, -1, -1, nullptr);
        LZB_CUDA(cudaEventRecord(ev_root_, s_));
        // band i: subtrees [k0, k1) of column a = k0 / 3, rows b0 = k0 % 3 .. b1 - 1;
        // assembly, then its sizes / scan / pack, all on the solve stream (the
        // persistent assembly kernel holds every SM while it runs, so a pack beside
        // it would starve)
        static constexpr int kBand[kBands + 1] = {0, 3, 6, 9};
        for (int i = 0; i < kBands; ++i) {
            const int k0 = kBand[i], k1 = kBand[i + 1], a = k0 / 3, b0 = k0 % 3, nb = k1 - k0;
            const int64_t s0 = 1 + k0 * S1, nslot = nb * S1;
            const int prow = nb * pw;  // patch rows of the band
            const int per = prow % 3 == 0 ? 3 : 1;
            assemble_rect(n, CellRect{a * w, w, b0 * w}, static_cast<int64_t>(w) * nb * w, s_);
            LZB_CUDA(cudaEventRecord(ev_asm_[i], s_));
            LZB_LAUNCH(k_record_sizes_patches, dim3(blocks_for(pw, 64), prow), 64, 0, s_, AL, rec_sizes_.p, a * pw, pw,
                       b0 * pw);
            for (int b = b0; b < b0 + nb && nup > 0; ++b)
                LZB_LAUNCH(k_record_sizes_upper, blocks_for(nup, kThreads), kThreads, 0, s_, AL, nup, rec_sizes_.p,
                           a, b);
            size_t tb = scan_tmp_.n;
            LZB_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp_.p, tb, rec_sizes_.p + s0, rec_offs_.p + s0,
                                                  static_cast<int>(nslot), s_));
            LZB_LAUNCH(k_chunk_base, 1, 1, 0, s_, rec_sizes_.p + s0, rec_offs_.p + s0, nslot, stream_base_.p + i);
            LZB_LAUNCH(k_pack_patches, dim3(blocks_for(pw, kPackWarps), prow / per), kPackWarps * 32, 0, s_, AL,
                       d_.field, T, per, rec_offs_.p, img_.p, ctx_->err.p, a * pw, pw, b0 * pw, stream_base_.p + i);
            for (int b = b0; b < b0 + nb && nup > 0; ++b)
                LZB_LAUNCH(k_pack_upper, blocks_for(nup, kThreads / 32), kThreads, 0, s_, AL, d_.field, nup,
                           rec_offs_.p, img_.p, ctx_->err.p, a, b, stream_base_.p + i);
            LZB_CUDA(cudaMemcpyAsync(hbase_ + i, stream_base_.p + i + 1, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                     s_));
            LZB_CUDA(cudaEventRecord(ev_pack_[i], s_));
        }
        // host: as each band's byte range becomes known, queue its copy (copy
        // engine, concurrent with the next bands' assembly)
        bool overflow = false;
        int64_t lo = 12;
        for (int a = 0; a < kBands; ++a) {
            LZB_CUDA(cudaEventSynchronize(ev_pack_[a]));
            const int64_t hi = 12 + hbase_[a];
            if (hi > cap) overflow = true;
            if (!overflow) {
                LZB_CUDA(cudaStreamWaitEvent(cp_, ev_pack_[a], 0));
                LZB_CUDA(cudaMemcpyAsync(out + lo, img_.p + lo, hi - lo, cudaMemcpyDeviceToHost, cp_));
            }
            LZB_CUDA(cudaEventRecord(ev_copy_[a], cp_));
            lo = hi;
        }
        LZB_CUDA(cudaStreamSynchronize(cp_));
        if (timeline)
            for (int a = 0; a < kBands; ++a) {
                LZB_CUDA(cudaEventElapsedTime(&timeline[a], ev_start_, ev_asm_[a]));
                LZB_CUDA(cudaEventElapsedTime(&timeline[kBands + a], ev_start_, ev_pack_[a]));
                LZB_CUDA(cudaEventElapsedTime(&timeline[2 * kBands + a], ev_start_, ev_copy_[a]));
            }
        sync_check();
        if (overflow) throw Error(LZB_ERR_INVALID, "stream image buffer too small");
        const uint32_t hdr[3] = {0x4c5a4d47u, 1u, static_cast<uint32_t>(total_cells_)};
        std::memcpy(out, hdr, 12);
        return lo;
    }

    // CellStream::save byte image: packed on the device (k_pack_patches) from the
    // decoded operators, copied once into the caller's buffer.
    int64_t image_into(uint8_t* out, int64_t cap) {
        int64_t size = scan_records();
        if (size > cap) throw Error(LZB_ERR_INVALID, "stream image buffer too small");
        if (img_.n < static_cast<size_t>(size)) img_.alloc(static_cast<size_t>(size) + (size >> 3));
        uint32_t hdr[3] = {0x4c5a4d47u, 1u, static_cast<uint32_t>(total_cells_)};
        std::memcpy(out, hdr, 12);
        pack_launches(img_.p);
        LZB_CUDA(cudaMemcpyAsync(out + 12, img_.p + 12, size - 12, cudaMemcpyDeviceToHost, s_));
        sync_check();
        return size;
    }

    // Device time of one hot kernel of the cycle / stream path on the solve
    // stream: `reps` back-to-back launches bracketed by CUDA events, average
    // ms per launch. The kernels run on the grid's live state (idempotent
    // except the Jacobi / prolongation updates of u, which only drift it).
    double time_kernel(int what, int reps) {
        if (reps < 1) throw Error(LZB_ERR_INVALID, "reps must be >= 1");
        const int l = D_;
        ensure_rhs();
        if (what == LZB_TK_PACK) {
            const int64_t size = scan_records();
            if (img_.n < static_cast<size_t>(size)) img_.alloc(static_cast<size_t>(size) + (size >> 3));
        }
        if ((what == LZB_TK_RESTRICT || what == LZB_TK_PROLONG) && D_ < 1)
            throw Error(LZB_ERR_INVALID, "needs depth >= 1");
        auto launch = [&] {
            switch (what) {
                case LZB_TK_UHAT:
                    LZB_LAUNCH(k_uhat, ugrid(l), kThreads, 0, s_, V(l), l > 0 ? V(l - 1) : V(l), l > 0 ? 1 : 0);
                    break;
                case LZB_TK_RESIDUAL: leaf_residual(0, L_[D_].N + 1); break;
                case LZB_TK_RESTRICT:
                    LZB_LAUNCH(k_restrict, vgrid(l - 1), kThreads, 0, s_, V(l), V(l - 1), 0, 0.0);
                    break;
                case LZB_TK_JACOBI: LZB_LAUNCH(k_jacobi, vgrid(l), kThreads, 0, s_, V(l), 0.0); break;
                case LZB_TK_PROLONG: LZB_LAUNCH(k_prolong, ugrid(l), kThreads, 0, s_, V(l), V(l - 1)); break;
                case LZB_TK_PACK:
                    pack_launches(img_.p);
                    break;
                case LZB_TK_FRONT: run_graph(g_front_, &Grid::front_body); break;
                case LZB_TK_BACK: run_graph(g_back_, &Grid::back_body); break;
                default: throw Error(LZB_ERR_INVALID, "unknown kernel id");
            }
        };
        launch();  // warm (and graph instantiation)
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
        sync_check();
        return static_cast<double>(ms) / reps;
    }

    std::vector<uint8_t> image() {
        std::vector<uint8_t> out(static_cast<size_t>(scan_records()));
        image_into(out.data(), static_cast<int64_t>(out.size()));
        return out;
    }

    void load(const uint8_t* in, int64_t size) {  // CellStream::load (stream.cpp:340-394)
        all_top_ = false;
        settled_ = false;
        if (size < 4) throw Error(LZB_ERR_CORRUPT, "truncated stream file");
        uint32_t hdr[3] = {0, 0, 0};
        std::memcpy(&hdr[0], in, 4);
        if (hdr[0] != 0x4c5a4d47u) throw Error(LZB_ERR_CORRUPT, "bad stream magic");
        if (size < 8) throw Error(LZB_ERR_CORRUPT, "truncated stream file");
        std::memcpy(&hdr[1], in + 4, 4);
        if (hdr[1] != 1u) throw Error(LZB_ERR_CORRUPT, "unsupported stream version");
        if (size < 12) throw Error(LZB_ERR_CORRUPT, "truncated stream file");
        std::memcpy(&hdr[2], in + 8, 4);
        if (hdr[2] != static_cast<uint32_t>(total_cells_))
            throw Error(LZB_ERR_CORRUPT, "stream cell count does not match the mesh");
        // sequential header walk in pre-order: the record sizes chain the offsets
        std::vector<int64_t> offsets(total_cells_);
        int64_t pos = 12, slot = 0;
        std::vector<int> stack;  // levels of the pre-order walk
        std::function<void(int)> walk = [&](int l) {
            if (pos >= size) throw Error(LZB_ERR_CORRUPT, "truncated stream file");
            uint8_t h = in[pos];
            int cls = (h >> 6) & 3, p3 = h & 0x0f;
            if (cls == 3 || p3 == 1 || p3 > 8) throw Error(LZB_ERR_CORRUPT, "invalid record header byte");
            offsets[slot++] = pos;
            int64_t len = 1;
            if (cls != 0 && p3 != 0) len += static_cast<int64_t>(p3) * (l == D_ ? 16 : 144);
            if (pos + len > size) throw Error(LZB_ERR_CORRUPT, "truncated record payload");
            pos += len;
            if (l < D_)
                for (int k = 0; k < 9; ++k) walk(l + 1);
        };
        walk(0);
        // p3 == 0 payload-less class-1/2 records of refined cells: only 1 byte (handled by len)
        DevBuf<int64_t> doff(total_cells_);
        DevBuf<uint8_t> din(size);
        LZB_CUDA(cudaMemcpyAsync(doff.p, offsets.data(), doff.bytes(), cudaMemcpyHostToDevice, s_));
        LZB_CUDA(cudaMemcpyAsync(din.p, in, size, cudaMemcpyHostToDevice, s_));
        for (int l = 0; l <= D_; ++l)
            LZB_LAUNCH(k_unpack, blocks_for(L_[l].nc, 64), 64, 0, s_, V(l), d_.field, l,
                       l == D_ ? 1 : 0, slots_, doff.p, din.p, d_.delta_max, cycle_, res_.p->s,
                       ctx_->err.p);
        sync_check();
        pending_ = count_pending();
    }

    int64_t pending() const { return pending_; }

    // The leaf state was modified outside the engine (e.g. rows received from
    // other ranks): re-derive the converged flag on the next leaf pass.
    void invalidate() {
        LZB_CUDA(cudaStreamSynchronize(s_));
        all_top_ = false;
        settled_ = false;
    }

    void plane_arrays(void** planes, void** cp3, int* width) {
        *planes = L_[D_].cplanes.p;
        *cp3 = L_[D_].cp3.p;
        *width = d_.plane_width;
    }

    void cell_arrays(int level, void** op, void** p1, void** n, void** p3, void** epoch, void** chg) {
        check_level(level);
        const Level& L = L_[level];
        if (op) *op = L.op.p;
        if (p1) *p1 = L.p1.p;
        if (n) *n = L.n.p;
        if (p3) *p3 = L.p3.p;
        if (epoch) *epoch = L.epoch.p;
        if (chg) *chg = L.chg.p;
    }
    double* device_field(int level, int field) {
        check_level(level);
        if (field < 0 || field >= LZB_V_NFIELDS) throw Error(LZB_ERR_INVALID, "bad vertex field");
        return L_[level].v[field].p;
    }

private:
    void check_level(int level) const {
        if (level < 0 || level > D_) throw Error(LZB_ERR_INVALID, "level out of range");
    }
    void check_cell(int level, int cx, int cy) const {
        check_level(level);
        if (cx < 0 || cy < 0 || cx >= L_[level].N || cy >= L_[level].N)
            throw Error(LZB_ERR_INVALID, "cell out of range");
    }

    lzb_ctx* ctx_;
    lzb_grid_desc d_;
    int D_;
    cudaStream_t s_;
    double* raw_ = nullptr;  // assemble_fixed_raw: integrated matrices out of the fused kernel
    DevBuf<double> sink_;    // forced tasks' discarded results
    std::vector<Level> L_;
    int64_t leaves_ = 0, total_cells_ = 0, total_vertices_ = 0;
    DevBuf<int32_t> list_, snap_;
    DevBuf<int> counter_, blockcnt_;
    DevBuf<unsigned> hist_;
    DevBuf<double> partial_;
    DevBuf<Result> res_;
    DevBuf<long long> keys_;
    TableSet tables_;
    // concurrent assembly
    cudaStream_t a_ = nullptr;
    TableSet atables_;
    DevBuf<int32_t> alist_, asnap_, sp1_, sn_;
    DevBuf<int> acounter_, ablockcnt_;
    DevBuf<unsigned> ahist_;
    DevBuf<double> sop_;
    DevBuf<int8_t> sp3_;
    DevBuf<uint32_t> sepoch_, schg_;
    cudaEvent_t ev_batch_ = nullptr, ev_spawn_ = nullptr;
    bool batch_inflight_ = false;
    int batch_n_ = 1;
    int64_t batches_launched_ = 0, batches_committed_ = 0;

public:
    int64_t batches_launched() const { return batches_launched_; }
    int64_t batches_committed() const { return batches_committed_; }

private:
    DevBuf<int64_t> rec_sizes_, rec_offs_, stream_base_;
    int64_t* hbase_ = nullptr;  // pinned: the running image base per band
    cudaStream_t cp_ = nullptr;
    static constexpr int kBands = 3;  // assemble_stream bands of level-1 subtrees
    cudaEvent_t ev_asm_[kBands] = {}, ev_pack_[kBands] = {}, ev_copy_[kBands] = {}, ev_root_ = nullptr,
                ev_start_ = nullptr;
    bool st_ready_ = false;
    DevBuf<unsigned char> scan_tmp_;
    DevBuf<uint8_t> img_;
    Result* hres_ = nullptr;
    unsigned* hhist_ = nullptr;
    SlotTable slots_{};
    DevBuf<int64_t> slot_x_[kMaxLevels], slot_y_[kMaxLevels];
    struct CentreParts {
        DevBuf<double> x, y;
    } centre_[2];  // levels D-1 and D
    uint32_t cycle_ = 0;
    uint32_t* hcycle_ = nullptr;  // pinned: read by the coarse-pass graph at replay
    int* herr_ = nullptr;         // pinned: device error flag copied out by the front graph
    DevBuf<uint32_t> dcycle_;
    bool use_graphs_ = true;
    DevBuf<double> caux_;         // scaled aux of level D-1 (k_update_fine)
    bool rhs_ready_ = false;      // leaf-level lumped load in place
    bool all_top_ = false;        // every leaf converged (no request_stencil work left)
    cudaGraphExec_t g_coarse_ = nullptr, g_front_ = nullptr, g_back_ = nullptr;
    cudaGraphExec_t g_front_quiet_ = nullptr;  // a settled cycle's front: no coarse pass, no stats
    cudaGraphExec_t g_vfront_ = nullptr, g_vback_ = nullptr;  // V-cycle: front, sweeps (for vnu_)
    cudaGraphExec_t g_loop_[2] = {nullptr, nullptr};  // the device-side cycle loop: [0] settled body, [1] full body
    bool settled_ = false;  // a full coarse pass found nothing to recompute and nothing has changed since
    bool loop_capture_ = false;         // capturing the loop body: the epoch is counted on the device
    DevBuf<Result> loop_hist_;
    DevBuf<LoopState> loop_state_;
    unsigned char* hloop_ = nullptr;  // pinned: LoopState + the loop's Results
    uint64_t loop_kernels_[2][2] = {{0, 0}, {0, 0}};  // [body][front part, update part] kernels per cycle
    int vnu_ = -1;
    bool uhat_is_u_ = false;
    uint64_t graph_kernels_[6] = {0, 0, 0, 0, 0, 0};
    double first_residual_ = -1.0;
    int slab_v0_ = 0, slab_v1_ = -1;  // leaf vertex rows of this rank's slab (-1: the whole level)
    std::chrono::steady_clock::time_point dist_t0_{};
    std::vector<double> history_;
    uint64_t dof_total_ = 0;
    int64_t pending_ = 0;
};

}  // namespace lzb

struct lzb_grid {
    lzb::Grid* g;
};

using namespace lzb;

extern "C" {

int lzb_grid_create(lzb_ctx* ctx, const lzb_grid_desc* desc, lzb_grid** out) { LZB_RANGE("lzb_grid_create");
    return guarded([&] {
        auto* g = new lzb_grid{nullptr};
        try {
            g->g = new Grid(ctx, *desc);
        } catch (...) {
            delete g;
            throw;
        }
        *out = g;
    });
}
void lzb_grid_destroy(lzb_grid* g) {
    if (!g) return;
    delete g->g;
    delete g;
}
int lzb_grid_init_noise(lzb_grid* g, uint64_t seed) { LZB_RANGE("lzb_grid_init_noise"); return guarded([&] { g->g->unsettle(); g->g->init_noise(seed); }); }
int lzb_grid_eager_setup(lzb_grid* g) { LZB_RANGE("lzb_grid_eager_setup");
    return guarded([&] { g->g->unsettle();
        g->g->eager_setup();
        g->g->sync_check();
    });
}
int lzb_grid_assemble_rows(lzb_grid* g, int n, int row0, int row1) { LZB_RANGE("lzb_grid_assemble_rows");
    return guarded([&] { g->g->unsettle();
        g->g->assemble_fixed_rows(n, row0, row1);
        g->g->sync_check();
    });
}
int lzb_grid_assemble_fixed_raw(lzb_grid* g, int n, double* host_raw) { LZB_RANGE("lzb_grid_assemble_fixed_raw");
    return guarded([&] { g->g->unsettle(); g->g->assemble_fixed_raw(n, host_raw); });
}
int lzb_grid_publish_level(lzb_grid* g, int level, const double* mats, const int32_t* n, int32_t p1) { LZB_RANGE("lzb_grid_publish_level");
    return guarded([&] { g->g->unsettle(); g->g->publish_level(level, mats, n, p1); });
}
int lzb_grid_vertex_stencils(lzb_grid* g, int level, int require_payload, double* out) { LZB_RANGE("lzb_grid_vertex_stencils");
    return guarded([&] { g->g->unsettle(); g->g->vertex_stencils(level, require_payload, out); });
}
int lzb_scatter_row(const double* element16, int corner, double* stencil9) {
    if (corner < 0 || corner > 3) {
        lzb::set_last_error("corner must be 0..3");
        return LZB_ERR_INVALID;
    }
    for (int c = 0; c < 4; ++c) {  // element.cpp:39-45
        const int dx = lzb::cdx(c) - lzb::cdx(corner), dy = lzb::cdy(c) - lzb::cdy(corner);
        stencil9[(dy + 1) * 3 + (dx + 1)] += element16[corner * 4 + c];
    }
    return LZB_OK;
}
int lzb_grid_invalidate(lzb_grid* g) {
    return guarded([&] { g->g->unsettle(); g->g->invalidate(); });
}
int lzb_grid_cell_arrays(lzb_grid* g, int level, void** op, void** p1, void** n, void** p3, void** epoch,
                         void** chg) {
    return guarded([&] { g->g->unsettle(); g->g->cell_arrays(level, op, p1, n, p3, epoch, chg); });
}
int lzb_grid_assemble_fixed(lzb_grid* g, int n) { LZB_RANGE("lzb_grid_assemble_fixed");
    return guarded([&] { g->g->unsettle();
        g->g->assemble_fixed(n);
        g->g->sync_check();
    });
}
int lzb_grid_step(lzb_grid* g, lzb_cycle_report* out) { LZB_RANGE("lzb_grid_step"); return guarded([&] { *out = g->g->step(); }); }
int lzb_grid_vcycle(lzb_grid* g, int nu, lzb_cycle_report* out) { LZB_RANGE("lzb_grid_vcycle");
    return guarded([&] { g->g->unsettle(); *out = g->g->vcycle(nu); });
}
int lzb_grid_run(lzb_grid* g, lzb_cycle_report* out, int cap, int* count) { LZB_RANGE("lzb_grid_run");
    return guarded([&] {
        auto reps = g->g->run();
        for (size_t i = 0; i < reps.size() && static_cast<int>(i) < cap; ++i) out[i] = reps[i];
        *count = static_cast<int>(reps.size());
    });
}
int lzb_grid_pass(lzb_grid* g, int which, double* value) { LZB_RANGE("lzb_grid_pass");
    return guarded([&] { g->g->unsettle();
        double v = g->g->pass(which);
        if (value) *value = v;
    });
}
int lzb_grid_cycle(lzb_grid* g) { return static_cast<int>(g->g->cycle()); }
int lzb_grid_vertices(lzb_grid* g, int level, int field, double* buf, int write) {
    return guarded([&] { g->g->unsettle(); g->g->vertices(level, field, buf, write != 0); });
}
int lzb_grid_cells(lzb_grid* g, int level, double* ops, int32_t* p1, int32_t* n, int32_t* p3,
                   uint32_t* epoch) {
    return guarded([&] { g->g->unsettle(); g->g->cells(level, ops, p1, n, p3, epoch); });
}
int lzb_grid_transfer(lzb_grid* g, int level, int cx, int cy, double* out64) {
    return guarded([&] { g->g->unsettle(); g->g->transfer(level, cx, cy, out64); });
}
int lzb_grid_publish_element(lzb_grid* g, int level, int cx, int cy, const double* m16, int n,
                             int32_t p1) {
    return guarded([&] { g->g->unsettle(); g->g->publish_element(level, cx, cy, m16, n, p1); });
}
int lzb_grid_adaptive_step(lzb_grid* g, int level, int cx, int cy) { LZB_RANGE("lzb_grid_adaptive_step");
    return guarded([&] { g->g->unsettle(); g->g->adaptive_step(level, cx, cy); });
}
int lzb_grid_stats(lzb_grid* g, lzb_compression_stats* out) { LZB_RANGE("lzb_grid_stats");
    return guarded([&] { g->g->unsettle(); *out = g->g->stats(); });
}
int lzb_grid_stream_image(lzb_grid* g, uint8_t* out, int64_t cap, int64_t* size) { LZB_RANGE("lzb_grid_stream_image");
    return guarded([&] { g->g->unsettle();
        if (!out) {
            *size = g->g->image_size();
            return;
        }
        *size = g->g->image_into(out, cap);
    });
}
int lzb_grid_plane_arrays(lzb_grid* g, void** planes, void** cp3, int* width) {
    return guarded([&] { g->g->unsettle(); g->g->plane_arrays(planes, cp3, width); });
}
int lzb_grid_desc_of(lzb_grid* g, lzb_grid_desc* out) {
    return guarded([&] { g->g->unsettle(); *out = g->g->desc(); });
}
int lzb_grid_info(lzb_grid* g, lzb_ctx** ctx, int* depth) {
    return guarded([&] { g->g->unsettle();
        if (ctx) *ctx = g->g->context();
        if (depth) *depth = g->g->depth();
    });
}
int lzb_grid_set_slab(lzb_grid* g, int v0, int v1) {
    return guarded([&] { g->g->unsettle(); g->g->set_slab(v0, v1); });
}
int lzb_grid_dist_phase(lzb_grid* g, int phase, int flags) { LZB_RANGE("lzb_grid_dist_phase");
    return guarded([&] { g->g->unsettle(); g->g->dist_phase(phase, flags); });
}
int lzb_grid_dist_result_dev(lzb_grid* g, void** result) {
    return guarded([&] { g->g->unsettle(); *result = g->g->dist_result_dev(); });
}
int lzb_grid_dist_result(lzb_grid* g, double* norm2, uint64_t* slots20) {
    return guarded([&] { g->g->unsettle(); g->g->dist_result(norm2, slots20); });
}
int lzb_grid_dist_report(lzb_grid* g, double norm2, const uint64_t* slots20, lzb_cycle_report* rep) {
    return guarded([&] { g->g->unsettle(); *rep = g->g->dist_report(norm2, slots20); });
}
int lzb_grid_assemble_stream(lzb_grid* g, int n, uint8_t* out, int64_t cap, int64_t* size, float* timeline) { LZB_RANGE("lzb_grid_assemble_stream");
    return guarded([&] { g->g->unsettle(); *size = g->g->assemble_stream(n, out, cap, timeline); });
}
int lzb_grid_time_kernel(lzb_grid* g, int what, int reps, double* avg_ms) {
    return guarded([&] { g->g->unsettle(); *avg_ms = g->g->time_kernel(what, reps); });
}
int lzb_grid_stream_load(lzb_grid* g, const uint8_t* in, int64_t size) { LZB_RANGE("lzb_grid_stream_load");
    return guarded([&] { g->g->unsettle(); g->g->load(in, size); });
}
int lzb_grid_save(lzb_grid* g, const char* path) { LZB_RANGE("lzb_grid_save");
    return guarded([&] { g->g->unsettle();
        auto img = g->g->image();
        std::ofstream f(path, std::ios::binary);
        if (!f) throw Error(LZB_ERR_IO, std::string("cannot open stream file for writing: ") + path);
        f.write(reinterpret_cast<const char*>(img.data()), static_cast<std::streamsize>(img.size()));
    });
}
int lzb_grid_load(lzb_grid* g, const char* path) { LZB_RANGE("lzb_grid_load");
    return guarded([&] { g->g->unsettle();
        std::ifstream f(path, std::ios::binary);
        if (!f) throw Error(LZB_ERR_IO, std::string("cannot open stream file: ") + path);
        std::vector<uint8_t> buf((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
        g->g->load(buf.data(), static_cast<int64_t>(buf.size()));
    });
}
int64_t lzb_grid_pending(lzb_grid* g) { return g->g->pending(); }
int lzb_grid_device_view(lzb_grid* g, int level, int field, void** ptr) {
    return guarded([&] { g->g->unsettle(); *ptr = g->g->device_field(level, field); });
}

}  // extern "C"

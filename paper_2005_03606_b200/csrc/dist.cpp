// dist.cpp — the slab-distributed data plane of liblzb.so,
// C++ behind the C-ABI: the context owns an NCCL communicator, and one cycle
// of a slab-distributed grid is the grid's compute phases (lzb_grid_dist_phase
// / lzb_grid3_dist_phase, grid.cu / grid3.cu) with the exchanges in between,
// all enqueued on the solve stream:
//   * halos: ncclSend / ncclRecv of whole vertex rows (2D) or planes (3D)
//     with the two neighbouring slabs, inside one ncclGroupStart/End, straight
//     from / into the grid's arrays (rows and planes are contiguous);
//   * the replicated level D-1: every rank's rows [c0, c1) to every rank by an
//     in-place ncclBroadcast per root in one group (slabs may be uneven, no
//     padding or staging copies);
//   * the norm and the telemetry counters: ncclAllReduce on the device result
//     (sum, and max for the three maxima), then ONE device-to-host read per
//     cycle, the termination decision's.
// The same plan runs over several slabs of one process through device copies
// (the loopback transport): the one-GPU test of the exchange plan, bit for bit
// against the undistributed cycle (tests/test_dist_cpp.py).
//
// NCCL is loaded at run time (dlopen of libnccl.so.2, reusing the copy torch
// has loaded when there is one), so liblzb.so has no link-time NCCL
// dependency and a process that never builds a communicator never loads it.
// The reference (/root/reference/proj) is shared-memory only
// (SPEC.md:96 lists domain decomposition as a non-goal): no counterpart.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine.hpp"
#include "lzb.h"

namespace lzb {
namespace {

// ------------------------------------------------------------ NCCL loader
struct Nccl {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

template <typename F>
void sym(void* h, const char* name, F& out) {
    out = reinterpret_cast<F>(dlsym(h, name));
    if (!out) throw Error(LZB_ERR_NCCL, std::string("libnccl.so.2 lacks ") + name);
}

Nccl& nccl() {
    static Nccl n;
    if (n.h) return n;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's copy (torch's)
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw Error(LZB_ERR_NCCL, std::string("cannot load libnccl.so.2: ") + dlerror());
    sym(h, "ncclGetUniqueId", n.GetUniqueId);
    sym(h, "ncclCommInitRank", n.CommInitRank);
    sym(h, "ncclCommDestroy", n.CommDestroy);
    sym(h, "ncclSend", n.Send);
    sym(h, "ncclRecv", n.Recv);
    sym(h, "ncclBroadcast", n.Broadcast);
    sym(h, "ncclAllReduce", n.AllReduce);
    sym(h, "ncclGroupStart", n.GroupStart);
    sym(h, "ncclGroupEnd", n.GroupEnd);
    sym(h, "ncclGetErrorString", n.GetErrorString);
    n.h = h;
    return n;
}

void nc(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error(LZB_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}
void check(int rc) {
    if (rc != LZB_OK) throw Error(rc, lzb_last_error());
}

// ------------------------------------------------------------ slab plan
// Leaf cell rows (2D) / planes (3D) [r0, r1) of slab `rank`: boundaries at
// multiples of 3 so that every level-(D-1) patch lies in one slab, sizes
// balanced to one patch row (parallel.py slab_rows).
void slab_rows(int n, int world, int rank, int& r0, int& r1) {
    const int units = (n + 2) / 3, base = units / world, extra = units % world;
    const int u0 = rank * base + std::min(rank, extra);
    const int u1 = u0 + base + (rank < extra ? 1 : 0);
    r0 = std::min(n, 3 * u0);
    r1 = std::min(n, 3 * u1);
}
struct Slab {
    int v0, v1;  // leaf vertex rows / planes [v0, v1) (the last slab owns row N)
    int c0, c1;  // level-(D-1) vertex rows / planes it computes
};
Slab slab_of(int N, int world, int rank) {
    if (N / 3 < world) throw Error(LZB_ERR_INVALID, "too many slabs for the grid (3 leaf rows per slab at least)");
    Slab s;
    int r0, r1;
    slab_rows(N, world, rank, r0, r1);
    s.v0 = r0;
    s.v1 = r1 >= N ? N + 1 : r1;
    s.c0 = s.v0 / 3;
    s.c1 = (s.v1 + 2) / 3;
    return s;
}

// Result slots reduced by max: S_MAXN, S_MAXDELTA (non-negative double bits), S_MAXSAMPLES.
bool max_slot(int k) { return k == 11 || k == 14 || k == 15; }

// One grid of either dimension, seen through the C-ABI.
struct GridRef {
    lzb_grid* g2 = nullptr;
    lzb_grid3* g3 = nullptr;
    lzb_ctx* ctx = nullptr;
    int D = 0, N = 1, dims = 2;
    Slab slab{};
    static GridRef of(lzb_grid* g) {
        GridRef r;
        r.g2 = g;
        check(lzb_grid_info(g, &r.ctx, &r.D));
        r.dims = 2;
        r.N = 1;
        for (int i = 0; i < r.D; ++i) r.N *= 3;
        return r;
    }
    static GridRef of(lzb_grid3* g) {
        GridRef r;
        r.g3 = g;
        check(lzb_grid3_info(g, &r.ctx, &r.D));
        r.dims = 3;
        r.N = 1;
        for (int i = 0; i < r.D; ++i) r.N *= 3;
        return r;
    }
    cudaStream_t stream() const { return static_cast<cudaStream_t>(lzb_ctx_solve_stream(ctx)); }
    // elements of one row (2D) / plane (3D) of vertices of a level
    size_t unit(int level) const {
        size_t n = 1;
        for (int i = 0; i < level; ++i) n *= 3;
        return dims == 2 ? n + 1 : (n + 1) * (n + 1);
    }
    double* field(int level, int f) const {
        void* p = nullptr;
        check(g2 ? lzb_grid_device_view(g2, level, f, &p) : lzb_grid3_device_view(g3, level, f, &p));
        return static_cast<double*>(p);
    }
    void set_slab() const { check(g2 ? lzb_grid_set_slab(g2, slab.v0, slab.v1) : lzb_grid3_set_slab(g3, slab.v0, slab.v1)); }
    void phase(int k, int flags) const {
        check(g2 ? lzb_grid_dist_phase(g2, k, flags | 2) : lzb_grid3_dist_phase_flags(g3, k, flags | 2));
    }
    void* result() const {
        void* p = nullptr;
        check(g2 ? lzb_grid_dist_result_dev(g2, &p) : lzb_grid3_dist_result_dev(g3, &p));
        return p;
    }
};

// ------------------------------------------------------------ transports
// halo: rows [v0 - depth, v0) from the slab below, [v1, v1 + depth) from the
// slab above; gather: every slab's rows [c0, c1) to every slab; reduce: the
// device results summed (maxima for the three max slots) into each slab's
// result and returned to the host.
struct Transport {
    virtual ~Transport() = default;
    virtual void halo(std::vector<GridRef>& s, int level, int f, int depth) = 0;
    virtual void gather(std::vector<GridRef>& s, int level, int f) = 0;
    virtual void gather_planes(std::vector<GridRef>& s, int level) = 0;  // 3D class planes of level D-1
    // returns norm^2 and the 20 slots (2D) of the reduced result
    virtual double reduce(std::vector<GridRef>& s, uint64_t* slots) = 0;
};

// level-(D-1) cell planes [p0, p1) whose children are slab s's leaf cells
void coarse_cell_planes(const GridRef& g, int& p0, int& p1) {
    p0 = g.slab.v0 / 3;
    p1 = std::min(g.slab.v1, g.N) / 3;
}

struct NcclTransport : Transport {
    ncclComm_t comm;
    int rank, world;
    explicit NcclTransport(lzb_ctx* c) {
        if (!c->comm) throw Error(LZB_ERR_INVALID, "the context has no communicator (lzb_ctx_comm_init)");
        comm = static_cast<ncclComm_t>(c->comm);
        rank = c->comm_rank;
        world = c->comm_size;
    }
    void halo(std::vector<GridRef>& s, int level, int f, int depth) override {
        GridRef& g = s[0];
        const size_t n = g.unit(level);
        const int rows = static_cast<int>(g.N) + 1;
        double* t = g.field(level, f);
        cudaStream_t st = g.stream();
        Nccl& x = nccl();
        nc(x.GroupStart(), "ncclGroupStart");
        if (rank > 0) {
            const int a = std::max(g.slab.v0 - depth, 0), e = std::min(g.slab.v0 + depth, g.slab.v1);
            nc(x.Send(t + g.slab.v0 * n, (e - g.slab.v0) * n, ncclFloat64, rank - 1, comm, st), "ncclSend");
            nc(x.Recv(t + a * n, (g.slab.v0 - a) * n, ncclFloat64, rank - 1, comm, st), "ncclRecv");
        }
        if (rank + 1 < world) {
            const int b = std::min(g.slab.v1 + depth, rows), e = std::max(g.slab.v1 - depth, g.slab.v0);
            nc(x.Send(t + e * n, (g.slab.v1 - e) * n, ncclFloat64, rank + 1, comm, st), "ncclSend");
            nc(x.Recv(t + g.slab.v1 * n, (b - g.slab.v1) * n, ncclFloat64, rank + 1, comm, st), "ncclRecv");
        }
        nc(x.GroupEnd(), "ncclGroupEnd");
    }
    void gather(std::vector<GridRef>& s, int level, int f) override {
        GridRef& g = s[0];
        const size_t n = g.unit(level);
        double* t = g.field(level, f);
        cudaStream_t st = g.stream();
        Nccl& x = nccl();
        nc(x.GroupStart(), "ncclGroupStart");
        for (int r = 0; r < world; ++r) {
            const Slab o = slab_of(g.N, world, r);
            if (o.c1 > o.c0)
                nc(x.Broadcast(t + o.c0 * n, t + o.c0 * n, (o.c1 - o.c0) * n, ncclFloat64, r, comm, st), "ncclBroadcast");
        }
        nc(x.GroupEnd(), "ncclGroupEnd");
    }
    void gather_planes(std::vector<GridRef>& s, int level) override {
        GridRef& g = s[0];
        void* p = nullptr;
        check(lzb_grid3_level_ops(g.g3, level, &p));
        double* ops = static_cast<double*>(p);
        const size_t Nc = g.N / 3, plane = Nc * Nc, ncells = Nc * Nc * Nc;
        cudaStream_t st = g.stream();
        Nccl& x = nccl();
        nc(x.GroupStart(), "ncclGroupStart");
        for (int r = 0; r < world; ++r) {
            GridRef o = g;
            o.slab = slab_of(g.N, world, r);
            int p0, p1;
            coarse_cell_planes(o, p0, p1);
            if (p1 <= p0) continue;
            for (int q = 0; q < 27; ++q) {  // class plane q, its cell planes [p0, p1)
                double* b = ops + q * ncells + p0 * plane;
                nc(x.Broadcast(b, b, (p1 - p0) * plane, ncclFloat64, r, comm, st), "ncclBroadcast");
            }
        }
        nc(x.GroupEnd(), "ncclGroupEnd");
    }
    double reduce(std::vector<GridRef>& s, uint64_t* slots) override {
        GridRef& g = s[0];
        cudaStream_t st = g.stream();
        Nccl& x = nccl();
        char* res = static_cast<char*>(g.result());
        double norm2 = 0.0;
        if (g.dims == 3) {
            nc(x.AllReduce(res, res, 1, ncclFloat64, ncclSum, comm, st), "ncclAllReduce");
            LZB_CUDA(cudaMemcpyAsync(&norm2, res, sizeof(double), cudaMemcpyDeviceToHost, st));
            LZB_CUDA(cudaStreamSynchronize(st));
            return norm2;
        }
        // 2D result: double norm, then 20 u64 slots; sums in place, maxima through a copy
        if (!scratch_) LZB_CUDA(cudaMalloc(&scratch_, 20 * sizeof(uint64_t)));
        uint64_t* sl = reinterpret_cast<uint64_t*>(res + 8);
        LZB_CUDA(cudaMemcpyAsync(scratch_, sl, 20 * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
        nc(x.GroupStart(), "ncclGroupStart");
        nc(x.AllReduce(res, res, 1, ncclFloat64, ncclSum, comm, st), "ncclAllReduce");
        nc(x.AllReduce(sl, sl, 20, ncclUint64, ncclSum, comm, st), "ncclAllReduce");
        nc(x.AllReduce(scratch_, scratch_, 20, ncclUint64, ncclMax, comm, st), "ncclAllReduce");
        nc(x.GroupEnd(), "ncclGroupEnd");
        uint64_t sum[20], mx[20];
        LZB_CUDA(cudaMemcpyAsync(&norm2, res, sizeof(double), cudaMemcpyDeviceToHost, st));
        LZB_CUDA(cudaMemcpyAsync(sum, sl, sizeof sum, cudaMemcpyDeviceToHost, st));
        LZB_CUDA(cudaMemcpyAsync(mx, scratch_, sizeof mx, cudaMemcpyDeviceToHost, st));
        LZB_CUDA(cudaStreamSynchronize(st));
        for (int k = 0; k < 20; ++k) slots[k] = max_slot(k) ? mx[k] : sum[k];
        return norm2;
    }
    ~NcclTransport() override {
        if (scratch_) cudaFree(scratch_);
    }
    void* scratch_ = nullptr;
};

// All slabs in this process (one GPU, one solve stream): device copies.
struct LoopTransport : Transport {
    void halo(std::vector<GridRef>& s, int level, int f, int depth) override {
        const size_t n = s[0].unit(level);
        const int rows = s[0].N + 1;
        cudaStream_t st = s[0].stream();
        for (size_t i = 0; i < s.size(); ++i) {
            double* t = s[i].field(level, f);
            if (i > 0) {
                const int a = std::max(s[i].slab.v0 - depth, 0);
                LZB_CUDA(cudaMemcpyAsync(t + a * n, s[i - 1].field(level, f) + a * n, (s[i].slab.v0 - a) * n * 8,
                                         cudaMemcpyDeviceToDevice, st));
            }
            if (i + 1 < s.size()) {
                const int b = std::min(s[i].slab.v1 + depth, rows);
                LZB_CUDA(cudaMemcpyAsync(t + s[i].slab.v1 * n, s[i + 1].field(level, f) + s[i].slab.v1 * n,
                                         (b - s[i].slab.v1) * n * 8, cudaMemcpyDeviceToDevice, st));
            }
        }
    }
    void gather(std::vector<GridRef>& s, int level, int f) override {
        const size_t n = s[0].unit(level);
        cudaStream_t st = s[0].stream();
        for (auto& a : s)
            for (auto& b : s)
                if (&a != &b && a.slab.c1 > a.slab.c0)
                    LZB_CUDA(cudaMemcpyAsync(b.field(level, f) + a.slab.c0 * n, a.field(level, f) + a.slab.c0 * n,
                                             (a.slab.c1 - a.slab.c0) * n * 8, cudaMemcpyDeviceToDevice, st));
    }
    void gather_planes(std::vector<GridRef>& s, int level) override {
        const size_t Nc = s[0].N / 3, plane = Nc * Nc, ncells = Nc * Nc * Nc;
        cudaStream_t st = s[0].stream();
        for (auto& a : s) {
            int p0, p1;
            coarse_cell_planes(a, p0, p1);
            void *pa = nullptr, *pb = nullptr;
            check(lzb_grid3_level_ops(a.g3, level, &pa));
            for (auto& b : s) {
                if (&a == &b || p1 <= p0) continue;
                check(lzb_grid3_level_ops(b.g3, level, &pb));
                for (int q = 0; q < 27; ++q)
                    LZB_CUDA(cudaMemcpyAsync(static_cast<double*>(pb) + q * ncells + p0 * plane,
                                             static_cast<double*>(pa) + q * ncells + p0 * plane,
                                             (p1 - p0) * plane * 8, cudaMemcpyDeviceToDevice, st));
            }
        }
    }
    double reduce(std::vector<GridRef>& s, uint64_t* slots) override {
        cudaStream_t st = s[0].stream();
        double norm2 = 0.0;
        if (s[0].dims == 3) {
            for (auto& g : s) {
                double v = 0.0;
                LZB_CUDA(cudaMemcpyAsync(&v, g.result(), sizeof v, cudaMemcpyDeviceToHost, st));
                LZB_CUDA(cudaStreamSynchronize(st));
                norm2 += v;
            }
            return norm2;
        }
        for (int k = 0; k < 20; ++k) slots[k] = 0;
        for (auto& g : s) {
            struct {
                double norm;
                uint64_t s[20];
            } r;
            LZB_CUDA(cudaMemcpyAsync(&r, g.result(), sizeof r, cudaMemcpyDeviceToHost, st));
            LZB_CUDA(cudaStreamSynchronize(st));
            norm2 += r.norm;
            for (int k = 0; k < 20; ++k) slots[k] = max_slot(k) ? std::max(slots[k], r.s[k]) : slots[k] + r.s[k];
        }
        return norm2;
    }
};

// ------------------------------------------------------------ the cycle
// parallel.py dist_cycle / dist_cycle3, in C++ on the solve stream.
lzb_cycle_report dist_cycle(std::vector<GridRef>& s, Transport& x) {
    const int D = s[0].D, dims = s[0].dims;
    for (size_t i = 0; i < s.size(); ++i) s[i].phase(0, (dims == 2 && s[i].slab.v0 == 0) ? 1 : 0);
    x.halo(s, D, LZB_V_RHAT, 3);  // the restriction reads r-hat 3 rows beyond the slab
    for (auto& g : s) g.phase(1, 0);
    x.gather(s, D - 1, LZB_V_FL);  // the restricted load of level D-1
    for (auto& g : s) g.phase(2, 0);
    uint64_t slots[20];
    const double norm2 = x.reduce(s, slots);
    std::vector<lzb_cycle_report> reps(s.size());
    for (size_t i = 0; i < s.size(); ++i)
        check(dims == 2 ? lzb_grid_dist_report(s[i].g2, norm2, slots, &reps[i])
                        : lzb_grid3_dist_report(s[i].g3, norm2, &reps[i]));
    const lzb_cycle_report rep = reps[0];
    if (rep.status == LZB_CONTINUE || rep.status == LZB_TIMEOUT) {
        int pi = 0;
        if (dims == 2) {
            lzb_grid_desc d;
            check(lzb_grid_desc_of(s[0].g2, &d));
            pi = d.variant == LZB_ADAFAC_PI;
        } else {
            pi = lzb_grid3_variant(s[0].g3) == LZB_ADAFAC_PI;
        }
        for (auto& g : s) g.phase(3, 0);
        if (pi) x.gather(s, D - 1, LZB_V_AUX);  // the injected residual of level D-1
        for (auto& g : s) g.phase(4, 0);
        x.gather(s, D - 1, LZB_V_U);  // the injected solution of level D-1
        for (auto& g : s) g.phase(5, 0);
        x.halo(s, D, LZB_V_U, 1);  // leaf u one row beyond the slab
    }
    LZB_CUDA(cudaStreamSynchronize(s[0].stream()));
    return rep;
}

// assign the slabs (rank r of world) and tell the grids
void plan(std::vector<GridRef>& s, int world, const int* ranks) {
    for (size_t i = 0; i < s.size(); ++i) {
        s[i].slab = slab_of(s[i].N, world, ranks ? ranks[i] : static_cast<int>(i));
        s[i].set_slab();
    }
}

// z-slab sharded 3D assembly (parallel.py distributed_assemble3): the leaf
// cell planes each slab's cycle reads, its level-(D-1) Galerkin planes, one
// exchange of those, the levels below recomputed everywhere
void dist_assemble3(std::vector<GridRef>& s, Transport& x, int n) {
    const int D = s[0].D;
    for (auto& g : s) {
        check(lzb_grid3_assemble_planes(g.g3, n, std::max(g.slab.v0 - 1, 0), std::min(g.slab.v1, g.N)));
        int p0, p1;
        coarse_cell_planes(g, p0, p1);
        check(lzb_grid3_galerkin_planes(g.g3, D - 1, p0, p1));
    }
    x.gather_planes(s, D - 1);
    for (auto& g : s) check(lzb_grid3_coarse_below(g.g3, D - 1));
    LZB_CUDA(cudaStreamSynchronize(s[0].stream()));
}

// 2D slab assembly: each slab integrates its leaf cell rows, then every
// slab's rows of the leaf state (operators, markers, change epochs; the
// compressed records when the residual reads them) go to every slab
void dist_assemble2(std::vector<GridRef>& s, Transport* nx, int n, int world, int rank) {
    const int D = s[0].D, N = s[0].N;
    cudaStream_t st = s[0].stream();
    struct Arr {
        char* p;
        size_t per_cell;
    };
    std::vector<std::vector<Arr>> arrs(s.size());
    for (size_t i = 0; i < s.size(); ++i) {
        int r0, r1;
        slab_rows(N, world, nx ? rank : static_cast<int>(i), r0, r1);
        if (r1 > r0) check(lzb_grid_assemble_rows(s[i].g2, n, r0, r1));
        void *op, *p1, *nn, *p3, *ep, *chg, *pl = nullptr, *cp3 = nullptr;
        int w = 0;
        check(lzb_grid_cell_arrays(s[i].g2, D, &op, &p1, &nn, &p3, &ep, &chg));
        check(lzb_grid_plane_arrays(s[i].g2, &pl, &cp3, &w));
        arrs[i] = {{static_cast<char*>(op), 128}, {static_cast<char*>(p1), 4}, {static_cast<char*>(nn), 4},
                   {static_cast<char*>(p3), 1}, {static_cast<char*>(ep), 4}, {static_cast<char*>(chg), 4}};
        if (w) {
            arrs[i].push_back({static_cast<char*>(pl), static_cast<size_t>(16 * w)});
            arrs[i].push_back({static_cast<char*>(cp3), 1});
        }
    }
    const size_t row = static_cast<size_t>(N);  // cells per cell row
    if (nx) {
        NcclTransport& t = *static_cast<NcclTransport*>(nx);
        Nccl& x = nccl();
        nc(x.GroupStart(), "ncclGroupStart");
        for (int r = 0; r < world; ++r) {
            int r0, r1;
            slab_rows(N, world, r, r0, r1);
            if (r1 <= r0) continue;
            for (auto& a : arrs[0]) {
                char* b = a.p + r0 * row * a.per_cell;
                nc(x.Broadcast(b, b, (r1 - r0) * row * a.per_cell, ncclUint8, r, t.comm, st), "ncclBroadcast");
            }
        }
        nc(x.GroupEnd(), "ncclGroupEnd");
    } else {
        for (size_t i = 0; i < s.size(); ++i) {
            int r0, r1;
            slab_rows(N, world, static_cast<int>(i), r0, r1);
            for (size_t j = 0; j < s.size(); ++j) {
                if (i == j || r1 <= r0) continue;
                for (size_t k = 0; k < arrs[i].size(); ++k) {
                    const size_t off = r0 * row * arrs[i][k].per_cell, len = (r1 - r0) * row * arrs[i][k].per_cell;
                    LZB_CUDA(cudaMemcpyAsync(arrs[j][k].p + off, arrs[i][k].p + off, len, cudaMemcpyDeviceToDevice, st));
                }
            }
        }
    }
    LZB_CUDA(cudaStreamSynchronize(st));
    for (auto& g : s) check(lzb_grid_invalidate(g.g2));
}

}  // namespace

void release_comm(lzb_ctx* c) {
    if (c && c->comm) {
        nccl().CommDestroy(static_cast<ncclComm_t>(c->comm));
        c->comm = nullptr;
    }
}

}  // namespace lzb

using namespace lzb;

extern "C" {

int lzb_nccl_unique_id(uint8_t* out128) { LZB_RANGE("lzb_nccl_unique_id");
    return guarded([&] {
        ncclUniqueId id;
        nc(nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out128, &id, sizeof id);
    });
}

int lzb_ctx_comm_init(lzb_ctx* ctx, const uint8_t* id128, int nranks, int rank) { LZB_RANGE("lzb_ctx_comm_init");
    return guarded([&] {
        if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(LZB_ERR_INVALID, "bad rank / nranks");
        release_comm(ctx);
        LZB_CUDA(cudaSetDevice(ctx->device));
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof id);
        ncclComm_t comm = nullptr;
        nc(nccl().CommInitRank(&comm, nranks, id, rank), "ncclCommInitRank");
        ctx->comm = comm;
        ctx->comm_rank = rank;
        ctx->comm_size = nranks;
    });
}

int lzb_ctx_comm_info(lzb_ctx* ctx, int* rank, int* nranks) {
    return guarded([&] {
        *rank = ctx->comm ? ctx->comm_rank : 0;
        *nranks = ctx->comm ? ctx->comm_size : 1;
    });
}

int lzb_grid_dist_cycle(lzb_grid* g, lzb_cycle_report* out) {
    return guarded([&] {
        std::vector<GridRef> s{GridRef::of(g)};
        NcclTransport x(s[0].ctx);
        plan(s, x.world, &x.rank);
        *out = dist_cycle(s, x);
    });
}

int lzb_grid_dist_cycle_loopback(lzb_grid* const* slabs, int nslabs, lzb_cycle_report* out) { LZB_RANGE("lzb_grid_dist_cycle_loopback");
    return guarded([&] {
        std::vector<GridRef> s;
        for (int i = 0; i < nslabs; ++i) s.push_back(GridRef::of(slabs[i]));
        LoopTransport x;
        plan(s, nslabs, nullptr);
        *out = dist_cycle(s, x);
    });
}

int lzb_grid_dist_assemble(lzb_grid* g, int n) { LZB_RANGE("lzb_grid_dist_assemble");
    return guarded([&] {
        std::vector<GridRef> s{GridRef::of(g)};
        NcclTransport x(s[0].ctx);
        dist_assemble2(s, &x, n, x.world, x.rank);
    });
}

int lzb_grid_dist_assemble_loopback(lzb_grid* const* slabs, int nslabs, int n) { LZB_RANGE("lzb_grid_dist_assemble_loopback");
    return guarded([&] {
        std::vector<GridRef> s;
        for (int i = 0; i < nslabs; ++i) s.push_back(GridRef::of(slabs[i]));
        dist_assemble2(s, nullptr, n, nslabs, 0);
    });
}

int lzb_grid3_create_slab(lzb_ctx* ctx, int depth, const lzb_field3* f, double delta_max, int fixed_p3,
                          int plane_width, int nslabs, int slab, lzb_grid3** out) { LZB_RANGE("lzb_grid3_create_slab");
    return guarded([&] {
        if (depth < 1 || depth > 6) throw Error(LZB_ERR_INVALID, "slab grids need depth in 1..6");
        if (nslabs < 1 || slab < 0 || slab >= nslabs) throw Error(LZB_ERR_INVALID, "bad slab / nslabs");
        int N = 1;
        for (int i = 0; i < depth; ++i) N *= 3;
        const Slab s = slab_of(N, nslabs, slab);
        // the leaf cell layers the slab's kernels read: its vertex planes' cells
        // and one layer below (residual, Jacobi diagonal); its level-(D-1)
        // Galerkin planes' children lie inside
        check(lzb_grid3_create_window(ctx, depth, f, delta_max, fixed_p3, plane_width, std::max(s.v0 - 1, 0),
                                      std::min(s.v1, N), out));
    });
}
int lzb_grid3_dist_cycle(lzb_grid3* g, lzb_cycle_report* out) {
    return guarded([&] {
        std::vector<GridRef> s{GridRef::of(g)};
        NcclTransport x(s[0].ctx);
        plan(s, x.world, &x.rank);
        *out = dist_cycle(s, x);
    });
}

int lzb_grid3_dist_cycle_loopback(lzb_grid3* const* slabs, int nslabs, lzb_cycle_report* out) { LZB_RANGE("lzb_grid3_dist_cycle_loopback");
    return guarded([&] {
        std::vector<GridRef> s;
        for (int i = 0; i < nslabs; ++i) s.push_back(GridRef::of(slabs[i]));
        LoopTransport x;
        plan(s, nslabs, nullptr);
        *out = dist_cycle(s, x);
    });
}

int lzb_grid3_dist_assemble(lzb_grid3* g, int n) { LZB_RANGE("lzb_grid3_dist_assemble");
    return guarded([&] {
        std::vector<GridRef> s{GridRef::of(g)};
        NcclTransport x(s[0].ctx);
        plan(s, x.world, &x.rank);
        dist_assemble3(s, x, n);
    });
}

int lzb_grid3_dist_assemble_loopback(lzb_grid3* const* slabs, int nslabs, int n) { LZB_RANGE("lzb_grid3_dist_assemble_loopback");
    return guarded([&] {
        std::vector<GridRef> s;
        for (int i = 0; i < nslabs; ++i) s.push_back(GridRef::of(slabs[i]));
        LoopTransport x;
        plan(s, nslabs, nullptr);
        dist_assemble3(s, x, n);
    });
}

}  // extern "C"

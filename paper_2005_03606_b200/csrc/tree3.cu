// tree3.cu — BASELINE configs[3] (C4), the assembly half: a 3D adaptive
// spacetree (k = 3) refined to level lmax inside a sphere and to level lbase
// elsewhere, its leaves at three levels with hanging nodes between them, the
// smoothed-interface sphere field eps (LZB_F3_SPHERE), fixed-p assembly of
// every leaf with the 27-class record coding of grid3.cu, and the delayed
// re-assembly of the interface shell at rising p. The reference is 2D only
// (types.hpp:13); its adaptive mesh is mesh.cpp:66-129,236-312 (cells exist
// only under refined parents, leaves on several levels). The cycle on the
// adaptive tree (hanging-node interpolation, mesh.cpp:182-224, in 3D) is not
// built yet.
//
// Leaves are a flat list (level, cx, cy, cz), level-major, in the order the
// levels are generated (parents in order, children z-major); operators are
// class planes over the leaf index (value q of leaf i at q * nleaves + i).
#include <algorithm>
#include <cmath>
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
    const int p3 = fixed_p3 ? fixed_p3 : choose_precision_regular<27>(sur, delta_max);
    if (p3 < 0) {
        atomicExch(err, 1);
        return;
    }
    double delta = 0.0;
#pragma unroll
    for (int q = 0; q < 27; ++q) {
        double rt;
        if (!roundtrip_fast(sur[q], p3, rt)) {
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
    int64_t set_shell(double band) {
        if (!(band >= 0.0)) throw Error(LZB_ERR_INVALID, "shell band must be >= 0");
        std::vector<int32_t> list;
        for (int64_t i = 0; i < n_leaves_; ++i) {
            const int4& c = leaves_[i];
            const double h = HL_.h[c.x];
            double lo, hi;
            box_range(c.y * h, c.z * h, c.w * h, h, lo, hi);
            if (hi >= rad_ - band && lo <= rad_ + band) list.push_back(static_cast<int32_t>(i));
        }
        n_shell_ = static_cast<int64_t>(list.size());
        shell_.alloc(std::max<int64_t>(n_shell_, 1));
        if (n_shell_)
            LZB_CUDA(cudaMemcpy(shell_.p, list.data(), n_shell_ * sizeof(int32_t), cudaMemcpyHostToDevice));
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
        if (lxyz) std::memcpy(lxyz, leaves_.data() + first, count * sizeof(int4));
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
    std::vector<int4> leaves_;
    int64_t per_level_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t n_leaves_ = 0, n_shell_ = 0;
    DevBuf<double> table_, op_;
    DevBuf<int4> dleaves_;
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
                     lzb_tree3** out) {
    return lzb::guarded([&] {
        auto t = std::make_unique<lzb_tree3>();
        t->t = std::make_unique<lzb::Tree3>(ctx, lbase, lmax, *f, delta_max, fixed_p3);
        *out = t.release();
    });
}
int lzb_tree3_destroy(lzb_tree3* t) {
    return lzb::guarded([&] { delete t; });
}
int lzb_tree3_counts(lzb_tree3* t, int64_t* per_level, int64_t* total) {
    return lzb::guarded([&] { t->t->counts(per_level, total); });
}
int lzb_tree3_assemble(lzb_tree3* t, int n) {
    return lzb::guarded([&] {
        t->t->assemble(n, false);
        t->t->sync();
    });
}
int lzb_tree3_set_shell(lzb_tree3* t, double band, int64_t* count) {
    return lzb::guarded([&] { *count = t->t->set_shell(band); });
}
int lzb_tree3_assemble_shell(lzb_tree3* t, int n) {
    return lzb::guarded([&] {
        t->t->assemble(n, true);
        t->t->sync();
    });
}
int lzb_tree3_stats(lzb_tree3* t, lzb_compression_stats* out) {
    return lzb::guarded([&] { *out = t->t->stats(); });
}
int lzb_tree3_cells(lzb_tree3* t, int64_t first, int64_t count, double* ops, int32_t* p3, int32_t* n,
                    int32_t* lxyz) {
    return lzb::guarded([&] { t->t->cells(first, count, ops, p3, n, lxyz); });
}

}  // extern "C"

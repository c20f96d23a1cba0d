// lazymg_b200.hpp — header-only C++ host shim over the lzb C-ABI.
//
// The reference's call sites (/root/reference/proj/src/*.cpp) use the lazymg::
// C++ API. This header offers the same names and semantics on top of
// liblzb.so, so a reference-side integration replaces `#include "lazymg/..."`
// by this header and links -llzb. It lives in its own
// namespace (lazymg_b200) so that it can be linked next to the reference
// without ODR clashes.
//
// Status codes are rethrown as the reference's exception types
// (types.hpp:68-76): protocol_error, corrupt_stream_error, resource_error,
// std::invalid_argument, std::runtime_error.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "lzb.h"

namespace lazymg_b200 {

struct protocol_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct corrupt_stream_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct resource_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == LZB_OK) return;
    std::string msg = lzb_last_error();
    switch (rc) {
        case LZB_ERR_PROTOCOL: throw protocol_error(msg);
        case LZB_ERR_CORRUPT: throw corrupt_stream_error(msg);
        case LZB_ERR_RESOURCE: throw resource_error(msg);
        case LZB_ERR_INVALID: throw std::invalid_argument(msg);
        default: throw std::runtime_error(msg);
    }
}

/// Mat4 of the reference (types.hpp:23-50): 16 doubles, row-major, corners SW,SE,NW,NE.
using Mat4 = std::array<double, 16>;
using TransferBlock = std::array<double, 64>;  // w[L*4 + c] (types.hpp:62-66)

/// Assembled 3x3 vertex stencil, index (dy+1)*3 + (dx+1) (types.hpp:53-58).
struct Stencil9 {
    std::array<double, 9> s{};
    double& at(int dx, int dy) { return s[(dy + 1) * 3 + (dx + 1)]; }
    double at(int dx, int dy) const { return s[(dy + 1) * 3 + (dx + 1)]; }
    double centre() const { return at(0, 0); }
};
/// scatter_row (element.hpp:53)
inline void scatter_row(const Mat4& element, int corner, Stencil9& stencil) {
    check(lzb_scatter_row(element.data(), corner, stencil.s.data()));
}

struct ElementMatrix {  // element.hpp:12-15
    Mat4 m{};
    int n = 0;
};
struct CellBox {  // element.hpp:25-27
    double x0 = 0.0, y0 = 0.0, h = 1.0;
};

/// Device + solve / assembly streams. One per process and GPU.
class Context {
public:
    explicit Context(int device = 0) { check(lzb_ctx_create(device, &ctx_)); }
    ~Context() { lzb_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    lzb_ctx* get() const { return ctx_; }

private:
    lzb_ctx* ctx_ = nullptr;
};

/// integrate_element(box, eps, n) (element.hpp:36-49): bit-identical to the
/// reference with LZB_INTEGRATE_EXACT.
inline ElementMatrix integrate_element(Context& ctx, const CellBox& box, const lzb_field& eps, int n,
                                       int integration = LZB_INTEGRATE_EXACT) {
    ElementMatrix out;
    out.n = n;
    int32_t nn = n;
    check(lzb_integrate_elements(ctx.get(), &eps, 1, &box.x0, &box.y0, &box.h, &nn, out.m.data(),
                                 integration));
    return out;
}

/// Batched form: the GPU-native entry the reference's per-cell loops map to.
inline std::vector<Mat4> integrate_elements(Context& ctx, const lzb_field& eps,
                                            const std::vector<CellBox>& boxes,
                                            const std::vector<int32_t>& n,
                                            int integration = LZB_INTEGRATE_EXACT) {
    std::vector<double> x0, y0, h;
    for (const auto& b : boxes) {
        x0.push_back(b.x0);
        y0.push_back(b.y0);
        h.push_back(b.h);
    }
    std::vector<Mat4> out(boxes.size());
    check(lzb_integrate_elements(ctx.get(), &eps, static_cast<int64_t>(boxes.size()), x0.data(), y0.data(),
                                 h.data(), n.data(), out.front().data(), integration));
    return out;
}

namespace codec {  // codec.hpp:17-37
inline constexpr int max_p3 = 8;
inline constexpr int mantissa_bits(int p3) { return 8 * (p3 - 1) - 1; }

inline void encode_value(Context& ctx, double x, int p3, uint8_t* out) {
    if (p3 == 0) return;
    check(lzb_codec_encode(ctx.get(), 1, &x, p3, out));
}
inline double decode_value(Context& ctx, const uint8_t* in, int p3) {
    double v = 0.0;
    check(lzb_codec_decode(ctx.get(), 1, in, p3, &v));
    return v;
}
inline double roundtrip(Context& ctx, double x, int p3) {
    if (p3 == 0) return 0.0;
    uint8_t buf[8];
    encode_value(ctx, x, p3, buf);
    return decode_value(ctx, buf, p3);
}
inline int choose_precision(Context& ctx, std::span<const double> surplus, double delta_max) {
    int32_t p3 = 0;
    check(lzb_codec_choose_precision(ctx.get(), 1, static_cast<int32_t>(surplus.size()), surplus.data(),
                                     delta_max, &p3));
    return p3;
}
}  // namespace codec

inline uint8_t pack_header(int32_t p1, bool p2, int p3) { return lzb_pack_header(p1, p2 ? 1 : 0, p3); }
inline void unpack_header(uint8_t h, int& p1_class, bool& p2, int& p3) {
    int b = 0;
    check(lzb_unpack_header(h, &p1_class, &b, &p3));
    p2 = b != 0;
}

inline TransferBlock geometric_prolongation() {
    TransferBlock P{};
    lzb_geometric_prolongation(P.data());
    return P;
}
/// galerkin_coarse_element(children, P) (transfer.hpp:31).
inline Mat4 galerkin_coarse_element(Context& ctx, const std::array<Mat4, 9>& children,
                                    const TransferBlock& P) {
    Mat4 out{};
    check(lzb_galerkin(ctx.get(), 1, children.front().data(), P.data(), out.data()));
    return out;
}
/// boxmg_prolongation(children) (transfer.hpp:28); returns the block, fallback rows in *fb.
inline TransferBlock boxmg_prolongation(Context& ctx, const std::array<Mat4, 9>& children,
                                        int* fb = nullptr) {
    TransferBlock P{};
    int32_t f = 0;
    check(lzb_boxmg(ctx.get(), 1, children.front().data(), P.data(), &f));
    if (fb) *fb = f;
    return P;
}

/// Mesh + CellStream + Assembler + AdditiveSolver of one regular 2D spacetree
/// (mesh.hpp:64, stream.hpp:72, assembly.hpp:38, solver.hpp:72), resident on
/// the GPU. Cells and vertices are addressed by (level, cx, cy) / (level, ix, iy).
class Grid {
public:
    Grid(Context& ctx, const lzb_grid_desc& desc) : desc_(desc) { check(lzb_grid_create(ctx.get(), &desc, &g_)); }
    ~Grid() { lzb_grid_destroy(g_); }
    Grid(const Grid&) = delete;
    Grid& operator=(const Grid&) = delete;

    void init_noise(uint64_t seed) { check(lzb_grid_init_noise(g_, seed)); }          // problem.hpp:50
    void eager_setup() { check(lzb_grid_eager_setup(g_)); }                            // assembly.hpp:47
    lzb_cycle_report step() {                                                          // solver.hpp:78
        lzb_cycle_report r;
        check(lzb_grid_step(g_, &r));
        return r;
    }
    std::vector<lzb_cycle_report> run_cycles() {                                       // solver.hpp:79
        std::vector<lzb_cycle_report> out(static_cast<size_t>(desc_.max_cycles) + 1);
        int n = 0;
        check(lzb_grid_run(g_, out.data(), static_cast<int>(out.size()), &n));
        out.resize(static_cast<size_t>(n) < out.size() ? n : out.size());
        return out;
    }
    double residual_pass() {  // solver.hpp:94
        double v = 0.0;
        check(lzb_grid_pass(g_, 1, &v));
        return v;
    }
    void assembly_pass() { check(lzb_grid_pass(g_, 0, nullptr)); }
    void update_pass() { check(lzb_grid_pass(g_, 2, nullptr)); }
    void prolong_corrections() { check(lzb_grid_pass(g_, 3, nullptr)); }
    void finish_cycle_sync() { check(lzb_grid_pass(g_, 4, nullptr)); }
    void drain() { check(lzb_grid_pass(g_, 7, nullptr)); }                              // TaskPool::drain_all

    /// CellStream::publish_element + p1 store; adaptive_step (assembly.hpp:40).
    void publish_element(int level, int cx, int cy, const Mat4& m, int n, int32_t p1) {
        check(lzb_grid_publish_element(g_, level, cx, cy, m.data(), n, p1));
    }
    void adaptive_step(int level, int cx, int cy) { check(lzb_grid_adaptive_step(g_, level, cx, cy)); }
    lzb_compression_stats compression_stats() {                                        // stream.hpp:118
        lzb_compression_stats s;
        check(lzb_grid_stats(g_, &s));
        return s;
    }
    void save(const std::string& path) { check(lzb_grid_save(g_, path.c_str())); }     // stream.hpp:123
    void load(const std::string& path) { check(lzb_grid_load(g_, path.c_str())); }     // stream.hpp:125
    std::vector<double> vertices(int level, int field) {
        int N = 1;
        for (int i = 0; i < level; ++i) N *= 3;
        std::vector<double> v(static_cast<size_t>(N + 1) * (N + 1));
        check(lzb_grid_vertices(g_, level, field, v.data(), 0));
        return v;
    }
    /// assemble_vertex_stencil (assembly.hpp:69-71) of vertex (ix, iy) of a level.
    Stencil9 assemble_vertex_stencil(int level, int ix, int iy, bool require_payload = false) {
        int N = 1;
        for (int i = 0; i < level; ++i) N *= 3;
        std::vector<double> all(static_cast<size_t>(N + 1) * (N + 1) * 9);
        check(lzb_grid_vertex_stencils(g_, level, require_payload ? 1 : 0, all.data()));
        Stencil9 st;
        for (int k = 0; k < 9; ++k) st.s[k] = all[9 * (static_cast<size_t>(iy) * (N + 1) + ix) + k];
        return st;
    }
    lzb_grid* raw() const { return g_; }

private:
    lzb_grid_desc desc_;
    lzb_grid* g_ = nullptr;
};

/// run_experiment(parse_config_file(path)) (experiment.hpp:75,89); returns the exit code.
inline int run_experiment(const std::string& cfg_path) {
    int ec = 0, n = 0;
    check(lzb_run_experiment_file(cfg_path.c_str(), &ec, &n));
    return ec;
}
inline std::string emit_table(const std::vector<std::string>& csv_paths) {
    std::string joined;
    for (const auto& p : csv_paths) joined += p + "\n";
    std::string out(1 << 20, '\0');
    check(lzb_emit_table(joined.c_str(), out.data(), static_cast<int64_t>(out.size())));
    out.resize(std::char_traits<char>::length(out.c_str()));
    return out;
}
inline std::string compare_runs(const std::string& a, const std::string& b) {
    std::string out(1 << 16, '\0');
    check(lzb_compare_runs(a.c_str(), b.c_str(), out.data(), static_cast<int64_t>(out.size())));
    out.resize(std::char_traits<char>::length(out.c_str()));
    return out;
}

}  // namespace lazymg_b200

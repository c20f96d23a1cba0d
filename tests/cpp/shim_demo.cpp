// A reference-style host program written against include/lazymg_b200.hpp
// (the drop-in C++ shim over the lzb C-ABI). Mirrors checks of the reference
// tests (test_element.cpp:9-21, test_codec.cpp:21-35, test_experiment.cpp).
// Exit code 0 = all checks passed, 77 = no GPU (skipped), 1 = failure.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "lazymg_b200.hpp"

namespace lm = lazymg_b200;

static int fails = 0;
#define CHECK(c)                                                    \
    do {                                                            \
        if (!(c)) {                                                 \
            std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++fails;                                                \
        }                                                           \
    } while (0)

int main(int argc, char** argv) {
    std::unique_ptr<lm::Context> ctx;
    try {
        ctx = std::make_unique<lm::Context>(0);
    } catch (const std::runtime_error& e) {
        std::printf("no device: %s\n", e.what());
        return 77;
    }
    // unit stiffness (test_element.cpp:9-21)
    lzb_field one{};
    one.kind = LZB_FIELD_CONSTANT;
    one.value = 1.0;
    lm::ElementMatrix em = lm::integrate_element(*ctx, {0, 0, 1}, one, 1);
    const double e = 1.0 / 6.0;
    const double want[16] = {4 * e, -e, -e, -2 * e, -e, 4 * e, -2 * e, -e,
                             -e, -2 * e, 4 * e, -e, -2 * e, -e, -e, 4 * e};
    for (int i = 0; i < 16; ++i) CHECK(std::fabs(em.m[i] - want[i]) <= 1e-14);
    // codec known answers (test_codec.cpp:21-35)
    uint8_t b[8];
    lm::codec::encode_value(*ctx, 1.0, 2, b);
    CHECK(b[0] == 0x00 && b[1] == 0x00);
    lm::codec::encode_value(*ctx, -0.75, 2, b);
    CHECK(b[0] == 0xC0 && static_cast<int8_t>(b[1]) == -1);
    CHECK(lm::codec::decode_value(*ctx, b, 2) == -0.75);
    bool threw = false;
    try {
        lm::codec::encode_value(*ctx, NAN, 4, b);
    } catch (const lm::protocol_error&) {
        threw = true;
    }
    CHECK(threw);
    const double ones[4] = {1.2345678901, -0.987654321, 1.5, 0.7777777};
    CHECK(lm::codec::choose_precision(*ctx, std::span<const double>(ones, 4), 1e-8) == 5);
    // a grid driven through the shim: eager run to convergence (test_solver.cpp:183-211)
    lzb_grid_desc d{};
    d.dim = 2;
    d.depth = 2;
    d.field = one;
    d.delta_max = 1e-8;
    d.variant = LZB_ADAFAC_PI;
    d.omega = 0.7;
    d.target = 1e-10;
    d.divergence = 1e2;
    d.max_cycles = 400;
    d.mode = LZB_EAGER;
    d.termination_c = 0.01;
    {
        lm::Grid g(*ctx, d);
        g.init_noise(0);
        auto reps = g.run_cycles();
        CHECK(!reps.empty() && reps.back().status == LZB_CONVERGED);
        CHECK(reps.size() == 67);  // golden exp_cmp_eager.csv: 67 cycles
        auto st = g.compression_stats();
        CHECK(st.fine_cells == 81 && st.fine_factor_totals == 128.0);
        // assembled interior stencil on the eps = 1 mesh (test_element.cpp:83-107)
        lm::Stencil9 s9 = g.assemble_vertex_stencil(2, 4, 4, true);
        for (int dx = -1; dx <= 1; ++dx)
            for (int dy = -1; dy <= 1; ++dy)
                CHECK(std::fabs(s9.at(dx, dy) - ((dx == 0 && dy == 0) ? 8.0 / 3.0 : -1.0 / 3.0)) <= 1e-12);
        lm::Stencil9 byhand;
        for (int c = 0; c < 4; ++c) lm::scatter_row(lm::Mat4(em.m), 3 - c, byhand);  // the 4 cells around a vertex
        for (int k = 0; k < 9; ++k) CHECK(std::fabs(byhand.s[k] - s9.s[k]) <= 1e-12);
    }
    // the experiment layer (config file -> CSV -> table)
    if (argc > 2) {
        int ec = lm::run_experiment(argv[1]);
        CHECK(ec == 3);  // exp_table_t1: 4 cycles, timeout
        std::string t = lm::emit_table({argv[2]});
        CHECK(t.find("theta = 1") != std::string::npos && t.find("128.00") != std::string::npos);
    }
    std::printf("%s (%d failed checks)\n", fails ? "FAIL" : "OK", fails);
    return fails ? 1 : 0;
}

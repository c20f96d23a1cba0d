// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// An extern "C" harness around the UNMODIFIED reference library, which
// oracle/Makefile compiles in place from /root/reference/proj/src/*.cpp into
// oracle/_ref/liblazymg_ref.so. tests/ and bench.py (--impl reference,
// cpu_baseline) load it through ctypes; nothing else may.
//
// Everything below calls the reference's own public API
// (/root/reference/proj/include/lazymg/*.hpp). The only restated pieces are
// the two BASELINE.json eps kinds the reference cannot express
// (checkerboard, sinusoid); they are passed to the
// reference's own integrate_element template (element.hpp:36-49), which
// accepts any callable.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <numbers>
#include <sstream>
#include <string>
#include <thread>
#include <unistd.h>
#include <vector>

#include "lazymg/assembly.hpp"
#include "lazymg/codec.hpp"
#include "lazymg/element.hpp"
#include "lazymg/experiment.hpp"
#include "lazymg/mesh.hpp"
#include "lazymg/problem.hpp"
#include "lazymg/solver.hpp"
#include "lazymg/stream.hpp"
#include "lazymg/transfer.hpp"
#include "lzb_types.h"

using namespace lazymg;

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
    g_err = what;
    return code;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return LZB_OK;
    } catch (const protocol_error& e) {
        return fail(LZB_ERR_PROTOCOL, e.what());
    } catch (const corrupt_stream_error& e) {
        return fail(LZB_ERR_CORRUPT, e.what());
    } catch (const resource_error& e) {
        return fail(LZB_ERR_RESOURCE, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(LZB_ERR_INVALID, e.what());
    } catch (const std::exception& e) {
        return fail(LZB_ERR_IO, e.what());
    }
}

// eps callable: kinds 0-2 go through the reference MaterialField, 3-4 are the
// BASELINE restatements (same expressions as the oracle and the device code).
struct FieldFn {
    lzb_field f;
    MaterialField mat;
    explicit FieldFn(const lzb_field& d) : f(d) {
        switch (d.kind) {
            case LZB_FIELD_THETA: mat = MaterialField::theta_field(d.theta); break;
            case LZB_FIELD_QUADRANT: mat = MaterialField::quadrant(d.eps_low); break;
            default: mat = MaterialField::constant(d.value); break;
        }
    }
    double operator()(double x, double y) const {
        switch (f.kind) {
            case LZB_FIELD_CHECKER: {
                int b = f.blocks;
                int bx = static_cast<int>(b * x), by = static_cast<int>(b * y);
                bx = std::min(bx, b - 1);
                by = std::min(by, b - 1);
                return f.table[bx * b + by];
            }
            case LZB_FIELD_SINUSOID:
                return 1.0 + f.amp * std::sin(f.freq * std::numbers::pi * x) *
                                 std::sin(f.freq * std::numbers::pi * y);
            default: return mat(x, y);
        }
    }
};

struct Rig {
    ExperimentConfig cfg;
    Mesh mesh;
    ProblemInstance problem;
    CellStream stream;
    TaskPool pool;
    Assembler assembler;
    AdditiveSolver solver;
    explicit Rig(const ExperimentConfig& c)
        : cfg(c),
          mesh(build_initial_mesh(c.depth)),
          problem(c.problem()),
          stream(mesh, problem.material, c.compression_threshold),
          pool(c.scheduler_config()),
          assembler(stream, c.assembly_config(), pool),
          solver(mesh, stream, assembler, pool, problem, c.solver_config(),
                 c.multilevel_config()) {
        // run_experiment's forced-task workload hook (experiment.cpp:260-270),
        // installed the same way through the public on_cycle_start member
        if (cfg.forced_task_fraction > 0.0) {
            solver.on_cycle_start = [this] {
                for (std::size_t id = 0; id < mesh.cell_count(); ++id) {
                    const Cell& cell = mesh.cell(static_cast<int32_t>(id));
                    if (cell.refined) continue;
                    const double roll = static_cast<double>(splitmix64(0x6f4ce1a3u ^ id) >> 11) * 0x1.0p-53;
                    if (roll < cfg.forced_task_fraction) assembler.spawn_forced(cell.id, cfg.forced_task_n);
                }
            };
        }
    }
};

void fill_report(const CycleReport& r, lzb_cycle_report* o) {
    std::memset(o, 0, sizeof *o);
    o->cycle = r.cycle;
    o->status = static_cast<int32_t>(r.status);
    o->residual = r.residual;
    o->normalized = r.normalized;
    o->dof_updates = r.dof_updates;
    o->dof_updates_total = r.dof_updates_total;
    o->coarse_updates = r.coarse_updates;
    o->pending_tasks = r.pending_tasks;
    o->max_n = r.max_n;
    o->max_samples = r.max_samples;
    o->avg_n = r.avg_n;
    o->factor_totals = r.factor_totals;
    o->factor_mean = r.factor_mean;
    o->enabled_mask = r.enabled_mask;
    o->levels = r.levels;
    o->cells = r.cells;
    o->dofs_fine_interior = r.dofs_fine_interior;
    o->grid_points_total = r.grid_points_total;
    o->wall_seconds = r.wall_seconds;
}

std::string write_temp(const char* text) {
    char path[] = "/tmp/lzb_ref_cfg_XXXXXX";
    int fd = mkstemp(path);
    if (fd < 0) throw std::runtime_error("mkstemp failed");
    ::close(fd);
    std::ofstream out(path);
    out << text;
    return path;
}

ExperimentConfig config_from_text(const char* text) {
    std::string p = write_temp(text);
    ExperimentConfig cfg;
    try {
        cfg = parse_config_file(p);
    } catch (...) {
        std::remove(p.c_str());
        throw;
    }
    std::remove(p.c_str());
    return cfg;
}

double* vertex_member(Vertex& v, int field) {
    switch (field) {
        case LZB_V_U: return &v.u;
        case LZB_V_FL: return &v.fl;
        case LZB_V_R: return &v.r;
        case LZB_V_RHAT: return &v.rhat;
        case LZB_V_UHAT: return &v.uhat;
        case LZB_V_DIAG: return &v.diag;
        case LZB_V_AUX: return &v.aux;
        default: return &v.usnap;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

double ref_eval_field(const lzb_field* f, double x, double y) { return FieldFn(*f)(x, y); }

int ref_integrate_element(const lzb_field* f, double x0, double y0, double h, int n,
                          double* out16) {
    return guarded([&] {
        FieldFn eps(*f);
        ElementMatrix em = integrate_element(CellBox{x0, y0, h}, eps, n);
        std::memcpy(out16, em.m.a.data(), 16 * sizeof(double));
    });
}

// Cells given by level coordinates; box exactly as cell_box() (element.hpp:29-32)
// with h = Mesh::level_h (mesh.hpp:87). nthreads > 1 splits the cells into
// disjoint ranges (the all-cores baseline harness of SURVEY.md §8d item 2).
int ref_integrate_cells(const lzb_field* f, int level, int64_t ncells, const int32_t* cx,
                        const int32_t* cy, const int32_t* n, double* out, int nthreads) {
    return guarded([&] {
        FieldFn eps(*f);
        const double h = std::pow(1.0 / Mesh::kRefine, level);
        auto work = [&](int64_t lo, int64_t hi) {
            for (int64_t i = lo; i < hi; ++i) {
                CellBox box{cx[i] * h, cy[i] * h, h};
                ElementMatrix em = integrate_element(box, eps, n[i]);
                std::memcpy(out + 16 * i, em.m.a.data(), 16 * sizeof(double));
            }
        };
        if (nthreads <= 1) {
            work(0, ncells);
            return;
        }
        std::vector<std::thread> th;
        int64_t chunk = (ncells + nthreads - 1) / nthreads;
        for (int t = 0; t < nthreads; ++t) {
            int64_t lo = t * chunk, hi = std::min<int64_t>(ncells, lo + chunk);
            if (lo < hi) th.emplace_back(work, lo, hi);
        }
        for (auto& x : th) x.join();
    });
}

void ref_unit_stiffness(double* out16) {
    std::memcpy(out16, unit_stiffness().a.data(), 16 * sizeof(double));
}

void ref_subcell_stiffness(double a, double b, double c, double d, double* out16) {
    Mat4 k = reference_subcell_stiffness(a, b, c, d);
    std::memcpy(out16, k.a.data(), 16 * sizeof(double));
}

// ---------------------------------------------------------------- codec
int ref_encode_value(double x, int p3, uint8_t* out) {
    return guarded([&] { codec::encode_value(x, p3, out); });
}
double ref_decode_value(const uint8_t* in, int p3) { return codec::decode_value(in, p3); }
int ref_encode_many(int64_t count, const double* x, int p3, uint8_t* out) {
    return guarded([&] {
        for (int64_t i = 0; i < count; ++i) codec::encode_value(x[i], p3, out + i * p3);
    });
}
void ref_decode_many(int64_t count, const uint8_t* in, int p3, double* out) {
    for (int64_t i = 0; i < count; ++i) out[i] = codec::decode_value(in + i * p3, p3);
}
int ref_choose_precision(const double* v, int64_t count, double delta, int* out_p3) {
    return guarded([&] {
        *out_p3 = codec::choose_precision(std::span<const double>(v, count), delta);
    });
}
int ref_choose_many(int64_t nrec, int entries, const double* v, double delta, int32_t* out,
                    int nthreads) {
    return guarded([&] {
        auto work = [&](int64_t lo, int64_t hi) {
            for (int64_t r = lo; r < hi; ++r)
                out[r] = codec::choose_precision(
                    std::span<const double>(v + r * entries, entries), delta);
        };
        if (nthreads <= 1) return work(0, nrec);
        std::vector<std::thread> th;
        int64_t chunk = (nrec + nthreads - 1) / nthreads;
        for (int t = 0; t < nthreads; ++t) {
            int64_t lo = t * chunk, hi = std::min<int64_t>(nrec, lo + chunk);
            if (lo < hi) th.emplace_back(work, lo, hi);
        }
        for (auto& x : th) x.join();
    });
}
uint8_t ref_pack_header(int32_t p1, int p2, int p3) { return pack_header(p1, p2 != 0, p3); }
int ref_unpack_header(uint8_t h, int* cls, int* p2, int* p3) {
    return guarded([&] {
        bool b = false;
        unpack_header(h, *cls, b, *p3);
        *p2 = b ? 1 : 0;
    });
}

// ---------------------------------------------------------------- transfer
void ref_geometric_prolongation(double* out64) {
    std::memcpy(out64, geometric_prolongation().w.data(), 64 * sizeof(double));
}
void ref_galerkin(const double* children144, const double* P64, double* out16) {
    PatchMatrices ch;
    for (int i = 0; i < 9; ++i) std::memcpy(ch[i].a.data(), children144 + 16 * i, 128);
    TransferBlock P;
    std::memcpy(P.w.data(), P64, 64 * sizeof(double));
    Mat4 m = galerkin_coarse_element(ch, P);
    std::memcpy(out16, m.a.data(), 128);
}
int ref_boxmg(const double* children144, double* out64) {
    PatchMatrices ch;
    for (int i = 0; i < 9; ++i) std::memcpy(ch[i].a.data(), children144 + 16 * i, 128);
    BoxmgResult r = boxmg_prolongation(ch);
    std::memcpy(out64, r.block.w.data(), 64 * sizeof(double));
    return r.fallback_rows;
}

// ---------------------------------------------------------------- rig
void* ref_rig_create(const char* cfg_text, int do_noise) {
    Rig* rig = nullptr;
    int rc = guarded([&] {
        ExperimentConfig cfg = config_from_text(cfg_text);
        rig = new Rig(cfg);
        if (do_noise) init_noise(rig->mesh, rig->problem);
    });
    return rc == LZB_OK ? rig : nullptr;
}
void ref_rig_destroy(void* p) {
    Rig* rig = static_cast<Rig*>(p);
    if (!rig) return;
    rig->pool.shutdown();
    delete rig;
}
int ref_rig_eager_setup(void* p) {
    return guarded([&] { static_cast<Rig*>(p)->assembler.eager_setup(); });
}
int ref_rig_step(void* p, lzb_cycle_report* out) {
    return guarded([&] {
        Rig* rig = static_cast<Rig*>(p);
        CycleReport r = rig->solver.step();
        if (!rig->cfg.timing) r.wall_seconds = 0.0;
        fill_report(r, out);
    });
}
int ref_rig_run(void* p, lzb_cycle_report* out, int cap, int* count) {
    return guarded([&] {
        Rig* rig = static_cast<Rig*>(p);
        auto reps = rig->solver.run_cycles(rig->cfg.amr_config());
        int k = 0;
        for (auto& r : reps) {
            if (!rig->cfg.timing) r.wall_seconds = 0.0;
            if (k < cap) fill_report(r, out + k);
            ++k;
        }
        *count = k;
    });
}
int ref_rig_pass(void* p, int which, double* value) {
    return guarded([&] {
        Rig* rig = static_cast<Rig*>(p);
        CycleReport dummy;
        switch (which) {
            case 0: rig->solver.assembly_pass(); break;
            case 1: *value = rig->solver.residual_pass(); break;
            case 2: rig->solver.update_pass(dummy); break;
            case 3: rig->solver.prolong_corrections(); break;
            case 4: rig->solver.finish_cycle_sync(); break;
            case 5: rig->stream.begin_cycle(static_cast<uint32_t>(rig->solver.cycle())); break;
            case 6: rig->pool.begin_cycle(); break;
            default: throw std::invalid_argument("unknown pass");
        }
    });
}
// Dense per-level vertex view: out[iy*(N+1)+ix], N = 3^level.
int ref_rig_vertices(void* p, int level, int field, double* out, int write) {
    return guarded([&] {
        Rig* rig = static_cast<Rig*>(p);
        int N = rig->mesh.level_cells_per_axis(level);
        for (int32_t vid : rig->mesh.level_vertices(level)) {
            Vertex& v = rig->mesh.vertex(vid);
            double* m = vertex_member(v, field);
            std::size_t k = static_cast<std::size_t>(v.iy) * (N + 1) + v.ix;
            if (write) *m = out[k];
            else out[k] = *m;
        }
    });
}
// Dense per-level cell view: index cy*N+cx.
int ref_rig_cells(void* p, int level, double* ops, int32_t* p1, int32_t* n, int32_t* p3,
                  uint32_t* epoch, int32_t* slot) {
    return guarded([&] {
        Rig* rig = static_cast<Rig*>(p);
        int N = rig->mesh.level_cells_per_axis(level);
        for (int32_t cid : rig->mesh.level_cells(level)) {
            const Cell& c = rig->mesh.cell(cid);
            std::size_t k = static_cast<std::size_t>(c.cy) * N + c.cx;
            const CellMarker& mk = rig->stream.marker(cid);
            OperatorSnapshot s = rig->stream.read_element(cid);
            Mat4 m = rig->stream.element_or_baseline(cid);
            if (ops) std::memcpy(ops + 16 * k, m.a.data(), 128);
            if (p1) p1[k] = mk.p1.load();
            if (n) n[k] = s.n;
            if (p3) p3[k] = mk.p3.load();
            if (epoch) epoch[k] = s.epoch;
            if (slot) slot[k] = c.slot;
        }
    });
}
int ref_rig_transfer(void* p, int level, int cx, int cy, double* out64) {
    return guarded([&] {
        Rig* rig = static_cast<Rig*>(p);
        int32_t cid = rig->mesh.find_cell(level, cx, cy);
        TransferBlock P = rig->stream.transfer_or_geometric(cid);
        std::memcpy(out64, P.w.data(), 512);
    });
}
int ref_rig_publish_element(void* p, int level, int cx, int cy, const double* m16, int n,
                            int32_t p1) {
    return guarded([&] {
        Rig* rig = static_cast<Rig*>(p);
        int32_t cid = rig->mesh.find_cell(level, cx, cy);
        Mat4 m;
        std::memcpy(m.a.data(), m16, 128);
        rig->stream.publish_element(cid, m, n);
        rig->stream.marker(cid).p1.store(p1);
    });
}
int ref_rig_adaptive_step(void* p, int level, int cx, int cy) {
    return guarded([&] {
        Rig* rig = static_cast<Rig*>(p);
        rig->assembler.adaptive_step(rig->mesh.find_cell(level, cx, cy));
    });
}
int ref_rig_stats(void* p, lzb_compression_stats* o) {
    return guarded([&] {
        CompressionStats s = static_cast<Rig*>(p)->stream.compression_stats();
        std::memset(o, 0, sizeof *o);
        o->fine_cells = s.fine_cells;
        o->fine_stored_bytes = s.fine_stored_bytes;
        o->fine_uncompressed_bytes = s.fine_uncompressed_bytes;
        o->fine_factor_totals = s.fine_factor_totals;
        o->fine_factor_mean = s.fine_factor_mean;
        o->max_n = s.max_n;
        o->max_sample_count = s.max_sample_count;
        o->avg_n = s.avg_n;
        o->max_delta = s.max_delta;
        for (int i = 0; i < 9; ++i) o->p3_histogram[i] = s.p3_histogram[i];
        o->total_stored_bytes = s.total_stored_bytes;
        o->total_uncompressed_bytes = s.total_uncompressed_bytes;
        o->total_factor = s.total_factor;
    });
}
int ref_rig_save(void* p, const char* path) {
    return guarded([&] { static_cast<Rig*>(p)->stream.save(path); });
}
int ref_rig_load(void* p, const char* path) {
    return guarded([&] { static_cast<Rig*>(p)->stream.load(path); });
}
int ref_rig_cycle(void* p) { return static_cast<Rig*>(p)->solver.cycle(); }

// ---------------------------------------------------------------- experiment
int ref_run_experiment_file(const char* cfg_path, int* exit_code, int* ncycles) {
    return guarded([&] {
        ExperimentConfig cfg = parse_config_file(cfg_path);
        ExperimentResult r = run_experiment(cfg);
        *exit_code = r.exit_code();
        *ncycles = static_cast<int>(r.reports.size());
    });
}
int ref_run_experiment_text(const char* cfg_text, int* exit_code, int* ncycles) {
    return guarded([&] {
        ExperimentConfig cfg = config_from_text(cfg_text);
        ExperimentResult r = run_experiment(cfg);
        *exit_code = r.exit_code();
        *ncycles = static_cast<int>(r.reports.size());
    });
}
int ref_config_keys(const char* cfg_text, char* out, int64_t cap) {
    return guarded([&] {
        ExperimentConfig cfg = config_from_text(cfg_text);
        std::string s;
        for (const auto& [k, v] : cfg.to_keys()) s += k + " = " + v + "\n";
        std::snprintf(out, static_cast<size_t>(cap), "%s", s.c_str());
    });
}
int ref_emit_table(const char* paths_nl, char* out, int64_t cap) {
    return guarded([&] {
        std::vector<std::string> paths;
        std::istringstream in(paths_nl);
        std::string line;
        while (std::getline(in, line))
            if (!line.empty()) paths.push_back(line);
        std::string t = emit_table(paths);
        std::snprintf(out, static_cast<size_t>(cap), "%s", t.c_str());
    });
}
int ref_compare_runs(const char* a, const char* b, char* out, int64_t cap) {
    return guarded([&] {
        std::string t = compare_runs(a, b);
        std::snprintf(out, static_cast<size_t>(cap), "%s", t.c_str());
    });
}

// ---------------------------------------------------------------- timing harnesses
// Times integrate_element over a bounded sample of cells of one level on
// `nthreads` host threads (disjoint ranges). Returns sub-samples / second.
double ref_time_integrate(const lzb_field* f, int level, int n, int64_t ncells, int nthreads,
                          double* seconds_out) {
    const int N = 1 << 30;
    (void)N;
    int per_axis = 1;
    for (int i = 0; i < level; ++i) per_axis *= 3;
    std::vector<int32_t> cx(ncells), cy(ncells), nn(ncells, n);
    for (int64_t i = 0; i < ncells; ++i) {
        int64_t k = i % (static_cast<int64_t>(per_axis) * per_axis);
        cx[i] = static_cast<int32_t>(k % per_axis);
        cy[i] = static_cast<int32_t>(k / per_axis);
    }
    std::vector<double> out(16 * ncells);
    auto t0 = std::chrono::steady_clock::now();
    ref_integrate_cells(f, level, ncells, cx.data(), cy.data(), nn.data(), out.data(), nthreads);
    double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (seconds_out) *seconds_out = s;
    volatile double sink = out[0];
    (void)sink;
    return static_cast<double>(ncells) * n * n / s;
}

}  // extern "C"

// experiment.cpp — the reference's config / telemetry interface
// (experiment.hpp:14-105) as host C++ over the lzb C-ABI.
//
// Config files use the reference's keys and parsing rules (experiment.cpp:
// 107-211). Extension keys (BASELINE fields, rhs kind, p schedule, sampling
// cap, integration arithmetic) are emitted by to_keys only when they differ
// from their defaults, so reference-compatible configs round-trip and write
// byte-identical telemetry preambles.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "lzb.h"

namespace lzb {
void set_last_error(const std::string& msg);  // runtime.cu: the lzb_last_error() slot
namespace {

thread_local std::vector<lzb_cycle_report> t_reports;

struct Fail : std::runtime_error {
    int code;
    Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

std::string num(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

struct ExperimentConfig {
    std::string setup = "constant";
    double eps_constant = 1.0, theta = 1.0, eps_low = 1e-3, rhs = 0.0;
    uint64_t seed = 0;
    int depth = 2;
    std::string solver = "adafac-pi";
    double omega = 0.7, target = 1e-10, divergence = 1e2;
    int max_cycles = 500;
    std::string assembly = "adaptive";
    double termination_c = 0.01;
    std::string transfer = "geometric", coarse_recompute = "always";
    bool gating = true;
    double compression_threshold = 1e-8;
    int workers = 1;
    uint64_t throttle = 0;
    bool amr = false;
    double amr_fraction = 0.1;
    int amr_interval = 2, amr_max_depth = 7, amr_max_events = -1;
    double forced_task_fraction = 0.0;
    int forced_task_n = 8;
    std::string csv;
    bool timing = true;
    // extensions (BASELINE.json configs)
    int dim = 2;
    uint64_t field_seed = 1;
    int blocks = 8;
    double amp = 0.9, freq = 6.0;
    std::string rhs_kind = "constant";
    double rhs_scale = 2.0 * 3.14159265358979323846 * 3.14159265358979323846;
    std::string schedule = "increment";
    int n_max = 0;
    std::string integration = "exact";
    std::string start = "sample";  // "geometric": BASELINE configs[1]'s eps = 1 start
    int device = 0;

    std::map<std::string, std::string> to_keys() const {
        std::map<std::string, std::string> k;
        k["setup"] = setup;
        k["eps"] = num(eps_constant);
        k["theta"] = num(theta);
        k["eps-low"] = num(eps_low);
        k["rhs"] = num(rhs);
        k["seed"] = std::to_string(seed);
        k["depth"] = std::to_string(depth);
        k["solver"] = solver;
        k["omega"] = num(omega);
        k["target"] = num(target);
        k["divergence"] = num(divergence);
        k["max-cycles"] = std::to_string(max_cycles);
        k["assembly"] = assembly;
        k["termination-c"] = num(termination_c);
        k["transfer"] = transfer;
        k["coarse-recompute"] = coarse_recompute;
        k["gating"] = gating ? "on" : "off";
        k["compression-threshold"] = num(compression_threshold);
        k["workers"] = std::to_string(workers);
        k["throttle"] = std::to_string(throttle);
        k["amr"] = amr ? "on" : "off";
        k["amr-fraction"] = num(amr_fraction);
        k["amr-interval"] = std::to_string(amr_interval);
        k["amr-max-depth"] = std::to_string(amr_max_depth);
        k["amr-max-events"] = std::to_string(amr_max_events);
        k["forced-task-fraction"] = num(forced_task_fraction);
        k["forced-task-n"] = std::to_string(forced_task_n);
        k["timing"] = timing ? "on" : "off";
        k["rng"] = "splitmix64";
        ExperimentConfig d;  // extension keys only when not default
        if (dim != d.dim) k["dim"] = std::to_string(dim);
        if (field_seed != d.field_seed) k["field-seed"] = std::to_string(field_seed);
        if (blocks != d.blocks) k["blocks"] = std::to_string(blocks);
        if (amp != d.amp) k["amp"] = num(amp);
        if (freq != d.freq) k["freq"] = num(freq);
        if (rhs_kind != d.rhs_kind) k["rhs-kind"] = rhs_kind;
        if (rhs_scale != d.rhs_scale) k["rhs-scale"] = num(rhs_scale);
        if (schedule != d.schedule) k["schedule"] = schedule;
        if (n_max != d.n_max) k["n-max"] = std::to_string(n_max);
        if (integration != d.integration) k["integration"] = integration;
        if (start != d.start) k["start"] = start;
        return k;
    }

    void set(const std::string& key, const std::string& value) {
        auto on = [&] {
            if (value == "on" || value == "true" || value == "1") return true;
            if (value == "off" || value == "false" || value == "0") return false;
            throw Fail(LZB_ERR_IO, "expected on/off for key " + key);
        };
        try {
            if (key == "setup") setup = value;
            else if (key == "eps") eps_constant = std::stod(value);
            else if (key == "theta") theta = std::stod(value);
            else if (key == "eps-low") eps_low = std::stod(value);
            else if (key == "rhs") rhs = std::stod(value);
            else if (key == "seed") seed = std::stoull(value);
            else if (key == "depth") depth = std::stoi(value);
            else if (key == "solver") solver = value;
            else if (key == "omega") omega = std::stod(value);
            else if (key == "target") target = std::stod(value);
            else if (key == "divergence") divergence = std::stod(value);
            else if (key == "max-cycles") max_cycles = std::stoi(value);
            else if (key == "assembly") assembly = value;
            else if (key == "termination-c") termination_c = std::stod(value);
            else if (key == "transfer") transfer = value;
            else if (key == "coarse-recompute") coarse_recompute = value;
            else if (key == "gating") gating = on();
            else if (key == "compression-threshold") compression_threshold = std::stod(value);
            else if (key == "workers") workers = std::stoi(value);
            else if (key == "throttle") throttle = std::stoull(value);
            else if (key == "amr") amr = on();
            else if (key == "amr-fraction") amr_fraction = std::stod(value);
            else if (key == "amr-interval") amr_interval = std::stoi(value);
            else if (key == "amr-max-depth") amr_max_depth = std::stoi(value);
            else if (key == "amr-max-events") amr_max_events = std::stoi(value);
            else if (key == "forced-task-fraction") forced_task_fraction = std::stod(value);
            else if (key == "forced-task-n") forced_task_n = std::stoi(value);
            else if (key == "timing") timing = on();
            else if (key == "csv") csv = value;
            else if (key == "rng") { /* informational */ }
            else if (key == "dim") dim = std::stoi(value);
            else if (key == "field-seed") field_seed = std::stoull(value);
            else if (key == "blocks") blocks = std::stoi(value);
            else if (key == "amp") amp = std::stod(value);
            else if (key == "freq") freq = std::stod(value);
            else if (key == "rhs-kind") rhs_kind = value;
            else if (key == "rhs-scale") rhs_scale = std::stod(value);
            else if (key == "schedule") schedule = value;
            else if (key == "n-max") n_max = std::stoi(value);
            else if (key == "integration") integration = value;
            else if (key == "start") start = value;
            else if (key == "device") device = std::stoi(value);
            else throw Fail(LZB_ERR_IO, "unknown config key: " + key);
        } catch (const std::invalid_argument&) {
            throw Fail(LZB_ERR_IO, "malformed value for key " + key + ": " + value);
        } catch (const std::out_of_range&) {
            throw Fail(LZB_ERR_IO, "value out of range for key " + key + ": " + value);
        }
    }

    lzb_grid_desc desc() const {
        lzb_grid_desc d;
        std::memset(&d, 0, sizeof d);
        d.dim = dim;
        d.depth = depth;
        if (setup == "theta") {
            d.field.kind = LZB_FIELD_THETA;
            d.field.value = 1.0;
            d.field.theta = theta;
        } else if (setup == "quadrant") {
            d.field.kind = LZB_FIELD_QUADRANT;
            d.field.value = 1.0;
            d.field.eps_low = eps_low;
        } else if (setup == "constant") {
            d.field.kind = LZB_FIELD_CONSTANT;
            d.field.value = eps_constant;
        } else if (setup == "checkerboard") {
            lzb_field_checkerboard(&d.field, field_seed, blocks);
        } else if (setup == "sinusoid") {
            d.field.kind = LZB_FIELD_SINUSOID;
            d.field.value = 1.0;
            d.field.amp = amp;
            d.field.freq = freq;
        } else {
            throw Fail(LZB_ERR_IO, "unknown setup: " + setup);
        }
        if (rhs_kind == "sinprod") {
            d.rhs.kind = LZB_RHS_SINPROD;
            d.rhs.value = rhs_scale;
        } else if (rhs_kind == "constant") {
            d.rhs.kind = LZB_RHS_CONSTANT;
            d.rhs.value = rhs;
        } else {
            throw Fail(LZB_ERR_IO, "unknown rhs-kind: " + rhs_kind);
        }
        d.delta_max = compression_threshold;
        if (solver == "additive") d.variant = LZB_ADDITIVE;
        else if (solver == "adafac-jac") d.variant = LZB_ADAFAC_JAC;
        else if (solver == "adafac-pi") d.variant = LZB_ADAFAC_PI;
        else throw Fail(LZB_ERR_IO, "unknown solver: " + solver);
        d.omega = omega;
        d.target = target;
        d.divergence = divergence;
        d.max_cycles = max_cycles;
        if (assembly == "eager") d.mode = LZB_EAGER;
        else if (assembly == "lazy") d.mode = LZB_LAZY;
        else if (assembly == "adaptive") d.mode = LZB_ADAPTIVE;
        else if (assembly == "anarchic") d.mode = LZB_ANARCHIC;
        else throw Fail(LZB_ERR_IO, "unknown assembly mode: " + assembly);
        d.termination_c = termination_c;
        if (transfer == "geometric") d.transfer = LZB_GEOMETRIC;
        else if (transfer == "boxmg") d.transfer = LZB_BOXMG;
        else throw Fail(LZB_ERR_IO, "unknown transfer: " + transfer);
        if (coarse_recompute == "always") d.policy = LZB_ALWAYS;
        else if (coarse_recompute == "ripple") d.policy = LZB_RIPPLE;
        else throw Fail(LZB_ERR_IO, "unknown coarse-recompute: " + coarse_recompute);
        d.gating = gating ? 1 : 0;
        if (schedule == "increment") d.schedule = LZB_SCHEDULE_INCREMENT;
        else if (schedule == "double") d.schedule = LZB_SCHEDULE_DOUBLE;
        else throw Fail(LZB_ERR_IO, "unknown schedule: " + schedule);
        d.n_max = n_max;
        if (integration == "exact") d.integration = LZB_INTEGRATE_EXACT;
        else if (integration == "fast") d.integration = LZB_INTEGRATE_FAST;
        else throw Fail(LZB_ERR_IO, "unknown integration: " + integration);
        // workers > 1: background integration (scheduler.cpp:5-12) = the concurrent
        // assembly stream; only anarchic mode ever spawns tasks
        d.concurrent = (workers > 1 && assembly == "anarchic") ? 1 : 0;
        d.throttle = throttle;
        d.noise_seed = seed;
        d.boundary_value = 0.0;
        if (start == "geometric") d.start_geometric = 1;
        else if (start != "sample") throw Fail(LZB_ERR_IO, "unknown start: " + start);
        // run_experiment's forced-task hook (experiment.cpp:260-270) on the device
        d.forced_fraction = forced_task_fraction;
        d.forced_n = forced_task_n;
        return d;
    }
};

std::string strip(const std::string& s, const char* ws) {
    auto a = s.find_first_not_of(ws);
    auto b = s.find_last_not_of(ws);
    return a == std::string::npos ? std::string() : s.substr(a, b - a + 1);
}

ExperimentConfig parse_stream(std::istream& in, const std::string& name) {
    ExperimentConfig cfg;
    std::string line;
    int lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        auto hash = line.find('#');
        if (hash != std::string::npos) line.erase(hash);
        if (strip(line, " \t\r").empty()) continue;
        auto eq = line.find('=');
        if (eq == std::string::npos)
            throw Fail(LZB_ERR_IO, name + ":" + std::to_string(lineno) + ": expected key = value");
        cfg.set(strip(line.substr(0, eq), " \t\r"), strip(line.substr(eq + 1), " \t\r"));
    }
    return cfg;
}

const char* status_name(int s) {
    switch (s) {
        case LZB_CONTINUE: return "continue";
        case LZB_CONVERGED: return "converged";
        case LZB_DIVERGED: return "diverged";
        case LZB_TIMEOUT: return "timeout";
    }
    return "unknown";
}

std::string telemetry_csv(const ExperimentConfig& cfg, const std::vector<lzb_cycle_report>& reps) {
    std::ostringstream out;
    out << "# lazymg telemetry v1\n";
    for (const auto& [k, v] : cfg.to_keys()) out << "# " << k << " = " << v << "\n";
    out << "cycle,residual,normalized,dof_updates,dof_updates_total,coarse_updates,"
           "pending_tasks,max_n,avg_n,max_samples,factor_totals,factor_mean,enabled_mask,"
           "levels,cells,dofs_fine_interior,grid_points_total,wall_seconds,status\n";
    char buf[512];
    for (const auto& r : reps) {
        std::snprintf(buf, sizeof buf,
                      "%d,%.17g,%.17g,%llu,%llu,%llu,%llu,%d,%.6f,%d,%.6f,%.6f,%u,%d,%llu,%llu,"
                      "%llu,%.6f,%s\n",
                      r.cycle, r.residual, r.normalized,
                      static_cast<unsigned long long>(r.dof_updates),
                      static_cast<unsigned long long>(r.dof_updates_total),
                      static_cast<unsigned long long>(r.coarse_updates),
                      static_cast<unsigned long long>(r.pending_tasks), r.max_n, r.avg_n,
                      r.max_samples, r.factor_totals, r.factor_mean, r.enabled_mask, r.levels,
                      static_cast<unsigned long long>(r.cells),
                      static_cast<unsigned long long>(r.dofs_fine_interior),
                      static_cast<unsigned long long>(r.grid_points_total), r.wall_seconds,
                      status_name(r.status));
        out << buf;
    }
    return out.str();
}

struct Ctx {
    lzb_ctx* c = nullptr;
    ~Ctx() { lzb_ctx_destroy(c); }
};
struct GridH {
    lzb_grid* g = nullptr;
    ~GridH() { lzb_grid_destroy(g); }
};

void check(int rc) {
    if (rc != LZB_OK) throw Fail(rc, lzb_last_error());
}

int run(const ExperimentConfig& cfg) {
    if (cfg.amr)
        throw Fail(LZB_ERR_INVALID, "amr = on: adaptive refinement is not on the device path (SURVEY §8f)");
    lzb_grid_desc d = cfg.desc();
    Ctx ctx;
    check(lzb_ctx_create(cfg.device, &ctx.c));
    GridH grid;
    check(lzb_grid_create(ctx.c, &d, &grid.g));
    check(lzb_grid_init_noise(grid.g, cfg.seed));
    std::vector<lzb_cycle_report> reps(static_cast<size_t>(std::max(cfg.max_cycles, 1)) + 1);
    int count = 0;
    check(lzb_grid_run(grid.g, reps.data(), static_cast<int>(reps.size()), &count));
    reps.resize(std::min<size_t>(reps.size(), static_cast<size_t>(count)));
    if (!cfg.timing)
        for (auto& r : reps) r.wall_seconds = 0.0;
    t_reports = reps;
    if (!cfg.csv.empty()) {
        std::ofstream out(cfg.csv);
        if (!out) throw Fail(LZB_ERR_IO, "cannot write telemetry: " + cfg.csv);
        out << telemetry_csv(cfg, reps);
    }
    int st = reps.empty() ? LZB_TIMEOUT : reps.back().status;
    switch (st) {  // ExperimentResult::exit_code, experiment.cpp:213-220
        case LZB_CONVERGED: return 0;
        case LZB_DIVERGED: return 2;
        case LZB_TIMEOUT: return 3;
        default: return 1;
    }
}

struct Telemetry {
    std::map<std::string, std::string> keys;
    std::vector<lzb_cycle_report> rows;
};

Telemetry read_telemetry(const std::string& path) {  // experiment.cpp:290-347
    std::ifstream in(path);
    if (!in) throw Fail(LZB_ERR_IO, "cannot open telemetry file: " + path);
    Telemetry tf;
    std::string line;
    bool header = false;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        if (line[0] == '#') {
            auto eq = line.find('=');
            if (eq != std::string::npos)
                tf.keys[strip(line.substr(0, eq), " \t#")] = strip(line.substr(eq + 1), " \t\r");
            continue;
        }
        if (!header) {
            header = true;
            continue;
        }
        std::vector<std::string> f;
        std::istringstream ss(line);
        std::string x;
        while (std::getline(ss, x, ',')) f.push_back(x);
        if (f.size() < 19) throw Fail(LZB_ERR_IO, "short telemetry row");
        lzb_cycle_report r;
        std::memset(&r, 0, sizeof r);
        r.cycle = std::stoi(f[0]);
        r.residual = std::stod(f[1]);
        r.normalized = std::stod(f[2]);
        r.dof_updates = std::stoull(f[3]);
        r.dof_updates_total = std::stoull(f[4]);
        r.coarse_updates = std::stoull(f[5]);
        r.pending_tasks = std::stoull(f[6]);
        r.max_n = std::stoi(f[7]);
        r.avg_n = std::stod(f[8]);
        r.max_samples = std::stoi(f[9]);
        r.factor_totals = std::stod(f[10]);
        r.factor_mean = std::stod(f[11]);
        r.enabled_mask = static_cast<uint32_t>(std::stoul(f[12]));
        r.levels = std::stoi(f[13]);
        r.cells = std::stoull(f[14]);
        r.dofs_fine_interior = std::stoull(f[15]);
        r.grid_points_total = std::stoull(f[16]);
        r.wall_seconds = std::stod(f[17]);
        const std::string& st = f[18];
        r.status = st == "converged" ? LZB_CONVERGED
                   : st == "diverged" ? LZB_DIVERGED
                   : st == "timeout"  ? LZB_TIMEOUT
                                      : LZB_CONTINUE;
        tf.rows.push_back(r);
    }
    return tf;
}

std::string emit_table(const std::vector<std::string>& paths) {  // experiment.cpp:349-383
    std::vector<Telemetry> files;
    size_t max_rows = 0;
    for (const auto& p : paths) {
        files.push_back(read_telemetry(p));
        max_rows = std::max(max_rows, files.back().rows.size());
    }
    std::ostringstream out;
    out << "Cycle";
    for (const auto& tf : files) {
        std::string label = tf.keys.count("setup") ? tf.keys.at("setup") : "run";
        if (label == "theta" && tf.keys.count("theta")) label = "theta = " + tf.keys.at("theta");
        else if (label == "quadrant" && tf.keys.count("eps-low"))
            label = "eps-low = " + tf.keys.at("eps-low");
        out << " | " << label << ": max{n}  avg n  compression";
    }
    out << "\n";
    char buf[128];
    for (size_t i = 0; i < max_rows; ++i) {
        out << (i + 1 < 10 ? "    " : "   ") << (i + 1);
        for (const auto& tf : files) {
            if (i < tf.rows.size()) {
                const auto& r = tf.rows[i];
                std::snprintf(buf, sizeof buf, " |        %6d  %5.2f  %11.2f", r.max_n, r.avg_n,
                              r.factor_totals);
                out << buf;
            } else {
                out << " |             -      -            -";
            }
        }
        out << "\n";
    }
    return out.str();
}

// Shortest round-trip rendering of a double (the JSON number style of the
// reference's compare_runs output).
std::string jnum(double v) {
    if (std::isnan(v) || std::isinf(v)) return "null";
    char buf[64];
    for (int p = 1; p <= 17; ++p) {
        std::snprintf(buf, sizeof buf, "%.*g", p, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    std::string s = buf;
    if (s.find_first_of(".en") == std::string::npos) s += ".0";
    return s;
}

std::string compare_runs(const std::string& a_path, const std::string& b_path) {  // experiment.cpp:385-424
    Telemetry a = read_telemetry(a_path), b = read_telemetry(b_path);
    for (const char* key : {"setup", "theta", "eps-low", "eps", "depth", "rhs"}) {
        std::string va = a.keys.count(key) ? a.keys.at(key) : "";
        std::string vb = b.keys.count(key) ? b.keys.at(key) : "";
        if (va != vb)
            throw Fail(LZB_ERR_IO, std::string("runs solve different problems (") + key + ": " + va +
                                       " vs " + vb + ")");
    }
    auto summarise = [](const Telemetry& tf, const std::string& path) {
        double target = tf.keys.count("target") ? std::stod(tf.keys.at("target")) : 1e-10;
        int cycles_to_target = -1;
        double time_to_target = -1.0, t = 0.0;
        for (const auto& r : tf.rows) {
            t += r.wall_seconds;
            if (cycles_to_target < 0 && r.normalized <= target) {
                cycles_to_target = r.cycle;
                time_to_target = t;
            }
        }
        std::map<std::string, std::string> j;  // keys sorted like a JSON object dump
        j["file"] = "\"" + path + "\"";
        j["target"] = jnum(target);
        j["cycles"] = std::to_string(tf.rows.size());
        j["cycles_to_target"] = std::to_string(cycles_to_target);
        j["time_to_target_seconds"] = jnum(time_to_target);
        j["total_time_seconds"] = jnum(t);
        if (!tf.rows.empty()) {
            j["final_normalized_residual"] = jnum(tf.rows.back().normalized);
            j["final_status"] = std::string("\"") + status_name(tf.rows.back().status) + "\"";
            j["dof_updates_total"] = std::to_string(tf.rows.back().dof_updates_total);
        }
        std::string s = "{\n";
        size_t i = 0;
        for (const auto& [k, v] : j)
            s += "    \"" + k + "\": " + v + (++i < j.size() ? ",\n" : "\n");
        return s + "  }";
    };
    return "{\n  \"a\": " + summarise(a, a_path) + ",\n  \"b\": " + summarise(b, b_path) + "\n}\n";
}

template <typename F>
int guard(F&& f) {
    try {
        f();
        return LZB_OK;
    } catch (const Fail& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return LZB_ERR_IO;
    }
}

void copy_out(const std::string& s, char* out, int64_t cap) {
    if (cap <= 0) return;
    std::snprintf(out, static_cast<size_t>(cap), "%s", s.c_str());
    if (static_cast<int64_t>(s.size()) >= cap) throw Fail(LZB_ERR_INVALID, "output buffer too small");
}

}  // namespace
}  // namespace lzb

using namespace lzb;

extern "C" {

int lzb_run_experiment_file(const char* cfg_path, int* exit_code, int* ncycles) {
    return guard([&] {
        std::ifstream in(cfg_path);
        if (!in) throw Fail(LZB_ERR_IO, std::string("cannot open config file: ") + cfg_path);
        ExperimentConfig cfg = parse_stream(in, cfg_path);
        *exit_code = run(cfg);
        *ncycles = static_cast<int>(t_reports.size());
    });
}

int lzb_run_experiment_text(const char* cfg_text, int* exit_code, int* ncycles) {
    return guard([&] {
        std::istringstream in(cfg_text);
        ExperimentConfig cfg = parse_stream(in, "<text>");
        *exit_code = run(cfg);
        *ncycles = static_cast<int>(t_reports.size());
    });
}

int lzb_last_reports(lzb_cycle_report* out, int cap, int* count) {
    for (size_t i = 0; i < t_reports.size() && static_cast<int>(i) < cap; ++i) out[i] = t_reports[i];
    *count = static_cast<int>(t_reports.size());
    return LZB_OK;
}

int lzb_config_keys(const char* cfg_text, char* out, int64_t cap) {
    return guard([&] {
        std::istringstream in(cfg_text);
        ExperimentConfig cfg = parse_stream(in, "<text>");
        std::string s;
        for (const auto& [k, v] : cfg.to_keys()) s += k + " = " + v + "\n";
        copy_out(s, out, cap);
    });
}

int lzb_emit_table(const char* paths_nl, char* out, int64_t cap) {
    return guard([&] {
        std::vector<std::string> paths;
        std::istringstream in(paths_nl);
        std::string line;
        while (std::getline(in, line))
            if (!line.empty()) paths.push_back(line);
        copy_out(emit_table(paths), out, cap);
    });
}

int lzb_compare_runs(const char* a, const char* b, char* out, int64_t cap) {
    return guard([&] { copy_out(compare_runs(a, b), out, cap); });
}

}  // extern "C"

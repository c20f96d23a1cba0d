/*
 * lzb_types.h — plain-C data formats shared by the B200 C-ABI (include/lzb.h),
 * the CPU oracle (oracle/) and the reference harness (oracle/ref_driver.cpp).
 *
 * Nothing here depends on CUDA or torch. Every struct is POD with fixed-width
 * members so that ctypes / cgo / JNI bindings can mirror it verbatim.
 *
 * Conventions follow the reference (`/root/reference/proj/include/lazymg/types.hpp`):
 *   corner c of a cell: SW,SE,NW,NE with offset (c & 1, c >> 1)      types.hpp:11-15
 *   element matrix: 16 doubles, row-major, rows/cols indexed by corner  types.hpp:23-50
 *   transfer block: 64 doubles, w[L*4 + c], lattice L = ly*4 + lx      types.hpp:17-20,62-66
 */
#ifndef LZB_TYPES_H
#define LZB_TYPES_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
/* One code per reference exception type (types.hpp:68-76 + std exceptions). */
enum lzb_status {
    LZB_OK = 0,
    LZB_ERR_PROTOCOL = 1, /* lazymg::protocol_error      (codec.cpp:10, assembly.cpp:127) */
    LZB_ERR_CORRUPT = 2,  /* lazymg::corrupt_stream_error (stream.cpp:53,346-379)          */
    LZB_ERR_RESOURCE = 3, /* lazymg::resource_error      (mesh.cpp:68,259)                */
    LZB_ERR_INVALID = 4,  /* std::invalid_argument       (mesh.cpp:254)                   */
    LZB_ERR_IO = 5,       /* std::runtime_error for config / file IO (experiment.cpp)     */
    LZB_ERR_CUDA = 6,     /* device fault / launch failure                                */
    LZB_ERR_NCCL = 7      /* collective failure                                           */
};

/* ------------------------------------------------------------ material eps */
/* Kinds 0-2 are the reference MaterialField (problem.hpp:12-26, problem.cpp:9-31).
 * Kinds 3-4 are the BASELINE.json fields; they have one
 * definition shared by the oracle and the device code. */
enum lzb_field_kind {
    LZB_FIELD_CONSTANT = 0, /* eps = value                                               */
    LZB_FIELD_THETA = 1,    /* 1 + 0.15 prod_i exp(-theta x_i) cos(pi theta x_i)         */
    LZB_FIELD_QUADRANT = 2, /* 1 on the diagonal pair, eps_low off-diagonal (centre 0.5+1/4374) */
    LZB_FIELD_CHECKER = 3,  /* T[min(B-1,floor(Bx))][min(B-1,floor(By))], B = blocks      */
    LZB_FIELD_SINUSOID = 4  /* 1 + amp sin(freq pi x) sin(freq pi y)                      */
};

#define LZB_CHECKER_MAX_BLOCKS 8

typedef struct lzb_field {
    int32_t kind;
    int32_t blocks;   /* checkerboard blocks per axis (<= 8)                  */
    double value;     /* constant                                             */
    double theta;     /* theta field                                          */
    double eps_low;   /* quadrant                                             */
    double amp;       /* sinusoid amplitude (0.9 for BASELINE config 2)       */
    double freq;      /* sinusoid frequency factor (6 for BASELINE config 2)  */
    double table[LZB_CHECKER_MAX_BLOCKS * LZB_CHECKER_MAX_BLOCKS]; /* T[bx*blocks+by] */
} lzb_field;

/* --------------------------------------------------------------- 3D fields
 * BASELINE configs[2..4] are 3D; the reference has no 3D code (types.hpp:13),
 * so these are restated extensions (SURVEY.md §8c "3D: parity unpinned by the
 * reference"). GRF: eps = exp(g), g trilinearly interpolated from a periodic
 * n^3 table (lzb_grf_table), index (i*n + j)*n + k for (x, y, z). EXTRUDED:
 * eps(x, y, z) = the 2D field at (x, y) (tensor-product checks). */
enum lzb_field3_kind { LZB_F3_CONSTANT = 0, LZB_F3_GRF = 1, LZB_F3_EXTRUDED = 2, LZB_F3_SPHERE = 3 };

/* SPHERE (BASELINE configs[3]): eps = eps_out + (eps_in - eps_out) s(t),
 * t = (radius - |x - centre|) / width, s(t) = (1 + tanh(2 atanh(0.8) t)) / 2,
 * so eps passes from 10 % to 90 % of the jump across the interface width. */
typedef struct lzb_field3 {
    int32_t kind;
    int32_t grf_n;        /* GRF table points per axis (64 for BASELINE)        */
    double value;         /* constant                                           */
    const double* grf;    /* host pointer to grf_n^3 values of g (copied)       */
    lzb_field xy;         /* EXTRUDED                                           */
    double centre[3];     /* SPHERE                                             */
    double radius, width, eps_in, eps_out;
} lzb_field3;

/* ------------------------------------------------------------ right-hand side */
/* The reference only has f = rhs_constant (problem.hpp:38,42) and applies the
 * lumped load only when it is non-zero (solver.cpp:106). SINPROD is the
 * BASELINE f = scale * sin(pi x) sin(pi y) (scale = 2 pi^2). */
enum lzb_rhs_kind { LZB_RHS_CONSTANT = 0, LZB_RHS_SINPROD = 1 };

typedef struct lzb_rhs {
    int32_t kind;
    int32_t pad_;
    double value; /* constant value, or the scale of SINPROD */
} lzb_rhs;

/* ------------------------------------------------------------ solver / grid */
enum lzb_variant { LZB_ADDITIVE = 0, LZB_ADAFAC_JAC = 1, LZB_ADAFAC_PI = 2 };     /* solver.hpp:14 */
enum lzb_assembly_mode { LZB_EAGER = 0, LZB_LAZY = 1, LZB_ADAPTIVE = 2, LZB_ANARCHIC = 3 }; /* assembly.hpp:10 */
enum lzb_transfer { LZB_GEOMETRIC = 0, LZB_BOXMG = 1 };                           /* solver.hpp:15 */
enum lzb_policy { LZB_ALWAYS = 0, LZB_RIPPLE = 1 };                               /* solver.hpp:16 */
enum lzb_run_status { LZB_CONTINUE = 0, LZB_CONVERGED = 1, LZB_DIVERGED = 2, LZB_TIMEOUT = 3 };
enum lzb_schedule { LZB_SCHEDULE_INCREMENT = 0, LZB_SCHEDULE_DOUBLE = 1 };
/* integration arithmetic: EXACT reproduces element.hpp:42-47 bit for bit
 * (same loop order, no FMA contraction); FAST is the separable FMA form
 * (within 1e-12 relative). */
enum lzb_integration { LZB_INTEGRATE_EXACT = 0, LZB_INTEGRATE_FAST = 1 };

typedef struct lzb_grid_desc {
    int32_t dim;              /* 2 (3D is a later round)                           */
    int32_t depth;            /* regular spacetree depth: 3^depth cells per axis   */
    lzb_field field;
    lzb_rhs rhs;
    double delta_max;         /* codec threshold (stream.hpp:74, default 1e-8)     */
    /* solver (SolverConfig solver.hpp:18-24) */
    int32_t variant;
    int32_t max_cycles;
    double omega;
    double target;
    double divergence;
    /* assembly (AssemblyConfig assembly.hpp:12-15) */
    int32_t mode;
    int32_t schedule;         /* n -> n+1 (reference) or n -> 2n                    */
    double termination_c;
    int32_t n_max;            /* 0 = unlimited; else cells reaching n_max become top */
    int32_t integration;      /* lzb_integration                                   */
    /* multilevel (MultilevelConfig solver.hpp:27-31) */
    int32_t transfer;
    int32_t policy;
    int32_t gating;
    /* scheduler (SchedulerConfig scheduler.hpp:26-29): workers == 1 semantics */
    int32_t concurrent;       /* 0: deterministic (tasks at next cycle start); 1: side stream */
    uint64_t throttle;        /* tasks per cycle, 0 = unlimited                     */
    uint64_t noise_seed;
    double boundary_value;
    /* extensions (no reference counterpart) */
    int32_t plane_width;      /* 0: the residual reads the decoded FP64 operators; 2..8: it
                                 decodes the leaf records' compressed surplus bytes (a slot of
                                 plane_width bytes per entry; wider records fall back to FP64) */
    int32_t fixed_p3;         /* 0: choose_precision per leaf record; 2..8: every leaf record
                                 at this width (the mantissa-width sweep, BASELINE configs[4]) */
    int32_t start_geometric;  /* 1: a leaf not yet integrated (p1 = bottom) reads the geometric
                                 stencil (eps = 1) instead of its n = 1 sample, and in anarchic
                                 mode its first integration is deferred to a task too -- the
                                 "delayed assembly starting from the geometric stencil" of
                                 BASELINE configs[1]; 0: the reference start (assembly.cpp:26-33,
                                 stream.cpp:82-84). The codec baseline stays A(n = 1). */
    int32_t forced_n;         /* spawn_forced sub-sample count (forced-task-n, experiment.hpp:56) */
    double forced_fraction;   /* forced-task-fraction (experiment.hpp:55, experiment.cpp:260-270):
                                 at every cycle start the leaves whose roll
                                 splitmix64(0x6f4ce1a3 ^ cell id) falls below it get a forced
                                 integrate task (Assembler::spawn_forced, assembly.cpp:138-154) */
} lzb_grid_desc;

/* CycleReport, solver.hpp:41-61 (field for field). */
typedef struct lzb_cycle_report {
    int32_t cycle;
    int32_t status; /* lzb_run_status */
    double residual;
    double normalized;
    uint64_t dof_updates;
    uint64_t dof_updates_total;
    uint64_t coarse_updates;
    uint64_t pending_tasks;
    int32_t max_n;
    int32_t max_samples;
    double avg_n;
    double factor_totals;
    double factor_mean;
    uint32_t enabled_mask;
    int32_t levels;
    uint64_t cells;
    uint64_t dofs_fine_interior;
    uint64_t grid_points_total;
    double wall_seconds;
} lzb_cycle_report;

/* CompressionStats, stream.hpp:49-66. */
typedef struct lzb_compression_stats {
    uint64_t fine_cells;
    uint64_t fine_stored_bytes;
    uint64_t fine_uncompressed_bytes;
    double fine_factor_totals;
    double fine_factor_mean;
    int32_t max_n;
    int32_t max_sample_count;
    double avg_n;
    double max_delta;
    uint64_t p3_histogram[9];
    uint64_t total_stored_bytes;
    uint64_t total_uncompressed_bytes;
    double total_factor;
} lzb_compression_stats;

/* Marker p1 encoding (stream.hpp:18-24). */
#define LZB_P1_BOTTOM 0
#define LZB_P1_TOP (-1)

/* Vertex field selectors for lzb_grid_get_level / set_level (mesh.hpp:27-36). */
enum lzb_vertex_field {
    LZB_V_U = 0, LZB_V_FL = 1, LZB_V_R = 2, LZB_V_RHAT = 3, LZB_V_UHAT = 4,
    LZB_V_DIAG = 5, LZB_V_AUX = 6, LZB_V_USNAP = 7, LZB_V_NFIELDS = 8
};

/* kernels timed by lzb_grid_time_kernel (leaf level) */
enum {
    LZB_TK_UHAT = 0, LZB_TK_RESIDUAL = 1, LZB_TK_RESTRICT = 2, LZB_TK_JACOBI = 3,
    LZB_TK_PROLONG = 4, LZB_TK_PACK = 5, LZB_TK_FRONT = 6, LZB_TK_BACK = 7
};

#ifdef __cplusplus
}
#endif
#endif /* LZB_TYPES_H */

/*
 * lzb.h — C-ABI of the B200-native delayed-assembly hot path (liblzb.so).
 *
 * Plain pointers and sizes only. Host-buffer entry points copy in/out inside
 * the call; *_dev entry points take device pointers and a cudaStream_t passed
 * as void* and are asynchronous on that stream.
 *
 * Each entry point names the reference interface it replaces
 * (the headers under /root/reference/proj/include/lazymg). The reference exposes C++
 * only; these are the symbols its call sites bind through the host shim
 * (INTEGRATION.md). Errors: every function returns an lzb_status; the
 * message is in lzb_last_error() (thread-local). A missing GPU is
 * LZB_ERR_CUDA — there is no CPU fallback.
 */
#ifndef LZB_H
#define LZB_H

#include <stddef.h>
#include <stdint.h>

#include "lzb_types.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ----------------------------------------------------------------- runtime */
const char* lzb_last_error(void);
int lzb_version(void);
/* Number of kernels this library has launched since load (evidence counter). */
uint64_t lzb_launch_count(void);
/* Measured FP64 FMA throughput of this device (TFLOP/s): the roofline
 * denominator for the FP64-bound integration kernel. */
int lzb_probe_fp64_tflops(int device, double* tflops);

typedef struct lzb_ctx lzb_ctx;
/* Device + two streams: solve (high priority) and assembly (low priority). */
int lzb_ctx_create(int device, lzb_ctx** out);
void lzb_ctx_destroy(lzb_ctx* ctx);
int lzb_ctx_synchronize(lzb_ctx* ctx);
/* Raw stream handles (cudaStream_t) for callers that mix their own work in. */
void* lzb_ctx_solve_stream(lzb_ctx* ctx);
void* lzb_ctx_assembly_stream(lzb_ctx* ctx);

/* ------------------------------------------------------------------ fields */
/* BASELINE config 1 checkerboard; host-side helper. */
void lzb_field_checkerboard(lzb_field* f, uint64_t seed, int blocks);
double lzb_field_eval_host(const lzb_field* f, double x, double y);

/* ----------------------------------------------------------------- element */
/* integrate_element(CellBox{x0,y0,h}, eps, n)          element.hpp:36-49
 * batched over cells; out = ncells x 16 doubles (row-major Mat4).
 * integration: LZB_INTEGRATE_EXACT (bit-identical) or LZB_INTEGRATE_FAST. */
int lzb_integrate_elements(lzb_ctx* ctx, const lzb_field* eps, int64_t ncells,
                           const double* x0, const double* y0, const double* h,
                           const int32_t* n, double* out, int integration);
int lzb_integrate_elements_dev(lzb_ctx* ctx, const lzb_field* eps, int64_t ncells,
                               const double* x0, const double* y0, const double* h,
                               const int32_t* n, double* out, int integration, void* stream);
/* All cells of one regular level at one n: out[(cy*N+cx)*16 + k], N = 3^level,
 * boxes as cell_box() (element.hpp:29-32) with h = pow(1/3, level) (mesh.hpp:87). */
int lzb_integrate_level_dev(lzb_ctx* ctx, const lzb_field* eps, int level, int n,
                            double* out, int integration, void* stream);
/* Same, host output buffer (the end-to-end entry: the field descriptor goes in,
 * N*N*16 doubles come back). */
int lzb_integrate_level(lzb_ctx* ctx, const lzb_field* eps, int level, int n, double* host_out,
                        int integration);
/* reference_subcell_stiffness(a,b,c,d)                   element.hpp:19 */
int lzb_subcell_stiffness(lzb_ctx* ctx, double a, double b, double c, double d, double* out16);

/* ------------------------------------------------------------------- codec */
/* codec::encode_value, batched: count values at one p3 -> count*p3 bytes. codec.hpp:23-26
 * Non-finite input -> LZB_ERR_PROTOCOL (codec.cpp:10). */
int lzb_codec_encode(lzb_ctx* ctx, int64_t count, const double* x, int p3, uint8_t* out);
/* codec::decode_value, batched.                                              codec.hpp:28 */
int lzb_codec_decode(lzb_ctx* ctx, int64_t count, const uint8_t* in, int p3, double* out);
/* codec::choose_precision over nrec records of `entries` values.          codec.hpp:35-37 */
int lzb_codec_choose_precision(lzb_ctx* ctx, int64_t nrec, int32_t entries, const double* values,
                               double delta_max, int32_t* out_p3);
int lzb_codec_choose_precision_dev(lzb_ctx* ctx, int64_t nrec, int32_t entries,
                                   const double* values, double delta_max, int32_t* out_p3,
                                   void* stream);
/* pack_header / unpack_header                                         stream.hpp:30-33 */
uint8_t lzb_pack_header(int32_t p1, int p2, int p3);
int lzb_unpack_header(uint8_t h, int* p1_class, int* p2, int* p3);

/* ---------------------------------------------------------------- transfer */
/* galerkin_coarse_element(children, P): npatch x (9x16 children, child lx*3+ly)
 * P = npatch x 64 or NULL for geometric_prolongation().       transfer.hpp:31-32 */
int lzb_galerkin(lzb_ctx* ctx, int64_t npatch, const double* children, const double* P,
                 double* out);
/* boxmg_prolongation(children) -> npatch x 64, fallback rows.   transfer.hpp:28 */
int lzb_boxmg(lzb_ctx* ctx, int64_t npatch, const double* children, double* P,
              int32_t* fallback_rows);
void lzb_geometric_prolongation(double* out64);

/* -------------------------------------------------------------------- grid */
/* One regular 2D spacetree with its operator stream, assembler and additive
 * multigrid solver resident in HBM: Mesh + CellStream + Assembler +
 * AdditiveSolver (mesh.hpp:64, stream.hpp:72, assembly.hpp:38, solver.hpp:72). */
typedef struct lzb_grid lzb_grid;
int lzb_grid_create(lzb_ctx* ctx, const lzb_grid_desc* desc, lzb_grid** out);
void lzb_grid_destroy(lzb_grid* g);
/* init_noise(mesh, problem)                                        problem.hpp:50 */
int lzb_grid_init_noise(lzb_grid* g, uint64_t seed);
/* Assembler::eager_setup                                          assembly.hpp:47 */
int lzb_grid_eager_setup(lzb_grid* g);
/* Fixed-p assembly (BASELINE config 1): every leaf integrated at n, published, p1 = top. */
int lzb_grid_assemble_fixed(lzb_grid* g, int n);
/* lzb_grid_assemble_fixed through the same fused integrate + compress +
 * publish kernel, also returning each leaf's integrated element matrix before
 * compression (host_raw: N*N*16 doubles, cy*N+cx): integrate_element
 * (element.hpp:36-49) of every leaf, for parity checks of the benched kernel. */
int lzb_grid_assemble_fixed_raw(lzb_grid* g, int n, double* host_raw);
/* CellStream::publish_element + p1 store for every leaf (stream.cpp:100-132,
 * batched): mats N*N*16 doubles, n per cell (host buffers). */
int lzb_grid_publish_level(lzb_grid* g, int level, const double* mats, const int32_t* n, int32_t p1);
/* Same for the leaf cell rows [row0, row1) only: one slab of a multi-GPU
 * decomposition (cells are independent). */
int lzb_grid_assemble_rows(lzb_grid* g, int n, int row0, int row1);
/* Device pointers of one level's cell arrays (op: 16 doubles per cell, p1 i32,
 * n i32, p3 i8, epoch u32, chg u32; index cy*N+cx), for in-place collectives. */
int lzb_grid_cell_arrays(lzb_grid* g, int level, void** op, void** p1, void** n, void** p3,
                         void** epoch, void** chg);
/* The cell state was written through lzb_grid_cell_arrays: re-derive the
 * engine's host-side bookkeeping before the next cycle. */
int lzb_grid_invalidate(lzb_grid* g);
/* AdditiveSolver::step / run_cycles                             solver.hpp:78-79 */
int lzb_grid_step(lzb_grid* g, lzb_cycle_report* out);
int lzb_grid_run(lzb_grid* g, lzb_cycle_report* out, int cap, int* count);
/* One multiplicative V(nu, nu) cycle with damped Jacobi (omega of the desc)
 * on the same levels, operators and transfers (BASELINE configs[1] names
 * V(1,1); restated extension, the reference's cycle is additive only). */
int lzb_grid_vcycle(lzb_grid* g, int nu, lzb_cycle_report* out);
/* Individual passes (solver.hpp:91-98): 0 assembly, 1 residual (value = norm),
 * 2 update, 3 prolong, 4 finish_cycle_sync, 5 stream begin_cycle, 6 pool begin_cycle,
 * 7 drain every pending assembly task (TaskPool::drain_all, scheduler.hpp:59). */
int lzb_grid_pass(lzb_grid* g, int which, double* value);
int lzb_grid_cycle(lzb_grid* g);
/* Dense per-level vertex field: (N+1)^2 doubles, index iy*(N+1)+ix. */
int lzb_grid_vertices(lzb_grid* g, int level, int field, double* buf, int write);
/* Dense per-level cells, index cy*N+cx: element_or_baseline (16 doubles), markers. */
int lzb_grid_cells(lzb_grid* g, int level, double* ops, int32_t* p1, int32_t* n, int32_t* p3,
                   uint32_t* epoch);
/* assemble_vertex_stencil (assembly.hpp:69-71, assembly.cpp:120-136) for every
 * vertex of a level: out (N+1)^2 x 9 doubles, vertex iy*(N+1)+ix, entry
 * (dy+1)*3+(dx+1) (Stencil9, types.hpp:53-58); missing cells contribute zero;
 * require_payload != 0 and a bottom neighbour -> LZB_ERR_PROTOCOL. */
int lzb_grid_vertex_stencils(lzb_grid* g, int level, int require_payload, double* out);
/* scatter_row (element.hpp:53, element.cpp:39-45): stencil9 += row `corner`
 * of element16 placed relative to that corner. Host only. */
int lzb_scatter_row(const double* element16, int corner, double* stencil9);
/* Transfer block of a refined cell (transfer_or_geometric, stream.hpp:106). */
int lzb_grid_transfer(lzb_grid* g, int level, int cx, int cy, double* out64);
/* CellStream::publish_element + marker store (stream.hpp:88, assembly protocol). */
int lzb_grid_publish_element(lzb_grid* g, int level, int cx, int cy, const double* m16,
                             int n, int32_t p1);
/* Assembler::adaptive_step(cell)                                   assembly.hpp:40 */
int lzb_grid_adaptive_step(lzb_grid* g, int level, int cx, int cy);
/* CellStream::compression_stats                                    stream.hpp:118 */
int lzb_grid_stats(lzb_grid* g, lzb_compression_stats* out);
/* CellStream::save/load byte image ("LZMG" v1, stream.cpp:303-394).
 * lzb_grid_stream_image with out == NULL returns the size in *size. */
int lzb_grid_stream_image(lzb_grid* g, uint8_t* out, int64_t cap, int64_t* size);
/* lzb_grid_assemble_fixed(g, n) then lzb_grid_stream_image(g, out, cap, size),
 * pipelined: three bands of level-1 subtrees (contiguous byte ranges in
 * pre-order) are packed and copied to `out` while the next band assembles.
 * Same bytes; LZB_ERR_INVALID if the image exceeds cap (nothing past cap is
 * written). timeline: NULL or 9 floats (device ms of each band's assembly,
 * pack and copy end). Replaces Assembler::eager_setup at fixed n +
 * CellStream::save (assembly.cpp:111-118, stream.cpp:303-338). */
int lzb_grid_assemble_stream(lzb_grid* g, int n, uint8_t* out, int64_t cap, int64_t* size, float* timeline);
int lzb_grid_stream_load(lzb_grid* g, const uint8_t* in, int64_t size);
int lzb_grid_save(lzb_grid* g, const char* path);
int lzb_grid_load(lzb_grid* g, const char* path);
/* Pending background tasks (TaskPool::pending_count, scheduler.hpp:45). */
int64_t lzb_grid_pending(lzb_grid* g);
/* Device pointers for callers composing their own kernels (read-only use). */
int lzb_grid_device_view(lzb_grid* g, int level, int field, void** ptr);
/* Slab-distributed cycle (no reference counterpart: the
 * reference is shared-memory only). One rank per GPU holds the whole grid;
 * the leaf level's vertex rows [v0, v1) (multiples of 3, v1 may be N+1) are
 * this rank's slab, the coarse levels run replicated. A cycle is
 * lzb_grid_dist_phase 0..5 with the host exchanges in between
 * (paper_2005_03606_b200/parallel.py: r̂ halo after 0, all-gather of level
 * D-1 fl after 1, all-reduce of lzb_grid_dist_result after 2 then
 * lzb_grid_dist_report, all-gather of aux / u of level D-1 after 3 / 4, u
 * halo after 5). flags bit 0 on phase 0: count the coarse levels' stats
 * (one rank). Every vertex value is bit-identical to the one-GPU cycle. */
int lzb_grid_set_slab(lzb_grid* g, int v0, int v1);
/* The leaf level's compressed records read by the residual (desc.plane_width
 * > 0; NULL otherwise): 16 slots of `width` bytes per cell, and the width
 * each cell's slots hold (> width: the FP64 operator is read). */
int lzb_grid_plane_arrays(lzb_grid* g, void** planes, void** cp3, int* width);
int lzb_grid_dist_phase(lzb_grid* g, int phase, int flags);
int lzb_grid_dist_result(lzb_grid* g, double* norm2, uint64_t* slots20);
int lzb_grid_dist_report(lzb_grid* g, double norm2, const uint64_t* slots20, lzb_cycle_report* rep);
/* ---- the slab-distributed data plane in C++ (csrc/dist.cpp)
 * The context owns an NCCL communicator (NCCL loaded at run time); one
 * distributed cycle is the phases above with NCCL send/recv halos, in-place
 * broadcasts of the replicated level D-1 rows and an on-device all-reduce of
 * the norm and counters, all on the solve stream, one host read per cycle.
 * The _loopback forms run the same plan over several slabs of one process
 * (device copies instead of NCCL): the one-GPU check of the plan. */
int lzb_nccl_unique_id(uint8_t* out128);
int lzb_ctx_comm_init(lzb_ctx* ctx, const uint8_t* id128, int nranks, int rank);
int lzb_ctx_comm_info(lzb_ctx* ctx, int* rank, int* nranks);
int lzb_grid_dist_cycle(lzb_grid* g, lzb_cycle_report* out);
int lzb_grid_dist_cycle_loopback(lzb_grid* const* slabs, int nslabs, lzb_cycle_report* out);
/* slab assembly (each rank its leaf cell rows) + exchange of the leaf state */
int lzb_grid_dist_assemble(lzb_grid* g, int n);
int lzb_grid_dist_assemble_loopback(lzb_grid* const* slabs, int nslabs, int n);
/* introspection for the data plane: context, depth, descriptor, the device
 * address of the phase-2 result (double norm^2, then 20 u64 counter slots) */
int lzb_grid_info(lzb_grid* g, lzb_ctx** ctx, int* depth);
int lzb_grid_desc_of(lzb_grid* g, lzb_grid_desc* out);
int lzb_grid_dist_result_dev(lzb_grid* g, void** result);
/* Device time (CUDA events on the solve stream) of one hot kernel of the
 * leaf level, averaged over `reps` back-to-back launches: LZB_TK_* ids.
 * No reference counterpart: the measurement hook behind bench.py's roofline. */
int lzb_grid_time_kernel(lzb_grid* g, int what, int reps, double* avg_ms);

/* -------------------------------------------------------------------- 3D
 * Restated 3D extension (BASELINE configs[2..4]; no reference counterpart):
 * trilinear hexahedra, corner a = ax + 2 ay + 4 az, 8x8 element matrices,
 * eps sampled at the n^3 sub-cell centres, K = sum eps * K_sub with K_sub
 * the exact sub-box stiffness (per-axis seg_int, element.cpp:8-32, in 3D).
 * Records: 64 entries, the same codec and surplus-over-A(n=1) coding. */
/* Gaussian random field g on a periodic n^3 grid (n a power of 2): Gaussian
 * covariance sigma2 * exp(-r^2 / (2 ell^2)), spectral synthesis from seeded
 * (splitmix64, Box-Muller) normals, inverse FFT; out: n^3 doubles. */
int lzb_grf_table(uint64_t seed, int n, double ell, double sigma2, double* out);
/* Batched 3D element integration (host buffers): count cells, out count*64. */
int lzb_integrate_elements3(lzb_ctx* ctx, const lzb_field3* f, int64_t count, const double* x0,
                            const double* y0, const double* z0, const double* h, const int32_t* n,
                            double* out);
typedef struct lzb_grid3 lzb_grid3;
/* A regular 3D grid of depth `depth` (3^depth cells per axis), leaves only:
 * fixed-p assembly + compression (fixed_p3 = 0: choose_precision per record). */
int lzb_grid3_create(lzb_ctx* ctx, int depth, const lzb_field3* f, double delta_max, int fixed_p3,
                     lzb_grid3** out);
/* The same with the leaf operators held only as compressed class planes of
 * plane_width W bytes per class value (2..8; 0 = FP64 class planes): the
 * residual and the Galerkin product decode them (BASELINE configs[4] width
 * sweep). A record whose p3 exceeds W fails the assembly with
 * LZB_ERR_RESOURCE. Restated 3D form of stream.cpp:82-111 + solver.cpp:145-175. */
int lzb_grid3_create_planes(lzb_ctx* ctx, int depth, const lzb_field3* f, double delta_max, int fixed_p3,
                            int plane_width, lzb_grid3** out);
/* The same storing only the leaf operators of cell layers [cz0, cz1) (-1, -1:
 * all): a z-slab window. Such a grid runs the plane-range assembly calls and
 * the distributed cycle (lzb_grid3_dist_*); the one-GPU cycle, which reads
 * every leaf, is rejected (LZB_ERR_INVALID). lzb_grid3_create_slab picks the
 * window of slab `slab` of `nslabs` of the z-slab plan (csrc/dist.cpp): the
 * leaf operators, 3/4 of a 729^3 grid's memory, then scale as 1/nslabs
 * (the reference is shared-memory only). */
int lzb_grid3_create_window(lzb_ctx* ctx, int depth, const lzb_field3* f, double delta_max, int fixed_p3,
                            int plane_width, int cz0, int cz1, lzb_grid3** out);
int lzb_grid3_create_slab(lzb_ctx* ctx, int depth, const lzb_field3* f, double delta_max, int fixed_p3,
                          int plane_width, int nslabs, int slab, lzb_grid3** out);
/* resident bytes of the leaf operator storage and the stored layer window */
int lzb_grid3_leaf_storage(lzb_grid3* g, int64_t* bytes, int* cz0, int* cz1);
int lzb_grid3_destroy(lzb_grid3* g);
int lzb_grid3_assemble_fixed(lzb_grid3* g, int n);
int lzb_grid3_stats(lzb_grid3* g, lzb_compression_stats* out);
/* Cells [first, first+count) (index (cz*N + cy)*N + cx): stored operators
 * (count*64) and widths. */
int lzb_grid3_cells(lzb_grid3* g, int64_t first, int64_t count, double* ops, int32_t* p3);
/* The additive multilevel cycle on the 3D grid (solver.cpp:99-347 restated):
 * levels 0..depth, Galerkin coarse operators from the assembled leaves,
 * trilinear geometric transfer, variant additive or adafac-pi, load
 * f = rhs_scale * prod sin(pi x_d) lumped with h^3/8, u0 = seeded noise. */
int lzb_grid3_init_cycle(lzb_grid3* g, int variant, double omega, double rhs_scale, uint64_t noise_seed,
                         int max_cycles, double target);
int lzb_grid3_step(lzb_grid3* g, lzb_cycle_report* out);
/* One multiplicative V(nu, nu) cycle with damped Jacobi (omega of
 * init_cycle) on the same levels, Galerkin operators and transfers
 * (BASELINE configs[1..2] V-cycles; restated, the reference is additive only). */
int lzb_grid3_vcycle(lzb_grid3* g, int nu, lzb_cycle_report* out);
int lzb_grid3_vertices(lzb_grid3* g, int level, int field, double* out);  /* (N+1)^3 doubles */
/* Slab-distributed 3D cycle: z-slabs of leaf vertex planes, coarse levels
 * replicated; phases 0..5 and exchanges as lzb_grid_dist_phase (driven by
 * paper_2005_03606_b200/parallel.py dist_cycle3). */
int lzb_grid3_set_slab(lzb_grid3* g, int v0, int v1);
int lzb_grid3_dist_phase(lzb_grid3* g, int phase);
int lzb_grid3_dist_result(lzb_grid3* g, double* norm2);
int lzb_grid3_dist_report(lzb_grid3* g, double norm2, lzb_cycle_report* out);
/* the C++ data plane for the 3D grid (see lzb_grid_dist_cycle); assemble:
 * the z-slab sharded assembly below with the level D-1 class planes exchanged */
int lzb_grid3_dist_cycle(lzb_grid3* g, lzb_cycle_report* out);
int lzb_grid3_dist_cycle_loopback(lzb_grid3* const* slabs, int nslabs, lzb_cycle_report* out);
int lzb_grid3_dist_assemble(lzb_grid3* g, int n);
int lzb_grid3_dist_assemble_loopback(lzb_grid3* const* slabs, int nslabs, int n);
int lzb_grid3_dist_phase_flags(lzb_grid3* g, int phase, int flags);
int lzb_grid3_dist_result_dev(lzb_grid3* g, void** norm2);
int lzb_grid3_info(lzb_grid3* g, lzb_ctx** ctx, int* depth);
int lzb_grid3_variant(lzb_grid3* g);
/* z-slab sharded 3D assembly (parallel.distributed_assemble3): fixed-p
 * assembly of the leaf cells in z planes [cz0, cz1); the Galerkin coarse
 * operators of `level` for its coarse cells in z planes [pz0, pz1); every
 * coarse level below `level` from it; the device class planes of a level
 * (27 planes of N^3 doubles, value q of cell c at q * N^3 + c) for the
 * all-gather. Restated 3D form of assembly.cpp:111-118 / solver.cpp:59-77. */
int lzb_grid3_assemble_planes(lzb_grid3* g, int n, int cz0, int cz1);
int lzb_grid3_galerkin_planes(lzb_grid3* g, int level, int pz0, int pz1);
int lzb_grid3_coarse_below(lzb_grid3* g, int level);
int lzb_grid3_level_ops(lzb_grid3* g, int level, void** ptr);
/* BASELINE configs[3] (C4), assembly: a 3D adaptive spacetree refined to
 * level lmax where a cell meets the ball |x - f->centre| <= f->radius and to
 * lbase elsewhere (leaves on up to three levels, hanging nodes between them;
 * the adaptive mesh of mesh.cpp:66-129,236-312 restated in 3D), fixed-p
 * assembly + 27-class record coding of every leaf, and the delayed
 * re-assembly of the leaves meeting the interface shell | |x - c| - r | <=
 * band. Leaves: (level, cx, cy, cz), level-major. */
typedef struct lzb_tree3 lzb_tree3;
int lzb_tree3_create(lzb_ctx* ctx, int lbase, int lmax, const lzb_field3* f, double delta_max, int fixed_p3,
                     lzb_tree3** out);
int lzb_tree3_destroy(lzb_tree3* t);
int lzb_tree3_counts(lzb_tree3* t, int64_t* per_level /* [8] */, int64_t* total);
int lzb_tree3_assemble(lzb_tree3* t, int n);
int lzb_tree3_set_shell(lzb_tree3* t, double band, int64_t* count);
int lzb_tree3_assemble_shell(lzb_tree3* t, int n);
int lzb_tree3_stats(lzb_tree3* t, lzb_compression_stats* out);
/* leaves [first, first + count): 64 entries (8x8 row-major), p3, n, (level, cx, cy, cz) */
int lzb_tree3_cells(lzb_tree3* t, int64_t first, int64_t count, double* ops, int32_t* p3, int32_t* n,
                    int32_t* lxyz);
/* The additive cycle on the tree (solver.cpp:99-347 on an adaptive mesh,
 * restated in 3D: hanging vertices interpolated from their parents,
 * mesh.cpp:115-138,182-234). init_cycle builds the levels, copies the leaves'
 * operators in and forms the refined cells' Galerkin operators; refresh_ops
 * redoes that after a (shell) re-assembly; vertices reads a dense level
 * ((3^l + 1)^3 values, [z][y][x]). */
int lzb_tree3_init_cycle(lzb_tree3* t, int variant, double omega, double rhs_scale, uint64_t noise_seed,
                         int max_cycles, double target);
int lzb_tree3_refresh_ops(lzb_tree3* t);
/* Re-refinement (BASELINE configs[3]: topology change forcing re-assembly;
 * the reference's apply_refinement_now + on_refinement, solver.cpp:402-418,
 * mesh.cpp:236-312, stream.cpp:262-266, restated for the sphere tree): the
 * refinement ball grows to `radius` (no coarsening, mesh.hpp:55), every leaf
 * meeting it below lmax is refined; surviving leaves keep their operators,
 * new leaves are assembled at n; during a cycle the new vertices start from
 * the parent interpolant and the levels / loads / Galerkin operators are
 * rebuilt. *new_leaves: the leaves created. */
int lzb_tree3_refine(lzb_tree3* t, double radius, int n, int64_t* new_leaves);
int lzb_tree3_step(lzb_tree3* t, lzb_cycle_report* out);
int lzb_tree3_vertices(lzb_tree3* t, int level, int field, double* out);
/* Average device ms of one leaf-level 3D cycle kernel (LZB_TK_UHAT .. LZB_TK_PROLONG). */
int lzb_grid3_time_kernel(lzb_grid3* g, int what, int reps, double* avg_ms);
int lzb_grid3_device_view(lzb_grid3* g, int level, int field, void** ptr);

/* -------------------------------------------------------------- experiment */
/* run_experiment(parse_config_file(path))               experiment.hpp:75,89
 * Writes the telemetry CSV when the config names one; returns the exit code
 * in *exit_code (0 converged, 2 diverged, 3 timeout, experiment.cpp:213-220). */
int lzb_run_experiment_file(const char* cfg_path, int* exit_code, int* ncycles);
int lzb_run_experiment_text(const char* cfg_text, int* exit_code, int* ncycles);
/* Reports of the last run_experiment on this thread. */
int lzb_last_reports(lzb_cycle_report* out, int cap, int* count);
/* ExperimentConfig::to_keys rendered as "key = value\n" lines. experiment.hpp:68 */
int lzb_config_keys(const char* cfg_text, char* out, int64_t cap);
/* emit_table / compare_runs                                   experiment.hpp:99-104 */
int lzb_emit_table(const char* csv_paths_newline_separated, char* out, int64_t cap);
int lzb_compare_runs(const char* csv_a, const char* csv_b, char* out, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* LZB_H */

/*
 * lzb_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference (/root/reference/proj) delayed-assembly
 * path on REGULAR 2D spacetrees, used as the parity checker for the B200
 * product. Every function cites the reference file:line it restates.
 * Pinned against the unmodified reference (oracle/_ref) and the six committed
 * telemetry CSVs (proj/exp_*.csv) by tests/test_oracle_pin.py.
 */
#ifndef LZB_ORACLE_H
#define LZB_ORACLE_H
#include <stdint.h>

#include "lzb_types.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- primitives ---- */
double orc_field_eval(const lzb_field* f, double x, double y);
void orc_field_checkerboard(lzb_field* f, uint64_t seed, int blocks);
uint64_t orc_splitmix64(uint64_t z);
void orc_subcell_stiffness(double a, double b, double c, double d, double* out16);
void orc_integrate_element(const lzb_field* f, double x0, double y0, double h, int n,
                           double* out16);
/* every cell of a regular level, threaded over disjoint cell ranges */
void orc_integrate_level(const lzb_field* f, int level, int n, double* out, int threads);
int orc_encode_value(double x, int p3, uint8_t* out); /* 0 ok, LZB_ERR_PROTOCOL */
double orc_decode_value(const uint8_t* in, int p3);
int orc_choose_precision(const double* v, int64_t count, double delta); /* <0: error */
uint8_t orc_pack_header(int32_t p1, int p2, int p3);
int orc_unpack_header(uint8_t h, int* cls, int* p2, int* p3);
void orc_geometric(double* P64);
void orc_patch_operator(const double* children144, double* A256);
void orc_galerkin(const double* children144, const double* P64, double* out16);
int orc_boxmg(const double* children144, double* P64);

/* ---- regular-grid solver state ---- */
typedef struct orc_grid orc_grid;
orc_grid* orc_grid_create(const lzb_grid_desc* d);
void orc_grid_destroy(orc_grid* g);
const char* orc_last_error(void);
int orc_init_noise(orc_grid* g, uint64_t seed);
int orc_eager_setup(orc_grid* g);
int orc_assemble_fixed(orc_grid* g, int n);
int orc_step(orc_grid* g, lzb_cycle_report* out);
int orc_run(orc_grid* g, lzb_cycle_report* out, int cap, int* count);
int orc_pass(orc_grid* g, int which, double* value);
int orc_vertices(orc_grid* g, int level, int field, double* buf, int write);
int orc_cells(orc_grid* g, int level, double* ops, int32_t* p1, int32_t* n, int32_t* p3,
              uint32_t* epoch);
int orc_publish_element(orc_grid* g, int level, int cx, int cy, const double* m, int n,
                        int32_t p1);
int orc_publish_level(orc_grid* g, int level, const double* mats, const int32_t* n, int32_t p1);
int orc_adaptive_step(orc_grid* g, int level, int cx, int cy);
int orc_stats(orc_grid* g, lzb_compression_stats* out);
int64_t orc_stream_image(orc_grid* g, uint8_t* out, int64_t cap);
int orc_stream_load(orc_grid* g, const uint8_t* in, int64_t size);
int orc_cycle(orc_grid* g);

#ifdef __cplusplus
}
#endif
#endif

/*
 * lzb_oracle.c — TEST INFRASTRUCTURE ONLY: CPU restatement of the reference
 * delayed-assembly path (/root/reference/proj) for REGULAR 2D spacetrees.
 *
 * It is the parity checker of the B200 product and nothing else: only
 * tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
 * reference) may load it. It is pinned against the unmodified reference
 * (oracle/_ref) and the six telemetry CSVs committed in the reference tree
 * (tests/test_oracle_pin.py).
 *
 * Data layout: per level l, N = 3^l cells per axis; cell (cx,cy) at cy*N+cx,
 * vertex (ix,iy) at iy*(N+1)+ix. The reference's hash-mapped AoS mesh
 * (mesh.hpp:17-51) is replaced by these dense arrays, but every loop that
 * accumulates floating point values visits cells/vertices in the reference's
 * order (level_cells creation order, level_vertices creation order) and
 * every expression keeps the reference's operand order, so results are bit
 * identical (compiled with -ffp-contract=off).
 */
#define _POSIX_C_SOURCE 200809L
#define _DEFAULT_SOURCE
#include "lzb_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static _Thread_local char g_err[256];
static int set_err(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
const char* orc_last_error(void) { return g_err; }

static inline int cdx(int c) { return c & 1; } /* types.hpp:14 */
static inline int cdy(int c) { return c >> 1; } /* types.hpp:15 */

/* ================================================================ eps, f */

/* problem.cpp:9-31 (kinds 0-2); kinds 3-4 are the BASELINE restatements. */
double orc_field_eval(const lzb_field* f, double x, double y) {
    switch (f->kind) {
        case LZB_FIELD_THETA: {
            const double amplitude = 0.3 / 2.0;
            double px = exp(-f->theta * x) * cos(M_PI * f->theta * x);
            double py = exp(-f->theta * y) * cos(M_PI * f->theta * y);
            return 1.0 + amplitude * px * py;
        }
        case LZB_FIELD_QUADRANT: {
            const double centre = 0.5 + 1.0 / (2.0 * 2187.0);
            int east = x >= centre, north = y >= centre;
            return east == north ? 1.0 : f->eps_low;
        }
        case LZB_FIELD_CHECKER: {
            int b = f->blocks;
            int bx = (int)(b * x), by = (int)(b * y);
            if (bx > b - 1) bx = b - 1;
            if (by > b - 1) by = b - 1;
            return f->table[bx * b + by];
        }
        case LZB_FIELD_SINUSOID:
            return 1.0 + f->amp * sin(f->freq * M_PI * x) * sin(f->freq * M_PI * y);
        default: return f->value;
    }
}

/* problem.cpp:43-48 */
uint64_t orc_splitmix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

/* BASELINE config 1 field table. */
void orc_field_checkerboard(lzb_field* f, uint64_t seed, int blocks) {
    memset(f, 0, sizeof *f);
    f->kind = LZB_FIELD_CHECKER;
    f->blocks = blocks;
    f->value = 1.0;
    for (int i = 0; i < blocks; ++i)
        for (int j = 0; j < blocks; ++j) {
            double u = (double)(orc_splitmix64(seed ^ (uint64_t)(blocks * i + j)) >> 11) *
                       0x1.0p-53;
            f->table[i * blocks + j] = pow(10.0, -2.0 + 4.0 * u);
        }
}

static double rhs_eval(const lzb_rhs* r, double x, double y) {
    if (r->kind == LZB_RHS_SINPROD) return r->value * sin(M_PI * x) * sin(M_PI * y);
    return r->value;
}
static int rhs_active(const lzb_rhs* r) {
    return r->kind == LZB_RHS_SINPROD || r->value != 0.0; /* solver.cpp:106 */
}

/* ================================================================ element */

/* element.cpp:8-15 */
static double seg_int(int si, int sj, double a, double b) {
    double a0 = si ? 0.0 : 1.0, a1 = si ? 1.0 : -1.0;
    double b0 = sj ? 0.0 : 1.0, b1 = sj ? 1.0 : -1.0;
    double Fb = a0 * b0 * b + (a0 * b1 + a1 * b0) * b * b / 2.0 + a1 * b1 * b * b * b / 3.0;
    double Fa = a0 * b0 * a + (a0 * b1 + a1 * b0) * a * a / 2.0 + a1 * b1 * a * a * a / 3.0;
    return Fb - Fa;
}

/* element.cpp:19-32 */
void orc_subcell_stiffness(double a, double b, double c, double d, double* K) {
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            double dXi = cdx(i) ? 1.0 : -1.0, dXj = cdx(j) ? 1.0 : -1.0;
            double dYi = cdy(i) ? 1.0 : -1.0, dYj = cdy(j) ? 1.0 : -1.0;
            K[i * 4 + j] = dXi * dXj * (b - a) * seg_int(cdy(i), cdy(j), c, d) +
                           dYi * dYj * (d - c) * seg_int(cdx(i), cdx(j), a, b);
        }
}

/* K_sub(i, j) of integrate_element at sub-sample count n (element.hpp:42-45):
 * reference_subcell_stiffness(i*inv, (i+1)*inv, j*inv, (j+1)*inv). It is a
 * pure function of (n, i, j), so it is tabulated once per n and per thread
 * with the very same call -- the bits are those of the per-sample call. */
static const double* ksub_table(int n) {
    static _Thread_local double* tab = NULL;
    static _Thread_local int tab_n = 0;
    if (tab_n != n) {
        free(tab);
        tab = malloc((size_t)n * n * 16 * sizeof(double));
        double inv = 1.0 / n;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                orc_subcell_stiffness(i * inv, (i + 1) * inv, j * inv, (j + 1) * inv, tab + ((size_t)i * n + j) * 16);
        tab_n = n;
    }
    return tab;
}

/* element.hpp:36-49: i (x) outer, j (y) inner, out += eps * K_sub. */
void orc_integrate_element(const lzb_field* f, double x0, double y0, double h, int n,
                           double* out) {
    double inv = 1.0 / n;
    const double* tab = ksub_table(n);
    for (int k = 0; k < 16; ++k) out[k] = 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double e = orc_field_eval(f, x0 + (i + 0.5) * inv * h, y0 + (j + 0.5) * inv * h);
            const double* K = tab + ((size_t)i * n + j) * 16;
            for (int k = 0; k < 16; ++k) out[k] += e * K[k];
        }
}

/* integrate_element over every cell of a regular level (boxes as cell_box,
 * element.hpp:29-32, h = pow(1/3, level) as mesh.hpp:87), cells split into
 * contiguous ranges over `threads` POSIX threads (the reference's pure
 * function on disjoint cells). out: N*N*16, cy*N+cx. */
typedef struct {
    const lzb_field* f;
    int N, n;
    double h;
    int64_t c0, c1;
    double* out;
} level_job;
static void* level_worker(void* arg) {
    level_job* j = (level_job*)arg;
    for (int64_t c = j->c0; c < j->c1; ++c)
        orc_integrate_element(j->f, (c % j->N) * j->h, (c / j->N) * j->h, j->h, j->n, j->out + 16 * c);
    return NULL;
}
void orc_integrate_level(const lzb_field* f, int level, int n, double* out, int threads) {
    int N = 1;
    for (int l = 0; l < level; ++l) N *= 3;
    double h = pow(1.0 / 3, level);
    int64_t nc = (int64_t)N * N;
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    level_job jobs[256];
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (level_job){f, N, n, h, nc * t / threads, nc * (t + 1) / threads, out};
        if (pthread_create(&tid[t], NULL, level_worker, &jobs[t]) != 0) {
            level_worker(&jobs[t]);
            tid[t] = 0;
        }
    }
    for (int t = 0; t < threads; ++t)
        if (tid[t]) pthread_join(tid[t], NULL);
}

/* ================================================================ codec */

static inline int mantissa_bits(int p3) { return 8 * (p3 - 1) - 1; } /* codec.hpp:20 */

/* codec.cpp:8-45 */
int orc_encode_value(double x, int p3, uint8_t* out) {
    if (p3 == 0) return 0;
    if (!isfinite(x)) return set_err(LZB_ERR_PROTOCOL, "cannot encode non-finite operator entry");
    if (p3 == 8) {
        memcpy(out, &x, 8);
        return 0;
    }
    const int m = mantissa_bits(p3);
    uint64_t frac_bits = 0;
    int sign = 0, e_hat = -128;
    if (x != 0.0) {
        sign = signbit(x) ? 1 : 0;
        int e;
        double f = frexp(fabs(x), &e);
        e -= 1;
        double frac = 2.0 * f - 1.0;
        e_hat = e < -128 ? -128 : (e > 127 ? 127 : e);
        frac_bits = (uint64_t)ldexp(frac, m);
    }
    uint64_t packed = ((uint64_t)sign << m) | frac_bits;
    int total_bits = m + 1;
    for (int b = 0; b < p3 - 1; ++b) out[b] = (uint8_t)(packed >> (total_bits - 8 * (b + 1)));
    out[p3 - 1] = (uint8_t)(int8_t)e_hat;
    return 0;
}

/* codec.cpp:47-63 */
double orc_decode_value(const uint8_t* in, int p3) {
    if (p3 == 8) {
        double x;
        memcpy(&x, in, 8);
        return x;
    }
    const int m = mantissa_bits(p3);
    uint64_t packed = 0;
    for (int b = 0; b < p3 - 1; ++b) packed = (packed << 8) | in[b];
    int sign = (int)((packed >> m) & 1u);
    uint64_t frac_bits = packed & ((1ull << m) - 1);
    int e_hat = (int8_t)in[p3 - 1];
    if (sign == 0 && frac_bits == 0 && e_hat == -128) return 0.0;
    double mant = 1.0 + ldexp((double)frac_bits, -m);
    double v = ldexp(mant, e_hat);
    return sign ? -v : v;
}

/* codec.hpp:28-33 */
static int roundtrip(double x, int p3, double* out) {
    if (p3 == 0) {
        *out = 0.0;
        return 0;
    }
    uint8_t buf[8];
    int rc = orc_encode_value(x, p3, buf);
    if (rc) return rc;
    *out = orc_decode_value(buf, p3);
    return 0;
}

/* codec.cpp:65-85 */
int orc_choose_precision(const double* v, int64_t count, double delta) {
    int all_small = 1;
    for (int64_t i = 0; i < count; ++i)
        if (fabs(v[i]) > delta) {
            all_small = 0;
            break;
        }
    if (all_small) return 0;
    for (int p3 = 2; p3 < 8; ++p3) {
        int ok = 1;
        for (int64_t i = 0; i < count; ++i) {
            double rt;
            if (roundtrip(v[i], p3, &rt)) return -LZB_ERR_PROTOCOL;
            if (fabs(rt - v[i]) > delta) {
                ok = 0;
                break;
            }
        }
        if (ok) return p3;
    }
    return 8;
}

/* stream.cpp:44-55 */
uint8_t orc_pack_header(int32_t p1, int p2, int p3) {
    int cls = p1 == LZB_P1_BOTTOM ? 0 : (p1 == LZB_P1_TOP ? 2 : 1);
    return (uint8_t)((cls << 6) | (p2 ? 0x20 : 0) | (p3 & 0x0f));
}
int orc_unpack_header(uint8_t h, int* cls, int* p2, int* p3) {
    *cls = (h >> 6) & 0x3;
    *p2 = (h & 0x20) != 0;
    *p3 = h & 0x0f;
    if (*cls == 3 || *p3 == 1 || *p3 > 8)
        return set_err(LZB_ERR_CORRUPT, "invalid record header byte");
    return 0;
}

/* ================================================================ transfer */

/* transfer.cpp:11-21 */
void orc_geometric(double* P) {
    for (int ly = 0; ly < 4; ++ly)
        for (int lx = 0; lx < 4; ++lx) {
            double fx = lx / 3.0, fy = ly / 3.0;
            int L = ly * 4 + lx;
            for (int c = 0; c < 4; ++c)
                P[L * 4 + c] = (cdx(c) ? fx : 1.0 - fx) * (cdy(c) ? fy : 1.0 - fy);
        }
}

/* transfer.cpp:81-93: child i = lx outer, j = ly inner, child index lx*3+ly */
void orc_patch_operator(const double* ch, double* A) {
    memset(A, 0, 256 * sizeof(double));
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            const double* K = ch + 16 * (i * 3 + j);
            int ids[4];
            for (int c = 0; c < 4; ++c) ids[c] = (j + cdy(c)) * 4 + (i + cdx(c));
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b) A[ids[a] * 16 + ids[b]] += K[a * 4 + b];
        }
}

/* transfer.cpp:182-200 (zero-skip on A entries kept) */
void orc_galerkin(const double* ch, const double* P, double* out) {
    double A[256], T[16][4];
    orc_patch_operator(ch, A);
    memset(T, 0, sizeof T);
    for (int r = 0; r < 16; ++r)
        for (int k = 0; k < 16; ++k) {
            double a = A[r * 16 + k];
            if (a == 0.0) continue;
            for (int c = 0; c < 4; ++c) T[r][c] += a * P[k * 4 + c];
        }
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) {
            double v = 0.0;
            for (int k = 0; k < 16; ++k) v += P[k * 4 + r] * T[k][c];
            out[r * 4 + c] = v;
        }
}

/* transfer.cpp:41-72 */
static int solve4(double M[4][4], double rhs[4][4]) {
    int perm[4] = {0, 1, 2, 3};
    for (int k = 0; k < 4; ++k) {
        int p = k;
        for (int r = k + 1; r < 4; ++r)
            if (fabs(M[perm[r]][k]) > fabs(M[perm[p]][k])) p = r;
        int t = perm[k];
        perm[k] = perm[p];
        perm[p] = t;
        double piv = M[perm[k]][k];
        if (fabs(piv) < 1e-14) return 0;
        for (int r = k + 1; r < 4; ++r) {
            double f = M[perm[r]][k] / piv;
            if (f == 0.0) continue;
            for (int c = k; c < 4; ++c) M[perm[r]][c] -= f * M[perm[k]][c];
            for (int c = 0; c < 4; ++c) rhs[perm[r]][c] -= f * rhs[perm[k]][c];
        }
    }
    for (int k = 3; k >= 0; --k)
        for (int c = 0; c < 4; ++c) {
            double v = rhs[perm[k]][c];
            for (int j = k + 1; j < 4; ++j) v -= M[perm[k]][j] * rhs[perm[j]][c];
            rhs[perm[k]][c] = v / M[perm[k]][k];
        }
    double tmp[4][4];
    for (int k = 0; k < 4; ++k)
        for (int c = 0; c < 4; ++c) tmp[k][c] = rhs[perm[k]][c];
    memcpy(rhs, tmp, sizeof tmp);
    return 1;
}

/* 3x3 patch stencil truncated at the patch boundary, transfer.cpp:29-39 */
static void stencil_of(const double* A, int L, double S[3][3]) {
    int lx = L % 4, ly = L / 4;
    for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
            int nx = lx + dx, ny = ly + dy;
            S[dy + 1][dx + 1] =
                (nx >= 0 && nx < 4 && ny >= 0 && ny < 4) ? A[L * 16 + ny * 4 + nx] : 0.0;
        }
}

/* transfer.cpp:95-180 */
int orc_boxmg(const double* ch, double* P) {
    int fallback = 0;
    double geo[64], A[256];
    orc_geometric(geo);
    orc_patch_operator(ch, A);
    memset(P, 0, 64 * sizeof(double));
    static const int corner_lattice[4] = {0, 3, 12, 15};
    for (int c = 0; c < 4; ++c) P[corner_lattice[c] * 4 + c] = 1.0;
    static const struct {
        int ids[2], endA, endB, along_x;
    } edges[4] = {{{1, 2}, 0, 1, 1}, {{13, 14}, 2, 3, 1}, {{4, 8}, 0, 2, 0}, {{7, 11}, 1, 3, 0}};
    for (int e = 0; e < 4; ++e) {
        double w[2], c[2], s[2];
        int ok = 1;
        for (int k = 0; k < 2; ++k) {
            double S[3][3];
            stencil_of(A, edges[e].ids[k], S);
            if (edges[e].along_x) {
                w[k] = S[0][0] + S[1][0] + S[2][0];
                c[k] = S[0][1] + S[1][1] + S[2][1];
                s[k] = S[0][2] + S[1][2] + S[2][2];
            } else {
                w[k] = S[0][0] + S[0][1] + S[0][2];
                c[k] = S[1][0] + S[1][1] + S[1][2];
                s[k] = S[2][0] + S[2][1] + S[2][2];
            }
            if (!(c[k] > 0.0)) ok = 0;
        }
        double det = c[0] * c[1] - s[0] * w[1];
        if (!ok || fabs(det) < 1e-300) {
            for (int k = 0; k < 2; ++k) {
                for (int cc = 0; cc < 4; ++cc)
                    P[edges[e].ids[k] * 4 + cc] = geo[edges[e].ids[k] * 4 + cc];
                ++fallback;
            }
            continue;
        }
        P[edges[e].ids[0] * 4 + edges[e].endA] = (-w[0] * c[1]) / det;
        P[edges[e].ids[1] * 4 + edges[e].endA] = (w[0] * w[1]) / det;
        P[edges[e].ids[0] * 4 + edges[e].endB] = (s[0] * s[1]) / det;
        P[edges[e].ids[1] * 4 + edges[e].endB] = (-c[0] * s[1]) / det;
    }
    static const int interior[4] = {5, 6, 9, 10};
    double M[4][4], rhs[4][4];
    memset(rhs, 0, sizeof rhs);
    for (int r = 0; r < 4; ++r)
        for (int q = 0; q < 4; ++q) M[r][q] = A[interior[r] * 16 + interior[q]];
    for (int r = 0; r < 4; ++r)
        for (int L = 0; L < 16; ++L) {
            int is_int = L == 5 || L == 6 || L == 9 || L == 10;
            if (is_int) continue;
            double a = A[interior[r] * 16 + L];
            if (a == 0.0) continue;
            for (int cc = 0; cc < 4; ++cc) rhs[r][cc] -= a * P[L * 4 + cc];
        }
    if (solve4(M, rhs)) {
        for (int r = 0; r < 4; ++r)
            for (int cc = 0; cc < 4; ++cc) P[interior[r] * 4 + cc] = rhs[r][cc];
    } else {
        for (int r = 0; r < 4; ++r) {
            for (int cc = 0; cc < 4; ++cc) P[interior[r] * 4 + cc] = geo[interior[r] * 4 + cc];
            ++fallback;
        }
    }
    return fallback;
}

/* ================================================================ grid */

typedef struct {
    int N;            /* cells per axis */
    double h;         /* Mesh::level_h = pow(1/3, l), mesh.hpp:87 */
    double inv3l;     /* pow(3.0, l): Vertex::x() divisor, mesh.hpp:159 */
    int32_t* order;   /* level_cells creation order (mesh.cpp:83-93) */
    int32_t* vorder;  /* level_vertices creation order (mesh.cpp:53-64) */
    int64_t* rx;      /* creation rank = rx[cx] + ry[cy] */
    int64_t* ry;
    double* op;       /* 16 per cell: decoded stored operator (stream.hpp:133-139) */
    double* P;        /* 64 per cell (refined levels only) */
    int32_t* p1;
    uint8_t* p2;
    int32_t* p3;
    int32_t* n;
    uint32_t* epoch;
    uint8_t* has_P;
    uint8_t* dirty; /* CellStream slot dirty[2] as bits 0/1 (stream.cpp:240-260) */
    double* v[LZB_V_NFIELDS];
} orc_level;

struct orc_grid {
    lzb_grid_desc d;
    int D;
    orc_level* L;
    uint32_t cycle;
    double first_residual;
    double* history;
    int nhist, cap_hist;
    uint64_t dof_updates_total;
    double max_delta_published;
    int max_samples;
    uint64_t zero_norm_accepts;
    /* TaskPool with workers = 1 (scheduler.cpp:88-111): FIFO of leaf cells */
    int32_t* queue;
    int64_t qhead, qtail, qcap;
    /* the high-priority class: coarse_recompute tasks (level, cell), FIFO */
    int32_t* hq;
    int64_t hhead, htail, hcap;
    uint64_t spawned, completed;
    double geo[64];
    double kunit[16];
};

static int64_t ipow3(int l) {
    int64_t p = 1;
    for (int i = 0; i < l; ++i) p *= 3;
    return p;
}

orc_grid* orc_grid_create(const lzb_grid_desc* d) {
    if (d->depth < 1) {
        set_err(LZB_ERR_INVALID, "mesh depth must be >= 1");
        return NULL;
    }
    orc_grid* g = calloc(1, sizeof *g);
    g->d = *d;
    g->D = d->depth;
    g->first_residual = -1.0;
    g->L = calloc((size_t)g->D + 1, sizeof(orc_level));
    orc_geometric(g->geo);
    orc_subcell_stiffness(0.0, 1.0, 0.0, 1.0, g->kunit);
    for (int l = 0; l <= g->D; ++l) {
        orc_level* L = &g->L[l];
        int N = (int)ipow3(l);
        int64_t nc = (int64_t)N * N, nv = (int64_t)(N + 1) * (N + 1);
        L->N = N;
        L->h = pow(1.0 / 3, l);
        L->inv3l = pow(3.0, l);
        L->order = malloc(nc * sizeof(int32_t));
        L->vorder = malloc(nv * sizeof(int32_t));
        L->rx = malloc(N * sizeof(int64_t));
        L->ry = malloc(N * sizeof(int64_t));
        L->op = calloc(nc * 16, sizeof(double));
        L->p1 = calloc(nc, sizeof(int32_t));
        L->p2 = calloc(nc, 1);
        L->p3 = calloc(nc, sizeof(int32_t));
        L->n = calloc(nc, sizeof(int32_t));
        L->epoch = calloc(nc, sizeof(uint32_t));
        L->has_P = calloc(nc, 1);
        L->dirty = calloc(nc, 1);
        if (l < g->D) L->P = calloc(nc * 64, sizeof(double));
        for (int f = 0; f < LZB_V_NFIELDS; ++f) L->v[f] = calloc(nv, sizeof(double));
        for (int c = 0; c < N; ++c) {
            L->rx[c] = l == 0 ? 0 : 9 * g->L[l - 1].rx[c / 3] + 3 * (c % 3);
            L->ry[c] = l == 0 ? 0 : 9 * g->L[l - 1].ry[c / 3] + (c % 3);
        }
        if (l == 0) {
            L->order[0] = 0;
            for (int k = 0; k < 4; ++k) L->vorder[k] = cdy(k) * 2 + cdx(k);
        } else {
            orc_level* Pl = &g->L[l - 1];
            uint8_t* seen = calloc(nv, 1);
            int64_t oc = 0, ov = 0;
            for (int64_t q = 0; q < (int64_t)Pl->N * Pl->N; ++q) {
                int pc = Pl->order[q], px = pc % Pl->N, py = pc / Pl->N;
                for (int lx = 0; lx < 3; ++lx)
                    for (int ly = 0; ly < 3; ++ly) {
                        int cx = 3 * px + lx, cy = 3 * py + ly;
                        L->order[oc++] = cy * N + cx;
                        for (int k = 0; k < 4; ++k) {
                            int vi = (cy + cdy(k)) * (N + 1) + cx + cdx(k);
                            if (!seen[vi]) {
                                seen[vi] = 1;
                                L->vorder[ov++] = vi;
                            }
                        }
                    }
            }
            free(seen);
        }
    }
    return g;
}

void orc_grid_destroy(orc_grid* g) {
    if (!g) return;
    for (int l = 0; l <= g->D; ++l) {
        orc_level* L = &g->L[l];
        free(L->order); free(L->vorder); free(L->rx); free(L->ry); free(L->op); free(L->P);
        free(L->p1); free(L->p2); free(L->p3); free(L->n); free(L->epoch); free(L->has_P); free(L->dirty);
        for (int f = 0; f < LZB_V_NFIELDS; ++f) free(L->v[f]);
    }
    free(g->L);
    free(g->history);
    free(g->queue);
    free(g->hq);
    free(g);
}

static inline int is_boundary(const orc_level* L, int ix, int iy) {
    return ix == 0 || iy == 0 || ix == L->N || iy == L->N; /* mesh.cpp:117-120 */
}
static inline int64_t crank(const orc_level* L, int cx, int cy) { return L->rx[cx] + L->ry[cy]; }

/* element_or_baseline / baseline, stream.cpp:82-84,206-210 */
static void baseline(const orc_grid* g, int l, int cx, int cy, double* out) {
    const orc_level* L = &g->L[l];
    orc_integrate_element(&g->d.field, cx * L->h, cy * L->h, L->h, 1, out);
}
static void element_or_baseline(const orc_grid* g, int l, int c, double* out) {
    const orc_level* L = &g->L[l];
    if (L->p1[c] != LZB_P1_BOTTOM) memcpy(out, L->op + 16 * c, 128);
    else if (g->d.start_geometric) memcpy(out, g->kunit, 128); /* extension: the geometric stencil (eps = 1) */
    else baseline(g, l, c % L->N, c / L->N, out);
}
static const double* transfer_or_geometric(const orc_grid* g, int l, int c) {
    const orc_level* L = &g->L[l];
    return L->has_P[c] ? L->P + 64 * c : g->geo; /* stream.cpp:212-216 */
}

/* CellStream::mark_parent_dirty (stream.cpp:240-245): the parent's flag of
 * the parity (cycle + 1) & 1, taken by the walk of the next cycle */
static void mark_parent_dirty(orc_grid* g, int l, int c) {
    if (l == 0) return;
    const orc_level* L = &g->L[l];
    int cx = c % L->N, cy = c / L->N;
    orc_level* P = &g->L[l - 1];
    P->dirty[(cy / 3) * P->N + cx / 3] |= (uint8_t)(1u << ((g->cycle + 1) & 1u));
}

/* stream.cpp:100-132 (caller sets p1, assembly.cpp) */
static int publish_element(orc_grid* g, int l, int c, const double* m, int n) {
    orc_level* L = &g->L[l];
    double base[16], surplus[16];
    baseline(g, l, c % L->N, c / L->N, base);
    for (int i = 0; i < 16; ++i) surplus[i] = m[i] - base[i];
    int p3 = orc_choose_precision(surplus, 16, g->d.delta_max);
    if (p3 < 0) return -p3;
    double delta = 0.0;
    for (int i = 0; i < 16; ++i) {
        double rt;
        int rc = roundtrip(surplus[i], p3, &rt);
        if (rc) return rc;
        double err = fabs(rt - surplus[i]);
        if (err > delta) delta = err;
        L->op[16 * c + i] = base[i] + rt;
    }
    if (delta > g->max_delta_published) g->max_delta_published = delta;
    if (n > g->max_samples) g->max_samples = n;
    L->n[c] = n;
    L->epoch[c] = g->cycle;
    L->p3[c] = p3;
    mark_parent_dirty(g, l, c);
    return 0;
}

/* stream.cpp:134-184; returns 1 when published */
static int publish_coarse(orc_grid* g, int l, int c, const double* m, const double* P, int* rc) {
    orc_level* L = &g->L[l];
    double base[16], joint[80], dec[16], Pd[64];
    baseline(g, l, c % L->N, c / L->N, base);
    for (int i = 0; i < 16; ++i) joint[i] = m[i] - base[i];
    for (int i = 0; i < 64; ++i) joint[16 + i] = P[i] - g->geo[i];
    int p3 = orc_choose_precision(joint, 80, g->d.delta_max);
    *rc = 0;
    if (p3 < 0) {
        *rc = -p3;
        return 0;
    }
    double delta = 0.0;
    for (int i = 0; i < 80; ++i) {
        double rt;
        if ((*rc = roundtrip(joint[i], p3, &rt))) return 0;
        double err = fabs(rt - joint[i]);
        if (err > delta) delta = err;
        if (i < 16) dec[i] = base[i] + rt;
        else Pd[i - 16] = g->geo[i - 16] + rt;
    }
    if (L->p1[c] == LZB_P1_TOP && L->has_P[c]) { /* std::array == (stream.cpp:153-158) */
        int same = 1;
        for (int i = 0; i < 16; ++i) same &= dec[i] == L->op[16 * c + i];
        for (int i = 0; i < 64; ++i) same &= Pd[i] == L->P[64 * c + i];
        if (same) return 0;
    }
    if (delta > g->max_delta_published) g->max_delta_published = delta;
    memcpy(L->op + 16 * c, dec, 128);
    memcpy(L->P + 64 * c, Pd, 512);
    L->has_P[c] = 1;
    L->n[c] = 1;
    L->epoch[c] = g->cycle;
    L->p3[c] = p3;
    L->p1[c] = LZB_P1_TOP;
    mark_parent_dirty(g, l, c);
    return 1;
}

static double max_abs16(const double* a) {
    double m = 0.0;
    for (int i = 0; i < 16; ++i) {
        double f = fabs(a[i]);
        if (m < f) m = f;
    }
    return m;
}

/* n -> n+1 (assembly.cpp:36-37) or, as the BASELINE knob, n -> 2n; capped at n_max */
static int next_n(const orc_grid* g, int n) {
    int nn = g->d.schedule == LZB_SCHEDULE_DOUBLE ? 2 * n : n + 1;
    if (g->d.n_max > 0 && nn > g->d.n_max) nn = g->d.n_max;
    return nn;
}

/* assembly.cpp:10-60 (n -> n+1; LZB_SCHEDULE_DOUBLE is the BASELINE knob) */
/* pre: NULL, or the integration at next_n(p1) computed ahead (a pure
 * function of the cell and n, see prefetch_integrations) */
static int adaptive_step_pre(orc_grid* g, int c, const double* pre);
static int adaptive_step(orc_grid* g, int c) { return adaptive_step_pre(g, c, NULL); }
static int adaptive_step_pre(orc_grid* g, int c, const double* pre) {
    orc_level* L = &g->L[g->D];
    int32_t p1 = L->p1[c];
    if (p1 == LZB_P1_TOP) return 0;
    int cx = c % L->N, cy = c / L->N;
    if (p1 == LZB_P1_BOTTOM) {
        double m[16];
        orc_integrate_element(&g->d.field, cx * L->h, cy * L->h, L->h, 1, m);
        int rc = publish_element(g, g->D, c, m, 1);
        if (rc) return rc;
        L->p1[c] = 1;
        return 0;
    }
    int n = p1, nn = next_n(g, n);
    if (g->d.n_max > 0 && n >= g->d.n_max) { /* extension: the sampling cap ends refinement */
        L->p1[c] = LZB_P1_TOP;
        return 0;
    }
    double fresh[16], diff[16];
    if (pre) memcpy(fresh, pre, sizeof fresh);
    else orc_integrate_element(&g->d.field, cx * L->h, cy * L->h, L->h, nn, fresh);
    const double* old = L->op + 16 * c;
    double denom = max_abs16(old), ratio = 0.0;
    if (denom == 0.0) {
        g->zero_norm_accepts++;
    } else {
        for (int i = 0; i < 16; ++i) diff[i] = fresh[i] - old[i];
        ratio = max_abs16(diff) / denom;
    }
    if (ratio < g->d.termination_c) {
        L->p1[c] = LZB_P1_TOP;
        return 0;
    }
    int rc = publish_element(g, g->D, c, fresh, nn);
    if (rc) return rc;
    L->p1[c] = nn;
    return 0;
}

static void spawn(orc_grid* g, int c) {
    orc_level* L = &g->L[g->D];
    if (L->p2[c]) return; /* assembly.cpp:64 */
    L->p2[c] = 1;
    if (g->qtail == g->qcap) {
        int64_t live = g->qtail - g->qhead;
        if (g->qhead > 0 && live < g->qcap / 2) {
            memmove(g->queue, g->queue + g->qhead, live * sizeof(int32_t));
        } else {
            g->qcap = g->qcap ? 2 * g->qcap : 1024;
            g->queue = realloc(g->queue, g->qcap * sizeof(int32_t));
            memmove(g->queue, g->queue + g->qhead, live * sizeof(int32_t));
        }
        g->qhead = 0;
        g->qtail = live;
    }
    g->queue[g->qtail++] = c;
    g->spawned++;
}

/* Assembler::spawn_forced (assembly.cpp:138-154): an integrate task that only
 * occupies the pool (its result is discarded); queued as -(c + 1). */
static void spawn_forced(orc_grid* g, int c) {
    orc_level* L = &g->L[g->D];
    if (L->p2[c]) return; /* assembly.cpp:140 */
    spawn(g, c);
    g->queue[g->qtail - 1] = -c - 1;
}

/* A coarse_recompute task (solver.cpp:86-90) in the high-priority class. */
static void spawn_coarse(orc_grid* g, int l, int c) {
    if (g->htail + 2 > g->hcap) {
        int64_t live = g->htail - g->hhead;
        g->hcap = g->hcap ? 2 * g->hcap : 1024;
        int32_t* q = malloc(g->hcap * sizeof(int32_t));
        memcpy(q, g->hq + g->hhead, live * sizeof(int32_t));
        free(g->hq);
        g->hq = q;
        g->hhead = 0;
        g->htail = live;
    }
    g->hq[g->htail++] = l;
    g->hq[g->htail++] = c;
    g->spawned++;
}

static int recompute_coarse(orc_grid* g, int l, int c, int* published);

/* TaskPool::begin_cycle with workers == 1: the high class first, then the
 * leaf tasks, FIFO, <= throttle tasks in all (scheduler.cpp:88-111) */
/* The leaf tasks a begin_cycle will run integrate at next_n(p1) of their
 * cell; p1 of a queued leaf cannot change before its task runs (p2 allows one
 * task per cell, coarse tasks do not touch leaves), so those integrations are
 * computed ahead on host threads, in any order -- each is the same pure
 * function call as inside adaptive_step. The protocol itself then runs
 * strictly in FIFO order. (A speed-up of the checker only.) */
typedef struct {
    const orc_grid* g;
    const int32_t* cells;
    int64_t k0, k1;
    double* out;
} pre_job;
static void* pre_worker(void* arg) {
    pre_job* j = (pre_job*)arg;
    const orc_level* L = &j->g->L[j->g->D];
    for (int64_t k = j->k0; k < j->k1; ++k) {
        int c = j->cells[k];
        if (c < 0) continue; /* a forced task */
        int p1 = L->p1[c];
        if (p1 == LZB_P1_TOP || p1 == LZB_P1_BOTTOM) continue;
        if (j->g->d.n_max > 0 && p1 >= j->g->d.n_max) continue;
        orc_integrate_element(&j->g->d.field, (c % L->N) * L->h, (c / L->N) * L->h, L->h, next_n(j->g, p1),
                              j->out + 16 * k);
    }
    return NULL;
}
static double* prefetch_integrations(orc_grid* g, int64_t count) {
    if (count < 4096) return NULL;
    double* out = malloc((size_t)count * 16 * sizeof(double));
    if (!out) return NULL;
    long nt = sysconf(_SC_NPROCESSORS_ONLN);
    int threads = nt < 1 ? 1 : (nt > 256 ? 256 : (int)nt);
    pthread_t tid[256];
    pre_job jobs[256];
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (pre_job){g, g->queue + g->qhead, count * t / threads, count * (t + 1) / threads, out};
        if (pthread_create(&tid[t], NULL, pre_worker, &jobs[t]) != 0) {
            pre_worker(&jobs[t]);
            tid[t] = 0;
        }
    }
    for (int t = 0; t < threads; ++t)
        if (tid[t]) pthread_join(tid[t], NULL);
    return out;
}

static int pool_begin_cycle(orc_grid* g) {
    uint64_t budget = g->d.throttle == 0 ? UINT64_MAX : g->d.throttle;
    /* leaf tasks this call will run: those the budget leaves after the high class */
    int64_t nleaf = g->qtail - g->qhead, nhigh = (g->htail - g->hhead) / 2;
    if (budget != UINT64_MAX) {
        int64_t left = (int64_t)budget - nhigh;
        if (left < nleaf) nleaf = left < 0 ? 0 : left;
    }
    const int64_t qbase = g->qhead;
    double* pre = prefetch_integrations(g, nleaf);
    while (g->hhead < g->htail || g->qhead < g->qtail) {
        if (budget == 0) break;
        if (budget != UINT64_MAX) --budget;
        int rc;
        if (g->hhead < g->htail) {
            int l = g->hq[g->hhead], c = g->hq[g->hhead + 1], pub;
            g->hhead += 2;
            rc = recompute_coarse(g, l, c, &pub);
        } else {
            int64_t k = g->qhead - qbase;
            int c = g->queue[g->qhead++];
            if (c < 0) { /* spawn_forced's task: integrate_element(box, eps, fixed_n), result discarded */
                g->L[g->D].p2[-c - 1] = 0;
            } else {
                rc = adaptive_step_pre(g, c, pre && k < nleaf ? pre + 16 * k : NULL);
                g->L[g->D].p2[c] = 0;
            }
        }
        g->completed++;
        if (rc) {
            free(pre);
            return rc;
        }
    }
    free(pre);
    return 0;
}

/* TaskPool::try_run_one (scheduler.cpp:113-128): the oldest task, high class
 * first, regardless of the cycle budget */
static int try_run_one(orc_grid* g) {
    int rc = 0;
    if (g->hhead < g->htail) {
        int l = g->hq[g->hhead], c = g->hq[g->hhead + 1], pub;
        g->hhead += 2;
        rc = recompute_coarse(g, l, c, &pub);
    } else if (g->qhead < g->qtail) {
        int c = g->queue[g->qhead++];
        if (c < 0) {
            g->L[g->D].p2[-c - 1] = 0;
        } else {
            rc = adaptive_step(g, c);
            g->L[g->D].p2[c] = 0;
        }
    } else {
        return 0;
    }
    g->completed++;
    return rc;
}

/* assembly.cpp:76-109 */
static int request_stencil(orc_grid* g, int c) {
    orc_level* L = &g->L[g->D];
    int rc = 0;
    switch (g->d.mode) {
        case LZB_EAGER:
        case LZB_LAZY:
            while (L->p1[c] != LZB_P1_TOP)
                if ((rc = adaptive_step(g, c))) return rc;
            return 0;
        case LZB_ADAPTIVE:
            /* block while a task of this cell is queued, running queued work
             * (assembly.cpp:86-93); only forced tasks set p2 in this mode */
            while (L->p2[c])
                if ((rc = try_run_one(g))) return rc;
            if (L->p1[c] != LZB_P1_TOP) rc = adaptive_step(g, c);
            return rc;
        case LZB_ANARCHIC:
            if (L->p1[c] == LZB_P1_BOTTOM && g->d.start_geometric) {
                /* extension: the first integration is deferred too */
                if (!L->p2[c]) spawn(g, c);
                return 0;
            }
            if (L->p1[c] == LZB_P1_BOTTOM) {
                if ((rc = adaptive_step(g, c))) return rc;
                spawn(g, c);
                return 0;
            }
            if (L->p1[c] != LZB_P1_TOP && !L->p2[c]) spawn(g, c);
            return 0;
    }
    return 0;
}

/* solver.cpp:59-77 */
static int recompute_coarse(orc_grid* g, int l, int c, int* published) {
    orc_level* L = &g->L[l];
    orc_level* F = &g->L[l + 1];
    int cx = c % L->N, cy = c / L->N;
    double ch[144], P[64], m[16];
    *published = 0;
    for (int lx = 0; lx < 3; ++lx)
        for (int ly = 0; ly < 3; ++ly) {
            int fc = (3 * cy + ly) * F->N + 3 * cx + lx;
            if (F->p1[fc] == LZB_P1_BOTTOM) return 0;
            memcpy(ch + 16 * (lx * 3 + ly), F->op + 16 * fc, 128);
        }
    if (g->d.transfer == LZB_BOXMG) orc_boxmg(ch, P);
    else memcpy(P, g->geo, sizeof P);
    orc_galerkin(ch, P, m);
    int rc;
    *published = publish_coarse(g, l, c, m, P, &rc);
    return rc;
}

/* pre-order walk, mesh.cpp:140-150; visit(l, cell) */
typedef int (*visit_fn)(orc_grid*, int l, int c, void* ctx);
static int walk(orc_grid* g, int l, int cx, int cy, visit_fn fn, void* ctx) {
    int rc = fn(g, l, cy * g->L[l].N + cx, ctx);
    if (rc) return rc;
    if (l == g->D) return 0;
    for (int lx = 0; lx < 3; ++lx)
        for (int ly = 0; ly < 3; ++ly)
            if ((rc = walk(g, l + 1, 3 * cx + lx, 3 * cy + ly, fn, ctx))) return rc;
    return 0;
}

/* take_dirty (stream.cpp:247-250): the flag of the current cycle's parity */
static int take_dirty(orc_grid* g, int l, int c) {
    uint8_t bit = (uint8_t)(1u << (g->cycle & 1u));
    int set = (g->L[l].dirty[c] & bit) != 0;
    g->L[l].dirty[c] &= (uint8_t)~bit;
    return set;
}

static int visit_assembly(orc_grid* g, int l, int c, void* ctx) { /* solver.cpp:79-97 */
    (void)ctx;
    if (l < g->D) {
        if (g->d.policy == LZB_RIPPLE) {
            if (take_dirty(g, l, c)) spawn_coarse(g, l, c);
            return 0;
        }
        int pub;
        int rc = recompute_coarse(g, l, c, &pub); /* policy always */
        take_dirty(g, l, c);                      /* consumed implicitly */
        return rc;
    }
    return request_stencil(g, c);
}

static int visit_eager(orc_grid* g, int l, int c, void* ctx) {
    (void)ctx;
    if (l < g->D) return 0;
    while (g->L[l].p1[c] != LZB_P1_TOP) {
        int rc = adaptive_step(g, c);
        if (rc) return rc;
    }
    return 0;
}

int orc_eager_setup(orc_grid* g) { return walk(g, 0, 0, 0, visit_eager, NULL); } /* assembly.cpp:111-118 */

int orc_assemble_fixed(orc_grid* g, int n) {
    orc_level* L = &g->L[g->D];
    double m[16];
    for (int c = 0; c < L->N * L->N; ++c) {
        orc_integrate_element(&g->d.field, (c % L->N) * L->h, (c / L->N) * L->h, L->h, n, m);
        int rc = publish_element(g, g->D, c, m, n);
        if (rc) return rc;
        L->p1[c] = LZB_P1_TOP;
    }
    return 0;
}

/* problem.cpp:50-68 */
int orc_init_noise(orc_grid* g, uint64_t seed) {
    for (int l = 0; l <= g->D; ++l) {
        orc_level* L = &g->L[l];
        for (int iy = 0; iy <= L->N; ++iy)
            for (int ix = 0; ix <= L->N; ++ix) {
                double* u = &L->v[LZB_V_U][iy * (L->N + 1) + ix];
                if (is_boundary(L, ix, iy)) {
                    *u = g->d.boundary_value;
                    continue;
                }
                uint64_t k = orc_splitmix64(
                    seed ^ orc_splitmix64(((uint64_t)l << 48) ^ ((uint64_t)(uint32_t)ix << 24) ^
                                          (uint64_t)(uint32_t)iy));
                *u = (4.0 / 3.0) * (double)(k >> 11) * 0x1.0p-53;
            }
    }
    /* inject_solution (mesh.cpp:226-234); no hanging vertices on regular grids */
    for (int l = g->D; l >= 1; --l) {
        orc_level *C = &g->L[l - 1], *F = &g->L[l];
        for (int iy = 0; iy <= C->N; ++iy)
            for (int ix = 0; ix <= C->N; ++ix)
                C->v[LZB_V_U][iy * (C->N + 1) + ix] = F->v[LZB_V_U][3 * iy * (F->N + 1) + 3 * ix];
    }
    return 0;
}

/* solver.cpp:39-57: the min-slot refined patch among those sharing the lattice vertex.
 * Same-level pre-order slots order like creation ranks. */
static int owns(const orc_grid* g, int l, int cx, int cy, int lx, int ly) {
    const orc_level* L = &g->L[l];
    int bx = lx == 0 || lx == 3, by = ly == 0 || ly == 3;
    if (!bx && !by) return 1;
    int64_t best = crank(L, cx, cy);
    int is_me = 1;
    for (int ox = (lx == 0 ? -1 : 0); ox <= (lx == 3 ? 1 : 0); ++ox)
        for (int oy = (ly == 0 ? -1 : 0); oy <= (ly == 3 ? 1 : 0); ++oy) {
            if (ox == 0 && oy == 0) continue;
            int nx = cx + ox, ny = cy + oy;
            if (nx < 0 || ny < 0 || nx >= L->N || ny >= L->N) continue;
            if (l >= g->D) continue; /* neighbour must be refined */
            int64_t r = crank(L, nx, ny);
            if (r < best) {
                best = r;
                is_me = 0;
            }
        }
    return is_me;
}

/* solver.cpp:99-118 */
static void init_level_rhs(orc_grid* g) {
    for (int l = 0; l <= g->D; ++l) {
        orc_level* L = &g->L[l];
        int64_t nv = (int64_t)(L->N + 1) * (L->N + 1);
        memset(L->v[LZB_V_FL], 0, nv * sizeof(double));
        memset(L->v[LZB_V_DIAG], 0, nv * sizeof(double));
    }
    if (!rhs_active(&g->d.rhs)) return;
    orc_level* L = &g->L[g->D];
    double w = L->h * L->h / 4.0;
    for (int64_t q = 0; q < (int64_t)L->N * L->N; ++q) {
        int c = L->order[q], cx = c % L->N, cy = c / L->N;
        for (int k = 0; k < 4; ++k) {
            int ix = cx + cdx(k), iy = cy + cdy(k);
            L->v[LZB_V_FL][iy * (L->N + 1) + ix] +=
                w * rhs_eval(&g->d.rhs, ix / L->inv3l, iy / L->inv3l);
        }
    }
}

/* solver.cpp:120-143 */
static void compute_uhat(orc_grid* g, int l) {
    orc_level* F = &g->L[l];
    int64_t nv = (int64_t)(F->N + 1) * (F->N + 1);
    memcpy(F->v[LZB_V_UHAT], F->v[LZB_V_U], nv * sizeof(double));
    if (l == 0) return;
    orc_level* C = &g->L[l - 1];
    for (int64_t q = 0; q < (int64_t)C->N * C->N; ++q) {
        int c = C->order[q], cx = c % C->N, cy = c / C->N;
        const double* P = transfer_or_geometric(g, l - 1, c);
        double uc[4];
        for (int k = 0; k < 4; ++k)
            uc[k] = C->v[LZB_V_U][(cy + cdy(k)) * (C->N + 1) + cx + cdx(k)];
        for (int ly = 0; ly < 4; ++ly)
            for (int lx = 0; lx < 4; ++lx) {
                if (!owns(g, l - 1, cx, cy, lx, ly)) continue;
                int fi = (3 * cy + ly) * (F->N + 1) + 3 * cx + lx;
                int Li = ly * 4 + lx;
                double interp = 0.0;
                for (int k = 0; k < 4; ++k) interp += P[Li * 4 + k] * uc[k];
                F->v[LZB_V_UHAT][fi] = F->v[LZB_V_U][fi] - interp;
            }
    }
}

/* solver.cpp:145-210 */
static double residual_pass(orc_grid* g) {
    init_level_rhs(g);
    for (int l = g->D; l >= 0; --l) {
        orc_level* L = &g->L[l];
        int NV = L->N + 1;
        compute_uhat(g, l);
        int64_t nv = (int64_t)NV * NV;
        memcpy(L->v[LZB_V_R], L->v[LZB_V_FL], nv * sizeof(double));
        memcpy(L->v[LZB_V_RHAT], L->v[LZB_V_FL], nv * sizeof(double));
        for (int64_t q = 0; q < (int64_t)L->N * L->N; ++q) {
            int c = L->order[q], cx = c % L->N, cy = c / L->N;
            double K[16], u[4], uh[4];
            int vi[4];
            element_or_baseline(g, l, c, K);
            for (int k = 0; k < 4; ++k) {
                vi[k] = (cy + cdy(k)) * NV + cx + cdx(k);
                u[k] = L->v[LZB_V_U][vi[k]];
                uh[k] = L->v[LZB_V_UHAT][vi[k]];
            }
            for (int row = 0; row < 4; ++row) {
                double au = 0.0, auh = 0.0;
                for (int col = 0; col < 4; ++col) {
                    au += K[row * 4 + col] * u[col];
                    auh += K[row * 4 + col] * uh[col];
                }
                L->v[LZB_V_R][vi[row]] -= au;
                L->v[LZB_V_RHAT][vi[row]] -= auh;
                L->v[LZB_V_DIAG][vi[row]] += K[row * 4 + row];
            }
        }
        for (int iy = 0; iy <= L->N; ++iy)
            for (int ix = 0; ix <= L->N; ++ix)
                if (is_boundary(L, ix, iy)) {
                    L->v[LZB_V_R][iy * NV + ix] = 0.0;
                    L->v[LZB_V_RHAT][iy * NV + ix] = 0.0;
                }
        if (l > 0) {
            orc_level* C = &g->L[l - 1];
            int NVc = C->N + 1;
            for (int64_t q = 0; q < (int64_t)C->N * C->N; ++q) {
                int c = C->order[q], cx = c % C->N, cy = c / C->N;
                const double* P = transfer_or_geometric(g, l - 1, c);
                for (int ly = 0; ly < 4; ++ly)
                    for (int lx = 0; lx < 4; ++lx) {
                        if (!owns(g, l - 1, cx, cy, lx, ly)) continue;
                        double rh = L->v[LZB_V_RHAT][(3 * cy + ly) * NV + 3 * cx + lx];
                        if (rh == 0.0) continue;
                        int Li = ly * 4 + lx;
                        for (int k = 0; k < 4; ++k)
                            C->v[LZB_V_FL][(cy + cdy(k)) * NVc + cx + cdx(k)] += P[Li * 4 + k] * rh;
                    }
            }
        }
    }
    double sq = 0.0;
    orc_level* L = &g->L[g->D]; /* fine_grid vertices: adjacent to a leaf (mesh.cpp:124-128) */
    for (int64_t q = 0; q < (int64_t)(L->N + 1) * (L->N + 1); ++q) {
        int vi = L->vorder[q], ix = vi % (L->N + 1), iy = vi / (L->N + 1);
        if (!is_boundary(L, ix, iy)) sq += L->v[LZB_V_R][vi] * L->v[LZB_V_R][vi];
    }
    return sqrt(sq);
}

/* solver.cpp:212-313 (no refinement: level_enabled is always true) */
static void update_pass(orc_grid* g, lzb_cycle_report* rep) {
    const double omega = g->d.omega;
    const int v = g->d.variant;
    for (int l = 0; l <= g->D; ++l) {
        orc_level* L = &g->L[l];
        int64_t nv = (int64_t)(L->N + 1) * (L->N + 1);
        memcpy(L->v[LZB_V_USNAP], L->v[LZB_V_U], nv * sizeof(double));
        memset(L->v[LZB_V_AUX], 0, nv * sizeof(double));
    }
    for (int l = g->D; l >= 0; --l) {
        orc_level* F = &g->L[l];
        int NV = F->N + 1;
        int aux_term = v != LZB_ADDITIVE && l > 0;
        if (aux_term) {
            orc_level* C = &g->L[l - 1];
            int NVc = C->N + 1;
            memset(C->v[LZB_V_AUX], 0, (size_t)NVc * NVc * sizeof(double));
            if (v == LZB_ADAFAC_PI) {
                for (int iy = 0; iy <= C->N; ++iy)
                    for (int ix = 0; ix <= C->N; ++ix)
                        C->v[LZB_V_AUX][iy * NVc + ix] = F->v[LZB_V_R][3 * iy * NV + 3 * ix];
            } else {
                memset(F->v[LZB_V_AUX], 0, (size_t)NV * NV * sizeof(double));
                for (int64_t q = 0; q < (int64_t)F->N * F->N; ++q) {
                    int c = F->order[q], cx = c % F->N, cy = c / F->N;
                    double K[16], rr[4];
                    int vi[4];
                    element_or_baseline(g, l, c, K);
                    for (int k = 0; k < 4; ++k) {
                        vi[k] = (cy + cdy(k)) * NV + cx + cdx(k);
                        rr[k] = F->v[LZB_V_R][vi[k]];
                    }
                    for (int row = 0; row < 4; ++row) {
                        double ar = 0.0;
                        for (int col = 0; col < 4; ++col) ar += K[row * 4 + col] * rr[col];
                        F->v[LZB_V_AUX][vi[row]] += ar;
                    }
                }
                for (int64_t q = 0; q < (int64_t)C->N * C->N; ++q) {
                    int c = C->order[q], cx = c % C->N, cy = c / C->N;
                    const double* P = transfer_or_geometric(g, l - 1, c);
                    double acc[4] = {0, 0, 0, 0};
                    for (int ly = 0; ly < 4; ++ly)
                        for (int lx = 0; lx < 4; ++lx) {
                            if (!owns(g, l - 1, cx, cy, lx, ly)) continue;
                            int fx = 3 * cx + lx, fy = 3 * cy + ly, fi = fy * NV + fx;
                            if (is_boundary(F, fx, fy)) continue;
                            double dg = F->v[LZB_V_DIAG][fi];
                            double sres = F->v[LZB_V_R][fi] -
                                          (dg != 0.0 ? omega / dg * F->v[LZB_V_AUX][fi] : 0.0);
                            int Li = ly * 4 + lx;
                            for (int k = 0; k < 4; ++k) acc[k] += P[Li * 4 + k] * sres;
                        }
                    for (int k = 0; k < 4; ++k)
                        C->v[LZB_V_AUX][(cy + cdy(k)) * NVc + cx + cdx(k)] += acc[k];
                }
            }
            for (int64_t q = 0; q < (int64_t)C->N * C->N; ++q) {
                int c = C->order[q], cx = c % C->N, cy = c / C->N;
                const double* P = transfer_or_geometric(g, l - 1, c);
                double caux[4];
                for (int k = 0; k < 4; ++k) {
                    int ix = cx + cdx(k), iy = cy + cdy(k), vi = iy * NVc + ix;
                    double dg = C->v[LZB_V_DIAG][vi];
                    caux[k] = (!is_boundary(C, ix, iy) && dg != 0.0)
                                  ? omega / dg * C->v[LZB_V_AUX][vi]
                                  : 0.0;
                }
                for (int ly = 0; ly < 4; ++ly)
                    for (int lx = 0; lx < 4; ++lx) {
                        if (!owns(g, l - 1, cx, cy, lx, ly)) continue;
                        int fx = 3 * cx + lx, fy = 3 * cy + ly;
                        if (is_boundary(F, fx, fy)) continue;
                        int Li = ly * 4 + lx;
                        double p = 0.0;
                        for (int k = 0; k < 4; ++k) p += P[Li * 4 + k] * caux[k];
                        F->v[LZB_V_U][fy * NV + fx] -= p;
                    }
            }
        }
        double damping = v == LZB_ADDITIVE ? pow(omega, g->D - l + 1) : omega;
        for (int iy = 0; iy <= F->N; ++iy)
            for (int ix = 0; ix <= F->N; ++ix) {
                if (is_boundary(F, ix, iy)) continue;
                int vi = iy * NV + ix;
                double dg = F->v[LZB_V_DIAG][vi];
                if (dg != 0.0) F->v[LZB_V_U][vi] += damping / dg * F->v[LZB_V_R][vi];
                if (l == g->D) rep->dof_updates += 1;
                else rep->coarse_updates += 1;
            }
    }
}

/* solver.cpp:315-342 */
static void prolong_corrections(orc_grid* g) {
    for (int l = 1; l <= g->D; ++l) {
        orc_level *C = &g->L[l - 1], *F = &g->L[l];
        int NVc = C->N + 1, NV = F->N + 1;
        for (int64_t q = 0; q < (int64_t)C->N * C->N; ++q) {
            int c = C->order[q], cx = c % C->N, cy = c / C->N;
            const double* P = transfer_or_geometric(g, l - 1, c);
            double delta[4];
            int any = 0;
            for (int k = 0; k < 4; ++k) {
                int vi = (cy + cdy(k)) * NVc + cx + cdx(k);
                delta[k] = C->v[LZB_V_U][vi] - C->v[LZB_V_USNAP][vi];
                any |= delta[k] != 0.0;
            }
            if (!any) continue;
            for (int ly = 0; ly < 4; ++ly)
                for (int lx = 0; lx < 4; ++lx) {
                    if (!owns(g, l - 1, cx, cy, lx, ly)) continue;
                    int fx = 3 * cx + lx, fy = 3 * cy + ly;
                    if (is_boundary(F, fx, fy)) continue;
                    int Li = ly * 4 + lx;
                    double p = 0.0;
                    for (int k = 0; k < 4; ++k) p += P[Li * 4 + k] * delta[k];
                    F->v[LZB_V_U][fy * NV + fx] += p;
                }
        }
    }
}

static void finish_cycle_sync(orc_grid* g) { /* solver.cpp:344-347 */
    for (int l = g->D; l >= 1; --l) {
        orc_level *C = &g->L[l - 1], *F = &g->L[l];
        for (int iy = 0; iy <= C->N; ++iy)
            for (int ix = 0; ix <= C->N; ++ix)
                C->v[LZB_V_U][iy * (C->N + 1) + ix] = F->v[LZB_V_U][3 * iy * (F->N + 1) + 3 * ix];
    }
}

/* stream.cpp:268-301 */
int orc_stats(orc_grid* g, lzb_compression_stats* st) {
    memset(st, 0, sizeof *st);
    double ratio_sum = 0.0;
    long double n_sum = 0.0;
    for (int l = 0; l <= g->D; ++l) {
        orc_level* L = &g->L[l];
        for (int64_t q = 0; q < (int64_t)L->N * L->N; ++q) {
            int c = L->order[q];
            int refined = l < g->D;
            uint64_t entries = refined ? 144 : 16;
            uint64_t bytes = L->p1[c] == LZB_P1_BOTTOM ? 1 : 1 + (uint64_t)L->p3[c] * entries;
            st->total_stored_bytes += bytes;
            st->total_uncompressed_bytes += 8 * entries;
            if (refined) continue;
            int p3 = L->p1[c] != LZB_P1_BOTTOM ? L->p3[c] : 0;
            st->p3_histogram[p3] += 1;
            st->fine_cells += 1;
            st->fine_stored_bytes += bytes;
            st->fine_uncompressed_bytes += 128;
            ratio_sum += 128.0 / (double)bytes;
            int n = L->p1[c] != LZB_P1_BOTTOM ? L->n[c] : 0;
            if (n > st->max_n) st->max_n = n;
            n_sum += n;
        }
    }
    if (st->fine_cells) {
        st->fine_factor_totals = (double)st->fine_uncompressed_bytes / (double)st->fine_stored_bytes;
        st->fine_factor_mean = ratio_sum / (double)st->fine_cells;
        st->avg_n = (double)(n_sum / st->fine_cells);
    }
    if (st->total_stored_bytes)
        st->total_factor = (double)st->total_uncompressed_bytes / (double)st->total_stored_bytes;
    st->max_delta = g->max_delta_published;
    st->max_sample_count = g->max_samples;
    return 0;
}

/* solver.cpp:8-16 */
static int check_termination(const orc_grid* g) {
    if (g->nhist == 0) return LZB_CONTINUE;
    double normalized = g->history[g->nhist - 1] / g->history[0];
    if (normalized <= g->d.target) return LZB_CONVERGED;
    if (normalized >= g->d.divergence) return LZB_DIVERGED;
    if ((int)g->cycle >= g->d.max_cycles) return LZB_TIMEOUT;
    return LZB_CONTINUE;
}

/* solver.cpp:349-400 */
int orc_step(orc_grid* g, lzb_cycle_report* rep) {
    memset(rep, 0, sizeof *rep);
    ++g->cycle;
    int rc = pool_begin_cycle(g);
    if (rc) return rc;
    rep->cycle = (int32_t)g->cycle;
    if (g->d.forced_fraction > 0.0) { /* on_cycle_start of run_experiment, experiment.cpp:260-270 */
        orc_level* L = &g->L[g->D];
        int64_t id0 = 0; /* cell ids: level by level in creation order (mesh.cpp:66-102, 253-272) */
        for (int l = 0; l < g->D; ++l) id0 += (int64_t)g->L[l].N * g->L[l].N;
        for (int64_t q = 0; q < (int64_t)L->N * L->N; ++q) {
            uint64_t id = (uint64_t)(id0 + q);
            double roll = (double)(orc_splitmix64(0x6f4ce1a3ull ^ id) >> 11) * 0x1.0p-53;
            if (roll < g->d.forced_fraction) spawn_forced(g, L->order[q]);
        }
    }
    if ((rc = walk(g, 0, 0, 0, visit_assembly, NULL))) return rc;
    rep->residual = residual_pass(g);
    if (g->first_residual < 0.0) g->first_residual = rep->residual > 0.0 ? rep->residual : 1.0;
    rep->normalized = rep->residual / g->first_residual;
    if (g->nhist == g->cap_hist) {
        g->cap_hist = g->cap_hist ? 2 * g->cap_hist : 256;
        g->history = realloc(g->history, g->cap_hist * sizeof(double));
    }
    g->history[g->nhist++] = rep->residual;
    rep->status = check_termination(g);
    if (rep->status == LZB_CONTINUE || rep->status == LZB_TIMEOUT) {
        update_pass(g, rep);
        prolong_corrections(g);
        finish_cycle_sync(g);
    }
    g->dof_updates_total += rep->dof_updates;
    rep->dof_updates_total = g->dof_updates_total;
    rep->pending_tasks = (uint64_t)(g->qtail - g->qhead) + (uint64_t)(g->htail - g->hhead) / 2;
    lzb_compression_stats cs;
    orc_stats(g, &cs);
    rep->max_n = cs.max_n;
    rep->avg_n = cs.avg_n;
    rep->max_samples = cs.max_sample_count;
    rep->factor_totals = cs.fine_factor_totals;
    rep->factor_mean = cs.fine_factor_mean;
    rep->levels = g->D + 1;
    uint64_t cells = 0, total = 0;
    for (int l = 0; l <= g->D; ++l) {
        uint64_t N = (uint64_t)g->L[l].N;
        cells += N * N;
        total += (N + 1) * (N + 1);
        if (l < 32) rep->enabled_mask |= 1u << l;
    }
    uint64_t Nf = (uint64_t)g->L[g->D].N;
    rep->cells = cells;
    rep->dofs_fine_interior = (Nf - 1) * (Nf - 1);
    rep->grid_points_total = total;
    rep->wall_seconds = 0.0;
    return 0;
}

/* solver.cpp:421-444 without AMR */
int orc_run(orc_grid* g, lzb_cycle_report* out, int cap, int* count) {
    int rc;
    if (g->d.mode == LZB_EAGER && (rc = orc_eager_setup(g))) return rc;
    int k = 0;
    for (;;) {
        lzb_cycle_report r;
        if ((rc = orc_step(g, &r))) return rc;
        if (k < cap) out[k] = r;
        ++k;
        if (r.status != LZB_CONTINUE) break;
    }
    *count = k;
    return 0;
}

int orc_pass(orc_grid* g, int which, double* value) {
    lzb_cycle_report dummy;
    memset(&dummy, 0, sizeof dummy);
    switch (which) {
        case 0: return walk(g, 0, 0, 0, visit_assembly, NULL);
        case 1: *value = residual_pass(g); return 0;
        case 2: update_pass(g, &dummy); return 0;
        case 3: prolong_corrections(g); return 0;
        case 4: finish_cycle_sync(g); return 0;
        case 5: return 0; /* begin_cycle of the stream: no per-cycle state on regular grids */
        case 6: return pool_begin_cycle(g);
        default: return set_err(LZB_ERR_INVALID, "unknown pass");
    }
}

int orc_cycle(orc_grid* g) { return (int)g->cycle; }

int orc_vertices(orc_grid* g, int level, int field, double* buf, int write) {
    if (level < 0 || level > g->D || field < 0 || field >= LZB_V_NFIELDS)
        return set_err(LZB_ERR_INVALID, "bad level/field");
    orc_level* L = &g->L[level];
    size_t bytes = (size_t)(L->N + 1) * (L->N + 1) * sizeof(double);
    if (write) memcpy(L->v[field], buf, bytes);
    else memcpy(buf, L->v[field], bytes);
    return 0;
}

int orc_cells(orc_grid* g, int level, double* ops, int32_t* p1, int32_t* n, int32_t* p3,
              uint32_t* epoch) {
    if (level < 0 || level > g->D) return set_err(LZB_ERR_INVALID, "bad level");
    orc_level* L = &g->L[level];
    for (int c = 0; c < L->N * L->N; ++c) {
        if (ops) element_or_baseline(g, level, c, ops + 16 * c);
        if (p1) p1[c] = L->p1[c];
        if (n) n[c] = L->p1[c] != LZB_P1_BOTTOM ? L->n[c] : 0;
        if (p3) p3[c] = L->p3[c];
        if (epoch) epoch[c] = L->p1[c] != LZB_P1_BOTTOM ? L->epoch[c] : 0;
    }
    return 0;
}

int orc_publish_element(orc_grid* g, int level, int cx, int cy, const double* m, int n,
                        int32_t p1) {
    orc_level* L = &g->L[level];
    int c = cy * L->N + cx;
    int rc = publish_element(g, level, c, m, n);
    if (rc) return rc;
    L->p1[c] = p1;
    return 0;
}

/* CellStream::publish_element + p1 store for every cell of a level, in cell
 * index order (a loop of the per-cell call; mats: N*N*16, n per cell). */
int orc_publish_level(orc_grid* g, int level, const double* mats, const int32_t* n, int32_t p1) {
    orc_level* L = &g->L[level];
    for (int64_t c = 0; c < (int64_t)L->N * L->N; ++c) {
        int rc = publish_element(g, level, (int)c, mats + 16 * c, n[c]);
        if (rc) return rc;
        L->p1[c] = p1;
    }
    return 0;
}

int orc_adaptive_step(orc_grid* g, int level, int cx, int cy) {
    if (level != g->D) return set_err(LZB_ERR_INVALID, "adaptive steps are for leaves");
    return adaptive_step(g, cy * g->L[level].N + cx);
}

/* ---------------------------------------------------------------- LZMG image */
typedef struct {
    uint8_t* out;
    int64_t cap, pos;
    int rc;
} img_ctx;

static void put(img_ctx* s, const void* p, int64_t n) {
    if (s->out && s->pos + n <= s->cap) memcpy(s->out + s->pos, p, n);
    s->pos += n;
}

/* stream.cpp:303-338 */
static int visit_save(orc_grid* g, int l, int c, void* vctx) {
    img_ctx* s = vctx;
    orc_level* L = &g->L[l];
    int32_t p1 = L->p1[c];
    int p3 = p1 != LZB_P1_BOTTOM ? L->p3[c] : 0;
    uint8_t hdr = orc_pack_header(p1, L->p2[c], p3);
    put(s, &hdr, 1);
    if (p1 == LZB_P1_BOTTOM || p3 == 0) return 0;
    double base[16];
    baseline(g, l, c % L->N, c / L->N, base);
    uint8_t buf[8];
    for (int i = 0; i < 16; ++i) {
        if ((s->rc = orc_encode_value(L->op[16 * c + i] - base[i], p3, buf))) return s->rc;
        put(s, buf, p3);
    }
    if (l < g->D) {
        const double* P = transfer_or_geometric(g, l, c);
        double ps[64];
        for (int i = 0; i < 64; ++i) ps[i] = P[i] - g->geo[i];
        for (int rep = 0; rep < 2; ++rep) /* P-hat, then the R-hat copy (stream.cpp:326-335) */
            for (int i = 0; i < 64; ++i) {
                if ((s->rc = orc_encode_value(ps[i], p3, buf))) return s->rc;
                put(s, buf, p3);
            }
    }
    return 0;
}

int64_t orc_stream_image(orc_grid* g, uint8_t* out, int64_t cap) {
    img_ctx s = {out, cap, 0, 0};
    uint32_t hdr[3] = {0x4c5a4d47u, 1u, 0};
    for (int l = 0; l <= g->D; ++l) hdr[2] += (uint32_t)(g->L[l].N * g->L[l].N);
    put(&s, hdr, 12);
    int rc = walk(g, 0, 0, 0, visit_save, &s);
    if (rc) return -rc;
    return s.pos;
}

typedef struct {
    const uint8_t* in;
    int64_t size, pos;
} load_ctx;

/* stream.cpp:340-394 */
static int visit_load(orc_grid* g, int l, int c, void* vctx) {
    load_ctx* s = vctx;
    orc_level* L = &g->L[l];
    if (s->pos >= s->size) return set_err(LZB_ERR_CORRUPT, "truncated stream file");
    uint8_t hb = s->in[s->pos++];
    int cls, p2, p3, rc;
    if ((rc = orc_unpack_header(hb, &cls, &p2, &p3))) return rc;
    L->p2[c] = (uint8_t)p2;
    if (cls == 0) {
        L->p1[c] = LZB_P1_BOTTOM;
        return 0;
    }
    int32_t p1 = cls == 2 ? LZB_P1_TOP : 1;
    double m[16], P[64];
    baseline(g, l, c % L->N, c / L->N, m);
    memcpy(P, g->geo, sizeof P);
    if (p3 != 0) {
        int64_t entries = l < g->D ? 144 : 16;
        if (s->pos + entries * p3 > s->size) return set_err(LZB_ERR_CORRUPT, "truncated record payload");
        const uint8_t* cur = s->in + s->pos;
        for (int i = 0; i < 16; ++i, cur += p3) m[i] += orc_decode_value(cur, p3);
        if (l < g->D)
            for (int i = 0; i < 64; ++i, cur += p3) P[i] += orc_decode_value(cur, p3);
        s->pos += entries * p3;
    }
    if (l < g->D) {
        int pub;
        (void)pub;
        publish_coarse(g, l, c, m, P, &rc);
        if (rc) return rc;
    } else if ((rc = publish_element(g, l, c, m, 1))) {
        return rc;
    }
    L->p1[c] = p1;
    L->p3[c] = p3;
    return 0;
}

int orc_stream_load(orc_grid* g, const uint8_t* in, int64_t size) {
    if (size < 12) return set_err(LZB_ERR_CORRUPT, "truncated stream file");
    uint32_t hdr[3];
    memcpy(hdr, in, 12);
    if (hdr[0] != 0x4c5a4d47u) return set_err(LZB_ERR_CORRUPT, "bad stream magic");
    if (hdr[1] != 1u) return set_err(LZB_ERR_CORRUPT, "unsupported stream version");
    uint32_t cells = 0;
    for (int l = 0; l <= g->D; ++l) cells += (uint32_t)(g->L[l].N * g->L[l].N);
    if (hdr[2] != cells) return set_err(LZB_ERR_CORRUPT, "stream cell count does not match the mesh");
    load_ctx s = {in, size, 12};
    return walk(g, 0, 0, 0, visit_load, &s);
}

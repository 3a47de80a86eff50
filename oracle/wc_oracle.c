/*
 * wc_oracle.c -- CPU ORACLE (test infrastructure only; see wc_oracle.h).
 *
 * Plain-C restatement of the reference render path.  Compiled with
 * -ffp-contract=off so that, like the numba kernels (which contain no FMA
 * instructions), every float64 operation rounds
 * individually and in source order.  The only tests, smoke() and
 * bench.py's cpu_baseline / --impl reference legs load it.
 */
#include "wc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define FINE_CELL 4.0
#define COARSE_CELL 16.0
#define ENTRY_EPS 4e-4   /* traversal.py:32 */
#define ENTRY_NUDGE 1e-7 /* blocktrace.py:31 */
#define AMBIENT 0.2      /* blocktrace.py:26 */

/* Reference invariant failures (AssertionError in the reference) end the
 * checker loudly with the reference's own message. */
#include <stdio.h>
#define ORC_ASSERT(cond, msg)                                      \
    do {                                                           \
        if (!(cond)) {                                             \
            fprintf(stderr, "oracle invariant failed: %s\n", msg); \
            abort();                                               \
        }                                                          \
    } while (0)

static void *xcalloc(size_t n, size_t sz) {
    void *p = calloc(n ? n : 1, sz ? sz : 1);
    if (!p) abort();
    return p;
}
static void *xmalloc(size_t n) {
    void *p = malloc(n ? n : 1);
    if (!p) abort();
    return p;
}

/* Python builtin max/min on floats as numba lowers them: the later argument
 * replaces the accumulator only when strictly greater (smaller). */
static inline double py_max(double a, double b) { return (b > a) ? b : a; }
static inline double py_min(double a, double b) { return (b < a) ? b : a; }
/* numpy maximum/minimum element rule (maxpd/minpd): a OP b ? a : b */
static inline double np_maximum(double a, double b) { return (a > b) ? a : b; }
static inline double np_minimum(double a, double b) { return (a < b) ? a : b; }

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ------------------------------------------------------------------ codec */

/* codec.py:143-168 _unpack_block */
static void unpack_block(const uint8_t *payload, int64_t block_id, int qbits,
                         int stride, float *out) {
    const int64_t base = block_id * (int64_t)stride;
    const uint16_t eu = (uint16_t)(payload[base] | (payload[base + 1] << 8));
    if (eu == 0x8000u) {
        for (int i = 0; i < 64; i++) out[i] = 0.0f;
        return;
    }
    const int64_t e = (int64_t)(int16_t)eu;
    const double s = (double)(((int64_t)1 << (qbits - 1)) - 1);
    const double scale = ldexp(1.0, (int)e); /* 2.0 ** e, exact */
    const int64_t mask = ((int64_t)1 << qbits) - 1;
    const int64_t sign_bit = (int64_t)1 << (qbits - 1);
    for (int i = 0; i < 64; i++) {
        const int64_t bitpos = 16 + (int64_t)i * qbits;
        const int64_t byte = base + (bitpos >> 3);
        const int shift = (int)(bitpos & 7);
        const int nbytes = (shift + qbits + 7) >> 3;
        int64_t acc = 0;
        for (int k = 0; k < nbytes; k++) acc |= (int64_t)payload[byte + k] << (8 * k);
        int64_t q = (acc >> shift) & mask;
        if (q & sign_bit) q -= (int64_t)1 << qbits;
        out[i] = (float)((double)q / s * scale);
    }
}

/* codec.py:171-174 _unpack_many */
void orc_decode_blocks(const uint8_t *payload, int qbits, int stride,
                       const int64_t *ids, int64_t n, float *out) {
    for (int64_t j = 0; j < n; j++) unpack_block(payload, ids[j], qbits, stride, out + 64 * j);
}

/* codec.py:100-105 _block_exponents + :183-185 quantisation + :120-140
 * _pack_blocks for one gathered block (blk: 64 edge-replicated values,
 * x fastest).  Returns the exponent. */
static int32_t pack_block(const float *blk, int qbits, uint8_t *rec) {
    const double s = (double)(((int64_t)1 << (qbits - 1)) - 1);
    const int64_t mask = ((int64_t)1 << qbits) - 1;
    float m = 0.0f;
    for (int i = 0; i < 64; i++) {
        const float a = fabsf(blk[i]);
        if (a > m) m = a;
    }
    int32_t e;
    if ((double)m == 0.0) {
        e = -32768;
    } else {
        int ex;
        const double mant = frexp((double)m, &ex);
        e = ex - (mant == 0.5);
    }
    const uint16_t eu = (uint16_t)(int16_t)e;
    rec[0] = (uint8_t)(eu & 0xFF);
    rec[1] = (uint8_t)((eu >> 8) & 0xFF);
    if (e == -32768) return e;
    const double scale = ldexp(1.0, -e);
    for (int i = 0; i < 64; i++) {
        const double qd = rint((double)blk[i] * scale * s); /* np.rint: half-even */
        const int64_t q = (int64_t)(int32_t)qd & mask;
        const int64_t bitpos = 16 + (int64_t)i * qbits;
        const int shift = (int)(bitpos & 7);
        const int64_t accv = q << shift;
        const int nbytes = (shift + qbits + 7) >> 3;
        for (int k = 0; k < nbytes; k++) rec[(bitpos >> 3) + k] |= (uint8_t)((accv >> (8 * k)) & 0xFF);
    }
    return e;
}

/* codec.py:81-97 _gather_blocks for block (bx,by,bz) of a field given by
 * a sampler; fills blk and the valid-voxel (min, max). */
typedef float (*orc_sampler)(const void *ctx, int x, int y, int z);

static void gather_block(orc_sampler f, const void *ctx, int nx, int ny, int nz, int bx, int by, int bz, float *blk,
                         float *mn_out, float *mx_out) {
    float mn = INFINITY, mx = -INFINITY;
    for (int k = 0; k < 4; k++)
        for (int j = 0; j < 4; j++)
            for (int i = 0; i < 4; i++) {
                int x = 4 * bx + i, y = 4 * by + j, z = 4 * bz + k;
                const int valid = x < nx && y < ny && z < nz;
                if (x >= nx) x = nx - 1; /* np.pad mode="edge" */
                if (y >= ny) y = ny - 1;
                if (z >= nz) z = nz - 1;
                const float v = f(ctx, x, y, z);
                blk[i + 4 * j + 16 * k] = v;
                if (valid) {
                    if (v < mn) mn = v;
                    if (v > mx) mx = v;
                }
            }
    *mn_out = mn;
    *mx_out = mx;
}

typedef struct {
    const float *v;
    int nx, ny;
} dense_ctx;

static float dense_sample(const void *ctx, int x, int y, int z) {
    const dense_ctx *c = (const dense_ctx *)ctx;
    return c->v[x + (int64_t)c->nx * (y + (int64_t)c->ny * z)];
}

typedef struct {
    int K, nx, ny, nz;
    const float *amp, *fx, *fy, *fz;
} sep_ctx;

/* separable field, float32 in the same order as volume.SeparableField */
static float sep_sample(const void *ctx, int x, int y, int z) {
    const sep_ctx *c = (const sep_ctx *)ctx;
    float v = 0.0f;
    for (int k = 0; k < c->K; k++)
        v = v + ((c->amp[k] * c->fz[(int64_t)k * c->nz + z]) * c->fy[(int64_t)k * c->ny + y]) * c->fx[(int64_t)k * c->nx + x];
    return v;
}

static void compress_layers(orc_sampler f, const void *ctx, int nx, int ny, int nz, int qbits, int bz0, int bz1,
                            uint8_t *payload, float *ranges, int32_t *exponents) {
    const int bdx = (nx + 3) / 4, bdy = (ny + 3) / 4;
    const int stride = ((16 + 64 * qbits + 31) / 32) * 4;
    float blk[64];
    for (int bz = bz0; bz < bz1; bz++)
        for (int by = 0; by < bdy; by++)
            for (int bx = 0; bx < bdx; bx++) {
                const int64_t b = bx + (int64_t)bdx * (by + (int64_t)bdy * bz);
                gather_block(f, ctx, nx, ny, nz, bx, by, bz, blk, &ranges[2 * b], &ranges[2 * b + 1]);
                const int32_t e = pack_block(blk, qbits, payload + b * stride);
                if (exponents) exponents[b] = e;
            }
}

/* codec.py:177-198 compress_volume (payload zeroed by the caller) */
void orc_compress(const float *values, int nx, int ny, int nz, int qbits,
                  uint8_t *payload, float *ranges, int32_t *exponents) {
    dense_ctx c = {values, nx, ny};
    compress_layers(dense_sample, &c, nx, ny, nz, qbits, 0, (nz + 3) / 4, payload, ranges, exponents);
}

/* Same for a separable synthetic field, block layers [bz0, bz1) only, so
 * callers can split an 8.05B-voxel volume across host threads. */
void orc_compress_separable(int K, const float *amp, const float *fx, const float *fy, const float *fz, int nx,
                            int ny, int nz, int qbits, int bz0, int bz1, uint8_t *payload, float *ranges) {
    sep_ctx c = {K, nx, ny, nz, amp, fx, fy, fz};
    compress_layers(sep_sample, &c, nx, ny, nz, qbits, bz0, bz1, payload, ranges, NULL);
}

/* codec.py:113-117 _bounds_from_exponents over codec.py:220-223 */
void orc_error_bounds(const uint8_t *payload, int64_t n_blocks, int qbits,
                      int stride, double *bounds) {
    const double s = (double)(((int64_t)1 << (qbits - 1)) - 1);
    for (int64_t b = 0; b < n_blocks; b++) {
        const uint16_t eu = (uint16_t)(payload[b * stride] | (payload[b * stride + 1] << 8));
        if (eu == 0x8000u)
            bounds[b] = 0.0;
        else
            bounds[b] = ldexp(1.0, (int)(int16_t)eu) / (2.0 * s);
    }
}

/* ------------------------------------------------------------------ grids */

/* grids.py:48-57 _octant_union: reduce over the 2x2x2 window anchored at
 * each cell, window cells outside the grid read `fill`. */
static void octant_union(const double *a, int dx, int dy, int dz, int is_max,
                         double *out) {
    const double fill = is_max ? -INFINITY : INFINITY;
    for (int z = 0; z < dz; z++)
        for (int y = 0; y < dy; y++)
            for (int x = 0; x < dx; x++) {
                double acc = fill;
                for (int oz = 0; oz < 2; oz++)
                    for (int oy = 0; oy < 2; oy++)
                        for (int ox = 0; ox < 2; ox++) {
                            const int X = x + ox, Y = y + oy, Z = z + oz;
                            double v = fill;
                            if (X < dx && Y < dy && Z < dz) v = a[X + (int64_t)dx * (Y + (int64_t)dy * Z)];
                            acc = is_max ? np_maximum(acc, v) : np_minimum(acc, v);
                        }
                out[x + (int64_t)dx * (y + (int64_t)dy * z)] = acc;
            }
}

/* grids.py:71-94 build_grids */
void orc_build_grids(const float *ranges, const double *bounds, int bdx,
                     int bdy, int bdz, double *fine_min, double *fine_max,
                     double *coarse_min, double *coarse_max) {
    const int64_t nb = (int64_t)bdx * bdy * bdz;
    double *wmin = xmalloc(sizeof(double) * nb), *wmax = xmalloc(sizeof(double) * nb);
    for (int64_t b = 0; b < nb; b++) {
        wmin[b] = (double)ranges[2 * b] - bounds[b];
        wmax[b] = (double)ranges[2 * b + 1] + bounds[b];
    }
    octant_union(wmin, bdx, bdy, bdz, 0, fine_min);
    octant_union(wmax, bdx, bdy, bdz, 1, fine_max);
    const int cdx = (bdx + 3) / 4, cdy = (bdy + 3) / 4, cdz = (bdz + 3) / 4;
    const int64_t nc = (int64_t)cdx * cdy * cdz;
    double *gmin = xmalloc(sizeof(double) * nc), *gmax = xmalloc(sizeof(double) * nc);
    for (int cz = 0; cz < cdz; cz++) /* grids.py:60-68 _group4 */
        for (int cy = 0; cy < cdy; cy++)
            for (int cx = 0; cx < cdx; cx++) {
                double lo = INFINITY, hi = -INFINITY;
                for (int k = 0; k < 4; k++)
                    for (int j = 0; j < 4; j++)
                        for (int i = 0; i < 4; i++) {
                            const int x = 4 * cx + i, y = 4 * cy + j, z = 4 * cz + k;
                            if (x >= bdx || y >= bdy || z >= bdz) continue;
                            const int64_t b = x + (int64_t)bdx * (y + (int64_t)bdy * z);
                            lo = np_minimum(lo, wmin[b]);
                            hi = np_maximum(hi, wmax[b]);
                        }
                gmin[cx + (int64_t)cdx * (cy + (int64_t)cdy * cz)] = lo;
                gmax[cx + (int64_t)cdx * (cy + (int64_t)cdy * cz)] = hi;
            }
    octant_union(gmin, cdx, cdy, cdz, 0, coarse_min);
    octant_union(gmax, cdx, cdy, cdz, 1, coarse_max);
    free(wmin);
    free(wmax);
    free(gmin);
    free(gmax);
}

/* ------------------------------------------------------------------- rays */

/* traversal.py:105-120 RaySoA.from_camera (direction part) */
void orc_camera_rays(const orc_camera *cam, const int64_t *pixel_ids,
                     int64_t n, double *origin, double *direction) {
    const int64_t w = cam->img_w, h = cam->img_h;
    const double aspect = (double)w / (double)h;
    for (int64_t r = 0; r < n; r++) {
        const int64_t p = pixel_ids ? pixel_ids[r] : r;
        const int64_t px = p % w, py = p / w;
        const double xs = ((2.0 * ((double)px + 0.5)) / (double)w - 1.0) * cam->tan_half * aspect;
        const double ys = (1.0 - (2.0 * ((double)py + 0.5)) / (double)h) * cam->tan_half;
        double d[3];
        for (int a = 0; a < 3; a++) d[a] = (cam->look[a] + xs * cam->right[a]) + ys * cam->up[a];
        const double nrm = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
        for (int a = 0; a < 3; a++) {
            direction[3 * r + a] = d[a] / nrm;
            origin[3 * r + a] = cam->eye[a];
        }
    }
}

/* traversal.py:181-187 _tmax_init for one axis */
static inline double tmax_init(double o, double d, int64_t cell, double size) {
    if (d == 0.0) return INFINITY;
    const double lo = (double)cell * size;
    const double target = d > 0 ? lo + size : lo;
    return (target - o) / d;
}

/* traversal.py:122-170 RaySoA.from_rays: slab clip + iterator seeds */
static void from_rays(const double *origin, const double *direction, int64_t n,
                      int nx, int ny, int nz, double *t_enter, double *t_exit,
                      uint8_t *status, uint8_t *exited, uint32_t *coarse_cell,
                      uint32_t *fine_cell, double *coarse_tmax, double *fine_tmax) {
    const double hi[3] = {(double)nx - 1.0, (double)ny - 1.0, (double)nz - 1.0};
    const int64_t fd[3] = {(nx + 3) / 4, (ny + 3) / 4, (nz + 3) / 4};
    const int64_t cd[3] = {(fd[0] + 3) / 4, (fd[1] + 3) / 4, (fd[2] + 3) / 4};
    for (int64_t r = 0; r < n; r++) {
        const double *o = origin + 3 * r, *d = direction + 3 * r;
        double near[3], far[3];
        for (int a = 0; a < 3; a++) {
            if (d[a] != 0.0) {
                const double t1 = (0.0 - o[a]) / d[a];
                const double t2 = (hi[a] - o[a]) / d[a];
                near[a] = np_minimum(t1, t2);
                far[a] = np_maximum(t1, t2);
            } else if (o[a] < 0.0 || o[a] > hi[a]) {
                near[a] = INFINITY;
                far[a] = -INFINITY;
            } else {
                near[a] = -INFINITY;
                far[a] = INFINITY;
            }
        }
        const double t_near = np_maximum(np_maximum(near[0], near[1]), near[2]);
        const double t_far = np_minimum(np_minimum(far[0], far[1]), far[2]);
        const int hit = (t_near <= t_far) && (t_far >= 0.0);
        t_enter[r] = np_maximum(t_near, 0.0);
        t_exit[r] = t_far;
        status[r] = hit ? 0 : 2;
        exited[r] = 0;
        coarse_cell[r] = ORC_UINT_MAX;
        fine_cell[r] = ORC_UINT_MAX;
        for (int a = 0; a < 3; a++) coarse_tmax[3 * r + a] = fine_tmax[3 * r + a] = 0.0;
        if (!hit) continue;
        int64_t fc[3], cc[3];
        for (int a = 0; a < 3; a++) {
            const double p0 = o[a] + d[a] * (t_enter[r] + ENTRY_EPS);
            int64_t c = (int64_t)floor(p0 / FINE_CELL);
            if (c < 0) c = 0;
            if (c > fd[a] - 1) c = fd[a] - 1;
            fc[a] = c;
            cc[a] = c / 4;
        }
        fine_cell[r] = (uint32_t)(fc[0] + fd[0] * (fc[1] + fd[1] * fc[2]));
        coarse_cell[r] = (uint32_t)(cc[0] + cd[0] * (cc[1] + cd[1] * cc[2]));
        for (int a = 0; a < 3; a++) {
            fine_tmax[3 * r + a] = tmax_init(o[a], d[a], fc[a], FINE_CELL);
            coarse_tmax[3 * r + a] = tmax_init(o[a], d[a], cc[a], COARSE_CELL);
        }
    }
}

/* ------------------------------------------------------------ intersection */

/* blocktrace.py:126-158 _cell_overlap; returns 0 when rejected early */
static inline void cell_overlap(double ox, double oy, double oz, double dx,
                                double dy, double dz, double cx, double cy,
                                double cz, double *t0o, double *t1o) {
    double t0 = -INFINITY, t1 = INFINITY, ta, tb;
    const double o[3] = {ox, oy, oz}, d[3] = {dx, dy, dz}, c[3] = {cx, cy, cz};
    for (int a = 0; a < 3; a++) {
        if (d[a] != 0.0) {
            ta = (c[a] - o[a]) / d[a];
            tb = (c[a] + 1.0 - o[a]) / d[a];
            if (ta > tb) {
                const double t = ta;
                ta = tb;
                tb = t;
            }
            t0 = py_max(t0, ta);
            t1 = py_min(t1, tb);
        } else if (o[a] < c[a] || o[a] > c[a] + 1.0) {
            *t0o = INFINITY;
            *t1o = -INFINITY;
            return;
        }
    }
    *t0o = t0;
    *t1o = t1;
}

/* blocktrace.py:161-190 _cubic_coeffs */
static inline void cubic_coeffs(const float *c, double ox, double oy, double oz,
                                double dx, double dy, double dz, double cx,
                                double cy, double cz, double *A, double *B,
                                double *C, double *D) {
    const double ax1 = ox - cx, ay1 = oy - cy, az1 = oz - cz;
    const double ax0 = 1.0 - ax1, ay0 = 1.0 - ay1, az0 = 1.0 - az1;
    double a = 0.0, b = 0.0, cc = 0.0, d = 0.0;
    for (int idx = 0; idx < 8; idx++) {
        const int i = idx & 1, j = (idx >> 1) & 1, k = (idx >> 2) & 1;
        const double axa = i ? ax1 : ax0, axb = i ? dx : -dx;
        const double aya = j ? ay1 : ay0, ayb = j ? dy : -dy;
        const double aza = k ? az1 : az0, azb = k ? dz : -dz;
        const double w = (double)c[idx];
        a += w * ((axb * ayb) * azb);
        b += w * (((axa * ayb) * azb + (axb * aya) * azb) + (axb * ayb) * aza);
        cc += w * (((axa * aya) * azb + (axa * ayb) * aza) + (axb * aya) * aza);
        d += w * ((axa * aya) * aza);
    }
    *A = a;
    *B = b;
    *C = cc;
    *D = d;
}

/* blocktrace.py:193-195 */
static inline double poly_eval(double A, double B, double C, double D, double t) {
    return ((A * t + B) * t + C) * t + D;
}

/* blocktrace.py:198-233 _refine_root (Illinois regula falsi + bisection) */
static double refine_root(double A, double B, double C, double D, double lo,
                          double hi, double g_lo, double g_hi) {
    const double tol = 1e-9 * (hi - lo);
    int side = 0;
    double tm = 0.5 * (lo + hi);
    for (int it = 0; it < 64; it++) {
        const double denom = g_lo - g_hi;
        if (denom != 0.0)
            tm = lo + (hi - lo) * (g_lo / denom);
        else
            tm = 0.5 * (lo + hi);
        if (tm <= lo || tm >= hi) tm = 0.5 * (lo + hi);
        const double gm = poly_eval(A, B, C, D, tm);
        if (gm == 0.0 || hi - lo < tol) return tm;
        if ((gm < 0.0) == (g_lo < 0.0)) {
            lo = tm;
            g_lo = gm;
            if (side == -1) g_hi *= 0.5;
            side = -1;
        } else {
            hi = tm;
            g_hi = gm;
            if (side == 1) g_lo *= 0.5;
            side = 1;
        }
    }
    return tm;
}

/* blocktrace.py:236-280 _intersect_cubic */
static double intersect_cubic(const float *c, double ox, double oy, double oz,
                              double dx, double dy, double dz, double cx,
                              double cy, double cz, double t0, double t1,
                              double iso) {
    double A, B, C, D;
    cubic_coeffs(c, ox, oy, oz, dx, dy, dz, cx, cy, cz, &A, &B, &C, &D);
    D -= iso;
    double bounds[4];
    int nb = 0;
    bounds[nb++] = t0;
    const double qa = 3.0 * A, qb = 2.0 * B;
    if (qa != 0.0) {
        const double disc = qb * qb - 4.0 * qa * C;
        if (disc > 0.0) {
            const double sq = sqrt(disc);
            const double q = qb >= 0.0 ? -0.5 * (qb + sq) : -0.5 * (qb - sq);
            double r1 = q / qa;
            double r2 = q != 0.0 ? C / q : r1;
            if (r1 > r2) {
                const double t = r1;
                r1 = r2;
                r2 = t;
            }
            if (t0 < r1 && r1 < t1) bounds[nb++] = r1;
            if (t0 < r2 && r2 < t1 && r2 != r1) bounds[nb++] = r2;
        }
    } else if (qb != 0.0) {
        const double r1 = -C / qb;
        if (t0 < r1 && r1 < t1) bounds[nb++] = r1;
    }
    bounds[nb++] = t1;
    double g_prev = poly_eval(A, B, C, D, bounds[0]);
    if (g_prev == 0.0) return bounds[0];
    for (int i = 1; i < nb; i++) {
        const double g_here = poly_eval(A, B, C, D, bounds[i]);
        if (g_here == 0.0) return bounds[i];
        if ((g_prev < 0.0) != (g_here < 0.0))
            return refine_root(A, B, C, D, bounds[i - 1], bounds[i], g_prev, g_here);
        g_prev = g_here;
    }
    return INFINITY;
}

double orc_intersect_cell(const float *corners, const double *o,
                          const double *d, const double *cell, double t0,
                          double t1, double iso) {
    return intersect_cubic(corners, o[0], o[1], o[2], d[0], d[1], d[2], cell[0],
                           cell[1], cell[2], t0, t1, iso);
}

/* blocktrace.py:283-303 _grad_at: corner differences are float32 ops */
static inline void grad_at(const float *c, double ux, double uy, double uz,
                           double *gx, double *gy, double *gz) {
    *gx = (((double)(c[1] - c[0]) * (1.0 - uy) * (1.0 - uz) + (double)(c[3] - c[2]) * uy * (1.0 - uz)) +
           (double)(c[5] - c[4]) * (1.0 - uy) * uz) +
          (double)(c[7] - c[6]) * uy * uz;
    *gy = (((double)(c[2] - c[0]) * (1.0 - ux) * (1.0 - uz) + (double)(c[3] - c[1]) * ux * (1.0 - uz)) +
           (double)(c[6] - c[4]) * (1.0 - ux) * uz) +
          (double)(c[7] - c[5]) * ux * uz;
    *gz = (((double)(c[4] - c[0]) * (1.0 - ux) * (1.0 - uy) + (double)(c[5] - c[1]) * ux * (1.0 - uy)) +
           (double)(c[6] - c[2]) * (1.0 - ux) * uy) +
          (double)(c[7] - c[3]) * ux * uy;
}

/* blocktrace.py:306-314 _shade */
static inline void shade(double gx, double gy, double gz, double dx, double dy,
                         double dz, double br, double bg, double bb,
                         double *r, double *g, double *b) {
    const double gl = sqrt((gx * gx + gy * gy) + gz * gz);
    double inten;
    if (gl == 0.0) {
        inten = AMBIENT;
    } else {
        const double cos_t = fabs((gx * dx + gy * dy) + gz * dz) / gl;
        inten = cos_t > AMBIENT ? cos_t : AMBIENT;
    }
    *r = br * inten;
    *g = bg * inten;
    *b = bb * inten;
}

/* blocktrace.py:317-449 _trace_region.  field is indexed
 * [z - foz][y - foy][x - fox] with row stride fsy, slice stride fsz. */
static double trace_region(const float *field, int64_t fsy, int64_t fsz,
                           int64_t fox, int64_t foy, int64_t foz, int64_t lo_x,
                           int64_t lo_y, int64_t lo_z, int64_t n_x, int64_t n_y,
                           int64_t n_z, double ox, double oy, double oz,
                           double dx, double dy, double dz, double ray_t_enter,
                           double iso, double br, double bg, double bb,
                           double *rgb) {
    if (n_x <= 0 || n_y <= 0 || n_z <= 0) return INFINITY;
    double t0 = ray_t_enter, t1 = INFINITY, ta, tb;
    const double o[3] = {ox, oy, oz}, d[3] = {dx, dy, dz};
    const int64_t lo[3] = {lo_x, lo_y, lo_z}, nn[3] = {n_x, n_y, n_z};
    for (int a = 0; a < 3; a++) {
        if (d[a] != 0.0) {
            ta = ((double)lo[a] - o[a]) / d[a];
            tb = ((double)(lo[a] + nn[a]) - o[a]) / d[a];
            if (ta > tb) {
                const double t = ta;
                ta = tb;
                tb = t;
            }
            t0 = py_max(t0, ta);
            t1 = py_min(t1, tb);
        } else if (o[a] < (double)lo[a] || o[a] > (double)(lo[a] + nn[a])) {
            return INFINITY;
        }
    }
    if (t0 > t1) return INFINITY;
    const double ts = t0 + ENTRY_NUDGE * py_max(1.0, t1 - t0);
    int64_t cx = (int64_t)floor(ox + dx * ts);
    int64_t cy = (int64_t)floor(oy + dy * ts);
    int64_t cz = (int64_t)floor(oz + dz * ts);
    cx = cx < lo_x ? lo_x : cx;
    cx = cx > lo_x + n_x - 1 ? lo_x + n_x - 1 : cx;
    cy = cy < lo_y ? lo_y : cy;
    cy = cy > lo_y + n_y - 1 ? lo_y + n_y - 1 : cy;
    cz = cz < lo_z ? lo_z : cz;
    cz = cz > lo_z + n_z - 1 ? lo_z + n_z - 1 : cz;
    const int sx = dx > 0.0 ? 1 : (dx < 0.0 ? -1 : 0);
    const int sy = dy > 0.0 ? 1 : (dy < 0.0 ? -1 : 0);
    const int sz = dz > 0.0 ? 1 : (dz < 0.0 ? -1 : 0);
    const double del_x = dx != 0.0 ? 1.0 / fabs(dx) : INFINITY;
    const double del_y = dy != 0.0 ? 1.0 / fabs(dy) : INFINITY;
    const double del_z = dz != 0.0 ? 1.0 / fabs(dz) : INFINITY;
    double tmx = dx > 0.0 ? ((double)(cx + 1) - ox) / dx : (dx < 0.0 ? ((double)cx - ox) / dx : INFINITY);
    double tmy = dy > 0.0 ? ((double)(cy + 1) - oy) / dy : (dy < 0.0 ? ((double)cy - oy) / dy : INFINITY);
    double tmz = dz > 0.0 ? ((double)(cz + 1) - oz) / dz : (dz < 0.0 ? ((double)cz - oz) / dz : INFINITY);
    float corners[8];
    for (;;) {
        const float *p = field + (cz - foz) * fsz + (cy - foy) * fsy + (cx - fox);
        corners[0] = p[0];
        corners[1] = p[1];
        corners[2] = p[fsy];
        corners[3] = p[fsy + 1];
        corners[4] = p[fsz];
        corners[5] = p[fsz + 1];
        corners[6] = p[fsz + fsy];
        corners[7] = p[fsz + fsy + 1];
        float cmin = corners[0], cmax = corners[0];
        for (int q = 1; q < 8; q++) {
            if (corners[q] < cmin) cmin = corners[q];
            if (corners[q] > cmax) cmax = corners[q];
        }
        if ((double)cmin <= iso && iso <= (double)cmax) {
            double ct0, ct1;
            cell_overlap(ox, oy, oz, dx, dy, dz, (double)cx, (double)cy, (double)cz, &ct0, &ct1);
            if (ct0 < ray_t_enter) ct0 = ray_t_enter;
            if (ct0 <= ct1) {
                const double th = intersect_cubic(corners, ox, oy, oz, dx, dy, dz, (double)cx,
                                                  (double)cy, (double)cz, ct0, ct1, iso);
                if (th != INFINITY) {
                    double ux = ox + dx * th - (double)cx;
                    double uy = oy + dy * th - (double)cy;
                    double uz = oz + dz * th - (double)cz;
                    ux = py_min(py_max(ux, 0.0), 1.0);
                    uy = py_min(py_max(uy, 0.0), 1.0);
                    uz = py_min(py_max(uz, 0.0), 1.0);
                    double gx, gy, gz;
                    grad_at(corners, ux, uy, uz, &gx, &gy, &gz);
                    shade(gx, gy, gz, dx, dy, dz, br, bg, bb, &rgb[0], &rgb[1], &rgb[2]);
                    return th;
                }
            }
        }
        if (tmx <= tmy && tmx <= tmz) {
            cx += sx;
            tmx += del_x;
            if (cx < lo_x || cx >= lo_x + n_x) return INFINITY;
        } else if (tmy <= tmz) {
            cy += sy;
            tmy += del_y;
            if (cy < lo_y || cy >= lo_y + n_y) return INFINITY;
        } else {
            cz += sz;
            tmz += del_z;
            if (cz < lo_z || cz >= lo_z + n_z) return INFINITY;
        }
    }
}

/* engine.py:152-158 _rgb_u8 (the engine passes float32 rgbz values, the
 * brute-force oracle passes the float64 shade result: oracle.py:88-90) */
static inline uint8_t rgb_u8_d(double v) {
    if (v < 0.0)
        v = 0.0;
    else if (v > 1.0)
        v = 1.0;
    return (uint8_t)(v * 255.0 + 0.5);
}
static inline uint8_t rgb_u8(float vf) {
    double v = (double)vf;
    if (v < 0.0)
        v = 0.0;
    else if (v > 1.0)
        v = 1.0;
    return (uint8_t)(v * 255.0 + 0.5);
}

/* oracle.py:42-122 brute-force reference render (status per from_rays) */
void orc_reference_render(const float *values, int nx, int ny, int nz,
                          const double *origin, const double *direction,
                          int64_t n, double iso, double base_r, double base_g,
                          double base_b, uint8_t *rgba, float *depth) {
    double *te = xmalloc(sizeof(double) * n), *tx = xmalloc(sizeof(double) * n);
    uint8_t *st = xmalloc(n), *ex = xmalloc(n);
    uint32_t *cc = xmalloc(4 * n), *fc = xmalloc(4 * n);
    double *ct = xmalloc(sizeof(double) * 3 * n), *ft = xmalloc(sizeof(double) * 3 * n);
    from_rays(origin, direction, n, nx, ny, nz, te, tx, st, ex, cc, fc, ct, ft);
    for (int64_t r = 0; r < n; r++) {
        rgba[4 * r] = rgba[4 * r + 1] = rgba[4 * r + 2] = 0;
        rgba[4 * r + 3] = 255;
        depth[r] = INFINITY;
        if (st[r] != 0) continue;
        const double *o = origin + 3 * r, *d = direction + 3 * r;
        double rgb[3];
        const double t = trace_region(values, nx, (int64_t)nx * ny, 0, 0, 0, 0, 0, 0, nx - 1, ny - 1,
                                      nz - 1, o[0], o[1], o[2], d[0], d[1], d[2], te[r], iso, base_r,
                                      base_g, base_b, rgb);
        if (t != INFINITY) {
            depth[r] = (float)t;
            rgba[4 * r] = rgb_u8_d(rgb[0]);
            rgba[4 * r + 1] = rgb_u8_d(rgb[1]);
            rgba[4 * r + 2] = rgb_u8_d(rgb[2]);
            rgba[4 * r + 3] = 255;
        }
    }
    free(te); free(tx); free(st); free(ex); free(cc); free(fc); free(ct); free(ft);
}

/* -------------------------------------------------------------- LRU cache */

/* cache.py:27-111 BlockCache */
struct orc_cache {
    int64_t cap;
    int64_t n_blocks;
    int64_t current_pass;
    float *slot_values;     /* cap x 64 */
    int64_t *block_of_slot; /* cap */
    int64_t *last_used;     /* cap */
    int32_t *slot_of_block; /* n_blocks, -1 = absent */
    int64_t *scratch_a, *scratch_b;
    int64_t scratch_cap;
};

orc_cache *orc_cache_create(int64_t capacity, int64_t n_blocks) {
    orc_cache *c = xcalloc(1, sizeof(orc_cache));
    c->cap = capacity < 1 ? 1 : capacity;
    c->n_blocks = n_blocks;
    c->slot_values = xcalloc((size_t)c->cap * 64, sizeof(float));
    c->block_of_slot = xmalloc(sizeof(int64_t) * c->cap);
    for (int64_t i = 0; i < c->cap; i++) c->block_of_slot[i] = -1;
    c->last_used = xcalloc(c->cap, sizeof(int64_t));
    c->slot_of_block = xmalloc(sizeof(int32_t) * (n_blocks ? n_blocks : 1));
    for (int64_t i = 0; i < n_blocks; i++) c->slot_of_block[i] = -1;
    return c;
}

void orc_cache_destroy(orc_cache *c) {
    if (!c) return;
    free(c->slot_values);
    free(c->block_of_slot);
    free(c->last_used);
    free(c->slot_of_block);
    free(c->scratch_a);
    free(c->scratch_b);
    free(c);
}

/* cache.py:42-53 _grow */
static void cache_grow(orc_cache *c, int64_t new_cap) {
    c->slot_values = realloc(c->slot_values, sizeof(float) * 64 * (size_t)new_cap);
    c->block_of_slot = realloc(c->block_of_slot, sizeof(int64_t) * new_cap);
    c->last_used = realloc(c->last_used, sizeof(int64_t) * new_cap);
    if (!c->slot_values || !c->block_of_slot || !c->last_used) abort();
    memset(c->slot_values + 64 * c->cap, 0, sizeof(float) * 64 * (size_t)(new_cap - c->cap));
    for (int64_t i = c->cap; i < new_cap; i++) {
        c->block_of_slot[i] = -1;
        c->last_used[i] = 0;
    }
    c->cap = new_cap;
}

static int cmp_u64(const void *a, const void *b) {
    const uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return x < y ? -1 : (x > y);
}

/* cache.py:66-111 ensure_resident; active_ids ascending */
void orc_cache_update(orc_cache *c, const uint8_t *payload, int qbits,
                      int stride, const int64_t *active_ids, int64_t n_active,
                      int64_t *stats) {
    c->current_pass += 1;
    const int64_t needed = n_active;
    if (needed > c->cap) cache_grow(c, (3 * needed + 1) / 2); /* ceil(1.5*needed) */
    if (c->scratch_cap < c->cap || c->scratch_cap < n_active) {
        c->scratch_cap = c->cap > n_active ? c->cap : n_active;
        free(c->scratch_a);
        free(c->scratch_b);
        c->scratch_a = xmalloc(sizeof(int64_t) * c->scratch_cap);
        c->scratch_b = xmalloc(sizeof(int64_t) * c->scratch_cap);
    }
    int64_t *miss = c->scratch_a, n_miss = 0;
    for (int64_t i = 0; i < n_active; i++) {
        const int64_t b = active_ids[i];
        const int32_t s = c->slot_of_block[b];
        if (s >= 0)
            c->last_used[s] = c->current_pass;
        else
            miss[n_miss++] = b;
    }
    int64_t evicted = 0;
    if (n_miss) {
        int64_t *free_slots = c->scratch_b, n_free = 0;
        for (int64_t s = 0; s < c->cap && n_free < n_miss; s++)
            if (c->block_of_slot[s] < 0) free_slots[n_free++] = s;
        int64_t n_evict = n_miss - n_free;
        if (n_evict > 0) {
            /* candidates sorted by (last_used, block_id): cache.py:84-91 */
            uint64_t *keys = xmalloc(sizeof(uint64_t) * c->cap);
            int64_t nc = 0;
            for (int64_t s = 0; s < c->cap; s++)
                if (c->block_of_slot[s] >= 0 && c->last_used[s] < c->current_pass)
                    keys[nc++] = ((uint64_t)c->last_used[s] << 32) | (uint64_t)c->block_of_slot[s];
            qsort(keys, nc, sizeof(uint64_t), cmp_u64);
            for (int64_t v = 0; v < n_evict; v++) {
                const int64_t b = (int64_t)(keys[v] & 0xFFFFFFFFull);
                const int64_t s = c->slot_of_block[b];
                c->slot_of_block[b] = -1;
                c->block_of_slot[s] = -1;
                free_slots[n_free++] = s;
            }
            evicted = n_evict;
            free(keys);
        }
        for (int64_t i = 0; i < n_miss; i++) {
            const int64_t s = free_slots[i], b = miss[i];
            unpack_block(payload, b, qbits, stride, c->slot_values + 64 * s);
            c->block_of_slot[s] = b;
            c->last_used[s] = c->current_pass;
            c->slot_of_block[b] = (int32_t)s;
        }
    }
    stats[0] = n_miss;
    stats[1] = evicted;
    stats[2] = c->cap;
}

int64_t orc_cache_lookup(const orc_cache *c, int64_t block_id) { return c->slot_of_block[block_id]; }
int64_t orc_cache_capacity_of(const orc_cache *c) { return c->cap; }
void orc_cache_state(const orc_cache *c, int64_t *block_of_slot,
                     int64_t *last_used, float *slot_values) {
    if (block_of_slot) memcpy(block_of_slot, c->block_of_slot, sizeof(int64_t) * c->cap);
    if (last_used) memcpy(last_used, c->last_used, sizeof(int64_t) * c->cap);
    if (slot_values) memcpy(slot_values, c->slot_values, sizeof(float) * 64 * (size_t)c->cap);
}

/* ---------------------------------------------------------------- session */

struct orc_session {
    const uint8_t *payload;
    const double *fmin, *fmax, *cmin, *cmax;
    int nx, ny, nz, qbits, stride;
    int64_t bdx, bdy, bdz, cdx, cdy, cdz, n_blocks;
    int64_t n, w, h;
    const double *origin, *direction;
    double *t_enter, *t_exit, *coarse_tmax, *fine_tmax;
    uint8_t *status, *exited;
    uint32_t *coarse_cell, *fine_cell, *block_slots, *ray_slots, *active_offsets;
    double iso, base[3];
    int speculation, max_spec, corrupt;
    orc_cache *cache;
    uint8_t *rgba;
    float *depth, *rgbz_rgb, *rgbz_z;
    uint64_t *vis_bm, *act_bm;
    uint32_t *visible_ids, *active_ids, *rays_per_block, *block_ray_offsets;
    uint32_t *sorted_ray_ids, *sorted_hit_slots, *valid_prefix;
    int64_t n_vis, n_actb, n_entries, slots_used, pass_index;
    int64_t *tmp_ids;
    int64_t tmp_cap;
};

orc_session *orc_session_create(const uint8_t *payload, const float *ranges,
                                const double *fine_min, const double *fine_max,
                                const double *coarse_min,
                                const double *coarse_max, int nx, int ny,
                                int nz, int qbits, int stride,
                                const double *origin, const double *direction,
                                int64_t n, int64_t w, int64_t h, double iso,
                                int speculation, int max_spec,
                                int64_t cache_capacity, int corrupt_cache) {
    (void)ranges;
    orc_session *s = xcalloc(1, sizeof(orc_session));
    s->payload = payload;
    s->fmin = fine_min;
    s->fmax = fine_max;
    s->cmin = coarse_min;
    s->cmax = coarse_max;
    s->nx = nx;
    s->ny = ny;
    s->nz = nz;
    s->qbits = qbits;
    s->stride = stride;
    s->bdx = (nx + 3) / 4;
    s->bdy = (ny + 3) / 4;
    s->bdz = (nz + 3) / 4;
    s->cdx = (s->bdx + 3) / 4;
    s->cdy = (s->bdy + 3) / 4;
    s->cdz = (s->bdz + 3) / 4;
    s->n_blocks = s->bdx * s->bdy * s->bdz;
    s->n = n;
    s->w = w;
    s->h = h;
    s->origin = origin;
    s->direction = direction;
    s->iso = iso;
    s->base[0] = s->base[1] = s->base[2] = 0.85; /* blocktrace.py:27 */
    s->speculation = speculation;
    s->max_spec = max_spec;
    s->corrupt = corrupt_cache;
    s->t_enter = xmalloc(sizeof(double) * n);
    s->t_exit = xmalloc(sizeof(double) * n);
    s->coarse_tmax = xmalloc(sizeof(double) * 3 * n);
    s->fine_tmax = xmalloc(sizeof(double) * 3 * n);
    s->status = xmalloc(n);
    s->exited = xmalloc(n);
    s->coarse_cell = xmalloc(4 * n);
    s->fine_cell = xmalloc(4 * n);
    s->block_slots = xmalloc(4 * n);
    s->ray_slots = xmalloc(4 * n);
    s->active_offsets = xmalloc(4 * n);
    s->valid_prefix = xmalloc(4 * n);
    s->sorted_ray_ids = xmalloc(4 * n);
    s->sorted_hit_slots = xmalloc(4 * n);
    s->visible_ids = xmalloc(4 * n);
    s->rays_per_block = xmalloc(4 * n);
    s->block_ray_offsets = xmalloc(4 * n);
    s->tmp_cap = 8 * n < s->n_blocks ? 8 * n : s->n_blocks;
    s->active_ids = xmalloc(4 * (s->tmp_cap + 1));
    s->tmp_ids = xmalloc(sizeof(int64_t) * (s->tmp_cap + 1));
    s->rgbz_rgb = xcalloc(3 * n, sizeof(float));
    s->rgbz_z = xmalloc(sizeof(float) * n);
    s->rgba = xmalloc(4 * n);
    s->depth = xmalloc(sizeof(float) * n);
    for (int64_t r = 0; r < n; r++) {
        s->rgba[4 * r] = s->rgba[4 * r + 1] = s->rgba[4 * r + 2] = 0; /* engine.py:29,56-60 */
        s->rgba[4 * r + 3] = 255;
        s->depth[r] = INFINITY;
        s->block_slots[r] = s->ray_slots[r] = ORC_UINT_MAX;
    }
    const int64_t words = (s->n_blocks + 63) / 64;
    s->vis_bm = xcalloc(words, 8);
    s->act_bm = xcalloc(words, 8);
    from_rays(origin, direction, n, nx, ny, nz, s->t_enter, s->t_exit, s->status, s->exited,
              s->coarse_cell, s->fine_cell, s->coarse_tmax, s->fine_tmax);
    if (cache_capacity <= 0) {
        cache_capacity = 2 * (w * h) / 64; /* cache.py:122-125 */
        if (cache_capacity < 1024) cache_capacity = 1024;
    }
    s->cache = orc_cache_create(cache_capacity, s->n_blocks);
    return s;
}

void orc_session_destroy(orc_session *s) {
    if (!s) return;
    free(s->t_enter); free(s->t_exit); free(s->coarse_tmax); free(s->fine_tmax);
    free(s->status); free(s->exited); free(s->coarse_cell); free(s->fine_cell);
    free(s->block_slots); free(s->ray_slots); free(s->active_offsets); free(s->valid_prefix);
    free(s->sorted_ray_ids); free(s->sorted_hit_slots); free(s->visible_ids);
    free(s->rays_per_block); free(s->block_ray_offsets); free(s->active_ids); free(s->tmp_ids);
    free(s->rgbz_rgb); free(s->rgbz_z); free(s->rgba); free(s->depth);
    free(s->vis_bm); free(s->act_bm);
    orc_cache_destroy(s->cache);
    free(s);
}

/* traversal.py:217-403 _traverse_kernel for one ray */
static void traverse_ray(orc_session *s, int64_t r, int64_t n_spec) {
    const double ox = s->origin[3 * r], oy = s->origin[3 * r + 1], oz = s->origin[3 * r + 2];
    const double dx = s->direction[3 * r], dy = s->direction[3 * r + 1], dz = s->direction[3 * r + 2];
    const double te = s->t_exit[r];
    const int64_t fdx = s->bdx, fdy = s->bdy, fdz = s->bdz, cdx = s->cdx, cdy = s->cdy, cdz = s->cdz;
    const double iso = s->iso;
    const int sx = dx > 0.0 ? 1 : (dx < 0.0 ? -1 : 0);
    const int sy = dy > 0.0 ? 1 : (dy < 0.0 ? -1 : 0);
    const int sz = dz > 0.0 ? 1 : (dz < 0.0 ? -1 : 0);
    const double fdel_x = dx != 0.0 ? 4.0 / fabs(dx) : INFINITY;
    const double fdel_y = dy != 0.0 ? 4.0 / fabs(dy) : INFINITY;
    const double fdel_z = dz != 0.0 ? 4.0 / fabs(dz) : INFINITY;
    const double cdel_x = dx != 0.0 ? 16.0 / fabs(dx) : INFINITY;
    const double cdel_y = dy != 0.0 ? 16.0 / fabs(dy) : INFINITY;
    const double cdel_z = dz != 0.0 ? 16.0 / fabs(dz) : INFINITY;
    const int64_t cc = s->coarse_cell[r];
    int64_t ccx = cc % cdx, ccy = (cc / cdx) % cdy, ccz = cc / (cdx * cdy);
    double ctx = s->coarse_tmax[3 * r], cty = s->coarse_tmax[3 * r + 1], ctz = s->coarse_tmax[3 * r + 2];
    const int64_t fc = s->fine_cell[r];
    int in_fine_run = fc != (int64_t)ORC_UINT_MAX;
    int64_t fcx = 0, fcy = 0, fcz = 0;
    if (in_fine_run) {
        fcx = fc % fdx;
        fcy = (fc / fdx) % fdy;
        fcz = fc / (fdx * fdy);
    }
    double ftx = s->fine_tmax[3 * r], fty = s->fine_tmax[3 * r + 1], ftz = s->fine_tmax[3 * r + 2];
    const int64_t base = (int64_t)s->active_offsets[r] * n_spec;
    int64_t emitted = 0;
    int ray_done = 0;
    double t_cross;
    for (;;) {
        if (in_fine_run) {
            for (;;) {
                const int64_t f_lin = fcx + fdx * (fcy + fdy * fcz);
                if (s->fmin[f_lin] <= iso && iso <= s->fmax[f_lin]) {
                    s->block_slots[base + emitted] = (uint32_t)f_lin;
                    s->ray_slots[base + emitted] = (uint32_t)r;
                    emitted++;
                }
                if (ftx <= fty && ftx <= ftz) {
                    t_cross = ftx;
                    fcx += sx;
                    ftx += fdel_x;
                } else if (fty <= ftz) {
                    t_cross = fty;
                    fcy += sy;
                    fty += fdel_y;
                } else {
                    t_cross = ftz;
                    fcz += sz;
                    ftz += fdel_z;
                }
                if (t_cross > te || fcx < 0 || fcx >= fdx || fcy < 0 || fcy >= fdy || fcz < 0 || fcz >= fdz) {
                    in_fine_run = 0;
                    ray_done = 1;
                } else if ((fcx >> 2) != ccx || (fcy >> 2) != ccy || (fcz >> 2) != ccz) {
                    in_fine_run = 0;
                }
                if (emitted == n_spec || !in_fine_run) break;
            }
            if (emitted == n_spec || ray_done) break;
        }
        if (ctx <= cty && ctx <= ctz) {
            t_cross = ctx;
            ccx += sx;
            ctx += cdel_x;
        } else if (cty <= ctz) {
            t_cross = cty;
            ccy += sy;
            cty += cdel_y;
        } else {
            t_cross = ctz;
            ccz += sz;
            ctz += cdel_z;
        }
        if (t_cross > te || ccx < 0 || ccx >= cdx || ccy < 0 || ccy >= cdy || ccz < 0 || ccz >= cdz) {
            ray_done = 1;
            break;
        }
        const int64_t c_lin = ccx + cdx * (ccy + cdy * ccz);
        if (s->cmin[c_lin] <= iso && iso <= s->cmax[c_lin]) {
            const double px = ox + dx * t_cross, py = oy + dy * t_cross, pz = oz + dz * t_cross;
            const int64_t lo_x = 4 * ccx, lo_y = 4 * ccy, lo_z = 4 * ccz;
            const int64_t hi_x = lo_x + 3 < fdx - 1 ? lo_x + 3 : fdx - 1;
            const int64_t hi_y = lo_y + 3 < fdy - 1 ? lo_y + 3 : fdy - 1;
            const int64_t hi_z = lo_z + 3 < fdz - 1 ? lo_z + 3 : fdz - 1;
            fcx = (int64_t)floor(px / 4.0);
            fcy = (int64_t)floor(py / 4.0);
            fcz = (int64_t)floor(pz / 4.0);
            if (fcx < lo_x) fcx = lo_x; else if (fcx > hi_x) fcx = hi_x;
            if (fcy < lo_y) fcy = lo_y; else if (fcy > hi_y) fcy = hi_y;
            if (fcz < lo_z) fcz = lo_z; else if (fcz > hi_z) fcz = hi_z;
            ftx = dx > 0.0 ? ((double)(fcx + 1) * 4.0 - ox) / dx : (dx < 0.0 ? ((double)fcx * 4.0 - ox) / dx : INFINITY);
            fty = dy > 0.0 ? ((double)(fcy + 1) * 4.0 - oy) / dy : (dy < 0.0 ? ((double)fcy * 4.0 - oy) / dy : INFINITY);
            ftz = dz > 0.0 ? ((double)(fcz + 1) * 4.0 - oz) / dz : (dz < 0.0 ? ((double)fcz * 4.0 - oz) / dz : INFINITY);
            in_fine_run = 1;
        }
    }
    if (ray_done) {
        s->exited[r] = 1;
        s->coarse_cell[r] = ORC_UINT_MAX;
        s->fine_cell[r] = ORC_UINT_MAX;
    } else {
        s->coarse_cell[r] = (uint32_t)(ccx + cdx * (ccy + cdy * ccz));
        s->fine_cell[r] = in_fine_run ? (uint32_t)(fcx + fdx * (fcy + fdy * fcz)) : ORC_UINT_MAX;
    }
    s->coarse_tmax[3 * r] = ctx;
    s->coarse_tmax[3 * r + 1] = cty;
    s->coarse_tmax[3 * r + 2] = ctz;
    s->fine_tmax[3 * r] = ftx;
    s->fine_tmax[3 * r + 1] = fty;
    s->fine_tmax[3 * r + 2] = ftz;
}

static int64_t bitmap_extract(uint64_t *bm, int64_t words, uint32_t *out) {
    int64_t k = 0;
    for (int64_t w = 0; w < words; w++) {
        uint64_t v = bm[w];
        if (!v) continue;
        bm[w] = 0;
        while (v) {
            const int b = __builtin_ctzll(v);
            out[k++] = (uint32_t)(64 * w + b);
            v &= v - 1;
        }
    }
    return k;
}

static int64_t lower_bound_u32(const uint32_t *a, int64_t n, uint32_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

/* engine.py:216-219 + blocktrace.py:49-94 for one visible block */
static void raytrace_block_entries(orc_session *s, int64_t v) {
    const int64_t b = s->visible_ids[v];
    const int64_t bx = b % s->bdx, by = (b / s->bdx) % s->bdy, bz = b / (s->bdx * s->bdy);
    float dual[125];
    memset(dual, 0, sizeof(dual));
    int64_t slot[8]; /* engine.py:286-305 _contributor_table */
    for (int oz = 0; oz < 2; oz++)
        for (int oy = 0; oy < 2; oy++)
            for (int ox = 0; ox < 2; ox++) {
                const int idx = ox + 2 * oy + 4 * oz;
                if (bx + ox < s->bdx && by + oy < s->bdy && bz + oz < s->bdz) {
                    const int64_t nid = (bx + ox) + s->bdx * ((by + oy) + s->bdy * (bz + oz));
                    slot[idx] = s->cache->slot_of_block[nid];
                } else {
                    slot[idx] = -1;
                }
            }
    ORC_ASSERT(slot[0] >= 0, "visible block not resident"); /* engine.py:302 */
    const float *sv = s->cache->slot_values;
    /* blocktrace.py:49-94 _assemble_dual */
    for (int k = 0; k < 5; k++)
        for (int j = 0; j < 5; j++)
            for (int i = 0; i < 5; i++) {
                const int ox = i == 4, oy = j == 4, oz = k == 4;
                const int64_t sl = slot[ox + 2 * oy + 4 * oz];
                if (sl < 0) continue;
                dual[i + 5 * j + 25 * k] = sv[64 * sl + (i & 3) + 4 * (j & 3) + 16 * (k & 3)];
            }
    int64_t cells[3];
    const int64_t dims[3] = {s->nx, s->ny, s->nz}, bc[3] = {bx, by, bz};
    for (int a = 0; a < 3; a++) {
        int64_t c = dims[a] - 1 - 4 * bc[a];
        cells[a] = c < 0 ? 0 : (c > 4 ? 4 : c);
    }
    const int64_t start = s->block_ray_offsets[v];
    for (int64_t j = start; j < start + s->rays_per_block[v]; j++) {
        const int64_t r = s->sorted_ray_ids[j];
        double rgb[3];
        const double *o = s->origin + 3 * r, *d = s->direction + 3 * r;
        const double t = trace_region(dual, 5, 25, 4 * bx, 4 * by, 4 * bz, 4 * bx, 4 * by, 4 * bz, cells[0],
                                      cells[1], cells[2], o[0], o[1], o[2], d[0], d[1], d[2], s->t_enter[r],
                                      s->iso, s->base[0], s->base[1], s->base[2], rgb);
        if (t != INFINITY) {
            const int64_t sl = s->sorted_hit_slots[j];
            s->rgbz_z[sl] = (float)t;
            s->rgbz_rgb[3 * sl] = (float)rgb[0];
            s->rgbz_rgb[3 * sl + 1] = (float)rgb[1];
            s->rgbz_rgb[3 * sl + 2] = (float)rgb[2];
        }
    }
}

/* engine.py:308-382, one pass */
int orc_session_pass(orc_session *s, orc_pass_stats *st) {
    const int64_t n = s->n;
    int64_t n_act = 0;
    for (int64_t r = 0; r < n; r++) n_act += s->status[r] == 0;
    if (n_act == 0) return 0;
    const double t_start = now_s();
    /* engine.py:331 exclusive_scan(active_mask) */
    int64_t acc = 0;
    for (int64_t r = 0; r < n; r++) {
        s->active_offsets[r] = (uint32_t)acc;
        acc += s->status[r] == 0;
    }
    /* engine.py:91-94,333 compute_n_spec */
    int64_t n_spec = 1;
    if (s->speculation) {
        int64_t q = (s->w * s->h) / n_act;
        if (q < 1) q = 1;
        n_spec = q < s->max_spec ? q : s->max_spec;
    }
    ORC_ASSERT(n_act * n_spec <= n, "slot budget exceeded"); /* traversal.py:422 */
    /* traversal.py:423-424 */
    for (int64_t i = 0; i < n; i++) s->block_slots[i] = s->ray_slots[i] = ORC_UINT_MAX;
    for (int64_t r = 0; r < n; r++)
        if (s->status[r] == 0) traverse_ray(s, r, n_spec);
    s->slots_used = n_act * n_spec;
    /* engine.py:97-118 mark_blocks */
    const int64_t words = (s->n_blocks + 63) / 64;
    for (int64_t i = 0; i < s->slots_used; i++) {
        const uint32_t b = s->block_slots[i];
        if (b == ORC_UINT_MAX) continue;
        s->vis_bm[b >> 6] |= 1ull << (b & 63);
    }
    s->n_vis = bitmap_extract(s->vis_bm, words, s->visible_ids);
    for (int64_t v = 0; v < s->n_vis; v++) {
        const int64_t b = s->visible_ids[v];
        const int64_t bx = b % s->bdx, by = (b / s->bdx) % s->bdy, bz = b / (s->bdx * s->bdy);
        for (int oz = 0; oz < 2; oz++)
            for (int oy = 0; oy < 2; oy++)
                for (int ox = 0; ox < 2; ox++) {
                    if (bx + ox >= s->bdx || by + oy >= s->bdy || bz + oz >= s->bdz) continue;
                    const int64_t nid = (bx + ox) + s->bdx * ((by + oy) + s->bdy * (bz + oz));
                    s->act_bm[nid >> 6] |= 1ull << (nid & 63);
                }
    }
    s->n_actb = bitmap_extract(s->act_bm, words, s->active_ids);
    for (int64_t i = 0; i < s->n_actb; i++) s->tmp_ids[i] = s->active_ids[i];
    /* engine.py:337 cache.ensure_resident */
    int64_t cst[3];
    orc_cache_update(s->cache, s->payload, s->qbits, s->stride, s->tmp_ids, s->n_actb, cst);
    if (s->corrupt) memset(s->cache->slot_values, 0, sizeof(float) * 64 * (size_t)s->cache->cap);
    /* engine.py:121-149 build_rt_inputs (stable counting sort by block) */
    int64_t ne = 0;
    for (int64_t i = 0; i < n; i++) {
        s->valid_prefix[i] = (uint32_t)ne;
        ne += s->block_slots[i] != ORC_UINT_MAX;
    }
    s->n_entries = ne;
    ORC_ASSERT(ne <= n, "slot budget exceeded"); /* engine.py:341 */
    for (int64_t v = 0; v < s->n_vis; v++) s->rays_per_block[v] = 0;
    for (int64_t i = 0; i < s->slots_used; i++) {
        const uint32_t b = s->block_slots[i];
        if (b == ORC_UINT_MAX) continue;
        s->rays_per_block[lower_bound_u32(s->visible_ids, s->n_vis, b)]++;
    }
    uint32_t run = 0;
    for (int64_t v = 0; v < s->n_vis; v++) {
        s->block_ray_offsets[v] = run;
        run += s->rays_per_block[v];
    }
    ORC_ASSERT((int64_t)run == ne, "ray-block grouping is inconsistent"); /* engine.py:140 */
    uint32_t *cursor = xmalloc(4 * (s->n_vis + 1));
    memcpy(cursor, s->block_ray_offsets, 4 * s->n_vis);
    for (int64_t i = 0; i < s->slots_used; i++) {
        const uint32_t b = s->block_slots[i];
        if (b == ORC_UINT_MAX) continue;
        const int64_t v = lower_bound_u32(s->visible_ids, s->n_vis, b);
        const uint32_t pos = cursor[v]++;
        s->sorted_ray_ids[pos] = s->ray_slots[i];
        s->sorted_hit_slots[pos] = s->valid_prefix[i];
    }
    free(cursor);
    /* engine.py:343-344 */
    for (int64_t i = 0; i < n; i++) {
        s->rgbz_z[i] = INFINITY;
        s->rgbz_rgb[3 * i] = s->rgbz_rgb[3 * i + 1] = s->rgbz_rgb[3 * i + 2] = 0.0f;
    }
    /* engine.py:345-366 */
    for (int64_t v = 0; v < s->n_vis; v++) raytrace_block_entries(s, v);
    /* engine.py:222-258 _composite_kernel */
    int64_t n_after = 0;
    for (int64_t r = 0; r < n; r++) {
        if (s->status[r] != 0) continue;
        const int64_t base = (int64_t)s->active_offsets[r] * n_spec;
        double best = INFINITY;
        int64_t best_slot = -1;
        for (int64_t k = 0; k < n_spec; k++) {
            const int64_t sidx = base + k;
            if (s->block_slots[sidx] != ORC_UINT_MAX) {
                const int64_t slot = s->valid_prefix[sidx];
                const float z = s->rgbz_z[slot];
                if ((double)z < best) {
                    best = (double)z;
                    best_slot = slot;
                }
            }
        }
        if (best_slot >= 0) {
            s->depth[r] = (float)best;
            s->rgba[4 * r] = rgb_u8(s->rgbz_rgb[3 * best_slot]);
            s->rgba[4 * r + 1] = rgb_u8(s->rgbz_rgb[3 * best_slot + 1]);
            s->rgba[4 * r + 2] = rgb_u8(s->rgbz_rgb[3 * best_slot + 2]);
            s->rgba[4 * r + 3] = 255;
            s->status[r] = 1;
        } else if (s->exited[r] == 1) {
            s->status[r] = 2;
        } else {
            n_after++;
        }
    }
    st->pass_index = s->pass_index;
    st->n_active_before = n_act;
    st->n_spec = n_spec;
    st->visible_blocks = s->n_vis;
    st->active_blocks = s->n_actb;
    st->new_decompressed = cst[0];
    st->evicted = cst[1];
    st->cache_slots = cst[2];
    st->n_entries = ne;
    st->n_active_after = n_after;
    st->utilization = (double)ne / (double)n;
    st->completeness = (double)(n - n_after) / (double)n;
    st->duration = now_s() - t_start;
    s->pass_index++;
    return 1;
}

void orc_get_rays(const orc_session *s, double *t_enter, double *t_exit,
                  uint8_t *status, uint8_t *exited, uint32_t *coarse_cell,
                  uint32_t *fine_cell, double *coarse_tmax, double *fine_tmax) {
    const int64_t n = s->n;
    if (t_enter) memcpy(t_enter, s->t_enter, 8 * n);
    if (t_exit) memcpy(t_exit, s->t_exit, 8 * n);
    if (status) memcpy(status, s->status, n);
    if (exited) memcpy(exited, s->exited, n);
    if (coarse_cell) memcpy(coarse_cell, s->coarse_cell, 4 * n);
    if (fine_cell) memcpy(fine_cell, s->fine_cell, 4 * n);
    if (coarse_tmax) memcpy(coarse_tmax, s->coarse_tmax, 24 * n);
    if (fine_tmax) memcpy(fine_tmax, s->fine_tmax, 24 * n);
}

void orc_get_framebuffer(const orc_session *s, uint8_t *rgba, float *depth) {
    if (rgba) memcpy(rgba, s->rgba, 4 * s->n);
    if (depth) memcpy(depth, s->depth, 4 * s->n);
}

void orc_get_pass_sizes(const orc_session *s, int64_t *sizes) {
    sizes[0] = s->slots_used;
    sizes[1] = s->n_vis;
    sizes[2] = s->n_actb;
    sizes[3] = s->n_entries;
}

void orc_get_slots(const orc_session *s, uint32_t *block_slots,
                   uint32_t *ray_slots, uint32_t *active_offsets) {
    if (block_slots) memcpy(block_slots, s->block_slots, 4 * s->n);
    if (ray_slots) memcpy(ray_slots, s->ray_slots, 4 * s->n);
    if (active_offsets) memcpy(active_offsets, s->active_offsets, 4 * s->n);
}

void orc_get_visible_active(const orc_session *s, uint32_t *visible_ids,
                            uint32_t *active_ids) {
    if (visible_ids) memcpy(visible_ids, s->visible_ids, 4 * s->n_vis);
    if (active_ids) memcpy(active_ids, s->active_ids, 4 * s->n_actb);
}

void orc_get_rt_inputs(const orc_session *s, uint32_t *rays_per_block,
                       uint32_t *block_ray_offsets, uint32_t *sorted_ray_ids,
                       uint32_t *sorted_hit_slots, uint32_t *valid_prefix) {
    if (rays_per_block) memcpy(rays_per_block, s->rays_per_block, 4 * s->n_vis);
    if (block_ray_offsets) memcpy(block_ray_offsets, s->block_ray_offsets, 4 * s->n_vis);
    if (sorted_ray_ids) memcpy(sorted_ray_ids, s->sorted_ray_ids, 4 * s->n_entries);
    if (sorted_hit_slots) memcpy(sorted_hit_slots, s->sorted_hit_slots, 4 * s->n_entries);
    if (valid_prefix) memcpy(valid_prefix, s->valid_prefix, 4 * s->n);
}

void orc_get_rgbz(const orc_session *s, float *rgb, float *z) {
    if (rgb) memcpy(rgb, s->rgbz_rgb, 12 * s->n);
    if (z) memcpy(z, s->rgbz_z, 4 * s->n);
}

int64_t orc_cache_capacity(const orc_session *s) { return s->cache->cap; }

void orc_session_set_base_color(orc_session *s, double r, double g, double b) {
    s->base[0] = r;
    s->base[1] = g;
    s->base[2] = b;
}

void orc_get_cache(const orc_session *s, int64_t *block_of_slot,
                   int64_t *last_used, float *slot_values) {
    orc_cache_state(s->cache, block_of_slot, last_used, slot_values);
}

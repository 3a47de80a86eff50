// wc_trace.cuh -- per-cell isosurface intersection and shading (device).
//
// Bit-exact restatement of blocktrace.py:126-449 for sm_100a.  Compiled with
// -fmad=false; every expression keeps the reference's evaluation order
// (Python is left-to-right, numba emits no FMA), float32 corner differences
// stay float32 (_grad_at, blocktrace.py:283-303), and Python's max/min
// keep the first argument on ties (blocktrace.py:136-137 etc.).
#pragma once

#include <math_constants.h>

#include "wc_common.cuh"

namespace wc {

constexpr double kAmbient = 0.2;       // blocktrace.py:26
constexpr double kEntryNudge = 1e-7;   // blocktrace.py:31
constexpr double kEntryEps = 4e-4;     // traversal.py:32

__device__ __forceinline__ double py_max(double a, double b) { return (b > a) ? b : a; }
__device__ __forceinline__ double py_min(double a, double b) { return (b < a) ? b : a; }

// blocktrace.py:126-158 _cell_overlap
// (rd: the reciprocals of d, recip_of; the quotients are exactly (x - o) / d)
__device__ __forceinline__ void cell_overlap(const double o[3], const double d[3], const Recip rd[3],
                                             const double c[3], double &t0o, double &t1o) {
    double t0 = -CUDART_INF, t1 = CUDART_INF;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        if (d[a] != 0.0) {
            double ta = div_by(c[a] - o[a], rd[a]);
            double tb = div_by(c[a] + 1.0 - o[a], rd[a]);
            if (ta > tb) {
                const double t = ta;
                ta = tb;
                tb = t;
            }
            t0 = py_max(t0, ta);
            t1 = py_min(t1, tb);
        } else if (o[a] < c[a] || o[a] > c[a] + 1.0) {
            t0o = CUDART_INF;
            t1o = -CUDART_INF;
            return;
        }
    }
    t0o = t0;
    t1o = t1;
}

// blocktrace.py:193-195
__device__ __forceinline__ double poly_eval(double A, double B, double C, double D, double t) {
    return ((A * t + B) * t + C) * t + D;
}

// blocktrace.py:198-233 _refine_root (Illinois regula falsi, bisection fallback)
static __device__ __noinline__ double refine_root(double A, double B, double C, double D, double lo, double hi,
                                           double g_lo, double g_hi) {
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

// blocktrace.py:161-190 _cubic_coeffs + blocktrace.py:236-280 _intersect_cubic
__device__ __forceinline__ double intersect_cubic(const float c[8], const double o[3], const double d[3],
                                                  const double cell[3], double t0, double t1, double iso) {
    const double ax1 = o[0] - cell[0], ay1 = o[1] - cell[1], az1 = o[2] - cell[2];
    const double ax0 = 1.0 - ax1, ay0 = 1.0 - ay1, az0 = 1.0 - az1;
    double A = 0.0, B = 0.0, C = 0.0, D = 0.0;
#pragma unroll
    for (int idx = 0; idx < 8; idx++) {
        const int i = idx & 1, j = (idx >> 1) & 1, k = (idx >> 2) & 1;
        const double axa = i ? ax1 : ax0, axb = i ? d[0] : -d[0];
        const double aya = j ? ay1 : ay0, ayb = j ? d[1] : -d[1];
        const double aza = k ? az1 : az0, azb = k ? d[2] : -d[2];
        const double w = (double)c[idx];
        A += w * ((axb * ayb) * azb);
        B += w * (((axa * ayb) * azb + (axb * aya) * azb) + (axb * ayb) * aza);
        C += w * (((axa * aya) * azb + (axa * ayb) * aza) + (axb * aya) * aza);
        D += w * ((axa * aya) * aza);
    }
    D -= iso;
    // split points t0 < [m1 < m2] < t1 (registers, no local array)
    double m1 = 0.0, m2 = 0.0;
    int nm = 0;
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
            if (t0 < r1 && r1 < t1) m1 = r1, nm = 1;
            if (t0 < r2 && r2 < t1 && r2 != r1) {
                if (nm == 0)
                    m1 = r2;
                else
                    m2 = r2;
                nm++;
            }
        }
    } else if (qb != 0.0) {
        const double r1 = -C / qb;
        if (t0 < r1 && r1 < t1) m1 = r1, nm = 1;
    }
    double t_prev = t0, g_prev = poly_eval(A, B, C, D, t0);
    if (g_prev == 0.0) return t0;
#pragma unroll
    for (int i = 1; i <= 3; i++) {
        if (i > nm + 1) break;
        const double t_here = i > nm ? t1 : (i == 1 ? m1 : m2);
        const double g_here = poly_eval(A, B, C, D, t_here);
        if (g_here == 0.0) return t_here;
        if ((g_prev < 0.0) != (g_here < 0.0)) return refine_root(A, B, C, D, t_prev, t_here, g_prev, g_here);
        t_prev = t_here;
        g_prev = g_here;
    }
    return CUDART_INF;
}

// blocktrace.py:283-303 _grad_at (corner differences in float32) and
// blocktrace.py:306-314 _shade (two-sided headlight, ambient floor).
__device__ __forceinline__ void grad_shade(const float c[8], double ux, double uy, double uz, const double d[3],
                                           double br, double bg, double bb, float rgb[3]) {
    const double gx = (((double)(c[1] - c[0]) * (1.0 - uy) * (1.0 - uz) + (double)(c[3] - c[2]) * uy * (1.0 - uz)) +
                       (double)(c[5] - c[4]) * (1.0 - uy) * uz) +
                      (double)(c[7] - c[6]) * uy * uz;
    const double gy = (((double)(c[2] - c[0]) * (1.0 - ux) * (1.0 - uz) + (double)(c[3] - c[1]) * ux * (1.0 - uz)) +
                       (double)(c[6] - c[4]) * (1.0 - ux) * uz) +
                      (double)(c[7] - c[5]) * ux * uz;
    const double gz = (((double)(c[4] - c[0]) * (1.0 - ux) * (1.0 - uy) + (double)(c[5] - c[1]) * ux * (1.0 - uy)) +
                       (double)(c[6] - c[2]) * (1.0 - ux) * uy) +
                      (double)(c[7] - c[3]) * ux * uy;
    const double gl = sqrt((gx * gx + gy * gy) + gz * gz);
    double inten;
    if (gl == 0.0) {
        inten = kAmbient;
    } else {
        const double cos_t = fabs((gx * d[0] + gy * d[1]) + gz * d[2]) / gl;
        inten = cos_t > kAmbient ? cos_t : kAmbient;
    }
    rgb[0] = (float)(br * inten);
    rgb[1] = (float)(bg * inten);
    rgb[2] = (float)(bb * inten);
}

// blocktrace.py:306-314 _shade on its own (the reference's `shade` API).
__device__ __forceinline__ void shade_grad(double gx, double gy, double gz, const double d[3], double br, double bg,
                                           double bb, double rgb[3]) {
    const double gl = sqrt((gx * gx + gy * gy) + gz * gz);
    double inten;
    if (gl == 0.0) {
        inten = kAmbient;
    } else {
        const double cos_t = fabs((gx * d[0] + gy * d[1]) + gz * d[2]) / gl;
        inten = cos_t > kAmbient ? cos_t : kAmbient;
    }
    rgb[0] = br * inten;
    rgb[1] = bg * inten;
    rgb[2] = bb * inten;
}

// Same, returning float64 colour (oracle.py:88-90 quantises the f64 value).
__device__ __forceinline__ void grad_shade_d(const float c[8], double ux, double uy, double uz, const double d[3],
                                             double br, double bg, double bb, double rgb[3]) {
    const double gx = (((double)(c[1] - c[0]) * (1.0 - uy) * (1.0 - uz) + (double)(c[3] - c[2]) * uy * (1.0 - uz)) +
                       (double)(c[5] - c[4]) * (1.0 - uy) * uz) +
                      (double)(c[7] - c[6]) * uy * uz;
    const double gy = (((double)(c[2] - c[0]) * (1.0 - ux) * (1.0 - uz) + (double)(c[3] - c[1]) * ux * (1.0 - uz)) +
                       (double)(c[6] - c[4]) * (1.0 - ux) * uz) +
                      (double)(c[7] - c[5]) * ux * uz;
    const double gz = (((double)(c[4] - c[0]) * (1.0 - ux) * (1.0 - uy) + (double)(c[5] - c[1]) * ux * (1.0 - uy)) +
                       (double)(c[6] - c[2]) * (1.0 - ux) * uy) +
                      (double)(c[7] - c[3]) * ux * uy;
    const double gl = sqrt((gx * gx + gy * gy) + gz * gz);
    double inten;
    if (gl == 0.0) {
        inten = kAmbient;
    } else {
        const double cos_t = fabs((gx * d[0] + gy * d[1]) + gz * d[2]) / gl;
        inten = cos_t > kAmbient ? cos_t : kAmbient;
    }
    rgb[0] = br * inten;
    rgb[1] = bg * inten;
    rgb[2] = bb * inten;
}

// Field accessor: corners of dual cell (cx,cy,cz) relative to the field
// origin; Field must provide load(lx, ly, lz) for local integer coords.
//
// blocktrace.py:317-449 _trace_region.  Returns t (+inf on miss) and, on a
// hit, the shaded colour through rgb (float32 for the engine, float64 for
// the brute-force oracle via RGB = double).
template <class Field, typename RGB>
__device__ double trace_region(const Field &field, int fox, int foy, int foz, int lo_x, int lo_y, int lo_z, int n_x,
                               int n_y, int n_z, const double o[3], const double d[3], double ray_t_enter, double iso,
                               double br, double bg, double bb, RGB *rgb) {
    if (n_x <= 0 || n_y <= 0 || n_z <= 0) return CUDART_INF;
    double t0 = ray_t_enter, t1 = CUDART_INF;
    const int lo[3] = {lo_x, lo_y, lo_z}, nn[3] = {n_x, n_y, n_z};
    const Recip rd[3] = {recip_of(d[0]), recip_of(d[1]), recip_of(d[2])};
#pragma unroll
    for (int a = 0; a < 3; a++) {
        if (d[a] != 0.0) {
            double ta = div_by((double)lo[a] - o[a], rd[a]);
            double tb = div_by((double)(lo[a] + nn[a]) - o[a], rd[a]);
            if (ta > tb) {
                const double t = ta;
                ta = tb;
                tb = t;
            }
            t0 = py_max(t0, ta);
            t1 = py_min(t1, tb);
        } else if (o[a] < (double)lo[a] || o[a] > (double)(lo[a] + nn[a])) {
            return CUDART_INF;
        }
    }
    if (t0 > t1) return CUDART_INF;
    const double ts = t0 + kEntryNudge * py_max(1.0, t1 - t0);
    int cx = (int)floor(o[0] + d[0] * ts);
    int cy = (int)floor(o[1] + d[1] * ts);
    int cz = (int)floor(o[2] + d[2] * ts);
    cx = min(max(cx, lo_x), lo_x + n_x - 1);
    cy = min(max(cy, lo_y), lo_y + n_y - 1);
    cz = min(max(cz, lo_z), lo_z + n_z - 1);
    const int sx = d[0] > 0.0 ? 1 : (d[0] < 0.0 ? -1 : 0);
    const int sy = d[1] > 0.0 ? 1 : (d[1] < 0.0 ? -1 : 0);
    const int sz = d[2] > 0.0 ? 1 : (d[2] < 0.0 ? -1 : 0);
    // 1 / |d| == |1 / d| (round to nearest is sign-symmetric)
    const double del_x = d[0] != 0.0 ? fabs(div_by(1.0, rd[0])) : CUDART_INF;
    const double del_y = d[1] != 0.0 ? fabs(div_by(1.0, rd[1])) : CUDART_INF;
    const double del_z = d[2] != 0.0 ? fabs(div_by(1.0, rd[2])) : CUDART_INF;
    double tmx = d[0] != 0.0 ? div_by((double)(d[0] > 0.0 ? cx + 1 : cx) - o[0], rd[0]) : CUDART_INF;
    double tmy = d[1] != 0.0 ? div_by((double)(d[1] > 0.0 ? cy + 1 : cy) - o[1], rd[1]) : CUDART_INF;
    double tmz = d[2] != 0.0 ? div_by((double)(d[2] > 0.0 ? cz + 1 : cz) - o[2], rd[2]) : CUDART_INF;
    float c[8];
    for (;;) {
        field.corners(cx - fox, cy - foy, cz - foz, c);
        float cmin = c[0], cmax = c[0];
#pragma unroll
        for (int q = 1; q < 8; q++) {
            if (c[q] < cmin) cmin = c[q];
            if (c[q] > cmax) cmax = c[q];
        }
        if ((double)cmin <= iso && iso <= (double)cmax) {
            const double cell[3] = {(double)cx, (double)cy, (double)cz};
            double ct0, ct1;
            cell_overlap(o, d, rd, cell, ct0, ct1);
            if (ct0 < ray_t_enter) ct0 = ray_t_enter;
            if (ct0 <= ct1) {
                const double th = intersect_cubic(c, o, d, cell, ct0, ct1, iso);
                if (th != CUDART_INF) {
                    double ux = o[0] + d[0] * th - cell[0];
                    double uy = o[1] + d[1] * th - cell[1];
                    double uz = o[2] + d[2] * th - cell[2];
                    ux = py_min(py_max(ux, 0.0), 1.0);
                    uy = py_min(py_max(uy, 0.0), 1.0);
                    uz = py_min(py_max(uz, 0.0), 1.0);
                    if constexpr (sizeof(RGB) == sizeof(float))
                        grad_shade(c, ux, uy, uz, d, br, bg, bb, rgb);
                    else
                        grad_shade_d(c, ux, uy, uz, d, br, bg, bb, rgb);
                    return th;
                }
            }
        }
        if (tmx <= tmy && tmx <= tmz) {
            cx += sx;
            tmx += del_x;
            if (cx < lo_x || cx >= lo_x + n_x) return CUDART_INF;
        } else if (tmy <= tmz) {
            cy += sy;
            tmy += del_y;
            if (cy < lo_y || cy >= lo_y + n_y) return CUDART_INF;
        } else {
            cz += sz;
            tmz += del_z;
            if (cz < lo_z || cz >= lo_z + n_z) return CUDART_INF;
        }
    }
}

// ---- trace_region split in three, for the two-phase raytrace ------------
// (walk the cells, solve every candidate cell with uniform SIMT work, shade
// the first hit).  Together they compute exactly trace_region: the first
// bracketing cell in DDA order whose cubic has a root in its overlap wins.

// blocktrace.py:346-418: clip the ray to the region and walk its dual cells;
// on_cell(cx, cy, cz, seq) is called, in DDA order, for every cell whose
// corner range brackets iso (seq = 0, 1, ...).
template <class Field, class OnCell>
__device__ void walk_bracketing_cells(const Field &field, int fox, int foy, int foz, int lo_x, int lo_y, int lo_z,
                                      int n_x, int n_y, int n_z, const double o[3], const double d[3],
                                      double ray_t_enter, double iso, OnCell on_cell) {
    if (n_x <= 0 || n_y <= 0 || n_z <= 0) return;
    double t0 = ray_t_enter, t1 = CUDART_INF;
    const int lo[3] = {lo_x, lo_y, lo_z}, nn[3] = {n_x, n_y, n_z};
#pragma unroll
    for (int a = 0; a < 3; a++) {
        if (d[a] != 0.0) {
            double ta = ((double)lo[a] - o[a]) / d[a];
            double tb = ((double)(lo[a] + nn[a]) - o[a]) / d[a];
            if (ta > tb) {
                const double t = ta;
                ta = tb;
                tb = t;
            }
            t0 = py_max(t0, ta);
            t1 = py_min(t1, tb);
        } else if (o[a] < (double)lo[a] || o[a] > (double)(lo[a] + nn[a])) {
            return;
        }
    }
    if (t0 > t1) return;
    const double ts = t0 + kEntryNudge * py_max(1.0, t1 - t0);
    int cx = (int)floor(o[0] + d[0] * ts);
    int cy = (int)floor(o[1] + d[1] * ts);
    int cz = (int)floor(o[2] + d[2] * ts);
    cx = min(max(cx, lo_x), lo_x + n_x - 1);
    cy = min(max(cy, lo_y), lo_y + n_y - 1);
    cz = min(max(cz, lo_z), lo_z + n_z - 1);
    const int sx = d[0] > 0.0 ? 1 : (d[0] < 0.0 ? -1 : 0);
    const int sy = d[1] > 0.0 ? 1 : (d[1] < 0.0 ? -1 : 0);
    const int sz = d[2] > 0.0 ? 1 : (d[2] < 0.0 ? -1 : 0);
    const double del_x = d[0] != 0.0 ? 1.0 / fabs(d[0]) : CUDART_INF;
    const double del_y = d[1] != 0.0 ? 1.0 / fabs(d[1]) : CUDART_INF;
    const double del_z = d[2] != 0.0 ? 1.0 / fabs(d[2]) : CUDART_INF;
    double tmx = d[0] > 0.0 ? ((double)(cx + 1) - o[0]) / d[0] : (d[0] < 0.0 ? ((double)cx - o[0]) / d[0] : CUDART_INF);
    double tmy = d[1] > 0.0 ? ((double)(cy + 1) - o[1]) / d[1] : (d[1] < 0.0 ? ((double)cy - o[1]) / d[1] : CUDART_INF);
    double tmz = d[2] > 0.0 ? ((double)(cz + 1) - o[2]) / d[2] : (d[2] < 0.0 ? ((double)cz - o[2]) / d[2] : CUDART_INF);
    // Corners are carried across steps: a step shares a face with the previous
    // cell, so only the 4 corners of the far face are loaded (same values).
    float c[8];
    field.corners(cx - fox, cy - foy, cz - foz, c);
    int seq = 0;
    for (;;) {
        float cmin = c[0], cmax = c[0];
#pragma unroll
        for (int q = 1; q < 8; q++) {
            if (c[q] < cmin) cmin = c[q];
            if (c[q] > cmax) cmax = c[q];
        }
        if ((double)cmin <= iso && iso <= (double)cmax) on_cell(cx, cy, cz, seq++);
        const int lx = cx - fox, ly = cy - foy, lz = cz - foz;
        if (tmx <= tmy && tmx <= tmz) {
            cx += sx;
            tmx += del_x;
            if (cx < lo_x || cx >= lo_x + n_x) return;
            // corner bit 0 is x: keep the shared face, load the new one
            // (compile-time corner indices: c[] stays in registers)
            if (sx > 0) {
#pragma unroll
                for (int q = 0; q < 8; q += 2) {
                    c[q] = c[q + 1];
                    c[q + 1] = field.point(lx + 2, ly + ((q >> 1) & 1), lz + (q >> 2));
                }
            } else {
#pragma unroll
                for (int q = 0; q < 8; q += 2) {
                    c[q + 1] = c[q];
                    c[q] = field.point(lx - 1, ly + ((q >> 1) & 1), lz + (q >> 2));
                }
            }
        } else if (tmy <= tmz) {
            cy += sy;
            tmy += del_y;
            if (cy < lo_y || cy >= lo_y + n_y) return;
            if (sy > 0) {
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    if (q & 2) continue;  // the corners with y bit 0
                    c[q] = c[q + 2];
                    c[q + 2] = field.point(lx + (q & 1), ly + 2, lz + (q >> 2));
                }
            } else {
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    if (q & 2) continue;
                    c[q + 2] = c[q];
                    c[q] = field.point(lx + (q & 1), ly - 1, lz + (q >> 2));
                }
            }
        } else {
            cz += sz;
            tmz += del_z;
            if (cz < lo_z || cz >= lo_z + n_z) return;
            if (sz > 0) {
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    c[q] = c[q + 4];
                    c[q + 4] = field.point(lx + (q & 1), ly + (q >> 1), lz + 2);
                }
            } else {
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    c[q + 4] = c[q];
                    c[q] = field.point(lx + (q & 1), ly + (q >> 1), lz - 1);
                }
            }
        }
    }
}

// Same walk in two phases, for memory-level parallelism: the DDA path
// through the region first (it never depends on the field: <= 10 cells of a
// 4^3 block region, as 6-bit local codes), then the bracketing tests with
// the next cell's 8 corners requested before the current cell's are used.
// on_cell sees the same cells, in the same order, as walk_bracketing_cells.
template <class Field, class OnCell>
__device__ __forceinline__ void walk_bracketing_cells_prefetch(const Field &field, int fox, int foy, int foz, int lo_x,
                                                               int lo_y, int lo_z, int n_x, int n_y, int n_z,
                                                               const double o[3], const double d[3],
                                                               double ray_t_enter, double iso, OnCell on_cell) {
    if (n_x <= 0 || n_y <= 0 || n_z <= 0) return;
    double t0 = ray_t_enter, t1 = CUDART_INF;
    const int lo[3] = {lo_x, lo_y, lo_z}, nn[3] = {n_x, n_y, n_z};
#pragma unroll
    for (int a = 0; a < 3; a++) {
        if (d[a] != 0.0) {
            double ta = ((double)lo[a] - o[a]) / d[a];
            double tb = ((double)(lo[a] + nn[a]) - o[a]) / d[a];
            if (ta > tb) {
                const double t = ta;
                ta = tb;
                tb = t;
            }
            t0 = py_max(t0, ta);
            t1 = py_min(t1, tb);
        } else if (o[a] < (double)lo[a] || o[a] > (double)(lo[a] + nn[a])) {
            return;
        }
    }
    if (t0 > t1) return;
    const double ts = t0 + kEntryNudge * py_max(1.0, t1 - t0);
    int cx = (int)floor(o[0] + d[0] * ts);
    int cy = (int)floor(o[1] + d[1] * ts);
    int cz = (int)floor(o[2] + d[2] * ts);
    cx = min(max(cx, lo_x), lo_x + n_x - 1);
    cy = min(max(cy, lo_y), lo_y + n_y - 1);
    cz = min(max(cz, lo_z), lo_z + n_z - 1);
    const int sx = d[0] > 0.0 ? 1 : (d[0] < 0.0 ? -1 : 0);
    const int sy = d[1] > 0.0 ? 1 : (d[1] < 0.0 ? -1 : 0);
    const int sz = d[2] > 0.0 ? 1 : (d[2] < 0.0 ? -1 : 0);
    const double del_x = d[0] != 0.0 ? 1.0 / fabs(d[0]) : CUDART_INF;
    const double del_y = d[1] != 0.0 ? 1.0 / fabs(d[1]) : CUDART_INF;
    const double del_z = d[2] != 0.0 ? 1.0 / fabs(d[2]) : CUDART_INF;
    double tmx = d[0] > 0.0 ? ((double)(cx + 1) - o[0]) / d[0] : (d[0] < 0.0 ? ((double)cx - o[0]) / d[0] : CUDART_INF);
    double tmy = d[1] > 0.0 ? ((double)(cy + 1) - o[1]) / d[1] : (d[1] < 0.0 ? ((double)cy - o[1]) / d[1] : CUDART_INF);
    double tmz = d[2] > 0.0 ? ((double)(cz + 1) - o[2]) / d[2] : (d[2] < 0.0 ? ((double)cz - o[2]) / d[2] : CUDART_INF);
    // the path (blocktrace.py:428-449 steps): cell k at bits [6k, 6k + 6)
    unsigned long long path = 0;
    int ncell = 0;
    for (;;) {
        path |= (unsigned long long)((cx - lo_x) | ((cy - lo_y) << 2) | ((cz - lo_z) << 4)) << (6 * ncell);
        ncell++;
        if (tmx <= tmy && tmx <= tmz) {
            cx += sx;
            tmx += del_x;
            if (cx < lo_x || cx >= lo_x + n_x) break;
        } else if (tmy <= tmz) {
            cy += sy;
            tmy += del_y;
            if (cy < lo_y || cy >= lo_y + n_y) break;
        } else {
            cz += sz;
            tmz += del_z;
            if (cz < lo_z || cz >= lo_z + n_z) break;
        }
    }
    // the tests, one cell of corner loads ahead
    float cur[8], nxt[8];
    auto cell_of = [&](int k, int &x, int &y, int &z) {
        const uint32_t code = (uint32_t)(path >> (6 * k)) & 63u;
        x = lo_x + (int)(code & 3u);
        y = lo_y + (int)((code >> 2) & 3u);
        z = lo_z + (int)(code >> 4);
    };
    int px, py, pz;
    cell_of(0, px, py, pz);
    field.corners(px - fox, py - foy, pz - foz, cur);
    int seq = 0;
    for (int k = 0; k < ncell; k++) {
        int qx = px, qy = py, qz = pz;
        if (k + 1 < ncell) {
            cell_of(k + 1, qx, qy, qz);
            field.corners(qx - fox, qy - foy, qz - foz, nxt);
        }
        float cmin = cur[0], cmax = cur[0];
#pragma unroll
        for (int q = 1; q < 8; q++) {
            if (cur[q] < cmin) cmin = cur[q];
            if (cur[q] > cmax) cmax = cur[q];
        }
        if ((double)cmin <= iso && iso <= (double)cmax) on_cell(px, py, pz, seq++);
#pragma unroll
        for (int q = 0; q < 8; q++) cur[q] = nxt[q];
        px = qx;
        py = qy;
        pz = qz;
    }
}

// blocktrace.py:420-427: the root in one bracketing cell, or +inf.
__device__ __forceinline__ double solve_cell(const float c[8], const double o[3], const double d[3], int cx, int cy,
                                             int cz, double ray_t_enter, double iso) {
    const double cell[3] = {(double)cx, (double)cy, (double)cz};
    double ct0, ct1;
    const Recip rd[3] = {recip_of(d[0]), recip_of(d[1]), recip_of(d[2])};
    cell_overlap(o, d, rd, cell, ct0, ct1);
    if (ct0 < ray_t_enter) ct0 = ray_t_enter;
    if (!(ct0 <= ct1)) return CUDART_INF;
    return intersect_cubic(c, o, d, cell, ct0, ct1, iso);
}

// blocktrace.py:428-433: shade the hit at parameter th in cell (cx, cy, cz).
__device__ __forceinline__ void shade_hit(const float c[8], const double o[3], const double d[3], int cx, int cy,
                                          int cz, double th, double br, double bg, double bb, float rgb[3]) {
    double ux = o[0] + d[0] * th - (double)cx;
    double uy = o[1] + d[1] * th - (double)cy;
    double uz = o[2] + d[2] * th - (double)cz;
    ux = py_min(py_max(ux, 0.0), 1.0);
    uy = py_min(py_max(uy, 0.0), 1.0);
    uz = py_min(py_max(uz, 0.0), 1.0);
    grad_shade(c, ux, uy, uz, d, br, bg, bb, rgb);
}

// engine.py:152-158 _rgb_u8: clamp, scale in float64, truncating cast.
__device__ __forceinline__ uint32_t rgb_u8(double v) {
    if (v < 0.0)
        v = 0.0;
    else if (v > 1.0)
        v = 1.0;
    return (uint32_t)(v * 255.0 + 0.5);
}

}  // namespace wc

/*
 * oracle/loops.c -- TEST INFRASTRUCTURE ONLY (parity checker and CPU baseline).
 *
 * Plain-C fp64 restatement of the three pixel loops the reference runs under
 * Numba.  Nothing in the product path links or calls this file: it is loaded
 * only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg (via oracle/cgs_oracle.py).
 *
 * Reference: /root/reference/pkg/src/cryosplat/_kernels.py
 *   tile binning   -> build_tile_work   (_kernels.py:17-63)
 *   forward pixels -> forward_tiles     (_kernels.py:66-125)
 *   backward sums  -> backward_pixels   (_kernels.py:128-190)
 *
 * Arithmetic follows the reference operation by operation in IEEE fp64
 * (compiled with -ffp-contract=off so no FMA contraction changes rounding),
 * so outputs agree with the Numba kernels to the last few ulps (tile lists
 * bit-exactly).  Arrays are C-contiguous, int64 where the reference uses
 * int64.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* floor division for the non-negative bbox coordinates used here */
static inline int64_t fdiv(int64_t a, int64_t b) { return a / b; }

/* Pass 1 of build_tile_work: per-tile item counts (_kernels.py:25-42).
 * counts has n_tiles+1 entries; counts[0] stays 0 so that the inclusive
 * cumulative sum is the tile_starts array (_kernels.py:43). */
int64_t oracle_tile_counts(const int64_t *bbox, int64_t n, int64_t tile_size,
                           int64_t n_tiles_x, int64_t n_tiles_y, int64_t *counts) {
    int64_t n_tiles = n_tiles_x * n_tiles_y;
    memset(counts, 0, sizeof(int64_t) * (size_t)(n_tiles + 1));
    for (int64_t g = 0; g < n; ++g) {
        const int64_t *bb = bbox + 4 * g;
        if (bb[0] > bb[1] || bb[2] > bb[3]) continue;
        int64_t tx0 = fdiv(bb[0], tile_size), tx1 = fdiv(bb[1], tile_size);
        int64_t ty0 = fdiv(bb[2], tile_size), ty1 = fdiv(bb[3], tile_size);
        for (int64_t ty = ty0; ty <= ty1; ++ty)
            for (int64_t tx = tx0; tx <= tx1; ++tx) counts[ty * n_tiles_x + tx + 1] += 1;
    }
    int64_t total = 0;
    for (int64_t t = 0; t <= n_tiles; ++t) { total += counts[t]; counts[t] = total; }
    return total; /* counts now holds tile_starts */
}

/* Pass 2 of build_tile_work: scatter ascending Gaussian ids (_kernels.py:44-63).
 * tile_starts from oracle_tile_counts; gauss_ids has tile_starts[n_tiles]. */
void oracle_tile_scatter(const int64_t *bbox, int64_t n, int64_t tile_size,
                         int64_t n_tiles_x, int64_t n_tiles_y,
                         const int64_t *tile_starts, int64_t *gauss_ids) {
    int64_t n_tiles = n_tiles_x * n_tiles_y;
    int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_tiles > 0 ? n_tiles : 1));
    memcpy(cursor, tile_starts, sizeof(int64_t) * (size_t)n_tiles);
    for (int64_t g = 0; g < n; ++g) {
        const int64_t *bb = bbox + 4 * g;
        if (bb[0] > bb[1] || bb[2] > bb[3]) continue;
        int64_t tx0 = fdiv(bb[0], tile_size), tx1 = fdiv(bb[1], tile_size);
        int64_t ty0 = fdiv(bb[2], tile_size), ty1 = fdiv(bb[3], tile_size);
        for (int64_t ty = ty0; ty <= ty1; ++ty)
            for (int64_t tx = tx0; tx <= tx1; ++tx) {
                int64_t tid = ty * n_tiles_x + tx;
                gauss_ids[cursor[tid]++] = g;
            }
    }
    free(cursor);
}

static inline int64_t i64max(int64_t a, int64_t b) { return a > b ? a : b; }
static inline int64_t i64min(int64_t a, int64_t b) { return a < b ? a : b; }

/* forward_tiles (_kernels.py:66-125): per tile, per listed Gaussian (ascending),
 * per row inside the cutoff ellipse, accumulate w * (exp(-q/2) - sub). */
void oracle_forward_tiles(double *pixels, int64_t D, const int64_t *gauss_ids,
                          const int64_t *tile_starts, int64_t n_tiles, int64_t n_tiles_x,
                          int64_t tile_size, const double *mean2, const double *prec,
                          const double *weight, const int64_t *bbox, double h, double c0,
                          double cutoff_sq, double sub) {
    for (int64_t tid = 0; tid < n_tiles; ++tid) {
        int64_t lo = tile_starts[tid], hi = tile_starts[tid + 1];
        if (lo == hi) continue;
        int64_t ty = tid / n_tiles_x, tx = tid % n_tiles_x;
        int64_t py0 = ty * tile_size, py1 = i64min(py0 + tile_size, D) - 1;
        int64_t px0 = tx * tile_size, px1 = i64min(px0 + tile_size, D) - 1;
        for (int64_t w = lo; w < hi; ++w) {
            int64_t g = gauss_ids[w];
            const int64_t *bb = bbox + 4 * g;
            int64_t x0 = i64max(bb[0], px0), x1 = i64min(bb[1], px1);
            int64_t y0 = i64max(bb[2], py0), y1 = i64min(bb[3], py1);
            if (x0 > x1 || y0 > y1) continue;
            double p00 = prec[3 * g], p01 = prec[3 * g + 1], p11 = prec[3 * g + 2];
            double mx = mean2[2 * g], my = mean2[2 * g + 1], wgt = weight[g];
            double mpx = mx / h + c0;
            for (int64_t iy = y0; iy <= y1; ++iy) {
                double dy = ((double)iy - c0) * h - my;
                double bh = p01 * dy;
                double disc = bh * bh - p00 * (p11 * dy * dy - cutoff_sq);
                if (disc <= 0.0) continue;
                double root = sqrt(disc);
                int64_t xa = i64max(x0, (int64_t)ceil((-bh - root) / (p00 * h) + mpx) - 1);
                int64_t xb = i64min(x1, (int64_t)floor((-bh + root) / (p00 * h) + mpx) + 1);
                for (int64_t ix = xa; ix <= xb; ++ix) {
                    double dx = ((double)ix - c0) * h - mx;
                    double q = p00 * dx * dx + 2.0 * p01 * dx * dy + p11 * dy * dy;
                    if (q < cutoff_sq) pixels[iy * D + ix] += wgt * (exp(-0.5 * q) - sub);
                }
            }
        }
    }
}

/* backward_pixels (_kernels.py:128-190): six raw sums per Gaussian over its
 * bbox with the forward's exact culling.  out is (n, 6), overwritten. */
void oracle_backward_pixels(const double *grad_pixels, int64_t D, int64_t n,
                            const double *mean2, const double *prec, const int64_t *bbox,
                            double h, double c0, double cutoff_sq, double sub, double *out) {
    for (int64_t g = 0; g < n; ++g) {
        const int64_t *bb = bbox + 4 * g;
        double *o = out + 6 * g;
        if (bb[0] > bb[1] || bb[2] > bb[3]) continue; /* reference leaves the row untouched */
        double p00 = prec[3 * g], p01 = prec[3 * g + 1], p11 = prec[3 * g + 2];
        double mx = mean2[2 * g], my = mean2[2 * g + 1];
        double mpx = mx / h + c0;
        double sA = 0.0, sx = 0.0, sy = 0.0, s00 = 0.0, s01 = 0.0, s11 = 0.0;
        for (int64_t iy = bb[2]; iy <= bb[3]; ++iy) {
            double dy = ((double)iy - c0) * h - my;
            double bh = p01 * dy;
            double disc = bh * bh - p00 * (p11 * dy * dy - cutoff_sq);
            if (disc <= 0.0) continue;
            double root = sqrt(disc);
            int64_t xa = i64max(bb[0], (int64_t)ceil((-bh - root) / (p00 * h) + mpx) - 1);
            int64_t xb = i64min(bb[1], (int64_t)floor((-bh + root) / (p00 * h) + mpx) + 1);
            for (int64_t ix = xa; ix <= xb; ++ix) {
                double dx = ((double)ix - c0) * h - mx;
                double q = p00 * dx * dx + 2.0 * p01 * dx * dy + p11 * dy * dy;
                if (q >= cutoff_sq) continue;
                double gp = grad_pixels[iy * D + ix];
                double e = exp(-0.5 * q);
                double v = e - sub;
                double pdx = p00 * dx + p01 * dy;
                double pdy = p01 * dx + p11 * dy;
                sA += gp * v;
                sx += gp * e * pdx;
                sy += gp * e * pdy;
                s00 += gp * (0.5 * e * pdx * pdx - 0.5 * v * p00);
                s01 += gp * (0.5 * e * pdx * pdy - 0.5 * v * p01);
                s11 += gp * (0.5 * e * pdy * pdy - 0.5 * v * p11);
            }
        }
        o[0] = sA; o[1] = sx; o[2] = sy; o[3] = s00; o[4] = s01; o[5] = s11;
    }
}

/* In-ellipse (image, Gaussian, pixel) pair count: the algorithmic work unit
 * of SURVEY.md section 8(d).  Same culling as backward_pixels. */
int64_t oracle_count_pairs(int64_t D, int64_t n, const double *mean2, const double *prec,
                           const int64_t *bbox, double h, double c0, double cutoff_sq) {
    int64_t total = 0;
    for (int64_t g = 0; g < n; ++g) {
        const int64_t *bb = bbox + 4 * g;
        if (bb[0] > bb[1] || bb[2] > bb[3]) continue;
        double p00 = prec[3 * g], p01 = prec[3 * g + 1], p11 = prec[3 * g + 2];
        double mx = mean2[2 * g], my = mean2[2 * g + 1];
        double mpx = mx / h + c0;
        for (int64_t iy = bb[2]; iy <= bb[3]; ++iy) {
            double dy = ((double)iy - c0) * h - my;
            double bh = p01 * dy;
            double disc = bh * bh - p00 * (p11 * dy * dy - cutoff_sq);
            if (disc <= 0.0) continue;
            double root = sqrt(disc);
            int64_t xa = i64max(bb[0], (int64_t)ceil((-bh - root) / (p00 * h) + mpx) - 1);
            int64_t xb = i64min(bb[1], (int64_t)floor((-bh + root) / (p00 * h) + mpx) + 1);
            for (int64_t ix = xa; ix <= xb; ++ix) {
                double dx = ((double)ix - c0) * h - mx;
                double q = p00 * dx * dx + 2.0 * p01 * dx * dy + p11 * dy * dy;
                total += (q < cutoff_sq);
            }
        }
    }
    return total;
}

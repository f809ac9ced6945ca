/*
 * tgv_synth.c -- seeded synthetic INPUT generator (shared by the oracle side
 * and the CUDA side as the only common code; holds none of the TGV method's
 * arithmetic: no operators, no prox, no projections, no energy).
 *
 * It produces per-voxel 8-bin vote histograms the way the paper builds its
 * data term:
 *   - analytic depth maps of sphere / plane / heightfield scenes, rendered by
 *     ray casting pinhole cameras (z-depth, reading R4), with
 *     optional Gaussian depth noise and "floater" outliers
 *     (SPEC.md:564 inject_outliers, depth x U(0.3, 0.9));
 *   - mipmap pyramids, level L+1 = mean of the valid children
 *     (§3.4; SPEC.md:66 build_pyramid);
 *   - Alg. 1: project the voxel centre, pick the pyramid
 *     level from the projected diameter, a = depth - distance,
 *     reject a < -eta, clamp a/delta to [-1,1], bin = floor((a+1)/2 * 8)
 *     clamped to 7, add the vote weight (1, or 5 for LIDAR).
 *     delta = 6 r, eta = 3 delta = 18 r, r = voxel radius.
 *
 * All randomness is a counter-based hash of (seed, camera, pixel, stream), so
 * every voxel's histogram depends only on its coordinates and the cameras:
 * slabs generated independently are identical to the same planes of the
 * monolithic grid.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define PRIM_SPHERE 0
#define PRIM_PLANE 1      /* horizontal ground plane z = a[0], seen from above */
#define PRIM_HEIGHTFIELD 2 /* z = a[0] + sum_{o<5} amp_o sin(kx_o x + ky_o y + phi_o) */
#define PRIM_BOX 3         /* axis-aligned box [a0, a3] x [a1, a4] x [a2, a5] (a building) */

typedef struct {
    int32_t kind;
    int32_t pad;
    double a[24];
} synth_prim;

typedef struct {
    double origin[3];
    double rot[9]; /* row-major world<-camera: world_dir = rot * cam_dir; columns = camera axes */
    double fx, fy, cx, cy;
    int32_t width, height;
    int32_t vote_weight;
    int32_t pad;
} synth_camera;

/* ---- counter-based RNG ------------------------------------------------- */
static inline uint64_t splitmix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
static inline double hash_uniform(uint64_t seed, uint64_t cam, uint64_t pix, uint64_t stream)
{
    uint64_t h = splitmix64(seed ^ splitmix64(cam * 0x100000001B3ull + stream));
    h = splitmix64(h ^ pix);
    return ((double)(h >> 11) + 0.5) * (1.0 / 9007199254740992.0); /* (0,1) */
}
static inline double hash_normal(uint64_t seed, uint64_t cam, uint64_t pix)
{
    double u1 = hash_uniform(seed, cam, pix, 1), u2 = hash_uniform(seed, cam, pix, 2);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

/* ---- ray casting ------------------------------------------------------- */
static double hf_height(const synth_prim* p, double x, double y)
{
    double z = p->a[0];
    for (int o = 0; o < 5; ++o)
        z += p->a[1 + 4 * o] * sin(p->a[2 + 4 * o] * x + p->a[3 + 4 * o] * y + p->a[4 + 4 * o]);
    return z;
}
/* returns ray parameter t > 0 of the first hit of o + t d, or INFINITY */
static double intersect(const synth_prim* p, const double o[3], const double d[3])
{
    if (p->kind == PRIM_SPHERE) {
        double oc[3] = {o[0] - p->a[0], o[1] - p->a[1], o[2] - p->a[2]};
        double A = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
        double B = 2.0 * (oc[0] * d[0] + oc[1] * d[1] + oc[2] * d[2]);
        double C = oc[0] * oc[0] + oc[1] * oc[1] + oc[2] * oc[2] - p->a[3] * p->a[3];
        double disc = B * B - 4.0 * A * C;
        if (disc < 0.0) return INFINITY;
        double sq = sqrt(disc);
        double t0 = (-B - sq) / (2.0 * A), t1 = (-B + sq) / (2.0 * A);
        if (t0 > 1e-9) return t0;
        if (t1 > 1e-9) return t1;
        return INFINITY;
    }
    if (p->kind == PRIM_PLANE) {
        if (d[2] >= 0.0) return INFINITY;
        double t = (p->a[0] - o[2]) / d[2];
        return t > 1e-9 ? t : INFINITY;
    }
    if (p->kind == PRIM_BOX) { /* slab test */
        double t0 = -INFINITY, t1 = INFINITY;
        for (int k = 0; k < 3; ++k) {
            if (d[k] == 0.0) {
                if (o[k] < p->a[k] || o[k] > p->a[3 + k]) return INFINITY;
                continue;
            }
            double ta = (p->a[k] - o[k]) / d[k], tb = (p->a[3 + k] - o[k]) / d[k];
            if (ta > tb) {
                double tt = ta;
                ta = tb;
                tb = tt;
            }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
        }
        if (t0 > t1) return INFINITY;
        if (t0 > 1e-9) return t0;
        if (t1 > 1e-9) return t1;
        return INFINITY;
    }
    if (p->kind == PRIM_HEIGHTFIELD) {
        /* a[21], a[22]: bounds zmin, zmax of the field; march then bisect */
        double zmin = p->a[21], zmax = p->a[22];
        double dl = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        double t = 0.0, tend;
        if (d[2] < 0.0) {
            if (o[2] > zmax) t = (zmax - o[2]) / d[2];
            tend = (zmin - o[2]) / d[2];
        } else {
            return INFINITY;
        }
        /* Lipschitz-bounded steps (a[23] bounds |grad H|): along the ray the height gap
         * f = z - H shrinks at most by (|d_z| + L |d_xy|) per unit t, so stepping by
         * f / that rate never jumps over the surface; the last bracket is bisected. */
        const double L = p->a[23] > 0.0 ? p->a[23] : 10.0;
        const double rate = fabs(d[2]) + L * sqrt(d[0] * d[0] + d[1] * d[1]);
        const double min_step = 0.05 / dl;
        double prev_t = t, prev_f = o[2] + t * d[2] - hf_height(p, o[0] + t * d[0], o[1] + t * d[1]);
        if (prev_f <= 0.0) return t > 1e-9 ? t : INFINITY;
        while (t <= tend) {
            double step = prev_f / rate;
            if (step < min_step) step = min_step;
            t += step;
            double f = o[2] + t * d[2] - hf_height(p, o[0] + t * d[0], o[1] + t * d[1]);
            if (f <= 0.0) {
                double lo = prev_t, hi = t;
                for (int it = 0; it < 24; ++it) {
                    double mid = 0.5 * (lo + hi);
                    double fm = o[2] + mid * d[2] - hf_height(p, o[0] + mid * d[0], o[1] + mid * d[1]);
                    if (fm > 0.0) lo = mid; else hi = mid;
                }
                return 0.5 * (lo + hi);
            }
            prev_t = t;
            prev_f = f;
        }
        (void)prev_f;
        return INFINITY;
    }
    return INFINITY;
}

/* Render the z-depth map of one camera (NaN = no surface). */
int synth_render(const synth_prim* prims, int nprims, const synth_camera* cam, int64_t cam_id,
                 uint64_t seed, double noise_sigma, double floater_frac, float* depth)
{
    const int W = cam->width, H = cam->height;
#pragma omp parallel for schedule(dynamic, 4)
    for (int py = 0; py < H; ++py)
        for (int px = 0; px < W; ++px) {
            /* camera-frame direction with unit z: the ray parameter IS the z-depth */
            double dc[3] = {(px + 0.5 - cam->cx) / cam->fx, (py + 0.5 - cam->cy) / cam->fy, 1.0};
            double dw[3];
            for (int r = 0; r < 3; ++r)
                dw[r] = cam->rot[3 * r + 0] * dc[0] + cam->rot[3 * r + 1] * dc[1] + cam->rot[3 * r + 2] * dc[2];
            double tbest = INFINITY;
            for (int i = 0; i < nprims; ++i) {
                double t = intersect(&prims[i], cam->origin, dw);
                if (t < tbest) tbest = t;
            }
            float out = NAN;
            if (isfinite(tbest)) {
                uint64_t pix = (uint64_t)py * (uint64_t)W + (uint64_t)px;
                double dd = tbest;
                if (noise_sigma > 0.0) dd += noise_sigma * hash_normal(seed, (uint64_t)cam_id, pix);
                if (floater_frac > 0.0 && hash_uniform(seed, (uint64_t)cam_id, pix, 3) < floater_frac)
                    dd *= 0.3 + 0.6 * hash_uniform(seed, (uint64_t)cam_id, pix, 4);
                if (dd > 0.0) out = (float)dd;
            }
            depth[(int64_t)py * W + px] = out;
        }
    return 0;
}

/* ---- pyramids ---------------------------------------------------------- */
typedef struct {
    int nlev;
    int w[32], h[32];
    float* lev[32];
} pyramid;

static void pyr_build(pyramid* P, const float* depth, int W, int H)
{
    int m = W > H ? W : H, n = 1;
    while ((1 << n) <= m) ++n; /* 1 + floor(log2(max(W,H))) */
    P->nlev = n;
    P->w[0] = W; P->h[0] = H;
    P->lev[0] = (float*)depth;
    for (int L = 1; L < n; ++L) {
        int w = (P->w[L - 1] + 1) / 2, h = (P->h[L - 1] + 1) / 2;
        P->w[L] = w; P->h[L] = h;
        P->lev[L] = (float*)malloc(sizeof(float) * (size_t)w * (size_t)h);
        const float* src = P->lev[L - 1];
        int sw = P->w[L - 1], sh = P->h[L - 1];
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x) {
                double s = 0.0;
                int c = 0;
                for (int dy = 0; dy < 2; ++dy)
                    for (int dx = 0; dx < 2; ++dx) {
                        int xx = 2 * x + dx, yy = 2 * y + dy;
                        if (xx < sw && yy < sh) {
                            float v = src[(int64_t)yy * sw + xx];
                            if (!isnan(v)) { s += v; ++c; }
                        }
                    }
                P->lev[L][(int64_t)y * w + x] = c ? (float)(s / c) : NAN;
            }
    }
}
static void pyr_free(pyramid* P)
{
    for (int L = 1; L < P->nlev; ++L) free(P->lev[L]);
}

/* ---- Alg. 1 ------------------------------------------------------------ */
/* One Alg. 1 vote: returns the bin (0..7) or -1 for no vote. */
int synth_alg1_bin(double depth, double distance, double r)
{
    const double delta = 6.0 * r, eta = 3.0 * delta;
    double a = depth - distance;
    if (a < -eta) return -1;
    a = a / delta;
    if (a < -1.0) a = -1.0;
    if (a > 1.0) a = 1.0;
    int bin = (int)floor((a + 1.0) / 2.0 * 8.0);
    return bin > 7 ? 7 : bin;
}

/* Vote every camera into the 8-bin histograms of the voxels of global planes
 * [z0, z1) of an nx x ny x nz grid.  Voxel (x,y,z) has its centre at the
 * point (x, y, z) and radius r.  counts: [z1-z0][ny][nx][8], zeroed here. */
/* The box [x0, x1) x [y0, y1) x [z0, z1) of the grid (a window: the same votes as the
 * full planes, cropped).  counts: [z1-z0][y1-y0][x1-x0][8], zeroed here. */
int synth_vote_box(const synth_camera* cams, int ncams, const float* const* depths, int64_t x0, int64_t x1,
                   int64_t y0, int64_t y1, int64_t z0, int64_t z1, double r, uint32_t* counts)
{
    const int NB = 8;
    const int64_t nx = x1 - x0, ny = y1 - y0;
    memset(counts, 0, sizeof(uint32_t) * (size_t)((z1 - z0) * ny * nx * NB));
    pyramid* pyr = (pyramid*)calloc((size_t)ncams, sizeof(pyramid));
    for (int c = 0; c < ncams; ++c) pyr_build(&pyr[c], depths[c], cams[c].width, cams[c].height);
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
    for (int64_t z = z0; z < z1; ++z)
        for (int64_t y = y0; y < y1; ++y)
            for (int64_t x = x0; x < x1; ++x) {
                uint32_t* hv = counts + (((z - z0) * ny + (y - y0)) * nx + (x - x0)) * NB;
                for (int c = 0; c < ncams; ++c) {
                    const synth_camera* C = &cams[c];
                    double dwp[3] = {x - C->origin[0], y - C->origin[1], z - C->origin[2]};
                    double pc[3]; /* camera frame = rot^T * (X - o) */
                    for (int k = 0; k < 3; ++k)
                        pc[k] = C->rot[0 * 3 + k] * dwp[0] + C->rot[1 * 3 + k] * dwp[1] + C->rot[2 * 3 + k] * dwp[2];
                    if (pc[2] <= 0.0) continue;
                    double u = C->fx * pc[0] / pc[2] + C->cx, v = C->fy * pc[1] / pc[2] + C->cy;
                    if (!(u >= 0.0 && u < C->width && v >= 0.0 && v < C->height)) continue;
                    /* level of detail from the projected diameter in level-0 pixels */
                    double diam = 2.0 * r * C->fx / pc[2];
                    int L = 0;
                    if (diam > 1.0) {
                        L = (int)floor(log2(diam) + 0.5);
                        if (L > pyr[c].nlev - 1) L = pyr[c].nlev - 1;
                    }
                    int ix = (int)floor(u / (double)(1 << L)), iy = (int)floor(v / (double)(1 << L));
                    if (ix >= pyr[c].w[L]) ix = pyr[c].w[L] - 1;
                    if (iy >= pyr[c].h[L]) iy = pyr[c].h[L] - 1;
                    float dep = pyr[c].lev[L][(int64_t)iy * pyr[c].w[L] + ix];
                    if (isnan(dep)) continue;                   /* depth = None */
                    int bin = synth_alg1_bin((double)dep, pc[2], r); /* a = depth - distance */
                    if (bin < 0) continue;                                /* occluded: no vote */
                    hv[bin] += (uint32_t)C->vote_weight;
                }
            }
    for (int c = 0; c < ncams; ++c) pyr_free(&pyr[c]);
    free(pyr);
    return 0;
}

int synth_vote(const synth_camera* cams, int ncams, const float* const* depths, int64_t nx, int64_t ny,
               int64_t z0, int64_t z1, double r, uint32_t* counts)
{
    return synth_vote_box(cams, ncams, depths, 0, nx, 0, ny, z0, z1, r, counts);
}


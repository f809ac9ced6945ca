/*
 * tgv_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, fp64, single-threaded-by-default CPU implementation of the
 * discrete TGV primal-dual scheme that the CUDA path computes.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library.  It shares no code, header, table or constant with
 * paper_2107_14790_b200/ (the product) and never includes include/tgv.h.
 *
 * What it follows (PAPER.md = /root/reference/PAPER.md, the paper's LaTeX):
 *   - Eq. 2 (§3.2): the TGV functional
 *         min_{u,v} sum alpha1 |grad u - v| + alpha0 |E(v)| + sum_i |u - f_i|
 *     with the data term written through the 8-bin histogram of §3.4
 *     (Alg. 1) as lambda sum_b h_b |u - c_b|
 *     (readings R1, R2, R3).
 *   - Eq. 3: E(v) = (grad v + grad v^T) / 2.
 *   - "we use the primal-dual method [pock2011tgv]": the
 *     Chambolle-Pock iteration
 *         p <- P_{alpha1}(p + sigma (grad ubar - vbar))
 *         q <- P_{alpha0}(q + sigma E(vbar))
 *         u+ <- clamp(prox_{tau lambda hist}(u + tau div p), -1, 1)
 *         v+ <- v + tau (p + div2 q)
 *         ubar <- 2 u+ - u,  vbar <- 2 v+ - v         (theta = 1)
 *     (readings R5-R9, R13).
 *   - the indicator range u in [-1, 1] (reading R8).
 *
 * Discrete operators (reading R6; forward/backward pair of
 * [bredies2010total]/[pock2011tgv], h = 1, Neumann boundary):
 *   D+_k w[l] = w[l+1] - w[l]   for l < n-1,   0 at l = n-1
 *   D-_k w[l] = wt[l] - wt[l-1] where wt[l] = w[l] for 0 <= l < n-1, else 0
 *   grad u = (D+_x u, D+_y u, D+_z u)
 *   E(v)_kl = 1/2 (D-_l v_k + D-_k v_l)
 *   div p = sum_k D-_k p_k               (= -grad^T p)
 *   (div2 q)_k = sum_l D+_l q_kl         (= -E^T q, Frobenius with both
 *                                           off-diagonal entries counted)
 *
 * Everything is computed in double precision with separate arrays per field
 * and Jacobi half-steps (each half-step reads only the previous half-step's
 * values).  An optional OpenMP z-loop (threads > 1) changes nothing in the
 * arithmetic, so results are bit-identical for any thread count.
 *
 * Slab mode: a state may own only global planes [zb, ze) of an nz-plane grid.
 * Its arrays then carry one halo plane below (global zb-1) and one above
 * (global ze); the caller fills them (tests/test_slab_gloo.py) and the
 * boundary rules above are applied with GLOBAL indices.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define NB_MAX 16

/* field ids (oracle's own numbering; the tests map them) */
enum { F_U = 0, F_V0 = 1, F_UBAR = 4, F_VBAR0 = 5, F_P0 = 8, F_Q0 = 11, F_COUNT = 17 };

/* symmetric tensor storage order xx, yy, zz, xy, xz, yz */
static const int QIDX[3][3] = {{0, 3, 4}, {3, 1, 5}, {4, 5, 2}};

typedef struct {
    int64_t nx, ny, nz;  /* global grid */
    int64_t zb, ze;      /* owned global planes [zb, ze) */
} grid_t;

typedef struct oracle_state {
    grid_t g;
    int nbins;
    double c[NB_MAX];
    double lambda, alpha0, alpha1, tau, sigma;
    double* f[F_COUNT]; /* each (ze-zb+2) planes of ny*nx, halo planes at both ends */
    double* h;          /* owned voxels x nbins (no halo) */
    int tvl1;           /* 1: TV-L1 model of Eq. 1 (v = q = 0 throughout), see oracle_set_tvl1 */
} oracle_state;

/* ---- indexing ---------------------------------------------------------- */
static inline int64_t idx(const grid_t* g, int64_t x, int64_t y, int64_t z)
{
    return ((z - g->zb + 1) * g->ny + y) * g->nx + x; /* z is GLOBAL, zb-1 <= z <= ze */
}
static inline int64_t hidx(const grid_t* g, int64_t x, int64_t y, int64_t z)
{
    return ((z - g->zb) * g->ny + y) * g->nx + x;
}
static inline int64_t n_local(const grid_t* g) { return (g->ze - g->zb + 2) * g->ny * g->nx; }

static inline int64_t coord(int axis, int64_t x, int64_t y, int64_t z)
{
    return axis == 0 ? x : (axis == 1 ? y : z);
}
static inline int64_t extent(const grid_t* g, int axis)
{
    return axis == 0 ? g->nx : (axis == 1 ? g->ny : g->nz);
}
static inline int64_t stride(const grid_t* g, int axis)
{
    return axis == 0 ? 1 : (axis == 1 ? g->nx : g->nx * g->ny);
}

/* ---- the two difference operators (reading R6) -------------------------- */
/* D+_k w at voxel (x,y,z): w[l+1] - w[l] if l < n-1, else 0. */
static double dplus(const grid_t* g, const double* w, int axis, int64_t x, int64_t y, int64_t z)
{
    int64_t l = coord(axis, x, y, z), n = extent(g, axis), i = idx(g, x, y, z);
    if (l < n - 1) return w[i + stride(g, axis)] - w[i];
    return 0.0;
}
/* D-_k w at voxel: wt[l] - wt[l-1] with wt[m] = w[m] for 0 <= m < n-1, else 0
 * (= -(D+_k)^T w: w[0] at l = 0, -w[n-2] at l = n-1, 0 if n = 1). */
static double dminus(const grid_t* g, const double* w, int axis, int64_t x, int64_t y, int64_t z)
{
    int64_t l = coord(axis, x, y, z), n = extent(g, axis), i = idx(g, x, y, z);
    double here = (l < n - 1) ? w[i] : 0.0;
    double below = (l > 0) ? w[i - stride(g, axis)] : 0.0;
    return here - below;
}

/* ---- operators at one voxel -------------------------------------------- */
static void grad_at(const grid_t* g, const double* u, int64_t x, int64_t y, int64_t z, double out[3])
{
    for (int k = 0; k < 3; ++k) out[k] = dplus(g, u, k, x, y, z);
}
/* E(v)_kl = 1/2 (D-_l v_k + D-_k v_l), Eq. 3 */
static void symgrad_at(const grid_t* g, double* const v[3], int64_t x, int64_t y, int64_t z,
                       double out[6])
{
    for (int k = 0; k < 3; ++k)
        for (int l = k; l < 3; ++l)
            out[QIDX[k][l]] = 0.5 * (dminus(g, v[k], l, x, y, z) + dminus(g, v[l], k, x, y, z));
}
/* div p = sum_k D-_k p_k */
static double div_at(const grid_t* g, double* const p[3], int64_t x, int64_t y, int64_t z)
{
    double s = 0.0;
    for (int k = 0; k < 3; ++k) s += dminus(g, p[k], k, x, y, z);
    return s;
}
/* (div2 q)_k = sum_l D+_l q_kl */
static void div2_at(const grid_t* g, double* const q[6], int64_t x, int64_t y, int64_t z, double out[3])
{
    for (int k = 0; k < 3; ++k) {
        double s = 0.0;
        for (int l = 0; l < 3; ++l) s += dplus(g, q[QIDX[k][l]], l, x, y, z);
        out[k] = s;
    }
}

/* ---- histogram data term ------------------------------------------------ */
/* G(u) = lambda * sum_b h_b |u - c_b|   (readings R1-R3) */
static double data_term(int nb, const double* h, const double* c, double lambda, double u)
{
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += h[b] * fabs(u - c[b]);
    return lambda * s;
}

/* prox: argmin_{u in [-1,1]} 1/2 (u - ut)^2 + t sum_b h_b |u - c_b|   (t = tau*lambda)
 * Plain definition: the objective is a convex quadratic on each interval
 * between consecutive bin centres (and the bounds -1, 1), so the minimiser is
 * the best of the per-interval minimisers.  On interval j (between c_{j-1} and
 * c_j) the derivative is  u - ut + t (sum_{b<j} h_b - sum_{b>=j} h_b), whose
 * root, clipped to the interval, is the interval's minimiser.  Clamping to
 * [-1, 1] is part of the interval bounds (reading R8). */
double oracle_prox(double ut, double t, int nb, const double* h, const double* c)
{
    double best_u = 0.0, best_f = INFINITY;
    for (int j = 0; j <= nb; ++j) {
        double lo = (j == 0) ? -1.0 : c[j - 1];
        double hi = (j == nb) ? 1.0 : c[j];
        if (lo < -1.0) lo = -1.0;
        if (hi > 1.0) hi = 1.0;
        if (lo > hi) continue;
        double below = 0.0, above = 0.0;
        for (int b = 0; b < j; ++b) below += h[b];
        for (int b = j; b < nb; ++b) above += h[b];
        double s = ut - t * (below - above);
        if (s < lo) s = lo;
        if (s > hi) s = hi;
        double f = 0.5 * (s - ut) * (s - ut);
        for (int b = 0; b < nb; ++b) f += t * h[b] * fabs(s - c[b]);
        if (f < best_f) {
            best_f = f;
            best_u = s;
        }
    }
    return best_u;
}

/* ---- state ------------------------------------------------------------- */
oracle_state* oracle_create(int64_t nx, int64_t ny, int64_t nz, int64_t zb, int64_t ze, int nbins,
                            const double* centers, double lambda, double alpha0, double alpha1,
                            double tau, double sigma)
{
    if (nx < 1 || ny < 1 || nz < 1 || zb < 0 || ze > nz || zb >= ze || nbins < 1 || nbins > NB_MAX)
        return NULL;
    oracle_state* s = (oracle_state*)calloc(1, sizeof(oracle_state));
    if (!s) return NULL;
    s->g.nx = nx; s->g.ny = ny; s->g.nz = nz; s->g.zb = zb; s->g.ze = ze;
    s->nbins = nbins;
    for (int b = 0; b < nbins; ++b) s->c[b] = centers[b];
    s->lambda = lambda; s->alpha0 = alpha0; s->alpha1 = alpha1; s->tau = tau; s->sigma = sigma;
    int64_t n = n_local(&s->g);
    for (int f = 0; f < F_COUNT; ++f) {
        s->f[f] = (double*)calloc((size_t)n, sizeof(double));
        if (!s->f[f]) return NULL;
    }
    s->h = (double*)calloc((size_t)((ze - zb) * ny * nx * nbins), sizeof(double));
    if (!s->h) return NULL;
    return s;
}

void oracle_destroy(oracle_state* s)
{
    if (!s) return;
    for (int f = 0; f < F_COUNT; ++f) free(s->f[f]);
    free(s->h);
    free(s);
}

/* counts: owned voxels [ze-zb][ny][nx][nbins].  Initialisation (reading R9):
 * u0 = sum_b h_b c_b / W (0 where W = 0), v0 = p0 = q0 = 0, ubar0 = u0, vbar0 = 0. */
void oracle_load(oracle_state* s, const uint32_t* counts)
{
    const grid_t* g = &s->g;
    for (int f = 0; f < F_COUNT; ++f) memset(s->f[f], 0, sizeof(double) * (size_t)n_local(g));
    for (int64_t z = g->zb; z < g->ze; ++z)
        for (int64_t y = 0; y < g->ny; ++y)
            for (int64_t x = 0; x < g->nx; ++x) {
                int64_t hv = hidx(g, x, y, z);
                double W = 0.0, m = 0.0;
                for (int b = 0; b < s->nbins; ++b) {
                    double hb = (double)counts[hv * s->nbins + b];
                    s->h[hv * s->nbins + b] = hb;
                    W += hb;
                    m += hb * s->c[b];
                }
                double u0 = (W > 0.0) ? m / W : 0.0;
                s->f[F_U][idx(g, x, y, z)] = u0;
                s->f[F_UBAR][idx(g, x, y, z)] = u0;
            }
}

/* NEXT-4: the TV-L1 functional of Eq. 1,
 *     min_u sum alpha1 |grad u| + lambda sum_b h_b |u - c_b|,
 * is the TGV scheme with v fixed at 0 and no q: p <- P_alpha1(p + sigma grad ubar),
 * u+ = clamp(prox(u + tau div p)).  (reading R21.) */
void oracle_set_tvl1(oracle_state* s, int on) { s->tvl1 = on ? 1 : 0; }

/* (a1) dual step: p <- P_alpha1(p + sigma(grad ubar - vbar)), q <- P_alpha0(q + sigma E(vbar)) */
void oracle_dual(oracle_state* s, int threads)
{
    const grid_t* g = &s->g;
    double* vbar[3] = {s->f[F_VBAR0], s->f[F_VBAR0 + 1], s->f[F_VBAR0 + 2]};
    double* p[3] = {s->f[F_P0], s->f[F_P0 + 1], s->f[F_P0 + 2]};
    double* q[6];
    for (int k = 0; k < 6; ++k) q[k] = s->f[F_Q0 + k];
    (void)threads;
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
    for (int64_t z = g->zb; z < g->ze; ++z)
        for (int64_t y = 0; y < g->ny; ++y)
            for (int64_t x = 0; x < g->nx; ++x) {
                int64_t i = idx(g, x, y, z);
                double gu[3], e[6], pn[3], qn[6];
                grad_at(g, s->f[F_UBAR], x, y, z, gu);
                /* TV-L1 (Eq. 1, reading R21) has no v: p + sigma grad ubar, v never read */
                for (int k = 0; k < 3; ++k) pn[k] = p[k][i] + s->sigma * (s->tvl1 ? gu[k] : gu[k] - vbar[k][i]);
                double np = sqrt(pn[0] * pn[0] + pn[1] * pn[1] + pn[2] * pn[2]);
                /* Euclidean projection onto {|p| <= alpha1} (reading R5) */
                double sp = (np > s->alpha1) ? s->alpha1 / np : 1.0;
                for (int k = 0; k < 3; ++k) p[k][i] = pn[k] * sp;
                if (s->tvl1) continue; /* TV-L1: no q (vbar stays 0) */

                symgrad_at(g, vbar, x, y, z, e);
                for (int m = 0; m < 6; ++m) qn[m] = q[m][i] + s->sigma * e[m];
                double nq2 = 0.0; /* Frobenius norm of the full symmetric 3x3 tensor */
                for (int k = 0; k < 3; ++k)
                    for (int l = 0; l < 3; ++l) nq2 += qn[QIDX[k][l]] * qn[QIDX[k][l]];
                double nq = sqrt(nq2);
                double sq = (nq > s->alpha0) ? s->alpha0 / nq : 1.0;
                for (int m = 0; m < 6; ++m) q[m][i] = qn[m] * sq;
            }
}

/* (a2)+(a3) primal step with theta = 1 over-relaxation */
void oracle_primal(oracle_state* s, int threads)
{
    const grid_t* g = &s->g;
    double* p[3] = {s->f[F_P0], s->f[F_P0 + 1], s->f[F_P0 + 2]};
    double* q[6];
    for (int k = 0; k < 6; ++k) q[k] = s->f[F_Q0 + k];
    const double t = s->tau * s->lambda;
    (void)threads;
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
    for (int64_t z = g->zb; z < g->ze; ++z)
        for (int64_t y = 0; y < g->ny; ++y)
            for (int64_t x = 0; x < g->nx; ++x) {
                int64_t i = idx(g, x, y, z);
                const double* hv = s->h + hidx(g, x, y, z) * s->nbins;
                double d = div_at(g, p, x, y, z);
                double uold = s->f[F_U][i];
                double unew = oracle_prox(uold + s->tau * d, t, s->nbins, hv, s->c);
                s->f[F_U][i] = unew;
                s->f[F_UBAR][i] = 2.0 * unew - uold;
                if (s->tvl1) continue; /* TV-L1: v stays 0 */
                double w[3];
                div2_at(g, q, x, y, z, w);
                for (int k = 0; k < 3; ++k) {
                    double vold = s->f[F_V0 + k][i];
                    double vnew = vold + s->tau * (p[k][i] + w[k]);
                    s->f[F_V0 + k][i] = vnew;
                    s->f[F_VBAR0 + k][i] = 2.0 * vnew - vold;
                }
            }
}

/* Slab mode, single-sweep multi-GPU plan: with the neighbours'
 * ubar, vbar and p (bottom halo plane zb-1) and ubar, vbar and q (top halo plane
 * ze) received, recompute the dual step ON the halo planes -- p at zb-1 and q at
 * ze, the only halo values the primal step reads -- instead of receiving them
 * after the dual.  The arithmetic is the per-voxel dual of oracle_dual. */
void oracle_dual_halo(oracle_state* s)
{
    const grid_t* g = &s->g;
    double* vbar[3] = {s->f[F_VBAR0], s->f[F_VBAR0 + 1], s->f[F_VBAR0 + 2]};
    double* p[3] = {s->f[F_P0], s->f[F_P0 + 1], s->f[F_P0 + 2]};
    double* q[6];
    for (int k = 0; k < 6; ++k) q[k] = s->f[F_Q0 + k];
    if (g->zb > 0) { /* p at plane zb-1 */
        const int64_t z = g->zb - 1;
        for (int64_t y = 0; y < g->ny; ++y)
            for (int64_t x = 0; x < g->nx; ++x) {
                int64_t i = idx(g, x, y, z);
                double gu[3], pn[3];
                grad_at(g, s->f[F_UBAR], x, y, z, gu);
                for (int k = 0; k < 3; ++k) pn[k] = p[k][i] + s->sigma * (s->tvl1 ? gu[k] : gu[k] - vbar[k][i]);
                double np = sqrt(pn[0] * pn[0] + pn[1] * pn[1] + pn[2] * pn[2]);
                double sp = (np > s->alpha1) ? s->alpha1 / np : 1.0;
                for (int k = 0; k < 3; ++k) p[k][i] = pn[k] * sp;
            }
    }
    if (g->ze < g->nz && !s->tvl1) { /* q at plane ze (TV-L1 has no q) */
        const int64_t z = g->ze;
        for (int64_t y = 0; y < g->ny; ++y)
            for (int64_t x = 0; x < g->nx; ++x) {
                int64_t i = idx(g, x, y, z);
                double e[6], qn[6];
                symgrad_at(g, vbar, x, y, z, e);
                for (int m = 0; m < 6; ++m) qn[m] = q[m][i] + s->sigma * e[m];
                double nq2 = 0.0;
                for (int k = 0; k < 3; ++k)
                    for (int l = 0; l < 3; ++l) nq2 += qn[QIDX[k][l]] * qn[QIDX[k][l]];
                double nq = sqrt(nq2);
                double sq = (nq > s->alpha0) ? s->alpha0 / nq : 1.0;
                for (int m = 0; m < 6; ++m) q[m][i] = qn[m] * sq;
            }
    }
}

void oracle_iterate(oracle_state* s, int n, int threads)
{
    for (int it = 0; it < n; ++it) {
        oracle_dual(s, threads);
        oracle_primal(s, threads);
    }
}

/* Energy of the current (u, v) and the box-restricted dual value D_V(p, q)
 * (reading R14):
 *   E   = sum alpha1 |grad u - v|_2 + alpha0 |E v|_F + lambda sum_b h_b |u - c_b|
 *   D_V = sum min_{u in [-1,1]} (lambda sum_b h_b|u - c_b| - u div p) - V |p + div2 q|_1
 * out = {E, alpha1-term, alpha0-term, data-term, gap = E - D_V, max|v|, D_V}.
 * TV-L1 (Eq. 1, reading R21): E = sum alpha1 |grad u| + data and D = D_0; v and q
 * are never read (V is ignored).
 * In slab mode only owned voxels contribute (halo planes must hold the
 * neighbours' u, v, p, q); the caller sums partial terms over slabs. */
void oracle_energy(const oracle_state* s, double V, double out[7])
{
    const grid_t* g = &s->g;
    double* v[3] = {s->f[F_V0], s->f[F_V0 + 1], s->f[F_V0 + 2]};
    double* p[3] = {s->f[F_P0], s->f[F_P0 + 1], s->f[F_P0 + 2]};
    double* q[6];
    for (int k = 0; k < 6; ++k) q[k] = s->f[F_Q0 + k];
    double t1 = 0.0, t0 = 0.0, td = 0.0, dv = 0.0, vmax = 0.0;
    for (int64_t z = g->zb; z < g->ze; ++z)
        for (int64_t y = 0; y < g->ny; ++y)
            for (int64_t x = 0; x < g->nx; ++x) {
                int64_t i = idx(g, x, y, z);
                const double* hv = s->h + hidx(g, x, y, z) * s->nbins;
                double u = s->f[F_U][i];
                double gu[3], e[6], w[3];
                grad_at(g, s->f[F_U], x, y, z, gu);
                double a = 0.0;
                if (s->tvl1) { /* Eq. 1 (reading R21): alpha1 |grad u| + data, no v, no q */
                    for (int k = 0; k < 3; ++k) a += gu[k] * gu[k];
                } else {
                    for (int k = 0; k < 3; ++k) a += (gu[k] - v[k][i]) * (gu[k] - v[k][i]);
                }
                t1 += s->alpha1 * sqrt(a);
                if (!s->tvl1) {
                    symgrad_at(g, v, x, y, z, e);
                    double b2 = 0.0;
                    for (int k = 0; k < 3; ++k)
                        for (int l = 0; l < 3; ++l) b2 += e[QIDX[k][l]] * e[QIDX[k][l]];
                    t0 += s->alpha0 * sqrt(b2);
                }
                td += data_term(s->nbins, hv, s->c, s->lambda, u);
                /* dual: the convex piecewise-linear min is attained at -1, 1 or a centre */
                double d = div_at(g, p, x, y, z);
                double best = INFINITY;
                for (int j = -1; j <= s->nbins; ++j) {
                    double uu = (j < 0) ? -1.0 : (j == s->nbins ? 1.0 : s->c[j]);
                    double f = data_term(s->nbins, hv, s->c, s->lambda, uu) - uu * d;
                    if (f < best) best = f;
                }
                if (s->tvl1) { /* no v to bound: the plain dual D_0 */
                    dv += best;
                    continue;
                }
                div2_at(g, q, x, y, z, w);
                double l1 = 0.0;
                for (int k = 0; k < 3; ++k) l1 += fabs(p[k][i] + w[k]);
                dv += best - V * l1;
                for (int k = 0; k < 3; ++k)
                    if (fabs(v[k][i]) > vmax) vmax = fabs(v[k][i]);
            }
    double E = t1 + t0 + td;
    out[0] = E; out[1] = t1; out[2] = t0; out[3] = td;
    out[4] = E - dv; out[5] = vmax; out[6] = dv;
}

/* ---- field access ------------------------------------------------------- */
/* owned planes of field f -> out[(ze-zb)*ny*nx] */
int oracle_get(const oracle_state* s, int f, double* out)
{
    if (f < 0 || f >= F_COUNT) return -1;
    const grid_t* g = &s->g;
    int64_t plane = g->nx * g->ny;
    memcpy(out, s->f[f] + plane, sizeof(double) * (size_t)(plane * (g->ze - g->zb)));
    return 0;
}
int oracle_set(oracle_state* s, int f, const double* in)
{
    if (f < 0 || f >= F_COUNT) return -1;
    const grid_t* g = &s->g;
    int64_t plane = g->nx * g->ny;
    memcpy(s->f[f] + plane, in, sizeof(double) * (size_t)(plane * (g->ze - g->zb)));
    return 0;
}
/* one plane (global z in [zb-1, ze], halos included) of field f */
int oracle_get_plane(const oracle_state* s, int f, int64_t z, double* out)
{
    const grid_t* g = &s->g;
    if (f < 0 || f >= F_COUNT || z < g->zb - 1 || z > g->ze) return -1;
    memcpy(out, s->f[f] + idx(g, 0, 0, z), sizeof(double) * (size_t)(g->nx * g->ny));
    return 0;
}
int oracle_set_plane(oracle_state* s, int f, int64_t z, const double* in)
{
    const grid_t* g = &s->g;
    if (f < 0 || f >= F_COUNT || z < g->zb - 1 || z > g->ze) return -1;
    memcpy(s->f[f] + idx(g, 0, 0, z), in, sizeof(double) * (size_t)(g->nx * g->ny));
    return 0;
}

/* ---- whole-grid operators for the pins (the same per-voxel code as above) */
static oracle_state* scratch(int64_t nx, int64_t ny, int64_t nz)
{
    double c = 0.0;
    return oracle_create(nx, ny, nz, 0, nz, 1, &c, 0, 0, 0, 0, 0);
}
/* u[N] -> g[3][N] */
int oracle_grad(int64_t nx, int64_t ny, int64_t nz, const double* u, double* out)
{
    oracle_state* s = scratch(nx, ny, nz);
    if (!s) return -1;
    int64_t N = nx * ny * nz;
    oracle_set(s, F_U, u);
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x) {
                double gu[3];
                grad_at(&s->g, s->f[F_U], x, y, z, gu);
                for (int k = 0; k < 3; ++k) out[k * N + (z * ny + y) * nx + x] = gu[k];
            }
    oracle_destroy(s);
    return 0;
}
/* p[3][N] -> div p [N] */
int oracle_div(int64_t nx, int64_t ny, int64_t nz, const double* p, double* out)
{
    oracle_state* s = scratch(nx, ny, nz);
    if (!s) return -1;
    int64_t N = nx * ny * nz;
    for (int k = 0; k < 3; ++k) oracle_set(s, F_P0 + k, p + k * N);
    double* pp[3] = {s->f[F_P0], s->f[F_P0 + 1], s->f[F_P0 + 2]};
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x) out[(z * ny + y) * nx + x] = div_at(&s->g, pp, x, y, z);
    oracle_destroy(s);
    return 0;
}
/* v[3][N] -> E(v) [6][N] (xx, yy, zz, xy, xz, yz) */
int oracle_symgrad(int64_t nx, int64_t ny, int64_t nz, const double* v, double* out)
{
    oracle_state* s = scratch(nx, ny, nz);
    if (!s) return -1;
    int64_t N = nx * ny * nz;
    for (int k = 0; k < 3; ++k) oracle_set(s, F_V0 + k, v + k * N);
    double* vv[3] = {s->f[F_V0], s->f[F_V0 + 1], s->f[F_V0 + 2]};
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x) {
                double e[6];
                symgrad_at(&s->g, vv, x, y, z, e);
                for (int m = 0; m < 6; ++m) out[m * N + (z * ny + y) * nx + x] = e[m];
            }
    oracle_destroy(s);
    return 0;
}
/* q[6][N] -> div2 q [3][N] */
int oracle_div2(int64_t nx, int64_t ny, int64_t nz, const double* q, double* out)
{
    oracle_state* s = scratch(nx, ny, nz);
    if (!s) return -1;
    int64_t N = nx * ny * nz;
    for (int m = 0; m < 6; ++m) oracle_set(s, F_Q0 + m, q + m * N);
    double* qq[6];
    for (int m = 0; m < 6; ++m) qq[m] = s->f[F_Q0 + m];
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x) {
                double w[3];
                div2_at(&s->g, qq, x, y, z, w);
                for (int k = 0; k < 3; ++k) out[k * N + (z * ny + y) * nx + x] = w[k];
            }
    oracle_destroy(s);
    return 0;
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ======================================================================== */
/* NEXT-2: histogram voting, Alg. 1 (§3.4 :236-250)       */
/* ======================================================================== */
/* A pinhole camera: world_dir = rot * cam_dir (row-major, columns = camera
 * axes), pixel (u, v) = (fx X/Z + cx, fy Y/Z + cy) for camera-frame (X, Y, Z);
 * depth maps hold the camera-frame z-depth, NaN = no depth (reading R4). */
typedef struct {
    double origin[3];
    double rot[9];
    double fx, fy, cx, cy;
    int32_t width, height;
    int32_t vote_weight;
    int32_t pad;
} oracle_camera;

/* Mipmap level L+1 = mean of the valid children of level L (ceil halves), NaN if
 * none ("depth map pyramids").  Returns the number
 * of levels, 1 + floor(log2(max(w, h))). */
static int pyramid(const float* d0, int w, int h, float** lev, int* lw, int* lh)
{
    int m = w > h ? w : h, n = 1;
    while ((1 << n) <= m) ++n;
    lev[0] = (float*)d0;
    lw[0] = w;
    lh[0] = h;
    for (int L = 1; L < n; ++L) {
        lw[L] = (lw[L - 1] + 1) / 2;
        lh[L] = (lh[L - 1] + 1) / 2;
        lev[L] = (float*)malloc(sizeof(float) * (size_t)lw[L] * (size_t)lh[L]);
        for (int y = 0; y < lh[L]; ++y)
            for (int x = 0; x < lw[L]; ++x) {
                double sum = 0.0;
                int cnt = 0;
                for (int dy = 0; dy < 2; ++dy)
                    for (int dx = 0; dx < 2; ++dx) {
                        int xx = 2 * x + dx, yy = 2 * y + dy;
                        if (xx < lw[L - 1] && yy < lh[L - 1]) {
                            float v = lev[L - 1][(int64_t)yy * lw[L - 1] + xx];
                            if (v == v) {
                                sum += (double)v;
                                ++cnt;
                            }
                        }
                    }
                lev[L][(int64_t)y * lw[L] + x] = cnt ? (float)(sum / (double)cnt) : NAN;
            }
    }
    return n;
}

/* Alg. 1 for every voxel of global planes [z0, z1) of an nx x ny grid and every
 * camera.  Voxel (x, y, z) has centre origin + voxel_size * (x, y, z) and radius r.
 *   project: camera-frame centre (X, Y, Z); Z <= 0 or pixel outside -> no vote
 *   level:   round(log2(projected diameter 2 r fx / Z)), ties up, clamped to the
 *            pyramid -- evaluated as the number of k >= 0 with diameter >= sqrt(2) 2^k
 *   depth:   the level's texel floor(u / 2^L), floor(v / 2^L); NaN -> no vote
 *   a = depth - Z; a < -eta -> no vote; a = clamp(a / delta, -1, 1);
 *   bin = min(floor((a + 1) / 2 * 8), 7); counts[bin] += vote_weight
 * with delta = 6 r, eta = 3 delta.  counts: uint32
 * [z1-z0][ny][nx][8], zeroed here. */
void oracle_alg1_vote(const oracle_camera* cams, int ncams, const float* const* depths, int64_t nx, int64_t ny,
                      int64_t z0, int64_t z1, const double origin[3], double voxel_size, double r, uint32_t* counts)
{
    const double delta = 6.0 * r, eta = 3.0 * delta;
    memset(counts, 0, sizeof(uint32_t) * (size_t)((z1 - z0) * ny * nx * 8));
    for (int c = 0; c < ncams; ++c) {
        const oracle_camera* C = &cams[c];
        float* lev[32];
        int lw[32], lh[32];
        const int nlev = pyramid(depths[c], C->width, C->height, lev, lw, lh);
#pragma omp parallel for schedule(static)
        for (int64_t z = z0; z < z1; ++z)
            for (int64_t y = 0; y < ny; ++y)
                for (int64_t x = 0; x < nx; ++x) {
                    const double pw[3] = {origin[0] + voxel_size * (double)x, origin[1] + voxel_size * (double)y,
                                          origin[2] + voxel_size * (double)z};
                    const double d[3] = {pw[0] - C->origin[0], pw[1] - C->origin[1], pw[2] - C->origin[2]};
                    double pc[3];
                    for (int k = 0; k < 3; ++k)
                        pc[k] = C->rot[0 * 3 + k] * d[0] + C->rot[1 * 3 + k] * d[1] + C->rot[2 * 3 + k] * d[2];
                    if (!(pc[2] > 0.0)) continue;
                    const double u = C->fx * pc[0] / pc[2] + C->cx, v = C->fy * pc[1] / pc[2] + C->cy;
                    if (!(u >= 0.0 && u < (double)C->width && v >= 0.0 && v < (double)C->height)) continue;
                    const double diam = 2.0 * r * C->fx / pc[2];
                    int L = 0;
                    double thr = 1.4142135623730951; /* sqrt(2) 2^k */
                    while (L < nlev - 1 && diam >= thr) {
                        ++L;
                        thr *= 2.0;
                    }
                    const double sc = (double)(1 << L);
                    int ix = (int)floor(u / sc), iy = (int)floor(v / sc);
                    if (ix > lw[L] - 1) ix = lw[L] - 1;
                    if (iy > lh[L] - 1) iy = lh[L] - 1;
                    const float dep = lev[L][(int64_t)iy * lw[L] + ix];
                    if (dep != dep) continue; /* depth = None */
                    double a = (double)dep - pc[2];
                    if (a < -eta) continue;
                    a = a / delta;
                    if (a < -1.0) a = -1.0;
                    if (a > 1.0) a = 1.0;
                    int bin = (int)floor((a + 1.0) / 2.0 * 8.0);
                    if (bin > 7) bin = 7;
                    counts[(((z - z0) * ny + y) * nx + x) * 8 + bin] += (uint32_t)C->vote_weight;
                }
        for (int L = 1; L < nlev; ++L) free(lev[L]);
    }
}

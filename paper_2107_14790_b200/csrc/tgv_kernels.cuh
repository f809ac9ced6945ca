// tgv_kernels.cuh -- sm_100a kernels of the TGV primal-dual hot path.
//
// Scheme (include/tgv.h):
//   dual    p <- P_a1(p + s(grad ubar - vbar)),   q <- P_a0(q + s E(vbar))
//   primal  u+ = clamp(prox(u + t div p), -1, 1), v+ = v + t(p + div2 q),
//           ubar = 2u+ - u, vbar = 2v+ - v       (over-relaxation fused)
// Difference operators (R6), l = coordinate, n = global extent:
//   D+ w[l] = w[l+1] - w[l] (l < n-1), 0 at l = n-1
//   D- w[l] = wt[l] - wt[l-1],  wt[m] = w[m] for 0 <= m < n-1 else 0
//
// Storage (DESIGN.md §4 "Data layout in HBM"): each of the 17 fp32 fields is
// an SoA array of (nzl + 2) planes (one halo plane below and above the slab)
// of ny rows of `px` floats (px = nx rounded up to 32 -> 128-B aligned rows).
// Histograms: 8 (or 16) u16 counts per voxel, one 16-B (or 2x16-B) vector per
// voxel, no halo.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tgvk {

enum : int { F_U = 0, F_V = 1, F_UBAR = 4, F_VBAR = 5, F_P = 8, F_Q = 11, NF = 17 };
// q components: xx=0 yy=1 zz=2 xy=3 xz=4 yz=5

struct Geo {
    int nx, ny, nzl;   // owned extent (x, y, local z)
    int nz, z0;        // global nz and global z of local plane 0
    int64_t px;        // row pitch (floats)
    int64_t plane;     // px * ny
    int64_t fs;        // field stride = (nzl + 2) * plane
};

struct Centers {
    float c[16];       // padded with +inf beyond nbins
};

struct StepParams {
    float sigma, tau, alpha1, alpha0, tl;  // tl = tau * lambda
};

// ---------------------------------------------------------------------------
// element access: field f, local (x, y, z), z in [-1, nzl]
__device__ __forceinline__ int64_t vidx(const Geo& g, int x, int y, int z)
{
    return (int64_t)(z + 1) * g.plane + (int64_t)y * g.px + x;
}

// exact weighted median of the histogram-L1 prox (DESIGN.md §5 "prox"):
//   s_j = ut + t (W - 2 C_j), C_j = sum_{b<j} h_b, c_nb = +inf
//   P = max_j min(s_j, c_j)   (s_j non-increasing, c_j increasing)
template <int SLOTS>
__device__ __forceinline__ float hist_prox(float ut, float t, const uint16_t* h, const Centers& C)
{
    float W = 0.f;
#pragma unroll
    for (int b = 0; b < SLOTS; ++b) W += (float)h[b];
    float r = W, P = -INFINITY;
#pragma unroll
    for (int j = 0; j < SLOTS; ++j) {
        P = fmaxf(P, fminf(fmaf(t, r, ut), C.c[j]));
        r -= 2.f * (float)h[j];
    }
    P = fmaxf(P, fmaf(t, r, ut));
    return fminf(fmaxf(P, -1.f), 1.f);
}

template <int SLOTS>
__device__ __forceinline__ void load_hist(const uint4* __restrict__ H, int64_t v, uint16_t h[SLOTS])
{
#pragma unroll
    for (int k = 0; k < SLOTS / 8; ++k) {
        uint4 w = __ldg(H + v * (SLOTS / 8) + k);
        uint32_t a[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            h[8 * k + 2 * m] = (uint16_t)(a[m] & 0xffffu);
            h[8 * k + 2 * m + 1] = (uint16_t)(a[m] >> 16);
        }
    }
}

// ---------------------------------------------------------------------------
// (a1) dual kernel, v1: one voxel per thread, neighbours through L1/L2.
__global__ void __launch_bounds__(256) dual_kernel(float* __restrict__ S, Geo g, StepParams sp)
{
    const int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y, z = blockIdx.z;
    if (x >= g.nx || y >= g.ny) return;
    const int zg = g.z0 + z;
    const int64_t i = vidx(g, x, y, z);
    const float* __restrict__ ub = S + F_UBAR * g.fs;
    const float* __restrict__ vb0 = S + (F_VBAR + 0) * g.fs;
    const float* __restrict__ vb1 = S + (F_VBAR + 1) * g.fs;
    const float* __restrict__ vb2 = S + (F_VBAR + 2) * g.fs;
    const bool xl = x < g.nx - 1, yl = y < g.ny - 1, zl = zg < g.nz - 1;
    const bool xf = x > 0, yf = y > 0, zf = zg > 0;
    const int64_t sx = 1, sy = g.px, sz = g.plane;

    const float u0 = ub[i];
    const float gx = xl ? ub[i + sx] - u0 : 0.f;
    const float gy = yl ? ub[i + sy] - u0 : 0.f;
    const float gz = zl ? ub[i + sz] - u0 : 0.f;
    const float vx = vb0[i], vy = vb1[i], vz = vb2[i];

    float* __restrict__ P0 = S + (F_P + 0) * g.fs;
    float* __restrict__ P1 = S + (F_P + 1) * g.fs;
    float* __restrict__ P2 = S + (F_P + 2) * g.fs;
    float p0 = fmaf(sp.sigma, gx - vx, P0[i]);
    float p1 = fmaf(sp.sigma, gy - vy, P1[i]);
    float p2 = fmaf(sp.sigma, gz - vz, P2[i]);
    const float sp_ = fminf(1.f, sp.alpha1 * rsqrtf(p0 * p0 + p1 * p1 + p2 * p2));
    P0[i] = p0 * sp_;
    P1[i] = p1 * sp_;
    P2[i] = p2 * sp_;

    // D- of each vbar component along each axis
    const float wx = xl ? 1.f : 0.f, wy = yl ? 1.f : 0.f, wz = zl ? 1.f : 0.f;
    auto dmx = [&](const float* w, float self) { return wx * self - (xf ? w[i - sx] : 0.f); };
    auto dmy = [&](const float* w, float self) { return wy * self - (yf ? w[i - sy] : 0.f); };
    auto dmz = [&](const float* w, float self) { return wz * self - (zf ? w[i - sz] : 0.f); };
    const float exx = dmx(vb0, vx), eyy = dmy(vb1, vy), ezz = dmz(vb2, vz);
    const float exy = 0.5f * (dmy(vb0, vx) + dmx(vb1, vy));
    const float exz = 0.5f * (dmz(vb0, vx) + dmx(vb2, vz));
    const float eyz = 0.5f * (dmz(vb1, vy) + dmy(vb2, vz));

    float* __restrict__ Q = S + F_Q * g.fs;
    float q[6];
    const float e[6] = {exx, eyy, ezz, exy, exz, eyz};
#pragma unroll
    for (int m = 0; m < 6; ++m) q[m] = fmaf(sp.sigma, e[m], Q[m * g.fs + i]);
    const float nq2 = q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + 2.f * (q[3] * q[3] + q[4] * q[4] + q[5] * q[5]);
    const float sq = fminf(1.f, sp.alpha0 * rsqrtf(nq2));
#pragma unroll
    for (int m = 0; m < 6; ++m) Q[m * g.fs + i] = q[m] * sq;
}

// (a2)+(a3) primal kernel, v1: one voxel per thread.
template <int SLOTS>
__global__ void __launch_bounds__(256)
    primal_kernel(float* __restrict__ S, const uint4* __restrict__ H, Geo g, StepParams sp, Centers C)
{
    const int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y, z = blockIdx.z;
    if (x >= g.nx || y >= g.ny) return;
    const int zg = g.z0 + z;
    const int64_t i = vidx(g, x, y, z);
    const bool xl = x < g.nx - 1, yl = y < g.ny - 1, zl = zg < g.nz - 1;
    const bool xf = x > 0, yf = y > 0, zf = zg > 0;
    const int64_t sx = 1, sy = g.px, sz = g.plane;
    const float* __restrict__ P0 = S + (F_P + 0) * g.fs;
    const float* __restrict__ P1 = S + (F_P + 1) * g.fs;
    const float* __restrict__ P2 = S + (F_P + 2) * g.fs;
    const float* __restrict__ Q = S + F_Q * g.fs;

    const float p0 = P0[i], p1 = P1[i], p2 = P2[i];
    // div p = sum_k D-_k p_k
    const float divp = ((xl ? p0 : 0.f) - (xf ? P0[i - sx] : 0.f)) + ((yl ? p1 : 0.f) - (yf ? P1[i - sy] : 0.f)) +
                       ((zl ? p2 : 0.f) - (zf ? P2[i - sz] : 0.f));
    float* __restrict__ U = S + F_U * g.fs;
    float* __restrict__ UB = S + F_UBAR * g.fs;
    const float uo = U[i];
    uint16_t h[SLOTS];
    load_hist<SLOTS>(H, (int64_t)z * g.plane + (int64_t)y * g.px + x, h);
    const float un = hist_prox<SLOTS>(fmaf(sp.tau, divp, uo), sp.tl, h, C);
    U[i] = un;
    UB[i] = 2.f * un - uo;

    // (div2 q)_k = sum_l D+_l q_kl
    const float* qxx = Q + 0 * g.fs;
    const float* qyy = Q + 1 * g.fs;
    const float* qzz = Q + 2 * g.fs;
    const float* qxy = Q + 3 * g.fs;
    const float* qxz = Q + 4 * g.fs;
    const float* qyz = Q + 5 * g.fs;
    const float cxx = qxx[i], cyy = qyy[i], czz = qzz[i], cxy = qxy[i], cxz = qxz[i], cyz = qyz[i];
    const float w0 = (xl ? qxx[i + sx] - cxx : 0.f) + (yl ? qxy[i + sy] - cxy : 0.f) + (zl ? qxz[i + sz] - cxz : 0.f);
    const float w1 = (xl ? qxy[i + sx] - cxy : 0.f) + (yl ? qyy[i + sy] - cyy : 0.f) + (zl ? qyz[i + sz] - cyz : 0.f);
    const float w2 = (xl ? qxz[i + sx] - cxz : 0.f) + (yl ? qyz[i + sy] - cyz : 0.f) + (zl ? qzz[i + sz] - czz : 0.f);
    float* __restrict__ V0 = S + (F_V + 0) * g.fs;
    float* __restrict__ V1 = S + (F_V + 1) * g.fs;
    float* __restrict__ V2 = S + (F_V + 2) * g.fs;
    float* __restrict__ VB0 = S + (F_VBAR + 0) * g.fs;
    float* __restrict__ VB1 = S + (F_VBAR + 1) * g.fs;
    float* __restrict__ VB2 = S + (F_VBAR + 2) * g.fs;
    const float vo0 = V0[i], vo1 = V1[i], vo2 = V2[i];
    const float vn0 = fmaf(sp.tau, p0 + w0, vo0);
    const float vn1 = fmaf(sp.tau, p1 + w1, vo1);
    const float vn2 = fmaf(sp.tau, p2 + w2, vo2);
    V0[i] = vn0;
    V1[i] = vn1;
    V2[i] = vn2;
    VB0[i] = 2.f * vn0 - vo0;
    VB1[i] = 2.f * vn1 - vo1;
    VB2[i] = 2.f * vn2 - vo2;
}

// ---------------------------------------------------------------------------
// load / reset
// counts chunk: dense uint32 [nzc][ny][nx][nbins] for local planes [zc0, zc0 + nzc)
template <int SLOTS>
__global__ void pack_counts_kernel(const uint32_t* __restrict__ src, int nzc, int zc0, Geo g, int nbins,
                                   uint16_t* __restrict__ H, unsigned int* __restrict__ maxc)
{
    const int64_t n = (int64_t)nzc * g.ny * g.nx;
    unsigned int m = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(v % g.nx);
        const int64_t r = v / g.nx;
        const int y = (int)(r % g.ny);
        const int z = (int)(r / g.ny) + zc0;
        uint16_t* dst = H + ((int64_t)z * g.plane + (int64_t)y * g.px + x) * SLOTS;
        for (int b = 0; b < SLOTS; ++b) {
            unsigned int c = b < nbins ? src[v * nbins + b] : 0u;
            m = max(m, c);
            dst[b] = (uint16_t)min(c, 65535u);
        }
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(maxc, m);
}

// u = sum h c / W (fp64, 0 where W = 0), ubar = u; all other fields are zeroed by the caller.
template <int SLOTS>
__global__ void init_state_kernel(float* __restrict__ S, const uint4* __restrict__ H, Geo g, Centers C)
{
    const int64_t n = (int64_t)g.nzl * g.ny * g.nx;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(v % g.nx);
        const int64_t r = v / g.nx;
        const int y = (int)(r % g.ny);
        const int z = (int)(r / g.ny);
        uint16_t h[SLOTS];
        load_hist<SLOTS>(H, (int64_t)z * g.plane + (int64_t)y * g.px + x, h);
        double W = 0.0, m = 0.0;
        for (int b = 0; b < SLOTS; ++b) {
            if (h[b]) {
                W += (double)h[b];
                m += (double)h[b] * (double)C.c[b];
            }
        }
        const float u0 = W > 0.0 ? (float)(m / W) : 0.f;
        const int64_t i = vidx(g, x, y, z);
        S[F_U * g.fs + i] = u0;
        S[F_UBAR * g.fs + i] = u0;
    }
}

// ---------------------------------------------------------------------------
// (a4) energy and restricted gap, fp64 per-voxel terms, deterministic reduction.
struct EnergyParams {
    double alpha1, alpha0, lambda, V;
    int nbins;
};

constexpr int EN_TERMS = 5;  // alpha1, alpha0, data, dual, vmax

__device__ __forceinline__ double warp_sum(double v)
{
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v)
{
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <int SLOTS>
__global__ void __launch_bounds__(256)
    energy_partial_kernel(const float* __restrict__ S, const uint4* __restrict__ H, Geo g, EnergyParams ep,
                          Centers C, double* __restrict__ partials)
{
    const int64_t n = (int64_t)g.nzl * g.ny * g.nx;
    double t1 = 0, t0 = 0, td = 0, dv = 0, vm = 0;
    const int64_t sx = 1, sy = g.px, sz = g.plane;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(v % g.nx);
        const int64_t r = v / g.nx;
        const int y = (int)(r % g.ny);
        const int z = (int)(r / g.ny);
        const int zg = g.z0 + z;
        const int64_t i = vidx(g, x, y, z);
        const bool xl = x < g.nx - 1, yl = y < g.ny - 1, zl = zg < g.nz - 1;
        const bool xf = x > 0, yf = y > 0, zf = zg > 0;
        auto F = [&](int f, int64_t off) { return (double)S[f * g.fs + i + off]; };
        auto dp = [&](int f, bool l, int64_t s) { return l ? F(f, s) - F(f, 0) : 0.0; };
        auto dm = [&](int f, bool l, bool fst, int64_t s) { return (l ? F(f, 0) : 0.0) - (fst ? F(f, -s) : 0.0); };
        const double u = F(F_U, 0);
        const double v0 = F(F_V, 0), v1 = F(F_V + 1, 0), v2 = F(F_V + 2, 0);
        const double a0 = dp(F_U, xl, sx) - v0, a1 = dp(F_U, yl, sy) - v1, a2 = dp(F_U, zl, sz) - v2;
        t1 += ep.alpha1 * sqrt(a0 * a0 + a1 * a1 + a2 * a2);
        const double exx = dm(F_V, xl, xf, sx), eyy = dm(F_V + 1, yl, yf, sy), ezz = dm(F_V + 2, zl, zf, sz);
        const double exy = 0.5 * (dm(F_V, yl, yf, sy) + dm(F_V + 1, xl, xf, sx));
        const double exz = 0.5 * (dm(F_V, zl, zf, sz) + dm(F_V + 2, xl, xf, sx));
        const double eyz = 0.5 * (dm(F_V + 1, zl, zf, sz) + dm(F_V + 2, yl, yf, sy));
        t0 += ep.alpha0 * sqrt(exx * exx + eyy * eyy + ezz * ezz + 2.0 * (exy * exy + exz * exz + eyz * eyz));
        uint16_t h[SLOTS];
        load_hist<SLOTS>(H, (int64_t)z * g.plane + (int64_t)y * g.px + x, h);
        double dterm = 0.0;
        for (int b = 0; b < ep.nbins; ++b) dterm += (double)h[b] * fabs(u - (double)C.c[b]);
        td += ep.lambda * dterm;
        const double divp = dm(F_P, xl, xf, sx) + dm(F_P + 1, yl, yf, sy) + dm(F_P + 2, zl, zf, sz);
        double best = INFINITY;
        for (int j = -1; j <= ep.nbins; ++j) {
            const double uu = j < 0 ? -1.0 : (j == ep.nbins ? 1.0 : (double)C.c[j]);
            double s = 0.0;
            for (int b = 0; b < ep.nbins; ++b) s += (double)h[b] * fabs(uu - (double)C.c[b]);
            best = fmin(best, ep.lambda * s - uu * divp);
        }
        const int qb = F_Q;  // xx yy zz xy xz yz
        const double w0 = dp(qb + 0, xl, sx) + dp(qb + 3, yl, sy) + dp(qb + 4, zl, sz);
        const double w1 = dp(qb + 3, xl, sx) + dp(qb + 1, yl, sy) + dp(qb + 5, zl, sz);
        const double w2 = dp(qb + 4, xl, sx) + dp(qb + 5, yl, sy) + dp(qb + 2, zl, sz);
        const double l1 = fabs(F(F_P, 0) + w0) + fabs(F(F_P + 1, 0) + w1) + fabs(F(F_P + 2, 0) + w2);
        dv += best - ep.V * l1;
        vm = fmax(vm, fmax(fabs(v0), fmax(fabs(v1), fabs(v2))));
    }
    __shared__ double red[EN_TERMS][8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    t1 = warp_sum(t1);
    t0 = warp_sum(t0);
    td = warp_sum(td);
    dv = warp_sum(dv);
    vm = warp_max(vm);
    if (lane == 0) {
        red[0][wid] = t1;
        red[1][wid] = t0;
        red[2][wid] = td;
        red[3][wid] = dv;
        red[4][wid] = vm;
    }
    __syncthreads();
    if (threadIdx.x < EN_TERMS) {
        const int k = threadIdx.x;
        const int nw = blockDim.x >> 5;
        double s = red[k][0];
        for (int w = 1; w < nw; ++w) s = (k == 4) ? fmax(s, red[k][w]) : s + red[k][w];
        partials[(int64_t)blockIdx.x * EN_TERMS + k] = s;
    }
}

// one block: fixed-order sum of the block partials -> out[EN_TERMS]
__global__ void energy_final_kernel(const double* __restrict__ partials, int nblocks, double* __restrict__ out)
{
    __shared__ double red[EN_TERMS][256];
    for (int k = 0; k < EN_TERMS; ++k) {
        double s = 0.0;
        for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
            const double x = partials[(int64_t)b * EN_TERMS + k];
            s = (k == 4) ? fmax(s, x) : s + x;
        }
        red[k][threadIdx.x] = s;
    }
    __syncthreads();
    if (threadIdx.x < EN_TERMS) {
        const int k = threadIdx.x;
        double s = red[k][0];
        for (int t = 1; t < (int)blockDim.x; ++t) s = (k == 4) ? fmax(s, red[k][t]) : s + red[k][t];
        out[k] = s;
    }
}

}  // namespace tgvk

// tgv_kernels.cuh -- sm_100a kernels of the TGV primal-dual hot path.
//
// Scheme (include/tgv.h), iteration k:
//   ubar_k = 2 u_k - u_{k-1},  vbar_k = 2 v_k - v_{k-1}            (a3, theta = 1)
//   p_{k+1} = P_a1(p_k + s(grad ubar_k - vbar_k)),  q_{k+1} = P_a0(q_k + s E(vbar_k))   (a1)
//   u_{k+1} = clamp(prox(u_k + t div p_{k+1}), -1, 1),  v_{k+1} = v_k + t(p_{k+1} + div2 q_{k+1})  (a2)
// The over-relaxed iterate is formed on the fly from (u_k, u_{k-1}); storing the
// previous iterate instead of ubar lets the single-sweep kernel write only
// u, v, p, q (136 B per voxel-iteration, SURVEY.md §8(d) "method minimum").
//
// Difference operators (R6), l = coordinate along the axis, n = global extent:
//   D+ w[l] = w[l+1] - w[l] (l < n-1), 0 at l = n-1
//   D- w[l] = wt[l] - wt[l-1],  wt[m] = w[m] for 0 <= m < n-1 else 0
//   grad = D+,  E(v)_kl = (D-_l v_k + D-_k v_l)/2,  div p = sum_k D-_k p_k,
//   (div2 q)_k = sum_l D+_l q_kl
//
// Storage: every field is an fp32 array of (nzl + 2) planes (one
// halo plane below and above the slab) of ny rows of px floats (px = nx rounded
// up to 32: 128-B aligned rows).  Element offsets within a field fit in int32.
// Histograms: 8 (or 16) counts per voxel, u8 when every count <= 255 else u16,
// one vector load per voxel, no halo planes.
#pragma once
#include <type_traits>
#include <cstdint>
#include <cuda_runtime.h>

namespace tgvk {

struct Geo {
    int nx, ny, nzl;  // owned extent (x, y, local z)
    int nz, z0;       // global nz and global z of local plane 0
    int px;           // row pitch (floats)
    int plane;        // px * ny
    int64_t fs;       // field stride = (nzl + 2) * plane (< 2^31)
};

struct Centers {
    float c[16];  // padded with +inf beyond nbins
};

struct StepParams {
    float sigma, tau, alpha1, alpha0, tl;  // tl = tau * lambda
};

constexpr unsigned FULL = 0xffffffffu;

// element offset of local voxel (x, y, z), z in [-1, nzl]
__device__ __forceinline__ int eoff(const Geo& g, int x, int y, int z) { return (z + 1) * g.plane + y * g.px + x; }

// ---------------------------------------------------------------------------
// histograms: raw vector per voxel and exact count extraction
template <int SLOTS, typename CT>
struct HistRaw {
    static constexpr int NW = SLOTS * (int)sizeof(CT) / 4;  // 32-bit words
    uint32_t w[NW];
};

template <int SLOTS, typename CT>
__device__ __forceinline__ HistRaw<SLOTS, CT> load_hist(const void* __restrict__ H, int64_t v)
{
    HistRaw<SLOTS, CT> r;
    constexpr int NW = HistRaw<SLOTS, CT>::NW;
    if constexpr (NW == 2) {
        uint2 a = __ldg(reinterpret_cast<const uint2*>(H) + v);
        r.w[0] = a.x;
        r.w[1] = a.y;
    } else {
#pragma unroll
        for (int k = 0; k < NW / 4; ++k) {
            uint4 a = __ldg(reinterpret_cast<const uint4*>(H) + v * (NW / 4) + k);
            r.w[4 * k] = a.x;
            r.w[4 * k + 1] = a.y;
            r.w[4 * k + 2] = a.z;
            r.w[4 * k + 3] = a.w;
        }
    }
    return r;
}

// count b as an exact float: place the byte(s) in the mantissa of 2^23 and subtract 2^23
template <int SLOTS, typename CT>
__device__ __forceinline__ float hist_count(const HistRaw<SLOTS, CT>& h, int b)
{
    uint32_t bits;
    if constexpr (sizeof(CT) == 1)
        bits = __byte_perm(h.w[b >> 2], 0x4B000000u, (b & 3) | 0x4 << 4 | 0x4 << 8 | 0x7 << 12);
    else
        bits = __byte_perm(h.w[b >> 1], 0x4B000000u, (2 * (b & 1)) | (2 * (b & 1) + 1) << 4 | 0x4 << 8 | 0x7 << 12);
    return __uint_as_float(bits) - 8388608.0f;
}

// Exact histogram-L1 prox, clamped to [-1, 1] (DESIGN.md §5 "prox"):
//   r_j = W - 2 C_j (C_j = sum_{b<j} h_b, exact in fp32), s_j = ut + t r_j,
//   P = max_j min(s_j, c_j) with c_nb = +inf   (s_j non-increasing, c_j increasing)
template <int SLOTS, typename CT>
__device__ __forceinline__ float hist_prox(float ut, float t, const HistRaw<SLOTS, CT>& h, const Centers& C)
{
    float cnt[SLOTS];
    float W = 0.f;
#pragma unroll
    for (int b = 0; b < SLOTS; ++b) cnt[b] = hist_count<SLOTS, CT>(h, b);
    if constexpr (sizeof(CT) == 1) {  // byte sums in the integer pipe (exact), then the same magic conversion
        unsigned int wsum = 0;
#pragma unroll
        for (int k = 0; k < SLOTS / 4; ++k) wsum = __dp4a(h.w[k], 0x01010101u, wsum);
        W = __uint_as_float(0x4B000000u | wsum) - 8388608.0f;  // W <= 16 * 255 < 2^23
    } else {
#pragma unroll
        for (int b = 0; b < SLOTS; ++b) W += cnt[b];
    }
    float r = W, P = -INFINITY;
#pragma unroll
    for (int j = 0; j < SLOTS; ++j) {
        P = fmaxf(P, fminf(fmaf(t, r, ut), C.c[j]));
        r = fmaf(-2.f, cnt[j], r);
    }
    P = fmaxf(P, fmaf(t, r, ut));
    return fminf(fmaxf(P, -1.f), 1.f);
}

// Euclidean projection factor onto the ball of radius a for squared norm n2:
// min(1, a / |x|)  (n2 = 0 -> 1; a = 0 -> 0 unless n2 = 0)
// (rsqrt.approx.ftz: one MUFU; a squared norm below 2^-126 counts as 0 -> factor 1)
__device__ __forceinline__ float proj_scale(float n2, float a)
{
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(n2));
    return fminf(1.f, a * r);
}

// ---------------------------------------------------------------------------
// Field pointers of one iteration (host fills them from the rotating buffers)
struct IterPtrs {
    const float* uk;     // u_k
    const float* um;     // u_{k-1}
    const float* vk[3];  // v_k
    const float* vm[3];  // v_{k-1}
    const float* pk[3];  // p_k
    const float* qk[6];  // q_k  (xx, yy, zz, xy, xz, yz)
    float* un;           // u_{k+1}
    float* vn[3];        // v_{k+1}
    float* pn[3];        // p_{k+1}
    float* qn[6];        // q_{k+1}
    const void* hist;
};

// ===========================================================================
// SPLIT schedule: (1) dual kernel, (2) primal kernel with fused over-relaxation
// bookkeeping.  One voxel per thread, neighbours through L1/L2, all loads issued
// before any store.  88+16 B and 68+hist B per voxel.
// ===========================================================================
__global__ void __launch_bounds__(256) split_dual_kernel(const IterPtrs a, const Geo g, const StepParams sp)
{
    const int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y, z = blockIdx.z;
    if (x >= g.nx || y >= g.ny) return;
    const int zg = g.z0 + z;
    const int i = eoff(g, x, y, z);
    const bool xl = x < g.nx - 1, yl = y < g.ny - 1, zl = zg < g.nz - 1;
    const bool xf = x > 0, yf = y > 0, zf = zg > 0;
    const int sy = g.px, sz = g.plane;
    auto ubar = [&](int o) { return fmaf(2.f, __ldg(a.uk + o), -__ldg(a.um + o)); };
    auto vbar = [&](int k, int o) { return fmaf(2.f, __ldg(a.vk[k] + o), -__ldg(a.vm[k] + o)); };
    // ---- loads
    const float u0 = ubar(i);
    const float ux = xl ? ubar(i + 1) : 0.f, uy = yl ? ubar(i + sy) : 0.f, uz = zl ? ubar(i + sz) : 0.f;
    float vb[3], vbx[3], vby[3], vbz[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        vb[k] = vbar(k, i);
        vbx[k] = xf ? vbar(k, i - 1) : 0.f;
        vby[k] = yf ? vbar(k, i - sy) : 0.f;
        vbz[k] = zf ? vbar(k, i - sz) : 0.f;
    }
    float p[3], q[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) p[k] = __ldg(a.pk[k] + i);
#pragma unroll
    for (int m = 0; m < 6; ++m) q[m] = __ldg(a.qk[m] + i);
    // ---- p
    const float g0 = xl ? ux - u0 : 0.f, g1 = yl ? uy - u0 : 0.f, g2 = zl ? uz - u0 : 0.f;
    p[0] = fmaf(sp.sigma, g0 - vb[0], p[0]);
    p[1] = fmaf(sp.sigma, g1 - vb[1], p[1]);
    p[2] = fmaf(sp.sigma, g2 - vb[2], p[2]);
    const float sp_ = proj_scale(p[0] * p[0] + p[1] * p[1] + p[2] * p[2], sp.alpha1);
    // ---- q: D-_x vb_k = (xl ? vb_k : 0) - vbx_k, etc.
    float dx[3], dy[3], dz[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        dx[k] = fmaf(xl ? 1.f : 0.f, vb[k], -vbx[k]);
        dy[k] = fmaf(yl ? 1.f : 0.f, vb[k], -vby[k]);
        dz[k] = fmaf(zl ? 1.f : 0.f, vb[k], -vbz[k]);
    }
    const float e[6] = {dx[0], dy[1], dz[2], 0.5f * (dy[0] + dx[1]), 0.5f * (dz[0] + dx[2]), 0.5f * (dz[1] + dy[2])};
#pragma unroll
    for (int m = 0; m < 6; ++m) q[m] = fmaf(sp.sigma, e[m], q[m]);
    const float sq = proj_scale(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + 2.f * (q[3] * q[3] + q[4] * q[4] + q[5] * q[5]),
                                sp.alpha0);
#pragma unroll
    for (int k = 0; k < 3; ++k) a.pn[k][i] = p[k] * sp_;
#pragma unroll
    for (int m = 0; m < 6; ++m) a.qn[m][i] = q[m] * sq;
}

// reads p_{k+1}, q_{k+1} (in a.pk / a.qk), u_k, v_k; writes u_{k+1}, v_{k+1}
template <int SLOTS, typename CT>
__global__ void __launch_bounds__(256) split_primal_kernel(const IterPtrs a, const Geo g, const StepParams sp,
                                                           const Centers C)
{
    const int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y, z = blockIdx.z;
    if (x >= g.nx || y >= g.ny) return;
    const int zg = g.z0 + z;
    const int i = eoff(g, x, y, z);
    const bool xl = x < g.nx - 1, yl = y < g.ny - 1, zl = zg < g.nz - 1;
    const bool xf = x > 0, yf = y > 0, zf = zg > 0;
    const int sy = g.px, sz = g.plane;
    // ---- loads
    float p[3], q[6], qx[3], qy[3], qz[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) p[k] = __ldg(a.pk[k] + i);
    const float pxm = xf ? __ldg(a.pk[0] + i - 1) : 0.f;
    const float pym = yf ? __ldg(a.pk[1] + i - sy) : 0.f;
    const float pzm = zf ? __ldg(a.pk[2] + i - sz) : 0.f;
#pragma unroll
    for (int m = 0; m < 6; ++m) q[m] = __ldg(a.qk[m] + i);
    // q_kl at +e_l:  x: xx, xy, xz   y: xy, yy, yz   z: xz, yz, zz
    const int QX[3] = {0, 3, 4}, QY[3] = {3, 1, 5}, QZ[3] = {4, 5, 2};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        qx[k] = xl ? __ldg(a.qk[QX[k]] + i + 1) : 0.f;
        qy[k] = yl ? __ldg(a.qk[QY[k]] + i + sy) : 0.f;
        qz[k] = zl ? __ldg(a.qk[QZ[k]] + i + sz) : 0.f;
    }
    const float uo = __ldg(a.uk + i);
    float vo[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) vo[k] = __ldg(a.vk[k] + i);
    const auto h = load_hist<SLOTS, CT>(a.hist, (int64_t)z * g.plane + y * g.px + x);
    // ---- u
    const float divp = fmaf(xl ? 1.f : 0.f, p[0], -pxm) + fmaf(yl ? 1.f : 0.f, p[1], -pym) +
                       fmaf(zl ? 1.f : 0.f, p[2], -pzm);
    const float un = hist_prox<SLOTS, CT>(fmaf(sp.tau, divp, uo), sp.tl, h, C);
    // ---- v: (div2 q)_k = sum_l D+_l q_kl
    float w[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
        w[k] = (xl ? qx[k] - q[QX[k]] : 0.f) + (yl ? qy[k] - q[QY[k]] : 0.f) + (zl ? qz[k] - q[QZ[k]] : 0.f);
    a.un[i] = un;
#pragma unroll
    for (int k = 0; k < 3; ++k) a.vn[k][i] = fmaf(sp.tau, p[k] + w[k], vo[k]);
}

// ===========================================================================
// NEXT-4 TV-L1 model (Eq. 1; R21): v = q = 0,
//   p_{k+1} = P_a1(p_k + s grad ubar_k),  u_{k+1} = clamp(prox(u_k + t div p_{k+1}), -1, 1)
// dual: reads u_k, u_{k-1}, p (5 floats), writes p (3): 32 B per voxel
// primal: reads p (3), u_k (1) + counts, writes u: 20 B + counts
// ===========================================================================
__global__ void __launch_bounds__(256) tvl1_dual_kernel(const IterPtrs a, const Geo g, const StepParams sp)
{
    const int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y, z = blockIdx.z;
    if (x >= g.nx || y >= g.ny) return;
    const int zg = g.z0 + z;
    const int i = eoff(g, x, y, z);
    const bool xl = x < g.nx - 1, yl = y < g.ny - 1, zl = zg < g.nz - 1;
    const int sy = g.px, sz = g.plane;
    auto ubar = [&](int o) { return fmaf(2.f, __ldg(a.uk + o), -__ldg(a.um + o)); };
    const float u0 = ubar(i);
    const float ux = xl ? ubar(i + 1) : 0.f, uy = yl ? ubar(i + sy) : 0.f, uz = zl ? ubar(i + sz) : 0.f;
    float p[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) p[k] = __ldg(a.pk[k] + i);
    const float g0 = xl ? ux - u0 : 0.f, g1 = yl ? uy - u0 : 0.f, g2 = zl ? uz - u0 : 0.f;
    p[0] = fmaf(sp.sigma, g0, p[0]);
    p[1] = fmaf(sp.sigma, g1, p[1]);
    p[2] = fmaf(sp.sigma, g2, p[2]);
    const float f = proj_scale(p[0] * p[0] + p[1] * p[1] + p[2] * p[2], sp.alpha1);
#pragma unroll
    for (int k = 0; k < 3; ++k) a.pn[k][i] = p[k] * f;
}

// reads p_{k+1} (in a.pk), u_k; writes u_{k+1}
template <int SLOTS, typename CT>
__global__ void __launch_bounds__(256) tvl1_primal_kernel(const IterPtrs a, const Geo g, const StepParams sp,
                                                          const Centers C)
{
    const int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y, z = blockIdx.z;
    if (x >= g.nx || y >= g.ny) return;
    const int zg = g.z0 + z;
    const int i = eoff(g, x, y, z);
    const bool xl = x < g.nx - 1, yl = y < g.ny - 1, zl = zg < g.nz - 1;
    const bool xf = x > 0, yf = y > 0, zf = zg > 0;
    const int sy = g.px, sz = g.plane;
    float p[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) p[k] = __ldg(a.pk[k] + i);
    const float pxm = xf ? __ldg(a.pk[0] + i - 1) : 0.f;
    const float pym = yf ? __ldg(a.pk[1] + i - sy) : 0.f;
    const float pzm = zf ? __ldg(a.pk[2] + i - sz) : 0.f;
    const float uo = __ldg(a.uk + i);
    const auto h = load_hist<SLOTS, CT>(a.hist, (int64_t)z * g.plane + y * g.px + x);
    const float divp = ((xl ? p[0] : 0.f) - pxm) + ((yl ? p[1] : 0.f) - pym) + ((zl ? p[2] : 0.f) - pzm);
    a.un[i] = hist_prox<SLOTS, CT>(fmaf(sp.tau, divp, uo), sp.tl, h, C);
}

// ===========================================================================
// FUSED schedule: one single-sweep kernel per iteration (136 B per voxel-iteration
// with u16 counts, 128 B with u8).
//
// CTA = 32 lanes x (TY + 2) rows of threads, one (x, y) column per thread,
// marching up a z-chunk [zs, ze).  A warp covers 32 consecutive x of which
// lanes 1..30 are owned and lanes 0 / 31 are the x-halo; rows 1..TY are owned,
// row 0 (y0-1) and row TY+1 (y0+TY) are the y-halo.  Halos are recomputed
// redundantly so that no CTA ever needs another CTA's results of the same
// launch; the inputs are (u_k, u_{k-1}, v_k, v_{k-1}, p_k, q_k) and every output
// goes to a different buffer (U/V rotate over 3, P/Q over 2), so there is no
// intra-launch hazard.  Step s computes the dual D(s) (p, q at plane s) and the
// primal Pm(s-1); x-neighbours come from warp shuffles, y-neighbours from two
// parity-double-buffered shared planes (one __syncthreads per step), z-neighbours
// from registers.  Inputs are prefetched one plane ahead.
// ===========================================================================
struct FusedArgs {
    IterPtrs a;
    Geo g;
    StepParams sp;
    Centers C;
    int z_lo, z_hi, zc;  // local planes [z_lo, z_hi) in chunks of zc, one chunk per blockIdx.z
    int keep_halo_dual;  // NEXT-3 leaves: also store p at plane -1 and q at plane nzl (no exchange refreshes them)
};

struct UV {
    float uk, um, vk[3], vm[3];
};
struct PQ {
    float p[3], q[6];
};

template <int TY, int SLOTS, typename CT>
__global__ void __launch_bounds__(32 * (TY + 2), 1) fused_kernel(const FusedArgs A)
{
    __shared__ float sm_uv[2][4][TY + 2][32];  // ubar, vbar_x, vbar_y, vbar_z of plane s
    __shared__ float sm_r[2][4][TY + 2][32];   // p_y, q_xy, q_yy, q_yz of D(s)
    const IterPtrs& a = A.a;
    const Geo& g = A.g;
    const StepParams& sp = A.sp;
    const int lane = threadIdx.x, ty = threadIdx.y;
    const int x = blockIdx.x * 30 - 1 + lane, y = blockIdx.y * TY - 1 + ty;
    const bool vxy = x >= 0 && x < g.nx && y >= 0 && y < g.ny;
    const bool own = vxy && lane >= 1 && lane <= 30 && ty >= 1 && ty <= TY;
    const bool xl = x < g.nx - 1, xf = x > 0, yl = y < g.ny - 1, yf = y > 0;
    const bool prow = ty <= TY;       // rows needing p_{k+1} (all but the top halo row)
    const bool qrow = ty >= 1;        // rows needing q_{k+1} (all but the bottom halo row)
    const bool mrow = qrow && prow;   // owned rows: primal
    const int zs = A.z_lo + blockIdx.z * A.zc;
    const int ze = min(zs + A.zc, A.z_hi);
    const int rowoff = y * g.px + x;

    auto load_uv = [&](int s) {
        UV r;
        const bool ok = vxy && s >= -1 && s <= g.nzl;
        const int o = (s + 1) * g.plane + rowoff;
        r.uk = ok ? __ldg(a.uk + o) : 0.f;
        r.um = ok ? __ldg(a.um + o) : 0.f;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            r.vk[k] = ok ? __ldg(a.vk[k] + o) : 0.f;
            r.vm[k] = ok ? __ldg(a.vm[k] + o) : 0.f;
        }
        return r;
    };
    auto load_pq = [&](int s) {
        PQ r;
        const bool ok = vxy && s >= -1 && s <= g.nzl;
        const int o = (s + 1) * g.plane + rowoff;
#pragma unroll
        for (int k = 0; k < 3; ++k) r.p[k] = (ok && prow) ? __ldg(a.pk[k] + o) : 0.f;
#pragma unroll
        for (int m = 0; m < 6; ++m) r.q[m] = (ok && qrow) ? __ldg(a.qk[m] + o) : 0.f;
        return r;
    };
    auto load_h = [&](int s) {
        HistRaw<SLOTS, CT> h{};
        if (own && s >= 0 && s < g.nzl) h = load_hist<SLOTS, CT>(a.hist, (int64_t)s * g.plane + rowoff);
        return h;
    };

    UV u0 = load_uv(zs - 1), u1 = load_uv(zs);
    PQ pq0 = load_pq(zs - 1);
    float vbp[3] = {0.f, 0.f, 0.f};  // vbar(s-1)
    float uk_p = 0.f, vk_p[3] = {0.f, 0.f, 0.f};
    HistRaw<SLOTS, CT> h0{};
    float pn_p[3] = {0.f, 0.f, 0.f}, pz_pp = 0.f, qn_p[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};

    for (int s = zs - 1; s <= ze; ++s) {
        // prefetch (consumed next step)
        const UV u2 = load_uv(s + 2);
        const PQ pq1 = load_pq(s + 1);
        const HistRaw<SLOTS, CT> h1 = load_h(s);
        const int par = s & 1;
        const int zg = g.z0 + s;
        const bool zl = zg < g.nz - 1, zf = zg > 0;

        // (a3) over-relaxed iterate at planes s and s+1
        const float ub = fmaf(2.f, u0.uk, -u0.um);
        float vb[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) vb[k] = fmaf(2.f, u0.vk[k], -u0.vm[k]);
        const float ub1 = fmaf(2.f, u1.uk, -u1.um);
        sm_uv[par][0][ty][lane] = ub;
        sm_uv[par][1][ty][lane] = vb[0];
        sm_uv[par][2][ty][lane] = vb[1];
        sm_uv[par][3][ty][lane] = vb[2];
        __syncthreads();

        // (a1) dual D(s)
        float pn[3] = {0.f, 0.f, 0.f}, qn[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (prow) {
            const float ux = __shfl_down_sync(FULL, ub, 1);
            const float uy = sm_uv[par][0][ty + 1][lane];
            const float g0 = xl ? ux - ub : 0.f, g1 = yl ? uy - ub : 0.f, g2 = zl ? ub1 - ub : 0.f;
            pn[0] = fmaf(sp.sigma, g0 - vb[0], pq0.p[0]);
            pn[1] = fmaf(sp.sigma, g1 - vb[1], pq0.p[1]);
            pn[2] = fmaf(sp.sigma, g2 - vb[2], pq0.p[2]);
            const float f = proj_scale(pn[0] * pn[0] + pn[1] * pn[1] + pn[2] * pn[2], sp.alpha1);
            pn[0] *= f;
            pn[1] *= f;
            pn[2] *= f;
        }
        if (qrow) {
            float dx[3], dy[3], dz[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const float vx = __shfl_up_sync(FULL, vb[k], 1);
                const float vy = sm_uv[par][1 + k][ty - 1][lane];
                dx[k] = fmaf(xl ? 1.f : 0.f, vb[k], -(xf ? vx : 0.f));
                dy[k] = fmaf(yl ? 1.f : 0.f, vb[k], -(yf ? vy : 0.f));
                dz[k] = fmaf(zl ? 1.f : 0.f, vb[k], -(zf ? vbp[k] : 0.f));
            }
            const float e[6] = {dx[0], dy[1], dz[2], 0.5f * (dy[0] + dx[1]), 0.5f * (dz[0] + dx[2]),
                                0.5f * (dz[1] + dy[2])};
#pragma unroll
            for (int m = 0; m < 6; ++m) qn[m] = fmaf(sp.sigma, e[m], pq0.q[m]);
            const float f = proj_scale(qn[0] * qn[0] + qn[1] * qn[1] + qn[2] * qn[2] +
                                           2.f * (qn[3] * qn[3] + qn[4] * qn[4] + qn[5] * qn[5]),
                                       sp.alpha0);
#pragma unroll
            for (int m = 0; m < 6; ++m) qn[m] *= f;
        }
        sm_r[par][0][ty][lane] = pn[1];
        sm_r[par][1][ty][lane] = qn[3];
        sm_r[par][2][ty][lane] = qn[1];
        sm_r[par][3][ty][lane] = qn[5];
        if (own && ((s >= zs && s < ze) || (A.keep_halo_dual && (s == -1 || s == g.nzl)))) {
            const int o = (s + 1) * g.plane + rowoff;
#pragma unroll
            for (int k = 0; k < 3; ++k) a.pn[k][o] = pn[k];
#pragma unroll
            for (int m = 0; m < 6; ++m) a.qn[m][o] = qn[m];
        }

        // (a2) primal Pm(s-1) on owned rows
        if (mrow && s - 1 >= zs) {
            const int pr = par ^ 1;
            const bool zl1 = zg - 1 < g.nz - 1, zf1 = zg - 1 > 0;
            const float pxm = __shfl_up_sync(FULL, pn_p[0], 1);
            const float pym = sm_r[pr][0][ty - 1][lane];
            const float divp = fmaf(xl ? 1.f : 0.f, pn_p[0], -(xf ? pxm : 0.f)) +
                               fmaf(yl ? 1.f : 0.f, pn_p[1], -(yf ? pym : 0.f)) +
                               fmaf(zl1 ? 1.f : 0.f, pn_p[2], -(zf1 ? pz_pp : 0.f));
            const float qxx = __shfl_down_sync(FULL, qn_p[0], 1);
            const float qxy = __shfl_down_sync(FULL, qn_p[3], 1);
            const float qxz = __shfl_down_sync(FULL, qn_p[4], 1);
            const float qyxy = sm_r[pr][1][ty + 1][lane];
            const float qyyy = sm_r[pr][2][ty + 1][lane];
            const float qyyz = sm_r[pr][3][ty + 1][lane];
            // (div2 q)_k = D+_x q_kx + D+_y q_ky + D+_z q_kz at plane s-1; q(s) = qn
            const float w0 = (xl ? qxx - qn_p[0] : 0.f) + (yl ? qyxy - qn_p[3] : 0.f) + (zl1 ? qn[4] - qn_p[4] : 0.f);
            const float w1 = (xl ? qxy - qn_p[3] : 0.f) + (yl ? qyyy - qn_p[1] : 0.f) + (zl1 ? qn[5] - qn_p[5] : 0.f);
            const float w2 = (xl ? qxz - qn_p[4] : 0.f) + (yl ? qyyz - qn_p[5] : 0.f) + (zl1 ? qn[2] - qn_p[2] : 0.f);
            if (own) {
                const float un = hist_prox<SLOTS, CT>(fmaf(sp.tau, divp, uk_p), sp.tl, h0, A.C);
                const int o = s * g.plane + rowoff;  // plane s-1
                a.un[o] = un;
                a.vn[0][o] = fmaf(sp.tau, pn_p[0] + w0, vk_p[0]);
                a.vn[1][o] = fmaf(sp.tau, pn_p[1] + w1, vk_p[1]);
                a.vn[2][o] = fmaf(sp.tau, pn_p[2] + w2, vk_p[2]);
            }
        }

        // rotate
        pz_pp = pn_p[2];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            pn_p[k] = pn[k];
            vbp[k] = vb[k];
            vk_p[k] = u0.vk[k];
        }
#pragma unroll
        for (int m = 0; m < 6; ++m) qn_p[m] = qn[m];
        uk_p = u0.uk;
        h0 = h1;
        u0 = u1;
        u1 = u2;
        pq0 = pq1;
    }
}

// ===========================================================================
// NEXT-4 TV-L1, FUSED schedule: one single-sweep kernel per iteration.
// Reads u_k, u_{k-1}, p_k and the counts, writes p_{k+1}, u_{k+1}:
// 4 (2 + 3) + counts + 4 (3 + 1) = 44 B per voxel-iteration with u8 counts (60 B split).
// Same thread layout as fused_kernel: 32 lanes x (TY + 2) rows, lanes 1..30 and
// rows 1..TY owned; lane 0 / row 0 compute the dual of the x-1 / y-1 neighbours
// (div p reads p_x(x-1), p_y(y-1)), lane 31 / row TY+1 only supply ubar(x+1),
// ubar(y+1).  Step s computes the dual D(s) (rows 0..TY) and the primal of plane
// s-1, whose p_y(y-1) comes from the shared plane written in step s-1, so one
// __syncthreads per step separates both exchanges (parity double buffers).  The
// arithmetic is that of tvl1_dual_kernel / tvl1_primal_kernel expression for
// expression (the two schedules agree bit for bit, tests/test_gpu_parity.py).
// ===========================================================================
template <int TY, int SLOTS, typename CT>
__global__ void __launch_bounds__(32 * (TY + 2)) tvl1_fused_kernel(const FusedArgs A)
{
    __shared__ float sm_u[2][TY + 2][32];  // ubar of plane s
    __shared__ float sm_p[2][TY + 2][32];  // p_y of D(s)
    const IterPtrs& a = A.a;
    const Geo& g = A.g;
    const StepParams& sp = A.sp;
    const int lane = threadIdx.x, ty = threadIdx.y;
    const int x = blockIdx.x * 30 - 1 + lane, y = blockIdx.y * TY - 1 + ty;
    const bool vxy = x >= 0 && x < g.nx && y >= 0 && y < g.ny;
    const bool own = vxy && lane >= 1 && lane <= 30 && ty >= 1 && ty <= TY;
    const bool xl = x < g.nx - 1, xf = x > 0, yl = y < g.ny - 1, yf = y > 0;
    const bool prow = ty <= TY;  // rows needing p_{k+1}
    const int zs = A.z_lo + blockIdx.z * A.zc;
    const int ze = min(zs + A.zc, A.z_hi);
    const int rowoff = y * g.px + x;

    // Loads use coordinates clamped into the slab (halo planes included): every
    // address is valid, and a value read for an out-of-grid thread or plane only
    // ever meets a zero boundary factor (xl, yl, zl, xf, yf, zf), so no predicate or
    // select is needed per load.
    const int rowc = min(max(y, 0), g.ny - 1) * g.px + min(max(x, 0), g.nx - 1);
    auto off = [&](int s) { return (min(max(s, -1), g.nzl) + 1) * g.plane + rowc; };
    int o0 = off(zs - 1), o1 = off(zs);
    float uk0 = __ldg(a.uk + o0), um0 = __ldg(a.um + o0);  // plane s
    float uk1 = __ldg(a.uk + o1), um1 = __ldg(a.um + o1);  // plane s+1
    float pk0[3];                                          // p_k(s)
#pragma unroll
    for (int d = 0; d < 3; ++d) pk0[d] = __ldg(a.pk[d] + o0);
    HistRaw<SLOTS, CT> h0{};
    float uk_p = 0.f, pn_p[3] = {0.f, 0.f, 0.f}, pz_pp = 0.f;

    for (int s = zs - 1; s <= ze; ++s) {
        // prefetch (consumed next step)
        const int o2 = off(s + 2);
        const float uk2 = __ldg(a.uk + o2), um2 = __ldg(a.um + o2);
        float pk1[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) pk1[d] = __ldg(a.pk[d] + o1);
        HistRaw<SLOTS, CT> h1{};
        if (own && s >= 0 && s < g.nzl) h1 = load_hist<SLOTS, CT>(a.hist, (int64_t)s * g.plane + rowoff);
        const int par = s & 1;
        const int zg = g.z0 + s;
        const bool zl = zg < g.nz - 1;

        const float ub = fmaf(2.f, uk0, -um0);
        const float ub1 = fmaf(2.f, uk1, -um1);
        sm_u[par][ty][lane] = ub;
        __syncthreads();

        // dual D(s) (tvl1_dual_kernel)
        float pn[3] = {0.f, 0.f, 0.f};
        if (prow && s < ze) {
            const float ux = __shfl_down_sync(FULL, ub, 1);
            const float uy = sm_u[par][ty + 1][lane];
            const float g0 = xl ? ux - ub : 0.f, g1 = yl ? uy - ub : 0.f, g2 = zl ? ub1 - ub : 0.f;
            pn[0] = fmaf(sp.sigma, g0, pk0[0]);
            pn[1] = fmaf(sp.sigma, g1, pk0[1]);
            pn[2] = fmaf(sp.sigma, g2, pk0[2]);
            const float f = proj_scale(pn[0] * pn[0] + pn[1] * pn[1] + pn[2] * pn[2], sp.alpha1);
            pn[0] *= f;
            pn[1] *= f;
            pn[2] *= f;
        }
        sm_p[par][ty][lane] = pn[1];
        if (own && s >= zs && s < ze) {
            const int o = (s + 1) * g.plane + rowoff;
#pragma unroll
            for (int d = 0; d < 3; ++d) a.pn[d][o] = pn[d];
        }

        // primal of plane s-1 (tvl1_primal_kernel)
        const float pxm_all = __shfl_up_sync(FULL, pn_p[0], 1);
        if (own && s - 1 >= zs) {
            const int zg1 = zg - 1;
            const bool zl1 = zg1 < g.nz - 1, zf1 = zg1 > 0;
            const float pxm = xf ? pxm_all : 0.f;
            const float pym = yf ? sm_p[par ^ 1][ty - 1][lane] : 0.f;
            const float pzm = zf1 ? pz_pp : 0.f;
            const float divp = ((xl ? pn_p[0] : 0.f) - pxm) + ((yl ? pn_p[1] : 0.f) - pym) +
                               ((zl1 ? pn_p[2] : 0.f) - pzm);
            a.un[s * g.plane + rowoff] = hist_prox<SLOTS, CT>(fmaf(sp.tau, divp, uk_p), sp.tl, h0, A.C);
        }

        // rotate
        pz_pp = pn_p[2];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            pn_p[d] = pn[d];
            pk0[d] = pk1[d];
        }
        uk_p = uk0;
        h0 = h1;
        uk0 = uk1;
        um0 = um1;
        uk1 = uk2;
        um1 = um2;
        o1 = o2;
    }
}

// ===========================================================================
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
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(FULL, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(maxc, m);
}

// u16 -> u8 copy of the whole store (only when every count <= 255)
__global__ void compact_counts_kernel(const uint16_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t n)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = (uint8_t)src[i];
}

// ---------------------------------------------------------------------------
// NEXT-1 coarse-to-fine (R18-R20)
// restriction: coarse voxel (X, Y, Z) sums the u16 counts of its <= 8 children
// (2X + {0,1}, 2Y + {0,1}, 2Z + {0,1}) inside the fine grid
template <int SLOTS>
__global__ void restrict_counts_kernel(const uint16_t* __restrict__ Hf, Geo gf, uint16_t* __restrict__ Hc, Geo gc,
                                       unsigned int* __restrict__ maxc)
{
    const int64_t n = (int64_t)gc.nzl * gc.ny * gc.nx;
    unsigned int m = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int X = (int)(v % gc.nx);
        const int64_t r = v / gc.nx;
        const int Y = (int)(r % gc.ny);
        const int Z = (int)(r / gc.ny);
        unsigned int acc[SLOTS];
        for (int b = 0; b < SLOTS; ++b) acc[b] = 0;
        for (int dz = 0; dz < 2; ++dz)
            for (int dy = 0; dy < 2; ++dy)
                for (int dx = 0; dx < 2; ++dx) {
                    const int x = 2 * X + dx, y = 2 * Y + dy, z = 2 * Z + dz;
                    if (x < gf.nx && y < gf.ny && z < gf.nzl) {
                        const uint16_t* src = Hf + ((int64_t)z * gf.plane + (int64_t)y * gf.px + x) * SLOTS;
                        for (int b = 0; b < SLOTS; ++b) acc[b] += src[b];
                    }
                }
        uint16_t* dst = Hc + ((int64_t)Z * gc.plane + (int64_t)Y * gc.px + X) * SLOTS;
        for (int b = 0; b < SLOTS; ++b) {
            m = max(m, acc[b]);
            dst[b] = (uint16_t)min(acc[b], 65535u);
        }
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(FULL, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(maxc, m);
}

// prolongation: every fine voxel takes its parent's u and v / 2 (v is a per-voxel
// slope, and a fine voxel is half as wide), as both the current and the previous
// iterate (restart: ubar = u, vbar = v); p and q are zeroed by the caller
__global__ void prolong_kernel(const float* __restrict__ uc, const float* __restrict__ vc0,
                               const float* __restrict__ vc1, const float* __restrict__ vc2, Geo gc,
                               float* __restrict__ uf, float* __restrict__ uf_prev, float* __restrict__ vf0,
                               float* __restrict__ vf1, float* __restrict__ vf2, float* __restrict__ vf0_prev,
                               float* __restrict__ vf1_prev, float* __restrict__ vf2_prev, Geo gf)
{
    const int64_t n = (int64_t)gf.nzl * gf.ny * gf.nx;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(v % gf.nx);
        const int64_t r = v / gf.nx;
        const int y = (int)(r % gf.ny);
        const int z = (int)(r / gf.ny);
        const int ic = eoff(gc, x / 2, y / 2, z / 2), i = eoff(gf, x, y, z);
        const float u = uc[ic];
        const float a = 0.5f * vc0[ic], b = 0.5f * vc1[ic], c = 0.5f * vc2[ic];
        uf[i] = u;
        uf_prev[i] = u;
        vf0[i] = a;
        vf1[i] = b;
        vf2[i] = c;
        vf0_prev[i] = a;
        vf1_prev[i] = b;
        vf2_prev[i] = c;
    }
}

// NEXT-3 leaves: counts of this context's planes [0, nzc) (chunk starting at local plane zc0)
// as sums over factor^3 fine voxels of a dense uint32 fine slab [nzf][nyf][nxf][nbins]
// (fine plane 0 of the slab = fine plane factor * (z0 + zc0))
template <int SLOTS, typename T>
__global__ void coarsen_counts_kernel(const T* __restrict__ fine, int nxf, int nyf, int nzf, int factor,
                                      int nbins, int nzc, int zc0, Geo g, uint16_t* __restrict__ H,
                                      unsigned int* __restrict__ maxc)
{
    const int64_t n = (int64_t)nzc * g.ny * g.nx;
    unsigned int m = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int X = (int)(v % g.nx);
        const int64_t r = v / g.nx;
        const int Y = (int)(r % g.ny);
        const int Zc = (int)(r / g.ny);  // plane within the chunk
        unsigned int acc[SLOTS];
        for (int b = 0; b < SLOTS; ++b) acc[b] = 0;
        for (int dz = 0; dz < factor; ++dz) {
            const int zf = Zc * factor + dz;
            if (zf >= nzf) break;
            for (int dy = 0; dy < factor; ++dy) {
                const int yf = Y * factor + dy;
                if (yf >= nyf) break;
                for (int dx = 0; dx < factor; ++dx) {
                    const int xf = X * factor + dx;
                    if (xf >= nxf) break;
                    const T* src = fine + (((int64_t)zf * nyf + yf) * nxf + xf) * nbins;
                    for (int b = 0; b < nbins; ++b) acc[b] += src[b];
                }
            }
        }
        uint16_t* dst = H + ((int64_t)(Zc + zc0) * g.plane + (int64_t)Y * g.px + X) * SLOTS;
        for (int b = 0; b < SLOTS; ++b) {
            m = max(m, acc[b]);
            dst[b] = (uint16_t)min(acc[b], 65535u);
        }
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(FULL, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(maxc, m);
}

// NEXT-3 leaves: prolongation from a dense coarse slab [cnz][cny][cnx] (u) / [3][...] (v)
// whose plane 0 is coarse global plane cz0, into local planes [zlo, zhi) (halo planes
// included) of this context: u = parent u, v = parent v / 2, in every slot listed.
__global__ void prolong_slab_kernel(const float* __restrict__ uc, const float* __restrict__ vc, int cnx, int cny,
                                    int cnz, int cz0, int zlo, int zhi, Geo g, float* const* __restrict__ us,
                                    int nus, float* const* __restrict__ vs, int nvs)
{
    const int64_t n = (int64_t)(zhi - zlo) * g.ny * g.nx;
    const int64_t cpl = (int64_t)cnx * cny * cnz;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(v % g.nx);
        const int64_t r = v / g.nx;
        const int y = (int)(r % g.ny);
        const int zl = (int)(r / g.ny) + zlo;
        const int zc = (g.z0 + zl) / 2 - cz0;  // parent plane within the coarse slab
        if (zc < 0 || zc >= cnz) continue;
        const int64_t ic = ((int64_t)zc * cny + y / 2) * cnx + x / 2;
        const int i = eoff(g, x, y, zl);
        const float u = uc[ic];
        for (int k = 0; k < nus; ++k) us[k][i] = u;
        for (int d = 0; d < 3; ++d) {
            const float a = 0.5f * vc[d * cpl + ic];
            for (int k = 0; k < nvs; ++k) vs[3 * k + d][i] = a;
        }
    }
}

// u_0 = sum h c / W (fp64, 0 where W = 0) into the current and previous u buffers
// (ubar_0 = 2 u_0 - u_0 = u_0); every other field is zeroed by the caller.
template <int SLOTS, typename CT>
__global__ void init_state_kernel(float* __restrict__ u_cur, float* __restrict__ u_prev, const void* __restrict__ H,
                                  Geo g, Centers C)
{
    const int64_t n = (int64_t)g.nzl * g.ny * g.nx;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(v % g.nx);
        const int64_t r = v / g.nx;
        const int y = (int)(r % g.ny);
        const int z = (int)(r / g.ny);
        const auto h = load_hist<SLOTS, CT>(H, (int64_t)z * g.plane + (int64_t)y * g.px + x);
        double W = 0.0, m = 0.0;
        for (int b = 0; b < SLOTS; ++b) {
            const double hb = (double)hist_count<SLOTS, CT>(h, b);
            if (hb != 0.0) {
                W += hb;
                m += hb * (double)C.c[b];
            }
        }
        const float u0 = W > 0.0 ? (float)(m / W) : 0.f;
        const int i = eoff(g, x, y, z);
        u_cur[i] = u0;
        u_prev[i] = u0;
    }
}

// ===========================================================================
// (a4) energy and restricted gap, fp64 per-voxel terms, deterministic reduction.
struct EnergyArgs {
    const float* u;
    const float* v[3];
    const float* p[3];
    const float* q[6];
    const void* hist;
    double alpha1, alpha0, lambda, V;
    int nbins;
};

constexpr int EN_TERMS = 5;  // alpha1, alpha0, data, dual, vmax

__device__ __forceinline__ double warp_sum(double v)
{
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v)
{
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

// fp64 constants of the data term and of the box-restricted dual (R14), from the bin
// centres: padded bins (b >= nbins, whose counts are 0) sit at +1, so every walk below
// runs over SLOTS bins at compile time with no local arrays
struct EnergyConsts {
    double c[16];   // c_b (1.0 beyond nbins)
    double c1[16];  // c_b + 1
    double dc[17];  // c_b - c_{b-1} with c_{-1} = -1; dc[16]: 1 - c_15 (unused, the walk ends at the last slot)
    double end;     // 1 - c_{SLOTS-1} for the template's SLOTS (set per launch)
    float cf[16], c1f[16], dcf[16], endf;  // the same in fp32 (dense energy kernel)
};

// count b as an exact double: the count in the low mantissa word of 2^52, minus 2^52
template <int SLOTS, typename CT>
__device__ __forceinline__ double hist_count_f64(const HistRaw<SLOTS, CT>& h, int b)
{
    uint32_t lo;
    if constexpr (sizeof(CT) == 1)
        lo = __byte_perm(h.w[b >> 2], 0u, (b & 3) | 0x4 << 4 | 0x4 << 8 | 0x4 << 12);
    else
        lo = __byte_perm(h.w[b >> 1], 0u, (2 * (b & 1)) | (2 * (b & 1) + 1) << 4 | 0x4 << 8 | 0x4 << 12);
    return __hiloint2double(0x43300000, (int)lo) - 4503599627370496.0;
}

template <int SLOTS, typename CT>
__device__ __forceinline__ uint32_t hist_total(const HistRaw<SLOTS, CT>& h)
{
    uint32_t W = 0;
    if constexpr (sizeof(CT) == 1) {
#pragma unroll
        for (int k = 0; k < SLOTS / 4; ++k) W = __dp4a(h.w[k], 0x01010101u, W);
    } else {
#pragma unroll
        for (int k = 0; k < SLOTS / 2; ++k) W += (h.w[k] & 0xffffu) + (h.w[k] >> 16);
    }
    return W;
}

// data_box_terms in fp32 (the dense energy kernel's per-voxel terms; fp64 accumulation)
template <int SLOTS, typename CT>
__device__ __forceinline__ void data_box_terms_f32(const HistRaw<SLOTS, CT>& h, const EnergyConsts& K, float lam,
                                                   float u, float divp, float& data, float& box)
{
    const uint32_t Wi = hist_total<SLOTS, CT>(h);
    if (Wi == 0) {  // no votes: G = 0, so min over [-1, 1] of -x divp is -|divp| (unobserved space)
        data = 0.f;
        box = -fabsf(divp);
        return;
    }
    float d = 0.f, G = 0.f, f = 0.f, best = 0.f;
    const float W = (float)Wi;
    float slope = -fmaf(lam, W, divp);
    const float l2 = 2.f * lam;
#pragma unroll
    for (int b = 0; b < SLOTS; ++b) {
        const float hb = hist_count<SLOTS, CT>(h, b);
        d = fmaf(hb, fabsf(u - K.cf[b]), d);
        G = fmaf(hb, K.c1f[b], G);
        f = fmaf(K.dcf[b], slope, f);
        best = fminf(best, f);
        slope = fmaf(l2, hb, slope);
    }
    f = fmaf(K.endf, slope, f);
    best = fminf(best, f);
    data = lam * d;
    box = fmaf(lam, G, divp) + best;
}

// Per voxel, in fp64 (PAPER.md:153 data term with the R2 histogram form; R14 box dual):
//   data = lam sum_b h_b |u - c_b|
//   box  = min_{x in [-1,1]} g(x),  g(x) = lam sum_b h_b |x - c_b| - x divp
// g is convex and piecewise linear with kinks at the centres, so its minimum over [-1, 1] is
// at -1, a centre or +1.  One left-to-right walk evaluates g at all of them: g(-1) = lam sum h (c+1)
// + divp, then g grows by (gap) x (slope) with slope = lam (2 C_b - W) - divp on (c_{b-1}, c_b).
template <int SLOTS, typename CT>
__device__ __forceinline__ void data_box_terms(const HistRaw<SLOTS, CT>& h, const EnergyConsts& K, double lam,
                                               double u, double divp, double& data, double& box)
{
    const double W = (double)hist_total<SLOTS, CT>(h);
    double d = 0.0, G = 0.0, f = 0.0, best = 0.0;
    double slope = -fma(lam, W, divp);
    const double l2 = 2.0 * lam;
#pragma unroll
    for (int b = 0; b < SLOTS; ++b) {
        const double hb = hist_count_f64<SLOTS, CT>(h, b);
        d = fma(hb, fabs(u - K.c[b]), d);
        G = fma(hb, K.c1[b], G);
        f = fma(K.dc[b], slope, f);  // g(c_b) - g(-1)
        best = fmin(best, f);
        slope = fma(l2, hb, slope);
    }
    f = fma(K.end, slope, f);  // g(1) - g(-1)
    best = fmin(best, f);
    data = lam * d;
    box = fma(lam, G, divp) + best;
}

// One voxel's inputs to the energy / restricted-gap terms: the centre values and the
// neighbours each difference reads (x / y / z suffixes: +1 for u and q, -1 for v and p).
struct EnVoxel {
    float uc, ux, uy, un;                            // u at (x,y,z), x+1, y+1, z+1
    float v0, v1, v2, v0x, v1x, v2x, v0y, v1y, v2y;  // v at (x,y,z), x-1, y-1
    float vm0, vm1, vm2;                             // v at z-1
    float p0, p1, p2, p0x, p1y, pzm;                 // p; p_x at x-1, p_y at y-1, p_z at z-1
    float qxx, qyy, qzz, qxy, qxz, qyz;              // q at (x,y,z)
    float qxxx, qxyx, qxzx, qxyy, qyyy, qyzy;        // q_xx, q_xy, q_xz at x+1; q_xy, q_yy, q_yz at y+1
    float qzzn, qxzn, qyzn;                          // q_zz, q_xz, q_yz at z+1
};

// Per-voxel energy terms (PAPER.md:133 E, R14 box-restricted dual), accumulated in fp64:
//   t1 += alpha1 |D+u - v|, t0 += alpha0 |E(v)| (Frobenius, R5), td += lam sum_b h_b |u - c_b|,
//   dv += min_{|x|<=1} (lam sum_b h_b |x - c_b| - x divp) - V ||p + div2 q||_1.
// The masks are R6's Neumann D+ / D-; INT: all of them true (voxels away from the faces).
template <int SLOTS, typename CT, bool INT>
__device__ __forceinline__ void energy_voxel_terms(const EnVoxel& e, const HistRaw<SLOTS, CT>& h,
                                                   const EnergyConsts& K, float al1, float al0, float lam, float VV,
                                                   bool xl, bool yl, bool zl, bool xf, bool yf, bool zf, double& t1,
                                                   double& t0, double& td, double& dv)
{
    const bool xl_ = INT || xl, yl_ = INT || yl, zl_ = INT || zl, xf_ = INT || xf, yf_ = INT || yf, zf_ = INT || zf;
    auto dp = [](bool l, float a, float b) { return l ? a - b : 0.f; };
    auto dm = [](bool l, bool f, float a, float b) { return (l ? a : 0.f) - (f ? b : 0.f); };
    const float a0 = dp(xl_, e.ux, e.uc) - e.v0, a1 = dp(yl_, e.uy, e.uc) - e.v1, a2 = dp(zl_, e.un, e.uc) - e.v2;
    t1 += (double)(al1 * sqrtf(fmaf(a0, a0, fmaf(a1, a1, a2 * a2))));
    const float exx = dm(xl_, xf_, e.v0, e.v0x), eyy = dm(yl_, yf_, e.v1, e.v1y), ezz = dm(zl_, zf_, e.v2, e.vm2);
    const float exy = 0.5f * (dm(yl_, yf_, e.v0, e.v0y) + dm(xl_, xf_, e.v1, e.v1x));
    const float exz = 0.5f * (dm(zl_, zf_, e.v0, e.vm0) + dm(xl_, xf_, e.v2, e.v2x));
    const float eyz = 0.5f * (dm(zl_, zf_, e.v1, e.vm1) + dm(yl_, yf_, e.v2, e.v2y));
    const float off = fmaf(exy, exy, fmaf(exz, exz, eyz * eyz));
    t0 += (double)(al0 * sqrtf(fmaf(exx, exx, fmaf(eyy, eyy, fmaf(ezz, ezz, 2.f * off)))));
    const float divp = dm(xl_, xf_, e.p0, e.p0x) + dm(yl_, yf_, e.p1, e.p1y) + dm(zl_, zf_, e.p2, e.pzm);
    const float w0 = dp(xl_, e.qxxx, e.qxx) + dp(yl_, e.qxyy, e.qxy) + dp(zl_, e.qxzn, e.qxz);
    const float w1 = dp(xl_, e.qxyx, e.qxy) + dp(yl_, e.qyyy, e.qyy) + dp(zl_, e.qyzn, e.qyz);
    const float w2 = dp(xl_, e.qxzx, e.qxz) + dp(yl_, e.qyzy, e.qyz) + dp(zl_, e.qzzn, e.qzz);
    const float l1 = fabsf(e.p0 + w0) + fabsf(e.p1 + w1) + fabsf(e.p2 + w2);
    float data, box;
    data_box_terms_f32<SLOTS, CT>(h, K, lam, e.uc, divp, data, box);
    td += (double)data;
    dv += (double)box - (double)(VV * l1);
}

// Grid of the energy sweep: warp = a 32-voxel x segment of one row, block = 8 consecutive
// rows of one x tile, item = (x tile, 8-row group, z chunk); each warp marches its chunk in z.
struct EnergySched {
    int ntx, nyg, zc, items;
};

// (a4) dense energy / restricted gap (R14).  HBM-bound: each of the
// 13 fields and the counts is read once (60 B per voxel with u8 counts); the z-neighbours
// ride in registers along the march, the x / y neighbours are L1 / L2 hits of the same or
// the neighbouring warp's rows.  The per-voxel terms are formed in fp32 from the fp32
// state (relative error of each term ~1e-7) and REDUCED in fp64: per-thread fp64 sums,
// warp shuffles, fixed-order block partials (energy_final_kernel): deterministic.  (An
// all-fp64 version spent its time in 38 fp32->fp64 conversions per voxel on the XU pipe:
// 0.43 of the copy roofline, profiles/r2b_energy_*.)  On C4 the halo rows / sectors of
// neighbouring items mostly miss L2 (DRAM reads 1.24x the algorithmic bytes,
// profiles/r2e_C4_launches_summary.txt); a barrier per plane to keep a block's rows in step
// made it worse (1.34x, profiles/r2f_*) and is not used.
template <int SLOTS, typename CT>
__global__ void __launch_bounds__(256, SLOTS == 8 ? 3 : 2)
    energy_partial_kernel(const EnergyArgs ea, Geo g, const EnergyConsts K, const EnergySched es,
                          double* __restrict__ partials)
{
    double t1 = 0, t0 = 0, td = 0, dv = 0;
    float vm = 0.f;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int sy = g.px, sz = g.plane;
    const float al1 = (float)ea.alpha1, al0 = (float)ea.alpha0, lam = (float)ea.lambda, VV = (float)ea.V;
    for (int it = blockIdx.x; it < es.items; it += gridDim.x) {
        const int xt = it % es.ntx, r = it / es.ntx;
        // cells past the grid's x / y ends (ragged last tile / row group) march along on a
        // clamped in-grid cell without accumulating: every thread reaches the per-plane barrier
        const int xr = xt * 32 + lane, yr = (r % es.nyg) * 8 + wid;
        const bool act = xr < g.nx && yr < g.ny;
        const int x = min(xr, g.nx - 1), y = min(yr, g.ny - 1);
        const int za = (r / es.nyg) * es.zc, zb = min(g.nzl, za + es.zc);
        const bool xl = x < g.nx - 1, yl = y < g.ny - 1, xf = x > 0, yf = y > 0;
        int i = eoff(g, x, y, za);
        int64_t hv = (int64_t)za * g.plane + (int64_t)y * g.px + x;
        auto L = [&](const float* f, int o) { return __ldg(f + o); };
        // carried along z: v (3) and p_z at z-1; u, q_zz, q_xz, q_yz at z (loaded as z+1)
        float vm0 = L(ea.v[0], i - sz), vm1 = L(ea.v[1], i - sz), vm2 = L(ea.v[2], i - sz), pzm = L(ea.p[2], i - sz);
        float uc = L(ea.u, i), qzz = L(ea.q[2], i), qxz = L(ea.q[4], i), qyz = L(ea.q[5], i);
        for (int z = za; z < zb; ++z, i += sz, hv += g.plane) {
            const int zg = g.z0 + z;
            const bool zl = zg < g.nz - 1, zf = zg > 0;
            // ---- loads: plane z+1 (carried fields), plane z centres and x / y neighbours
            const float un = L(ea.u, i + sz), qzzn = L(ea.q[2], i + sz), qxzn = L(ea.q[4], i + sz),
                        qyzn = L(ea.q[5], i + sz);
            const float v0 = L(ea.v[0], i), v1 = L(ea.v[1], i), v2 = L(ea.v[2], i);
            const float p0 = L(ea.p[0], i), p1 = L(ea.p[1], i), p2 = L(ea.p[2], i);
            const float qxx = L(ea.q[0], i), qyy = L(ea.q[1], i), qxy = L(ea.q[3], i);
            const float ux = L(ea.u, i + 1), uy = L(ea.u, i + sy);
            const float qxxx = L(ea.q[0], i + 1), qxyx = L(ea.q[3], i + 1), qxzx = L(ea.q[4], i + 1);
            const float qxyy = L(ea.q[3], i + sy), qyyy = L(ea.q[1], i + sy), qyzy = L(ea.q[5], i + sy);
            const float v0x = L(ea.v[0], i - 1), v1x = L(ea.v[1], i - 1), v2x = L(ea.v[2], i - 1), p0x = L(ea.p[0], i - 1);
            const float v0y = L(ea.v[0], i - sy), v1y = L(ea.v[1], i - sy), v2y = L(ea.v[2], i - sy),
                        p1y = L(ea.p[1], i - sy);
            const auto h = load_hist<SLOTS, CT>(ea.hist, hv);
            if (act) {
                EnVoxel e;
                e.uc = uc, e.ux = ux, e.uy = uy, e.un = un;
                e.v0 = v0, e.v1 = v1, e.v2 = v2, e.v0x = v0x, e.v1x = v1x, e.v2x = v2x;
                e.v0y = v0y, e.v1y = v1y, e.v2y = v2y, e.vm0 = vm0, e.vm1 = vm1, e.vm2 = vm2;
                e.p0 = p0, e.p1 = p1, e.p2 = p2, e.p0x = p0x, e.p1y = p1y, e.pzm = pzm;
                e.qxx = qxx, e.qyy = qyy, e.qzz = qzz, e.qxy = qxy, e.qxz = qxz, e.qyz = qyz;
                e.qxxx = qxxx, e.qxyx = qxyx, e.qxzx = qxzx, e.qxyy = qxyy, e.qyyy = qyyy, e.qyzy = qyzy;
                e.qzzn = qzzn, e.qxzn = qxzn, e.qyzn = qyzn;
                if (xl && xf && yl && yf && zl && zf)
                    energy_voxel_terms<SLOTS, CT, true>(e, h, K, al1, al0, lam, VV, xl, yl, zl, xf, yf, zf, t1, t0, td,
                                                        dv);
                else
                    energy_voxel_terms<SLOTS, CT, false>(e, h, K, al1, al0, lam, VV, xl, yl, zl, xf, yf, zf, t1, t0,
                                                         td, dv);
                vm = fmaxf(vm, fmaxf(fabsf(v0), fmaxf(fabsf(v1), fabsf(v2))));
            }
            // ---- carry
            vm0 = v0, vm1 = v1, vm2 = v2, pzm = p2;
            uc = un, qzz = qzzn, qxz = qxzn, qyz = qyzn;
        }
    }
    __shared__ double red[EN_TERMS][8];
    double vmd = (double)vm;
    t1 = warp_sum(t1);
    t0 = warp_sum(t0);
    td = warp_sum(td);
    dv = warp_sum(dv);
    vmd = warp_max(vmd);
    if (lane == 0) {
        red[0][wid] = t1;
        red[1][wid] = t0;
        red[2][wid] = td;
        red[3][wid] = dv;
        red[4][wid] = vmd;
    }
    __syncthreads();
    if (threadIdx.x < EN_TERMS) {
        const int k = threadIdx.x;
        double s = red[k][0];
        for (int w = 1; w < 8; ++w) s = (k == 4) ? fmax(s, red[k][w]) : s + red[k][w];
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

// tgv_bricks.cuh -- NEXT-3 block-sparse brick sets (include/tgv_bricks.h; R24).
//
// A level is a list of bricks of E^3 voxels (E = 2^LE), each solved (set A) or
// frozen (set B), that reach their six face neighbours through a neighbour table
// (PAPER.md:221-225 stores neighbour references per cube; PAPER.md:446-453 freezes
// the cubes just outside a part).  The difference operators of tgv_kernels.cuh are
// restricted to the union Omega of the bricks: a forward difference exists where the
// forward neighbour voxel is in Omega, exactly as the dense kernels' "l < n-1" masks
// (a box of solved bricks reproduces the SPLIT schedule bit for bit).
//
// Storage: every field slot is one array of nbricks * E^3 floats, brick-major, z, y,
// x inside a brick; a warp covers 32 consecutive voxels of one brick row-block, so
// within a brick the loads are the dense SPLIT kernels' coalesced rows.  Counts:
// [voxel][SLOTS] of u8 / u16.  The rotating slots of tgv_runtime.cu (u, v over 3
// iterates, p, q over 2) are reused as they are.
//
// Kernels (one voxel per thread, 256 threads, every load issued before any store):
//   brick_dual_kernel    p, q at every voxel of S (A + frozen voxels face-adjacent to A)  104 B per voxel
//   brick_primal_kernel  u, v at A (B skipped)                                        76 / 84 B per voxel
//   brick_energy_kernel  fp64 terms, block partials (energy_final_kernel sums them)
#pragma once
#include "tgv_kernels.cuh"

namespace tgvk {

struct BrickGeo {
    int nvox;              // nbricks * E^3 (< 2^31, checked at create)
    const int* nbr;        // [nbricks][6]: brick index of the -x, +x, -y, +y, -z, +z neighbour, or -1
    const uint8_t* frozen; // [nbricks]: 1 = set B
    const uint8_t* aface;  // [nbricks]: bit 2k + d set if the face neighbour along axis k (d = 0: -, 1: +) is solved
};

// voxel i = ((b * E + z) * E + y) * E + x and its face neighbours (-1: outside Omega)
template <int LE>
struct BrickIdx {
    static constexpr int E = 1 << LE;
    int i, b, c[3];
    __device__ __forceinline__ explicit BrickIdx(int i_) : i(i_)
    {
        c[0] = i & (E - 1);
        c[1] = (i >> LE) & (E - 1);
        c[2] = (i >> (2 * LE)) & (E - 1);
        b = i >> (3 * LE);
    }
    // a frozen voxel belongs to S (R24) iff a face neighbour is a solved voxel:
    // it sits on a face of its brick whose neighbour brick across that face is solved
    __device__ __forceinline__ bool on_solved_face(unsigned int af) const
    {
        return ((c[0] == 0) & af) | ((c[0] == E - 1) & (af >> 1)) | ((c[1] == 0) & (af >> 2)) |
               ((c[1] == E - 1) & (af >> 3)) | ((c[2] == 0) & (af >> 4)) | ((c[2] == E - 1) & (af >> 5));
    }
    __device__ __forceinline__ int fwd(const int* __restrict__ nbr, int k) const
    {
        const int st = 1 << (LE * k);
        if (c[k] < E - 1) return i + st;
        const int n = __ldg(nbr + 6 * b + 2 * k + 1);
        return n < 0 ? -1 : i + ((n - b) << (3 * LE)) - (E - 1) * st;
    }
    __device__ __forceinline__ int bwd(const int* __restrict__ nbr, int k) const
    {
        const int st = 1 << (LE * k);
        if (c[k] > 0) return i - st;
        const int n = __ldg(nbr + 6 * b + 2 * k);
        return n < 0 ? -1 : i + ((n - b) << (3 * LE)) + (E - 1) * st;
    }
};

// (a1) at every voxel of S (solved voxels, and frozen voxels face-adjacent to them,
// which lie on the frozen bricks' faces towards solved bricks; the duals elsewhere
// stay 0) -- the expressions of split_dual_kernel with the neighbour masks taken
// from the brick table
// One body, two index spaces (MODE): 0 = every voxel of the solved bricks of `list`
// (n = |list| E^3 threads); 1 = the faces of frozen bricks that touch a solved brick,
// list = (brick, face) pairs, E^2 threads per face (a voxel on two such faces is
// computed twice, identically: reads and writes use different slots).
template <int LE, int MODE>
__device__ __forceinline__ int brick_list_voxel(const int* __restrict__ list, int t)
{
    constexpr int E = 1 << LE;
    if constexpr (MODE == 0) {
        return (__ldg(list + (t >> (3 * LE))) << (3 * LE)) | (t & (E * E * E - 1));
    } else {
        const int j = t >> (2 * LE);
        const int b = __ldg(list + 2 * j), f = __ldg(list + 2 * j + 1);
        const int k = f >> 1, side = (f & 1) ? E - 1 : 0;
        const int a = t & (E - 1), c = (t >> LE) & (E - 1);
        int x, y, z;  // x fastest where the face allows it (coalesced rows)
        if (k == 2) x = a, y = c, z = side;
        else if (k == 1) x = a, y = side, z = c;
        else x = side, y = a, z = c;
        return (((b << LE | z) << LE | y) << LE) | x;
    }
}

template <int LE, int MODE>
__global__ void __launch_bounds__(256) brick_dual_kernel(const IterPtrs a, const BrickGeo bg, const StepParams sp,
                                                         const int* __restrict__ list, int n)
{
    const int t = blockIdx.x * 256 + threadIdx.x;
    if (t >= n) return;
    const int i = brick_list_voxel<LE, MODE>(list, t);
    const BrickIdx<LE> I(i);
    const int fx = I.fwd(bg.nbr, 0), fy = I.fwd(bg.nbr, 1), fz = I.fwd(bg.nbr, 2);
    const int bx = I.bwd(bg.nbr, 0), by = I.bwd(bg.nbr, 1), bz = I.bwd(bg.nbr, 2);
    const bool xl = fx >= 0, yl = fy >= 0, zl = fz >= 0;
    const bool xf = bx >= 0, yf = by >= 0, zf = bz >= 0;
    auto ubar = [&](int o) { return fmaf(2.f, __ldg(a.uk + o), -__ldg(a.um + o)); };
    auto vbar = [&](int k, int o) { return fmaf(2.f, __ldg(a.vk[k] + o), -__ldg(a.vm[k] + o)); };
    const float u0 = ubar(i);
    const float ux = xl ? ubar(fx) : 0.f, uy = yl ? ubar(fy) : 0.f, uz = zl ? ubar(fz) : 0.f;
    float vb[3], vbx[3], vby[3], vbz[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        vb[k] = vbar(k, i);
        vbx[k] = xf ? vbar(k, bx) : 0.f;
        vby[k] = yf ? vbar(k, by) : 0.f;
        vbz[k] = zf ? vbar(k, bz) : 0.f;
    }
    float p[3], q[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) p[k] = __ldg(a.pk[k] + i);
#pragma unroll
    for (int m = 0; m < 6; ++m) q[m] = __ldg(a.qk[m] + i);
    const float g0 = xl ? ux - u0 : 0.f, g1 = yl ? uy - u0 : 0.f, g2 = zl ? uz - u0 : 0.f;
    p[0] = fmaf(sp.sigma, g0 - vb[0], p[0]);
    p[1] = fmaf(sp.sigma, g1 - vb[1], p[1]);
    p[2] = fmaf(sp.sigma, g2 - vb[2], p[2]);
    const float sp_ = proj_scale(p[0] * p[0] + p[1] * p[1] + p[2] * p[2], sp.alpha1);
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

// (a2) + (a3) at A -- the expressions of split_primal_kernel; B is skipped (warp-
// uniform: a brick holds a multiple of 32 voxels): its u and v sit in all three
// rotating slots (tgv_bricks_set_primal / prolong_from), so ubar = u, vbar = v there
template <int LE, int SLOTS, typename CT>
__global__ void __launch_bounds__(256) brick_primal_kernel(const IterPtrs a, const BrickGeo bg, const StepParams sp,
                                                           const Centers C, const int* __restrict__ list, int n)
{
    const int t = blockIdx.x * 256 + threadIdx.x;
    if (t >= n) return;
    const int i = brick_list_voxel<LE, 0>(list, t);  // solved bricks only
    const BrickIdx<LE> I(i);
    const int fx = I.fwd(bg.nbr, 0), fy = I.fwd(bg.nbr, 1), fz = I.fwd(bg.nbr, 2);
    const int bx = I.bwd(bg.nbr, 0), by = I.bwd(bg.nbr, 1), bz = I.bwd(bg.nbr, 2);
    const bool xl = fx >= 0, yl = fy >= 0, zl = fz >= 0;
    const bool xf = bx >= 0, yf = by >= 0, zf = bz >= 0;
    float p[3], q[6], qx[3], qy[3], qz[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) p[k] = __ldg(a.pk[k] + i);
    const float pxm = xf ? __ldg(a.pk[0] + bx) : 0.f;
    const float pym = yf ? __ldg(a.pk[1] + by) : 0.f;
    const float pzm = zf ? __ldg(a.pk[2] + bz) : 0.f;
#pragma unroll
    for (int m = 0; m < 6; ++m) q[m] = __ldg(a.qk[m] + i);
    const int QX[3] = {0, 3, 4}, QY[3] = {3, 1, 5}, QZ[3] = {4, 5, 2};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        qx[k] = xl ? __ldg(a.qk[QX[k]] + fx) : 0.f;
        qy[k] = yl ? __ldg(a.qk[QY[k]] + fy) : 0.f;
        qz[k] = zl ? __ldg(a.qk[QZ[k]] + fz) : 0.f;
    }
    const float uo = __ldg(a.uk + i);
    float vo[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) vo[k] = __ldg(a.vk[k] + i);
    const auto h = load_hist<SLOTS, CT>(a.hist, i);
    const float divp = fmaf(xl ? 1.f : 0.f, p[0], -pxm) + fmaf(yl ? 1.f : 0.f, p[1], -pym) +
                       fmaf(zl ? 1.f : 0.f, p[2], -pzm);
    const float un = hist_prox<SLOTS, CT>(fmaf(sp.tau, divp, uo), sp.tl, h, C);
    float w[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
        w[k] = (xl ? qx[k] - q[QX[k]] : 0.f) + (yl ? qy[k] - q[QY[k]] : 0.f) + (zl ? qz[k] - q[QZ[k]] : 0.f);
    a.un[i] = un;
#pragma unroll
    for (int k = 0; k < 3; ++k) a.vn[k][i] = fmaf(sp.tau, p[k] + w[k], vo[k]);
}

// host counts [nv][nbins] (u8 / u16 / u32) -> u16 [nv][SLOTS] (zero padded), max count
template <typename T, int SLOTS>
__global__ void brick_pack_kernel(const T* __restrict__ src, int64_t nv, int nbins, uint16_t* __restrict__ dst,
                                  unsigned int* __restrict__ maxc)
{
    unsigned int m = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
        for (int b = 0; b < SLOTS; ++b) {
            const unsigned int c = b < nbins ? (unsigned int)src[v * nbins + b] : 0u;
            m = max(m, c);
            dst[v * SLOTS + b] = (uint16_t)min(c, 65535u);
        }
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(FULL, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(maxc, m);
}

// u_0 on A (R9), 0 on B, into the current and previous u slots
template <int LE, int SLOTS, typename CT>
__global__ void brick_init_kernel(float* __restrict__ u_cur, float* __restrict__ u_prev, const void* __restrict__ H,
                                  const BrickGeo bg, const Centers C)
{
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < bg.nvox; v += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)v;
        float u0 = 0.f;
        if (!bg.frozen[i >> (3 * LE)]) {
            const auto h = load_hist<SLOTS, CT>(H, i);
            double W = 0.0, m = 0.0;
            for (int b = 0; b < SLOTS; ++b) {
                const double hb = (double)hist_count<SLOTS, CT>(h, b);
                if (hb != 0.0) {
                    W += hb;
                    m += hb * (double)C.c[b];
                }
            }
            u0 = W > 0.0 ? (float)(m / W) : 0.f;
        }
        u_cur[i] = u0;
        u_prev[i] = u0;
    }
}

// (a4) on a brick set (R24): regulariser over S, data and the box term of
// the dual over A, the frozen primal's saddle term -u div p - v.(p + div2 q) over B
// (duals are 0 outside S); vmax over A.  Partials in the layout of energy_partial_kernel.
template <int LE, int SLOTS, typename CT>
__global__ void __launch_bounds__(256)
    brick_energy_kernel(const EnergyArgs ea, const BrickGeo bg, const EnergyConsts K, double* __restrict__ partials)
{
    double t1 = 0, t0 = 0, td = 0, dv = 0, vm = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < bg.nvox; v += (int64_t)gridDim.x * blockDim.x) {
        const BrickIdx<LE> I((int)v);
        const int i = (int)v;
        const int fw[3] = {I.fwd(bg.nbr, 0), I.fwd(bg.nbr, 1), I.fwd(bg.nbr, 2)};
        const int bw[3] = {I.bwd(bg.nbr, 0), I.bwd(bg.nbr, 1), I.bwd(bg.nbr, 2)};
        const bool frozen = bg.frozen[I.b] != 0;
        auto F = [&](const float* f, int o) { return (double)f[o]; };
        auto dp = [&](const float* f, int k) { return fw[k] >= 0 ? F(f, fw[k]) - F(f, i) : 0.0; };
        auto dm = [&](const float* f, int k) { return (fw[k] >= 0 ? F(f, i) : 0.0) - (bw[k] >= 0 ? F(f, bw[k]) : 0.0); };
        const double u = F(ea.u, i);
        const double v0 = F(ea.v[0], i), v1 = F(ea.v[1], i), v2 = F(ea.v[2], i);
        if (!frozen || I.on_solved_face(bg.aface[I.b])) {  // regulariser over S
            const double a0 = dp(ea.u, 0) - v0, a1 = dp(ea.u, 1) - v1, a2 = dp(ea.u, 2) - v2;
            t1 += ea.alpha1 * sqrt(a0 * a0 + a1 * a1 + a2 * a2);
            const double exx = dm(ea.v[0], 0), eyy = dm(ea.v[1], 1), ezz = dm(ea.v[2], 2);
            const double exy = 0.5 * (dm(ea.v[0], 1) + dm(ea.v[1], 0));
            const double exz = 0.5 * (dm(ea.v[0], 2) + dm(ea.v[2], 0));
            const double eyz = 0.5 * (dm(ea.v[1], 2) + dm(ea.v[2], 1));
            t0 += ea.alpha0 * sqrt(exx * exx + eyy * eyy + ezz * ezz + 2.0 * (exy * exy + exz * exz + eyz * eyz));
        }
        const double divp = dm(ea.p[0], 0) + dm(ea.p[1], 1) + dm(ea.p[2], 2);
        const double w0 = F(ea.p[0], i) + dp(ea.q[0], 0) + dp(ea.q[3], 1) + dp(ea.q[4], 2);
        const double w1 = F(ea.p[1], i) + dp(ea.q[3], 0) + dp(ea.q[1], 1) + dp(ea.q[5], 2);
        const double w2 = F(ea.p[2], i) + dp(ea.q[4], 0) + dp(ea.q[5], 1) + dp(ea.q[2], 2);
        if (frozen) {
            dv += -u * divp - (v0 * w0 + v1 * w1 + v2 * w2);
            continue;
        }
        const auto h = load_hist<SLOTS, CT>(ea.hist, i);
        double data, best;
        data_box_terms<SLOTS, CT>(h, K, ea.lambda, u, divp, data, best);
        td += data;
        dv += best - ea.V * (fabs(w0) + fabs(w1) + fabs(w2));
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
        double s = red[k][0];
        for (int w = 1; w < 8; ++w) s = (k == 4) ? fmax(s, red[k][w]) : s + red[k][w];
        partials[(int64_t)blockIdx.x * EN_TERMS + k] = s;
    }
}

}  // namespace tgvk

// ---------------------------------------------------------------------------
// Brick-set companions of the dense helpers: Alg. 1 votes, count read-back,
// refinement flags, prolongation from the parent level.
#include "tgv_vote.cuh"

namespace tgvk {

// Alg. 1 (NEXT-2) at every voxel of every brick: the voxel centre is
// origin + h (E * brick coordinate + in-brick offset); same per-point arithmetic as
// vote_kernel (vote_point), so a brick's counts equal a dense vote of its box
// Mixed-level sets (R27; levels != NULL): brick b is voted at voxel size h 2^l and radius
// r 2^l of its level l (exact power-of-two scalings), as its level's own dense vote.
template <int LE, int SLOTS>
__global__ void __launch_bounds__(256) brick_vote_kernel(const VoteCam* __restrict__ cams, int ncams,
                                                         const float* __restrict__ depth, const int* __restrict__ coords,
                                                         int nvox, double ox, double oy, double oz, double h0, double r0,
                                                         uint16_t* __restrict__ H, unsigned int* __restrict__ maxc,
                                                         const uint8_t* __restrict__ levels = nullptr)
{
    constexpr int E = 1 << LE;
    unsigned int m = 0;
    for (int64_t vi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; vi < nvox; vi += (int64_t)gridDim.x * blockDim.x) {
        const BrickIdx<LE> I((int)vi);
        const int lv = levels ? levels[I.b] : 0;
        const double h = ldexp(h0, lv), r = ldexp(r0, lv);
        const double delta = __dmul_rn(6.0, r), eta = __dmul_rn(3.0, delta);
        const int gx = coords[3 * I.b] * E + I.c[0], gy = coords[3 * I.b + 1] * E + I.c[1],
                  gz = coords[3 * I.b + 2] * E + I.c[2];
        const double pw0 = __dadd_rn(ox, __dmul_rn(h, (double)gx));
        const double pw1 = __dadd_rn(oy, __dmul_rn(h, (double)gy));
        const double pw2 = __dadd_rn(oz, __dmul_rn(h, (double)gz));
        unsigned int acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        vote_point(cams, ncams, depth, pw0, pw1, pw2, r, delta, eta, acc);
        uint16_t* dst = H + vi * SLOTS;
#pragma unroll
        for (int b = 0; b < SLOTS; ++b) {
            const unsigned int cb = b < 8 ? acc[b] : 0u;
            m = max(m, cb);
            dst[b] = (uint16_t)min(cb, 65535u);
        }
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(FULL, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(maxc, m);
}

// stored counts -> uint32 [nvox][nbins]
template <typename CT>
__global__ void brick_unpack_kernel(const CT* __restrict__ H, int64_t nvox, int slots, int nbins,
                                    uint32_t* __restrict__ out)
{
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvox; v += (int64_t)gridDim.x * blockDim.x)
        for (int b = 0; b < nbins; ++b) out[v * nbins + b] = H[v * slots + b];
}

// flags[b * 8 + octant] = 1 if a voxel of solved brick b in that octant has at least
// min_votes votes outside the last (free-space) bin; the caller zeroes flags
template <int LE, typename CT>
__global__ void brick_refine_kernel(const CT* __restrict__ H, const uint8_t* __restrict__ frozen, int nvox, int slots,
                                    int nbins, int min_votes, uint8_t* __restrict__ flags)
{
    constexpr int E = 1 << LE;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nvox; v += (int64_t)gridDim.x * blockDim.x) {
        const BrickIdx<LE> I((int)v);
        if (frozen[I.b]) continue;
        int s = 0;
        for (int b = 0; b < nbins - 1; ++b) s += H[v * slots + b];
        if (s >= min_votes) {
            const int oct = (I.c[0] >= E / 2) | (I.c[1] >= E / 2) << 1 | (I.c[2] >= E / 2) << 2;
            flags[I.b * 8 + oct] = 1;  // identical writes only
        }
    }
}

// Prolongation from the parent level (R19 on brick sets): fine voxel
// (brick b, offset c) lies in parent brick parent[b] at offset (E (coord_b & 1) + c) / 2;
// u = parent u, v = parent v / 2 into all three rotating slots (the frozen bricks are
// never written again)
template <int LE>
__global__ void brick_prolong_kernel(const float* __restrict__ uc, const float* __restrict__ vc0,
                                     const float* __restrict__ vc1, const float* __restrict__ vc2,
                                     const int* __restrict__ parent, const int* __restrict__ coords, int nvox,
                                     float* __restrict__ u_cur, float* __restrict__ u_prev, float* __restrict__ u_next,
                                     float* __restrict__ v_cur0, float* __restrict__ v_cur1, float* __restrict__ v_cur2,
                                     float* __restrict__ v_prev0, float* __restrict__ v_prev1,
                                     float* __restrict__ v_prev2, float* __restrict__ v_next0,
                                     float* __restrict__ v_next1, float* __restrict__ v_next2,
                                     const uint8_t* __restrict__ levels = nullptr)
{
    constexpr int E = 1 << LE;
    for (int64_t vi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; vi < nvox; vi += (int64_t)gridDim.x * blockDim.x) {
        const BrickIdx<LE> I((int)vi);
        const int pb = parent[I.b];
        int px = ((coords[3 * I.b] & 1) * E + I.c[0]) >> 1;
        int py = ((coords[3 * I.b + 1] & 1) * E + I.c[1]) >> 1;
        int pz = ((coords[3 * I.b + 2] & 1) * E + I.c[2]) >> 1;
        if (levels && levels[I.b] == 1) {  // a mixed set's level-1 brick is its parent level's own brick
            px = I.c[0];
            py = I.c[1];
            pz = I.c[2];
        }
        const int j = (((pb << LE) + pz) << LE | py) << LE | px;
        const float u = uc[j];
        const float v0 = 0.5f * vc0[j], v1 = 0.5f * vc1[j], v2 = 0.5f * vc2[j];
        u_cur[vi] = u;
        u_prev[vi] = u;
        u_next[vi] = u;
        v_cur0[vi] = v0;
        v_prev0[vi] = v0;
        v_next0[vi] = v0;
        v_cur1[vi] = v1;
        v_prev1[vi] = v1;
        v_next1[vi] = v1;
        v_cur2[vi] = v2;
        v_prev2[vi] = v2;
        v_next2[vi] = v2;
    }
}

}  // namespace tgvk

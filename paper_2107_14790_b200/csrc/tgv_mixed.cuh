// tgv_mixed.cuh -- NEXT-3 2:1 mixed-level brick sets (include/tgv_bricks.h
// tgv_bricks_create_mixed; reading R27).
//
// The paper's octree is 2:1 balanced, "leading to the point when each cube has only 4
// or less neighbors over each face"; a part's border cubes are the
// frozen parents.  Here every brick carries a level l (voxel edge
// h = 2^l in finest-level units) and a face of a brick is one of
//   kind 0  none                      (Neumann)
//   kind 1  a brick of the same level (the R24 operators scaled by 1/h)
//   kind 2  a brick one level coarser (each voxel faces one coarse voxel)
//   kind 3  up to four bricks one level finer, one per quadrant of the face (each
//           voxel faces 2 x 2 fine voxels of one of them)
// and R27's operators are, for voxel i and axis k:
//   D+_k u(i) = (mean of u over the +k face neighbours - u(i)) / d,   d = (h_i + h_n) / 2
//   D-_k p(i) = b_i p(i) - c_i * (sum of p over the -k face neighbours),
//     b_i = 1/d of i's own forward difference (0 without + neighbours),
//     c_i = 1/h (same level), 4/(3h) (one coarser neighbour), 1/(6h) (four finer):
//   the adjoint of D+ in the cell-volume-weighted inner product (the CPU pins write
//   these cases out by hand).  With every brick at level 0 the expressions are
//   the uniform brick kernels' (tgv_bricks.cuh) term for term, so a one-level set is
//   the SPLIT brick schedule bit for bit (tests/test_gpu_mixed.py).
//
// SPLIT schedule, one voxel per thread (the brick kernels' layout and lists):
//   mixed_dual_kernel    p, q on S (solved voxels; frozen voxels on faces towards a solved
//                        neighbour, restricted to the quadrants whose neighbour is solved)
//   mixed_primal_kernel  u, v on A
//   mixed_energy_kernel  h^3-weighted fp64 terms, partials for energy_final_kernel
#pragma once
#include "tgv_bricks.cuh"

namespace tgvk {

struct MixGeo {
    int nvox;
    const uint8_t* level;   // [nbricks]
    const uint8_t* kind;    // [nbricks][6] faces -x, +x, -y, +y, -z, +z
    const int* nbr4;        // [nbricks][6][4]: kind 1 / 2: [0]; kind 3: quadrant q (-1 absent)
    const uint8_t* par;     // [nbricks]: bit k = brick coordinate k & 1
    const uint8_t* frozen;  // [nbricks]
    const uint8_t* sface;   // [nbricks][6]: bit q set if the neighbour voxels of quadrant q are solved
};

// lateral axes of axis k (increasing) and the quadrant of a face voxel
__device__ __forceinline__ void lat_axes(int k, int& l0, int& l1)
{
    l0 = k == 0 ? 1 : 0;
    l1 = k == 2 ? 1 : 2;
}

template <int LE>
struct MixIdx {
    static constexpr int E = 1 << LE;
    int i, b, c[3], lev;
    float h;
    __device__ __forceinline__ MixIdx(int i_, const MixGeo& g) : i(i_)
    {
        c[0] = i & (E - 1);
        c[1] = (i >> LE) & (E - 1);
        c[2] = (i >> (2 * LE)) & (E - 1);
        b = i >> (3 * LE);
        lev = __ldg(g.level + b);
        h = (float)(1 << lev);
    }
    __device__ __forceinline__ static int vox(int brick, int x, int y, int z)
    {
        return (((brick << LE | z) << LE | y) << LE) | x;
    }
    __device__ __forceinline__ int quad(int k) const
    {
        int l0, l1;
        lat_axes(k, l0, l1);
        return (c[l0] >= E / 2 ? 1 : 0) | (c[l1] >= E / 2 ? 2 : 0);
    }
    // the face neighbours of voxel i across its face (k, side): n (0, 1 or 4) voxel indices;
    // kind of the face (1 inside the brick)
    __device__ __forceinline__ int face(const MixGeo& g, int k, int side, int idx[4], int& n) const
    {
        const int st = 1 << (LE * k);
        const bool inner = side ? c[k] < E - 1 : c[k] > 0;
        if (inner) {
            idx[0] = side ? i + st : i - st;
            n = 1;
            return 1;
        }
        const int f = 2 * k + side;
        const int kd = __ldg(g.kind + 6 * b + f);
        n = 0;
        if (kd == 0) return 0;
        int l0, l1;
        lat_axes(k, l0, l1);
        int cc[3] = {c[0], c[1], c[2]};
        cc[k] = side ? 0 : E - 1;  // the neighbour's voxel layer touching this face
        if (kd == 1) {
            idx[0] = vox(__ldg(g.nbr4 + 4 * (6 * b + f)), cc[0], cc[1], cc[2]);
            n = 1;
        } else if (kd == 2) {  // coarser: the quadrant of its face this brick covers
            const int pr = __ldg(g.par + b);
            cc[l0] = (((pr >> l0) & 1) * E + c[l0]) >> 1;
            cc[l1] = (((pr >> l1) & 1) * E + c[l1]) >> 1;
            idx[0] = vox(__ldg(g.nbr4 + 4 * (6 * b + f)), cc[0], cc[1], cc[2]);
            n = 1;
        } else {  // finer: 2 x 2 voxels of the quadrant's brick
            const int q = quad(k);
            const int fb = __ldg(g.nbr4 + 4 * (6 * b + f) + q);
            if (fb < 0) return 3;
            cc[l0] = 2 * c[l0] - ((q & 1) ? E : 0);
            cc[l1] = 2 * c[l1] - ((q & 2) ? E : 0);
            const int base = vox(fb, cc[0], cc[1], cc[2]);
            const int s0 = 1 << (LE * l0), s1 = 1 << (LE * l1);
            idx[0] = base;
            idx[1] = base + s0;
            idx[2] = base + s1;
            idx[3] = base + s0 + s1;
            n = 4;
        }
        return kd;
    }
};

// one axis of R27's stencil at a voxel: forward set (mean, 1/d) and backward set (sum, c)
struct MixAxis {
    int fn, bn, kf, kb;  // set sizes (0, 1, 4) and face kinds
    int fi[4], bi[4];
    float inv_d;  // b_i of D- (0 without + neighbours)
    float cb;     // c_i of D-
};
// the same coefficients in fp64 (energy)
__device__ __forceinline__ double mix_inv_d64(const MixAxis& a, double ih)
{
    return a.fn == 0 ? 0.0 : (a.kf == 1 ? ih : (a.kf == 2 ? ih * (2.0 / 3.0) : ih * (4.0 / 3.0)));
}
__device__ __forceinline__ double mix_cb64(const MixAxis& a, double ih)
{
    return a.bn == 0 ? 0.0 : (a.kb == 1 ? ih : (a.kb == 2 ? ih * (4.0 / 3.0) : ih * (1.0 / 6.0)));
}
__device__ __forceinline__ double mix_dplus64(const MixAxis& a, const float* __restrict__ f, double ctr, double ih)
{
    if (a.fn == 0) return 0.0;
    auto F = [&](int o) { return (double)__ldg(f + o); };
    const double m = a.fn == 1 ? F(a.fi[0]) : 0.25 * ((F(a.fi[0]) + F(a.fi[1])) + (F(a.fi[2]) + F(a.fi[3])));
    return (m - ctr) * mix_inv_d64(a, ih);
}
__device__ __forceinline__ double mix_dminus64(const MixAxis& a, const float* __restrict__ f, double ctr, double ih)
{
    auto F = [&](int o) { return (double)__ldg(f + o); };
    double s = 0.0;
    if (a.bn == 1) s = F(a.bi[0]);
    else if (a.bn == 4) s = (F(a.bi[0]) + F(a.bi[1])) + (F(a.bi[2]) + F(a.bi[3]));
    return mix_inv_d64(a, ih) * ctr - mix_cb64(a, ih) * s;
}

template <int LE>
__device__ __forceinline__ MixAxis mix_axis(const MixIdx<LE>& I, const MixGeo& g, int k)
{
    MixAxis a;
    const int kf = I.face(g, k, 1, a.fi, a.fn);
    const int kb = I.face(g, k, 0, a.bi, a.bn);
    a.kf = kf;
    a.kb = kb;
    const float ih = 1.f / I.h;  // exact: h is a power of two
    a.inv_d = a.fn == 0 ? 0.f : (kf == 1 ? ih : (kf == 2 ? ih * (2.f / 3.f) : ih * (4.f / 3.f)));
    a.cb = a.bn == 0 ? 0.f : (kb == 1 ? ih : (kb == 2 ? ih * (4.f / 3.f) : ih * (1.f / 6.f)));
    return a;
}

// D+ of a field given its value at the voxel (loads of the forward set)
template <typename F>
__device__ __forceinline__ float mix_dplus(const MixAxis& a, float center, F&& load)
{
    if (a.fn == 0) return 0.f;
    const float m = a.fn == 1 ? load(a.fi[0]) : 0.25f * ((load(a.fi[0]) + load(a.fi[1])) + (load(a.fi[2]) + load(a.fi[3])));
    return (m - center) * a.inv_d;
}
// the backward sum times c_i (0 without - neighbours)
template <typename F>
__device__ __forceinline__ float mix_bsum(const MixAxis& a, F&& load)
{
    if (a.bn == 0) return 0.f;
    const float s = a.bn == 1 ? load(a.bi[0]) : (load(a.bi[0]) + load(a.bi[1])) + (load(a.bi[2]) + load(a.bi[3]));
    return a.cb * s;
}

// (a1) on S: MODE 0 every voxel of the solved bricks in `list`; MODE 1 the faces of
// frozen bricks towards solved neighbours, list = (brick, face | quadrant mask << 3)
// pairs, E^2 threads per face (threads outside the mask return)
template <int LE, int MODE>
__global__ void __launch_bounds__(256) mixed_dual_kernel(const IterPtrs a, const MixGeo g, const StepParams sp,
                                                         const int* __restrict__ list, int n)
{
    constexpr int E = 1 << LE;
    const int t = blockIdx.x * 256 + threadIdx.x;
    if (t >= n) return;
    int i;
    if constexpr (MODE == 0) {
        i = brick_list_voxel<LE, 0>(list, t);
    } else {
        const int j = t >> (2 * LE);
        const int b = __ldg(list + 2 * j), fm = __ldg(list + 2 * j + 1);
        const int f = fm & 7, mask = fm >> 3;
        const int k = f >> 1, side = (f & 1) ? E - 1 : 0;
        const int aa = t & (E - 1), cc = (t >> LE) & (E - 1);
        int x, y, z;
        if (k == 2) x = aa, y = cc, z = side;
        else if (k == 1) x = aa, y = side, z = cc;
        else x = side, y = aa, z = cc;
        int l0, l1, c3[3] = {x, y, z};
        lat_axes(k, l0, l1);
        const int q = (c3[l0] >= E / 2 ? 1 : 0) | (c3[l1] >= E / 2 ? 2 : 0);
        if (!((mask >> q) & 1)) return;
        i = MixIdx<LE>::vox(b, x, y, z);
    }
    const MixIdx<LE> I(i, g);
    const MixAxis ax[3] = {mix_axis<LE>(I, g, 0), mix_axis<LE>(I, g, 1), mix_axis<LE>(I, g, 2)};
    auto ubar = [&](int o) { return fmaf(2.f, __ldg(a.uk + o), -__ldg(a.um + o)); };
    const float u0 = ubar(i);
    float gr[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) gr[k] = mix_dplus(ax[k], u0, ubar);
    float vb[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) vb[k] = fmaf(2.f, __ldg(a.vk[k] + i), -__ldg(a.vm[k] + i));
    // D-_l vbar_k for every (k, l)
    float dm[3][3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        auto vbk = [&](int o) { return fmaf(2.f, __ldg(a.vk[k] + o), -__ldg(a.vm[k] + o)); };
#pragma unroll
        for (int l = 0; l < 3; ++l) dm[k][l] = fmaf(ax[l].inv_d, vb[k], -mix_bsum(ax[l], vbk));
    }
    float p[3], q[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) p[k] = __ldg(a.pk[k] + i);
#pragma unroll
    for (int m = 0; m < 6; ++m) q[m] = __ldg(a.qk[m] + i);
#pragma unroll
    for (int k = 0; k < 3; ++k) p[k] = fmaf(sp.sigma, gr[k] - vb[k], p[k]);
    const float sp_ = proj_scale(p[0] * p[0] + p[1] * p[1] + p[2] * p[2], sp.alpha1);
    const float e[6] = {dm[0][0], dm[1][1], dm[2][2], 0.5f * (dm[0][1] + dm[1][0]), 0.5f * (dm[0][2] + dm[2][0]),
                        0.5f * (dm[1][2] + dm[2][1])};
#pragma unroll
    for (int m = 0; m < 6; ++m) q[m] = fmaf(sp.sigma, e[m], q[m]);
    const float sq = proj_scale(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + 2.f * (q[3] * q[3] + q[4] * q[4] + q[5] * q[5]),
                                sp.alpha0);
#pragma unroll
    for (int k = 0; k < 3; ++k) a.pn[k][i] = p[k] * sp_;
#pragma unroll
    for (int m = 0; m < 6; ++m) a.qn[m][i] = q[m] * sq;
}

// (a2) + (a3) on A (u, v of B never change)
template <int LE, int SLOTS, typename CT>
__global__ void __launch_bounds__(256) mixed_primal_kernel(const IterPtrs a, const MixGeo g, const StepParams sp,
                                                           const Centers C, const int* __restrict__ list, int n)
{
    const int t = blockIdx.x * 256 + threadIdx.x;
    if (t >= n) return;
    const int i = brick_list_voxel<LE, 0>(list, t);
    const MixIdx<LE> I(i, g);
    const MixAxis ax[3] = {mix_axis<LE>(I, g, 0), mix_axis<LE>(I, g, 1), mix_axis<LE>(I, g, 2)};
    float p[3], q[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) p[k] = __ldg(a.pk[k] + i);
#pragma unroll
    for (int m = 0; m < 6; ++m) q[m] = __ldg(a.qk[m] + i);
    float divp = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        auto pk = [&](int o) { return __ldg(a.pk[k] + o); };
        divp += fmaf(ax[k].inv_d, p[k], -mix_bsum(ax[k], pk));
    }
    const int QI[3][3] = {{0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
    float w[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float s = 0.f;
#pragma unroll
        for (int l = 0; l < 3; ++l) {
            const float* qf = a.qk[QI[k][l]];
            s += mix_dplus(ax[l], q[QI[k][l]], [&](int o) { return __ldg(qf + o); });
        }
        w[k] = s;
    }
    const float uo = __ldg(a.uk + i);
    const auto h = load_hist<SLOTS, CT>(a.hist, i);
    const float un = hist_prox<SLOTS, CT>(fmaf(sp.tau, divp, uo), sp.tl, h, C);
    a.un[i] = un;
#pragma unroll
    for (int k = 0; k < 3; ++k) a.vn[k][i] = fmaf(sp.tau, p[k] + w[k], __ldg(a.vk[k] + i));
}

// (a4) on a mixed set: every term h^3-weighted (R27); regulariser over S, data and the
// box term of the dual over A, the frozen saddle term over B; vmax over A.
template <int LE, int SLOTS, typename CT>
__global__ void __launch_bounds__(256)
    mixed_energy_kernel(const EnergyArgs ea, const MixGeo g, const EnergyConsts K, double* __restrict__ partials)
{
    constexpr int E = 1 << LE;
    double t1 = 0, t0 = 0, td = 0, dv = 0, vm = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < g.nvox; v += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)v;
        const MixIdx<LE> I(i, g);
        const MixAxis ax[3] = {mix_axis<LE>(I, g, 0), mix_axis<LE>(I, g, 1), mix_axis<LE>(I, g, 2)};
        const bool frozen = __ldg(g.frozen + I.b) != 0;
        bool inS = !frozen;
        if (frozen) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int q = I.quad(k);
                if (I.c[k] == 0) inS |= (__ldg(g.sface + 6 * I.b + 2 * k) >> q) & 1;
                if (I.c[k] == E - 1) inS |= (__ldg(g.sface + 6 * I.b + 2 * k + 1) >> q) & 1;
            }
        }
        const double w = (double)I.h * I.h * I.h;  // cell volume
        const double ih = 1.0 / (double)I.h;
        auto F = [](const float* f, int o) { return (double)__ldg(f + o); };
        const double u = F(ea.u, i);
        const double v0 = F(ea.v[0], i), v1 = F(ea.v[1], i), v2 = F(ea.v[2], i);
        const double vv[3] = {v0, v1, v2};
        const float* vf[3] = {ea.v[0], ea.v[1], ea.v[2]};
        auto Dp = [&](int k, const float* f, double ctr) { return mix_dplus64(ax[k], f, ctr, ih); };
        auto Dm = [&](int k, const float* f, double ctr) { return mix_dminus64(ax[k], f, ctr, ih); };
        if (inS) {
            const double a0 = Dp(0, ea.u, u) - v0, a1 = Dp(1, ea.u, u) - v1, a2 = Dp(2, ea.u, u) - v2;
            t1 += w * ea.alpha1 * sqrt(a0 * a0 + a1 * a1 + a2 * a2);
            double dm[3][3];
            for (int k = 0; k < 3; ++k)
                for (int l = 0; l < 3; ++l) dm[k][l] = Dm(l, vf[k], vv[k]);
            const double exy = 0.5 * (dm[0][1] + dm[1][0]), exz = 0.5 * (dm[0][2] + dm[2][0]),
                         eyz = 0.5 * (dm[1][2] + dm[2][1]);
            t0 += w * ea.alpha0 *
                  sqrt(dm[0][0] * dm[0][0] + dm[1][1] * dm[1][1] + dm[2][2] * dm[2][2] +
                       2.0 * (exy * exy + exz * exz + eyz * eyz));
        }
        const double divp = Dm(0, ea.p[0], F(ea.p[0], i)) + Dm(1, ea.p[1], F(ea.p[1], i)) + Dm(2, ea.p[2], F(ea.p[2], i));
        const int QI[3][3] = {{0, 3, 4}, {3, 1, 5}, {4, 5, 2}};
        double wq[3];
        for (int k = 0; k < 3; ++k) {
            double s = F(ea.p[k], i);
            for (int l = 0; l < 3; ++l) s += Dp(l, ea.q[QI[k][l]], F(ea.q[QI[k][l]], i));
            wq[k] = s;
        }
        if (frozen) {
            dv += w * (-u * divp - (v0 * wq[0] + v1 * wq[1] + v2 * wq[2]));
            continue;
        }
        const auto hh = load_hist<SLOTS, CT>(ea.hist, i);
        double data, best;
        data_box_terms<SLOTS, CT>(hh, K, ea.lambda, u, divp, data, best);
        td += w * data;
        dv += w * (best - ea.V * (fabs(wq[0]) + fabs(wq[1]) + fabs(wq[2])));
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
        for (int ww = 1; ww < 8; ++ww) s = (k == 4) ? fmax(s, red[k][ww]) : s + red[k][ww];
        partials[(int64_t)blockIdx.x * EN_TERMS + k] = s;
    }
}

}  // namespace tgvk

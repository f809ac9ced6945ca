// tgv_bricks_fused.cuh -- single-sweep iteration over the solved bricks of a brick set
// (NEXT-3; R24, §5).  One launch per iteration after the frozen-face dual
// launch (brick_dual_kernel<LE, 1>, which stores the duals of S on the frozen
// bricks); 128 B per solved voxel-iteration with u8 counts instead of the SPLIT
// schedule's 180.
//
// CTA = one solved brick (E = 32) and one half of its rows (TY = 16 owned rows),
// 20 warps:
//   warps 0 .. 17 : one row each, y = y0 - 1 + w (rows 0 and 17 are the y-halo),
//                   lane = x (the 32 columns of the brick)
//   warp 18 / 19  : the x-halo columns x = -1 / x = 32, lane = row (0 .. 17)
// marching the planes s = -1 .. E: step s computes the dual D(s) and the primal of
// plane s - 1, exactly as fused_tma_kernel does on the dense grid, with the same
// expressions as brick_dual_kernel / brick_primal_kernel (the schedules agree bit
// for bit).  Halo cells lie in the face and edge neighbour bricks (a 27-entry
// neighbour table per solved brick); their duals are recomputed from the inputs of
// iteration k and never stored (a solved neighbour stores its own, the frozen-face
// launch stores those of S on frozen bricks).  Cells outside Omega load 0 and every
// stencil term that reaches them is masked as in the SPLIT kernels.  x and y
// neighbours go through two parity-double-buffered shared planes (one __syncthreads
// per step), z neighbours stay in registers, inputs are prefetched one plane ahead.
#pragma once
#include "tgv_bricks.cuh"

namespace tgvk {

constexpr int BF_TY = 16;            // owned rows per CTA
constexpr int BF_R = BF_TY + 2;      // rows incl. the y-halo
constexpr int BF_W = 34;             // exchange-plane width: x = -1 .. 32
constexpr int BF_WARPS = BF_R + 2;   // + the two x-halo warps

struct BrickFusedSmem {
    float suv[2][4][BF_R][BF_W];  // ubar, vbar(3) of plane s (parity)
    float sr[2][7][BF_R][BF_W];   // p_x, p_y, q_xx, q_xy, q_xz, q_yy, q_yz of D(s) (parity)
    float xb[3][2][BF_R][8];      // x-face cells (plane mod 3, column): v_k, v_{k-1} at x = -2 / u_k, u_{k-1} at x = E + 1
    float hr[4][2][32][17];       // x-halo columns' inputs (plane mod 4, column, lane): u_k, u_{k-1}, v_k(3), v_{k-1}(3), p(3), q(6)
    int nb[27];
};

// 4-byte asynchronous global -> shared copy (no register staging; visible to the
// issuing thread after cp.async.wait_all)
__device__ __forceinline__ void bf_cp_async4(void* dst, const float* src)
{
    asm volatile(
        "{\n .reg .u64 g;\n cvta.to.global.u64 g, %1;\n cp.async.ca.shared.global [%0], [g], 4;\n}\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(dst)),
        "l"(src)
        : "memory");
}

struct BrickFusedArgs {
    IterPtrs a;
    StepParams sp;
    Centers C;
    const int* nb27;  // [n_alist][27]: brick index at (dz+1)*9 + (dy+1)*3 + (dx+1) around each solved brick, or -1
    const uint8_t* frozen;  // [nbricks]
    int n_alist;
    int fold_x;             // 1: this kernel stores the frozen x-faces' duals (else the face launch does)
};

template <int LE, int SLOTS, typename CT>
__global__ void __launch_bounds__(32 * BF_WARPS, 1) brick_fused_kernel(const BrickFusedArgs A)
{
    constexpr int E = 1 << LE;
    static_assert(E == 2 * BF_TY, "two CTAs per brick");
    extern __shared__ __align__(16) uint8_t bf_smem[];  // BrickFusedSmem (54 KB: dynamic)
    BrickFusedSmem& S = *reinterpret_cast<BrickFusedSmem*>(bf_smem);
    auto& suv = S.suv;
    auto& sr = S.sr;
    auto& nb = S.nb;
    const IterPtrs& a = A.a;
    const StepParams& sp = A.sp;
    const int lane = threadIdx.x, w = threadIdx.y;
    const int j = blockIdx.x >> 1, y0 = (blockIdx.x & 1) * BF_TY;
    if (w == 0 && lane < 27) nb[lane] = __ldg(A.nb27 + 27 * j + lane);
    __syncthreads();

    // ---- this thread's cell column (x, y), relative to the brick
    int r, x;
    if (w < BF_R) {
        r = w, x = lane;
    } else {
        r = min(lane, BF_R - 1), x = (w == BF_R) ? -1 : E;
    }
    const int y = y0 - 1 + r, cc = x + 1;
    const int role = w == BF_R ? 3 : (w == BF_R + 1 ? 4 : (r == 0 ? 1 : (r == BF_R - 1 ? 2 : 0)));
    // roles: 0 owned row (p, q, primal), 1 bottom halo row (p), 2 top halo row (q),
    //        3 column x = -1 (p on the owned rows), 4 column x = E (q on the owned rows)
    const bool haloq_row = (role == 4) && r >= 1 && r <= BF_TY;
    const bool halop_row = (role == 3) && r >= 1 && r <= BF_TY;
    // a frozen x-neighbour: its face cells (x = -1 or E on the owned rows) are in S, and
    // this CTA computes and stores their full duals (the frozen-face launch does y and z
    // faces only): x-faces are strided in the x-major bricks, this warp reads them anyway
    const bool xm_fz = A.fold_x && nb[12] >= 0 && __ldg(A.frozen + nb[12]);
    const bool xp_fz = A.fold_x && nb[14] >= 0 && __ldg(A.frozen + nb[14]);
    const bool xface = (role == 3 && xm_fz && halop_row) || (role == 4 && xp_fz && haloq_row);
    const bool needP = role == 0 || role == 1 || halop_row || xface;
    const bool needQ = role == 0 || role == 2 || haloq_row || xface;
    auto dcoord = [](int c) { return c < 0 ? -1 : (c >= E ? 1 : 0); };
    auto brick_at = [&](int xx, int yy, int dz) { return nb[(dz + 1) * 9 + (dcoord(yy) + 1) * 3 + dcoord(xx) + 1]; };
    // existence of the neighbours this cell's stencils reach, per brick layer dz = -1, 0, 1
    // (bit d + 1 of each mask; registers, no dynamically indexed arrays)
    unsigned own_ex = 0, xl_m = 0, yl_m = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        own_ex |= (brick_at(x, y, d - 1) >= 0) << d;
        xl_m |= (brick_at(x + 1, y, d - 1) >= 0) << d;
        yl_m |= (brick_at(x, y + 1, d - 1) >= 0) << d;
    }
    const bool xf0 = brick_at(x - 1, y, 0) >= 0, yf0 = brick_at(x, y - 1, 0) >= 0;
    const int xin = x - dcoord(x) * E, yin = y - dcoord(y) * E;
    const int col = (yin << LE) | xin;
    // element index of (xin, yin, z = 0) in the brick of layer dz = -1, 0, 1, or -1
    const int bm = brick_at(x, y, -1), b0 = brick_at(x, y, 0), bp = brick_at(x, y, 1);
    const int base_m = bm < 0 ? -1 : (bm << (3 * LE)) | col;
    const int base_0 = b0 < 0 ? -1 : (b0 << (3 * LE)) | col;
    const int base_p = bp < 0 ? -1 : (bp << (3 * LE)) | col;
    auto at = [&](int s) {  // element index of plane s of this column, or -1
        if (s < -1 || s > E + 1) return -1;
        const int bb = s < 0 ? base_m : (s >= E ? base_p : base_0);
        const int zin = s < 0 ? s + E : (s >= E ? s - E : s);
        return bb < 0 ? -1 : bb + (zin << (2 * LE));
    };
    auto bit = [](unsigned m, int s) { return ((m >> (s < 0 ? 0 : (s >= E ? 2 : 1))) & 1u) != 0; };

    struct U2 {
        float uk, um;
    };
    struct X {
        float vk[3], vm[3], p[3], q[6];
    };
    auto load_u = [&](int s) {
        U2 o{0.f, 0.f};
        if (role >= 3) return o;  // x-halo columns: staged by cp.async (hissue)
        const int i = at(s);
        if (i >= 0) {
            o.uk = __ldg(a.uk + i);
            o.um = __ldg(a.um + i);
        }
        return o;
    };
    auto load_x = [&](int s) {
        X o{};
        if (role >= 3) return o;
        const int i = (s <= E) ? at(s) : -1;
        if (i >= 0) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                o.vk[k] = __ldg(a.vk[k] + i);
                o.vm[k] = __ldg(a.vm[k] + i);
            }
            if (needP) {
#pragma unroll
                for (int k = 0; k < 3; ++k) o.p[k] = __ldg(a.pk[k] + i);
            }
            if (needQ) {
#pragma unroll
                for (int m = 0; m < 6; ++m) o.q[m] = __ldg(a.qk[m] + i);
            }
        }
        return o;
    };
    auto load_h = [&](int s) {
        HistRaw<SLOTS, CT> h{};
        if (role == 0 && s >= 0 && s < E) h = load_hist<SLOTS, CT>(a.hist, base_0 + (s << (2 * LE)));
        return h;
    };

    auto xissue = [&](int t) {  // x-face cells: plane t's second column into smem
        float* d = S.xb[(t + 3) % 3][role - 3][r];
        const int i = at(t);
        if (i < 0) {
#pragma unroll
            for (int k = 0; k < 6; ++k) d[k] = 0.f;
        } else if (role == 3) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                bf_cp_async4(d + k, a.vk[k] + i - 1);
                bf_cp_async4(d + 3 + k, a.vm[k] + i - 1);
            }
        } else {
            bf_cp_async4(d, a.uk + i + 1);
            bf_cp_async4(d + 1, a.um + i + 1);
        }
    };
    // x-halo columns: their inputs are one strided 4-B value per 32-B sector, so they come
    // by cp.async two planes ahead of use (u one more: ubar at s+1) instead of one plane
    // ahead in registers.  One commit group per plane; each lane owns its ring row.
    auto hissue = [&](int t) {
        float* d = S.hr[(t + 4) & 3][role - 3][lane];
        const int i = (t <= E + 1) ? at(t) : -1;
        if (i < 0) {
#pragma unroll
            for (int f = 0; f < 17; ++f) d[f] = 0.f;
        } else {
            bf_cp_async4(d + 0, a.uk + i);
            bf_cp_async4(d + 1, a.um + i);
            if (t <= E) {
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    bf_cp_async4(d + 2 + k, a.vk[k] + i);
                    bf_cp_async4(d + 5 + k, a.vm[k] + i);
                }
                if (needP) {
#pragma unroll
                    for (int k = 0; k < 3; ++k) bf_cp_async4(d + 8 + k, a.pk[k] + i);
                }
                if (needQ) {
#pragma unroll
                    for (int m = 0; m < 6; ++m) bf_cp_async4(d + 11 + m, a.qk[m] + i);
                }
            }
        }
    };
    // commit groups of the x-halo columns: G(s) = {h(s+3), x(s+2)}, issued at step s; at
    // step s all but the newest group have landed: h(s), h(s+1), x(s)
    if (role >= 3) {
        hissue(-1);
        hissue(0);
        if (xface) xissue(-1);
        asm volatile("cp.async.commit_group;" ::: "memory");
        hissue(1);
        if (xface) xissue(0);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }

    struct Carry {
        float vb[3];      // vbar(s-1)
        float uk, vk[3];  // u_k, v_k at s-1
        HistRaw<SLOTS, CT> h;
        float pn[3], pz;  // p_{k+1}(s-1), p_z{k+1}(s-2)
        float qn[6];      // q_{k+1}(s-1)
    };
    Carry ca{};
    U2 u0 = load_u(-1), u1 = load_u(0);
    X x0 = load_x(-1);
    HistRaw<SLOTS, CT> h0{};

    for (int s = -1; s <= E; ++s) {
        const int par = s & 1, pr = par ^ 1;
        // prefetch: u at s+2, the other fields and the counts at s+1
        const U2 u2 = load_u(s + 2);
        const X x1 = load_x(s + 1);
        const HistRaw<SLOTS, CT> h1 = load_h(s + 1);

        const bool xl = bit(xl_m, s), yl = bit(yl_m, s), zl = bit(own_ex, s + 1);
        if (role >= 3) {  // the x-halo columns' current planes from the ring
            asm volatile("cp.async.wait_group 1;" ::: "memory");
            const float* d0 = S.hr[(s + 4) & 3][role - 3][lane];
            const float* d1 = S.hr[(s + 5) & 3][role - 3][lane];
            u0.uk = d0[0], u0.um = d0[1], u1.uk = d1[0], u1.um = d1[1];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                x0.vk[k] = d0[2 + k];
                x0.vm[k] = d0[5 + k];
                x0.p[k] = d0[8 + k];
            }
#pragma unroll
            for (int m = 0; m < 6; ++m) x0.q[m] = d0[11 + m];
        }
        // x-face cells: the second column into the frozen brick (same 32-B sectors),
        // copied one plane ahead with cp.async
        float ux2 = 0.f, vbx2[3] = {0.f, 0.f, 0.f};
        if (xface) {  // landed with G(s-2)
            const float* xv = S.xb[(s + 3) % 3][role - 3][r];
            if (role == 3) {  // x = -2: vbar for D-_x
#pragma unroll
                for (int k = 0; k < 3; ++k) vbx2[k] = fmaf(2.f, xv[k], -xv[3 + k]);
            } else {  // x = E + 1: ubar for D+_x
                ux2 = fmaf(2.f, xv[0], -xv[1]);
            }
        }
        if (role >= 3) {  // G(s)
            hissue(s + 3);
            if (xface && s + 2 <= E) xissue(s + 2);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        // (a3) over-relaxed iterate at planes s and s+1
        const float ub = fmaf(2.f, u0.uk, -u0.um);
        const float ub1 = fmaf(2.f, u1.uk, -u1.um);
        float vb[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) vb[k] = fmaf(2.f, x0.vk[k], -x0.vm[k]);
        suv[par][0][r][cc] = ub;
        suv[par][1][r][cc] = vb[0];
        suv[par][2][r][cc] = vb[1];
        suv[par][3][r][cc] = vb[2];
        __syncthreads();

        // (a1) dual D(s): brick_dual_kernel's expressions
        float pn[3] = {0.f, 0.f, 0.f}, qn[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (needP) {
            const float ux = xl ? (role == 4 ? ux2 : suv[par][0][r][cc + 1]) : 0.f;
            const float uy = yl ? suv[par][0][r + 1][cc] : 0.f;
            const float uz = zl ? ub1 : 0.f;
            float p[3] = {x0.p[0], x0.p[1], x0.p[2]};
            const float g0 = xl ? ux - ub : 0.f, g1 = yl ? uy - ub : 0.f, g2 = zl ? uz - ub : 0.f;
            p[0] = fmaf(sp.sigma, g0 - vb[0], p[0]);
            p[1] = fmaf(sp.sigma, g1 - vb[1], p[1]);
            p[2] = fmaf(sp.sigma, g2 - vb[2], p[2]);
            const float sp_ = proj_scale(p[0] * p[0] + p[1] * p[1] + p[2] * p[2], sp.alpha1);
#pragma unroll
            for (int k = 0; k < 3; ++k) pn[k] = p[k] * sp_;
        }
        if (needQ) {
            // neighbours outside Omega were loaded as 0, which is the SPLIT kernel's masked value
            float dx[3], dy[3], dz[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const float vbx = role == 3 ? vbx2[k] : suv[par][1 + k][r][cc - 1];
                const float vby = suv[par][1 + k][r - 1][cc];
                dx[k] = fmaf(xl ? 1.f : 0.f, vb[k], -vbx);
                dy[k] = fmaf(yl ? 1.f : 0.f, vb[k], -vby);
                dz[k] = fmaf(zl ? 1.f : 0.f, vb[k], -ca.vb[k]);
            }
            float q[6];
#pragma unroll
            for (int m = 0; m < 6; ++m) q[m] = x0.q[m];
            const float e[6] = {dx[0], dy[1], dz[2], 0.5f * (dy[0] + dx[1]), 0.5f * (dz[0] + dx[2]),
                                0.5f * (dz[1] + dy[2])};
#pragma unroll
            for (int m = 0; m < 6; ++m) q[m] = fmaf(sp.sigma, e[m], q[m]);
            const float sq = proj_scale(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] +
                                            2.f * (q[3] * q[3] + q[4] * q[4] + q[5] * q[5]),
                                        sp.alpha0);
#pragma unroll
            for (int m = 0; m < 6; ++m) qn[m] = q[m] * sq;
        }
        if (needP) {
            sr[par][0][r][cc] = pn[0];
            sr[par][1][r][cc] = pn[1];
        }
        if (needQ) {
            sr[par][2][r][cc] = qn[0];
            sr[par][3][r][cc] = qn[3];
            sr[par][4][r][cc] = qn[4];
            sr[par][5][r][cc] = qn[1];
            sr[par][6][r][cc] = qn[5];
        }
        if (xface && s >= 0 && s < E) {  // the frozen x-neighbour's face cell of plane s (in S)
            const int o = at(s);
#pragma unroll
            for (int k = 0; k < 3; ++k) a.pn[k][o] = pn[k];
#pragma unroll
            for (int m = 0; m < 6; ++m) a.qn[m][o] = qn[m];
        }
        if (role == 0) {
            if (s >= 0 && s < E) {  // p, q of the owned plane s
                const int o = base_0 + (s << (2 * LE));
#pragma unroll
                for (int k = 0; k < 3; ++k) a.pn[k][o] = pn[k];
#pragma unroll
                for (int m = 0; m < 6; ++m) a.qn[m][o] = qn[m];
            }
            if (s - 1 >= 0) {  // (a2) primal of plane s-1: brick_primal_kernel's expressions
                const bool zl1 = bit(own_ex, s), zf1 = bit(own_ex, s - 2);
                const bool xl1 = (xl_m >> 1) & 1u, yl1 = (yl_m >> 1) & 1u;
                const float pxm = xf0 ? sr[pr][0][r][cc - 1] : 0.f;
                const float pym = yf0 ? sr[pr][1][r - 1][cc] : 0.f;
                const float pzm = zf1 ? ca.pz : 0.f;
                const float qx0 = xl1 ? sr[pr][2][r][cc + 1] : 0.f, qx1 = xl1 ? sr[pr][3][r][cc + 1] : 0.f,
                            qx2 = xl1 ? sr[pr][4][r][cc + 1] : 0.f;
                const float qy0 = yl1 ? sr[pr][3][r + 1][cc] : 0.f, qy1 = yl1 ? sr[pr][5][r + 1][cc] : 0.f,
                            qy2 = yl1 ? sr[pr][6][r + 1][cc] : 0.f;
                const float qz0 = zl1 ? qn[4] : 0.f, qz1 = zl1 ? qn[5] : 0.f, qz2 = zl1 ? qn[2] : 0.f;
                const float* p = ca.pn;
                const float* q = ca.qn;
                const float divp = fmaf(xl1 ? 1.f : 0.f, p[0], -pxm) + fmaf(yl1 ? 1.f : 0.f, p[1], -pym) +
                                   fmaf(zl1 ? 1.f : 0.f, p[2], -pzm);
                const float un = hist_prox<SLOTS, CT>(fmaf(sp.tau, divp, ca.uk), sp.tl, ca.h, A.C);
                const float w0 = (xl1 ? qx0 - q[0] : 0.f) + (yl1 ? qy0 - q[3] : 0.f) + (zl1 ? qz0 - q[4] : 0.f);
                const float w1 = (xl1 ? qx1 - q[3] : 0.f) + (yl1 ? qy1 - q[1] : 0.f) + (zl1 ? qz1 - q[5] : 0.f);
                const float w2 = (xl1 ? qx2 - q[4] : 0.f) + (yl1 ? qy2 - q[5] : 0.f) + (zl1 ? qz2 - q[2] : 0.f);
                const int o = base_0 + ((s - 1) << (2 * LE));
                a.un[o] = un;
                a.vn[0][o] = fmaf(sp.tau, p[0] + w0, ca.vk[0]);
                a.vn[1][o] = fmaf(sp.tau, p[1] + w1, ca.vk[1]);
                a.vn[2][o] = fmaf(sp.tau, p[2] + w2, ca.vk[2]);
            }
        }
        // ---- carry to step s+1
        ca.pz = ca.pn[2];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            ca.pn[k] = pn[k];
            ca.vb[k] = vb[k];
            ca.vk[k] = x0.vk[k];
        }
#pragma unroll
        for (int m = 0; m < 6; ++m) ca.qn[m] = qn[m];
        ca.uk = u0.uk;
        ca.h = h0;
        h0 = h1;
        u0 = u1;
        u1 = u2;
        x0 = x1;
    }
}

}  // namespace tgvk

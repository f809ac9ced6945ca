// tgv_tvl1_tma.cuh -- NEXT-4 TV-L1 single sweep with TMA-staged planes (sm_100a).
//
// Eq. 1 (R21): the TGV scheme with v = q = 0,
//   p_{k+1} = P_a1(p_k + s grad ubar_k),  u_{k+1} = clamp(prox(u_k + t div p_{k+1}), -1, 1),
// the arithmetic of tvl1_dual_kernel / tvl1_primal_kernel (tgv_kernels.cuh)
// expression for expression, in one launch per iteration: reads u_k, u_{k-1}, p_k and
// the counts, writes p_{k+1}, u_{k+1} (44 B per voxel-iteration with u8 counts).
//
// Same machinery as fused_tma_kernel (tgv_fused_tma.cuh), with its tile geometry:
//   warps 0 .. TY+1 : one row each (row 0 = y0-1 supplies p_y(y-1) to row 1, row TY+1 =
//                     y0+TY supplies ubar(y+1) to row TY), lane = x - x0
//   warp  TY+2      : lanes 0..15 column x0-1 (p_x(x0-1) for div p), lanes 16..31 column
//                     x0+32 (ubar(x0+32) for the dual of column x0+31)
// u rings (u_k, u_{k-1}; read at planes s and s+1) and x rings (p_k and the counts) are
// filled by TMA, completion on mbarriers, three planes in flight on the x ring; outputs
// are staged in parity-double-buffered shared memory and written with TMA stores issued
// after the next step's barrier.  Step s computes the dual D(s) and the primal of plane
// s-1 (whose p_x(x-1), p_y(y-1) are the exchange planes of step s-1): one
// __syncthreads per step.
#pragma once
#include "tgv_fused_tma.cuh"

namespace tgvk {

template <int HB>
struct TvRings {
    static constexpr int NU = 4, NX = 4;
};

template <int TY, int HB>
struct alignas(128) TvSmem {
    static constexpr int R = TY + 2;
    using Rg = TvRings<HB>;
    float u[Rg::NU][2][R][TMA_BW];   // ring: u_k, u_{k-1}
    float p[Rg::NX][3][R][TMA_BW];   // ring: p_k(3)
    float out[2][4][TY][32];          // staged outputs of step s (parity): u (plane s-1), p(3) (plane s)
    uint8_t h[Rg::NX][TY][32 * HB];  // ring: histograms of the owned rows
    float suv[2][R][TMA_CW];          // ubar of plane s (parity)
    float sr[2][2][R][TMA_CW];        // p_x, p_y of D(s) (parity)
    uint64_t bar_u[Rg::NU], bar_x[Rg::NX];
};

template <int TY, int SLOTS, typename CT>
__global__ void __launch_bounds__(32 * (TY + 3), 2)
    tvl1_tma_kernel(const __grid_constant__ CUtensorMap m_ld1, const __grid_constant__ CUtensorMap m_ld3,
                    const __grid_constant__ CUtensorMap m_st1, const __grid_constant__ CUtensorMap m_st3,
                    const __grid_constant__ CUtensorMap m_h, const TmaArgs A)
{
    constexpr int HB = SLOTS * (int)sizeof(CT);
    constexpr int R = TY + 2;
    using Smem = TvSmem<TY, HB>;
    using Hist = HistRaw<SLOTS, CT>;
    using Rg = TvRings<HB>;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const Geo& g = A.g;
    const StepParams& sp = A.sp;

    const int lane = threadIdx.x, w = threadIdx.y;
    const bool tid0 = lane == 0 && w == 0;
    const bool halo = w == TY + 2;

    struct Cur {
        int st;
        uint32_t ph;
    };
    auto adv = [](Cur& c, int n) {
        if (++c.st == n) {
            c.st = 0;
            c.ph ^= 1u;
        }
    };
    Cur iu{0, 0u}, ix{0, 0u};
    Cur cu{0, 0u}, cx{0, 0u};

    if (tid0) {
        if (smem_addr(smem_raw) & 127) __trap();
        prefetch_map(&m_ld1);
        prefetch_map(&m_ld3);
        prefetch_map(&m_h);
        for (int k = 0; k < Rg::NU; ++k) mbar_init(&S.bar_u[k], 1);
        for (int k = 0; k < Rg::NX; ++k) mbar_init(&S.bar_x[k], 1);
        fence_mbar_init();
    }
    __syncthreads();

    const int tiles_x = (g.nx + 31) / 32;
    for (int sgi = A.sched_off[blockIdx.x]; sgi < A.sched_off[blockIdx.x + 1]; ++sgi) {
        const int4 sg = A.sched[sgi];
        const int t = sg.x, zs = sg.y, ze = sg.z;
        const int x0 = (t % tiles_x) * 32, y0 = (t / tiles_x) * TY;

        int r, bc, cc, x;
        if (!halo) {
            r = w, bc = lane + 4, cc = lane + 1, x = x0 + lane;
        } else if (lane < 16) {  // rows beyond R (TY < 14) duplicate row R-1 exactly: identical writes
            r = min(lane, R - 1), bc = 3, cc = 0, x = x0 - 1;
        } else {
            r = min(lane - 16, R - 1), bc = 36, cc = TMA_CW - 1, x = x0 + 32;
        }
        const int y = y0 - 1 + r;
        const bool own = !halo && r >= 1 && r <= TY;
        // p is needed on rows 0..TY and, in the halo warp, at column x0-1 of the owned rows
        const bool needP = halo ? (lane < 16 && r >= 1 && r <= TY) : r <= TY;
        const bool xl = x < g.nx - 1, xf = x > 0, yl = y < g.ny - 1, yf = y > 0;

        auto zclamp = [&](int s) { return min(max(s + 1, 0), g.nzl + 1); };
        auto issue_u = [&](int s) {
            const int st = iu.st;
            adv(iu, Rg::NU);
            mbar_expect_tx(&S.bar_u[st], 2 * R * TMA_BW * 4);
            tma_load4(&S.u[st][0][0][0], &m_ld1, &S.bar_u[st], x0 - 4, y0 - 1, zclamp(s), A.s_uk);
            tma_load4(&S.u[st][1][0][0], &m_ld1, &S.bar_u[st], x0 - 4, y0 - 1, zclamp(s), A.s_um);
        };
        auto issue_x = [&](int s) {  // p_k and the counts of plane s
            const int st = ix.st;
            adv(ix, Rg::NX);
            mbar_expect_tx(&S.bar_x[st], 3 * R * TMA_BW * 4 + TY * 32 * HB);
            tma_load4(&S.p[st][0][0][0], &m_ld3, &S.bar_x[st], x0 - 4, y0 - 1, zclamp(s), A.s_pk);
            tma_load3(&S.h[st][0][0], &m_h, &S.bar_x[st], 8 * x0, y0, min(max(s, 0), g.nzl - 1));
        };

        const int jr = sgi - A.sched_off[blockIdx.x];  // this CTA's segment index (= round while < rounds)
        if (tid0) {
            for (int tz = zs - 1; tz < zs - 1 + Rg::NU - 1; ++tz) issue_u(tz);
            for (int tz = zs - 1; tz < zs - 1 + Rg::NX - 1; ++tz) issue_x(tz);
            round_wait(A.round_ctr, jr, A.rounds);  // lock-step rounds, as fused_tma_kernel
        }
        mbar_wait(&S.bar_u[cu.st], cu.ph);  // u at plane zs-1
        int su = cu.st;
        adv(cu, Rg::NU);

        // TMA stores of the outputs step t staged in out[b]: p(t) at plane t, u(t-1) at plane t-1
        auto store = [&](int b, int t) {
            if (t >= zs && t < ze) tma_store4(&m_st3, &S.out[b][1][0][0], x0, y0, t + 1, A.s_pn);
            if (t - 1 >= zs) tma_store4(&m_st1, &S.out[b][0][0][0], x0, y0, t, A.s_un);
            tma_commit();
        };

        struct Carry {
            float uk;     // u_k at s-1
            Hist h;       // histogram of s-1
            float pn[3];  // p_{k+1}(s-1)
            float pz;     // p_z{k+1}(s-2)
        };
        Carry ca{}, cb{};

        auto step = [&](auto PAR, int s, const Carry& in, Carry& o) {
            constexpr int par = decltype(PAR)::value, pr = par ^ 1;
            const int zg = g.z0 + s;
            mbar_wait(&S.bar_u[cu.st], cu.ph);
            mbar_wait(&S.bar_x[cx.st], cx.ph);

            constexpr int F = R * TMA_BW;
            const float* U0 = &S.u[su][0][r][bc];
            const float* U1 = &S.u[cu.st][0][r][bc];
            const float* P0 = &S.p[cx.st][0][r][bc];
            const float uk = U0[0];
            const float ub = fmaf(2.f, uk, -U0[F]);         // ubar(s)
            const float ub1 = fmaf(2.f, U1[0], -U1[F]);     // ubar(s+1)
            const float pk0 = P0[0], pk1 = P0[F], pk2 = P0[2 * F];
            Hist hc{};
            if (own) {
                const uint8_t* hp = &S.h[cx.st][r - 1][lane * HB];
                if constexpr (HB == 8) {
                    const uint2 v2 = *reinterpret_cast<const uint2*>(hp);
                    hc.w[0] = v2.x;
                    hc.w[1] = v2.y;
                } else {
#pragma unroll
                    for (int q4 = 0; q4 < HB / 16; ++q4) {
                        const uint4 v4 = reinterpret_cast<const uint4*>(hp)[q4];
                        hc.w[4 * q4] = v4.x;
                        hc.w[4 * q4 + 1] = v4.y;
                        hc.w[4 * q4 + 2] = v4.z;
                        hc.w[4 * q4 + 3] = v4.w;
                    }
                }
            }
            S.suv[par][r][cc] = ub;
            if (tid0) tma_wait_read0();  // the stores of step s-2 have read out[par]
            __syncthreads();             // S1: also completes the out[pr] writes of step s-1
            if (tid0) {
                if (s + Rg::NU - 1 <= ze + 1) issue_u(s + Rg::NU - 1);
                if (s + Rg::NX - 1 <= ze) issue_x(s + Rg::NX - 1);
                if (s > zs - 1) store(pr, s - 1);  // the outputs of step s-1
            }
            su = cu.st;
            adv(cu, Rg::NU);
            adv(cx, Rg::NX);

            // dual D(s) (tvl1_dual_kernel)
            float pn[3] = {0.f, 0.f, 0.f};
            if (needP) {
                const bool zl = zg < g.nz - 1;
                const float ux = S.suv[par][r][cc + 1];
                const float uy = S.suv[par][r + 1][cc];
                const float g0 = xl ? ux - ub : 0.f, g1 = yl ? uy - ub : 0.f, g2 = zl ? ub1 - ub : 0.f;
                pn[0] = fmaf(sp.sigma, g0, pk0);
                pn[1] = fmaf(sp.sigma, g1, pk1);
                pn[2] = fmaf(sp.sigma, g2, pk2);
                const float f = proj_scale(pn[0] * pn[0] + pn[1] * pn[1] + pn[2] * pn[2], sp.alpha1);
                pn[0] *= f;
                pn[1] *= f;
                pn[2] *= f;
                S.sr[par][0][r][cc] = pn[0];
                S.sr[par][1][r][cc] = pn[1];
            }
            if (own) {
#pragma unroll
                for (int k = 0; k < 3; ++k) S.out[par][1 + k][r - 1][lane] = pn[k];
                if (s - 1 >= zs) {  // primal of plane s-1 (tvl1_primal_kernel)
                    const bool zl1 = zg - 1 < g.nz - 1, zf1 = zg - 1 > 0;
                    const float pxm = xf ? S.sr[pr][0][r][cc - 1] : 0.f;
                    const float pym = yf ? S.sr[pr][1][r - 1][cc] : 0.f;
                    const float pzm = zf1 ? in.pz : 0.f;
                    const float divp = ((xl ? in.pn[0] : 0.f) - pxm) + ((yl ? in.pn[1] : 0.f) - pym) +
                                       ((zl1 ? in.pn[2] : 0.f) - pzm);
                    S.out[par][0][r - 1][lane] = hist_prox<SLOTS, CT>(fmaf(sp.tau, divp, in.uk), sp.tl, in.h, A.C);
                }
            }
            fence_proxy_async();  // out[par] is stored by the async proxy after the next S1
            o.pz = in.pn[2];
#pragma unroll
            for (int k = 0; k < 3; ++k) o.pn[k] = pn[k];
            o.uk = uk;
            o.h = hc;
        };

        for (int s = zs - 1; s <= ze; s += 2) {
            step(std::integral_constant<int, 0>{}, s, ca, cb);
            if (s + 1 > ze) break;
            step(std::integral_constant<int, 1>{}, s + 1, cb, ca);
        }
        __syncthreads();  // the last step's outputs are complete (its parity counts from step zs-1)
        if (tid0) store((ze - (zs - 1)) & 1, ze);
        if (tid0) round_done(A.round_ctr, jr, A.rounds);
    }
    if (tid0) tma_wait0();
}

}  // namespace tgvk

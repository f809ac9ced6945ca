// tgv_energy_tma.cuh -- (a4) dense energy / restricted gap as a TMA-staged z-sweep (sm_100a).
//
// E(u, v) and the box-restricted dual D_V (R14) need,
// per voxel, D+u, the symmetrised D- of v, div p (D-) and div2 q (D+ of q): a one-voxel
// stencil over the 13 state fields, every neighbour an INPUT (no computed value is
// exchanged, unlike the iteration sweep).  So each CTA stages whole planes of its tile
// -- one 40 x (TY+2) box per field (x0-4 .. x0+35, y0-1 .. y0+TY: the +-1 halo) and the
// counts of the owned rows -- by TMA into an mbarrier ring, and every thread reads its
// own voxel and its x / y / z+1 neighbours straight from shared memory; the z-1
// neighbours (v, p_z) ride in registers.  HBM sees each field once (60 B per voxel with u8
// counts); the halo boxes overlap neighbouring tiles, whose reads L2 serves because the
// CTAs march the same lock-step (tile, z-chunk) schedule as the iteration sweep.
//
// Per-voxel terms are the fp32 expressions of energy_partial_kernel (one shared device
// function), summed in fp64 per thread, per warp (shuffles) and per CTA in a fixed
// order: deterministic.  The register-streaming energy_partial_kernel read 1.24x the
// algorithmic bytes on C4 at 0.55-0.64 of the copy roofline (profiles/r2e_*, r2f_*).
#pragma once
#include "tgv_fused_tma.cuh"

namespace tgvk {

// NS: ring depth (planes s and s+1 are read at step s, the rest are in flight); NS = 3 runs
// two CTAs per SM (u8 counts, 8 bins), deeper rings one
template <int TY, int HB, int NS_>
struct alignas(128) EnSmem {
    static constexpr int R = TY + 2, NS = NS_;
    float f[NS][13][R][TMA_BW];   // u, v(3), p(3), q(6) of one plane (state slot order)
    uint8_t h[NS][TY][32 * HB];  // counts of the owned rows
    uint64_t bar[NS];
    double red[EN_TERMS][TY];
};

struct EnTmaArgs {
    Geo g;
    int s_u, s_v, s_p, s_q;  // state slots of u_k, v_k (3), p_k (3), q_k (6)
    const int4* sched;       // persistent (tile, z_begin, z_end) segments, as the fused sweep's
    const int* sched_off;
    float alpha1, alpha0, lambda, V;
    unsigned long long* round_ctr;  // lock-step rounds (as fused_tma_kernel), or null
    int rounds;
};

template <int TY, int SLOTS, typename CT, int NS>
__global__ void __launch_bounds__(32 * TY, NS <= 3 ? 2 : 1)
    energy_tma_kernel(const __grid_constant__ CUtensorMap m_ld1, const __grid_constant__ CUtensorMap m_ld3,
                      const __grid_constant__ CUtensorMap m_ld6, const __grid_constant__ CUtensorMap m_h,
                      const EnTmaArgs A, const EnergyConsts K, double* __restrict__ partials)
{
    constexpr int HB = SLOTS * (int)sizeof(CT);
    constexpr int R = TY + 2;
    constexpr int F = R * TMA_BW;  // field stride in a ring slot
    using Smem = EnSmem<TY, HB, NS>;
    using Hist = HistRaw<SLOTS, CT>;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const Geo& g = A.g;
    const int lane = threadIdx.x, w = threadIdx.y;
    const bool tid0 = lane == 0 && w == 0;
    const int r = w + 1, bc = lane + 4;  // this thread's cell in the boxes (row 0 = y0-1, column 0 = x0-4)

    struct Cur {
        int st;
        uint32_t ph;
    };
    auto adv = [](Cur& c) {
        if (++c.st == NS) {
            c.st = 0;
            c.ph ^= 1u;
        }
    };
    Cur iss{0, 0u}, cw{0, 0u};  // issue cursor (tid0) and wait cursor (all), in plane order
    if (tid0) {
        if (smem_addr(smem_raw) & 127) __trap();
        prefetch_map(&m_ld1);
        prefetch_map(&m_ld3);
        prefetch_map(&m_ld6);
        prefetch_map(&m_h);
        for (int k = 0; k < NS; ++k) mbar_init(&S.bar[k], 1);
        fence_mbar_init();
    }
    __syncthreads();

    double t1 = 0, t0 = 0, td = 0, dv = 0;
    float vm = 0.f;
    const float al1 = A.alpha1, al0 = A.alpha0, lam = A.lambda, VV = A.V;
    const int tiles_x = (g.nx + 31) / 32;
    for (int sgi = A.sched_off[blockIdx.x]; sgi < A.sched_off[blockIdx.x + 1]; ++sgi) {
        const int4 sg = A.sched[sgi];
        const int zs = sg.y, ze = sg.z;
        const int x0 = (sg.x % tiles_x) * 32, y0 = (sg.x / tiles_x) * TY;
        const int x = x0 + lane, y = y0 + w;
        const bool act = x < g.nx && y < g.ny;
        const bool xl = x < g.nx - 1, yl = y < g.ny - 1, xf = x > 0, yf = y > 0;
        const bool tile_int = x0 >= 1 && x0 + 32 <= g.nx - 1 && y0 >= 1 && y0 + TY <= g.ny - 1;

        // planes zs-1 .. ze (z-1 neighbour of zs, z+1 neighbour of ze-1), in ring order;
        // only the planes zs .. ze-1 carry counts
        auto issue = [&](int pl) {
            const int st = iss.st;
            adv(iss);
            const bool hh = pl >= zs && pl < ze;
            mbar_expect_tx(&S.bar[st], 13 * F * 4 + (hh ? TY * 32 * HB : 0));
            const int zp = pl + 1;  // slot-plane coordinate (plane -1 is the bottom halo)
            tma_load4(&S.f[st][0][0][0], &m_ld1, &S.bar[st], x0 - 4, y0 - 1, zp, A.s_u);
            tma_load4(&S.f[st][1][0][0], &m_ld3, &S.bar[st], x0 - 4, y0 - 1, zp, A.s_v);
            tma_load4(&S.f[st][4][0][0], &m_ld3, &S.bar[st], x0 - 4, y0 - 1, zp, A.s_p);
            tma_load4(&S.f[st][7][0][0], &m_ld6, &S.bar[st], x0 - 4, y0 - 1, zp, A.s_q);
            if (hh) tma_load3(&S.h[st][0][0], &m_h, &S.bar[st], 8 * x0, y0, pl);
        };
        // prologue: planes zs-1 .. zs+NS-2 fill the ring; after step s's barrier the slots of
        // planes <= s are free and the ring runs up to plane s+NS
        int nxt = zs - 1;
        const int jr = sgi - A.sched_off[blockIdx.x];  // this CTA's segment index (= round while < rounds)
        if (tid0) {
            for (; nxt <= ze && nxt < zs - 1 + NS; ++nxt) issue(nxt);
            round_wait(A.round_ctr, jr, A.rounds);  // lock-step rounds, as fused_tma_kernel
        }

        // carry-in: v and p_z of plane zs-1 (its slot is refilled after step zs's barrier)
        mbar_wait(&S.bar[cw.st], cw.ph);
        float vz0, vz1, vz2, pzm;
        {
            const float* a = &S.f[cw.st][0][r][bc];
            vz0 = a[F], vz1 = a[2 * F], vz2 = a[3 * F], pzm = a[6 * F];
        }
        adv(cw);
        mbar_wait(&S.bar[cw.st], cw.ph);  // plane zs
        int sc = cw.st;
        adv(cw);
        for (int s = zs; s < ze; ++s) {
            mbar_wait(&S.bar[cw.st], cw.ph);  // plane s+1 (plane s arrived a step earlier)
            const int sn = cw.st;
            const float* a = &S.f[sc][0][r][bc];
            const float* b = &S.f[sn][0][r][bc];
            const int zg = g.z0 + s;
            const bool zl = zg < g.nz - 1, zf = zg > 0;
            const float v0 = a[F], v1 = a[2 * F], v2 = a[3 * F], p2 = a[6 * F];
            if (act) {
                Hist h;
                const uint8_t* hp = &S.h[sc][w][lane * HB];
                if constexpr (HB == 8) {
                    const uint2 q2 = *reinterpret_cast<const uint2*>(hp);
                    h.w[0] = q2.x;
                    h.w[1] = q2.y;
                } else {
#pragma unroll
                    for (int k = 0; k < HB / 16; ++k) {
                        const uint4 q4 = reinterpret_cast<const uint4*>(hp)[k];
                        h.w[4 * k] = q4.x;
                        h.w[4 * k + 1] = q4.y;
                        h.w[4 * k + 2] = q4.z;
                        h.w[4 * k + 3] = q4.w;
                    }
                }
                EnVoxel e;
                e.uc = a[0], e.ux = a[1], e.uy = a[TMA_BW], e.un = b[0];
                e.v0 = v0, e.v1 = v1, e.v2 = v2;
                e.v0x = a[F - 1], e.v1x = a[2 * F - 1], e.v2x = a[3 * F - 1];
                e.v0y = a[F - TMA_BW], e.v1y = a[2 * F - TMA_BW], e.v2y = a[3 * F - TMA_BW];
                e.vm0 = vz0, e.vm1 = vz1, e.vm2 = vz2;
                e.p0 = a[4 * F], e.p1 = a[5 * F], e.p2 = p2;
                e.p0x = a[4 * F - 1], e.p1y = a[5 * F - TMA_BW], e.pzm = pzm;
                e.qxx = a[7 * F], e.qyy = a[8 * F], e.qzz = a[9 * F], e.qxy = a[10 * F], e.qxz = a[11 * F],
                e.qyz = a[12 * F];
                e.qxxx = a[7 * F + 1], e.qxyx = a[10 * F + 1], e.qxzx = a[11 * F + 1];
                e.qxyy = a[10 * F + TMA_BW], e.qyyy = a[8 * F + TMA_BW], e.qyzy = a[12 * F + TMA_BW];
                e.qzzn = b[9 * F], e.qxzn = b[11 * F], e.qyzn = b[12 * F];
                if (tile_int && zl && zf)
                    energy_voxel_terms<SLOTS, CT, true>(e, h, K, al1, al0, lam, VV, xl, yl, zl, xf, yf, zf, t1, t0,
                                                        td, dv);
                else
                    energy_voxel_terms<SLOTS, CT, false>(e, h, K, al1, al0, lam, VV, xl, yl, zl, xf, yf, zf, t1, t0,
                                                         td, dv);
                vm = fmaxf(vm, fmaxf(fabsf(v0), fmaxf(fabsf(v1), fabsf(v2))));
            }
            vz0 = v0, vz1 = v1, vz2 = v2, pzm = p2;
            __syncthreads();  // every thread is done with the slots of planes <= s
            if (tid0)
                for (; nxt <= ze && nxt <= s + NS; ++nxt) issue(nxt);
            sc = sn;
            adv(cw);
        }
        __syncthreads();  // the next segment's prologue refills every slot
        if (tid0) round_done(A.round_ctr, jr, A.rounds);
    }

    double vmd = (double)vm;
    t1 = warp_sum(t1);
    t0 = warp_sum(t0);
    td = warp_sum(td);
    dv = warp_sum(dv);
    vmd = warp_max(vmd);
    if (lane == 0) {
        S.red[0][w] = t1;
        S.red[1][w] = t0;
        S.red[2][w] = td;
        S.red[3][w] = dv;
        S.red[4][w] = vmd;
    }
    __syncthreads();
    if (w == 0 && lane < EN_TERMS) {
        const int k = lane;
        double s = S.red[k][0];
        for (int j = 1; j < TY; ++j) s = (k == 4) ? fmax(s, S.red[k][j]) : s + S.red[k][j];
        partials[(int64_t)blockIdx.x * EN_TERMS + k] = s;
    }
}

}  // namespace tgvk

// tgv_fused_tma.cuh -- single-sweep TGV iteration with TMA-staged planes (sm_100a).
//
// Same scheme and same fp32 expressions as split_dual_kernel + split_primal_kernel
// (tgv_kernels.cuh), one launch per iteration, 128 / 136 B per voxel-iteration.
//
// CTA = (TY + 3) warps over a 32 x TY owned tile of (x, y), marching up a z-chunk:
//   warps 0 .. TY+1 : one row each (row 0 = y0-1 and row TY+1 = y0+TY are the
//                     y-halo), lane = x - x0 (32 owned columns, 128-B aligned)
//   warp  TY+2      : the x-halo: lanes 0..15 column x0-1 (p only),
//                     lanes 16..31 column x0+32 (q only), one row per lane
// Inputs arrive by TMA (cp.async.bulk.tensor) into shared-memory rings, one
// box of 40 x (TY+2) per field and plane (x0-4 .. x0+35: the +-1 halo; the
// inner start coordinate must be 16-B aligned), completion signalled on mbarriers; the planes of step s+2 are in
// flight while step s computes.  Out-of-range boxes (grid and slab edges) are
// zero-filled by the TMA unit, so there are no per-element guards.  x and y
// neighbours are exchanged through two small parity-double-buffered planes
// (over-relaxed inputs, and the dual results); z neighbours stay in registers.
// Outputs are staged in shared memory and written with TMA bulk tensor stores
// (which clip at nx, ny).  Two __syncthreads per step.
#pragma once
#include <cuda.h>

#include <type_traits>

#include "tgv_kernels.cuh"

namespace tgvk {

// ---- PTX helpers ---------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// wait for the phase with the given parity; a watchdog traps (kernel error, no hang)
// if the transaction never completes
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    uint32_t n = 0;
    while (!mbar_try(bar, parity))
        if (++n > (1u << 26)) __trap();
}
__device__ __forceinline__ void tma_load4(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                          int c3)
{
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
        "[%2];" ::"r"(smem_addr(dst)),
        "l"(map), "r"(smem_addr(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
        "[%2];" ::"r"(smem_addr(dst)),
        "l"(map), "r"(smem_addr(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
// L2 eviction-priority policies (createpolicy) and the hinted TMA forms: data no CTA
// will read again (the outputs, the counts) can leave L2 first, keeping it for the halo
// rows / columns that neighbouring tiles re-read
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load3_hint(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                               uint64_t pol)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
        "%4, %5}], [%2], %6;" ::"r"(smem_addr(dst)),
        "l"(map), "r"(smem_addr(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_store4_hint(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3,
                                                uint64_t pol)
{
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4, %5}], [%1], %6;" ::"l"(map),
                 "r"(smem_addr(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void tma_store4(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3)
{
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(map),
                 "r"(smem_addr(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}
__device__ __forceinline__ void tma_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void tma_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void prefetch_map(const CUtensorMap* m)
{
    asm volatile("prefetch.tensormap [%0];" ::"l"(m) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }

// Lock-step round sync of the persistent sweeps: before its round jr the
// issuing thread of a CTA waits until all gridDim.x CTAs finished round jr-1 (ctr counts the
// finished rounds, the launch's last increment resets it).  The wait is bounded and never a
// correctness dependency: one that runs out (the grid's CTAs not all resident, e.g. another
// kernel holding SMs) sets the launch's give-up word ctr[4], and no CTA waits again until the
// launch ends.
__device__ __forceinline__ void round_wait(unsigned long long* ctr, int jr, int rounds)
{
    if (!ctr || jr < 1 || jr >= rounds || *(volatile unsigned long long*)(ctr + 4)) return;
    const unsigned long long want = (unsigned long long)jr * gridDim.x;
    for (uint32_t n = 0; ld_acquire_sys(ctr) < want; ++n) {
        if (n > (1u << 18)) {  // ~20-40 ms: far beyond any honest skew between CTAs of one round
            atomicExch(ctr + 4, 1ull);
            return;
        }
        __nanosleep(64);
    }
}
__device__ __forceinline__ void round_done(unsigned long long* ctr, int jr, int rounds)
{
    if (ctr && jr < rounds && atomicAdd(ctr, 1ull) == (unsigned long long)rounds * gridDim.x - 1) {
        atomicExch(ctr, 0ull);  // the launch's last increment: no CTA waits any more, the next
        atomicExch(ctr + 4, 0ull);  // launch (stream-ordered) starts from zero
    }
}

// ---- shared memory ---------------------------------------------------------------
constexpr int TMA_BW = 40;  // input box width: x0-4 .. x0+35 (the inner start must be 16-B aligned)
constexpr int TMA_CW = 34;  // exchange plane width: x0-1 .. x0+32

// Ring depths: u is read at planes s and s+1, v / p / q / histogram at plane s only;
// each ring prefetches two planes beyond what step s reads.
// v, p, q and the histogram of a plane travel together on one ring ("x").
template <int HB>
struct TmaRings {
    static constexpr int NU = 4, NX = HB <= 16 ? 3 : 2;
};

template <int TY, int HB>
struct alignas(128) TmaSmem {
    static constexpr int R = TY + 2;
    using Rg = TmaRings<HB>;
    float u[Rg::NU][2][R][TMA_BW];   // ring: u_k, u_{k-1}
    float v[Rg::NX][6][R][TMA_BW];   // ring: v_k(3), v_{k-1}(3)
    float pq[Rg::NX][9][R][TMA_BW];  // ring: p_k(3), q_k(6)
    float out[13][TY][32];            // staged outputs: u, v(3), p(3), q(6) of iteration k+1
    uint8_t h[Rg::NX][TY][32 * HB];  // ring: histograms of the owned rows
    float suv[2][4][R][TMA_CW];       // ubar, vbar(3) of plane s (parity)
    float sr[2][7][R][TMA_CW];        // p_x, p_y, q_xx, q_xy, q_xz, q_yy, q_yz of D(s) (parity)
    uint64_t bar_u[Rg::NU], bar_x[Rg::NX];
};

struct TmaArgs {
    Geo g;
    StepParams sp;
    Centers C;
    int z_lo, z_hi, zc;
    const int4* sched;      // segments (tile, z_begin, z_end, -) of all CTAs, see tma_schedule()
    const int* sched_off;   // CTA b owns sched[sched_off[b] .. sched_off[b+1])
    int s_uk, s_um, s_vk, s_vm, s_pk, s_qk;  // input slots (v/p/q: first of 3/3/6 consecutive)
    int s_un, s_vn, s_pn, s_qn;              // output slots
    int keep_halo_dual;  // NEXT-3 leaves: also store p at plane -1 and q at plane nzl (no exchange refreshes them)
    int hints;           // L2 policy: bit 0 the output stores evict first, bit 1 the count loads evict first
    // Lock-step rounds (optional): the first `rounds` segments of every CTA are whole
    // (tile, chunk) items dealt round-robin; before its round j a CTA waits (bounded: never
    // a correctness dependency) until all G CTAs finished round j-1, so that persistent CTAs
    // cannot drift rounds apart and neighbouring tiles keep sharing their halos in L2.
    unsigned long long* round_ctr;  // null: off; else + 1 per CTA per round, reset by the last increment
    int rounds;
    // Peer halo mode: the kernel itself writes the next iterate of its
    // boundary planes into the neighbours' halo planes (NVLink / same-device stores,
    // tile by tile as they are computed) -- down: u, v, q of plane 0 into the lower
    // neighbour's top halo; up: u, v, p of plane nzl-1 into the upper neighbour's bottom
    // halo -- and hands over with a flag per neighbour: the last CTA to finish publishes
    // `seq`; the next launch waits until both neighbours published `wait_seq`.
    float* pdn;            // lower neighbour's state (slot 0), or null
    int64_t pdn_fs;        // its slot stride (floats)
    int pdn_top;           // its top halo plane, in slot-plane coordinates (its nzl + 1)
    float* pup;            // upper neighbour's state, or null (its bottom halo is plane 0)
    int64_t pup_fs;
    unsigned long long* done;            // this rank's CTA completion counter (null: no peer mode)
    unsigned long long* flag_dn_remote;  // the lower neighbour's "from up" flag
    unsigned long long* flag_up_remote;  // the upper neighbour's "from down" flag
    const unsigned long long* flag_in_dn;  // written by the lower neighbour
    const unsigned long long* flag_in_up;  // written by the upper neighbour
    unsigned long long seq, wait_seq;
};

// PEER: the peer halo mode instantiation (the single-GPU kernel carries none of its code)
template <int TY, int SLOTS, typename CT, bool PEER = false>
__global__ void __launch_bounds__(32 * (TY + 3), 1)
    fused_tma_kernel(const __grid_constant__ CUtensorMap m_ld1, const __grid_constant__ CUtensorMap m_ld3,
                     const __grid_constant__ CUtensorMap m_ld6, const __grid_constant__ CUtensorMap m_st1,
                     const __grid_constant__ CUtensorMap m_st3, const __grid_constant__ CUtensorMap m_st6,
                     const __grid_constant__ CUtensorMap m_h, const TmaArgs A)
{
    constexpr int HB = SLOTS * (int)sizeof(CT);
    constexpr int R = TY + 2;
    using Smem = TmaSmem<TY, HB>;
    using Hist = HistRaw<SLOTS, CT>;
    using Rg = TmaRings<HB>;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);  // dynamic smem starts 128-B aligned (checked below)
    const Geo& g = A.g;
    const StepParams& sp = A.sp;

    const int lane = threadIdx.x, w = threadIdx.y;
    const bool tid0 = lane == 0 && w == 0;
    const bool halo = w == TY + 2;
    const uint64_t pol_ef = A.hints ? policy_evict_first() : 0ull;

    // ring cursors: next slot to fill (issue side) and next slot / phase to wait for.
    // Fills and waits happen in the same order on every ring, across all segments.
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
    Cur iu{0, 0u}, ix{0, 0u};  // issue cursors (tid0 only)
    Cur cu{0, 0u}, cx{0, 0u};  // wait cursors (all threads)

    if (tid0) {
        if (smem_addr(smem_raw) & 127) __trap();
        prefetch_map(&m_ld1);
        prefetch_map(&m_ld3);
        prefetch_map(&m_ld6);
        prefetch_map(&m_h);
        for (int k = 0; k < Rg::NU; ++k) mbar_init(&S.bar_u[k], 1);
        for (int k = 0; k < Rg::NX; ++k) mbar_init(&S.bar_x[k], 1);
        fence_mbar_init();
        if (PEER && A.wait_seq) {  // peer mode: the neighbours' previous launches wrote our halo planes
            uint32_t n = 0;
            while ((A.pdn && ld_acquire_sys(A.flag_in_dn) < A.wait_seq) ||
                   (A.pup && ld_acquire_sys(A.flag_in_up) < A.wait_seq))
                if (++n > (1u << 28)) __trap();  // watchdog: a kernel error, never a hang
            fence_proxy_async_all();  // their generic-proxy stores, before our TMA reads
        }
    }
    __syncthreads();

    // Persistent CTA: it runs the segments (one tile over a z-range) the host schedule
    // assigned to it -- whole z-chunks round-robin over the CTAs, so that all CTAs
    // advance through the chunks together and neighbouring tiles' halos stay in L2,
    // and the chunks that do not fill a last round split evenly over all CTAs.
    const int tiles_x = (g.nx + 31) / 32;
    for (int sgi = A.sched_off[blockIdx.x]; sgi < A.sched_off[blockIdx.x + 1]; ++sgi) {
        const int4 sg = A.sched[sgi];
        const int t = sg.x, zs = sg.y, ze = sg.z;
        const int x0 = (t % tiles_x) * 32, y0 = (t / tiles_x) * TY;

        // ---- this thread's cell
        int r, bc, cc, x;
        if (!halo) {
            r = w, bc = lane + 4, cc = lane + 1, x = x0 + lane;
        } else if (lane < 16) {  // rows beyond R (TY < 14) duplicate row R-1 exactly: identical writes
            r = min(lane, R - 1), bc = 3, cc = 0, x = x0 - 1;
        } else {
            r = min(lane - 16, R - 1), bc = 36, cc = TMA_CW - 1, x = x0 + 32;
        }
        const int y = y0 - 1 + r;
        // p is needed on rows 0..TY (row 0 feeds D-_y of row 1) and at column x0-1;
        // q on rows 1..TY+1 and at column x0+32 (halo lanes: owned rows only)
        const bool own = !halo && r >= 1 && r <= TY;  // owned row (TMA stores clip at nx, ny)
        // warp role: 0 owned row, 1 bottom y-halo row (p only), 2 top y-halo row (q only), 3 x-halo
        const int role = halo ? 3 : (r == 0 ? 1 : (r == TY + 1 ? 2 : 0));
        // every cell of the tile and its halo is at distance >= 1 from the x and y grid ends
        const bool tile_int = x0 >= 2 && x0 + 32 <= g.nx - 2 && y0 >= 2 && y0 + TY <= g.ny - 2;
        const bool xl = x < g.nx - 1, xf = x > 0, yl = y < g.ny - 1, yf = y > 0;
        const float mxl = xl ? 1.f : 0.f, myl = yl ? 1.f : 0.f;

        // Every plane of the segment's sequence is loaded so that each ring slot is
        // filled in order (mbarrier phase = fill count); planes past the stored range are
        // clamped to the nearest stored plane (no box is ever entirely out of bounds) --
        // those values only feed results that are never used (p at plane nzl, the primal
        // of planes -1 / nzl).
        auto zclamp = [&](int s) { return min(max(s + 1, 0), g.nzl + 1); };
        auto issue_u = [&](int s) {
            const int st = iu.st;
            adv(iu, Rg::NU);
            mbar_expect_tx(&S.bar_u[st], 2 * R * TMA_BW * 4);
            tma_load4(&S.u[st][0][0][0], &m_ld1, &S.bar_u[st], x0 - 4, y0 - 1, zclamp(s), A.s_uk);
            tma_load4(&S.u[st][1][0][0], &m_ld1, &S.bar_u[st], x0 - 4, y0 - 1, zclamp(s), A.s_um);
        };
        auto issue_x = [&](int s) {  // v_k, v_{k-1}, p_k, q_k and the counts of plane s
            const int st = ix.st;
            adv(ix, Rg::NX);
            mbar_expect_tx(&S.bar_x[st], 15 * R * TMA_BW * 4 + TY * 32 * HB);
            tma_load4(&S.v[st][0][0][0], &m_ld3, &S.bar_x[st], x0 - 4, y0 - 1, zclamp(s), A.s_vk);
            tma_load4(&S.v[st][3][0][0], &m_ld3, &S.bar_x[st], x0 - 4, y0 - 1, zclamp(s), A.s_vm);
            tma_load4(&S.pq[st][0][0][0], &m_ld3, &S.bar_x[st], x0 - 4, y0 - 1, zclamp(s), A.s_pk);
            tma_load4(&S.pq[st][3][0][0], &m_ld6, &S.bar_x[st], x0 - 4, y0 - 1, zclamp(s), A.s_qk);
            if (A.hints & 2)
                tma_load3_hint(&S.h[st][0][0], &m_h, &S.bar_x[st], 8 * x0, y0, min(max(s, 0), g.nzl - 1), pol_ef);
            else
                tma_load3(&S.h[st][0][0], &m_h, &S.bar_x[st], 8 * x0, y0, min(max(s, 0), g.nzl - 1));
        };

        const int jr = sgi - A.sched_off[blockIdx.x];  // this CTA's segment index (= round while < rounds)
        if (tid0) {  // prologue: all but one slot of every ring (planes zs-1, zs, ...)
            for (int tz = zs - 1; tz < zs - 1 + Rg::NU - 1; ++tz) issue_u(tz);
            for (int tz = zs - 1; tz < zs - 1 + Rg::NX - 1; ++tz) issue_x(tz);
            round_wait(A.round_ctr, jr, A.rounds);  // (the other threads wait at S1)
        }
        mbar_wait(&S.bar_u[cu.st], cu.ph);  // u at plane zs-1
        int su = cu.st;
        adv(cu, Rg::NU);

        // carried from step s-1 to step s (double-buffered by the 2x-unrolled loop)
        struct Carry {
            float vb[3];      // vbar(s-1)
            float uk, vk[3];  // u_k, v_k at s-1 (the primal of plane s-1)
            Hist h;           // histogram of s-1
            float pn[3], pz;  // p_{k+1}(s-1), p_z{k+1}(s-2)
            float qn[6];      // q_{k+1}(s-1)
        };
        Carry ca{}, cb{};

        auto step = [&](auto PAR, int s, const Carry& in, Carry& o) {
            constexpr int par = decltype(PAR)::value, pr = par ^ 1;
            const int zg = g.z0 + s;

            mbar_wait(&S.bar_u[cu.st], cu.ph);
            mbar_wait(&S.bar_x[cx.st], cx.ph);

            // ---- phase B: this cell's inputs of plane s (and u at s+1) into registers
            const float* U0 = &S.u[su][0][r][bc];
            const float* U1 = &S.u[cu.st][0][r][bc];
            auto OUT = [&](int f, int row) -> float* { return &S.out[f][row][0]; };
            const float* V0 = &S.v[cx.st][0][r][bc];
            const float* PQ = &S.pq[cx.st][0][r][bc];
            constexpr int F = R * TMA_BW;  // field stride in a ring slot
            const float uk = U0[0], um = U0[F];
            float vk[3], vb[3];
    #pragma unroll
            for (int k = 0; k < 3; ++k) {
                vk[k] = V0[k * F];
                vb[k] = fmaf(2.f, vk[k], -V0[(3 + k) * F]);
            }
            const float ub = fmaf(2.f, uk, -um);           // (a3) ubar(s)
            const float ub1 = fmaf(2.f, U1[0], -U1[F]);    // ubar(s+1)
            float pk[3], qk[6];
    #pragma unroll
            for (int k = 0; k < 3; ++k) pk[k] = PQ[k * F];
    #pragma unroll
            for (int m = 0; m < 6; ++m) qk[m] = PQ[(3 + m) * F];
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
            S.suv[par][0][r][cc] = ub;
            S.suv[par][1][r][cc] = vb[0];
            S.suv[par][2][r][cc] = vb[1];
            S.suv[par][3][r][cc] = vb[2];
            if (tid0) tma_wait_read0();  // the previous step's output staging has been read
            __syncthreads();             // S1
            if (tid0) {  // the ring slots of plane s-1 are free: prefetch what later steps consume
                if (s + Rg::NU - 1 <= ze + 1) issue_u(s + Rg::NU - 1);
                if (s + Rg::NX - 1 <= ze) issue_x(s + Rg::NX - 1);
            }
            su = cu.st;
            adv(cu, Rg::NU);
            adv(cx, Rg::NX);

            // ---- phases E (a1: dual D(s)) and F (a2: primal Pm(s-1)), specialised per warp
            // role and, for the owned rows of interior tiles away from the z ends, without
            // the boundary masks (all of them are true there)
            float pn[3] = {0.f, 0.f, 0.f}, qn[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            auto ef = [&](auto ROLEc, auto INTc) {
                constexpr int ROLE = decltype(ROLEc)::value;
                constexpr bool INT = decltype(INTc)::value;
                const bool zl = INT || zg < g.nz - 1;
                const bool needP = ROLE == 0 || ROLE == 1 || (ROLE == 3 && lane < 16 && r >= 1 && r <= TY);
                const bool needQ = ROLE == 0 || ROLE == 2 || (ROLE == 3 && lane >= 16 && r >= 1 && r <= TY);
                const bool xl_ = INT || xl, yl_ = INT || yl, xf_ = INT || xf, yf_ = INT || yf;
                if (needP) {
                    const float ux = S.suv[par][0][r][cc + 1];
                    const float uy = S.suv[par][0][r + 1][cc];
                    const float g0 = xl_ ? ux - ub : 0.f, g1 = yl_ ? uy - ub : 0.f, g2 = zl ? ub1 - ub : 0.f;
                    pn[0] = fmaf(sp.sigma, g0 - vb[0], pk[0]);
                    pn[1] = fmaf(sp.sigma, g1 - vb[1], pk[1]);
                    pn[2] = fmaf(sp.sigma, g2 - vb[2], pk[2]);
                    const float f = proj_scale(pn[0] * pn[0] + pn[1] * pn[1] + pn[2] * pn[2], sp.alpha1);
                    pn[0] *= f;
                    pn[1] *= f;
                    pn[2] *= f;
                }
                if (needQ) {
                    // vbar is exactly 0 outside the grid (TMA zero fill, zero halo planes at the
                    // global z ends), so the "l > 0" guards of D- are implicit
                    float dx[3], dy[3], dz[3];
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        const float vx = S.suv[par][1 + k][r][cc - 1];
                        const float vy = S.suv[par][1 + k][r - 1][cc];
                        dx[k] = fmaf(INT ? 1.f : mxl, vb[k], -vx);  // (x < nx-1 ? vb : 0) - vb(x-1)
                        dy[k] = fmaf(INT ? 1.f : myl, vb[k], -vy);
                        dz[k] = fmaf(zl ? 1.f : 0.f, vb[k], -in.vb[k]);
                    }
                    const float e[6] = {dx[0], dy[1], dz[2], 0.5f * (dy[0] + dx[1]), 0.5f * (dz[0] + dx[2]),
                                        0.5f * (dz[1] + dy[2])};
#pragma unroll
                    for (int m = 0; m < 6; ++m) qn[m] = fmaf(sp.sigma, e[m], qk[m]);
                    const float f = proj_scale(qn[0] * qn[0] + qn[1] * qn[1] + qn[2] * qn[2] +
                                                   2.f * (qn[3] * qn[3] + qn[4] * qn[4] + qn[5] * qn[5]),
                                               sp.alpha0);
#pragma unroll
                    for (int m = 0; m < 6; ++m) qn[m] *= f;
                }
                if (ROLE != 2) {  // p_x, p_y (x- and y-neighbours' div p)
                    S.sr[par][0][r][cc] = pn[0];
                    S.sr[par][1][r][cc] = pn[1];
                }
                if (ROLE != 1) {  // q_xx, q_xy, q_xz (x-neighbour) and q_xy, q_yy, q_yz (y-neighbour of div2 q)
                    S.sr[par][2][r][cc] = qn[0];
                    S.sr[par][3][r][cc] = qn[3];
                    S.sr[par][4][r][cc] = qn[4];
                    S.sr[par][5][r][cc] = qn[1];
                    S.sr[par][6][r][cc] = qn[5];
                }
                if constexpr (ROLE == 0) {
#pragma unroll
                    for (int k = 0; k < 3; ++k) OUT(4 + k, r - 1)[lane] = pn[k];
#pragma unroll
                    for (int m = 0; m < 6; ++m) OUT(7 + m, r - 1)[lane] = qn[m];
                    [[maybe_unused]] const bool inb = x < g.nx && y < g.ny;
                    [[maybe_unused]] const int64_t cell = (int64_t)y * g.px + x;
                    if (PEER && A.pdn && s == 0 && s >= zs && s < ze && inb) {  // q of plane 0 -> lower neighbour's top halo
                        float* o = A.pdn + (int64_t)A.pdn_top * g.plane + cell;
#pragma unroll
                        for (int m = 0; m < 6; ++m) o[(A.s_qn + m) * A.pdn_fs] = qn[m];
                    }
                    if (PEER && A.pup && s == g.nzl - 1 && s >= zs && s < ze && inb) {  // p of plane nzl-1 -> upper neighbour
                        float* o = A.pup + cell;
#pragma unroll
                        for (int k = 0; k < 3; ++k) o[(A.s_pn + k) * A.pup_fs] = pn[k];
                    }
                    if (s - 1 >= zs) {  // (a2) primal Pm(s-1)
                        const bool zl1 = INT || zg - 1 < g.nz - 1, zf1 = INT || zg - 1 > 0;
                        const float pxm = S.sr[pr][0][r][cc - 1];
                        const float pym = S.sr[pr][1][r - 1][cc];
                        const float divp = fmaf(INT ? 1.f : mxl, in.pn[0], -(xf_ ? pxm : 0.f)) +
                                           fmaf(INT ? 1.f : myl, in.pn[1], -(yf_ ? pym : 0.f)) +
                                           fmaf(zl1 ? 1.f : 0.f, in.pn[2], -(zf1 ? in.pz : 0.f));
                        const float qxx = S.sr[pr][2][r][cc + 1], qxy = S.sr[pr][3][r][cc + 1],
                                    qxz = S.sr[pr][4][r][cc + 1];
                        const float qyxy = S.sr[pr][3][r + 1][cc], qyyy = S.sr[pr][5][r + 1][cc],
                                    qyyz = S.sr[pr][6][r + 1][cc];
                        const float w0 = (xl_ ? qxx - in.qn[0] : 0.f) + (yl_ ? qyxy - in.qn[3] : 0.f) +
                                         (zl1 ? qn[4] - in.qn[4] : 0.f);
                        const float w1 = (xl_ ? qxy - in.qn[3] : 0.f) + (yl_ ? qyyy - in.qn[1] : 0.f) +
                                         (zl1 ? qn[5] - in.qn[5] : 0.f);
                        const float w2 = (xl_ ? qxz - in.qn[4] : 0.f) + (yl_ ? qyyz - in.qn[5] : 0.f) +
                                         (zl1 ? qn[2] - in.qn[2] : 0.f);
                        const float un = hist_prox<SLOTS, CT>(fmaf(sp.tau, divp, in.uk), sp.tl, in.h, A.C);
                        const float v0 = fmaf(sp.tau, in.pn[0] + w0, in.vk[0]);
                        const float v1 = fmaf(sp.tau, in.pn[1] + w1, in.vk[1]);
                        const float v2 = fmaf(sp.tau, in.pn[2] + w2, in.vk[2]);
                        OUT(0, r - 1)[lane] = un;
                        OUT(1, r - 1)[lane] = v0;
                        OUT(2, r - 1)[lane] = v1;
                        OUT(3, r - 1)[lane] = v2;
                        // u, v of a boundary plane -> the neighbour's halo (peer mode)
                        if constexpr (PEER) {
                        float* po = nullptr;
                        int64_t pfs = 0;
                        if (A.pdn && s - 1 == 0 && inb) {
                            po = A.pdn + (int64_t)A.pdn_top * g.plane + cell;
                            pfs = A.pdn_fs;
                        } else if (A.pup && s - 1 == g.nzl - 1 && inb) {
                            po = A.pup + cell;
                            pfs = A.pup_fs;
                        }
                        if (po) {
                            po[A.s_un * pfs] = un;
                            po[A.s_vn * pfs] = v0;
                            po[(A.s_vn + 1) * pfs] = v1;
                            po[(A.s_vn + 2) * pfs] = v2;
                        }
                        if (A.pdn && A.pup && s - 1 == 0 && s - 1 == g.nzl - 1 && inb) {  // 1-plane slab: both
                            float* o2 = A.pup + cell;
                            o2[A.s_un * A.pup_fs] = un;
                            o2[A.s_vn * A.pup_fs] = v0;
                            o2[(A.s_vn + 1) * A.pup_fs] = v1;
                            o2[(A.s_vn + 2) * A.pup_fs] = v2;
                        }
                        }
                    }
                }
            };
            using F0 = std::false_type;
            switch (role) {  // warp-uniform
                case 0:
                    if (tile_int && zg - 1 > 0 && zg < g.nz - 1)
                        ef(std::integral_constant<int, 0>{}, std::true_type{});
                    else
                        ef(std::integral_constant<int, 0>{}, F0{});
                    break;
                case 1: ef(std::integral_constant<int, 1>{}, F0{}); break;
                case 2: ef(std::integral_constant<int, 2>{}, F0{}); break;
                default: ef(std::integral_constant<int, 3>{}, F0{}); break;
            }
            fence_proxy_async();
            __syncthreads();  // S2 (as an mbarrier only the storing thread waits on: 25.2 vs 24.2 ms on C4)
            if (tid0) {
                if ((s >= zs && s < ze) || (A.keep_halo_dual && (s == -1 || s == g.nzl))) {
                    if (A.hints & 1) {
                        tma_store4_hint(&m_st3, OUT(4, 0), x0, y0, s + 1, A.s_pn, pol_ef);
                        tma_store4_hint(&m_st6, OUT(7, 0), x0, y0, s + 1, A.s_qn, pol_ef);
                    } else {
                        tma_store4(&m_st3, OUT(4, 0), x0, y0, s + 1, A.s_pn);
                        tma_store4(&m_st6, OUT(7, 0), x0, y0, s + 1, A.s_qn);
                    }
                }
                if (s - 1 >= zs) {
                    if (A.hints & 1) {
                        tma_store4_hint(&m_st1, OUT(0, 0), x0, y0, s, A.s_un, pol_ef);
                        tma_store4_hint(&m_st3, OUT(1, 0), x0, y0, s, A.s_vn, pol_ef);
                    } else {
                        tma_store4(&m_st1, OUT(0, 0), x0, y0, s, A.s_un);
                        tma_store4(&m_st3, OUT(1, 0), x0, y0, s, A.s_vn);
                    }
                }
                tma_commit();
            }

            // ---- carry to step s+1
            o.pz = in.pn[2];
    #pragma unroll
            for (int k = 0; k < 3; ++k) {
                o.pn[k] = pn[k];
                o.vb[k] = vb[k];
                o.vk[k] = vk[k];
            }
    #pragma unroll
            for (int m = 0; m < 6; ++m) o.qn[m] = qn[m];
            o.uk = uk;
            o.h = hc;
        };


        // steps s = zs-1 .. ze; the shared exchange planes alternate with the step's parity
        for (int s = zs - 1; s <= ze; s += 2) {
            step(std::integral_constant<int, 0>{}, s, ca, cb);
            if (s + 1 > ze) break;
            step(std::integral_constant<int, 1>{}, s + 1, cb, ca);
        }
        if (tid0) round_done(A.round_ctr, jr, A.rounds);  // round jr done (after S2 of its last step)
    }
    if (PEER && A.done) {  // peer mode: publish once every CTA's halo stores are visible system-wide
        __threadfence_system();
        __syncthreads();
        if (tid0 && atomicAdd(A.done, 1ull) == gridDim.x - 1) {
            atomicExch(A.done, 0ull);
            __threadfence_system();
            if (A.flag_dn_remote) st_release_sys(A.flag_dn_remote, A.seq);
            if (A.flag_up_remote) st_release_sys(A.flag_up_remote, A.seq);
        }
    }
    if (tid0) tma_wait0();
}

}  // namespace tgvk

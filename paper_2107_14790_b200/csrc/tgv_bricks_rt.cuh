// tgv_bricks_rt.cuh -- context and C ABI of the block-sparse brick-set solver
// (include/tgv_bricks.h; R24).  Included at the end of tgv_runtime.cu
// (one translation unit: the kernels of tgv_kernels.cuh are shared, not duplicated).
//
// The context owns the fp32 state (30 rotating slots of nbricks * E^3 floats, the
// slot rotation of tgv_runtime.cu), the neighbour table and frozen flags, the
// counts (u8 when every count <= 255, else u16), a stream and timing events.
#include <unordered_map>

#include "../../include/tgv_bricks.h"
#include "tgv_bricks.cuh"
#include "tgv_bricks_fused.cuh"
#include "tgv_mixed.cuh"

struct tgv_bricks {
    int device = 0;
    int LE = 0, E = 0;
    int64_t nbricks = 0, nvox = 0;
    int nbins = 0, slots = 8, count_bytes = 0;
    float centers[16]{};
    float lambda = 0, alpha0 = 0, alpha1 = 0, tau = 0, sigma = 0;

    float* state = nullptr;     // NSLOT slots of nvox floats
    int* nbr = nullptr;         // [nbricks][6]
    uint8_t* frozen = nullptr;  // [nbricks]
    uint8_t* aface = nullptr;   // [nbricks]: solved face neighbours (BrickGeo::aface)
    int64_t nfrozen = 0;
    int* d_alist = nullptr;     // solved brick indices
    int* d_faces = nullptr;     // (frozen brick, face) pairs with a solved brick across the face: y, z faces first
    int n_alist = 0, n_faces = 0, n_faces_yz = 0;  // the fused sweep computes the x faces itself
    int* d_nb27 = nullptr;      // [n_alist][27] neighbourhood of each solved brick (fused schedule)
    int schedule = TGV_SCHEDULE_SPLIT;
    int64_t s_voxels = 0;       // voxels of S (solved + frozen face-adjacent to solved)
    int* d_coords = nullptr;    // [nbricks][3]
    int* d_parent = nullptr;    // [nbricks]: parent brick index (tgv_bricks_prolong_from)
    std::vector<int32_t> coords_h;
    void* hist = nullptr;       // [nvox][slots] of u8 / u16
    double* partials = nullptr;
    double* d_out = nullptr;
    unsigned int* d_maxc = nullptr;
    int energy_blocks = 0;
    int64_t device_bytes = 0;

    int64_t k = 0;
    bool loaded = false, poisoned = false;
    cudaStream_t stream = nullptr;
    char err[512] = "";

    // 2:1 mixed-level sets (tgv_bricks_create_mixed, R27)
    bool mixed = false;
    std::vector<uint8_t> levels_h;
    uint8_t* d_level = nullptr;  // [nbricks]
    uint8_t* d_kind = nullptr;   // [nbricks][6]
    int* d_nbr4 = nullptr;       // [nbricks][6][4]
    uint8_t* d_par = nullptr;    // [nbricks]
    uint8_t* d_sface = nullptr;  // [nbricks][6]
    int* d_mfaces = nullptr;     // (frozen brick, face | quadrant mask << 3) towards solved voxels
    int n_mfaces = 0;
    // solved bricks split by stencil: level 0 with only same-level (or no) face neighbours
    // run the uniform brick kernels (R27's operators are R24's there, bit for bit), the
    // rest the mixed kernels
    int* d_alist_reg = nullptr;
    int* d_alist_gen = nullptr;
    int n_alist_reg = 0, n_alist_gen = 0;
    // FUSED schedule of a mixed set (E = 32): solved level-0 bricks whose whole 26-neighbourhood
    // is level 0 or empty run the fused brick sweep (their 27-entry tables); every other
    // solved brick the mixed SPLIT kernels
    int* d_fnb27 = nullptr;
    int* d_alist_fgen = nullptr;  // the solved bricks the fused sweep does not cover
    int n_fused = 0, n_fgen = 0;

    bool timing = false;
    std::vector<cudaEvent_t> ev;  // pairs
    std::vector<int> ev_kind;     // 0 dual, 1 primal, 2 energy, 3 fused
    double t_ms[4]{};
    int64_t t_n[4]{};
};

namespace {

thread_local char g_bricks_error[512] = "";

int bfail(tgv_bricks* c, int code, const char* fmt, ...)
{
    char* dst = c ? c->err : g_bricks_error;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(dst, 512, fmt, ap);
    va_end(ap);
    if (c && code == TGV_ECUDA) c->poisoned = true;
    return code;
}

#define BCU(call)                                                                                  \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return bfail(c, TGV_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
    } while (0)

inline float* bslot(tgv_bricks* c, int s) { return c->state + (int64_t)s * c->nvox; }

int bready(tgv_bricks* c)
{
    if (!c) return TGV_EINVAL;
    if (c->poisoned) return bfail(c, TGV_ESTATE, "context poisoned by an earlier CUDA failure");
    if (cudaSetDevice(c->device) != cudaSuccess) {
        cudaGetLastError();
        return bfail(c, TGV_ECUDA, "cudaSetDevice(%d) failed", c->device);
    }
    return TGV_OK;
}

BrickGeo bgeo(const tgv_bricks* c) { return BrickGeo{(int)c->nvox, c->nbr, c->frozen, c->aface}; }
MixGeo mgeo(const tgv_bricks* c)
{
    return MixGeo{(int)c->nvox, c->d_level, c->d_kind, c->d_nbr4, c->d_par, c->frozen, c->d_sface};
}

IterPtrs biter_ptrs(tgv_bricks* c, int64_t k)
{
    const Bufs b = bufs(k);
    IterPtrs a{};
    a.uk = bslot(c, slotU(b.cu));
    a.um = bslot(c, slotU(b.pu));
    a.un = bslot(c, slotU(b.nu));
    for (int d = 0; d < 3; ++d) {
        a.vk[d] = bslot(c, slotV(b.cu, d));
        a.vm[d] = bslot(c, slotV(b.pu, d));
        a.vn[d] = bslot(c, slotV(b.nu, d));
        a.pk[d] = bslot(c, slotP(b.cp, d));
        a.pn[d] = bslot(c, slotP(b.np, d));
    }
    for (int m = 0; m < 6; ++m) {
        a.qk[m] = bslot(c, slotQ(b.cp, m));
        a.qn[m] = bslot(c, slotQ(b.np, m));
    }
    a.hist = c->hist;
    return a;
}

Centers bcenters(const tgv_bricks* c)
{
    Centers C;
    for (int b = 0; b < 16; ++b) C.c[b] = b < c->nbins ? c->centers[b] : INFINITY;
    return C;
}

int btimer(tgv_bricks* c, int kind, bool end)
{
    if (!c->timing) return TGV_OK;
    if (!end) {
        cudaEvent_t e[2];
        BCU(cudaEventCreate(&e[0]));
        BCU(cudaEventCreate(&e[1]));
        c->ev.push_back(e[0]);
        c->ev.push_back(e[1]);
        c->ev_kind.push_back(kind);
        BCU(cudaEventRecord(e[0], c->stream));
    } else {
        BCU(cudaEventRecord(c->ev.back(), c->stream));
    }
    return TGV_OK;
}

int btimer_collect(tgv_bricks* c)
{
    for (size_t j = 0; j < c->ev_kind.size(); ++j) {
        float ms = 0.f;
        BCU(cudaEventElapsedTime(&ms, c->ev[2 * j], c->ev[2 * j + 1]));
        c->t_ms[c->ev_kind[j]] += ms;
        c->t_n[c->ev_kind[j]] += 1;
    }
    for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
    c->ev.clear();
    c->ev_kind.clear();
    return TGV_OK;
}

template <int LE>
void launch_brick_primal_le(tgv_bricks* c, const IterPtrs& a, const StepParams& sp)
{
    const BrickGeo bg = bgeo(c);
    const Centers C = bcenters(c);
    const int n = c->n_alist << (3 * LE), blocks = (n + 255) / 256;
    if (!n) return;
    const int* L = c->d_alist;
    if (c->slots == 8 && c->count_bytes == 1) brick_primal_kernel<LE, 8, uint8_t><<<blocks, 256, 0, c->stream>>>(a, bg, sp, C, L, n);
    else if (c->slots == 8) brick_primal_kernel<LE, 8, uint16_t><<<blocks, 256, 0, c->stream>>>(a, bg, sp, C, L, n);
    else if (c->count_bytes == 1) brick_primal_kernel<LE, 16, uint8_t><<<blocks, 256, 0, c->stream>>>(a, bg, sp, C, L, n);
    else brick_primal_kernel<LE, 16, uint16_t><<<blocks, 256, 0, c->stream>>>(a, bg, sp, C, L, n);
}

template <int LE>
void launch_brick_init_le(tgv_bricks* c)
{
    const BrickGeo bg = bgeo(c);
    const Centers C = bcenters(c);
    float* u0 = bslot(c, slotU(0));
    float* u2 = bslot(c, slotU(2));  // bufs(0): current 0, previous 2
    if (c->slots == 8 && c->count_bytes == 1) brick_init_kernel<LE, 8, uint8_t><<<148 * 8, 256, 0, c->stream>>>(u0, u2, c->hist, bg, C);
    else if (c->slots == 8) brick_init_kernel<LE, 8, uint16_t><<<148 * 8, 256, 0, c->stream>>>(u0, u2, c->hist, bg, C);
    else if (c->count_bytes == 1) brick_init_kernel<LE, 16, uint8_t><<<148 * 8, 256, 0, c->stream>>>(u0, u2, c->hist, bg, C);
    else brick_init_kernel<LE, 16, uint16_t><<<148 * 8, 256, 0, c->stream>>>(u0, u2, c->hist, bg, C);
}

template <int LE>
void launch_brick_energy_le(tgv_bricks* c, const EnergyArgs& ea)
{
    const BrickGeo bg = bgeo(c);
    const EnergyConsts K8 = energy_consts(c->centers, c->nbins, 8), K16 = energy_consts(c->centers, c->nbins, 16);
    const int nb = c->energy_blocks;
    if (c->slots == 8 && c->count_bytes == 1) brick_energy_kernel<LE, 8, uint8_t><<<nb, 256, 0, c->stream>>>(ea, bg, K8, c->partials);
    else if (c->slots == 8) brick_energy_kernel<LE, 8, uint16_t><<<nb, 256, 0, c->stream>>>(ea, bg, K8, c->partials);
    else if (c->count_bytes == 1) brick_energy_kernel<LE, 16, uint8_t><<<nb, 256, 0, c->stream>>>(ea, bg, K16, c->partials);
    else brick_energy_kernel<LE, 16, uint16_t><<<nb, 256, 0, c->stream>>>(ea, bg, K16, c->partials);
}

template <int LE>
void launch_mixed_energy_le(tgv_bricks* c, const EnergyArgs& ea)
{
    const MixGeo g = mgeo(c);
    const EnergyConsts K8 = energy_consts(c->centers, c->nbins, 8), K16 = energy_consts(c->centers, c->nbins, 16);
    const int nb = c->energy_blocks;
    if (c->slots == 8 && c->count_bytes == 1) mixed_energy_kernel<LE, 8, uint8_t><<<nb, 256, 0, c->stream>>>(ea, g, K8, c->partials);
    else if (c->slots == 8) mixed_energy_kernel<LE, 8, uint16_t><<<nb, 256, 0, c->stream>>>(ea, g, K8, c->partials);
    else if (c->count_bytes == 1) mixed_energy_kernel<LE, 16, uint8_t><<<nb, 256, 0, c->stream>>>(ea, g, K16, c->partials);
    else mixed_energy_kernel<LE, 16, uint16_t><<<nb, 256, 0, c->stream>>>(ea, g, K16, c->partials);
}

template <int LE>
void launch_mixed_dual_le(tgv_bricks* c, const IterPtrs& a, const StepParams& sp)
{
    const int nr = c->n_alist_reg << (3 * LE), n0 = c->n_alist_gen << (3 * LE), n1 = c->n_mfaces << (2 * LE);
    if (nr) brick_dual_kernel<LE, 0><<<(nr + 255) / 256, 256, 0, c->stream>>>(a, bgeo(c), sp, c->d_alist_reg, nr);
    if (n0) mixed_dual_kernel<LE, 0><<<(n0 + 255) / 256, 256, 0, c->stream>>>(a, mgeo(c), sp, c->d_alist_gen, n0);
    if (n1) mixed_dual_kernel<LE, 1><<<(n1 + 255) / 256, 256, 0, c->stream>>>(a, mgeo(c), sp, c->d_mfaces, n1);
}

template <int LE>
void launch_mixed_primal_le(tgv_bricks* c, const IterPtrs& a, const StepParams& sp)
{
    const Centers C = bcenters(c);
    const int nr = c->n_alist_reg << (3 * LE), br = (nr + 255) / 256;
    if (nr) {
        const BrickGeo bg = bgeo(c);
        const int* R = c->d_alist_reg;
        if (c->slots == 8 && c->count_bytes == 1) brick_primal_kernel<LE, 8, uint8_t><<<br, 256, 0, c->stream>>>(a, bg, sp, C, R, nr);
        else if (c->slots == 8) brick_primal_kernel<LE, 8, uint16_t><<<br, 256, 0, c->stream>>>(a, bg, sp, C, R, nr);
        else if (c->count_bytes == 1) brick_primal_kernel<LE, 16, uint8_t><<<br, 256, 0, c->stream>>>(a, bg, sp, C, R, nr);
        else brick_primal_kernel<LE, 16, uint16_t><<<br, 256, 0, c->stream>>>(a, bg, sp, C, R, nr);
    }
    const int n = c->n_alist_gen << (3 * LE), blocks = (n + 255) / 256;
    if (!n) return;
    const int* L = c->d_alist_gen;
    const MixGeo g = mgeo(c);
    if (c->slots == 8 && c->count_bytes == 1) mixed_primal_kernel<LE, 8, uint8_t><<<blocks, 256, 0, c->stream>>>(a, g, sp, C, L, n);
    else if (c->slots == 8) mixed_primal_kernel<LE, 8, uint16_t><<<blocks, 256, 0, c->stream>>>(a, g, sp, C, L, n);
    else if (c->count_bytes == 1) mixed_primal_kernel<LE, 16, uint8_t><<<blocks, 256, 0, c->stream>>>(a, g, sp, C, L, n);
    else mixed_primal_kernel<LE, 16, uint16_t><<<blocks, 256, 0, c->stream>>>(a, g, sp, C, L, n);
}

#define BRICK_LE_DISPATCH(fn, ...)            \
    switch (c->LE) {                          \
        case 2: fn<2>(__VA_ARGS__); break;    \
        case 3: fn<3>(__VA_ARGS__); break;    \
        case 4: fn<4>(__VA_ARGS__); break;    \
        default: fn<5>(__VA_ARGS__); break;   \
    }

// the solved bricks, then the frozen bricks' faces towards solved bricks (same stream:
// the face launch only reads inputs of this iteration and writes other voxels)
template <int LE>
void launch_brick_dual_le(tgv_bricks* c, const IterPtrs& a, const StepParams& sp)
{
    const int n0 = c->n_alist << (3 * LE), n1 = c->n_faces << (2 * LE);
    if (n0) brick_dual_kernel<LE, 0><<<(n0 + 255) / 256, 256, 0, c->stream>>>(a, bgeo(c), sp, c->d_alist, n0);
    if (n1) brick_dual_kernel<LE, 1><<<(n1 + 255) / 256, 256, 0, c->stream>>>(a, bgeo(c), sp, c->d_faces, n1);
}

template <int SLOTS, typename CT>
void launch_brick_fused_t(tgv_bricks* c, const BrickFusedArgs& A)
{
    auto kern = brick_fused_kernel<5, SLOTS, CT>;
    static thread_local int configured_dev = -1;  // the attribute is per device
    if (configured_dev != c->device) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BrickFusedSmem));
        configured_dev = c->device;
    }
    // two CTAs per swept brick: A.n_alist rows of A.nb27 (all solved bricks, or the mixed
    // set's fused subset -- never c->n_alist there)
    if (A.n_alist) kern<<<2 * A.n_alist, dim3(32, BF_WARPS), sizeof(BrickFusedSmem), c->stream>>>(A);
}

// FUSED schedule: the frozen-face duals, then one single sweep over the solved bricks
int brick_iterate_fused(tgv_bricks* c, int32_t n)
{
    const StepParams sp{c->sigma, c->tau, c->alpha1, c->alpha0, c->tau * c->lambda};
    int rc;
    for (int32_t it = 0; it < n; ++it) {
        const IterPtrs a = biter_ptrs(c, c->k);
        const int fold_x = (int)env_int("TGV_BRICK_FOLD_X", 1);
        const int nf = fold_x ? c->n_faces_yz : c->n_faces;
        if (nf) {  // y and z faces (and x faces unless the fused sweep stores them)
            const int n1 = nf << (2 * 5);
            if ((rc = btimer(c, 0, false))) return rc;
            brick_dual_kernel<5, 1><<<(n1 + 255) / 256, 256, 0, c->stream>>>(a, bgeo(c), sp, c->d_faces, n1);
            BCU(cudaGetLastError());
            if ((rc = btimer(c, 0, true))) return rc;
        }
        if (c->n_alist) {
            BrickFusedArgs A{a, sp, bcenters(c), c->d_nb27, c->frozen, c->n_alist, fold_x};
            if ((rc = btimer(c, 3, false))) return rc;
            if (c->slots == 8 && c->count_bytes == 1) launch_brick_fused_t<8, uint8_t>(c, A);
            else if (c->slots == 8) launch_brick_fused_t<8, uint16_t>(c, A);
            else if (c->count_bytes == 1) launch_brick_fused_t<16, uint8_t>(c, A);
            else launch_brick_fused_t<16, uint16_t>(c, A);
            BCU(cudaGetLastError());
            if ((rc = btimer(c, 3, true))) return rc;
        }
        c->k += 1;
    }
    return TGV_OK;
}

// FUSED schedule of a mixed set (R27): per iteration (1) the duals of S on the frozen
// bricks (mixed face launch, every face kind) and of the solved bricks the fused sweep does
// not cover (mixed dual), (2) the fused sweep over the solved level-0 bricks whose whole
// 26-neighbourhood is level 0 or empty (there R27's operators are R24's, and the sweep
// recomputes every halo dual it needs), (3) the mixed primal of the remaining solved
// bricks, which reads the duals (1) and (2) stored.
int mixed_iterate_fused(tgv_bricks* c, int32_t n)
{
    const StepParams sp{c->sigma, c->tau, c->alpha1, c->alpha0, c->tau * c->lambda};
    int rc;
    for (int32_t it = 0; it < n; ++it) {
        const IterPtrs a = biter_ptrs(c, c->k);
        if ((rc = btimer(c, 0, false))) return rc;
        {
            const int n0 = c->n_fgen << 15, n1 = c->n_mfaces << 10;
            if (n0) mixed_dual_kernel<5, 0><<<(n0 + 255) / 256, 256, 0, c->stream>>>(a, mgeo(c), sp, c->d_alist_fgen, n0);
            if (n1) mixed_dual_kernel<5, 1><<<(n1 + 255) / 256, 256, 0, c->stream>>>(a, mgeo(c), sp, c->d_mfaces, n1);
        }
        BCU(cudaGetLastError());
        if ((rc = btimer(c, 0, true))) return rc;
        if (c->n_fused) {
            BrickFusedArgs A{a, sp, bcenters(c), c->d_fnb27, c->frozen, c->n_fused, 0};
            if ((rc = btimer(c, 3, false))) return rc;
            if (c->slots == 8 && c->count_bytes == 1) launch_brick_fused_t<8, uint8_t>(c, A);
            else if (c->slots == 8) launch_brick_fused_t<8, uint16_t>(c, A);
            else if (c->count_bytes == 1) launch_brick_fused_t<16, uint8_t>(c, A);
            else launch_brick_fused_t<16, uint16_t>(c, A);
            BCU(cudaGetLastError());
            if ((rc = btimer(c, 3, true))) return rc;
        }
        if (c->n_fgen) {
            IterPtrs ap = a;
            for (int d = 0; d < 3; ++d) ap.pk[d] = a.pn[d];
            for (int m = 0; m < 6; ++m) ap.qk[m] = a.qn[m];
            const Centers C = bcenters(c);
            const int n0 = c->n_fgen << 15, blocks = (n0 + 255) / 256;
            const MixGeo g = mgeo(c);
            const int* L = c->d_alist_fgen;
            if ((rc = btimer(c, 1, false))) return rc;
            if (c->slots == 8 && c->count_bytes == 1) mixed_primal_kernel<5, 8, uint8_t><<<blocks, 256, 0, c->stream>>>(ap, g, sp, C, L, n0);
            else if (c->slots == 8) mixed_primal_kernel<5, 8, uint16_t><<<blocks, 256, 0, c->stream>>>(ap, g, sp, C, L, n0);
            else if (c->count_bytes == 1) mixed_primal_kernel<5, 16, uint8_t><<<blocks, 256, 0, c->stream>>>(ap, g, sp, C, L, n0);
            else mixed_primal_kernel<5, 16, uint16_t><<<blocks, 256, 0, c->stream>>>(ap, g, sp, C, L, n0);
            BCU(cudaGetLastError());
            if ((rc = btimer(c, 1, true))) return rc;
        }
        c->k += 1;
    }
    return TGV_OK;
}

int brick_iterate_enqueue(tgv_bricks* c, int32_t n)
{
    if (c->schedule == TGV_SCHEDULE_FUSED && c->mixed) return mixed_iterate_fused(c, n);
    if (c->schedule == TGV_SCHEDULE_FUSED) return brick_iterate_fused(c, n);
    const StepParams sp{c->sigma, c->tau, c->alpha1, c->alpha0, c->tau * c->lambda};
    int rc;
    for (int32_t it = 0; it < n; ++it) {
        const IterPtrs a = biter_ptrs(c, c->k);
        if ((rc = btimer(c, 0, false))) return rc;
        if (c->mixed) {
            BRICK_LE_DISPATCH(launch_mixed_dual_le, c, a, sp);
        } else {
            BRICK_LE_DISPATCH(launch_brick_dual_le, c, a, sp);
        }
        BCU(cudaGetLastError());
        if ((rc = btimer(c, 0, true))) return rc;
        // the primal reads p_{k+1}, q_{k+1}: the dual's outputs
        IterPtrs ap = a;
        for (int d = 0; d < 3; ++d) ap.pk[d] = a.pn[d];
        for (int m = 0; m < 6; ++m) ap.qk[m] = a.qn[m];
        if ((rc = btimer(c, 1, false))) return rc;
        if (c->mixed) {
            BRICK_LE_DISPATCH(launch_mixed_primal_le, c, ap, sp);
        } else {
            BRICK_LE_DISPATCH(launch_brick_primal_le, c, ap, sp);
        }
        BCU(cudaGetLastError());
        if ((rc = btimer(c, 1, true))) return rc;
        c->k += 1;
    }
    return TGV_OK;
}

template <typename T>
void launch_brick_pack(tgv_bricks* c, const void* src, int64_t nv, uint16_t* dst)
{
    if (c->slots == 8)
        brick_pack_kernel<T, 8><<<148 * 8, 256, 0, c->stream>>>((const T*)src, nv, c->nbins, dst, c->d_maxc);
    else
        brick_pack_kernel<T, 16><<<148 * 8, 256, 0, c->stream>>>((const T*)src, nv, c->nbins, dst, c->d_maxc);
}

int bricks_init_state(tgv_bricks* c);

// Stream-ordered allocations of the big per-context buffers (the state, the counts and the
// load staging) from the device's default memory pool, whose release threshold is set to
// "keep everything": a context destroyed and the next one created -- the parts of a brick
// level streamed through one GPU -- reuse the same reserved device memory instead of
// unmapping and re-mapping 10+ GB (cudaFree of a part's state took 6 ms to 2 s, and its
// implicit device synchronisation stalls every stream; profiles/r2s_parts_probe.txt).
void* pool_alloc(tgv_bricks* c, size_t bytes)
{
    static std::atomic<uint64_t> thr_set{0};
    const uint64_t bit = 1ull << (c->device & 63);
    if (!(thr_set.load() & bit)) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, c->device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaGetLastError();
        thr_set.fetch_or(bit);
    }
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes, c->stream) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}
void pool_free(tgv_bricks* c, void* p)
{
    if (p) cudaFreeAsync(p, c->stream);
}

// shared tail of tgv_bricks_load / tgv_bricks_vote_depth_maps: range check of the
// u16 counts in h16 (max in c->d_maxc), u8 narrowing, state initialisation (R9)
int bricks_finish_counts(tgv_bricks* c, const uint16_t* h16)
{
    const size_t n16 = (size_t)c->nvox * c->slots;
    unsigned int maxc = 0;
    BCU(cudaMemcpyAsync(&maxc, c->d_maxc, sizeof maxc, cudaMemcpyDeviceToHost, c->stream));
    BCU(cudaStreamSynchronize(c->stream));
    if (maxc > 65535u) return bfail(c, TGV_ERANGE, "histogram count %u exceeds 65535", maxc);
    const int cb = maxc <= 255u && env_int("TGV_FORCE_U16", 0) == 0 ? 1 : 2;
    if (c->hist && cb != c->count_bytes) {
        pool_free(c, c->hist);
        c->device_bytes -= (int64_t)n16 * c->count_bytes;
        c->hist = nullptr;
    }
    if (!c->hist) {
        if (!(c->hist = pool_alloc(c, n16 * cb))) return bfail(c, TGV_ENOMEM, "count store allocation failed");
        c->device_bytes += (int64_t)n16 * cb;
    }
    c->count_bytes = cb;
    if (cb == 1) compact_counts_kernel<<<148 * 8, 256, 0, c->stream>>>(h16, (uint8_t*)c->hist, (int64_t)n16);
    else BCU(cudaMemcpyAsync(c->hist, h16, sizeof(uint16_t) * n16, cudaMemcpyDeviceToDevice, c->stream));
    BCU(cudaGetLastError());
    return bricks_init_state(c);
}

// initial state (R9): zero every slot, then u_0 into the current and previous u
int bricks_init_state(tgv_bricks* c)
{
    BCU(cudaMemsetAsync(c->state, 0, sizeof(float) * (size_t)NSLOT * c->nvox, c->stream));
    BRICK_LE_DISPATCH(launch_brick_init_le, c);
    BCU(cudaGetLastError());
    BCU(cudaStreamSynchronize(c->stream));
    c->k = 0;
    c->loaded = true;
    return TGV_OK;
}

}  // namespace

extern "C" {

const char* tgv_bricks_last_error(const tgv_bricks* c) { return c ? c->err : g_bricks_error; }

}  // extern "C"

namespace {
int build_mixed_tables(tgv_bricks* c, const tgv_brickset* S, const uint8_t* levels, const std::vector<uint8_t>& fr);

int bricks_create_impl(const tgv_brickset* S, const tgv_params* P, int dev, tgv_bricks** out, const uint8_t* levels)
{
    tgv_bricks* c = nullptr;
    if (!S || !P || !out) return bfail(c, TGV_EINVAL, "NULL argument");
    *out = nullptr;
    int LE = -1;
    for (int l = 2; l <= 5; ++l)
        if (S->edge == (1 << l)) LE = l;
    if (LE < 0) return bfail(c, TGV_EINVAL, "brick edge %d not in {4, 8, 16, 32}", S->edge);
    if (S->nbricks < 1 || !S->coords) return bfail(c, TGV_EINVAL, "need nbricks >= 1 and coords");
    const int64_t nvox = S->nbricks << (3 * LE);
    if (nvox >= (int64_t(1) << 31)) return bfail(c, TGV_EINVAL, "nbricks * E^3 must be < 2^31");
    if (P->nbins < 1 || P->nbins > 16) return bfail(c, TGV_EINVAL, "nbins must be in [1, 16]");
    if (!P->bin_centers) return bfail(c, TGV_EINVAL, "bin_centers is NULL");
    for (int b = 0; b < P->nbins; ++b) {
        const float cb = P->bin_centers[b];
        if (!std::isfinite(cb) || cb < -1.f || cb > 1.f) return bfail(c, TGV_EINVAL, "bin centre %d outside [-1,1]", b);
        if (b > 0 && !(cb > P->bin_centers[b - 1])) return bfail(c, TGV_EINVAL, "bin centres not strictly increasing");
    }
    const float vals[5] = {P->lambda, P->alpha0, P->alpha1, P->tau, P->sigma};
    for (float v : vals)
        if (!std::isfinite(v) || v < 0.f) return bfail(c, TGV_EINVAL, "parameters must be finite and >= 0");
    if (!(P->tau > 0.f) || !(P->sigma > 0.f)) return bfail(c, TGV_EINVAL, "tau and sigma must be > 0");
    if ((double)P->tau * (double)P->sigma * 16.0 > 1.0 + 1e-6)
        return bfail(c, TGV_EINVAL, "step sizes violate tau*sigma*16 <= 1 (tau=%g sigma=%g)", P->tau, P->sigma);

    // neighbour table from the coordinates
    const int64_t nb = S->nbricks;
    std::vector<int> nbr((size_t)nb * 6, -1);
    {
        std::unordered_map<uint64_t, int> at;
        at.reserve((size_t)nb * 2);
        // (level, coordinates): a one-level set has level 0 everywhere
        auto key = [](int64_t l, int64_t x, int64_t y, int64_t z) {
            return (uint64_t)x | (uint64_t)y << 20 | (uint64_t)z << 40 | (uint64_t)l << 60;
        };
        for (int64_t b = 0; b < nb; ++b) {
            const int32_t* q = S->coords + 3 * b;
            for (int a = 0; a < 3; ++a)
                if (q[a] < 0 || q[a] >= (1 << 20)) return bfail(c, TGV_EINVAL, "brick %lld coordinate outside [0, 2^20)", (long long)b);
            if (levels && levels[b] > 7) return bfail(c, TGV_EINVAL, "brick %lld level %d > 7", (long long)b, levels[b]);
            if (!at.emplace(key(levels ? levels[b] : 0, q[0], q[1], q[2]), (int)b).second)
                return bfail(c, TGV_EINVAL, "duplicate brick coordinates (%d, %d, %d)", q[0], q[1], q[2]);
        }
        for (int64_t b = 0; b < nb; ++b) {
            const int32_t* q = S->coords + 3 * b;
            const int lv = levels ? levels[b] : 0;
            for (int a = 0; a < 3; ++a)
                for (int d = 0; d < 2; ++d) {
                    int64_t r[3] = {q[0], q[1], q[2]};
                    r[a] += d ? 1 : -1;
                    if (r[a] < 0 || r[a] >= (1 << 20)) continue;
                    auto it = at.find(key(lv, r[0], r[1], r[2]));
                    if (it != at.end()) nbr[(size_t)b * 6 + 2 * a + d] = it->second;
                }
        }
    }

    c = new (std::nothrow) tgv_bricks();
    if (!c) return bfail(nullptr, TGV_ENOMEM, "host allocation failed");
    auto bail = [&](int code) {
        snprintf(g_bricks_error, sizeof g_bricks_error, "%s", c->err);
        tgv_bricks_destroy(c);
        return code;
    };
    c->device = dev;
    c->LE = LE;
    c->E = 1 << LE;
    c->nbricks = nb;
    c->nvox = nvox;
    c->nbins = P->nbins;
    c->slots = P->nbins <= 8 ? 8 : 16;
    for (int b = 0; b < P->nbins; ++b) c->centers[b] = P->bin_centers[b];
    c->lambda = P->lambda;
    c->alpha0 = P->alpha0;
    c->alpha1 = P->alpha1;
    c->tau = P->tau;
    c->sigma = P->sigma;
    if (cudaSetDevice(dev) != cudaSuccess) {
        cudaGetLastError();
        bfail(c, TGV_ECUDA, "cudaSetDevice(%d) failed", dev);
        return bail(TGV_ECUDA);
    }
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        bfail(c, TGV_ECUDA, "stream creation failed");
        return bail(TGV_ECUDA);
    }
    c->energy_blocks = 148 * 4;
    const size_t state_bytes = sizeof(float) * (size_t)NSLOT * (size_t)nvox;
    if (!(c->state = (float*)pool_alloc(c, state_bytes)) || cudaMalloc(&c->nbr, sizeof(int) * 6 * (size_t)nb) != cudaSuccess ||
        cudaMalloc(&c->frozen, (size_t)nb) != cudaSuccess || cudaMalloc(&c->aface, (size_t)nb) != cudaSuccess ||
        cudaMalloc(&c->partials, sizeof(double) * EN_TERMS * c->energy_blocks) != cudaSuccess ||
        cudaMalloc(&c->d_out, sizeof(double) * EN_TERMS) != cudaSuccess ||
        cudaMalloc(&c->d_maxc, sizeof(unsigned int)) != cudaSuccess) {
        cudaGetLastError();
        bfail(c, TGV_ENOMEM, "device allocation failed (%zu B of state)", state_bytes);
        return bail(TGV_ENOMEM);
    }
    cudaStreamSynchronize(c->stream);  // the pool allocation is usable from any stream from here on
    c->device_bytes = (int64_t)state_bytes + 7 * nb + (int64_t)sizeof(double) * EN_TERMS * (c->energy_blocks + 1);
    std::vector<uint8_t> fr((size_t)nb, 0), af((size_t)nb, 0);
    if (S->frozen)
        for (int64_t b = 0; b < nb; ++b) fr[(size_t)b] = S->frozen[b] ? 1 : 0;
    const int64_t E2 = (int64_t)c->E * c->E;
    c->s_voxels = 0;
    for (int64_t b = 0; b < nb; ++b) {
        for (int f = 0; f < 6; ++f) {
            const int n = nbr[(size_t)b * 6 + f];
            if (n >= 0 && !fr[(size_t)n]) af[(size_t)b] |= (uint8_t)(1u << f);
        }
        if (!fr[(size_t)b]) {
            c->s_voxels += E2 * c->E;
            continue;
        }
        ++c->nfrozen;
        // frozen voxels on the solved faces (inclusion-exclusion over the faces' edges and corners)
        int cnt[3] = {0, 0, 0};
        for (int k = 0; k < 3; ++k) cnt[k] = ((af[(size_t)b] >> (2 * k)) & 1) + ((af[(size_t)b] >> (2 * k + 1)) & 1);
        const int64_t Em2[3] = {c->E - cnt[0], c->E - cnt[1], c->E - cnt[2]};
        c->s_voxels += E2 * c->E - Em2[0] * Em2[1] * Em2[2];
    }
    std::vector<int> alist, faces;
    for (int pass = 0; pass < 2; ++pass) {  // y / z faces, then x faces
        for (int64_t b = 0; b < nb; ++b) {
            if (!fr[(size_t)b]) {
                if (pass == 0) alist.push_back((int)b);
                continue;
            }
            for (int f = pass == 0 ? 2 : 0; f < (pass == 0 ? 6 : 2); ++f)
                if (af[(size_t)b] >> f & 1) {
                    faces.push_back((int)b);
                    faces.push_back(f);
                }
        }
        if (pass == 0) c->n_faces_yz = (int)faces.size() / 2;
    }
    // optional Morton order of the solved bricks (TGV_BRICK_MORTON=1); the result does
    // not depend on the order (Jacobi sweeps)
    {
        auto spread = [](uint64_t v) {
            v &= 0x1FFFFF;
            v = (v | v << 32) & 0x1F00000000FFFFull;
            v = (v | v << 16) & 0x1F0000FF0000FFull;
            v = (v | v << 8) & 0x100F00F00F00F00Full;
            v = (v | v << 4) & 0x10C30C30C30C30C3ull;
            v = (v | v << 2) & 0x1249249249249249ull;
            return v;
        };
        auto mort = [&](int b) {
            const int32_t* q = S->coords + 3 * (int64_t)b;
            return spread((uint64_t)q[0]) | spread((uint64_t)q[1]) << 1 | spread((uint64_t)q[2]) << 2;
        };
        // TGV_BRICK_ORDER: 0 storage order, 1 Morton (measured 3-4 % slower on C5), 2 (z, 8 x 8 tiles
        // of (x, y), y, x): a CTA wave covers a compact x-y tile, so y-halo rows are read
        // while the neighbour brick's own CTAs have them in L2
        const int64_t order = env_int("TGV_BRICK_ORDER", 0);
        if (order == 1)
            std::stable_sort(alist.begin(), alist.end(), [&](int a1, int a2) { return mort(a1) < mort(a2); });
        if (order == 2) {
            auto key = [&](int b) {
                const int32_t* q = S->coords + 3 * (int64_t)b;
                return (uint64_t)q[2] << 44 | (uint64_t)(q[1] >> 3) << 32 | (uint64_t)(q[0] >> 3) << 20 |
                       (uint64_t)(q[1] & 7) << 10 | (uint64_t)(q[0] & 7);
            };
            std::stable_sort(alist.begin(), alist.end(), [&](int a1, int a2) { return key(a1) < key(a2); });
        }
    }
    c->n_alist = (int)alist.size();
    c->n_faces = (int)faces.size() / 2;
    if (cudaMalloc(&c->d_alist, sizeof(int) * std::max<size_t>(1, alist.size())) != cudaSuccess ||
        cudaMalloc(&c->d_faces, sizeof(int) * std::max<size_t>(1, faces.size())) != cudaSuccess ||
        (!alist.empty() && cudaMemcpy(c->d_alist, alist.data(), sizeof(int) * alist.size(), cudaMemcpyHostToDevice) != cudaSuccess) ||
        (!faces.empty() && cudaMemcpy(c->d_faces, faces.data(), sizeof(int) * faces.size(), cudaMemcpyHostToDevice) != cudaSuccess)) {
        cudaGetLastError();
        bfail(c, TGV_ENOMEM, "brick list allocation failed");
        return bail(TGV_ENOMEM);
    }
    if (c->E == 32 && !levels) {  // the fused schedule's neighbourhood table (and its default)
        std::vector<int> nb27((size_t)alist.size() * 27, -1);
        std::unordered_map<uint64_t, int> at2;
        at2.reserve((size_t)nb * 2);
        auto key2 = [](int64_t x, int64_t y, int64_t z) { return (uint64_t)x | (uint64_t)y << 21 | (uint64_t)z << 42; };
        for (int64_t b = 0; b < nb; ++b) at2.emplace(key2(S->coords[3 * b], S->coords[3 * b + 1], S->coords[3 * b + 2]), (int)b);
        for (size_t jj = 0; jj < alist.size(); ++jj) {
            const int32_t* q = S->coords + 3 * (int64_t)alist[jj];
            for (int dz = -1; dz <= 1; ++dz)
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        const int64_t X = q[0] + dx, Y = q[1] + dy, Z = q[2] + dz;
                        if (X < 0 || Y < 0 || Z < 0) continue;
                        auto it = at2.find(key2(X, Y, Z));
                        if (it != at2.end()) nb27[jj * 27 + (size_t)((dz + 1) * 9 + (dy + 1) * 3 + dx + 1)] = it->second;
                    }
        }
        if (cudaMalloc(&c->d_nb27, sizeof(int) * std::max<size_t>(1, nb27.size())) != cudaSuccess ||
            (!nb27.empty() && cudaMemcpy(c->d_nb27, nb27.data(), sizeof(int) * nb27.size(), cudaMemcpyHostToDevice) != cudaSuccess)) {
            cudaGetLastError();
            bfail(c, TGV_ENOMEM, "neighbourhood table allocation failed");
            return bail(TGV_ENOMEM);
        }
        c->device_bytes += (int64_t)sizeof(int) * nb27.size();
        c->schedule = env_int("TGV_BRICK_SCHEDULE", TGV_SCHEDULE_FUSED) == TGV_SCHEDULE_SPLIT ? TGV_SCHEDULE_SPLIT
                                                                                              : TGV_SCHEDULE_FUSED;
    }
    c->coords_h.assign(S->coords, S->coords + 3 * nb);
    if (cudaMalloc(&c->d_coords, sizeof(int) * 3 * (size_t)nb) != cudaSuccess ||
        cudaMalloc(&c->d_parent, sizeof(int) * (size_t)nb) != cudaSuccess) {
        cudaGetLastError();
        bfail(c, TGV_ENOMEM, "table allocation failed");
        return bail(TGV_ENOMEM);
    }
    c->device_bytes += 16 * nb;
    if (cudaMemcpy(c->d_coords, S->coords, sizeof(int) * 3 * (size_t)nb, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->nbr, nbr.data(), sizeof(int) * nbr.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->frozen, fr.data(), fr.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->aface, af.data(), af.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaGetLastError();
        bfail(c, TGV_ECUDA, "table upload failed");
        return bail(TGV_ECUDA);
    }
    if (levels) {
        int rc = build_mixed_tables(c, S, levels, fr);
        if (rc) return bail(rc);
    }
    *out = c;
    return TGV_OK;
}

// R27 tables of a 2:1 mixed-level set: face kinds, neighbour bricks (four quadrants for
// a finer face), coordinate parities, solved-quadrant masks, the frozen faces of S, |S|
int build_mixed_tables(tgv_bricks* c, const tgv_brickset* S, const uint8_t* levels, const std::vector<uint8_t>& fr)
{
    const int64_t nb = c->nbricks;
    const int E = c->E;
    std::unordered_map<uint64_t, int> at;
    at.reserve((size_t)nb * 2);
    auto key = [](int64_t l, int64_t x, int64_t y, int64_t z) {
        return (uint64_t)x | (uint64_t)y << 20 | (uint64_t)z << 40 | (uint64_t)l << 60;
    };
    auto find = [&](int64_t l, int64_t x, int64_t y, int64_t z) -> int {
        if (l < 0 || l > 7 || x < 0 || y < 0 || z < 0 || x >= (1 << 20) || y >= (1 << 20) || z >= (1 << 20)) return -1;
        auto it = at.find(key(l, x, y, z));
        return it == at.end() ? -1 : it->second;
    };
    for (int64_t b = 0; b < nb; ++b) at.emplace(key(levels[b], S->coords[3 * b], S->coords[3 * b + 1], S->coords[3 * b + 2]), (int)b);
    // disjoint: no brick has an ancestor position occupied by another brick
    for (int64_t b = 0; b < nb; ++b)
        for (int j = 1; levels[b] + j <= 7; ++j)
            if (find(levels[b] + j, S->coords[3 * b] >> j, S->coords[3 * b + 1] >> j, S->coords[3 * b + 2] >> j) >= 0)
                return bfail(c, TGV_EINVAL, "brick %lld overlaps a coarser brick", (long long)b);
    std::vector<uint8_t> kind((size_t)nb * 6, 0), par((size_t)nb, 0), sface((size_t)nb * 6, 0);
    std::vector<int> nbr4((size_t)nb * 24, -1);
    for (int64_t b = 0; b < nb; ++b) {
        const int l = levels[b];
        const int64_t P[3] = {S->coords[3 * b], S->coords[3 * b + 1], S->coords[3 * b + 2]};
        par[(size_t)b] = (uint8_t)((P[0] & 1) | (P[1] & 1) << 1 | (P[2] & 1) << 2);
        for (int k = 0; k < 3; ++k) {
            const int l0 = k == 0 ? 1 : 0, l1 = k == 2 ? 1 : 2;
            for (int d = 0; d < 2; ++d) {
                const int f = 2 * k + d;
                int64_t Q[3] = {P[0], P[1], P[2]};
                Q[k] += d ? 1 : -1;
                if (Q[k] < 0) continue;
                int* nb4 = &nbr4[(size_t)(b * 6 + f) * 4];
                int j = find(l, Q[0], Q[1], Q[2]);
                if (j >= 0) {
                    kind[(size_t)b * 6 + f] = 1;
                    nb4[0] = j;
                    sface[(size_t)b * 6 + f] = fr[(size_t)j] ? 0 : 0xF;
                    continue;
                }
                j = find(l + 1, Q[0] >> 1, Q[1] >> 1, Q[2] >> 1);
                if (j >= 0) {
                    kind[(size_t)b * 6 + f] = 2;
                    nb4[0] = j;
                    sface[(size_t)b * 6 + f] = fr[(size_t)j] ? 0 : 0xF;
                    continue;
                }
                for (int jj = 2; l + jj <= 7; ++jj)
                    if (find(l + jj, Q[0] >> jj, Q[1] >> jj, Q[2] >> jj) >= 0)
                        return bfail(c, TGV_EINVAL, "not 2:1 balanced: brick %lld face %d meets a brick %d levels coarser",
                                     (long long)b, f, jj);
                if (l == 0) continue;
                bool any = false;
                for (int q = 0; q < 4; ++q) {
                    int64_t F[3];
                    F[k] = d ? 2 * Q[k] : 2 * Q[k] + 1;
                    F[l0] = 2 * P[l0] + (q & 1);
                    F[l1] = 2 * P[l1] + (q >> 1);
                    const int fb = find(l - 1, F[0], F[1], F[2]);
                    nb4[q] = fb;
                    if (fb >= 0) {
                        any = true;
                        if (!fr[(size_t)fb]) sface[(size_t)b * 6 + f] |= (uint8_t)(1u << q);
                    }
                    // nothing two levels finer may touch the face
                    if (l >= 2)
                        for (int a2 = 0; a2 < 2; ++a2)
                            for (int b2 = 0; b2 < 2; ++b2) {
                                int64_t G[3];
                                G[k] = d ? 2 * F[k] : 2 * F[k] + 1;
                                G[l0] = 2 * F[l0] + a2;
                                G[l1] = 2 * F[l1] + b2;
                                if (find(l - 2, G[0], G[1], G[2]) >= 0)
                                    return bfail(c, TGV_EINVAL, "not 2:1 balanced at brick %lld face %d", (long long)b, f);
                            }
                }
                if (any) kind[(size_t)b * 6 + f] = 3;
            }
        }
    }
    // the frozen faces of S (quadrant masks) and |S|
    std::vector<int> mf;
    int64_t sv = 0;
    std::vector<uint8_t> mark((size_t)E * E * E);
    for (int64_t b = 0; b < nb; ++b) {
        if (!fr[(size_t)b]) {
            sv += (int64_t)E * E * E;
            continue;
        }
        std::fill(mark.begin(), mark.end(), 0);
        for (int f = 0; f < 6; ++f) {
            const int m = sface[(size_t)b * 6 + f];
            if (!m) continue;
            mf.push_back((int)b);
            mf.push_back(f | m << 3);
            const int k = f >> 1, l0 = k == 0 ? 1 : 0, l1 = k == 2 ? 1 : 2;
            for (int a1 = 0; a1 < E; ++a1)
                for (int a0 = 0; a0 < E; ++a0) {
                    const int q = (a0 >= E / 2 ? 1 : 0) | (a1 >= E / 2 ? 2 : 0);
                    if (!((m >> q) & 1)) continue;
                    int cc[3];
                    cc[k] = (f & 1) ? E - 1 : 0;
                    cc[l0] = a0;
                    cc[l1] = a1;
                    mark[((size_t)cc[2] * E + cc[1]) * E + cc[0]] = 1;
                }
        }
        for (uint8_t m : mark) sv += m;
    }
    c->s_voxels = sv;
    c->n_mfaces = (int)mf.size() / 2;
    std::vector<int> reg, gen;
    for (int64_t b = 0; b < nb; ++b) {
        if (fr[(size_t)b]) continue;
        bool regular = levels[b] == 0;
        for (int f = 0; f < 6; ++f) regular &= kind[(size_t)b * 6 + f] <= 1;
        (regular ? reg : gen).push_back((int)b);
    }
    c->n_alist_reg = (int)reg.size();
    c->n_alist_gen = (int)gen.size();
    if (E == 32) {  // the FUSED schedule's split of the solved bricks (see struct tgv_bricks)
        std::vector<int> fnb, fgen;
        for (int64_t b = 0; b < nb; ++b) {
            if (fr[(size_t)b]) continue;
            bool ok = levels[b] == 0;
            int row[27];
            const int64_t P[3] = {S->coords[3 * b], S->coords[3 * b + 1], S->coords[3 * b + 2]};
            for (int dz = -1; dz <= 1 && ok; ++dz)
                for (int dy = -1; dy <= 1 && ok; ++dy)
                    for (int dx = -1; dx <= 1 && ok; ++dx) {
                        const int64_t X = P[0] + dx, Y = P[1] + dy, Z = P[2] + dz;
                        const int j = find(0, X, Y, Z);
                        row[(dz + 1) * 9 + (dy + 1) * 3 + dx + 1] = j;
                        if (j < 0 && X >= 0 && Y >= 0 && Z >= 0)
                            for (int l = 1; l <= 7 && ok; ++l)
                                if (find(l, X >> l, Y >> l, Z >> l) >= 0) ok = false;  // a coarser brick is there
                    }
            if (ok) fnb.insert(fnb.end(), row, row + 27);
            else fgen.push_back((int)b);
        }
        c->n_fused = (int)fnb.size() / 27;
        c->n_fgen = (int)fgen.size();
        if (cudaMalloc(&c->d_fnb27, sizeof(int) * std::max<size_t>(1, fnb.size())) != cudaSuccess ||
            cudaMalloc(&c->d_alist_fgen, sizeof(int) * std::max<size_t>(1, fgen.size())) != cudaSuccess ||
            (!fnb.empty() && cudaMemcpy(c->d_fnb27, fnb.data(), sizeof(int) * fnb.size(), cudaMemcpyHostToDevice) != cudaSuccess) ||
            (!fgen.empty() && cudaMemcpy(c->d_alist_fgen, fgen.data(), sizeof(int) * fgen.size(), cudaMemcpyHostToDevice) != cudaSuccess)) {
            cudaGetLastError();
            return bfail(c, TGV_ENOMEM, "mixed-level fused tables allocation failed");
        }
        c->device_bytes += (int64_t)sizeof(int) * (fnb.size() + fgen.size());
    }
    if (cudaMalloc(&c->d_alist_reg, sizeof(int) * std::max<size_t>(1, reg.size())) != cudaSuccess ||
        cudaMalloc(&c->d_alist_gen, sizeof(int) * std::max<size_t>(1, gen.size())) != cudaSuccess ||
        (!reg.empty() && cudaMemcpy(c->d_alist_reg, reg.data(), sizeof(int) * reg.size(), cudaMemcpyHostToDevice) != cudaSuccess) ||
        (!gen.empty() && cudaMemcpy(c->d_alist_gen, gen.data(), sizeof(int) * gen.size(), cudaMemcpyHostToDevice) != cudaSuccess)) {
        cudaGetLastError();
        return bfail(c, TGV_ENOMEM, "mixed-level brick lists allocation failed");
    }
    c->mixed = true;
    // SPLIT by default: on C5's mixed finest level it measured 19.6 G solved vox-it/s against
    // FUSED's 19.0 G on the same box (profiles/r2t_*); tgv_bricks_set_schedule(FUSED) for E = 32
    c->schedule = TGV_SCHEDULE_SPLIT;
    c->levels_h.assign(levels, levels + nb);
    if (cudaMalloc(&c->d_level, (size_t)nb) != cudaSuccess || cudaMalloc(&c->d_kind, (size_t)nb * 6) != cudaSuccess ||
        cudaMalloc(&c->d_nbr4, sizeof(int) * (size_t)nb * 24) != cudaSuccess ||
        cudaMalloc(&c->d_par, (size_t)nb) != cudaSuccess || cudaMalloc(&c->d_sface, (size_t)nb * 6) != cudaSuccess ||
        cudaMalloc(&c->d_mfaces, sizeof(int) * std::max<size_t>(2, mf.size())) != cudaSuccess) {
        cudaGetLastError();
        return bfail(c, TGV_ENOMEM, "mixed-level table allocation failed");
    }
    c->device_bytes += 14 * nb + 96 * nb + (int64_t)sizeof(int) * mf.size();
    if (cudaMemcpy(c->d_level, levels, (size_t)nb, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->d_kind, kind.data(), kind.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->d_nbr4, nbr4.data(), sizeof(int) * nbr4.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->d_par, par.data(), par.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->d_sface, sface.data(), sface.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        (!mf.empty() && cudaMemcpy(c->d_mfaces, mf.data(), sizeof(int) * mf.size(), cudaMemcpyHostToDevice) != cudaSuccess)) {
        cudaGetLastError();
        return bfail(c, TGV_ECUDA, "mixed-level table upload failed");
    }
    return TGV_OK;
}
}  // namespace

extern "C" {

int tgv_bricks_create(const tgv_brickset* S, const tgv_params* P, int dev, tgv_bricks** out)
{
    return bricks_create_impl(S, P, dev, out, nullptr);
}

int tgv_bricks_create_mixed(const tgv_brickset* S, const uint8_t* levels, const tgv_params* P, int dev,
                            tgv_bricks** out)
{
    if (!levels) {
        if (out) *out = nullptr;
        return bfail(nullptr, TGV_EINVAL, "levels is NULL");
    }
    return bricks_create_impl(S, P, dev, out, levels);
}

int tgv_bricks_load(tgv_bricks* c, const void* counts, int count_bytes, int64_t n_counts)
{
    int rc = bready(c);
    if (rc) return rc;
    if (!counts) return bfail(c, TGV_EINVAL, "counts is NULL");
    if (count_bytes != 1 && count_bytes != 2 && count_bytes != 4) return bfail(c, TGV_EINVAL, "count_bytes must be 1, 2 or 4");
    if (n_counts != c->nvox * c->nbins)
        return bfail(c, TGV_EINVAL, "n_counts %lld != %lld", (long long)n_counts, (long long)(c->nvox * c->nbins));
    c->loaded = false;
    // u16 store of every count, filled chunk by chunk from a device staging buffer
    const size_t n16 = (size_t)c->nvox * c->slots;
    uint16_t* h16 = (uint16_t*)pool_alloc(c, sizeof(uint16_t) * n16);
    if (!h16) return bfail(c, TGV_ENOMEM, "u16 count staging allocation failed");
    const int64_t chunk = std::max<int64_t>(1, (64ll << 20) / (c->nbins * count_bytes));  // voxels per chunk
    void* stg = pool_alloc(c, (size_t)std::min(chunk, c->nvox) * c->nbins * count_bytes);
    if (!stg) {
        pool_free(c, h16);
        return bfail(c, TGV_ENOMEM, "count staging allocation failed");
    }
    auto done = [&](int code) {  // stream-ordered: after the pack kernels that read them
        pool_free(c, stg);
        pool_free(c, h16);
        return code;
    };
    if (cudaMemsetAsync(c->d_maxc, 0, sizeof(unsigned int), c->stream) != cudaSuccess) return done(bfail(c, TGV_ECUDA, "memset"));
    for (int64_t v0 = 0; v0 < c->nvox; v0 += chunk) {
        const int64_t nv = std::min(chunk, c->nvox - v0);
        const size_t bytes = (size_t)nv * c->nbins * count_bytes;
        if (cudaMemcpyAsync(stg, (const uint8_t*)counts + (size_t)v0 * c->nbins * count_bytes, bytes, cudaMemcpyHostToDevice,
                            c->stream) != cudaSuccess)
            return done(bfail(c, TGV_ECUDA, "count upload failed"));
        uint16_t* dst = h16 + (size_t)v0 * c->slots;
        if (count_bytes == 1) launch_brick_pack<uint8_t>(c, stg, nv, dst);
        else if (count_bytes == 2) launch_brick_pack<uint16_t>(c, stg, nv, dst);
        else launch_brick_pack<uint32_t>(c, stg, nv, dst);
        if (cudaGetLastError() != cudaSuccess) return done(bfail(c, TGV_ECUDA, "pack kernel launch failed"));
    }
    return done(bricks_finish_counts(c, h16));
}

int tgv_bricks_set_primal(tgv_bricks* c, const float* u, const float* v, int64_t n)
{
    int rc = bready(c);
    if (rc) return rc;
    if (!u) return bfail(c, TGV_EINVAL, "u is NULL");
    if (n != c->nvox) return bfail(c, TGV_EINVAL, "n_voxels %lld != %lld", (long long)n, (long long)c->nvox);
    if (!c->loaded) return bfail(c, TGV_ESTATE, "set_primal before load");
    const size_t fb = sizeof(float) * (size_t)c->nvox;
    c->k = 0;
    const Bufs b = bufs(0);
    BCU(cudaMemsetAsync(c->state, 0, sizeof(float) * (size_t)NSLOT * c->nvox, c->stream));
    for (int s : {b.cu, b.pu, b.nu}) {  // all three: the frozen bricks are never written again
        BCU(cudaMemcpyAsync(bslot(c, slotU(s)), u, fb, cudaMemcpyHostToDevice, c->stream));
        if (v)
            for (int d = 0; d < 3; ++d)
                BCU(cudaMemcpyAsync(bslot(c, slotV(s, d)), v + (size_t)d * c->nvox, fb, cudaMemcpyHostToDevice, c->stream));
    }
    BCU(cudaStreamSynchronize(c->stream));
    return TGV_OK;
}

int tgv_bricks_iterate(tgv_bricks* c, int32_t n)
{
    NvtxRange nv("tgv_bricks_iterate");
    int rc = bready(c);
    if (rc) return rc;
    if (n < 0) return bfail(c, TGV_EINVAL, "n must be >= 0");
    if (!c->loaded) return bfail(c, TGV_ESTATE, "iterate before load");
    if ((rc = brick_iterate_enqueue(c, n))) return rc;
    BCU(cudaStreamSynchronize(c->stream));
    return TGV_OK;
}

int tgv_bricks_read(tgv_bricks* c, int f, float* out, int64_t n)
{
    int rc = bready(c);
    if (rc) return rc;
    if (!out) return bfail(c, TGV_EINVAL, "out is NULL");
    if (n != c->nvox) return bfail(c, TGV_EINVAL, "n_voxels %lld != %lld", (long long)n, (long long)c->nvox);
    if (f < 0 || f >= TGV_NUM_FIELDS) return bfail(c, TGV_EINVAL, "bad field id %d", f);
    if (!c->loaded) return bfail(c, TGV_ESTATE, "read before load");
    const Bufs b = bufs(c->k);
    const size_t fb = sizeof(float) * (size_t)c->nvox;
    if (f == TGV_FIELD_UBAR || (f >= TGV_FIELD_VBAR && f < TGV_FIELD_VBAR + 3))
        return bfail(c, TGV_EINVAL, "ubar / vbar are formed inside the kernels, not stored: read u, v");
    int s;
    if (f == TGV_FIELD_U) s = slotU(b.cu);
    else if (f < TGV_FIELD_UBAR) s = slotV(b.cu, f - TGV_FIELD_V);
    else if (f < TGV_FIELD_Q) s = slotP(b.cp, f - TGV_FIELD_P);
    else s = slotQ(b.cp, f - TGV_FIELD_Q);
    BCU(cudaMemcpyAsync(out, bslot(c, s), fb, cudaMemcpyDeviceToHost, c->stream));
    BCU(cudaStreamSynchronize(c->stream));
    return TGV_OK;
}

int tgv_bricks_energy(tgv_bricks* c, double out[6])
{
    NvtxRange nv("tgv_bricks_energy");
    int rc = bready(c);
    if (rc) return rc;
    if (!out) return bfail(c, TGV_EINVAL, "out is NULL");
    if (!c->loaded) return bfail(c, TGV_ESTATE, "energy before load");
    const Bufs b = bufs(c->k);
    EnergyArgs ea{};
    ea.u = bslot(c, slotU(b.cu));
    for (int d = 0; d < 3; ++d) {
        ea.v[d] = bslot(c, slotV(b.cu, d));
        ea.p[d] = bslot(c, slotP(b.cp, d));
    }
    for (int m = 0; m < 6; ++m) ea.q[m] = bslot(c, slotQ(b.cp, m));
    ea.hist = c->hist;
    ea.alpha1 = c->alpha1;
    ea.alpha0 = c->alpha0;
    ea.lambda = c->lambda;
    ea.V = 2.0;
    ea.nbins = c->nbins;
    if ((rc = btimer(c, 2, false))) return rc;
    if (c->mixed) {
        BRICK_LE_DISPATCH(launch_mixed_energy_le, c, ea);
    } else {
        BRICK_LE_DISPATCH(launch_brick_energy_le, c, ea);
    }
    BCU(cudaGetLastError());
    energy_final_kernel<<<1, 256, 0, c->stream>>>(c->partials, c->energy_blocks, c->d_out);
    BCU(cudaGetLastError());
    if ((rc = btimer(c, 2, true))) return rc;
    double h[EN_TERMS];
    BCU(cudaMemcpyAsync(h, c->d_out, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    BCU(cudaStreamSynchronize(c->stream));
    energy_out(h, out);
    return TGV_OK;
}

int tgv_bricks_set_schedule(tgv_bricks* c, int schedule)
{
    int rc = bready(c);
    if (rc) return rc;
    if (schedule != TGV_SCHEDULE_FUSED && schedule != TGV_SCHEDULE_SPLIT) return bfail(c, TGV_EINVAL, "bad schedule %d", schedule);
    if (schedule == TGV_SCHEDULE_FUSED && c->E != 32) return bfail(c, TGV_EINVAL, "the fused schedule needs E = 32");

    c->schedule = schedule;
    return TGV_OK;
}

int tgv_bricks_set_timing(tgv_bricks* c, int enable)
{
    int rc = bready(c);
    if (rc) return rc;
    BCU(cudaStreamSynchronize(c->stream));
    for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
    c->ev.clear();
    c->ev_kind.clear();
    for (int j = 0; j < 4; ++j) {
        c->t_ms[j] = 0.0;
        c->t_n[j] = 0;
    }
    c->timing = enable != 0;
    return TGV_OK;
}

int tgv_bricks_get_timing(tgv_bricks* c, tgv_timing* o)
{
    int rc = bready(c);
    if (rc) return rc;
    if (!o) return bfail(c, TGV_EINVAL, "out is NULL");
    BCU(cudaStreamSynchronize(c->stream));
    if ((rc = btimer_collect(c))) return rc;
    *o = tgv_timing{};
    o->dual_ms = c->t_ms[0];
    o->primal_ms = c->t_ms[1];
    o->energy_ms = c->t_ms[2];
    o->fused_ms = c->t_ms[3];
    o->fused_launches = c->t_n[3];
    o->dual_launches = c->t_n[0];
    o->primal_launches = c->t_n[1];
    o->energy_launches = c->t_n[2];
    return TGV_OK;
}

int tgv_bricks_info(const tgv_bricks* c, tgv_bricks_info_t* o)
{
    if (!c || !o) return TGV_EINVAL;
    *o = tgv_bricks_info_t{};
    o->device_bytes = c->device_bytes;
    o->count_bytes = c->count_bytes;
    o->edge = c->E;
    o->nbricks = c->nbricks;
    o->nfrozen = c->nfrozen;
    o->solved_voxels = (c->nbricks - c->nfrozen) * c->E * c->E * c->E;
    o->s_voxels = c->s_voxels;
    o->schedule = c->schedule;
    return TGV_OK;
}

void tgv_bricks_destroy(tgv_bricks* c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
    pool_free(c, c->state);
    cudaFree(c->nbr);
    cudaFree(c->frozen);
    cudaFree(c->aface);
    cudaFree(c->d_alist);
    cudaFree(c->d_nb27);
    cudaFree(c->d_faces);
    cudaFree(c->d_coords);
    cudaFree(c->d_parent);
    cudaFree(c->d_level);
    cudaFree(c->d_kind);
    cudaFree(c->d_nbr4);
    cudaFree(c->d_par);
    cudaFree(c->d_sface);
    cudaFree(c->d_mfaces);
    cudaFree(c->d_alist_reg);
    cudaFree(c->d_alist_gen);
    cudaFree(c->d_fnb27);
    cudaFree(c->d_alist_fgen);
    pool_free(c, c->hist);
    cudaFree(c->partials);
    cudaFree(c->d_out);
    cudaFree(c->d_maxc);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

int tgv_bricks_reset(tgv_bricks* c)
{
    int rc = bready(c);
    if (rc) return rc;
    if (!c->hist) return bfail(c, TGV_ESTATE, "reset before load");
    return bricks_init_state(c);
}

int tgv_bricks_vote_depth_maps(tgv_bricks* c, const tgv_camera* cams, int ncams, const float* const* depths,
                               const double grid_origin[3], double voxel_size, double voxel_radius)
{
    int rc = bready(c);
    if (rc) return rc;
    if (!cams || !depths || !grid_origin || ncams < 0) return bfail(c, TGV_EINVAL, "NULL argument");
    if (c->nbins != 8) return bfail(c, TGV_EINVAL, "Alg. 1 votes into 8 bins; this context has %d", c->nbins);
    if (!(voxel_size > 0.0) || !(voxel_radius > 0.0)) return bfail(c, TGV_EINVAL, "voxel size and radius must be > 0");
    c->loaded = false;
    float* d_depth = nullptr;
    VoteCam* d_cams = nullptr;
    char msg[512];
    if ((rc = vote_upload(c->stream, cams, ncams, depths, &d_depth, &d_cams, msg))) return bfail(c, rc, "%s", msg);
    uint16_t* h16 = nullptr;
    const size_t n16 = (size_t)c->nvox * c->slots;
    if (cudaMalloc(&h16, sizeof(uint16_t) * n16) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(d_depth);
        cudaFree(d_cams);
        return bfail(c, TGV_ENOMEM, "u16 count staging allocation failed");
    }
    cudaError_t e = cudaMemsetAsync(c->d_maxc, 0, sizeof(unsigned int), c->stream);
    const int nv = (int)c->nvox;
    const double ox = grid_origin[0], oy = grid_origin[1], oz = grid_origin[2];
#define BVOTE(LE_)                                                                                                \
    (c->slots == 8 ? brick_vote_kernel<LE_, 8><<<148 * 8, 256, 0, c->stream>>>(d_cams, ncams, d_depth, c->d_coords, \
                                                                             nv, ox, oy, oz, voxel_size,          \
                                                                             voxel_radius, h16, c->d_maxc,        \
                                                                             c->d_level)                          \
                   : brick_vote_kernel<LE_, 16><<<148 * 8, 256, 0, c->stream>>>(d_cams, ncams, d_depth,            \
                                                                              c->d_coords, nv, ox, oy, oz,         \
                                                                              voxel_size, voxel_radius, h16,       \
                                                                              c->d_maxc, c->d_level))
    if (e == cudaSuccess) {
        switch (c->LE) {
            case 2: BVOTE(2); break;
            case 3: BVOTE(3); break;
            case 4: BVOTE(4); break;
            default: BVOTE(5); break;
        }
#undef BVOTE
        e = cudaGetLastError();
    }
    cudaStreamSynchronize(c->stream);
    cudaFree(d_depth);
    cudaFree(d_cams);
    if (e != cudaSuccess) {
        cudaFree(h16);
        return bfail(c, TGV_ECUDA, "voting: %s", cudaGetErrorString(e));
    }
    rc = bricks_finish_counts(c, h16);
    cudaFree(h16);
    return rc;
}

int tgv_bricks_read_counts(tgv_bricks* c, uint32_t* out, int64_t n)
{
    int rc = bready(c);
    if (rc) return rc;
    if (!out) return bfail(c, TGV_EINVAL, "out is NULL");
    if (!c->hist) return bfail(c, TGV_ESTATE, "no counts loaded");
    if (n != c->nvox * c->nbins)
        return bfail(c, TGV_EINVAL, "n_counts %lld != %lld", (long long)n, (long long)(c->nvox * c->nbins));
    const int64_t chunk = std::max<int64_t>(1, (64ll << 20) / c->nbins);
    uint32_t* d = nullptr;
    if (cudaMalloc(&d, sizeof(uint32_t) * (size_t)std::min(chunk, c->nvox) * c->nbins) != cudaSuccess) {
        cudaGetLastError();
        return bfail(c, TGV_ENOMEM, "read-back staging allocation failed");
    }
    cudaError_t e = cudaSuccess;
    for (int64_t v0 = 0; v0 < c->nvox && e == cudaSuccess; v0 += chunk) {
        const int64_t nv = std::min(chunk, c->nvox - v0);
        if (c->count_bytes == 1)
            brick_unpack_kernel<uint8_t><<<148 * 8, 256, 0, c->stream>>>((const uint8_t*)c->hist + v0 * c->slots, nv,
                                                                         c->slots, c->nbins, d);
        else
            brick_unpack_kernel<uint16_t><<<148 * 8, 256, 0, c->stream>>>((const uint16_t*)c->hist + v0 * c->slots,
                                                                          nv, c->slots, c->nbins, d);
        e = cudaGetLastError();
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(out + v0 * c->nbins, d, sizeof(uint32_t) * nv * c->nbins, cudaMemcpyDeviceToHost,
                                c->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    }
    cudaFree(d);
    if (e != cudaSuccess) return bfail(c, TGV_ECUDA, "count read-back: %s", cudaGetErrorString(e));
    return TGV_OK;
}

int tgv_bricks_refine_flags(tgv_bricks* c, int32_t min_votes, uint8_t* flags, int64_t n)
{
    int rc = bready(c);
    if (rc) return rc;
    if (!flags) return bfail(c, TGV_EINVAL, "flags is NULL");
    if (n != 8 * c->nbricks) return bfail(c, TGV_EINVAL, "n %lld != 8 * nbricks", (long long)n);
    if (min_votes < 1) return bfail(c, TGV_EINVAL, "min_votes must be >= 1");
    if (!c->hist) return bfail(c, TGV_ESTATE, "no counts loaded");
    uint8_t* d = nullptr;
    if (cudaMalloc(&d, (size_t)n) != cudaSuccess) {
        cudaGetLastError();
        return bfail(c, TGV_ENOMEM, "flag allocation failed");
    }
    cudaError_t e = cudaMemsetAsync(d, 0, (size_t)n, c->stream);
    const int nv = (int)c->nvox;
#define BREF(LE_)                                                                                                    \
    (c->count_bytes == 1                                                                                             \
         ? brick_refine_kernel<LE_, uint8_t><<<148 * 8, 256, 0, c->stream>>>((const uint8_t*)c->hist, c->frozen, nv,  \
                                                                             c->slots, c->nbins, min_votes, d)        \
         : brick_refine_kernel<LE_, uint16_t><<<148 * 8, 256, 0, c->stream>>>((const uint16_t*)c->hist, c->frozen,   \
                                                                              nv, c->slots, c->nbins, min_votes, d))
    if (e == cudaSuccess) {
        switch (c->LE) {
            case 2: BREF(2); break;
            case 3: BREF(3); break;
            case 4: BREF(4); break;
            default: BREF(5); break;
        }
#undef BREF
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(flags, d, (size_t)n, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    cudaFree(d);
    if (e != cudaSuccess) return bfail(c, TGV_ECUDA, "refine flags: %s", cudaGetErrorString(e));
    return TGV_OK;
}

int tgv_bricks_prolong_from(tgv_bricks* f, const tgv_bricks* pc)
{
    tgv_bricks* c = f;
    int rc = bready(c);
    if (rc) return rc;
    if (!pc) return bfail(c, TGV_EINVAL, "coarse context is NULL");
    if (pc->device != c->device) return bfail(c, TGV_EINVAL, "coarse context on device %d, fine on %d", pc->device, c->device);
    if (pc->E != c->E) return bfail(c, TGV_EINVAL, "brick edges differ (%d vs %d)", pc->E, c->E);
    if (!c->loaded || !pc->loaded) return bfail(c, TGV_ESTATE, "both levels must be loaded");
    if (pc->poisoned) return bfail(c, TGV_ESTATE, "coarse context poisoned");
    std::unordered_map<uint64_t, int> at;
    at.reserve((size_t)pc->nbricks * 2);
    auto key = [](int64_t x, int64_t y, int64_t z) { return (uint64_t)x | (uint64_t)y << 21 | (uint64_t)z << 42; };
    for (int64_t b = 0; b < pc->nbricks; ++b)
        at.emplace(key(pc->coords_h[3 * b], pc->coords_h[3 * b + 1], pc->coords_h[3 * b + 2]), (int)b);
    if (pc->mixed) return bfail(c, TGV_EINVAL, "the coarse context must be a one-level set");
    std::vector<int> parent((size_t)c->nbricks);
    for (int64_t b = 0; b < c->nbricks; ++b) {
        const int32_t* q = &c->coords_h[3 * b];
        const int lv = c->mixed ? c->levels_h[(size_t)b] : 0;
        if (lv > 1) return bfail(c, TGV_EINVAL, "prolongation into a mixed set needs levels 0 and 1 only");
        auto it = at.find(lv == 1 ? key(q[0], q[1], q[2]) : key(q[0] >> 1, q[1] >> 1, q[2] >> 1));
        if (it == at.end())
            return bfail(c, TGV_EINVAL, "brick (%d, %d, %d) has no parent brick in the coarse level", q[0], q[1], q[2]);
        parent[(size_t)b] = it->second;
    }
    // the coarse level's current iterate (its stream is synchronised first: the two
    // contexts use different streams)
    if (cudaStreamSynchronize(pc->stream) != cudaSuccess) {
        cudaGetLastError();
        return bfail(c, TGV_ECUDA, "coarse stream synchronisation failed");
    }
    const Bufs cb = bufs(pc->k);
    auto cslot = [&](int s) { return (const float*)(pc->state + (int64_t)s * pc->nvox); };
    BCU(cudaMemcpyAsync(c->d_parent, parent.data(), sizeof(int) * parent.size(), cudaMemcpyHostToDevice, c->stream));
    BCU(cudaMemsetAsync(c->state, 0, sizeof(float) * (size_t)NSLOT * c->nvox, c->stream));
    const Bufs b = bufs(0);
    const int nv = (int)c->nvox;
#define BPRO(LE_)                                                                                                   \
    brick_prolong_kernel<LE_><<<148 * 8, 256, 0, c->stream>>>(                                                      \
        cslot(slotU(cb.cu)), cslot(slotV(cb.cu, 0)), cslot(slotV(cb.cu, 1)), cslot(slotV(cb.cu, 2)), c->d_parent,   \
        c->d_coords, nv, bslot(c, slotU(b.cu)), bslot(c, slotU(b.pu)), bslot(c, slotU(b.nu)),                         \
        bslot(c, slotV(b.cu, 0)), bslot(c, slotV(b.cu, 1)), bslot(c, slotV(b.cu, 2)), bslot(c, slotV(b.pu, 0)),       \
        bslot(c, slotV(b.pu, 1)), bslot(c, slotV(b.pu, 2)), bslot(c, slotV(b.nu, 0)), bslot(c, slotV(b.nu, 1)),       \
        bslot(c, slotV(b.nu, 2)), c->d_level)
    switch (c->LE) {
        case 2: BPRO(2); break;
        case 3: BPRO(3); break;
        case 4: BPRO(4); break;
        default: BPRO(5); break;
    }
#undef BPRO
    BCU(cudaGetLastError());
    BCU(cudaStreamSynchronize(c->stream));
    c->k = 0;
    return TGV_OK;
}

}  // extern "C"


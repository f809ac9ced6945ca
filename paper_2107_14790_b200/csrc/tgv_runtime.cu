// tgv_runtime.cu -- context, C ABI (include/tgv.h) and NCCL z-slab halo
// exchange of the B200 TGV solver.
//
// One context per (process, GPU).  The context owns the fp32 state, the
// histogram store, a compute stream, CUDA events for kernel timing and, for
// nranks > 1, an NCCL communicator over NVLink/NVSwitch (NCCL is dlopen'ed).
//
// State representation: iteration k keeps (u_k, u_{k-1}),
// (v_k, v_{k-1}), p_k, q_k.  u and v rotate over 3 buffers, p and q over 2, so a
// single-sweep kernel never overwrites anything another CTA of the same launch
// still reads.  30 field slots of (nzl + 2) planes each (one halo plane below
// and above the slab).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <atomic>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges cost nothing unless a tool (nsys / ncu) attaches

#include "../../include/tgv.h"
#include "nccl_api.h"
#include "tgv_fused_tma.cuh"
#include "tgv_energy_tma.cuh"
#include "tgv_tvl1_tma.cuh"
#include "tgv_kernels.cuh"
#include "tgv_vote.cuh"

using namespace tgvk;

// NVTX range for one ABI call or phase (nsys timeline: iterate / halo / energy / load)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

namespace {

thread_local char g_create_error[512] = "";

constexpr int NSLOT = 30;
constexpr int slotU(int b) { return b; }
constexpr int slotV(int b, int k) { return 3 + 3 * b + k; }
constexpr int slotP(int b, int k) { return 12 + 3 * b + k; }
constexpr int slotQ(int b, int m) { return 18 + 6 * b + m; }  // m: xx yy zz xy xz yz

constexpr int FUSED_TY = 14;  // register fused kernel: 30 x 14 owned voxels, 32 x 16 threads
constexpr int TMA_TY = 14;    // TMA fused kernel: 32 x 14 owned voxels, 32 x 17 threads (box rows 16 -> 128-B fields)

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

enum TimerKind { T_DUAL = 0, T_PRIMAL, T_FUSED, T_ENERGY, T_HALO, T_KINDS };

}  // namespace

struct tgv_ctx {
    tgv_layout L{};
    int nbins = 0;
    float centers[16]{};
    float lambda = 0, alpha0 = 0, alpha1 = 0, tau = 0, sigma = 0;
    int rank = 0, nranks = 1, device = 0;
    int schedule = TGV_SCHEDULE_FUSED;
    int model = TGV_MODEL_TGV;
    bool leaf = false;  // NEXT-3: frozen-border leaf (tgv_create_leaf)
    // peer halo mode: the fused TMA kernel writes the neighbours' halo planes
    bool peer = false;          // neighbours' state and flags are mapped
    bool peer_same_dev = false; // a mapped neighbour runs on this context's GPU
    bool halo_fresh = false;    // our halos hold the current iterate (the neighbours' last launch wrote them)
    float* pdn = nullptr;       // lower / upper neighbour's state (same-process pointer or CUDA IPC mapping)
    float* pup = nullptr;
    int64_t pdn_fs = 0, pup_fs = 0;
    int pdn_top = 0;
    unsigned long long* flags = nullptr;  // [0] CTA counter, [1] written by the lower neighbour, [2] by the upper
    unsigned long long* flag_dn_remote = nullptr;
    unsigned long long* flag_up_remote = nullptr;
    unsigned long long seq = 0, peer_wait = 0;
    bool peer_now = false;      // the next fused launch writes the neighbours' halos
    void* ipc_open[4] = {nullptr, nullptr, nullptr, nullptr};  // IPC mappings to close at destroy
    int fused_zc = 0;       // 0 = automatic
    int num_sms = 148;
    int4* d_sched = nullptr;  // persistent-kernel schedule (fused TMA kernel)
    int* d_sched_off = nullptr;
    int sched_ctas = 0, sched_zc = -1, sched_per_sm = 1;
    int sched_rounds = 0;                 // whole lock-step rounds of the schedule (items / G)
    cudaGraphExec_t gexec = nullptr;      // GRAPH_K iterations, re-captured and updated per tgv_iterate call
    int4* d_esched = nullptr;  // the energy sweep's own copy (its chunk and CTA count never change)
    int* d_esched_off = nullptr;
    int esched_ctas = 0, esched_zc = -1, esched_rounds = 0, esched_per_sm = 0;
    bool fused_tma = true;  // TMA-staged fused kernel (TGV_FUSED_IMPL=regs selects the register one)
    CUtensorMap m_ld1{}, m_ld3{}, m_ld6{}, m_st1{}, m_st3{}, m_st6{}, m_h{};

    Geo g{};
    int slots = 8;            // histogram slots per voxel
    int count_bytes = 2;      // 1 (u8) or 2 (u16), decided per load
    float* state = nullptr;   // NSLOT * g.fs floats
    uint16_t* hist16 = nullptr;
    uint8_t* hist8 = nullptr;
    double* partials = nullptr;
    double* d_out = nullptr;
    unsigned int* d_maxc = nullptr;
    uint32_t* staging = nullptr;
    float* upload = nullptr;  // grow-only device buffer for tgv_prolong_slab's coarse fields
    size_t upload_bytes = 0;
    int64_t staging_elems = 0;
    // pipelined host I/O (tgv_stage_histograms / tgv_load_staged / tgv_read_u_async)
    void* stage = nullptr;          // whole-slab count staging (count_bytes per count)
    size_t stage_bytes = 0;
    int stage_cb = 0;               // count_bytes of the staged counts, 0: nothing staged
    float* usnap = nullptr;         // u snapshot read by the asynchronous D2H
    cudaStream_t s_in = nullptr, s_out = nullptr;
    cudaEvent_t ev_staged = nullptr, ev_stage_free = nullptr, ev_snap = nullptr, ev_read = nullptr;
    int energy_blocks = 0;
    int64_t device_bytes = 0;
    int64_t k = 0;  // iteration counter

    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;
    // in-process slab group (tgv_create_group): members exchange halos by device copies
    std::vector<tgv_ctx*>* group = nullptr;  // shared by the members, owned by the last one destroyed
    cudaEvent_t ev_step = nullptr;           // recorded after each of this member's sweeps
    const NcclApi* nccl = nullptr;  // resolved at create when nranks > 1

    bool loaded = false;
    bool poisoned = false;
    char err[512] = "";

    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<int> ev_kind;  // kind per recorded pair
    size_t ev_used = 0;
    double t_ms[T_KINDS]{};
    int64_t t_n[T_KINDS]{};
};

namespace {

int fail(tgv_ctx* c, int code, const char* fmt, ...)
{
    char* dst = c ? c->err : g_create_error;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(dst, 512, fmt, ap);
    va_end(ap);
    if (c && (code == TGV_ECUDA || code == TGV_ENCCL)) c->poisoned = true;
    return code;
}

#define CU(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return fail(c, TGV_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
    } while (0)
#define NC(call)                                                                                   \
    do {                                                                                           \
        ncclResult_t r_ = (call);                                                                  \
        if (r_ != ncclSuccess)                                                                     \
            return fail(c, TGV_ENCCL, "%s:%d %s: %s", __FILE__, __LINE__, #call, nccl->GetErrorString(r_)); \
    } while (0)

inline float* slot(tgv_ctx* c, int s) { return c->state + (int64_t)s * c->g.fs; }
// pointer to local plane z (z in [-1, nzl]) of slot s
inline float* plane_ptr(tgv_ctx* c, int s, int z) { return slot(c, s) + (int64_t)(z + 1) * c->g.plane; }
inline const void* hist_ptr(const tgv_ctx* c) { return c->count_bytes == 1 ? (const void*)c->hist8 : c->hist16; }

struct Bufs {
    int cu, pu, nu, cp, np;
};
inline Bufs bufs(int64_t k) { return Bufs{(int)(k % 3), (int)((k + 2) % 3), (int)((k + 1) % 3), (int)(k % 2), (int)((k + 1) % 2)}; }

int check_ready(tgv_ctx* c)
{
    if (!c) return TGV_EINVAL;
    if (c->poisoned) return fail(c, TGV_ESTATE, "context poisoned by an earlier CUDA/NCCL failure");
    // every call runs on the context's device, whatever the calling thread's current device
    if (cudaSetDevice(c->device) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, TGV_ECUDA, "cudaSetDevice(%d) failed", c->device);
    }
    return TGV_OK;
}

// ---- timing -----------------------------------------------------------------
int timer_begin(tgv_ctx* c, int kind, size_t* slot_)
{
    if (!c->timing) return TGV_OK;
    if (c->ev_used + 2 > c->ev_pool.size()) {
        size_t grow = std::max<size_t>(64, c->ev_pool.size());
        for (size_t k = 0; k < grow; ++k) {
            cudaEvent_t e;
            CU(cudaEventCreate(&e));
            c->ev_pool.push_back(e);
        }
    }
    *slot_ = c->ev_used;
    c->ev_used += 2;
    c->ev_kind.push_back(kind);
    CU(cudaEventRecord(c->ev_pool[*slot_], c->stream));
    return TGV_OK;
}
int timer_end(tgv_ctx* c, size_t slot_)
{
    if (!c->timing) return TGV_OK;
    CU(cudaEventRecord(c->ev_pool[slot_ + 1], c->stream));
    return TGV_OK;
}
int timer_collect(tgv_ctx* c)
{
    if (!c->timing) return TGV_OK;
    for (size_t k = 0; k < c->ev_kind.size(); ++k) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, c->ev_pool[2 * k], c->ev_pool[2 * k + 1]));
        c->t_ms[c->ev_kind[k]] += ms;
        c->t_n[c->ev_kind[k]] += 1;
    }
    c->ev_kind.clear();
    c->ev_used = 0;
    return TGV_OK;
}

// ---- launches ---------------------------------------------------------------
StepParams step_params(const tgv_ctx* c)
{
    return StepParams{c->sigma, c->tau, c->alpha1, c->alpha0, c->tau * c->lambda};
}
Centers centers(const tgv_ctx* c)
{
    Centers C;
    for (int b = 0; b < 16; ++b) C.c[b] = b < c->nbins ? c->centers[b] : INFINITY;
    return C;
}

// pointers of iteration k: inputs (u_k, u_{k-1}, v_k, v_{k-1}, p_k, q_k), outputs of k+1
IterPtrs iter_ptrs(tgv_ctx* c, int64_t k)
{
    const Bufs b = bufs(k);
    IterPtrs a{};
    a.uk = slot(c, slotU(b.cu));
    a.um = slot(c, slotU(b.pu));
    a.un = slot(c, slotU(b.nu));
    for (int d = 0; d < 3; ++d) {
        a.vk[d] = slot(c, slotV(b.cu, d));
        a.vm[d] = slot(c, slotV(b.pu, d));
        a.vn[d] = slot(c, slotV(b.nu, d));
        a.pk[d] = slot(c, slotP(b.cp, d));
        a.pn[d] = slot(c, slotP(b.np, d));
    }
    for (int m = 0; m < 6; ++m) {
        a.qk[m] = slot(c, slotQ(b.cp, m));
        a.qn[m] = slot(c, slotQ(b.np, m));
    }
    a.hist = hist_ptr(c);
    return a;
}

template <int SLOTS, typename CT>
void launch_split_primal_t(tgv_ctx* c, const IterPtrs& a, dim3 grd, dim3 blk)
{
    split_primal_kernel<SLOTS, CT><<<grd, blk, 0, c->stream>>>(a, c->g, step_params(c), centers(c));
}

int launch_split(tgv_ctx* c, int phase /*0 dual, 1 primal*/)
{
    size_t sl = 0;
    int rc = timer_begin(c, phase == 0 ? T_DUAL : T_PRIMAL, &sl);
    if (rc) return rc;
    dim3 blk(32, 8), grd((c->g.nx + 31) / 32, (c->g.ny + 7) / 8, c->g.nzl);
    IterPtrs a = iter_ptrs(c, c->k);
    if (phase == 0) {
        split_dual_kernel<<<grd, blk, 0, c->stream>>>(a, c->g, step_params(c));
    } else {
        // the primal reads the dual's outputs p_{k+1}, q_{k+1}
        for (int d = 0; d < 3; ++d) a.pk[d] = a.pn[d];
        for (int m = 0; m < 6; ++m) a.qk[m] = a.qn[m];
        if (c->slots == 8 && c->count_bytes == 1) launch_split_primal_t<8, uint8_t>(c, a, grd, blk);
        else if (c->slots == 8) launch_split_primal_t<8, uint16_t>(c, a, grd, blk);
        else if (c->count_bytes == 1) launch_split_primal_t<16, uint8_t>(c, a, grd, blk);
        else launch_split_primal_t<16, uint16_t>(c, a, grd, blk);
    }
    CU(cudaGetLastError());
    return timer_end(c, sl);
}

template <int SLOTS, typename CT>
void launch_tvl1_primal_t(tgv_ctx* c, const IterPtrs& a, dim3 grd, dim3 blk)
{
    tvl1_primal_kernel<SLOTS, CT><<<grd, blk, 0, c->stream>>>(a, c->g, step_params(c), centers(c));
}

// NEXT-4 TV-L1 (two kernels; v and q stay zero)
int launch_tvl1(tgv_ctx* c, int phase)
{
    size_t sl = 0;
    int rc = timer_begin(c, phase == 0 ? T_DUAL : T_PRIMAL, &sl);
    if (rc) return rc;
    dim3 blk(32, 8), grd((c->g.nx + 31) / 32, (c->g.ny + 7) / 8, c->g.nzl);
    IterPtrs a = iter_ptrs(c, c->k);
    if (phase == 0) {
        tvl1_dual_kernel<<<grd, blk, 0, c->stream>>>(a, c->g, step_params(c));
    } else {
        for (int d = 0; d < 3; ++d) a.pk[d] = a.pn[d];
        if (c->slots == 8 && c->count_bytes == 1) launch_tvl1_primal_t<8, uint8_t>(c, a, grd, blk);
        else if (c->slots == 8) launch_tvl1_primal_t<8, uint16_t>(c, a, grd, blk);
        else if (c->count_bytes == 1) launch_tvl1_primal_t<16, uint8_t>(c, a, grd, blk);
        else launch_tvl1_primal_t<16, uint16_t>(c, a, grd, blk);
    }
    CU(cudaGetLastError());
    return timer_end(c, sl);
}

template <int SLOTS, typename CT>
void launch_tvl1_fused_t(tgv_ctx* c, const FusedArgs& A, dim3 grd)
{
    tvl1_fused_kernel<FUSED_TY, SLOTS, CT><<<grd, dim3(32, FUSED_TY + 2), 0, c->stream>>>(A);
}

int build_schedule(tgv_ctx* c, int zc, int per_sm = 1, bool energy = false);
int64_t env_int(const char* name, int64_t dflt);
int fused_zc(const tgv_ctx* c);

template <int SLOTS, typename CT>
int launch_tvl1_tma_t(tgv_ctx* c, const TmaArgs& A, dim3 grd)
{
    constexpr int HB = SLOTS * (int)sizeof(CT);
    const size_t smem = sizeof(TvSmem<TMA_TY, HB>) + 128;
    static std::atomic<uint64_t> attr_set{0};
    const uint64_t bit = 1ull << (c->device & 63);
    if (!(attr_set.load() & bit)) {
        CU(cudaFuncSetAttribute(tvl1_tma_kernel<TMA_TY, SLOTS, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
        attr_set.fetch_or(bit);
    }
    tvl1_tma_kernel<TMA_TY, SLOTS, CT><<<grd, dim3(32, TMA_TY + 3), smem, c->stream>>>(c->m_ld1, c->m_ld3, c->m_st1,
                                                                                        c->m_st3, c->m_h, A);
    return TGV_OK;
}

// NEXT-4 single sweep (44 B per voxel-iteration with u8 counts): the TMA kernel on the
// persistent schedule of the TGV kernel, or (TGV_FUSED_IMPL=regs) the register kernel
int launch_tvl1_fused(tgv_ctx* c)
{
    size_t sl = 0;
    int rc = timer_begin(c, T_FUSED, &sl);
    if (rc) return rc;
    if (c->fused_tma) {
        const Bufs b = bufs(c->k);
        TmaArgs A{};
        A.g = c->g;
        A.sp = step_params(c);
        A.C = centers(c);
        A.z_lo = 0;
        A.z_hi = c->g.nzl;
        // lock-step chunks for 2 CTAs per SM: at least as many (tile, chunk) items as CTAs,
        // so that neighbouring tiles' halo re-reads meet in L2
        {
            const int tiles = ((c->g.nx + 31) / 32) * ((c->g.ny + TMA_TY - 1) / TMA_TY);
            const int nch = std::max((c->g.nzl + 255) / 256, (2 * c->num_sms + tiles - 1) / tiles);
            A.zc = c->fused_zc > 0 ? c->fused_zc : std::max(1, (c->g.nzl + nch - 1) / nch);
        }
        A.s_uk = slotU(b.cu);
        A.s_um = slotU(b.pu);
        A.s_pk = slotP(b.cp, 0);
        A.s_un = slotU(b.nu);
        A.s_pn = slotP(b.np, 0);
        // two CTAs per SM: one TV-L1 plane step is short, so a second CTA hides the waits
        if ((c->sched_zc != A.zc || c->sched_per_sm != 2) && (rc = build_schedule(c, A.zc, 2))) return rc;
        A.sched = c->d_sched;
        A.sched_off = c->d_sched_off;
        if (env_int("TGV_ROUND_SYNC", 1) && c->sched_rounds > 1 && !c->group) {  // as launch_fused_tma
            A.round_ctr = c->flags + 4;
            A.rounds = c->sched_rounds;
        }
        dim3 grd(c->sched_ctas, 1, 1);
        if (c->slots == 8 && c->count_bytes == 1) rc = launch_tvl1_tma_t<8, uint8_t>(c, A, grd);
        else if (c->slots == 8) rc = launch_tvl1_tma_t<8, uint16_t>(c, A, grd);
        else if (c->count_bytes == 1) rc = launch_tvl1_tma_t<16, uint8_t>(c, A, grd);
        else rc = launch_tvl1_tma_t<16, uint16_t>(c, A, grd);
        if (rc) return rc;
        CU(cudaGetLastError());
        return timer_end(c, sl);
    }
    FusedArgs A;
    A.a = iter_ptrs(c, c->k);
    A.g = c->g;
    A.sp = step_params(c);
    A.C = centers(c);
    A.z_lo = 0;
    A.z_hi = c->g.nzl;
    A.keep_halo_dual = 0;
    // z-chunks for about eight CTAs per SM in total (each chunk re-reads about 2 planes)
    const int tiles = ((c->g.nx + 29) / 30) * ((c->g.ny + FUSED_TY - 1) / FUSED_TY);
    const int chunks = std::max(1, std::min(c->g.nzl / 16 + 1, (8 * c->num_sms + tiles - 1) / tiles));
    A.zc = c->fused_zc > 0 ? c->fused_zc : std::max(1, (c->g.nzl + chunks - 1) / chunks);
    dim3 grd((c->g.nx + 29) / 30, (c->g.ny + FUSED_TY - 1) / FUSED_TY, (c->g.nzl + A.zc - 1) / A.zc);
    if (c->slots == 8 && c->count_bytes == 1) launch_tvl1_fused_t<8, uint8_t>(c, A, grd);
    else if (c->slots == 8) launch_tvl1_fused_t<8, uint16_t>(c, A, grd);
    else if (c->count_bytes == 1) launch_tvl1_fused_t<16, uint8_t>(c, A, grd);
    else launch_tvl1_fused_t<16, uint16_t>(c, A, grd);
    CU(cudaGetLastError());
    return timer_end(c, sl);
}

int fused_zc(const tgv_ctx* c)
{
    if (c->fused_zc > 0) return c->fused_zc;
    if (c->fused_tma) {  // lock-step chunk of the persistent schedule
        // <= 256 planes: one chunk.  Deeper slabs: 128-plane chunks (a divisor near 128 if
        // there is one).  The CTAs of a round march the chunk side by side and drift apart
        // as they go; a neighbour's halo rows only hit L2 while the drift stays within the
        // ~10 planes L2 holds, so shorter chunks keep more halo re-reads in L2.  Measured on
        // C4 (1024^3, one B200, profiles/r2b_C4_probes.txt, r2c): zc 256 27.2-29.9 ms per
        // launch, 128 25.8-26.4 ms, 96 27.8, 64 26.1-26.5 (chunk starts cost a plane each).
        if (c->g.nzl <= 256) return c->g.nzl;
        for (int d = 128; d >= 112; --d)
            if (c->g.nzl % d == 0) return d;
        return 128;
    }
    const int tiles = c->fused_tma ? ((c->g.nx + 31) / 32) * ((c->g.ny + TMA_TY - 1) / TMA_TY)
                                   : ((c->g.nx + 29) / 30) * ((c->g.ny + FUSED_TY - 1) / FUSED_TY);
    const int want = 4 * 148;  // about four waves of one CTA per SM
    int chunks = std::max(1, std::min(c->g.nzl, (want + tiles - 1) / tiles));
    return std::max(1, (c->g.nzl + chunks - 1) / chunks);
}

template <int SLOTS, typename CT>
void launch_fused_t(tgv_ctx* c, const FusedArgs& A, dim3 grd)
{
    fused_kernel<FUSED_TY, SLOTS, CT><<<grd, dim3(32, FUSED_TY + 2), 0, c->stream>>>(A);
}

// ---- TMA descriptors ------------------------------------------------------------
EncodeTiledFn encode_fn()
{
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// L2 sector promotion of the TMA loads (TGV_TMA_PROMO: 0 none, 1 64 B, 2 128 B, 3 256 B = default)
CUtensorMapL2promotion tma_promo()
{
    switch (env_int("TGV_TMA_PROMO", 3)) {
        case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
        case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
        case 2: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
        default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    }
}

// state as a 4-D tensor {x: nx, y: ny, plane: nzl+2 (halo'd), slot: NSLOT}; boxes of nf slots
int make_state_map(tgv_ctx* c, CUtensorMap* m, int bw, int bh, int nf)
{
    EncodeTiledFn enc = encode_fn();
    if (!enc) return fail(c, TGV_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const Geo& g = c->g;
    cuuint64_t dims[4] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)(g.nzl + 2), (cuuint64_t)NSLOT};
    cuuint64_t strides[3] = {(cuuint64_t)g.px * 4, (cuuint64_t)g.plane * 4, (cuuint64_t)g.fs * 4};
    cuuint32_t box[4] = {(cuuint32_t)bw, (cuuint32_t)bh, 1, (cuuint32_t)nf};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, c->state, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, tma_promo(),
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(c, TGV_ECUDA, "cuTensorMapEncodeTiled(state, box %dx%dx%d) = %d", bw, bh, nf, (int)r);
    return TGV_OK;
}

// histogram store as 3-D {8 elements per voxel x nx, ny, nzl}, element = bytes-per-voxel / 8
int make_hist_map(tgv_ctx* c)
{
    EncodeTiledFn enc = encode_fn();
    if (!enc) return fail(c, TGV_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const Geo& g = c->g;
    const int e = c->slots * c->count_bytes / 8;
    const CUtensorMapDataType dt = e == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                   : e == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_UINT32;
    cuuint64_t dims[3] = {(cuuint64_t)8 * g.nx, (cuuint64_t)g.ny, (cuuint64_t)g.nzl};
    cuuint64_t strides[2] = {(cuuint64_t)8 * g.px * e, (cuuint64_t)8 * g.plane * e};
    cuuint32_t box[3] = {256, (cuuint32_t)TMA_TY, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&c->m_h, dt, 3, const_cast<void*>(hist_ptr(c)), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, tma_promo(),
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(c, TGV_ECUDA, "cuTensorMapEncodeTiled(hist) = %d", (int)r);
    return TGV_OK;
}

int make_state_maps(tgv_ctx* c)
{
    int rc;
    if ((rc = make_state_map(c, &c->m_ld1, TMA_BW, TMA_TY + 2, 1))) return rc;
    if ((rc = make_state_map(c, &c->m_ld3, TMA_BW, TMA_TY + 2, 3))) return rc;
    if ((rc = make_state_map(c, &c->m_ld6, TMA_BW, TMA_TY + 2, 6))) return rc;
    if ((rc = make_state_map(c, &c->m_st1, 32, TMA_TY, 1))) return rc;
    if ((rc = make_state_map(c, &c->m_st3, 32, TMA_TY, 3))) return rc;
    return make_state_map(c, &c->m_st6, 32, TMA_TY, 6);
}

// Schedule of the persistent fused kernel: items = (z-chunk, tile) in chunk-major
// order; the first floor(items / G) * G items go round-robin to the G CTAs (each
// CTA runs whole chunks, all CTAs in lock-step through z); the planes of the
// remaining items are split evenly over all G CTAs as contiguous segments.
int64_t env_int(const char* name, int64_t dflt);

int build_schedule(tgv_ctx* c, int zc, int per_sm, bool energy)
{
    const int tiles = ((c->g.nx + 31) / 32) * ((c->g.ny + TMA_TY - 1) / TMA_TY);
    const int nzl = c->g.nzl;
    const int nch = (nzl + zc - 1) / zc;
    const int64_t items = (int64_t)tiles * nch;
    const int64_t planes = (int64_t)tiles * nzl;
    // TGV_PERSIST_CTAS (dev knob) caps the persistent grid; TGV_PERSIST_OVERSUB (test hook)
    // multiplies it beyond what can be resident, which only the round sync's give-up path survives
    const int ctas = (int)(std::min<int64_t>((int64_t)c->num_sms * per_sm,
                                             env_int("TGV_PERSIST_CTAS", (int64_t)c->num_sms * per_sm)) *
                           (energy ? 1 : std::max<int64_t>(1, env_int("TGV_PERSIST_OVERSUB", 1))));
    const int G = (int)std::max<int64_t>(1, std::min<int64_t>(ctas, (planes + 7) / 8));
    std::vector<std::vector<int4>> per(G);
    // items in chunk-major order: every tile of chunk 0, then chunk 1, ...  (A band-major
    // order -- G tiles climbing all the chunks before the next band -- measured no different
    // on C4 with the round sync, profiles/r2m_bands_probe.txt.)
    const int64_t whole = items / G * G;
    auto item = [&](int64_t i, int* t, int* z0, int* z1) {
        const int ch = (int)(i / tiles);
        *t = (int)(i % tiles);
        *z0 = ch * zc;
        *z1 = std::min(nzl, *z0 + zc);
    };
    for (int64_t i = 0; i < whole; ++i) {
        int t, z0, z1;
        item(i, &t, &z0, &z1);
        per[i % G].push_back(make_int4(t, z0, z1, 0));
    }
    // the rest: a contiguous walk over their planes, cut into G equal shares
    std::vector<int4> rest;
    int64_t rest_planes = 0;
    for (int64_t i = whole; i < items; ++i) {
        int t, z0, z1;
        item(i, &t, &z0, &z1);
        rest.push_back(make_int4(t, z0, z1, 0));
        rest_planes += z1 - z0;
    }
    int64_t pos = 0;
    size_t ri = 0;
    int zoff = 0;
    for (int b = 0; b < G && ri < rest.size(); ++b) {
        int64_t quota = rest_planes * (b + 1) / G - pos;
        while (quota > 0 && ri < rest.size()) {
            const int4 it = rest[ri];
            const int z0 = it.y + zoff, take = (int)std::min<int64_t>(quota, it.z - z0);
            per[b].push_back(make_int4(it.x, z0, z0 + take, 0));
            quota -= take;
            pos += take;
            zoff += take;
            if (it.y + zoff >= it.z) {
                ++ri;
                zoff = 0;
            }
        }
    }
    std::vector<int4> flat;
    std::vector<int> off(1, 0);
    for (auto& v : per) {
        flat.insert(flat.end(), v.begin(), v.end());
        off.push_back((int)flat.size());
    }
    int4*& d = energy ? c->d_esched : c->d_sched;
    int*& d_off = energy ? c->d_esched_off : c->d_sched_off;
    cudaFree(d);
    cudaFree(d_off);
    d = nullptr;
    d_off = nullptr;
    CU(cudaMalloc(&d, sizeof(int4) * std::max<size_t>(1, flat.size())));
    CU(cudaMalloc(&d_off, sizeof(int) * off.size()));
    CU(cudaMemcpy(d, flat.data(), sizeof(int4) * flat.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_off, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice));
    if (energy) {
        c->esched_ctas = G;
        c->esched_zc = zc;
        c->esched_rounds = (int)(whole / G);
        c->esched_per_sm = per_sm;
    } else {
        c->sched_ctas = G;
        c->sched_zc = zc;
        c->sched_per_sm = per_sm;
        c->sched_rounds = (int)(whole / G);
    }
    return TGV_OK;
}

template <int SLOTS, typename CT, bool PEER>
int launch_fused_tma_tp(tgv_ctx* c, const TmaArgs& A, dim3 grd)
{
    constexpr int HB = SLOTS * (int)sizeof(CT);
    const size_t smem = sizeof(TmaSmem<TMA_TY, HB>) + 128;
    // the attribute is per device: set it once for each device this process launches on
    static std::atomic<uint64_t> attr_set{0};
    const uint64_t bit = 1ull << (c->device & 63);
    if (!(attr_set.load() & bit)) {
        CU(cudaFuncSetAttribute(fused_tma_kernel<TMA_TY, SLOTS, CT, PEER>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_set.fetch_or(bit);
    }
    fused_tma_kernel<TMA_TY, SLOTS, CT, PEER><<<grd, dim3(32, TMA_TY + 3), smem, c->stream>>>(
        c->m_ld1, c->m_ld3, c->m_ld6, c->m_st1, c->m_st3, c->m_st6, c->m_h, A);
    return TGV_OK;
}
template <int SLOTS, typename CT>
int launch_fused_tma_t(tgv_ctx* c, const TmaArgs& A, dim3 grd)
{
    return c->peer_now ? launch_fused_tma_tp<SLOTS, CT, true>(c, A, grd) : launch_fused_tma_tp<SLOTS, CT, false>(c, A, grd);
}

int launch_fused_tma(tgv_ctx* c)
{
    const Bufs b = bufs(c->k);
    TmaArgs A{};
    A.g = c->g;
    A.sp = step_params(c);
    A.C = centers(c);
    A.z_lo = 0;
    A.z_hi = c->g.nzl;
    A.keep_halo_dual = c->leaf ? 1 : 0;
    A.zc = fused_zc(c);
    A.hints = (int)env_int("TGV_L2_HINTS", 0);  // dev knob until measured
    A.s_uk = slotU(b.cu);
    A.s_um = slotU(b.pu);
    A.s_vk = slotV(b.cu, 0);
    A.s_vm = slotV(b.pu, 0);
    A.s_pk = slotP(b.cp, 0);
    A.s_qk = slotQ(b.cp, 0);
    A.s_un = slotU(b.nu);
    A.s_vn = slotV(b.nu, 0);
    A.s_pn = slotP(b.np, 0);
    A.s_qn = slotQ(b.np, 0);
    if (c->peer_now) {  // peer halo mode: write the neighbours' halos, publish / wait for the hand-over flags
        A.pdn = c->pdn;
        A.pdn_fs = c->pdn_fs;
        A.pdn_top = c->pdn_top;
        A.pup = c->pup;
        A.pup_fs = c->pup_fs;
        A.done = c->flags;
        A.flag_dn_remote = c->flag_dn_remote;
        A.flag_up_remote = c->flag_up_remote;
        A.flag_in_dn = c->flags + 1;
        A.flag_in_up = c->flags + 2;
        A.seq = ++c->seq;
        A.wait_seq = c->peer_wait;
    }
    // persistent grid: one CTA per SM (the kernel's shared memory allows one)
    int rc;
    if ((c->sched_zc != A.zc || c->sched_per_sm != 1) && (rc = build_schedule(c, A.zc, 1))) return rc;
    A.sched = c->d_sched;
    A.sched_off = c->d_sched_off;
    // lock-step rounds (flags[4] counts finished rounds): C4 24.2 vs 26.0-26.2 ms per launch
    // without (profiles/r2l_*); TGV_ROUND_SYNC=0 turns it off.  Only for a kernel that has the
    // GPU to itself: the members of an in-process group (and peer-mode ranks whose neighbour
    // shares the GPU) run concurrently, and a round wait needs every CTA of its grid resident.
    if (env_int("TGV_ROUND_SYNC", 1) && c->sched_rounds > 1 && !c->group && !(c->peer_now && c->peer_same_dev)) {
        A.round_ctr = c->flags + 4;
        A.rounds = c->sched_rounds;
    }
    dim3 grd(c->sched_ctas, 1, 1);
    if (c->slots == 8 && c->count_bytes == 1) rc = launch_fused_tma_t<8, uint8_t>(c, A, grd);
    else if (c->slots == 8) rc = launch_fused_tma_t<8, uint16_t>(c, A, grd);
    else if (c->count_bytes == 1) rc = launch_fused_tma_t<16, uint8_t>(c, A, grd);
    else rc = launch_fused_tma_t<16, uint16_t>(c, A, grd);
    if (rc) return rc;
    CU(cudaGetLastError());
    return TGV_OK;
}

int launch_fused(tgv_ctx* c)
{
    size_t sl = 0;
    int rc = timer_begin(c, T_FUSED, &sl);
    if (rc) return rc;
    if (c->fused_tma) {
        if ((rc = launch_fused_tma(c))) return rc;
        return timer_end(c, sl);
    }
    FusedArgs A{};
    A.a = iter_ptrs(c, c->k);
    A.g = c->g;
    A.sp = step_params(c);
    A.C = centers(c);
    A.z_lo = 0;
    A.z_hi = c->g.nzl;
    A.keep_halo_dual = c->leaf ? 1 : 0;
    A.zc = fused_zc(c);
    dim3 grd((c->g.nx + 29) / 30, (c->g.ny + FUSED_TY - 1) / FUSED_TY, (c->g.nzl + A.zc - 1) / A.zc);
    if (c->slots == 8 && c->count_bytes == 1) launch_fused_t<8, uint8_t>(c, A, grd);
    else if (c->slots == 8) launch_fused_t<8, uint16_t>(c, A, grd);
    else if (c->count_bytes == 1) launch_fused_t<16, uint8_t>(c, A, grd);
    else launch_fused_t<16, uint16_t>(c, A, grd);
    CU(cudaGetLastError());
    return timer_end(c, sl);
}

// ---- halo exchange (plans pinned on CPU by tests/test_slab_gloo.py)
// "down": this rank's BOTTOM owned plane -> rank-1's top halo plane;
// "up":   this rank's TOP owned plane    -> rank+1's bottom halo plane.
struct HaloPlan {
    int ndown = 0, nup = 0;
    int down[16], up[16];
    void add_down(int s) { down[ndown++] = s; }
    void add_up(int s) { up[nup++] = s; }
};

int halo_exchange(tgv_ctx* c, const HaloPlan& hp)
{
    if (c->nranks == 1) return TGV_OK;
    NvtxRange nv("tgv halo exchange (NCCL)");
    const NcclApi* nccl = c->nccl;
    size_t sl = 0;
    int rc = timer_begin(c, T_HALO, &sl);
    if (rc) return rc;
    const size_t n = (size_t)c->g.plane;
    const int nzl = c->g.nzl;
    NC(nccl->GroupStart());
    for (int k = 0; k < hp.ndown; ++k) {
        if (c->rank > 0) NC(nccl->Send(plane_ptr(c, hp.down[k], 0), n, ncclFloat, c->rank - 1, c->comm, c->stream));
        if (c->rank < c->nranks - 1)
            NC(nccl->Recv(plane_ptr(c, hp.down[k], nzl), n, ncclFloat, c->rank + 1, c->comm, c->stream));
    }
    for (int k = 0; k < hp.nup; ++k) {
        if (c->rank < c->nranks - 1)
            NC(nccl->Send(plane_ptr(c, hp.up[k], nzl - 1), n, ncclFloat, c->rank + 1, c->comm, c->stream));
        if (c->rank > 0) NC(nccl->Recv(plane_ptr(c, hp.up[k], -1), n, ncclFloat, c->rank - 1, c->comm, c->stream));
    }
    NC(nccl->GroupEnd());
    return timer_end(c, sl);
}

// split schedule, before the dual: grad ubar needs ubar(z+1) -> (u_k, u_{k-1}) down;
// E(vbar) needs vbar(z-1) -> (v_k, v_{k-1}) up
HaloPlan plan_split_a(int64_t k)
{
    const Bufs b = bufs(k);
    HaloPlan h;
    h.add_down(slotU(b.cu));
    h.add_down(slotU(b.pu));
    for (int d = 0; d < 3; ++d) {
        h.add_up(slotV(b.cu, d));
        h.add_up(slotV(b.pu, d));
    }
    return h;
}
// split schedule, before the primal: div2 q needs q_xz, q_yz, q_zz(z+1) down; div p needs p_z(z-1) up
HaloPlan plan_split_b(int64_t k)
{
    const Bufs b = bufs(k);
    HaloPlan h;
    h.add_down(slotQ(b.np, 4));
    h.add_down(slotQ(b.np, 5));
    h.add_down(slotQ(b.np, 2));
    h.add_up(slotP(b.np, 2));
    return h;
}
// fused schedule, once per iteration: the kernel recomputes the dual on the halo
// planes (p at plane -1, q at plane nzl), so it needs the full inputs there:
//   down: u, u_prev, v, v_prev, q (14 planes);  up: u, u_prev, v, v_prev, p (11 planes)
HaloPlan plan_fused(int64_t k)
{
    const Bufs b = bufs(k);
    HaloPlan h;
    for (int s : {slotU(b.cu), slotU(b.pu)}) {
        h.add_down(s);
        h.add_up(s);
    }
    for (int d = 0; d < 3; ++d)
        for (int bb : {b.cu, b.pu}) {
            h.add_down(slotV(bb, d));
            h.add_up(slotV(bb, d));
        }
    for (int m = 0; m < 6; ++m) h.add_down(slotQ(b.cp, m));
    for (int d = 0; d < 3; ++d) h.add_up(slotP(b.cp, d));
    return h;
}
// TV-L1, before the dual: grad ubar needs (u_k, u_{k-1})(z+1); before the primal: p_z(z-1)
HaloPlan plan_tvl1_a(int64_t k)
{
    const Bufs b = bufs(k);
    HaloPlan h;
    h.add_down(slotU(b.cu));
    h.add_down(slotU(b.pu));
    return h;
}
// TV-L1 single sweep, once per iteration: the kernel recomputes p at plane -1 from
// (u_k, u_{k-1}, p_k) there and reads ubar at plane nzl
//   down: u, u_prev (2 planes);  up: u, u_prev, p (5 planes)
HaloPlan plan_tvl1_fused(int64_t k)
{
    const Bufs b = bufs(k);
    HaloPlan h;
    for (int s : {slotU(b.cu), slotU(b.pu)}) {
        h.add_down(s);
        h.add_up(s);
    }
    for (int d = 0; d < 3; ++d) h.add_up(slotP(b.cp, d));
    return h;
}
HaloPlan plan_tvl1_b(int64_t k)
{
    const Bufs b = bufs(k);
    HaloPlan h;
    h.add_up(slotP(b.np, 2));
    return h;
}
// energy: grad u (u(z+1)), div2 q (q_xz, q_yz, q_zz(z+1)) down; E(v) (v(z-1)), div p (p_z(z-1)) up
HaloPlan plan_energy(int64_t k)
{
    const Bufs b = bufs(k);
    HaloPlan h;
    h.add_down(slotU(b.cu));
    h.add_down(slotQ(b.cp, 4));
    h.add_down(slotQ(b.cp, 5));
    h.add_down(slotQ(b.cp, 2));
    for (int d = 0; d < 3; ++d) h.add_up(slotV(b.cu, d));
    h.add_up(slotP(b.cp, 2));
    return h;
}
// TV-L1 energy: grad u (u(z+1)) down, div p (p_z(z-1)) up; v and q stay zero
HaloPlan plan_energy_tvl1(int64_t k)
{
    const Bufs b = bufs(k);
    HaloPlan h;
    h.add_down(slotU(b.cu));
    h.add_up(slotP(b.cp, 2));
    return h;
}
HaloPlan plan_energy_for(const tgv_ctx* c, int64_t k)
{
    return c->model == TGV_MODEL_TVL1 ? plan_energy_tvl1(k) : plan_energy(k);
}

int sync_stream(tgv_ctx* c)
{
    CU(cudaStreamSynchronize(c->stream));
    if (c->comm) {
        const NcclApi* nccl = c->nccl;
        ncclResult_t ar = ncclSuccess;
        NC(nccl->CommGetAsyncError(c->comm, &ar));
        if (ar != ncclSuccess) return fail(c, TGV_ENCCL, "NCCL async error: %s", nccl->GetErrorString(ar));
    }
    return timer_collect(c);
}

template <int SLOTS, typename CT>
void launch_init_t(tgv_ctx* c)
{
    init_state_kernel<SLOTS, CT><<<148 * 8, 256, 0, c->stream>>>(slot(c, slotU(0)), slot(c, slotU(2)), hist_ptr(c),
                                                                 c->g, centers(c));
}

int init_from_hist(tgv_ctx* c)
{
    c->halo_fresh = false;
    CU(cudaMemsetAsync(c->state, 0, sizeof(float) * (size_t)NSLOT * (size_t)c->g.fs, c->stream));
    c->k = 0;  // u_0 in U[0], u_{-1} = u_0 in U[2]
    if (c->slots == 8 && c->count_bytes == 1) launch_init_t<8, uint8_t>(c);
    else if (c->slots == 8) launch_init_t<8, uint16_t>(c);
    else if (c->count_bytes == 1) launch_init_t<16, uint8_t>(c);
    else launch_init_t<16, uint16_t>(c);
    CU(cudaGetLastError());
    return TGV_OK;
}

// fp64 constants of the energy's data / box-dual walk (tgv_kernels.cuh data_box_terms)
EnergyConsts energy_consts(const float* centers, int nbins, int slots)
{
    EnergyConsts K{};
    double prev = -1.0;
    for (int b = 0; b < 16; ++b) {
        K.c[b] = b < nbins ? (double)centers[b] : 1.0;
        K.c1[b] = K.c[b] + 1.0;
        K.dc[b] = K.c[b] - prev;
        prev = K.c[b];
    }
    K.dc[16] = 1.0 - prev;
    K.end = 1.0 - K.c[slots - 1];
    for (int b = 0; b < 16; ++b) {
        K.cf[b] = (float)K.c[b];
        K.c1f[b] = K.cf[b] + 1.f;
        K.dcf[b] = K.cf[b] - (b ? K.cf[b - 1] : -1.f);
    }
    K.endf = 1.f - K.cf[slots - 1];
    return K;
}

// z-marching items of the energy sweep: at least 8 per block (a short last round) and
// chunks of <= 64 planes: the blocks of a round march side by side, and a neighbouring
// row group's halo rows only hit L2 while their drift stays small (C4 with whole
// 1024-plane columns read 24 % more DRAM than the algorithmic bytes, profiles/r2d_*)
EnergySched energy_sched(const Geo& g, int blocks)
{
    EnergySched es{};
    es.ntx = (g.nx + 31) / 32;
    es.nyg = (g.ny + 7) / 8;
    const int64_t cols = (int64_t)es.ntx * es.nyg;
    const int64_t want = std::max<int64_t>((g.nzl + 63) / 64, (8LL * blocks + cols - 1) / cols);
    const int64_t nch = std::max<int64_t>(1, std::min<int64_t>(g.nzl, want));
    es.zc = (int)((g.nzl + nch - 1) / nch);
    es.items = (int)(cols * ((g.nzl + es.zc - 1) / es.zc));
    return es;
}

// chunk of the energy sweep's lock-step schedule: the iteration sweep's rule (fused_zc)
int energy_zc(const Geo& g)
{
    if (g.nzl <= 256) return g.nzl;
    for (int d = 128; d >= 112; --d)
        if (g.nzl % d == 0) return d;
    return 128;
}

// (a4) energy partials; returns the number of partial blocks (energy_final_kernel's input).
// Default (u8 counts, 8 bins): the TMA-staged sweep (tgv_energy_tma.cuh) with two CTAs per SM
// and 3-plane rings on the lock-step round schedule wherever the grid makes a whole round of
// 2 x 148 (tile, chunk) items with chunks of >= 32 planes: C4 13.7 ms = 0.72 of the measured
// copy (register sweep 17.3 ms), C2 with 128-plane chunks 0.248 ms (register sweep 0.287,
// one round-less 256-plane chunk 0.45); elsewhere the register-streaming
// energy_partial_kernel.  TGV_ENERGY_IMPL=regs | tma | tma2 forces one
// (profiles/r2n_energy_zc_tvl1_probes.txt, r2o_probes.txt, r2x_energy_zc_probe.txt).
template <int SLOTS, typename CT, int NS>
int launch_energy_tma(tgv_ctx* c, const EnergyArgs& ea, const EnergyConsts& K, const Bufs& b, int per_sm, int zc,
                      int* nblocks)
{
    constexpr int HB = SLOTS * (int)sizeof(CT);
    zc = (int)std::max<int64_t>(1, env_int("TGV_ENERGY_ZC", zc));  // dev knob
    int rc;
    if ((c->esched_zc != zc || c->esched_per_sm != per_sm) && (rc = build_schedule(c, zc, per_sm, true))) return rc;
    EnTmaArgs A{};
    A.g = c->g;
    A.s_u = slotU(b.cu);
    A.s_v = slotV(b.cu, 0);
    A.s_p = slotP(b.cp, 0);
    A.s_q = slotQ(b.cp, 0);
    A.sched = c->d_esched;
    A.sched_off = c->d_esched_off;
    A.alpha1 = (float)ea.alpha1;
    A.alpha0 = (float)ea.alpha0;
    A.lambda = (float)ea.lambda;
    A.V = (float)ea.V;
    if (env_int("TGV_ROUND_SYNC", 1) && c->esched_rounds > 1 && !c->group) {  // as launch_fused_tma
        A.round_ctr = c->flags + 5;
        A.rounds = c->esched_rounds;
    }
    const size_t smem = sizeof(EnSmem<TMA_TY, HB, NS>) + 128;
    static std::atomic<uint64_t> attr_set{0};
    const uint64_t bit = 1ull << (c->device & 63);
    if (!(attr_set.load() & bit)) {
        CU(cudaFuncSetAttribute(energy_tma_kernel<TMA_TY, SLOTS, CT, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
        attr_set.fetch_or(bit);
    }
    energy_tma_kernel<TMA_TY, SLOTS, CT, NS><<<c->esched_ctas, dim3(32, TMA_TY), smem, c->stream>>>(
        c->m_ld1, c->m_ld3, c->m_ld6, c->m_h, A, K, c->partials);
    *nblocks = c->esched_ctas;
    return TGV_OK;
}

template <int SLOTS, typename CT>
int launch_energy_t(tgv_ctx* c, const EnergyArgs& ea, const Bufs& b, int* nblocks)
{
    constexpr int HB = SLOTS * (int)sizeof(CT);
    const EnergyConsts K = energy_consts(c->centers, c->nbins, SLOTS);
    const char* impl = getenv("TGV_ENERGY_IMPL");  // dev knob (A/B)
    // two CTAs per SM need at least one whole round of 2 x 148 (tile, chunk) items: deep grids
    // take the iteration sweep's chunks, shallower ones chunks cut to make the round (>= 32 planes)
    const int tiles = ((c->g.nx + 31) / 32) * ((c->g.ny + TMA_TY - 1) / TMA_TY);
    int zc2 = energy_zc(c->g);
    if ((int64_t)tiles * ((c->g.nzl + zc2 - 1) / zc2) < 2 * c->num_sms) {
        const int nch = (2 * c->num_sms + tiles - 1) / tiles;
        zc2 = (c->g.nzl + nch - 1) / nch;
    }
    const bool two = HB == 8 && (impl ? !strcmp(impl, "tma2") : zc2 >= 32);
    if (two) return launch_energy_tma<SLOTS, CT, 3>(c, ea, K, b, 2, zc2, nblocks);
    if (impl && !strncmp(impl, "tma", 3))
        return launch_energy_tma<SLOTS, CT, HB <= 16 ? 5 : 4>(c, ea, K, b, 1, energy_zc(c->g), nblocks);
    const EnergySched es = energy_sched(c->g, c->energy_blocks);
    energy_partial_kernel<SLOTS, CT><<<c->energy_blocks, 256, 0, c->stream>>>(ea, c->g, K, es, c->partials);
    *nblocks = c->energy_blocks;
    return TGV_OK;
}

int64_t env_int(const char* name, int64_t dflt)
{
    const char* s = getenv(name);
    return s && *s ? strtoll(s, nullptr, 10) : dflt;
}

}  // namespace

// =============================================================================
namespace {
int finish_counts(tgv_ctx* c);
}

template <typename T>
void launch_coarsen_t(tgv_ctx* c, const void* staging, int nxf, int nyf, int nzf, int factor, int nzc, int z0)
{
    if (c->slots == 8)
        coarsen_counts_kernel<8, T><<<148 * 8, 256, 0, c->stream>>>(static_cast<const T*>(staging), nxf, nyf, nzf,
                                                                     factor, c->nbins, nzc, z0, c->g, c->hist16,
                                                                     c->d_maxc);
    else
        coarsen_counts_kernel<16, T><<<148 * 8, 256, 0, c->stream>>>(static_cast<const T*>(staging), nxf, nyf, nzf,
                                                                      factor, c->nbins, nzc, z0, c->g, c->hist16,
                                                                      c->d_maxc);
}


extern "C" {

const char* tgv_status_string(int s)
{
    switch (s) {
        case TGV_OK: return "TGV_OK";
        case TGV_EINVAL: return "TGV_EINVAL: invalid argument";
        case TGV_ENOMEM: return "TGV_ENOMEM: allocation failed";
        case TGV_ECUDA: return "TGV_ECUDA: CUDA failure";
        case TGV_ENCCL: return "TGV_ENCCL: NCCL failure";
        case TGV_ESTATE: return "TGV_ESTATE: call not valid in this state";
        case TGV_ERANGE: return "TGV_ERANGE: histogram count out of range";
        default: return "unknown status";
    }
}

const char* tgv_last_error(const tgv_ctx* c) { return c ? c->err : g_create_error; }

int tgv_get_unique_id(uint8_t uid[128])
{
    tgv_ctx* c = nullptr;
    if (!uid) return fail(c, TGV_EINVAL, "uid is NULL");
    const NcclApi* nccl = nccl_api(g_create_error, sizeof g_create_error);
    if (!nccl) return TGV_ENCCL;
    ncclUniqueId id;
    NC(nccl->GetUniqueId(&id));
    static_assert(sizeof(id.internal) == 128, "NCCL unique id size");
    memcpy(uid, id.internal, 128);
    return TGV_OK;
}

struct IpcRecord {
    cudaIpcMemHandle_t state, flags;
    int64_t fs, nzl;
    unsigned char uuid[16];  // the exporter's GPU (neighbours sharing a GPU: no lock-step round sync)
};
static_assert(sizeof(IpcRecord) <= 192, "tgv_peer_export record size");

static int peer_export(tgv_ctx* c, IpcRecord* rec)
{
    if (cudaIpcGetMemHandle(&rec->state, c->state) != cudaSuccess ||
        cudaIpcGetMemHandle(&rec->flags, c->flags) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, TGV_ECUDA, "cudaIpcGetMemHandle failed");
    }
    rec->fs = c->g.fs;
    rec->nzl = c->g.nzl;
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, c->device) == cudaSuccess) memcpy(rec->uuid, prop.uuid.bytes, 16);
    cudaGetLastError();
    return TGV_OK;
}

// side 0: the lower neighbour (its top halo receives our plane 0), 1: the upper neighbour
static int peer_import(tgv_ctx* c, int side, const IpcRecord& n)
{
    void *ps = nullptr, *pf = nullptr;
    if (cudaIpcOpenMemHandle(&ps, n.state, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, TGV_ECUDA, "cudaIpcOpenMemHandle(state) failed (no peer access between the GPUs?)");
    }
    c->ipc_open[2 * side] = ps;
    if (cudaIpcOpenMemHandle(&pf, n.flags, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, TGV_ECUDA, "cudaIpcOpenMemHandle(flags) failed");
    }
    c->ipc_open[2 * side + 1] = pf;
    if (side == 0) {
        c->pdn = static_cast<float*>(ps);
        c->pdn_fs = n.fs;
        c->pdn_top = (int)n.nzl + 1;
        c->flag_dn_remote = static_cast<unsigned long long*>(pf) + 2;  // its "from the upper neighbour" flag
    } else {
        c->pup = static_cast<float*>(ps);
        c->pup_fs = n.fs;
        c->flag_up_remote = static_cast<unsigned long long*>(pf) + 1;  // its "from the lower neighbour" flag
    }
    c->peer = true;
    c->halo_fresh = false;
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, c->device) != cudaSuccess || !memcmp(prop.uuid.bytes, n.uuid, 16))
        c->peer_same_dev = true;  // (or unknown: assume shared)
    cudaGetLastError();
    return TGV_OK;
}

static int map_ipc_neighbours(tgv_ctx* c)
{
    const NcclApi* nccl = c->nccl;
    IpcRecord mine{};
    int rc = peer_export(c, &mine);
    if (rc) return rc;
    std::vector<IpcRecord> all((size_t)c->nranks);
    char* d = nullptr;
    if (cudaMalloc(&d, sizeof(IpcRecord) * (size_t)c->nranks) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, TGV_ENOMEM, "IPC record buffer");
    }
    cudaMemcpy(d + sizeof(IpcRecord) * (size_t)c->rank, &mine, sizeof mine, cudaMemcpyHostToDevice);
    ncclResult_t r = nccl->AllGather(d + sizeof(IpcRecord) * (size_t)c->rank, d, sizeof(IpcRecord), ncclChar,
                                     c->comm, c->stream);
    cudaStreamSynchronize(c->stream);
    cudaMemcpy(all.data(), d, sizeof(IpcRecord) * (size_t)c->nranks, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (r != ncclSuccess) return fail(c, TGV_ENCCL, "IPC all-gather: %s", nccl->GetErrorString(r));
    if (c->rank > 0 && (rc = peer_import(c, 0, all[(size_t)c->rank - 1]))) return rc;
    if (c->rank + 1 < c->nranks && (rc = peer_import(c, 1, all[(size_t)c->rank + 1]))) return rc;
    return TGV_OK;
}

static int create_impl(const tgv_layout* L, const tgv_params* P, int rank, int nranks, const uint8_t* uid, int dev,
                       bool grouped, tgv_ctx** out, bool leaf = false)
{
    tgv_ctx* c = nullptr;
    g_create_error[0] = 0;
    if (!out) return fail(c, TGV_EINVAL, "out is NULL");
    *out = nullptr;
    if (!L || !P) return fail(c, TGV_EINVAL, "layout or params is NULL");
    if (L->nx < 1 || L->ny < 1 || L->nz < 1) return fail(c, TGV_EINVAL, "grid extents must be >= 1");
    if (L->z_begin < 0 || L->z_end > L->nz || L->z_begin >= L->z_end)
        return fail(c, TGV_EINVAL, "slab [%lld, %lld) outside [0, %lld) or empty", (long long)L->z_begin,
                    (long long)L->z_end, (long long)L->nz);
    {
        const int64_t px = (L->nx + 31) / 32 * 32;
        if (L->nz > (1 << 30) || px * L->ny * (L->z_end - L->z_begin + 2) >= (int64_t(1) << 31))
            return fail(c, TGV_EINVAL, "slab too large: one field of a slab must hold < 2^31 elements");
    }
    if (L->brick[0] || L->brick[1] || L->brick[2])
        return fail(c, TGV_EINVAL, "brick layouts are not supported (brick must be {0,0,0})");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(c, TGV_EINVAL, "bad rank %d / nranks %d", rank, nranks);
    if (!grouped && (nranks == 1) != (uid == nullptr)) return fail(c, TGV_EINVAL, "uid must be NULL iff nranks == 1");
    if (nranks == 1 && !leaf && (L->z_begin != 0 || L->z_end != L->nz))
        return fail(c, TGV_EINVAL, "single rank must own the whole grid");
    if (P->nbins < 1 || P->nbins > 16) return fail(c, TGV_EINVAL, "nbins must be in [1, 16]");
    if (!P->bin_centers) return fail(c, TGV_EINVAL, "bin_centers is NULL");
    for (int b = 0; b < P->nbins; ++b) {
        const float cb = P->bin_centers[b];
        if (!std::isfinite(cb) || cb < -1.f || cb > 1.f) return fail(c, TGV_EINVAL, "bin centre %d outside [-1,1]", b);
        if (b > 0 && !(cb > P->bin_centers[b - 1])) return fail(c, TGV_EINVAL, "bin centres not strictly increasing");
    }
    const float vals[5] = {P->lambda, P->alpha0, P->alpha1, P->tau, P->sigma};
    for (float v : vals)
        if (!std::isfinite(v) || v < 0.f) return fail(c, TGV_EINVAL, "parameters must be finite and >= 0");
    if (!(P->tau > 0.f) || !(P->sigma > 0.f)) return fail(c, TGV_EINVAL, "tau and sigma must be > 0");
    if ((double)P->tau * (double)P->sigma * 16.0 > 1.0 + 1e-6)
        return fail(c, TGV_EINVAL, "step sizes violate tau*sigma*16 <= 1 (tau=%g sigma=%g)", P->tau, P->sigma);

    c = new (std::nothrow) tgv_ctx();
    if (!c) return fail(nullptr, TGV_ENOMEM, "host allocation failed");
    auto bail = [&](int code) {
        snprintf(g_create_error, sizeof g_create_error, "%s", c->err);
        tgv_destroy(c);
        return code;
    };
    c->L = *L;
    c->nbins = P->nbins;
    for (int b = 0; b < P->nbins; ++b) c->centers[b] = P->bin_centers[b];
    c->lambda = P->lambda;
    c->alpha0 = P->alpha0;
    c->alpha1 = P->alpha1;
    c->tau = P->tau;
    c->sigma = P->sigma;
    c->rank = rank;
    c->nranks = nranks;
    c->device = dev;
    c->slots = P->nbins <= 8 ? 8 : 16;
    c->leaf = leaf;
    c->schedule = (int)env_int("TGV_SCHEDULE", TGV_SCHEDULE_FUSED);
    if (c->schedule != TGV_SCHEDULE_SPLIT || leaf) c->schedule = TGV_SCHEDULE_FUSED;
    c->fused_zc = (int)env_int("TGV_FUSED_ZC", 0);
    {
        const char* impl = getenv("TGV_FUSED_IMPL");
        c->fused_tma = !(impl && strcmp(impl, "regs") == 0);
    }

    Geo& g = c->g;
    g.nx = (int)L->nx;
    g.ny = (int)L->ny;
    g.nzl = (int)(L->z_end - L->z_begin);
    g.nz = (int)L->nz;
    g.z0 = (int)L->z_begin;
    g.px = (int)((L->nx + 31) / 32 * 32);
    g.plane = g.px * g.ny;
    // Fields are (nzl + 2) planes apart plus a 512 KiB pad: without it every field's
    // plane z sits at the same offset modulo a large power of two (4 MiB planes at
    // 1024^2), and the 17 streams of one step collide in the DRAM / L2 address
    // mapping -- measured on a 1024 x 1024 x 512 slab: 37-38.5 G vox-it/s unpadded,
    // 43.0-43.4 G with 256-512 KiB of pad.
    g.fs = (int64_t)(g.nzl + 2) * g.plane + (env_int("TGV_FIELD_PAD", 131072) + 31) / 32 * 32;

    if (cudaSetDevice(dev) != cudaSuccess) {
        fail(c, TGV_ECUDA, "cudaSetDevice(%d) failed", dev);
        return bail(TGV_ECUDA);
    }
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
        fail(c, TGV_ECUDA, "stream creation failed");
        return bail(TGV_ECUDA);
    }
    const size_t state_bytes = sizeof(float) * (size_t)NSLOT * (size_t)g.fs;
    const size_t hist_bytes = sizeof(uint16_t) * (size_t)c->slots * (size_t)g.nzl * (size_t)g.plane;
    c->energy_blocks = 148 * 3;  // energy_partial_kernel: 3 blocks of 256 per SM (<= 85 registers)
    if (cudaMalloc(&c->state, state_bytes) != cudaSuccess || cudaMalloc(&c->hist16, hist_bytes) != cudaSuccess ||
        cudaMalloc(&c->partials, sizeof(double) * EN_TERMS * c->energy_blocks) != cudaSuccess ||
        cudaMalloc(&c->d_out, sizeof(double) * 8) != cudaSuccess ||
        cudaMalloc(&c->d_maxc, sizeof(unsigned int)) != cudaSuccess ||
        cudaMalloc(&c->flags, 256) != cudaSuccess) {
        cudaGetLastError();
        fail(c, TGV_ENOMEM, "device allocation of %.2f GB failed", (state_bytes + hist_bytes) / 1e9);
        return bail(TGV_ENOMEM);
    }
    c->device_bytes = (int64_t)(state_bytes + hist_bytes);
    if (cudaMemsetAsync(c->state, 0, state_bytes, c->stream) != cudaSuccess ||
        cudaMemsetAsync(c->hist16, 0, hist_bytes, c->stream) != cudaSuccess ||
        cudaMemsetAsync(c->flags, 0, 256, c->stream) != cudaSuccess) {
        fail(c, TGV_ECUDA, "memset failed");
        return bail(TGV_ECUDA);
    }

    if (nranks > 1 && !grouped) {
        const NcclApi* nccl = c->nccl = nccl_api(c->err, sizeof c->err);
        if (!nccl) return bail(TGV_ENCCL);
        ncclUniqueId id;
        memcpy(id.internal, uid, 128);
        ncclResult_t r = nccl->CommInitRank(&c->comm, nranks, id, rank);
        if (r != ncclSuccess) {
            c->comm = nullptr;
            fail(c, TGV_ENCCL, "ncclCommInitRank: %s", nccl->GetErrorString(r));
            return bail(TGV_ENCCL);
        }
        // every rank checks that the slabs tile [0, nz) in rank order
        int64_t* d_sl = nullptr;
        std::vector<int64_t> sl(2 * (size_t)nranks);
        if (cudaMalloc(&d_sl, sizeof(int64_t) * 2 * nranks) != cudaSuccess) {
            fail(c, TGV_ENOMEM, "slab check alloc");
            return bail(TGV_ENOMEM);
        }
        int64_t mine[2] = {L->z_begin, L->z_end};
        cudaMemcpy(d_sl + 2 * rank, mine, sizeof mine, cudaMemcpyHostToDevice);
        r = nccl->AllGather(d_sl + 2 * rank, d_sl, 2, ncclInt64, c->comm, c->stream);
        cudaStreamSynchronize(c->stream);
        cudaMemcpy(sl.data(), d_sl, sizeof(int64_t) * 2 * nranks, cudaMemcpyDeviceToHost);
        cudaFree(d_sl);
        if (r != ncclSuccess) {
            fail(c, TGV_ENCCL, "slab allgather: %s", nccl->GetErrorString(r));
            return bail(TGV_ENCCL);
        }
        bool ok = sl[0] == 0 && sl[2 * (nranks - 1) + 1] == L->nz;
        for (int k = 1; k < nranks; ++k) ok = ok && sl[2 * k] == sl[2 * k - 1];
        if (!ok) {
            fail(c, TGV_EINVAL, "slabs do not tile [0, nz) in rank order");
            return bail(TGV_EINVAL);
        }
        // peer halo mode across processes (default; TGV_PEER_HALO=0 keeps the NCCL exchange):
        // map the neighbours' state and flags with CUDA IPC, handles exchanged by an NCCL
        // all-gather.  Every rank must end up in the same mode (a mapped rank waits for its
        // neighbours' flags), so the outcome is agreed by an all-reduce; on any failure all
        // ranks fall back to the NCCL halo exchange.
        if (env_int("TGV_PEER_HALO", 1) != 0) {
            int ok = map_ipc_neighbours(c) == TGV_OK ? 1 : 0;
            int* d_ok = nullptr;
            int all_ok = 0;
            if (cudaMalloc(&d_ok, sizeof(int)) == cudaSuccess) {
                cudaMemcpy(d_ok, &ok, sizeof ok, cudaMemcpyHostToDevice);
                if (nccl->AllReduce(d_ok, d_ok, 1, ncclInt32, ncclMin, c->comm, c->stream) == ncclSuccess &&
                    cudaStreamSynchronize(c->stream) == cudaSuccess)
                    cudaMemcpy(&all_ok, d_ok, sizeof all_ok, cudaMemcpyDeviceToHost);
                cudaFree(d_ok);
            }
            cudaGetLastError();
            if (!all_ok) {  // back to the NCCL exchange on every rank
                for (void*& q : c->ipc_open)
                    if (q) {
                        cudaIpcCloseMemHandle(q);
                        q = nullptr;
                    }
                c->peer = false;
                c->pdn = c->pup = nullptr;
                c->flag_dn_remote = c->flag_up_remote = nullptr;
                c->err[0] = 0;
            }
        }
    }
    if (make_state_maps(c)) return bail(TGV_ECUDA);
    if (cudaEventCreateWithFlags(&c->ev_step, cudaEventDisableTiming) != cudaSuccess) {
        fail(c, TGV_ECUDA, "event creation failed");
        return bail(TGV_ECUDA);
    }
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) {
        fail(c, TGV_ECUDA, "create sync failed");
        return bail(TGV_ECUDA);
    }
    *out = c;
    return TGV_OK;
}

int tgv_create(const tgv_layout* L, const tgv_params* P, int rank, int nranks, const uint8_t* uid, int dev,
               tgv_ctx** out)
{
    return create_impl(L, P, rank, nranks, uid, dev, false, out);
}

// ---- NEXT-3 frozen-border leaves ------------------------------------------------------
int tgv_create_leaf(const tgv_layout* L, const tgv_params* P, int dev, tgv_ctx** out)
{
    return create_impl(L, P, 0, 1, nullptr, dev, false, out, true);
}

int tgv_peer_export(tgv_ctx* c, uint8_t rec[192])
{
    int rc = check_ready(c);
    if (rc) return rc;
    if (!rec) return fail(c, TGV_EINVAL, "rec is NULL");
    IpcRecord r{};
    if ((rc = peer_export(c, &r))) return rc;
    memset(rec, 0, 192);
    memcpy(rec, &r, sizeof r);
    return TGV_OK;
}

int tgv_peer_import(tgv_ctx* c, int side, const uint8_t rec[192])
{
    int rc = check_ready(c);
    if (rc) return rc;
    if (!rec || (side != 0 && side != 1)) return fail(c, TGV_EINVAL, "NULL record or side not 0 / 1");
    if (c->group) return fail(c, TGV_ESTATE, "group members map each other already");
    if ((side == 0 && c->g.z0 == 0) || (side == 1 && c->g.z0 + c->g.nzl == c->g.nz))
        return fail(c, TGV_EINVAL, "no neighbour on that side of the grid");
    if (c->ipc_open[2 * side]) return fail(c, TGV_ESTATE, "that side is mapped already");
    IpcRecord r;
    memcpy(&r, rec, sizeof r);
    return peer_import(c, side, r);
}

int tgv_leaf_rebind(tgv_ctx* c, int64_t z_begin, int64_t z_end)
{
    int rc = check_ready(c);
    if (rc) return rc;
    if (!c->leaf) return fail(c, TGV_ESTATE, "rebind applies to leaf contexts (tgv_create_leaf)");
    if (z_begin < 0 || z_end > c->L.nz || z_end - z_begin != c->g.nzl)
        return fail(c, TGV_EINVAL, "rebind to [%lld, %lld): the slab must lie in [0, %lld) and keep %d planes",
                    (long long)z_begin, (long long)z_end, (long long)c->L.nz, c->g.nzl);
    CU(cudaStreamSynchronize(c->stream));
    c->L.z_begin = z_begin;
    c->L.z_end = z_end;
    c->g.z0 = (int)z_begin;
    c->loaded = false;  // the counts of the old slab are not this slab's
    return TGV_OK;
}

int tgv_set_border(tgv_ctx* c, int side, const float* u, const float* v, const float* p, const float* q)
{
    int rc = check_ready(c);
    if (rc) return rc;
    c->halo_fresh = false;  // the state changes outside an iteration
    if (!c->leaf) return fail(c, TGV_ESTATE, "borders belong to leaf contexts (tgv_create_leaf)");
    if (!c->loaded) return fail(c, TGV_ESTATE, "set borders after load / prolong (they reset the state)");
    if (side != 0 && side != 1) return fail(c, TGV_EINVAL, "side must be 0 (below) or 1 (above)");
    const Geo& g = c->g;
    const int z = side == 0 ? -1 : g.nzl;
    const size_t rowb = sizeof(float) * g.nx, pitchb = sizeof(float) * g.px;
    const int64_t pl = (int64_t)g.nx * g.ny;
    auto put = [&](int sl, const float* src) -> int {
        if (src)
            CU(cudaMemcpy2DAsync(plane_ptr(c, sl, z), pitchb, src, rowb, rowb, g.ny, cudaMemcpyHostToDevice, c->stream));
        else
            CU(cudaMemset2DAsync(plane_ptr(c, sl, z), pitchb, 0, rowb, g.ny, c->stream));
        return TGV_OK;
    };
    // the same frozen values in every rotating buffer: ubar = u, vbar = v on the border
    for (int b = 0; b < 3; ++b) {
        if ((rc = put(slotU(b), u))) return rc;
        for (int k = 0; k < 3; ++k)
            if ((rc = put(slotV(b, k), v ? v + k * pl : nullptr))) return rc;
    }
    for (int b = 0; b < 2; ++b) {
        for (int k = 0; k < 3; ++k)
            if ((rc = put(slotP(b, k), p ? p + k * pl : nullptr))) return rc;
        for (int m = 0; m < 6; ++m)
            if ((rc = put(slotQ(b, m), q ? q + m * pl : nullptr))) return rc;
    }
    CU(cudaStreamSynchronize(c->stream));
    return TGV_OK;
}

int tgv_load_histograms_coarsened(tgv_ctx* c, const void* fine_v, int count_bytes, int64_t n_fine, int64_t nxf,
                                  int64_t nyf, int64_t nzf, int factor)
{
    NvtxRange nv("tgv_load_histograms_coarsened");
    int rc = check_ready(c);
    if (rc) return rc;
    const Geo& g = c->g;
    const char* fine = static_cast<const char*>(fine_v);
    if (!fine || factor < 1 || factor > 64) return fail(c, TGV_EINVAL, "NULL counts or factor outside [1, 64]");
    if (count_bytes != 1 && count_bytes != 2 && count_bytes != 4)
        return fail(c, TGV_EINVAL, "count_bytes must be 1, 2 or 4");
    if ((nxf + factor - 1) / factor != g.nx || (nyf + factor - 1) / factor != g.ny ||
        (nzf + factor - 1) / factor != g.nz)
        return fail(c, TGV_EINVAL, "grid is not the fine grid coarsened by %d", factor);
    const int64_t fz0 = (int64_t)g.z0 * factor, fz1 = std::min<int64_t>(nzf, (int64_t)(g.z0 + g.nzl) * factor);
    const int64_t per_fplane = nxf * nyf * c->nbins;
    if (n_fine != (fz1 - fz0) * per_fplane)
        return fail(c, TGV_EINVAL, "n_fine %lld != fine planes [%lld, %lld) x %lld", (long long)n_fine,
                    (long long)fz0, (long long)fz1, (long long)per_fplane);
    c->loaded = false;
    // chunks of whole coarse planes (factor fine planes each), staging up to ~256 MB
    const int64_t per_cplane = per_fplane * factor;
    const int cpc = (int)std::max<int64_t>(1, std::min<int64_t>(g.nzl, (256ll << 20) / count_bytes / per_cplane));
    const int64_t need = (per_cplane * cpc * count_bytes + 3) / 4;  // staging is counted in uint32
    if (c->staging_elems < need) {
        if (c->staging) cudaFree(c->staging);
        c->staging = nullptr;
        c->staging_elems = 0;
        if (cudaMalloc(&c->staging, sizeof(uint32_t) * (size_t)need) != cudaSuccess) {
            cudaGetLastError();
            return fail(c, TGV_ENOMEM, "staging allocation failed");
        }
        c->staging_elems = need;
    }
    CU(cudaMemsetAsync(c->d_maxc, 0, sizeof(unsigned int), c->stream));
    for (int z0 = 0; z0 < g.nzl; z0 += cpc) {
        const int nzc = std::min(cpc, g.nzl - z0);
        const int64_t f0 = (int64_t)z0 * factor, f1 = std::min<int64_t>(fz1 - fz0, (int64_t)(z0 + nzc) * factor);
        CU(cudaMemcpyAsync(c->staging, fine + f0 * per_fplane * count_bytes,
                           (size_t)count_bytes * (size_t)((f1 - f0) * per_fplane), cudaMemcpyHostToDevice, c->stream));
        if (count_bytes == 1)
            launch_coarsen_t<uint8_t>(c, c->staging, (int)nxf, (int)nyf, (int)(f1 - f0), factor, nzc, z0);
        else if (count_bytes == 2)
            launch_coarsen_t<uint16_t>(c, c->staging, (int)nxf, (int)nyf, (int)(f1 - f0), factor, nzc, z0);
        else
            launch_coarsen_t<uint32_t>(c, c->staging, (int)nxf, (int)nyf, (int)(f1 - f0), factor, nzc, z0);
        CU(cudaGetLastError());
    }
    return finish_counts(c);
}

int tgv_prolong_slab(tgv_ctx* c, const float* u_c, const float* v_c, int64_t cnx, int64_t cny, int64_t cz0,
                     int64_t cnz)
{
    int rc = check_ready(c);
    if (rc) return rc;
    c->halo_fresh = false;  // the state changes outside an iteration
    const Geo& g = c->g;
    if (!u_c || !v_c) return fail(c, TGV_EINVAL, "NULL coarse fields");
    if (cnx != (g.nx + 1) / 2 || cny != (g.ny + 1) / 2) return fail(c, TGV_EINVAL, "coarse slab is not nx/2 x ny/2");
    if (!c->loaded) return fail(c, TGV_ESTATE, "prolong into a context without histograms");
    // planes to fill: own planes, plus the frozen border planes of a leaf that exist in the grid
    const int zlo = (c->leaf && g.z0 > 0) ? -1 : 0;
    const int zhi = (c->leaf && g.z0 + g.nzl < g.nz) ? g.nzl + 1 : g.nzl;
    const int64_t need_lo = (g.z0 + zlo) / 2, need_hi = (g.z0 + zhi - 1) / 2;
    if (cz0 > need_lo || cz0 + cnz <= need_hi)
        return fail(c, TGV_EINVAL, "coarse slab [%lld, %lld) misses parents [%lld, %lld]", (long long)cz0,
                    (long long)(cz0 + cnz), (long long)need_lo, (long long)need_hi);
    CU(cudaMemsetAsync(c->state, 0, sizeof(float) * (size_t)NSLOT * (size_t)g.fs, c->stream));
    c->k = 0;
    const size_t nc = (size_t)(cnx * cny * cnz);
    // a grow-only buffer: after the first leaf of a size no allocation (and no
    // device-wide synchronisation) happens here
    const size_t need = sizeof(float) * 4 * nc + sizeof(float*) * 12;
    if (c->upload_bytes < need) {
        CU(cudaStreamSynchronize(c->stream));
        cudaFree(c->upload);
        c->upload = nullptr;
        c->upload_bytes = 0;
        if (cudaMalloc(&c->upload, need) != cudaSuccess) {
            cudaGetLastError();
            return fail(c, TGV_ENOMEM, "coarse slab upload buffer");
        }
        c->upload_bytes = need;
    }
    float* d = c->upload;
    float** d_ptrs = reinterpret_cast<float**>(d + 4 * nc);  // byte offset 16 nc: pointer-aligned
    // leaves: the border planes are frozen in every rotating slot; otherwise u_0 = u_{-1}
    float* ptrs[12];
    const int nus = c->leaf ? 3 : 2;
    for (int k = 0; k < nus; ++k) ptrs[k] = slot(c, slotU(c->leaf ? k : (k == 0 ? 0 : 2)));
    for (int k = 0; k < nus; ++k)
        for (int dd = 0; dd < 3; ++dd) ptrs[3 + 3 * k + dd] = slot(c, slotV(c->leaf ? k : (k == 0 ? 0 : 2), dd));
    cudaError_t e = cudaMemcpyAsync(d, u_c, sizeof(float) * nc, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(d + nc, v_c, sizeof(float) * 3 * nc, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_ptrs, ptrs, sizeof(float*) * 12, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) {
        prolong_slab_kernel<<<148 * 8, 256, 0, c->stream>>>(d, d + nc, (int)cnx, (int)cny, (int)cnz, (int)cz0, zlo,
                                                             zhi, g, d_ptrs, nus, d_ptrs + 3, nus);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return fail(c, TGV_ECUDA, "prolong slab: %s", cudaGetErrorString(e));
    return TGV_OK;
}

int tgv_set_model(tgv_ctx* c, int model)
{
    int rc = check_ready(c);
    if (rc) return rc;
    if (model != TGV_MODEL_TGV && model != TGV_MODEL_TVL1) return fail(c, TGV_EINVAL, "unknown model %d", model);
    if (c->leaf && model != TGV_MODEL_TGV) return fail(c, TGV_EINVAL, "leaves run the TGV model only");
    c->model = model;
    if (c->loaded) {  // restart from the initialisation (v = q = 0 for both models)
        if ((rc = init_from_hist(c))) return rc;
        CU(cudaStreamSynchronize(c->stream));
    }
    return TGV_OK;
}

int tgv_set_schedule(tgv_ctx* c, int schedule)
{
    int rc = check_ready(c);
    if (rc) return rc;
    if (schedule != TGV_SCHEDULE_FUSED && schedule != TGV_SCHEDULE_SPLIT)
        return fail(c, TGV_EINVAL, "unknown schedule %d", schedule);
    if (c->leaf && schedule != TGV_SCHEDULE_FUSED)
        return fail(c, TGV_EINVAL, "leaves run the fused schedule only (it updates the border duals)");
    c->schedule = schedule;  // the state representation is shared: switching keeps the iterate
    return TGV_OK;
}

}  // extern "C"

namespace {
// after the u16 store (hist16) and the running max (d_maxc) are written: range check,
// u8 compaction when every count fits, TMA map of the chosen store, state init
int finish_counts(tgv_ctx* c)
{
    const Geo& g = c->g;
    int rc;
    unsigned int maxc = 0;
    CU(cudaMemcpyAsync(&maxc, c->d_maxc, sizeof maxc, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    if (maxc > 65535u) return fail(c, TGV_ERANGE, "histogram count %u exceeds 65535", maxc);
    const bool want8 = maxc <= 255u && env_int("TGV_FORCE_U16", 0) == 0;
    if (want8) {
        const int64_t n = (int64_t)c->slots * g.nzl * g.plane;
        if (!c->hist8) {
            if (cudaMalloc(&c->hist8, (size_t)n) != cudaSuccess) {
                cudaGetLastError();
                return fail(c, TGV_ENOMEM, "u8 histogram allocation failed");
            }
            c->device_bytes += n;
        }
        compact_counts_kernel<<<148 * 8, 256, 0, c->stream>>>(c->hist16, c->hist8, n);
        CU(cudaGetLastError());
    }
    c->count_bytes = want8 ? 1 : 2;
    if ((rc = make_hist_map(c))) return rc;
    rc = init_from_hist(c);
    if (rc) return rc;
    CU(cudaStreamSynchronize(c->stream));
    c->loaded = true;
    return TGV_OK;
}

}  // namespace

extern "C" {

int tgv_load_histograms(tgv_ctx* c, const uint32_t* counts, int64_t n_counts)
{
    NvtxRange nv("tgv_load_histograms");
    int rc = check_ready(c);
    if (rc) return rc;
    const Geo& g = c->g;
    const int64_t per_plane = (int64_t)g.nx * g.ny * c->nbins;
    if (!counts) return fail(c, TGV_EINVAL, "counts is NULL");
    if (n_counts != per_plane * g.nzl)
        return fail(c, TGV_EINVAL, "n_counts %lld != %lld", (long long)n_counts, (long long)(per_plane * g.nzl));
    c->loaded = false;
    // staging buffer of whole planes, up to ~256 MB
    const int planes_per_chunk = (int)std::max<int64_t>(1, std::min<int64_t>(g.nzl, (64ll << 20) / per_plane));
    const int64_t need = per_plane * planes_per_chunk;
    if (c->staging_elems < need) {
        if (c->staging) cudaFree(c->staging);
        c->staging = nullptr;
        c->staging_elems = 0;
        if (cudaMalloc(&c->staging, sizeof(uint32_t) * (size_t)need) != cudaSuccess) {
            cudaGetLastError();
            return fail(c, TGV_ENOMEM, "staging allocation failed");
        }
        c->staging_elems = need;
    }
    CU(cudaMemsetAsync(c->d_maxc, 0, sizeof(unsigned int), c->stream));
    for (int z0 = 0; z0 < g.nzl; z0 += planes_per_chunk) {
        const int nzc = std::min(planes_per_chunk, g.nzl - z0);
        CU(cudaMemcpyAsync(c->staging, counts + (int64_t)z0 * per_plane, sizeof(uint32_t) * per_plane * nzc,
                           cudaMemcpyHostToDevice, c->stream));
        const int blocks = 148 * 8;
        if (c->slots == 8)
            pack_counts_kernel<8><<<blocks, 256, 0, c->stream>>>(c->staging, nzc, z0, g, c->nbins, c->hist16,
                                                                  c->d_maxc);
        else
            pack_counts_kernel<16><<<blocks, 256, 0, c->stream>>>(c->staging, nzc, z0, g, c->nbins, c->hist16,
                                                                   c->d_maxc);
        CU(cudaGetLastError());
    }
    return finish_counts(c);
}

// ---- NEXT-1 coarse-to-fine -------------------------------------------------------
static bool coarse_of(const tgv_ctx* coarse, const tgv_ctx* fine)
{
    return coarse->g.nx == (fine->g.nx + 1) / 2 && coarse->g.ny == (fine->g.ny + 1) / 2 &&
           coarse->g.nz == (fine->g.nz + 1) / 2 && coarse->nranks == 1 && fine->nranks == 1 &&
           coarse->nbins == fine->nbins && coarse->device == fine->device && !coarse->leaf && !fine->leaf;
}

int tgv_restrict_from(tgv_ctx* c, const tgv_ctx* fine)
{
    int rc = check_ready(c);
    if (rc) return rc;
    if (!fine || !fine->loaded) return fail(c, TGV_ESTATE, "fine context missing or not loaded");
    if (!coarse_of(c, fine))
        return fail(c, TGV_EINVAL, "not a 2x coarsening of the fine grid (single-rank contexts on one device)");
    c->loaded = false;
    CU(cudaStreamSynchronize(fine->stream));
    CU(cudaMemsetAsync(c->d_maxc, 0, sizeof(unsigned int), c->stream));
    if (c->slots == 8)
        restrict_counts_kernel<8><<<148 * 8, 256, 0, c->stream>>>(fine->hist16, fine->g, c->hist16, c->g, c->d_maxc);
    else
        restrict_counts_kernel<16><<<148 * 8, 256, 0, c->stream>>>(fine->hist16, fine->g, c->hist16, c->g,
                                                                    c->d_maxc);
    CU(cudaGetLastError());
    return finish_counts(c);
}

int tgv_prolong_from(tgv_ctx* c, const tgv_ctx* coarse)
{
    int rc = check_ready(c);
    if (rc) return rc;
    c->halo_fresh = false;  // the state changes outside an iteration
    if (!coarse || !coarse->loaded) return fail(c, TGV_ESTATE, "coarse context missing or not loaded");
    if (!c->loaded) return fail(c, TGV_ESTATE, "prolong into a context without histograms");
    if (!coarse_of(coarse, c))
        return fail(c, TGV_EINVAL, "not a 2x coarsening of this grid (single-rank contexts on one device)");
    CU(cudaStreamSynchronize(coarse->stream));
    CU(cudaMemsetAsync(c->state, 0, sizeof(float) * (size_t)NSLOT * (size_t)c->g.fs, c->stream));
    c->k = 0;  // current buffers 0, previous buffers 2
    tgv_ctx* cc = const_cast<tgv_ctx*>(coarse);
    const Bufs b = bufs(cc->k);
    prolong_kernel<<<148 * 8, 256, 0, c->stream>>>(
        slot(cc, slotU(b.cu)), slot(cc, slotV(b.cu, 0)), slot(cc, slotV(b.cu, 1)), slot(cc, slotV(b.cu, 2)), cc->g,
        slot(c, slotU(0)), slot(c, slotU(2)), slot(c, slotV(0, 0)), slot(c, slotV(0, 1)), slot(c, slotV(0, 2)),
        slot(c, slotV(2, 0)), slot(c, slotV(2, 1)), slot(c, slotV(2, 2)), c->g);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(c->stream));
    return TGV_OK;
}

// ---- NEXT-2 GPU histogram voting ---------------------------------------------------
}  // extern "C"

namespace {
// Alg. 1 inputs on the device: the cameras (VoteCam) and every depth map's mip
// pyramid (means of the valid children), uploaded / built on stream st.
// Returns TGV_OK, TGV_EINVAL (bad camera), TGV_ENOMEM or TGV_ECUDA with err set;
// on success the caller owns *d_depth and *d_cams (free after the vote kernel).
int vote_upload(cudaStream_t st, const tgv_camera* cams, int ncams, const float* const* depths, float** d_depth_out,
                VoteCam** d_cams_out, char* err)
{
    std::vector<VoteCam> vc((size_t)ncams);
    int64_t total = 0;
    for (int i = 0; i < ncams; ++i) {
        const tgv_camera& C = cams[i];
        if (C.width < 1 || C.height < 1 || C.width > (1 << 22) || C.height > (1 << 22) || !depths[i] ||
            C.vote_weight < 0 || !(C.fx > 0.0) || !(C.fy > 0.0)) {
            snprintf(err, 512, "camera %d: bad size, focal, weight or NULL depth map", i);
            return TGV_EINVAL;
        }
        VoteCam& V = vc[(size_t)i];
        memcpy(V.origin, C.origin, sizeof V.origin);
        memcpy(V.rot, C.rot, sizeof V.rot);
        V.fx = C.fx;
        V.fy = C.fy;
        V.cx = C.cx;
        V.cy = C.cy;
        V.width = C.width;
        V.height = C.height;
        V.vote_weight = C.vote_weight;
        const int mx = std::max(C.width, C.height);
        int nl = 1;
        while ((1 << nl) <= mx) ++nl;  // 1 + floor(log2(max(w, h)))
        V.nlev = nl;
        int w = C.width, h = C.height;
        for (int L = 0; L < nl; ++L) {
            V.lw[L] = w;
            V.lh[L] = h;
            V.lev_off[L] = total;
            total += (int64_t)w * h;
            w = (w + 1) / 2;
            h = (h + 1) / 2;
        }
    }
    float* d_depth = nullptr;
    VoteCam* d_cams = nullptr;
    if (cudaMalloc(&d_depth, sizeof(float) * (size_t)std::max<int64_t>(1, total)) != cudaSuccess ||
        cudaMalloc(&d_cams, sizeof(VoteCam) * (size_t)std::max(1, ncams)) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(d_depth);
        snprintf(err, 512, "depth pyramid allocation of %.2f GB failed", total * 4e-9);
        return TGV_ENOMEM;
    }
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < ncams && e == cudaSuccess; ++i) {
        const VoteCam& V = vc[(size_t)i];
        e = cudaMemcpyAsync(d_depth + V.lev_off[0], depths[i], sizeof(float) * (size_t)V.lw[0] * V.lh[0],
                            cudaMemcpyHostToDevice, st);
        for (int L = 1; L < V.nlev && e == cudaSuccess; ++L) {
            pyramid_level_kernel<<<148 * 4, 256, 0, st>>>(d_depth + V.lev_off[L - 1], V.lw[L - 1], V.lh[L - 1],
                                                           d_depth + V.lev_off[L], V.lw[L], V.lh[L]);
            e = cudaGetLastError();
        }
    }
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(d_cams, vc.data(), sizeof(VoteCam) * (size_t)ncams, cudaMemcpyHostToDevice, st);
    // the host camera table must stay alive until the copy is done
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        cudaStreamSynchronize(st);
        cudaFree(d_depth);
        cudaFree(d_cams);
        snprintf(err, 512, "depth upload / pyramids: %s", cudaGetErrorString(e));
        return TGV_ECUDA;
    }
    *d_depth_out = d_depth;
    *d_cams_out = d_cams;
    return TGV_OK;
}
}  // namespace

extern "C" {

int tgv_vote_depth_maps(tgv_ctx* c, const tgv_camera* cams, int ncams, const float* const* depths,
                        const double grid_origin[3], double voxel_size, double voxel_radius)
{
    int rc = check_ready(c);
    if (rc) return rc;
    if (!cams || !depths || !grid_origin || ncams < 0) return fail(c, TGV_EINVAL, "NULL argument");
    if (c->nbins != 8) return fail(c, TGV_EINVAL, "Alg. 1 votes into 8 bins; this context has %d", c->nbins);
    if (!(voxel_size > 0.0) || !(voxel_radius > 0.0)) return fail(c, TGV_EINVAL, "voxel size and radius must be > 0");
    c->loaded = false;
    float* d_depth = nullptr;
    VoteCam* d_cams = nullptr;
    char msg[512];
    if ((rc = vote_upload(c->stream, cams, ncams, depths, &d_depth, &d_cams, msg))) return fail(c, rc, "%s", msg);
    cudaError_t e = cudaMemsetAsync(c->d_maxc, 0, sizeof(unsigned int), c->stream);
    if (e == cudaSuccess) {
        if (c->slots == 8)
            vote_kernel<8><<<148 * 8, 256, 0, c->stream>>>(d_cams, ncams, d_depth, c->g, grid_origin[0], grid_origin[1],
                                                           grid_origin[2], voxel_size, voxel_radius, c->hist16,
                                                           c->d_maxc);
        else
            vote_kernel<16><<<148 * 8, 256, 0, c->stream>>>(d_cams, ncams, d_depth, c->g, grid_origin[0],
                                                            grid_origin[1], grid_origin[2], voxel_size, voxel_radius,
                                                            c->hist16, c->d_maxc);
        e = cudaGetLastError();
    }
    cudaStreamSynchronize(c->stream);
    cudaFree(d_depth);
    cudaFree(d_cams);
    if (e != cudaSuccess) return fail(c, TGV_ECUDA, "voting: %s", cudaGetErrorString(e));
    return finish_counts(c);
}

int tgv_read_counts(tgv_ctx* c, uint32_t* out, int64_t n)
{
    int rc = check_ready(c);
    if (rc) return rc;
    if (!out) return fail(c, TGV_EINVAL, "out is NULL");
    if (!c->loaded) return fail(c, TGV_ESTATE, "no histograms");
    const int64_t need = (int64_t)c->g.nzl * c->g.ny * c->g.nx * c->nbins;
    if (n != need) return fail(c, TGV_EINVAL, "n_counts %lld != %lld", (long long)n, (long long)need);
    uint32_t* d = nullptr;
    if (cudaMalloc(&d, sizeof(uint32_t) * (size_t)need) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, TGV_ENOMEM, "readback buffer");
    }
    unpack_counts_kernel<<<148 * 8, 256, 0, c->stream>>>(c->hist16, c->g, c->slots, c->nbins, d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(out, d, sizeof(uint32_t) * (size_t)need, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    cudaFree(d);
    if (e != cudaSuccess) return fail(c, TGV_ECUDA, "read counts: %s", cudaGetErrorString(e));
    return TGV_OK;
}

int tgv_reset(tgv_ctx* c)
{
    NvtxRange nv("tgv_reset");
    int rc = check_ready(c);
    if (rc) return rc;
    if (!c->loaded) return fail(c, TGV_ESTATE, "reset before load");
    rc = init_from_hist(c);
    if (rc) return rc;
    CU(cudaStreamSynchronize(c->stream));
    return TGV_OK;
}

static int iterate_enqueue(tgv_ctx* c, int32_t n);

// the fused TMA TGV sweep with mapped neighbours runs in peer halo mode
static bool peer_ready(const tgv_ctx* c)
{
    return c->peer && c->fused_tma && c->model == TGV_MODEL_TGV && c->schedule == TGV_SCHEDULE_FUSED;
}

int tgv_iterate(tgv_ctx* c, int32_t n)
{
    NvtxRange nv("tgv_iterate");
    int rc = iterate_enqueue(c, n);
    if (rc) return rc;
    return sync_stream(c);
}

int tgv_iterate_async(tgv_ctx* c, int32_t n)
{
    int rc = check_ready(c);
    if (rc) return rc;
    if (c->timing) return fail(c, TGV_ESTATE, "per-kernel timing needs the synchronous tgv_iterate");
    if (c->nranks > 1) return fail(c, TGV_ESTATE, "multi-rank contexts iterate with tgv_iterate");
    return iterate_enqueue(c, n);
}

int tgv_sync(tgv_ctx* c)
{
    int rc = check_ready(c);
    if (rc) return rc;
    return sync_stream(c);
}

// One iteration's launches (and, with several ranks, its halo exchanges) on c->stream.
static int iterate_one(tgv_ctx* c)
{
    int rc;
    if (c->model == TGV_MODEL_TVL1 && c->schedule == TGV_SCHEDULE_FUSED) {
        if ((rc = halo_exchange(c, plan_tvl1_fused(c->k)))) return rc;
        if ((rc = launch_tvl1_fused(c))) return rc;
    } else if (c->model == TGV_MODEL_TVL1) {
        if ((rc = halo_exchange(c, plan_tvl1_a(c->k)))) return rc;
        if ((rc = launch_tvl1(c, 0))) return rc;
        if ((rc = halo_exchange(c, plan_tvl1_b(c->k)))) return rc;
        if ((rc = launch_tvl1(c, 1))) return rc;
    } else if (c->schedule == TGV_SCHEDULE_SPLIT) {
        if ((rc = halo_exchange(c, plan_split_a(c->k)))) return rc;
        if ((rc = launch_split(c, 0))) return rc;
        if ((rc = halo_exchange(c, plan_split_b(c->k)))) return rc;
        if ((rc = launch_split(c, 1))) return rc;
    } else if (peer_ready(c)) {  // peer halo mode: the previous launch already wrote our halos
        if (c->halo_fresh) {
            c->peer_wait = c->seq;
        } else {
            if ((rc = halo_exchange(c, plan_fused(c->k)))) return rc;
            c->peer_wait = 0;
        }
        c->peer_now = true;
        rc = launch_fused(c);
        c->peer_now = false;
        if (rc) return rc;
        c->halo_fresh = true;
    } else {
        if ((rc = halo_exchange(c, plan_fused(c->k)))) return rc;
        if ((rc = launch_fused(c))) return rc;
    }
    if (!peer_ready(c)) c->halo_fresh = false;
    c->k += 1;
    return TGV_OK;
}

// CUDA graph of the iteration loop (one GPU, no exchanges, no per-launch timing): the state
// buffers rotate with period GRAPH_K (u / v over 3 slots, p / q over 2), so GRAPH_K
// iterations captured from k = 0 mod GRAPH_K replay for every later block.  Each
// tgv_iterate call re-captures them (whatever changed since -- schedule, model, counts,
// knobs -- is captured as it is now) and updates the executable graph in place; the first
// iterations of the call run directly, so every lazily built resource (persistent
// schedule, kernel attributes) exists before the capture.  TGV_GRAPH=0 turns it off.
constexpr int GRAPH_K = 6;

static bool graph_ok(tgv_ctx* c, int32_t n)
{
    return n >= 3 * GRAPH_K && c->nranks == 1 && !c->timing && !peer_ready(c) && env_int("TGV_GRAPH", 1);
}

// capture GRAPH_K iterations into c->gexec; false (nothing enqueued, k unchanged) on failure
static bool graph_capture(tgv_ctx* c)
{
    const int64_t k0 = c->k;
    const bool poisoned0 = c->poisoned;  // a call the capture rejects is not a device fault
    if (cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    int rc = TGV_OK;
    for (int i = 0; i < GRAPH_K && rc == TGV_OK; ++i) rc = iterate_one(c);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    c->k = k0;
    c->halo_fresh = false;
    bool ok = rc == TGV_OK && e == cudaSuccess && g;
    if (ok && c->gexec) {
        cudaGraphExecUpdateResultInfo info{};
        if (cudaGraphExecUpdate(c->gexec, g, &info) != cudaSuccess) {
            cudaGetLastError();
            cudaGraphExecDestroy(c->gexec);
            c->gexec = nullptr;
        }
    }
    if (ok && !c->gexec && cudaGraphInstantiate(&c->gexec, g, 0) != cudaSuccess) {
        c->gexec = nullptr;
        ok = false;
    }
    if (g) cudaGraphDestroy(g);
    if (!ok) {  // the direct path runs instead (and meets any real fault itself)
        cudaGetLastError();
        c->poisoned = poisoned0;
        c->err[0] = 0;
    }
    return ok;
}

static int iterate_enqueue(tgv_ctx* c, int32_t n)
{
    int rc = check_ready(c);
    if (rc) return rc;
    if (n < 0) return fail(c, TGV_EINVAL, "n < 0");
    if (!c->loaded) return fail(c, TGV_ESTATE, "iterate before load");
    if (c->group) return fail(c, TGV_ESTATE, "grouped context: use tgv_group_iterate");
    int32_t it = 0;
    if (graph_ok(c, n)) {
        // direct until k = 0 mod GRAPH_K, at least one iteration
        do {
            if ((rc = iterate_one(c))) return rc;
            ++it;
        } while (c->k % GRAPH_K);
        if (graph_capture(c)) {
            for (; n - it >= GRAPH_K; it += GRAPH_K) {
                CU(cudaGraphLaunch(c->gexec, c->stream));
                c->k += GRAPH_K;
            }
        }
    }
    for (; it < n; ++it)
        if ((rc = iterate_one(c))) return rc;
    return TGV_OK;
}

// ---- field access -------------------------------------------------------------
static int copy_out(tgv_ctx* c, int s, float* out)
{
    const Geo& g = c->g;
    CU(cudaMemcpy2DAsync(out, sizeof(float) * g.nx, plane_ptr(c, s, 0), sizeof(float) * g.px, sizeof(float) * g.nx,
                         (size_t)g.ny * g.nzl, cudaMemcpyDeviceToHost, c->stream));
    return TGV_OK;
}
static int copy_in(tgv_ctx* c, int s, const float* in)
{
    const Geo& g = c->g;
    CU(cudaMemcpy2DAsync(plane_ptr(c, s, 0), sizeof(float) * g.px, in, sizeof(float) * g.nx, sizeof(float) * g.nx,
                         (size_t)g.ny * g.nzl, cudaMemcpyHostToDevice, c->stream));
    return TGV_OK;
}
// ABI field id -> (current slot, previous slot or -1)
static void field_slots(const tgv_ctx* c, int f, int* cur, int* prev)
{
    const Bufs b = bufs(c->k);
    *prev = -1;
    if (f == TGV_FIELD_U) *cur = slotU(b.cu);
    else if (f >= TGV_FIELD_V && f < TGV_FIELD_V + 3) *cur = slotV(b.cu, f - TGV_FIELD_V);
    else if (f == TGV_FIELD_UBAR) *cur = slotU(b.cu), *prev = slotU(b.pu);
    else if (f >= TGV_FIELD_VBAR && f < TGV_FIELD_VBAR + 3)
        *cur = slotV(b.cu, f - TGV_FIELD_VBAR), *prev = slotV(b.pu, f - TGV_FIELD_VBAR);
    else if (f >= TGV_FIELD_P && f < TGV_FIELD_P + 3) *cur = slotP(b.cp, f - TGV_FIELD_P);
    else *cur = slotQ(b.cp, f - TGV_FIELD_Q);
}

int tgv_read_field(tgv_ctx* c, int f, float* out, int64_t n)
{
    int rc = check_ready(c);
    if (rc) return rc;
    if (!out) return fail(c, TGV_EINVAL, "out is NULL");
    if (f < 0 || f >= TGV_NUM_FIELDS) return fail(c, TGV_EINVAL, "bad field id %d", f);
    if (n != (int64_t)c->g.nx * c->g.ny * c->g.nzl) return fail(c, TGV_EINVAL, "n_voxels mismatch");
    if (!c->loaded) return fail(c, TGV_ESTATE, "read before load");
    int cur, prev;
    field_slots(c, f, &cur, &prev);
    if ((rc = copy_out(c, cur, out))) return rc;
    if (prev >= 0) {  // over-relaxed iterate: 2 x_k - x_{k-1} (exactly the kernels' rounding)
        std::vector<float> pv((size_t)n);
        if ((rc = copy_out(c, prev, pv.data()))) return rc;
        CU(cudaStreamSynchronize(c->stream));
        for (int64_t i = 0; i < n; ++i) out[i] = 2.f * out[i] - pv[(size_t)i];
        return TGV_OK;
    }
    CU(cudaStreamSynchronize(c->stream));
    return TGV_OK;
}

// ---- pipelined host I/O: the next step's counts H2D and this step's u D2H on copy streams,
// overlapped with the iterations (bench.py e2e; include/tgv.h)
static int io_streams(tgv_ctx* c)
{
    if (c->s_in) return TGV_OK;
    CU(cudaStreamCreateWithFlags(&c->s_in, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&c->s_out, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&c->ev_staged, &c->ev_stage_free, &c->ev_snap, &c->ev_read})
        CU(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    CU(cudaEventRecord(c->ev_stage_free, c->stream));
    CU(cudaEventRecord(c->ev_read, c->s_out));
    return TGV_OK;
}

int tgv_stage_histograms(tgv_ctx* c, const void* counts, int count_bytes, int64_t n_counts)
{
    NvtxRange nv("tgv_stage_histograms");
    int rc = check_ready(c);
    if (rc) return rc;
    if (!counts) return fail(c, TGV_EINVAL, "counts is NULL");
    if (count_bytes != 1 && count_bytes != 2 && count_bytes != 4)
        return fail(c, TGV_EINVAL, "count_bytes must be 1, 2 or 4");
    const Geo& g = c->g;
    const int64_t want = (int64_t)g.nzl * g.ny * g.nx * c->nbins;
    if (n_counts != want) return fail(c, TGV_EINVAL, "n_counts %lld != %lld", (long long)n_counts, (long long)want);
    if ((rc = io_streams(c))) return rc;
    const size_t bytes = (size_t)n_counts * count_bytes;
    if (c->stage_bytes < bytes) {
        CU(cudaStreamWaitEvent(c->s_in, c->ev_stage_free, 0));
        CU(cudaStreamSynchronize(c->s_in));
        cudaFree(c->stage);
        c->stage = nullptr;
        c->stage_bytes = 0;
        if (cudaMalloc(&c->stage, bytes) != cudaSuccess) {
            cudaGetLastError();
            return fail(c, TGV_ENOMEM, "count staging allocation of %.2f GB failed", bytes / 1e9);
        }
        c->stage_bytes = bytes;
    }
    // the previous staged counts must have been consumed before they are overwritten
    CU(cudaStreamWaitEvent(c->s_in, c->ev_stage_free, 0));
    CU(cudaMemcpyAsync(c->stage, counts, bytes, cudaMemcpyHostToDevice, c->s_in));
    CU(cudaEventRecord(c->ev_staged, c->s_in));
    c->stage_cb = count_bytes;
    return TGV_OK;
}

int tgv_load_staged(tgv_ctx* c)
{
    NvtxRange nv("tgv_load_staged");
    int rc = check_ready(c);
    if (rc) return rc;
    if (!c->stage_cb) return fail(c, TGV_ESTATE, "nothing staged");
    const Geo& g = c->g;
    c->loaded = false;
    CU(cudaStreamWaitEvent(c->stream, c->ev_staged, 0));
    CU(cudaMemsetAsync(c->d_maxc, 0, sizeof(unsigned int), c->stream));
    const int64_t per_plane = (int64_t)g.nx * g.ny * c->nbins * c->stage_cb;
    const int cpc = (int)std::max<int64_t>(1, std::min<int64_t>(g.nzl, (256ll << 20) / per_plane));
    for (int z0 = 0; z0 < g.nzl; z0 += cpc) {  // the coarsening kernels with factor 1, straight from the staging
        const int nzc = std::min(cpc, g.nzl - z0);
        const void* src = static_cast<const char*>(c->stage) + (size_t)z0 * per_plane;
        if (c->stage_cb == 1) launch_coarsen_t<uint8_t>(c, src, g.nx, g.ny, nzc, 1, nzc, z0);
        else if (c->stage_cb == 2) launch_coarsen_t<uint16_t>(c, src, g.nx, g.ny, nzc, 1, nzc, z0);
        else launch_coarsen_t<uint32_t>(c, src, g.nx, g.ny, nzc, 1, nzc, z0);
        CU(cudaGetLastError());
    }
    CU(cudaEventRecord(c->ev_stage_free, c->stream));
    c->stage_cb = 0;
    return finish_counts(c);
}

int tgv_read_u_async(tgv_ctx* c, float* u, int64_t n)
{
    NvtxRange nv("tgv_read_u_async");
    int rc = check_ready(c);
    if (rc) return rc;
    if (!u) return fail(c, TGV_EINVAL, "u is NULL");
    const Geo& g = c->g;
    if (n != (int64_t)g.nzl * g.ny * g.nx) return fail(c, TGV_EINVAL, "n_voxels mismatch");
    if (!c->loaded) return fail(c, TGV_ESTATE, "read before load");
    if ((rc = io_streams(c))) return rc;
    if (!c->usnap && cudaMalloc(&c->usnap, sizeof(float) * (size_t)g.nzl * g.plane) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, TGV_ENOMEM, "u snapshot allocation failed");
    }
    // the previous read must have left the snapshot before it is overwritten
    CU(cudaStreamWaitEvent(c->stream, c->ev_read, 0));
    CU(cudaMemcpyAsync(c->usnap, plane_ptr(c, slotU(bufs(c->k).cu), 0), sizeof(float) * (size_t)g.nzl * g.plane,
                       cudaMemcpyDeviceToDevice, c->stream));
    CU(cudaEventRecord(c->ev_snap, c->stream));
    CU(cudaStreamWaitEvent(c->s_out, c->ev_snap, 0));
    CU(cudaMemcpy2DAsync(u, sizeof(float) * g.nx, c->usnap, sizeof(float) * g.px, sizeof(float) * g.nx,
                         (size_t)g.ny * g.nzl, cudaMemcpyDeviceToHost, c->s_out));
    CU(cudaEventRecord(c->ev_read, c->s_out));
    return TGV_OK;
}

int tgv_wait_io(tgv_ctx* c)
{
    int rc = check_ready(c);
    if (rc) return rc;
    if (c->s_in) CU(cudaStreamSynchronize(c->s_in));
    if (c->s_out) CU(cudaStreamSynchronize(c->s_out));
    return TGV_OK;
}

int tgv_read_u(tgv_ctx* c, float* u, int64_t n)
{
    NvtxRange nv("tgv_read_u");
    return tgv_read_field(c, TGV_FIELD_U, u, n);
}

int tgv_write_field(tgv_ctx* c, int f, const float* in, int64_t n)
{
    int rc = check_ready(c);
    if (rc) return rc;
    c->halo_fresh = false;  // the state changes outside an iteration
    if (!in) return fail(c, TGV_EINVAL, "in is NULL");
    if (f < 0 || f >= TGV_NUM_FIELDS) return fail(c, TGV_EINVAL, "bad field id %d", f);
    if (n != (int64_t)c->g.nx * c->g.ny * c->g.nzl) return fail(c, TGV_EINVAL, "n_voxels mismatch");
    if (!c->loaded) return fail(c, TGV_ESTATE, "write before load");
    int cur, prev;
    field_slots(c, f, &cur, &prev);
    if (prev < 0) {
        if ((rc = copy_in(c, cur, in))) return rc;
    } else {  // ubar / vbar: set the previous iterate to 2 x_k - in
        std::vector<float> xk((size_t)n);
        if ((rc = copy_out(c, cur, xk.data()))) return rc;
        CU(cudaStreamSynchronize(c->stream));
        for (int64_t i = 0; i < n; ++i) xk[(size_t)i] = 2.f * xk[(size_t)i] - in[i];
        if ((rc = copy_in(c, prev, xk.data()))) return rc;
    }
    CU(cudaStreamSynchronize(c->stream));
    return TGV_OK;
}

static int energy_launch(tgv_ctx* c)
{
    int rc;
    size_t sl = 0;
    if ((rc = timer_begin(c, T_ENERGY, &sl))) return rc;
    const Bufs b = bufs(c->k);
    EnergyArgs ea{};
    ea.u = slot(c, slotU(b.cu));
    for (int d = 0; d < 3; ++d) {
        ea.v[d] = slot(c, slotV(b.cu, d));
        ea.p[d] = slot(c, slotP(b.cp, d));
    }
    for (int m = 0; m < 6; ++m) ea.q[m] = slot(c, slotQ(b.cp, m));
    ea.hist = hist_ptr(c);
    ea.alpha1 = c->alpha1;
    ea.alpha0 = c->alpha0;
    ea.lambda = c->lambda;
    ea.V = c->model == TGV_MODEL_TVL1 ? 0.0 : 2.0;  // TV-L1 has no v to bound (R14, R21)
    ea.nbins = c->nbins;
    int nb = 0;
    if (c->slots == 8 && c->count_bytes == 1) rc = launch_energy_t<8, uint8_t>(c, ea, b, &nb);
    else if (c->slots == 8) rc = launch_energy_t<8, uint16_t>(c, ea, b, &nb);
    else if (c->count_bytes == 1) rc = launch_energy_t<16, uint8_t>(c, ea, b, &nb);
    else rc = launch_energy_t<16, uint16_t>(c, ea, b, &nb);
    if (rc) return rc;
    CU(cudaGetLastError());
    energy_final_kernel<<<1, 256, 0, c->stream>>>(c->partials, nb, c->d_out);
    CU(cudaGetLastError());
    return timer_end(c, sl);
}

// {alpha1, alpha0, data, dual, vmax} sums -> ABI out[6]
static void energy_out(const double h[EN_TERMS], double out[6])
{
    const double E = h[0] + h[1] + h[2];
    out[0] = E;
    out[1] = h[0];
    out[2] = h[1];
    out[3] = h[2];
    out[4] = E - h[3];
    out[5] = h[4];
}

int tgv_energy(tgv_ctx* c, double out[6])
{
    NvtxRange nv("tgv_energy");
    int rc = check_ready(c);
    if (rc) return rc;
    if (!out) return fail(c, TGV_EINVAL, "out is NULL");
    if (!c->loaded) return fail(c, TGV_ESTATE, "energy before load");
    if (c->group) return fail(c, TGV_ESTATE, "grouped context: use tgv_group_energy");
    if ((rc = halo_exchange(c, plan_energy_for(c, c->k)))) return rc;
    if ((rc = energy_launch(c))) return rc;
    if (c->nranks > 1) {
        const NcclApi* nccl = c->nccl;
        NC(nccl->AllReduce(c->d_out, c->d_out, 4, ncclFloat64, ncclSum, c->comm, c->stream));
        NC(nccl->AllReduce(c->d_out + 4, c->d_out + 4, 1, ncclFloat64, ncclMax, c->comm, c->stream));
    }
    double h[EN_TERMS];
    CU(cudaMemcpyAsync(h, c->d_out, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    if ((rc = sync_stream(c))) return rc;
    energy_out(h, out);
    return TGV_OK;
}

// ============================================================================
// in-process slab groups
// ============================================================================
// every member waits for its neighbours' last recorded step, then copies the
// neighbours' boundary planes of the plan's slots into its halo planes
static int group_exchange(tgv_ctx* const* m, int n, const HaloPlan& hp)
{
    for (int r = 0; r < n; ++r) {
        tgv_ctx* c = m[r];
        CU(cudaSetDevice(c->device));
        size_t sl = 0;
        int rc = timer_begin(c, T_HALO, &sl);
        if (rc) return rc;
        const size_t bytes = sizeof(float) * (size_t)c->g.plane;
        if (r + 1 < n) {  // top halo <- bottom plane of r+1
            tgv_ctx* o = m[r + 1];
            CU(cudaStreamWaitEvent(c->stream, o->ev_step, 0));
            for (int k = 0; k < hp.ndown; ++k)
                CU(cudaMemcpyPeerAsync(plane_ptr(c, hp.down[k], c->g.nzl), c->device, plane_ptr(o, hp.down[k], 0),
                                       o->device, bytes, c->stream));
        }
        if (r > 0) {  // bottom halo <- top plane of r-1
            tgv_ctx* o = m[r - 1];
            CU(cudaStreamWaitEvent(c->stream, o->ev_step, 0));
            for (int k = 0; k < hp.nup; ++k)
                CU(cudaMemcpyPeerAsync(plane_ptr(c, hp.up[k], -1), c->device, plane_ptr(o, hp.up[k], o->g.nzl - 1),
                                       o->device, bytes, c->stream));
        }
        if ((rc = timer_end(c, sl))) return rc;
    }
    return TGV_OK;
}

static int group_record(tgv_ctx* const* m, int n)
{
    for (int r = 0; r < n; ++r) {
        tgv_ctx* c = m[r];
        CU(cudaSetDevice(c->device));
        CU(cudaEventRecord(c->ev_step, c->stream));
    }
    return TGV_OK;
}

static int group_check(tgv_ctx* const* m, int n)
{
    if (!m || n < 1) return TGV_EINVAL;
    for (int r = 0; r < n; ++r) {
        int rc = check_ready(m[r]);
        if (rc) return rc;
        tgv_ctx* c = m[r];
        if (!c->group || (int)c->group->size() != n || (*c->group)[r] != c)
            return fail(c, TGV_EINVAL, "contexts are not the members of one group, in rank order");
        if (!c->loaded) return fail(c, TGV_ESTATE, "group member %d not loaded", r);
        if (c->k != m[0]->k || c->schedule != m[0]->schedule || c->model != m[0]->model)
            return fail(c, TGV_ESTATE, "group members at different iterations or schedules");
    }
    return TGV_OK;
}

int tgv_create_group(const tgv_layout* layouts, const tgv_params* P, int n, const int* devices, tgv_ctx** out)
{
    tgv_ctx* c = nullptr;
    g_create_error[0] = 0;
    if (!layouts || !out || !devices || n < 1) return fail(c, TGV_EINVAL, "NULL argument or n < 1");
    for (int r = 0; r < n; ++r) out[r] = nullptr;
    for (int r = 0; r < n; ++r) {
        const tgv_layout& L = layouts[r];
        if (L.nx != layouts[0].nx || L.ny != layouts[0].ny || L.nz != layouts[0].nz)
            return fail(c, TGV_EINVAL, "group members must share nx, ny, nz");
        if ((r == 0 && L.z_begin != 0) || (r > 0 && L.z_begin != layouts[r - 1].z_end) ||
            (r == n - 1 && L.z_end != L.nz))
            return fail(c, TGV_EINVAL, "group slabs must tile [0, nz) in order");
    }
    auto* grp = new (std::nothrow) std::vector<tgv_ctx*>((size_t)n, nullptr);
    if (!grp) return fail(c, TGV_ENOMEM, "host allocation failed");
    for (int r = 0; r < n; ++r) {
        int rc = create_impl(&layouts[r], P, r, n, nullptr, devices[r], true, &out[r]);
        if (rc) {
            for (int k = 0; k < r; ++k) {
                out[k]->group = nullptr;
                tgv_destroy(out[k]);
                out[k] = nullptr;
            }
            delete grp;
            return rc;
        }
        (*grp)[r] = out[r];
        out[r]->group = grp;
    }
    bool all_peer = true;
    for (int r = 0; r < n; ++r)  // peer access between distinct devices (NVLink copies and stores)
        for (int o = 0; o < n; ++o)
            if (devices[r] != devices[o]) {
                int can = 0;
                cudaDeviceCanAccessPeer(&can, devices[r], devices[o]);
                if (can) {
                    cudaSetDevice(devices[r]);
                    cudaError_t e = cudaDeviceEnablePeerAccess(devices[o], 0);
                    if (e != cudaSuccess) cudaGetLastError();  // already enabled
                } else if (o == r - 1 || o == r + 1) {
                    all_peer = false;
                }
            }
    // peer halo mode (TGV_PEER_HALO=0 turns it off): each member maps its neighbours
    if (all_peer && n > 1 && env_int("TGV_PEER_HALO", 1) != 0)
        for (int r = 0; r < n; ++r) {
            tgv_ctx* c = out[r];
            c->peer = true;
            if (r > 0) {
                tgv_ctx* d = out[r - 1];
                c->pdn = d->state;
                c->pdn_fs = d->g.fs;
                c->pdn_top = d->g.nzl + 1;
                c->flag_dn_remote = d->flags + 2;  // its "from the upper neighbour" flag
            }
            if (r + 1 < n) {
                tgv_ctx* u = out[r + 1];
                c->pup = u->state;
                c->pup_fs = u->g.fs;
                c->flag_up_remote = u->flags + 1;  // its "from the lower neighbour" flag
            }
        }
    return TGV_OK;
}

int tgv_group_iterate(tgv_ctx* const* m, int n, int32_t iters)
{
    NvtxRange nv("tgv_group_iterate");
    int rc = group_check(m, n);
    if (rc) return rc;
    if (iters < 0) return fail(m[0], TGV_EINVAL, "n < 0");
    tgv_ctx* c = m[0];
    CU(cudaSetDevice(c->device));
    if ((rc = group_record(m, n))) return rc;  // the current state is each member's last step
    for (int32_t it = 0; it < iters; ++it) {
        const int64_t k = m[0]->k;
        if (m[0]->model == TGV_MODEL_TVL1 && m[0]->schedule == TGV_SCHEDULE_FUSED) {
            if ((rc = group_exchange(m, n, plan_tvl1_fused(k)))) return rc;
            for (int r = 0; r < n; ++r) {
                CU(cudaSetDevice(m[r]->device));
                if ((rc = launch_tvl1_fused(m[r]))) return rc;
            }
        } else if (m[0]->model == TGV_MODEL_TVL1) {
            if ((rc = group_exchange(m, n, plan_tvl1_a(k)))) return rc;
            for (int r = 0; r < n; ++r) {
                CU(cudaSetDevice(m[r]->device));
                if ((rc = launch_tvl1(m[r], 0))) return rc;
            }
            if ((rc = group_record(m, n))) return rc;
            if ((rc = group_exchange(m, n, plan_tvl1_b(k)))) return rc;
            for (int r = 0; r < n; ++r) {
                CU(cudaSetDevice(m[r]->device));
                if ((rc = launch_tvl1(m[r], 1))) return rc;
            }
        } else if (m[0]->schedule == TGV_SCHEDULE_SPLIT) {
            if ((rc = group_exchange(m, n, plan_split_a(k)))) return rc;
            for (int r = 0; r < n; ++r) {
                CU(cudaSetDevice(m[r]->device));
                if ((rc = launch_split(m[r], 0))) return rc;
            }
            if ((rc = group_record(m, n))) return rc;
            if ((rc = group_exchange(m, n, plan_split_b(k)))) return rc;
            for (int r = 0; r < n; ++r) {
                CU(cudaSetDevice(m[r]->device));
                if ((rc = launch_split(m[r], 1))) return rc;
            }
        } else if (peer_ready(m[0])) {  // peer halo mode (the members share peer, schedule and model)
            bool fresh = true;
            for (int r = 0; r < n; ++r) fresh = fresh && m[r]->halo_fresh;
            if (!fresh) {
                if ((rc = group_exchange(m, n, plan_fused(k)))) return rc;
            } else {  // order after the neighbours' previous launches (they wrote our halos, we write theirs)
                for (int r = 0; r < n; ++r) {
                    CU(cudaSetDevice(m[r]->device));
                    if (r > 0) CU(cudaStreamWaitEvent(m[r]->stream, m[r - 1]->ev_step, 0));
                    if (r + 1 < n) CU(cudaStreamWaitEvent(m[r]->stream, m[r + 1]->ev_step, 0));
                }
            }
            for (int r = 0; r < n; ++r) {
                CU(cudaSetDevice(m[r]->device));
                m[r]->peer_wait = fresh ? m[r]->seq : 0;
                m[r]->peer_now = true;
                rc = launch_fused(m[r]);
                m[r]->peer_now = false;
                if (rc) return rc;
                m[r]->halo_fresh = true;
            }
        } else {
            if ((rc = group_exchange(m, n, plan_fused(k)))) return rc;
            for (int r = 0; r < n; ++r) {
                CU(cudaSetDevice(m[r]->device));
                if ((rc = launch_fused(m[r]))) return rc;
            }
        }
        if (!peer_ready(m[0]))
            for (int r = 0; r < n; ++r) m[r]->halo_fresh = false;
        if ((rc = group_record(m, n))) return rc;
        for (int r = 0; r < n; ++r) m[r]->k += 1;
    }
    for (int r = 0; r < n; ++r) {
        c = m[r];
        CU(cudaSetDevice(c->device));
        if ((rc = sync_stream(c))) return rc;
    }
    return TGV_OK;
}

int tgv_group_energy(tgv_ctx* const* m, int n, double out[6])
{
    int rc = group_check(m, n);
    if (rc) return rc;
    if (!out) return fail(m[0], TGV_EINVAL, "out is NULL");
    tgv_ctx* c = m[0];
    if ((rc = group_record(m, n))) return rc;
    if ((rc = group_exchange(m, n, plan_energy_for(m[0], m[0]->k)))) return rc;
    double tot[EN_TERMS] = {0, 0, 0, 0, 0};
    for (int r = 0; r < n; ++r) {  // fixed rank order: deterministic
        c = m[r];
        CU(cudaSetDevice(c->device));
        if ((rc = energy_launch(c))) return rc;
        double h[EN_TERMS];
        CU(cudaMemcpyAsync(h, c->d_out, sizeof h, cudaMemcpyDeviceToHost, c->stream));
        if ((rc = sync_stream(c))) return rc;
        for (int t = 0; t < 4; ++t) tot[t] += h[t];
        tot[4] = std::max(tot[4], h[4]);
    }
    energy_out(tot, out);
    return TGV_OK;
}

int tgv_set_timing(tgv_ctx* c, int enable)
{
    if (!c) return TGV_EINVAL;
    c->timing = enable != 0;
    for (int k = 0; k < T_KINDS; ++k) {
        c->t_ms[k] = 0;
        c->t_n[k] = 0;
    }
    c->ev_kind.clear();
    c->ev_used = 0;
    return TGV_OK;
}

int tgv_get_timing(const tgv_ctx* c, tgv_timing* o)
{
    if (!c || !o) return TGV_EINVAL;
    o->dual_ms = c->t_ms[T_DUAL];
    o->primal_ms = c->t_ms[T_PRIMAL];
    o->fused_ms = c->t_ms[T_FUSED];
    o->energy_ms = c->t_ms[T_ENERGY];
    o->halo_ms = c->t_ms[T_HALO];
    o->dual_launches = c->t_n[T_DUAL];
    o->primal_launches = c->t_n[T_PRIMAL];
    o->fused_launches = c->t_n[T_FUSED];
    o->energy_launches = c->t_n[T_ENERGY];
    o->halo_exchanges = c->t_n[T_HALO];
    return TGV_OK;
}

int tgv_info(const tgv_ctx* c, tgv_info_t* o)
{
    if (!c || !o) return TGV_EINVAL;
    o->row_pitch = c->g.px;
    o->device_bytes = c->device_bytes;
    o->count_bytes = c->count_bytes;
    o->count_slots = c->slots;
    o->schedule = c->schedule;
    o->model = c->model;
    const int64_t hb = (int64_t)c->count_bytes * c->slots;
    // algorithmic HBM bytes per voxel of one launch:
    // split dual: reads u_k, u_{k-1}, v_k, v_{k-1}, p_k, q_k (17 floats), writes p, q (9)
    o->bytes_dual = 4 * (17 + 9);
    // split primal: reads p, q (new), u_k, v_k (13 floats) + histogram, writes u, v (4)
    o->bytes_primal = 4 * (13 + 4) + hb;
    // fused: reads 17 floats + histogram, writes u, v, p, q (13 floats)
    o->bytes_fused = 4 * (17 + 13) + hb;
    if (c->model == TGV_MODEL_TVL1) {  // TV-L1: dual reads u_k, u_{k-1}, p, writes p; primal reads p, u + counts, writes u
        o->bytes_dual = 4 * (5 + 3);
        o->bytes_primal = 4 * (4 + 1) + hb;
        o->bytes_fused = 4 * (5 + 4) + hb;
    }
    o->fused_zc = fused_zc(c);
    o->fused_tma = c->fused_tma ? 1 : 0;
    o->nranks = c->nranks;
    o->peer_halo = c->peer ? 1 : 0;
    o->pad = 0;
    o->rank = c->rank;
    o->iteration = c->k;
    return TGV_OK;
}

void tgv_destroy(tgv_ctx* c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->group) {  // leave the group; the last member frees the member table
        bool last = true;
        for (auto& mbr : *c->group) {
            if (mbr == c) mbr = nullptr;
            else if (mbr) last = false;
        }
        if (last) delete c->group;
        c->group = nullptr;
    }
    if (c->ev_step) cudaEventDestroy(c->ev_step);
    if (c->comm) {
        const NcclApi* nccl = c->nccl;
        if (c->poisoned)
            nccl->CommAbort(c->comm);
        else
            nccl->CommDestroy(c->comm);
    }
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    for (void* p : c->ipc_open)
        if (p) cudaIpcCloseMemHandle(p);
    cudaFree(c->flags);
    cudaFree(c->state);
    cudaFree(c->hist16);
    cudaFree(c->hist8);
    cudaFree(c->partials);
    cudaFree(c->d_out);
    cudaFree(c->d_maxc);
    cudaFree(c->staging);
    cudaFree(c->upload);
    if (c->s_in) cudaStreamSynchronize(c->s_in);
    if (c->s_out) cudaStreamSynchronize(c->s_out);
    cudaFree(c->stage);
    cudaFree(c->usnap);
    for (cudaEvent_t e : {c->ev_staged, c->ev_stage_free, c->ev_snap, c->ev_read})
        if (e) cudaEventDestroy(e);
    if (c->s_in) cudaStreamDestroy(c->s_in);
    if (c->s_out) cudaStreamDestroy(c->s_out);
    cudaFree(c->d_sched);
    cudaFree(c->d_sched_off);
    cudaFree(c->d_esched);
    cudaFree(c->d_esched_off);
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

}  // extern "C"

// NEXT-3 block-sparse brick sets (same translation unit: shares the kernels above)
#include "tgv_bricks_rt.cuh"

// tgv_runtime.cu -- context, C ABI (include/tgv.h) and NCCL z-slab halo
// exchange of the B200 TGV solver.
//
// One context per (process, GPU).  The context owns the fp32 SoA state
// (17 fields, each with one halo plane below and above the slab), the u16
// histogram store, a compute stream, CUDA events for kernel timing and, for
// nranks > 1, an NCCL communicator over NVLink/NVSwitch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/tgv.h"
#include "nccl_api.h"
#include "tgv_kernels.cuh"

using namespace tgvk;

namespace {

thread_local char g_create_error[512] = "";

// Halo plan (pinned on CPU by tests/test_slab_gloo.py).
// "down": this rank's BOTTOM owned plane goes to rank-1 (its top halo).
// "up":   this rank's TOP owned plane goes to rank+1 (its bottom halo).
struct HaloPlan {
    int ndown, nup;
    int down[4], up[4];
};
// before the dual step: grad ubar needs ubar(z+1); E(vbar) needs vbar_k(z-1)
constexpr HaloPlan HALO_A = {1, 3, {F_UBAR}, {F_VBAR + 0, F_VBAR + 1, F_VBAR + 2}};
// before the primal step: div p needs p_z(z-1); div2 q needs q_xz, q_yz, q_zz(z+1)
constexpr HaloPlan HALO_B = {3, 1, {F_Q + 4, F_Q + 5, F_Q + 2}, {F_P + 2}};
// energy: grad u (u(z+1)), E(v) (v(z-1)), div p, div2 q
constexpr HaloPlan HALO_E = {4, 4, {F_U, F_Q + 4, F_Q + 5, F_Q + 2}, {F_V + 0, F_V + 1, F_V + 2, F_P + 2}};

enum TimerKind { T_DUAL = 0, T_PRIMAL, T_ENERGY, T_HALO, T_KINDS };

}  // namespace

struct tgv_ctx {
    tgv_layout L{};
    int nbins = 0;
    float centers[16]{};
    float lambda = 0, alpha0 = 0, alpha1 = 0, tau = 0, sigma = 0;
    int rank = 0, nranks = 1, device = 0;

    Geo g{};
    int slots = 8;           // histogram slots per voxel
    float* state = nullptr;  // NF * g.fs floats
    uint16_t* hist = nullptr;
    double* partials = nullptr;
    double* d_out = nullptr;
    unsigned int* d_maxc = nullptr;
    uint32_t* staging = nullptr;
    int64_t staging_elems = 0;
    int energy_blocks = 0;
    int64_t device_bytes = 0;

    cudaStream_t stream = nullptr;
    ncclComm_t comm = nullptr;
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

inline float* field(tgv_ctx* c, int f) { return c->state + (int64_t)f * c->g.fs; }
// pointer to local plane z (z in [-1, nzl]) of field f
inline float* plane_ptr(tgv_ctx* c, int f, int z) { return field(c, f) + (int64_t)(z + 1) * c->g.plane; }

int check_ready(tgv_ctx* c)
{
    if (!c) return TGV_EINVAL;
    if (c->poisoned) return fail(c, TGV_ESTATE, "context poisoned by an earlier CUDA/NCCL failure");
    return TGV_OK;
}

// ---- timing -----------------------------------------------------------------
int timer_begin(tgv_ctx* c, int kind, size_t* slot)
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
    *slot = c->ev_used;
    c->ev_used += 2;
    c->ev_kind.push_back(kind);
    CU(cudaEventRecord(c->ev_pool[*slot], c->stream));
    return TGV_OK;
}
int timer_end(tgv_ctx* c, size_t slot)
{
    if (!c->timing) return TGV_OK;
    CU(cudaEventRecord(c->ev_pool[slot + 1], c->stream));
    return TGV_OK;
}
// after a stream sync: fold recorded pairs into the sums
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

int launch_dual(tgv_ctx* c)
{
    size_t slot = 0;
    int rc = timer_begin(c, T_DUAL, &slot);
    if (rc) return rc;
    dim3 blk(32, 8), grd((c->g.nx + 31) / 32, (c->g.ny + 7) / 8, c->g.nzl);
    dual_kernel<<<grd, blk, 0, c->stream>>>(c->state, c->g, step_params(c));
    CU(cudaGetLastError());
    return timer_end(c, slot);
}

int launch_primal(tgv_ctx* c)
{
    size_t slot = 0;
    int rc = timer_begin(c, T_PRIMAL, &slot);
    if (rc) return rc;
    dim3 blk(32, 8), grd((c->g.nx + 31) / 32, (c->g.ny + 7) / 8, c->g.nzl);
    const uint4* H = reinterpret_cast<const uint4*>(c->hist);
    if (c->slots == 8)
        primal_kernel<8><<<grd, blk, 0, c->stream>>>(c->state, H, c->g, step_params(c), centers(c));
    else
        primal_kernel<16><<<grd, blk, 0, c->stream>>>(c->state, H, c->g, step_params(c), centers(c));
    CU(cudaGetLastError());
    return timer_end(c, slot);
}

int halo_exchange(tgv_ctx* c, const HaloPlan& hp)
{
    if (c->nranks == 1) return TGV_OK;
    const NcclApi* nccl = c->nccl;
    size_t slot = 0;
    int rc = timer_begin(c, T_HALO, &slot);
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
    return timer_end(c, slot);
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

int init_from_hist(tgv_ctx* c)
{
    CU(cudaMemsetAsync(c->state, 0, sizeof(float) * (size_t)NF * (size_t)c->g.fs, c->stream));
    const uint4* H = reinterpret_cast<const uint4*>(c->hist);
    const int blocks = 148 * 8;
    if (c->slots == 8)
        init_state_kernel<8><<<blocks, 256, 0, c->stream>>>(c->state, H, c->g, centers(c));
    else
        init_state_kernel<16><<<blocks, 256, 0, c->stream>>>(c->state, H, c->g, centers(c));
    CU(cudaGetLastError());
    return TGV_OK;
}

}  // namespace

// =============================================================================
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

int tgv_create(const tgv_layout* L, const tgv_params* P, int rank, int nranks, const uint8_t* uid, int dev,
               tgv_ctx** out)
{
    tgv_ctx* c = nullptr;
    g_create_error[0] = 0;
    if (!out) return fail(c, TGV_EINVAL, "out is NULL");
    *out = nullptr;
    if (!L || !P) return fail(c, TGV_EINVAL, "layout or params is NULL");
    if (L->nx < 1 || L->ny < 1 || L->nz < 1) return fail(c, TGV_EINVAL, "grid extents must be >= 1");
    if (L->nx > (1 << 30) || L->ny > (1 << 30) || L->nz > (1 << 30)) return fail(c, TGV_EINVAL, "grid too large");
    if (L->z_begin < 0 || L->z_end > L->nz || L->z_begin >= L->z_end)
        return fail(c, TGV_EINVAL, "slab [%lld, %lld) outside [0, %lld) or empty", (long long)L->z_begin,
                    (long long)L->z_end, (long long)L->nz);
    if (L->brick[0] || L->brick[1] || L->brick[2])
        return fail(c, TGV_EINVAL, "brick layouts are not supported (brick must be {0,0,0})");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(c, TGV_EINVAL, "bad rank %d / nranks %d", rank, nranks);
    if ((nranks == 1) != (uid == nullptr)) return fail(c, TGV_EINVAL, "uid must be NULL iff nranks == 1");
    if (nranks == 1 && (L->z_begin != 0 || L->z_end != L->nz))
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

    Geo& g = c->g;
    g.nx = (int)L->nx;
    g.ny = (int)L->ny;
    g.nzl = (int)(L->z_end - L->z_begin);
    g.nz = (int)L->nz;
    g.z0 = (int)L->z_begin;
    g.px = (L->nx + 31) / 32 * 32;
    g.plane = g.px * L->ny;
    g.fs = (int64_t)(g.nzl + 2) * g.plane;

    int rc;
    if (cudaSetDevice(dev) != cudaSuccess) {
        fail(c, TGV_ECUDA, "cudaSetDevice(%d) failed", dev);
        return bail(TGV_ECUDA);
    }
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
        fail(c, TGV_ECUDA, "stream creation failed");
        return bail(TGV_ECUDA);
    }
    const size_t state_bytes = sizeof(float) * (size_t)NF * (size_t)g.fs;
    const size_t hist_bytes = sizeof(uint16_t) * (size_t)c->slots * (size_t)g.nzl * (size_t)g.plane;
    c->energy_blocks = 148 * 4;
    if (cudaMalloc(&c->state, state_bytes) != cudaSuccess || cudaMalloc(&c->hist, hist_bytes) != cudaSuccess ||
        cudaMalloc(&c->partials, sizeof(double) * EN_TERMS * c->energy_blocks) != cudaSuccess ||
        cudaMalloc(&c->d_out, sizeof(double) * 8) != cudaSuccess ||
        cudaMalloc(&c->d_maxc, sizeof(unsigned int)) != cudaSuccess) {
        cudaGetLastError();
        fail(c, TGV_ENOMEM, "device allocation of %.2f GB failed", (state_bytes + hist_bytes) / 1e9);
        return bail(TGV_ENOMEM);
    }
    c->device_bytes = (int64_t)(state_bytes + hist_bytes);
    if (cudaMemsetAsync(c->state, 0, state_bytes, c->stream) != cudaSuccess ||
        cudaMemsetAsync(c->hist, 0, hist_bytes, c->stream) != cudaSuccess) {
        fail(c, TGV_ECUDA, "memset failed");
        return bail(TGV_ECUDA);
    }

    if (nranks > 1) {
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
    }
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) {
        fail(c, TGV_ECUDA, "create sync failed");
        return bail(TGV_ECUDA);
    }
    (void)rc;
    *out = c;
    return TGV_OK;
}

int tgv_load_histograms(tgv_ctx* c, const uint32_t* counts, int64_t n_counts)
{
    int rc = check_ready(c);
    if (rc) return rc;
    const Geo& g = c->g;
    const int64_t per_plane = (int64_t)g.nx * g.ny * c->nbins;
    if (!counts) return fail(c, TGV_EINVAL, "counts is NULL");
    if (n_counts != per_plane * g.nzl)
        return fail(c, TGV_EINVAL, "n_counts %lld != %lld", (long long)n_counts, (long long)(per_plane * g.nzl));
    c->loaded = false;
    // staging buffer of whole planes, up to ~256 MB
    int planes_per_chunk = (int)std::max<int64_t>(1, std::min<int64_t>(g.nzl, (64ll << 20) / per_plane));
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
            pack_counts_kernel<8><<<blocks, 256, 0, c->stream>>>(c->staging, nzc, z0, g, c->nbins, c->hist, c->d_maxc);
        else
            pack_counts_kernel<16><<<blocks, 256, 0, c->stream>>>(c->staging, nzc, z0, g, c->nbins, c->hist,
                                                                   c->d_maxc);
        CU(cudaGetLastError());
    }
    unsigned int maxc = 0;
    CU(cudaMemcpyAsync(&maxc, c->d_maxc, sizeof maxc, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    if (maxc > 65535u) return fail(c, TGV_ERANGE, "histogram count %u exceeds 65535", maxc);
    rc = init_from_hist(c);
    if (rc) return rc;
    CU(cudaStreamSynchronize(c->stream));
    c->loaded = true;
    return TGV_OK;
}

int tgv_reset(tgv_ctx* c)
{
    int rc = check_ready(c);
    if (rc) return rc;
    if (!c->loaded) return fail(c, TGV_ESTATE, "reset before load");
    rc = init_from_hist(c);
    if (rc) return rc;
    CU(cudaStreamSynchronize(c->stream));
    return TGV_OK;
}

int tgv_iterate(tgv_ctx* c, int32_t n)
{
    int rc = check_ready(c);
    if (rc) return rc;
    if (n < 0) return fail(c, TGV_EINVAL, "n < 0");
    if (!c->loaded) return fail(c, TGV_ESTATE, "iterate before load");
    for (int32_t it = 0; it < n; ++it) {
        if ((rc = halo_exchange(c, HALO_A))) return rc;
        if ((rc = launch_dual(c))) return rc;
        if ((rc = halo_exchange(c, HALO_B))) return rc;
        if ((rc = launch_primal(c))) return rc;
    }
    return sync_stream(c);
}

static int copy_field_out(tgv_ctx* c, int f, float* out, int64_t n)
{
    const Geo& g = c->g;
    CU(cudaMemcpy2DAsync(out, sizeof(float) * g.nx, plane_ptr(c, f, 0), sizeof(float) * g.px, sizeof(float) * g.nx,
                         (size_t)g.ny * g.nzl, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    (void)n;
    return TGV_OK;
}

int tgv_read_field(tgv_ctx* c, int f, float* out, int64_t n)
{
    int rc = check_ready(c);
    if (rc) return rc;
    if (!out) return fail(c, TGV_EINVAL, "out is NULL");
    if (f < 0 || f >= NF) return fail(c, TGV_EINVAL, "bad field id %d", f);
    if (n != (int64_t)c->g.nx * c->g.ny * c->g.nzl) return fail(c, TGV_EINVAL, "n_voxels mismatch");
    if (!c->loaded) return fail(c, TGV_ESTATE, "read before load");
    return copy_field_out(c, f, out, n);
}

int tgv_read_u(tgv_ctx* c, float* u, int64_t n) { return tgv_read_field(c, TGV_FIELD_U, u, n); }

int tgv_write_field(tgv_ctx* c, int f, const float* in, int64_t n)
{
    int rc = check_ready(c);
    if (rc) return rc;
    if (!in) return fail(c, TGV_EINVAL, "in is NULL");
    if (f < 0 || f >= NF) return fail(c, TGV_EINVAL, "bad field id %d", f);
    if (n != (int64_t)c->g.nx * c->g.ny * c->g.nzl) return fail(c, TGV_EINVAL, "n_voxels mismatch");
    if (!c->loaded) return fail(c, TGV_ESTATE, "write before load");
    const Geo& g = c->g;
    CU(cudaMemcpy2DAsync(plane_ptr(c, f, 0), sizeof(float) * g.px, in, sizeof(float) * g.nx, sizeof(float) * g.nx,
                         (size_t)g.ny * g.nzl, cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return TGV_OK;
}

int tgv_energy(tgv_ctx* c, double out[6])
{
    int rc = check_ready(c);
    if (rc) return rc;
    if (!out) return fail(c, TGV_EINVAL, "out is NULL");
    if (!c->loaded) return fail(c, TGV_ESTATE, "energy before load");
    if ((rc = halo_exchange(c, HALO_E))) return rc;
    size_t slot = 0;
    if ((rc = timer_begin(c, T_ENERGY, &slot))) return rc;
    EnergyParams ep{c->alpha1, c->alpha0, c->lambda, 2.0, c->nbins};
    const uint4* H = reinterpret_cast<const uint4*>(c->hist);
    if (c->slots == 8)
        energy_partial_kernel<8><<<c->energy_blocks, 256, 0, c->stream>>>(c->state, H, c->g, ep, centers(c),
                                                                          c->partials);
    else
        energy_partial_kernel<16><<<c->energy_blocks, 256, 0, c->stream>>>(c->state, H, c->g, ep, centers(c),
                                                                           c->partials);
    CU(cudaGetLastError());
    energy_final_kernel<<<1, 256, 0, c->stream>>>(c->partials, c->energy_blocks, c->d_out);
    CU(cudaGetLastError());
    if ((rc = timer_end(c, slot))) return rc;
    if (c->nranks > 1) {
        const NcclApi* nccl = c->nccl;
        NC(nccl->AllReduce(c->d_out, c->d_out, 4, ncclFloat64, ncclSum, c->comm, c->stream));
        NC(nccl->AllReduce(c->d_out + 4, c->d_out + 4, 1, ncclFloat64, ncclMax, c->comm, c->stream));
    }
    double h[EN_TERMS];
    CU(cudaMemcpyAsync(h, c->d_out, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    if ((rc = sync_stream(c))) return rc;
    const double E = h[0] + h[1] + h[2];
    out[0] = E;
    out[1] = h[0];
    out[2] = h[1];
    out[3] = h[2];
    out[4] = E - h[3];
    out[5] = h[4];
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
    o->energy_ms = c->t_ms[T_ENERGY];
    o->halo_ms = c->t_ms[T_HALO];
    o->dual_launches = c->t_n[T_DUAL];
    o->primal_launches = c->t_n[T_PRIMAL];
    o->energy_launches = c->t_n[T_ENERGY];
    o->halo_exchanges = c->t_n[T_HALO];
    return TGV_OK;
}

int tgv_info(const tgv_ctx* c, tgv_info_t* o)
{
    if (!c || !o) return TGV_EINVAL;
    o->row_pitch = c->g.px;
    o->device_bytes = c->device_bytes;
    o->count_bytes = 2;
    o->count_slots = c->slots;
    // algorithmic bytes per voxel: dual reads ubar, vbar(3), p(3), q(6) and
    // writes p, q; primal reads p(3), q(6), u, v(3), histogram and writes u, v, ubar, vbar.
    o->bytes_dual = 4 * (13 + 9);
    o->bytes_primal = 4 * (13 + 8) + 2 * c->slots;
    o->nranks = c->nranks;
    o->rank = c->rank;
    return TGV_OK;
}

void tgv_destroy(tgv_ctx* c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->comm) {
        const NcclApi* nccl = c->nccl;
        if (c->poisoned)
            nccl->CommAbort(c->comm);
        else
            nccl->CommDestroy(c->comm);
    }
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    cudaFree(c->state);
    cudaFree(c->hist);
    cudaFree(c->partials);
    cudaFree(c->d_out);
    cudaFree(c->d_maxc);
    cudaFree(c->staging);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

}  // extern "C"

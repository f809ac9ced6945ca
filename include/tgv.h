/*
 * tgv.h -- C ABI of the B200 (sm_100a) TGV primal-dual solver.
 *
 * The library minimises, over an nx x ny x nz voxel grid (x fastest), the
 * discrete TGV functional of PAPER.md Eq. 2 (§3.2)
 *
 *     E(u, v) = sum_x  alpha1 |grad u - v|_2 + alpha0 |E(v)|_F
 *                      + lambda sum_b h_b |u - c_b|
 *
 * with E(v) = (grad v + grad v^T)/2 (Eq. 3), the indicator
 * u in [-1, 1] and the data term written through per-voxel
 * vote histograms h_b over bin centres c_b (Alg. 1
 * PAPER.md:252-278), by the primal-dual method the paper cites
 * ("we use the primal-dual method [pock2011tgv]").  The
 * discretisation and every reading of a point the paper leaves open are listed
 * in DESIGN.md §2 (R1-R17); the defining passages are cited per call below.
 *
 * Conventions for every call:
 *   - returns int status: TGV_OK (0) or a negative TGV_E* code; no C++
 *     exception ever crosses the ABI;
 *   - host buffers are owned by the caller, read or written only during the
 *     call and never retained; pinned (page-locked) buffers make the copies
 *     faster but are not required;
 *   - the context owns ALL device memory, streams, events and the NCCL
 *     communicator; one context per (process, GPU); calls on one context must
 *     not run concurrently;
 *   - a CUDA or NCCL failure poisons the context: that call returns
 *     TGV_ECUDA / TGV_ENCCL and every later call except tgv_destroy,
 *     tgv_last_error and tgv_status_string returns TGV_ESTATE;
 *   - calls marked COLLECTIVE must be made by every rank of the communicator
 *     in the same order.
 */
#ifndef TGV_H
#define TGV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define TGV_OK 0
#define TGV_EINVAL (-1) /* bad argument: NULL pointer, size mismatch, invalid parameter */
#define TGV_ENOMEM (-2) /* device or pinned-host allocation failed */
#define TGV_ECUDA (-3)  /* CUDA runtime failure (context poisoned) */
#define TGV_ENCCL (-4)  /* NCCL failure (context poisoned) */
#define TGV_ESTATE (-5) /* call not valid in this state (e.g. iterate before load; poisoned) */
#define TGV_ERANGE (-6) /* a histogram count exceeds 65535 (device counts are u16) */

/* ---- field ids for tgv_read_field / tgv_write_field -------------------- */
#define TGV_FIELD_U 0      /* primal indicator u                                   */
#define TGV_FIELD_V 1      /* primal vector field v: 1 + k, k = x, y, z            */
#define TGV_FIELD_UBAR 4   /* over-relaxed u: ubar = 2 u_new - u_old               */
#define TGV_FIELD_VBAR 5   /* over-relaxed v: 5 + k                                */
#define TGV_FIELD_P 8      /* dual of grad u - v: 8 + k                            */
#define TGV_FIELD_Q 11     /* dual of E(v): 11 + m, m = xx, yy, zz, xy, xz, yz     */
#define TGV_NUM_FIELDS 17

typedef struct tgv_ctx tgv_ctx; /* opaque */

/* Grid layout.  The global dense grid is nx x ny x nz voxels, voxel (x,y,z)
 * stored x fastest.  This rank owns the z-slab [z_begin, z_end)
 * (multi-GPU: contiguous slabs, rank r below rank r+1, every slab non-empty;
 * SURVEY.md §8(e)).  brick = {0,0,0} selects the plain linear layout; any
 * other value is reserved for block-sparse brick sets (SURVEY.md §8(f)
 * NEXT-3) and currently returns TGV_EINVAL. */
typedef struct {
    int64_t nx, ny, nz;
    int64_t z_begin, z_end;
    int32_t brick[3];
} tgv_layout;

/* Solver parameters (R1, R3, R5, R7).
 *   nbins        number of histogram bins, 1..16 (the paper uses 8, Alg. 1)
 *   bin_centers  nbins floats, strictly increasing, within [-1, 1]; copied at create.
 *                The paper's bins are c_b = -0.875 + 0.25 b (R3).
 *   lambda       data-term weight (>= 0); Eq. 2 literally is lambda = 1 (R1)
 *   alpha0       weight of |E(v)| (>= 0);  alpha1 weight of |grad u - v| (>= 0)
 *   tau, sigma   primal / dual step sizes (> 0), required tau*sigma*16 <= 1
 *                (16 bounds ||K||^2 of the discrete operator, R7). */
typedef struct {
    int32_t nbins;
    const float* bin_centers;
    float lambda, alpha0, alpha1, tau, sigma;
} tgv_params;

/* Iteration schedules (same scheme, same results up to fp32 rounding order;
 * DESIGN.md §5).  FUSED: one single-sweep kernel per iteration (dual, primal and
 * over-relaxation fused; 136 B per voxel-iteration with u16 counts, 128 B with
 * u8).  SPLIT: a dual kernel then a primal kernel (188 / 180 B). */
#define TGV_SCHEDULE_FUSED 0
#define TGV_SCHEDULE_SPLIT 1

/* Models.  TGV: Eq. 2, the default.  TVL1: Eq. 1
 * (PAPER.md:135-144), min_u sum alpha1 |grad u| + lambda sum_b h_b |u - c_b|,
 * the same scheme with v = q = 0 (R21).  Under
 * FUSED it runs as one TMA single-sweep kernel per iteration (44 B per
 * voxel-iteration with u8 counts), under SPLIT as a dual kernel and a primal
 * kernel (60 B); its restricted gap uses V = 0. */
#define TGV_MODEL_TGV 0
#define TGV_MODEL_TVL1 1

/* Kernel timing (device time from CUDA events on the launching stream). */
typedef struct {
    double dual_ms, primal_ms, fused_ms, energy_ms, halo_ms; /* summed device ms since last enable */
    int64_t dual_launches, primal_launches, fused_launches, energy_launches, halo_exchanges;
} tgv_timing;

/* Static facts about a context. */
typedef struct {
    int64_t row_pitch;        /* floats per stored row (>= nx, multiple of 32)             */
    int64_t device_bytes;     /* device memory owned by the context                        */
    int32_t count_bytes;      /* bytes per stored histogram count: 1 (u8) or 2 (u16)       */
    int32_t count_slots;      /* histogram slots stored per voxel (8 or 16)                */
    int32_t schedule;         /* TGV_SCHEDULE_*                                            */
    int32_t model;            /* TGV_MODEL_*                                               */
    int32_t fused_zc;         /* z-planes per CTA of the fused kernel                      */
    int32_t fused_tma;        /* 1: the fused kernel stages planes with TMA (default)      */
    int64_t bytes_dual;       /* algorithmic HBM bytes per voxel of one SPLIT dual launch  */
    int64_t bytes_primal;     /* ... of one SPLIT primal launch                            */
    int64_t bytes_fused;      /* ... of one FUSED launch (one whole iteration)             */
    int32_t nranks, rank;
    int64_t iteration;        /* iterations since the last load / reset                    */
    int32_t peer_halo;        /* 1: peer halo mode (the kernel writes the neighbours' halos) */
    int32_t pad;
} tgv_info_t;

/* Rank 0 creates the NCCL unique id; the caller broadcasts the 128 bytes
 * (e.g. with torch.distributed) to every rank before tgv_create. */
int tgv_get_unique_id(uint8_t uid[128]);

/* COLLECTIVE (nranks > 1).  Validates layout and parameters, selects
 * cuda_device, allocates the state (u and v at the current and two previous
 * iterates, p and q at two, in fp32 SoA planes with one halo plane below and
 * above the slab: 120 B per voxel) and the histogram store (16 B per voxel,
 * plus 8 B when u8 counts are used), creates streams/events and, if nranks > 1, the NCCL
 * communicator from uid (uid must be NULL iff nranks == 1).
 * Peer halo mode (nranks > 1, unless TGV_PEER_HALO=0 at create):
 * the neighbours' state and hand-over flags are mapped with CUDA IPC (handles
 * exchanged by an NCCL all-gather) and the fused TGV kernel writes its boundary
 * planes straight into the neighbours' halo planes; if any rank cannot map its
 * neighbours, every rank keeps the NCCL halo exchange.  tgv_destroy itself makes
 * no collective call, but in peer mode the ranks must be synchronised before it
 * (e.g. a barrier after their last tgv_iterate): no rank may free its state while
 * a neighbour's kernel can still write it.
 * Errors: TGV_EINVAL for any invalid argument (see tgv_params / tgv_layout;
 * also non-contiguous slabs across ranks), TGV_ENOMEM, TGV_ECUDA, TGV_ENCCL.
 * On error *out is NULL. */
int tgv_create(const tgv_layout* layout, const tgv_params* params, int rank, int nranks, const uint8_t* uid,
               int cuda_device, tgv_ctx** out);

/* Load this rank's histograms and reset the state.
 *   counts    host, uint32 [z_end - z_begin][ny][nx][nbins] (row-major, bins fastest)
 *   n_counts  number of uint32 elements; must equal (z_end-z_begin)*ny*nx*nbins
 * The counts are copied to the device in chunks and packed to u16, then to u8
 * when every count is <= 255 (the kernels read 8 instead of 16 B per voxel;
 * environment TGV_FORCE_U16=1 keeps u16).  Then
 * (R9): u = sum_b h_b c_b / W (0 where W = 0), v = p = q = 0,
 * ubar = u, vbar = 0, iteration counter 0.
 * Errors: TGV_EINVAL (NULL, size mismatch), TGV_ERANGE (a count > 65535; the
 * previous histograms are then lost and the context needs another load),
 * TGV_ECUDA.  Not collective. */
int tgv_load_histograms(tgv_ctx* ctx, const uint32_t* counts, int64_t n_counts);

/* Reset the state from the loaded histograms as tgv_load_histograms does,
 * without a host copy.  TGV_ESTATE before the first successful load. */
int tgv_reset(tgv_ctx* ctx);

/* NEXT-2: a pinhole range image for tgv_vote_depth_maps (§3.1).
 * world_dir = rot * cam_dir (rot row-major, its columns the camera axes);
 * a camera-frame point (X, Y, Z), Z > 0, lands on pixel (fx X/Z + cx, fy Y/Z + cy);
 * the depth map holds the camera-frame Z of the surface per pixel, NaN = none
 * (R4); vote_weight is Alg. 1's depthmap_vote (1, or 5 for LIDAR). */
typedef struct {
    double origin[3];
    double rot[9];
    double fx, fy, cx, cy;
    int32_t width, height;
    int32_t vote_weight;
    int32_t pad;
} tgv_camera;

/* NEXT-2: compute this slab's histograms on the GPU with Alg. 1 (
 * DESIGN.md R22) from host depth maps, then reset the state as
 * tgv_load_histograms does.  Voxel (x, y, z) (z global) has its centre at
 * grid_origin + voxel_size * (x, y, z) and radius voxel_radius (delta = 6 r,
 * eta = 18 r).  depths[i] is float [height][width] of camera i,
 * read during the call only; mipmap pyramids (mean of valid children) are built
 * on the device.  Needs nbins == 8.  Counts are bit-identical to the CPU
 * definition (fp64 without contraction).  Errors: TGV_EINVAL, TGV_ENOMEM,
 * TGV_ERANGE (a count > 65535), TGV_ECUDA. */
int tgv_vote_depth_maps(tgv_ctx* ctx, const tgv_camera* cams, int ncams, const float* const* depths,
                        const double grid_origin[3], double voxel_size, double voxel_radius);

/* Copy this slab's histogram counts to the host as uint32
 * [z_end-z_begin][ny][nx][nbins].  Errors: TGV_EINVAL, TGV_ESTATE, TGV_ECUDA. */
int tgv_read_counts(tgv_ctx* ctx, uint32_t* counts_out, int64_t n_counts);

/* NEXT-3 out-of-core leaves with frozen borders (§4.5, Fig. 9:
 * "we update the indicator for all cubes inside the current leaf's border (set A)
 * while the indicator for neighboring cubes outside of the border (set B) is
 * frozen"; R23).  tgv_create_leaf makes a single-GPU context over the
 * z-slab [z_begin, z_end) of an nx x ny x nz grid (a leaf); its halo planes hold
 * the B set and are never exchanged.  The primal (u, v) on B is frozen; the dual
 * variables the leaf's update reads there (p on the plane below, q on the plane
 * above) keep evolving from the frozen primal exactly as a slab's halo duals do
 * in the fused schedule.  Leaves run the fused TGV schedule only (set_schedule
 * SPLIT / set_model TVL1 return TGV_EINVAL).  tgv_set_border writes the border
 * plane below (side 0, global z_begin - 1) or above (side 1, global z_end):
 * u, v (3 planes), p (3), q (6), each [ny][nx] floats, NULL = zeros; call it
 * after tgv_load_histograms / tgv_reset / tgv_prolong_slab (which reset the
 * state; tgv_prolong_slab also fills the borders from the parents).  A leaf at
 * the global end has no border on that side.  Errors: TGV_EINVAL, TGV_ESTATE,
 * TGV_ECUDA. */
int tgv_create_leaf(const tgv_layout* layout, const tgv_params* params, int cuda_device, tgv_ctx** out);
int tgv_set_border(tgv_ctx* ctx, int side, const float* u, const float* v, const float* p, const float* q);

/* NEXT-3: move a leaf to another z-slab [z_begin, z_end) of the same grid with the
 * same number of planes, keeping its device memory (a pool of leaves streams a level
 * without allocating).  The context is unloaded afterwards: load its histograms
 * next.  Errors: TGV_EINVAL (bad slab / different size), TGV_ESTATE (not a leaf). */
int tgv_leaf_rebind(tgv_ctx* ctx, int64_t z_begin, int64_t z_end);

/* Peer halo mapping for contexts in different processes, the step
 * tgv_create performs over NCCL when TGV_PEER_HALO=1: tgv_peer_export writes a
 * 192-byte record (CUDA IPC handles of this context's state and hand-over flags,
 * its slot stride and plane count); the neighbour passes it to tgv_peer_import with
 * side 0 if the record's owner is its lower neighbour (slab just below) or 1 if its
 * upper.  From then on the fused TGV kernel of the importer writes its boundary
 * planes into that neighbour's halo planes and both hand over through the flags;
 * both neighbours must map each other, and the ranks must then be synchronised
 * before tgv_destroy (which itself makes no collective call, see tgv_create).
 * Errors: TGV_EINVAL, TGV_ESTATE, TGV_ECUDA. */
int tgv_peer_export(tgv_ctx* ctx, uint8_t rec[192]);
int tgv_peer_import(tgv_ctx* ctx, int side, const uint8_t rec[192]);

/* NEXT-1/3: this context's histograms as sums of factor^3 fine voxels (DESIGN.md
 * R18) of a finer grid nxf x nyf x nzf with ceil(n_fine / factor) = n on every axis;
 * fine_counts: host unsigned integers of count_bytes = 1, 2 or 4 bytes each,
 * [fz1-fz0][nyf][nxf][nbins], for the fine planes [factor * z_begin,
 * min(factor * z_end, nzf)) this slab covers (n_fine elements); then the state is
 * reset as by tgv_load_histograms.  Narrow counts cut the host-to-device bytes;
 * the sums are formed in 32 bits on the device.  Pinned host memory overlaps the
 * copies with other contexts' work.
 * Errors: TGV_EINVAL, TGV_ERANGE (a sum > 65535), TGV_ENOMEM, TGV_ECUDA. */
int tgv_load_histograms_coarsened(tgv_ctx* ctx, const void* fine_counts, int count_bytes, int64_t n_fine,
                                  int64_t nxf, int64_t nyf, int64_t nzf, int factor);

/* NEXT-1/3: restart this (loaded) context from a coarser solution held on the host:
 * u_c [cnz][cny][cnx] and v_c [3][cnz][cny][cnx] of coarse global planes
 * [cz0, cz0 + cnz) of the 2x-coarser grid (cnx = ceil(nx/2), cny = ceil(ny/2)).
 * u = parent u, v = parent v / 2, ubar = u, vbar = v, p = q = 0 (R19); for a leaf
 * the frozen border planes get their parents' u and v as well (the B set of
 * "equal to indicator values of their parenting cubes").
 * The slab must contain every needed parent.  Errors: TGV_EINVAL, TGV_ESTATE,
 * TGV_ENOMEM, TGV_ECUDA. */
int tgv_prolong_slab(tgv_ctx* ctx, const float* u_c, const float* v_c, int64_t cnx, int64_t cny, int64_t cz0,
                     int64_t cnz);

/* NEXT-1 coarse-to-fine ("coarse-to-fine scheme ... 200 iterations
 * ... on each level"; :431-433 §4.5; R18-R20).  Both need single-rank
 * contexts on one device with coarse = ceil(fine / 2) on every axis.
 *
 * tgv_restrict_from: this (coarse) context's histograms become the sums of the
 *   <= 8 children's counts of the loaded fine context; then the state is reset as
 *   by tgv_load_histograms.  Errors: TGV_EINVAL (not a 2x coarsening), TGV_ESTATE
 *   (fine not loaded), TGV_ERANGE (a sum > 65535), TGV_ECUDA.
 * tgv_prolong_from: this (fine, loaded) context's state restarts from the coarse
 *   solution: u = u_parent, v = v_parent / 2 (per-voxel slope on a grid of half
 *   spacing), ubar = u, vbar = v, p = q = 0, iteration counter 0.
 *   Errors: TGV_EINVAL, TGV_ESTATE, TGV_ECUDA. */
int tgv_restrict_from(tgv_ctx* coarse, const tgv_ctx* fine);
int tgv_prolong_from(tgv_ctx* fine, const tgv_ctx* coarse);

/* COLLECTIVE.  Run n >= 0 full iterations of the scheme:
 *   p <- P_alpha1(p + sigma (grad ubar - vbar)),  q <- P_alpha0(q + sigma E(vbar))
 *   u+ = clamp(prox_{tau lambda h}(u + tau div p), -1, 1),  v+ = v + tau (p + div2 q)
 *   ubar = 2 u+ - u,  vbar = 2 v+ - v
 * where P_a is the Euclidean (Frobenius for q) projection onto the ball of
 * radius a and the prox is the exact weighted median of the histogram-L1
 * term.  Multi-GPU: FUSED exchanges the one-plane halos of its
 * plan once per iteration by NCCL send/recv, SPLIT before each half-step; in
 * peer halo mode the fused kernel itself stores its boundary planes into the
 * neighbours' halo planes (no exchange between iterations).  On one GPU
 * without per-kernel timing, long runs replay a captured CUDA graph of six
 * iterations (the buffer-rotation period; TGV_GRAPH=0 disables it; the results
 * are bitwise those of plain launches).  Blocks until the device work is done.
 * Errors: TGV_EINVAL (n < 0), TGV_ESTATE (before load / poisoned), TGV_ECUDA, TGV_ENCCL. */
int tgv_iterate(tgv_ctx* ctx, int32_t n);

/* tgv_iterate without the final wait: returns once the n iterations are enqueued
 * on the context's CUDA stream, so the host can stage another context meanwhile
 * (NEXT-3 leaf pipelining).  Launch errors are returned; execution errors surface
 * at the next synchronising call (tgv_sync, tgv_read_*, tgv_energy, tgv_iterate).
 * Single-rank contexts without per-kernel timing only.
 * Errors: as tgv_iterate, plus TGV_ESTATE (timing enabled / nranks > 1). */
int tgv_iterate_async(tgv_ctx* ctx, int32_t n);

/* Wait for the context's enqueued work; reports asynchronous CUDA / NCCL errors.
 * Errors: TGV_ECUDA, TGV_ENCCL. */
int tgv_sync(tgv_ctx* ctx);

/* Copy this rank's u to the host: u_out float [z_end-z_begin][ny][nx];
 * n_voxels must equal (z_end-z_begin)*ny*nx.  Errors: TGV_EINVAL, TGV_ESTATE, TGV_ECUDA. */
int tgv_read_u(tgv_ctx* ctx, float* u_out, int64_t n_voxels);

/* Pipelined host I/O (a solve loop that overlaps the next step's input upload and this
 * step's result download with the iterations; DESIGN.md §7 "e2e"):
 *   tgv_stage_histograms  enqueue the H2D copy of this rank's counts (layout of
 *                         tgv_load_histograms, unsigned integers of count_bytes = 1, 2 or 4
 *                         bytes) into a device staging area on the context's upload stream
 *                         and return; it first waits (on the device) until the previously
 *                         staged counts were consumed.  The host buffer must stay valid and
 *                         unchanged until the next tgv_load_staged returns; pinned memory
 *                         lets the copy run beside the iterations.
 *   tgv_load_staged       tgv_load_histograms from the staged counts (waits for the copy on
 *                         the device; state reset as in tgv_load_histograms).  Blocks.
 *   tgv_read_u_async      snapshot u on the device (ordered after the iterations enqueued
 *                         so far), then copy it to u_out on the download stream and return;
 *                         u_out must stay valid until tgv_wait_io.  A second call first waits
 *                         (on the device) until the previous download has left the snapshot.
 *   tgv_wait_io           wait for both copy streams.
 * The staging area holds one whole slab of counts (count_bytes per count) and the snapshot one
 * slab of u; both are allocated at first use.
 * Errors: TGV_EINVAL (NULL, size, count_bytes), TGV_ESTATE (load_staged with nothing staged,
 * read before load), TGV_ERANGE (a count > 65535), TGV_ENOMEM, TGV_ECUDA. */
int tgv_stage_histograms(tgv_ctx* ctx, const void* counts, int count_bytes, int64_t n_counts);
int tgv_load_staged(tgv_ctx* ctx);
int tgv_read_u_async(tgv_ctx* ctx, float* u_out, int64_t n_voxels);
int tgv_wait_io(tgv_ctx* ctx);

/* Copy one state field (TGV_FIELD_*) of this rank to the host, same layout
 * and size rule as tgv_read_u.  Errors as tgv_read_u; TGV_EINVAL for a bad id. */
int tgv_read_field(tgv_ctx* ctx, int field, float* out, int64_t n_voxels);

/* Overwrite one state field from the host (test hook; the halo planes are
 * refreshed by the next iterate / energy).  TGV_FIELD_UBAR / VBAR set the
 * previous iterate to 2 x - in, so write U / V before UBAR / VBAR.
 * Errors as tgv_read_field. */
int tgv_write_field(tgv_ctx* ctx, int field, const float* in, int64_t n_voxels);

/* COLLECTIVE.  Energy and restricted primal-dual gap of the current state
 * (R14): per-voxel terms formed in fp32 from the
 * fp32 state (one TMA-staged sweep over the grid), summed in fp64 in a fixed
 * order (deterministic), fp64 NCCL all-reduce across ranks:
 *   out[0] E = alpha1-term + alpha0-term + data-term
 *   out[1] sum alpha1 |grad u - v|_2          out[2] sum alpha0 |E(v)|_F
 *   out[3] sum lambda sum_b h_b |u - c_b|
 *   out[4] gap_V = E - D_V,  D_V = sum min_{u in [-1,1]}(lambda sum_b h_b |u - c_b| - u div p)
 *                                  - V |p + div2 q|_1,  V = 2
 *   out[5] max_x,k |v_k|  (gap_V >= 0 is guaranteed while this is <= V)
 * Errors: TGV_EINVAL (NULL), TGV_ESTATE, TGV_ECUDA, TGV_ENCCL. */
int tgv_energy(tgv_ctx* ctx, double out[6]);

/* In-process slab group: n contexts for the z-slabs layouts[0..n-1] of ONE grid
 * (same nx, ny, nz; slabs tile [0, nz) in order), created in this process on
 * devices[0..n-1] (several slabs may share a device).  Members exchange their
 * one-plane halos by device-to-device copies (peer copies over NVLink between
 * GPUs), with the same halo plans as the NCCL path; the result is
 * bitwise equal to one context over the whole grid.  out receives n contexts.
 * Per-member calls (load, reset, read, write, info, timing, schedule) work as
 * usual; iterate and energy go through tgv_group_iterate / tgv_group_energy
 * (tgv_iterate / tgv_energy on a member return TGV_ESTATE).
 * Members run in peer halo mode unless TGV_PEER_HALO=0 (or neighbouring devices
 * lack peer access): the fused TGV kernel of each member writes its boundary planes
 * into the neighbours' halo planes, so after the first iteration of a call no halo
 * copy runs.
 * Errors: TGV_EINVAL, TGV_ENOMEM, TGV_ECUDA. */
int tgv_create_group(const tgv_layout* layouts, const tgv_params* params, int n, const int* devices,
                     tgv_ctx** out);

/* n >= 0 iterations of every member of a group (members passed in rank order,
 * all loaded, same schedule and iteration count).  Blocks until done. */
int tgv_group_iterate(tgv_ctx* const* members, int n, int32_t iterations);

/* Energy of the whole grid of a group (same out[6] as tgv_energy), members'
 * partial sums added on the host in rank order. */
int tgv_group_energy(tgv_ctx* const* members, int n, double out[6]);

/* Select the model (TGV_MODEL_TGV, the default, or TGV_MODEL_TVL1).  A loaded
 * context restarts from the initialisation.  Errors: TGV_EINVAL, TGV_ESTATE. */
int tgv_set_model(tgv_ctx* ctx, int model);

/* Select the iteration schedule (TGV_SCHEDULE_FUSED, the default, or
 * TGV_SCHEDULE_SPLIT; the environment variable TGV_SCHEDULE sets the default at
 * create).  The state is shared, so switching keeps the current iterate.
 * Errors: TGV_EINVAL (unknown schedule), TGV_ESTATE. */
int tgv_set_schedule(tgv_ctx* ctx, int schedule);

/* Enable (1) / disable (0) per-kernel CUDA-event timing inside tgv_iterate
 * and tgv_energy; tgv_get_timing returns the sums since the last enable. */
int tgv_set_timing(tgv_ctx* ctx, int enable);
int tgv_get_timing(const tgv_ctx* ctx, tgv_timing* out);

/* Static facts (pitch, device bytes, algorithmic bytes per voxel per launch). */
int tgv_info(const tgv_ctx* ctx, tgv_info_t* out);

/* Release everything; NULL-safe.  Makes no collective call (the NCCL comm is
 * aborted if a peer failed, destroyed otherwise); in peer halo mode synchronise
 * the ranks first (see tgv_create). */
void tgv_destroy(tgv_ctx* ctx);

/* Static string for a status code. */
const char* tgv_status_string(int status);

/* Human-readable detail of the last failure on ctx ("" if none; ctx may be NULL
 * for failures of tgv_create, which are kept per thread). */
const char* tgv_last_error(const tgv_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* TGV_H */

/*
 * tgv_bricks.h -- C ABI of the block-sparse brick-set solver (SURVEY.md §8(f)
 * NEXT-3, BASELINE.json configs[4]; same library as tgv.h, libtgv.so).
 *
 * The paper minimises each level over the cubes of a sparse octree that reach
 * their neighbours through stored references (§4.2), part by
 * part, updating the cubes inside a part's border (set A) while the cubes just
 * outside it (set B) stay frozen at the values of the previous level
 * (§4.5, Fig. 9).  A brick set is one level of that,
 * block-sparse (reading R24):
 *
 *   - nbricks bricks of edge E voxels (E = 4, 8, 16 or 32) at integer brick
 *     coordinates (bx, by, bz), each SOLVED (set A) or FROZEN (set B);
 *   - the domain Omega is the union of the bricks' voxels; the difference
 *     operators of tgv.h (R6) are restricted to Omega:
 *       D+_k w[x] = w[x + e_k] - w[x] if x + e_k is in Omega, else 0
 *       D-_k w[x] = [x + e_k in Omega] w[x] - [x - e_k in Omega] w[x - e_k]
 *     (Neumann / zero flux across the boundary of Omega);
 *   - S = A plus the frozen voxels with a face neighbour in A: the terms of the
 *     functional at any other voxel do not involve A (constants of the solve) and
 *     the primal step on A reads duals on S only;
 *   - one iteration is the scheme of tgv.h (dual step on the voxels of S, the
 *     duals elsewhere staying 0; primal step and over-relaxation on the voxels of
 *     A); u and v of B keep the values given by tgv_bricks_set_primal /
 *     tgv_bricks_prolong_from;
 *   - a box-shaped set of solved bricks is exactly the dense grid of tgv.h.
 *
 * Layout of every per-voxel host array: brick-major in the order the bricks were
 * given, inside a brick z, y, x (x fastest): element (b, z, y, x) is at
 * ((b * E + z) * E + y) * E + x.  Conventions (status codes, ownership,
 * poisoning) are those of tgv.h.  One iteration is a single sweep over the solved
 * bricks (128 B per voxel with u8 counts) after the duals of the frozen faces, or
 * (SPLIT, tgv_bricks_set_schedule) a dual kernel over S (104 B per voxel) and a
 * primal kernel over A (76 B per voxel with u8 counts, 84 B with u16).
 */
#ifndef TGV_BRICKS_H
#define TGV_BRICKS_H

#include <stdint.h>

#include "tgv.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tgv_bricks tgv_bricks; /* opaque */

/* Brick set of one level.
 *   edge     brick edge E in voxels: 4, 8, 16 or 32
 *   nbricks  number of bricks, >= 1, nbricks * E^3 < 2^31
 *   coords   int32 [nbricks][3] brick coordinates (bx, by, bz), each in [0, 2^20),
 *            pairwise distinct; copied at create
 *   frozen   uint8 [nbricks]: 0 = solved (set A), 1 = frozen (set B); NULL = all
 *            solved; copied at create */
typedef struct {
    int32_t edge;
    int64_t nbricks;
    const int32_t* coords;
    const uint8_t* frozen;
} tgv_brickset;

/* Create a brick-set context on cuda_device with the parameters of tgv.h
 * (tgv_params, same validity rules).  The neighbour table (6 face neighbours
 * per brick, or -1) is built here from the coordinates.
 * Errors: TGV_EINVAL (NULL, bad edge / count / coordinates, duplicate bricks,
 * invalid parameters), TGV_ENOMEM, TGV_ECUDA.  The reason is in
 * tgv_last_error(NULL) when *out could not be created. */
int tgv_bricks_create(const tgv_brickset* set, const tgv_params* params, int cuda_device, tgv_bricks** out);

/* NEXT-3 2:1 mixed-level set (reading R27; "each cube has
 * only 4 or less neighbors over each face", PAPER.md:446-453 frozen parent cubes).
 *   levels  uint8 [nbricks], 0 = finest, <= 7; brick b's voxels have edge h = 2^levels[b]
 *           in finest-level units and coords[b] is in its own level's brick units, so its
 *           voxel (x, y, z) is the cube h (E coords[b] + (x, y, z)) + [0, h)^3; copied.
 * The bricks must be disjoint and 2:1 balanced (face-adjacent bricks at most one level
 * apart; a coarser brick's face may be covered by up to four finer bricks, one per
 * quadrant, or partly by none).  Operators (R27): D+_k u(i) = (mean of u over the
 * voxels across i's +k face - u(i)) / ((h_i + h_n) / 2), 0 without a neighbour;
 * D-_k = -(D+_k)^* in the cell-volume-weighted inner product; every term of the energy
 * and of the restricted gap is weighted by h^3.  A one-level set (all levels equal 0) is
 * tgv_bricks_create's set bit for bit.  Schedules: SPLIT (any E), and for E = 32 FUSED
 * (the default there): the fused sweep over the solved level-0 bricks whose whole
 * 26-neighbourhood is level 0 or empty, the mixed SPLIT kernels over the other solved bricks,
 * bit for bit the SPLIT schedule's iterates.  tgv_bricks_vote_depth_maps votes brick b at
 * voxel size voxel_size 2^l and
 * radius voxel_radius 2^l; tgv_bricks_prolong_from accepts levels 0 and 1 (a level-1
 * brick copies the coarse brick at its own coordinates: u, v / 2).  Everything else as
 * tgv_bricks_create.  Errors: TGV_EINVAL (also NULL levels, a level > 7, overlapping or
 * unbalanced bricks), TGV_ENOMEM, TGV_ECUDA. */
int tgv_bricks_create_mixed(const tgv_brickset* set, const uint8_t* levels, const tgv_params* params, int cuda_device,
                            tgv_bricks** out);

/* Load the histograms and initialise (R9): counts [nbricks][E^3][nbins]
 * of unsigned integers of count_bytes bytes (1, 2 or 4), host memory; frozen
 * bricks' entries are ignored.  On A: u = ubar = vote-weighted mean of the bin
 * centres (0 where there is no vote); everywhere else and for every other field 0;
 * the iteration counter goes to 0.
 * Errors: TGV_EINVAL (NULL, n_counts != nbricks*E^3*nbins, bad count_bytes),
 * TGV_ERANGE (a count > 65535), TGV_ENOMEM, TGV_ECUDA. */
int tgv_bricks_load(tgv_bricks* ctx, const void* counts, int count_bytes, int64_t n_counts);

/* NEXT-2 on a brick set: Alg. 1 votes of the depth maps into
 * every voxel of every brick, then the initialisation of tgv_bricks_load.  The
 * voxel centre of brick b, offset (x, y, z) is grid_origin + voxel_size * (E *
 * coords[b] + (x, y, z)); cameras, depth maps, voxel_radius and the arithmetic
 * (fp64, nearest texel of the mip level chosen by the projected diameter) are
 * those of tgv_vote_depth_maps (tgv.h), so a brick's counts are bit-identical to
 * a dense vote of its box.  Requires nbins = 8.
 * Errors: TGV_EINVAL, TGV_ERANGE, TGV_ENOMEM, TGV_ECUDA. */
int tgv_bricks_vote_depth_maps(tgv_bricks* ctx, const tgv_camera* cams, int ncams, const float* const* depths,
                               const double grid_origin[3], double voxel_size, double voxel_radius);

/* Copy the stored counts to the host: counts_out uint32 [nbricks][E^3][nbins];
 * n_counts = nbricks*E^3*nbins.  Errors: TGV_EINVAL, TGV_ESTATE (no counts), TGV_ECUDA. */
int tgv_bricks_read_counts(tgv_bricks* ctx, uint32_t* counts_out, int64_t n_counts);

/* Re-initialise the state from the resident counts (as tgv_bricks_load, without
 * the upload).  Errors: TGV_EINVAL, TGV_ESTATE (no counts), TGV_ECUDA. */
int tgv_bricks_reset(tgv_bricks* ctx);

/* Refinement of the next finer level (R24, "where the samples are"):
 * flags uint8 [nbricks][8], flags[b][o] = 1 iff brick b is solved and a voxel of its
 * octant o = (x >= E/2) + 2 (y >= E/2) + 4 (z >= E/2) holds >= min_votes votes
 * outside the last (free-space) bin, else 0; octant o of brick (bx, by, bz) is the
 * finer level's brick (2bx + (o & 1), 2by + (o >> 1 & 1), 2bz + (o >> 2)).
 * n = 8 * nbricks.  Errors: TGV_EINVAL, TGV_ESTATE (no counts), TGV_ECUDA. */
int tgv_bricks_refine_flags(tgv_bricks* ctx, int32_t min_votes, uint8_t* flags, int64_t n);

/* Coarse-to-fine on brick sets (NEXT-1 with DESIGN.md R19; PAPER.md:167-168,
 * :431-433): every brick (bx, by, bz) of `fine` takes u = u and v = v / 2 of the
 * voxel of brick (bx/2, by/2, bz/2) of `coarse` (same edge E, same device; both
 * loaded) that contains it, into u, ubar, v and vbar; p = q = 0; the iteration
 * counter goes to 0.  Frozen bricks of `fine` keep these values from here on (the
 * borders of PAPER.md:449-453).
 * Errors: TGV_EINVAL (NULL, edges / devices differ, a brick without a parent),
 * TGV_ESTATE, TGV_ECUDA. */
int tgv_bricks_prolong_from(tgv_bricks* fine, const tgv_bricks* coarse);

/* Set u and v on every brick (A and B) and restart: ubar = u, vbar = v,
 * p = q = 0, iteration counter 0 (the prolongation restart of DESIGN.md R19;
 * the values on B stay frozen from here on).  u float [nbricks][E^3],
 * v float [3][nbricks][E^3] (component-major) or NULL for v = 0; n_voxels must
 * be nbricks*E^3.  Requires a previous tgv_bricks_load.
 * Errors: TGV_EINVAL, TGV_ESTATE, TGV_ECUDA. */
int tgv_bricks_set_primal(tgv_bricks* ctx, const float* u, const float* v, int64_t n_voxels);

/* Iteration schedule (same results bit for bit):
 *   TGV_SCHEDULE_FUSED (default for E = 32, the only edge it supports): per
 *     iteration the frozen-face dual launch, then one single-sweep launch over the
 *     solved bricks, two CTAs per brick (128 B per solved voxel with u8 counts);
 *   TGV_SCHEDULE_SPLIT (default otherwise): a dual launch over S and a primal
 *     launch over the solved bricks (180 B per solved voxel).
 * Errors: TGV_EINVAL (bad value; FUSED with E != 32). */
int tgv_bricks_set_schedule(tgv_bricks* ctx, int schedule);

/* Run n >= 0 iterations of the context's schedule and wait.
 * Errors: TGV_EINVAL (n < 0), TGV_ESTATE (before load), TGV_ECUDA. */
int tgv_bricks_iterate(tgv_bricks* ctx, int32_t n);

/* Copy one field (TGV_FIELD_U, V + k, P + k, Q + m of tgv.h) of every brick to
 * the host: out float [nbricks][E^3]; n_voxels = nbricks*E^3.  The over-relaxed
 * iterates are formed inside the kernels and not stored (TGV_FIELD_UBAR / VBAR
 * return TGV_EINVAL).  Errors: TGV_EINVAL, TGV_ESTATE, TGV_ECUDA. */
int tgv_bricks_read(tgv_bricks* ctx, int field, float* out, int64_t n_voxels);

/* Energy and restricted gap (R24, fp64 per-voxel terms, deterministic
 * reduction): the regulariser over S, the data term over A,
 *   out[0] E   out[1] alpha1-term   out[2] alpha0-term   out[3] data-term
 *   out[4] gap_V = E - D_V with
 *          D_V = sum_A [min_{u in [-1,1]} (lambda sum_b h_b |u - c_b| - u div p) - V |p + div2 q|_1]
 *              + sum_B [-u div p - v.(p + div2 q)],   V = 2
 *   out[5] max |v_k| over A.
 * Errors: TGV_EINVAL (NULL), TGV_ESTATE, TGV_ECUDA. */
int tgv_bricks_energy(tgv_bricks* ctx, double out[6]);

/* Per-kernel device timing with CUDA events on the context's stream (dual_ms --
 * the frozen-face launch included --, primal_ms, fused_ms, energy_ms and the launch
 * counts of tgv_timing; halo members are 0).  Enabling resets the sums.  Errors: TGV_EINVAL, TGV_ECUDA. */
int tgv_bricks_set_timing(tgv_bricks* ctx, int enable);
int tgv_bricks_get_timing(tgv_bricks* ctx, tgv_timing* out);

/* Static facts about a brick-set context.  S (R24) is the set of voxels
 * whose duals an iteration updates: the solved voxels and the frozen voxels with a
 * solved face neighbour; an iteration processes s_voxels in the dual kernel and
 * solved_voxels in the primal kernel. */
typedef struct {
    int64_t device_bytes;   /* device memory owned by the context                 */
    int32_t count_bytes;    /* stored bytes per count: 1 (u8) or 2 (u16), 0 before load */
    int32_t edge;           /* E                                                  */
    int64_t nbricks, nfrozen;
    int64_t solved_voxels;  /* (nbricks - nfrozen) * E^3                          */
    int64_t s_voxels;       /* |S|                                                */
    int32_t schedule;       /* TGV_SCHEDULE_FUSED or TGV_SCHEDULE_SPLIT           */
    int32_t pad;
} tgv_bricks_info_t;
int tgv_bricks_info(const tgv_bricks* ctx, tgv_bricks_info_t* out);

/* Detail of the last failure on ctx (or of the last failed create, ctx = NULL). */
const char* tgv_bricks_last_error(const tgv_bricks* ctx);

/* Free everything the context owns.  NULL-safe. */
void tgv_bricks_destroy(tgv_bricks* ctx);

#ifdef __cplusplus
}
#endif

#endif /* TGV_BRICKS_H */

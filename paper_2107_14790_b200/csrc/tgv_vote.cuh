// tgv_vote.cuh -- NEXT-2: histogram voting of Alg. 1 on the GPU (PAPER.md:252-278,
// §3.4 :236-250; §4.4 :390-402).
//
// Every voxel of the slab projects its centre into every camera, picks the
// depth-map pyramid level from its projected diameter, reads one texel and adds
// the camera's vote to one of the 8 bins.  The arithmetic that decides an integer
// (the pixel, the level, the bin) is IEEE fp64 with explicit round-to-nearest
// intrinsics (no FMA contraction), the level is the tie-up rounding of
// log2(diameter) evaluated as comparisons with sqrt(2) 2^k, so the counts are
// bit-identical to the plain CPU implementation of the same steps.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tgvk {

struct VoteCam {
    double origin[3];
    double rot[9];  // row-major world<-camera
    double fx, fy, cx, cy;
    int width, height, vote_weight, nlev;
    int64_t lev_off[24];  // offset of each pyramid level in the depth buffer (floats)
    int lw[24], lh[24];
};

// level L+1 texel = mean of the valid children of level L (NaN if none), fp64 sum in a fixed order
__global__ void pyramid_level_kernel(const float* __restrict__ src, int sw, int sh, float* __restrict__ dst, int w,
                                     int h)
{
    const int64_t n = (int64_t)w * h;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(i % w), y = (int)(i / w);
        double sum = 0.0;
        int cnt = 0;
        for (int dy = 0; dy < 2; ++dy)
            for (int dx = 0; dx < 2; ++dx) {
                const int xx = 2 * x + dx, yy = 2 * y + dy;
                if (xx < sw && yy < sh) {
                    const float v = src[(int64_t)yy * sw + xx];
                    if (v == v) {
                        sum = __dadd_rn(sum, (double)v);
                        ++cnt;
                    }
                }
            }
        dst[i] = cnt ? (float)__ddiv_rn(sum, (double)cnt) : __int_as_float(0x7fc00000);
    }
}

// Alg. 1 for one voxel centre pw (world coordinates): every camera's vote into acc[8]
__device__ __forceinline__ void vote_point(const VoteCam* __restrict__ cams, int ncams,
                                           const float* __restrict__ depth, double pw0, double pw1, double pw2,
                                           double r, double delta, double eta, unsigned int (&acc)[8])
{
    for (int c = 0; c < ncams; ++c) {
        const VoteCam& C = cams[c];
        const double d0 = __dsub_rn(pw0, C.origin[0]), d1 = __dsub_rn(pw1, C.origin[1]),
                     d2 = __dsub_rn(pw2, C.origin[2]);
        double pc[3];
#pragma unroll
        for (int k = 0; k < 3; ++k)
            pc[k] = __dadd_rn(__dadd_rn(__dmul_rn(C.rot[k], d0), __dmul_rn(C.rot[3 + k], d1)),
                              __dmul_rn(C.rot[6 + k], d2));
        if (!(pc[2] > 0.0)) continue;
        const double u = __dadd_rn(__ddiv_rn(__dmul_rn(C.fx, pc[0]), pc[2]), C.cx);
        const double v = __dadd_rn(__ddiv_rn(__dmul_rn(C.fy, pc[1]), pc[2]), C.cy);
        if (!(u >= 0.0 && u < (double)C.width && v >= 0.0 && v < (double)C.height)) continue;
        const double diam = __ddiv_rn(__dmul_rn(__dmul_rn(2.0, r), C.fx), pc[2]);
        int L = 0;
        double thr = 1.4142135623730951;  // sqrt(2) 2^k
        while (L < C.nlev - 1 && diam >= thr) {
            ++L;
            thr = __dmul_rn(thr, 2.0);
        }
        const double sc = (double)(1 << L);
        int ix = (int)floor(__ddiv_rn(u, sc)), iy = (int)floor(__ddiv_rn(v, sc));
        ix = min(ix, C.lw[L] - 1);
        iy = min(iy, C.lh[L] - 1);
        const float dep = __ldg(depth + C.lev_off[L] + (int64_t)iy * C.lw[L] + ix);
        if (dep != dep) continue;  // depth = None
        double a = __dsub_rn((double)dep, pc[2]);
        if (a < -eta) continue;  // occluded: no vote
        a = __ddiv_rn(a, delta);
        a = fmin(fmax(a, -1.0), 1.0);
        const int bin = min((int)floor(__dmul_rn(__ddiv_rn(__dadd_rn(a, 1.0), 2.0), 8.0)), 7);
        acc[bin] += (unsigned)C.vote_weight;
    }
}

// counts of local planes [0, nzl) of the slab, u16 store (SLOTS per voxel, bins 0..7
// used), running maximum for the range check / u8 decision
template <int SLOTS>
__global__ void __launch_bounds__(256) vote_kernel(const VoteCam* __restrict__ cams, int ncams,
                                                   const float* __restrict__ depth, Geo g, double ox, double oy,
                                                   double oz, double h, double r, uint16_t* __restrict__ H,
                                                   unsigned int* __restrict__ maxc)
{
    const int64_t n = (int64_t)g.nzl * g.ny * g.nx;
    const double delta = __dmul_rn(6.0, r), eta = __dmul_rn(3.0, delta);
    unsigned int m = 0;
    for (int64_t vi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; vi < n; vi += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(vi % g.nx);
        const int64_t rr = vi / g.nx;
        const int y = (int)(rr % g.ny);
        const int zl = (int)(rr / g.ny);
        const double pw0 = __dadd_rn(ox, __dmul_rn(h, (double)x));
        const double pw1 = __dadd_rn(oy, __dmul_rn(h, (double)y));
        const double pw2 = __dadd_rn(oz, __dmul_rn(h, (double)(g.z0 + zl)));
        unsigned int acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        vote_point(cams, ncams, depth, pw0, pw1, pw2, r, delta, eta, acc);
        uint16_t* dst = H + ((int64_t)zl * g.plane + (int64_t)y * g.px + x) * SLOTS;
#pragma unroll
        for (int b = 0; b < SLOTS; ++b) {
            const unsigned int cb = b < 8 ? acc[b] : 0u;
            m = max(m, cb);
            dst[b] = (uint16_t)min(cb, 65535u);
        }
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(FULL, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(maxc, m);
}

// u16 store -> uint32 [nzl][ny][nx][nbins] (dense, for tgv_read_counts)
__global__ void unpack_counts_kernel(const uint16_t* __restrict__ H, Geo g, int slots, int nbins,
                                     uint32_t* __restrict__ out)
{
    const int64_t n = (int64_t)g.nzl * g.ny * g.nx;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(v % g.nx);
        const int64_t r = v / g.nx;
        const int y = (int)(r % g.ny);
        const int z = (int)(r / g.ny);
        const uint16_t* src = H + ((int64_t)z * g.plane + (int64_t)y * g.px + x) * slots;
        for (int b = 0; b < nbins; ++b) out[v * nbins + b] = src[b];
    }
}

}  // namespace tgvk

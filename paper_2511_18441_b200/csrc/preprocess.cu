// K1 per-gaussian preprocess + K2 tile binning (render.py:172-229 restated for
// sm_100a).
//
// Everything that drives a discrete decision is evaluated in fp64 with the
// reference's own operation order: the world->camera FMA chain (numpy/OpenBLAS
// P @ R.T + t), the near clip, mean2d = fx*x/z + cx, the 3-sigma viewport cull,
// and the depth keys.  The raster consumes fp32 records plus per-gaussian
// guard bands (p_lo/p_hi/delta) that route the rare near-threshold decisions
// back to fp64 (see raster.cu).
//
// Pipeline per view (one handle):
//   k1_cull      per gaussian: fp64 projection -> kept flag + z key (+ key min/max)
//                and, for kept gaussians, the raster + exact records, z, footprint
//                tile rect and tile count, all by scene index g
//   scan/compact stable list of kept scene indices (ascending index)
//   radix sort   stable LSD sort of the z bit patterns over their varying bits
//                (== np.argsort(z, kind="stable"), render.py:216) -> gid[s]
//   k1_rank      rank_of[g] = s, tile counts in depth order
//   scan         emission offsets offs[s] (pairs emitted in rank order)
//   k2_emit      one (tile, g) pair per overlapped tile, in depth order
//   radix sort   stable sort on tile id -> (tile, depth) order
//   k2_ranges    per-tile [start, end)
// Records are stored by scene index: tile lists carry g, so no pass is needed to
// lay them out in depth order (nothing reads them in that order).
#include <cuda_fp16.h>
#include <math.h>

#include "common.cuh"
#include "shmath.cuh"

namespace rcgs {

struct Rect {
    int16_t x0, y0, x1, y1;  // inclusive tile rect; x1 < x0 => empty
};

struct ProjF64 {
    bool kept;
    double z, mx, my, a, b, c, det;
};

__device__ __forceinline__ ProjF64 project_one(const double* __restrict__ pos,
                                               const double* __restrict__ cov3d, int64_t g,
                                               const rcgs_camera& cam,
                                               const rcgs_raster_config& cfg) {
    ProjF64 p;
    const double p0 = pos[3 * g], p1 = pos[3 * g + 1], p2 = pos[3 * g + 2];
    const double x = cam_coord(cam.R, cam.t, 0, p0, p1, p2);
    const double y = cam_coord(cam.R, cam.t, 1, p0, p1, p2);
    const double z = cam_coord(cam.R, cam.t, 2, p0, p1, p2);
    p.z = z;
    p.kept = false;
    if (!(z > cfg.near_clip)) return p;  // render.py:176
    // mean2d = fx * x / z + cx (render.py:182), evaluated left to right, unfused
    p.mx = __dadd_rn(__ddiv_rn(__dmul_rn(cam.fx, x), z), cam.cx);
    p.my = __dadd_rn(__ddiv_rn(__dmul_rn(cam.fy, y), z), cam.cy);
    // EWA Jacobian and cov2d = (J W) Sigma (J W)^T + dilation (render.py:184-194),
    // with numpy's exact operation sequence (every op explicitly rounded: nvcc
    // would otherwise contract * + into FMAs), restated in oracle/c/rcgs_oracle.c:
    //   jac entries: plain ops;
    //   t = jac @ R: the stacked matmul runs through OpenBLAS dgemm, the fused chain
    //     fma(a2, b2, fma(a1, b1, a0 * b0)) with jac's structural zeros multiplied in;
    //   cov2 = einsum("nij,njk,nlk->nil", t, S, t): sum over j (outer), k (inner)
    //     of (t_ij * S_jk) * t_lk, accumulated left to right.
    const double zz = __dmul_rn(z, z);
    const double j00 = __ddiv_rn(cam.fx, z);
    const double j02 = __ddiv_rn(__dmul_rn(-cam.fx, x), zz);
    const double j11 = __ddiv_rn(cam.fy, z);
    const double j12 = __ddiv_rn(__dmul_rn(-cam.fy, y), zz);
    const double* R = cam.R;
    double t0[3], t1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        t0[k] = __fma_rn(j02, R[6 + k], __fma_rn(0.0, R[3 + k], __dmul_rn(j00, R[k])));
        t1[k] = __fma_rn(j12, R[6 + k], __fma_rn(j11, R[3 + k], __dmul_rn(0.0, R[k])));
    }
    const double* S6 = cov3d + 6 * g;  // xx xy xz yy yz zz
    const double S[3][3] = {{S6[0], S6[1], S6[2]}, {S6[1], S6[3], S6[4]}, {S6[2], S6[4], S6[5]}};
    auto quad = [&](const double* ti, const double* tl) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int k = 0; k < 3; ++k) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(ti[j], S[j][k]), tl[k]));
        return acc;
    };
    const double a = __dadd_rn(quad(t0, t0), cfg.covariance_dilation);
    const double b = quad(t0, t1);
    const double c = __dadd_rn(quad(t1, t1), cfg.covariance_dilation);
    // det, lambda_max, 3-sigma radius and viewport test (render.py:196-205), unfused
    const double det = __dsub_rn(__dmul_rn(a, c), __dmul_rn(b, b));
    const double mid = __dmul_rn(0.5, __dadd_rn(a, c));
    const double lam = __dadd_rn(mid, sqrt(fmax(__dsub_rn(__dmul_rn(mid, mid), det), 0.0)));
    const double radius = __dmul_rn(cfg.footprint_sigmas, sqrt(lam));
    const double w1 = (double)(cam.width - 1), h1 = (double)(cam.height - 1);
    p.kept = (det > 0) && (__dadd_rn(p.mx, radius) >= 0) && (__dsub_rn(p.mx, radius) <= w1) &&
             (__dadd_rn(p.my, radius) >= 0) && (__dsub_rn(p.my, radius) <= h1);
    p.a = a;
    p.b = b;
    p.c = c;
    p.det = det;
    return p;
}

// ---------------------------------------------------------------- scene
__global__ void cov3d_kernel(const double* __restrict__ rot, const double* __restrict__ scale,
                             int64_t n, double* __restrict__ cov) {
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const double w = rot[4 * g], x = rot[4 * g + 1], y = rot[4 * g + 2], z = rot[4 * g + 3];
    // quaternion_to_rotation (scene.py:98-112) and m = R diag(s): elementwise numpy
    // ops, each explicitly rounded (no FMA contraction); then m @ m^T, which numpy
    // runs through OpenBLAS dgemm: the fused chain (oracle/c/rcgs_oracle.c)
    auto sq2 = [](double p, double q) { return __dadd_rn(__dmul_rn(p, p), __dmul_rn(q, q)); };
    double r[3][3];
    r[0][0] = __dsub_rn(1.0, __dmul_rn(2.0, sq2(y, z)));
    r[0][1] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(x, y), __dmul_rn(w, z)));
    r[0][2] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, z), __dmul_rn(w, y)));
    r[1][0] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, y), __dmul_rn(w, z)));
    r[1][1] = __dsub_rn(1.0, __dmul_rn(2.0, sq2(x, z)));
    r[1][2] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(y, z), __dmul_rn(w, x)));
    r[2][0] = __dmul_rn(2.0, __dsub_rn(__dmul_rn(x, z), __dmul_rn(w, y)));
    r[2][1] = __dmul_rn(2.0, __dadd_rn(__dmul_rn(y, z), __dmul_rn(w, x)));
    r[2][2] = __dsub_rn(1.0, __dmul_rn(2.0, sq2(x, y)));
    double m[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) m[i][j] = __dmul_rn(r[i][j], scale[3 * g + j]);
    double s[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            s[i][j] = __fma_rn(m[i][2], m[j][2], __fma_rn(m[i][1], m[j][1], __dmul_rn(m[i][0], m[j][0])));
    double* o = cov + 6 * g;
    o[0] = s[0][0];
    o[1] = s[0][1];
    o[2] = s[0][2];
    o[3] = s[1][1];
    o[4] = s[1][2];
    o[5] = s[2][2];
}

// ---------------------------------------------------------------- K1a cull + keys
__global__ void k1_cull_kernel(const double* __restrict__ pos, const double* __restrict__ cov3d,
                               const double* __restrict__ opac, int64_t n, rcgs_camera cam,
                               rcgs_raster_config cfg, uint32_t* __restrict__ flag, uint64_t* __restrict__ key,
                               unsigned long long* __restrict__ minmax, double* __restrict__ z_out,
                               RasterRec* __restrict__ rec, ExactRec* __restrict__ exact,
                               Rect* __restrict__ rect, uint32_t* __restrict__ count,
                               MaskRec* __restrict__ mrec, int32_t* __restrict__ rank_of,
                               uint2* __restrict__ ranges, int ntiles, uint32_t* __restrict__ fix) {
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // the view's empty tile ranges (k2_ranges fills the non-empty ones) and the
    // culled default of rank_of (k1_rank writes the kept ranks), instead of memsets
    if (g < ntiles) ranges[g] = make_uint2(0u, 0u);
    if (g == 0) *fix = 0u;  // the colour fixup queue (Adam colour epilogue) starts empty
    unsigned long long kmin = ~0ull, kmax = 0ull;
    if (g < n) {
        rank_of[g] = -1;
        const ProjF64 p = project_one(pos, cov3d, g, cam, cfg);
        flag[g] = p.kept ? 1u : 0u;
        uint64_t k = (uint64_t)__double_as_longlong(p.z);  // z > near_clip > 0: bits order like values
        key[g] = k;
        if (p.kept) {
            kmin = k;
            kmax = k;
            z_out[g] = p.z;
            // raster + exact records, footprint tile rect and tile count, by scene index
            const double op = opac[g];
            // conic = inverse(cov2d) (render.py:221-223)
            const double ca = __ddiv_rn(p.c, p.det), cb = __ddiv_rn(-p.b, p.det), cc = __ddiv_rn(p.a, p.det);
            ExactRec ex;
            ex.mx = p.mx;
            ex.my = p.my;
            ex.ca = ca;
            ex.cb = cb;
            ex.cc = cc;
            ex.op = op;
            exact[g] = ex;

            // alpha >= skip  <=>  power >= P := log(skip / op).  The fp32 power error is bounded
            // by |power| * 2 / (1 - |rho|) * 5.4e-7 (rho = conic correlation); with a 4x safety
            // factor kappa = 4.4e-6 / (1 - |rho|) and the exact-check band is P -+ |P| kappa.
            const double P = log(cfg.alpha_skip / op);
            const double rho = fmin(fabs(cb) / sqrt(ca * cc), 0.999999);
            const double kappa = 4.4e-6 / (1.0 - rho);
            const double margin = fabs(P) * kappa + 1e-6;
            // opacity-aware footprint: alpha >= skip inside d^T conic d <= r2 = 2 ln(op/skip);
            // axis half widths r * sqrt(cov2d diag), padded for fp64 rounding.
            const double r2 = -2.0 * P;
            const double ex_ = r2 >= 0.0 ? sqrt(r2 * p.a) * (1.0 + 1e-7) + 1e-4 : 0.0;
            const double ey_ = r2 >= 0.0 ? sqrt(r2 * p.c) * (1.0 + 1e-7) + 1e-4 : 0.0;
            // half extents rounded up to fp16 (+0.01 px) for the raster's sub-tile culling
            const __half hx = __float2half_ru((float)fmin(ex_ + 0.01, 60000.0));
            const __half hy = __float2half_ru((float)fmin(ey_ + 0.01, 60000.0));
            const unsigned packed = (unsigned)__half_as_ushort(hx) | ((unsigned)__half_as_ushort(hy) << 16);
            // raster record in log2 units (power2 = log2(e) * power, so alpha = op * 2^power2)
            constexpr double kL = 1.4426950408889634;
            RasterRec r;
            const float mxh = (float)p.mx, myh = (float)p.my;
            r.a = make_float4(mxh, myh, __uint_as_float(packed), (float)log2(op));
            r.b = make_float4((float)(p.mx - (double)mxh), (float)(p.my - (double)myh), (float)((P - margin) * kL),
                              (float)((P + margin) * kL));
            r.c = make_float4((float)(-0.5 * ca * kL), (float)(-cb * kL), (float)(-0.5 * cc * kL), 0.f);
            rec[g] = r;
            if (mrec) mrec[g] = mask_setup(r.a, r.b, r.c);

            Rect rc;
            rc.x0 = 0;
            rc.y0 = 0;
            rc.x1 = -1;
            rc.y1 = -1;
            if (r2 >= 0.0) {
                const double umin = fmax(ceil(p.mx - ex_), 0.0), umax = fmin(floor(p.mx + ex_), cam.width - 1.0);
                const double vmin = fmax(ceil(p.my - ey_), 0.0), vmax = fmin(floor(p.my + ey_), cam.height - 1.0);
                if (umin <= umax && vmin <= vmax) {
                    rc.x0 = (int16_t)((int)umin / kTile);
                    rc.x1 = (int16_t)((int)umax / kTile);
                    rc.y0 = (int16_t)((int)vmin / kTile);
                    rc.y1 = (int16_t)((int)vmax / kTile);
                }
            }
            rect[g] = rc;
            count[g] = rc.x1 >= rc.x0 ? (uint32_t)(rc.x1 - rc.x0 + 1) * (uint32_t)(rc.y1 - rc.y0 + 1) : 0u;
        }
    }
    // block min/max -> one atomic per warp
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    // zero-initialised control words: the minimum is kept complemented (max of ~key)
    if ((threadIdx.x & 31) == 0 && kmax != 0ull) {
        atomicMax(&minmax[0], ~kmin);
        atomicMax(&minmax[1], kmax);
    }
}

// Compaction straight to the 4-byte truncated, rebased depth keys (the common
// path; compact_kernel + key_rebase_kernel feed the full 64-bit sort).
__global__ void compact_k32_kernel(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                                   const uint64_t* __restrict__ key, int64_t n, uint64_t kmin, int shift,
                                   uint32_t* __restrict__ k32, uint32_t* __restrict__ kgid) {
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n && flag[g]) {
        const uint32_t d = pos[g];
        k32[d] = (uint32_t)((key[g] - kmin) >> shift);
        kgid[d] = (uint32_t)g;
    }
}

__global__ void compact_kernel(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                               const uint64_t* __restrict__ key, int64_t n,
                               uint64_t* __restrict__ kkey, uint32_t* __restrict__ kgid) {
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n && flag[g]) {
        uint32_t d = pos[g];
        kkey[d] = key[g];
        kgid[d] = (uint32_t)g;
    }
}

// ---------------------------------------------------------------- depth order, 32-bit keys
constexpr int kRetryFullSort = 100;
// depth keys: the top 24 varying bits of the rebased fp64 z (3 radix passes);
// equal truncated keys are repaired by the exact fp64 key (depth_fixup_kernel)
#ifndef RCGS_DEPTH_KEY_BITS
#define RCGS_DEPTH_KEY_BITS 24
#endif
constexpr int kDepthKeyBits = RCGS_DEPTH_KEY_BITS;

__global__ void key_rebase_kernel(uint64_t* __restrict__ key, int64_t k, uint64_t kmin) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < k) key[i] -= kmin;
}

// Runs of equal truncated keys are re-sorted by the full fp64 key, ties by scene
// index (the stable input order of np.argsort, render.py:216): runs of at most 32
// by one thread (insertion sort); the start of every longer run is queued for
// long_run_sort_kernel, which measures, checks and (only if needed) sorts the run
// with a whole CTA.  Long runs are mostly exact fp64 ties (gaussians of a plane on
// a line of equal depth), already in index order from the stable LSD passes; a
// serial per-run scan with dependent gathers had been the launch's tail.
constexpr int kLongRun = 2048;

__global__ void depth_fixup_kernel(const uint32_t* __restrict__ k32, uint32_t* __restrict__ gid,
                                   const uint64_t* __restrict__ key_of, int64_t k, uint32_t* __restrict__ long_runs,
                                   uint32_t* __restrict__ n_long, uint32_t max_long) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    const uint32_t h = k32[i];
    if ((i > 0 && k32[i - 1] == h) || i + 1 >= k || k32[i + 1] != h) return;  // run starts only
    int64_t e = i + 1;
    while (e < k && k32[e] == h && e - i <= 32) ++e;
    if (e - i > 32) {  // a long run: measured, checked and sorted by a CTA
        const uint32_t slot = atomicAdd(n_long, 1u);
        if (slot < max_long) long_runs[slot] = (uint32_t)i;
        return;
    }
    const int len = (int)(e - i);
    uint64_t kk[32];
    uint32_t gg[32];
    for (int a = 0; a < len; ++a) {
        gg[a] = gid[i + a];
        kk[a] = key_of[gg[a]];
    }
    for (int a = 1; a < len; ++a) {  // insertion sort, stable, by (key, index)
        const uint64_t ck = kk[a];
        const uint32_t cg = gg[a];
        int b = a - 1;
        while (b >= 0 && (kk[b] > ck || (kk[b] == ck && gg[b] > cg))) {
            kk[b + 1] = kk[b];
            gg[b + 1] = gg[b];
            --b;
        }
        kk[b + 1] = ck;
        gg[b + 1] = cg;
    }
    for (int a = 0; a < len; ++a) gid[i + a] = gg[a];
}

// One CTA per queued long run (grid-stride over the queue): the run's length by a
// parallel scan of the truncated keys; runs already in (fp64 key, index) order
// (checked in parallel) are left alone, others of at most kLongRun entries get a
// bitonic sort of their (key, index) pairs in shared memory (padded to a power of
// two with +inf keys; keys are unique per index, so the result is the stable
// order).  Unsorted runs beyond kLongRun, or beyond the queue, are left to the
// order check (which then triggers the full 64-bit sort).
__global__ void __launch_bounds__(1024) long_run_sort_kernel(const uint32_t* __restrict__ k32,
                                                             uint32_t* __restrict__ gid,
                                                             const uint64_t* __restrict__ key_of, int64_t k,
                                                             const uint32_t* __restrict__ long_runs,
                                                             const uint32_t* __restrict__ n_long, uint32_t max_long) {
    __shared__ uint64_t sk[kLongRun];
    __shared__ uint32_t sg[kLongRun];
    __shared__ int s_len;
    const uint32_t nr = min(*n_long, max_long);
    for (uint32_t r = blockIdx.x; r < nr; r += gridDim.x) {
        const int64_t i0 = long_runs[r];
        const uint32_t h = k32[i0];
        // run length, capped at kLongRun + 1 (first differing position)
        if (threadIdx.x == 0) s_len = kLongRun + 1;
        __syncthreads();
        for (int a = threadIdx.x; a <= kLongRun; a += blockDim.x) {
            const int64_t e = i0 + a;
            if (e >= k || k32[e] != h) atomicMin(&s_len, a);
        }
        __syncthreads();
        const int len = s_len;
        if (len > kLongRun) {  // too long to sort here; the order check decides
            __syncthreads();
            continue;
        }
        int unsorted = 0;
        for (int a = threadIdx.x; a < len; a += blockDim.x) {
            const uint32_t g = gid[i0 + a];
            sg[a] = g;
            sk[a] = key_of[g];
        }
        __syncthreads();
        for (int a = threadIdx.x; a + 1 < len; a += blockDim.x)
            unsorted |= sk[a] > sk[a + 1] || (sk[a] == sk[a + 1] && sg[a] > sg[a + 1]);
        if (!__syncthreads_or(unsorted)) continue;
        int np2 = 64;  // the run padded to a power of two
        while (np2 < len) np2 <<= 1;
        for (int a = len + threadIdx.x; a < np2; a += blockDim.x) {
            sg[a] = 0xffffffffu;
            sk[a] = ~0ull;
        }
        __syncthreads();
        for (int size = 2; size <= np2; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int a = threadIdx.x; a < np2; a += blockDim.x) {
                    const int b = a ^ stride;
                    if (b > a) {
                        const bool up = (a & size) == 0;
                        const bool gt = sk[a] > sk[b] || (sk[a] == sk[b] && sg[a] > sg[b]);
                        if (gt == up) {
                            const uint64_t tk = sk[a];
                            sk[a] = sk[b];
                            sk[b] = tk;
                            const uint32_t tg = sg[a];
                            sg[a] = sg[b];
                            sg[b] = tg;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (int a = threadIdx.x; a < len; a += blockDim.x) gid[i0 + a] = sg[a];
        __syncthreads();
    }
}

// Flags any adjacent pair out of (fp64 key, index) order (only possible inside a
// tie run longer than kLongRun with differing low bits).
__global__ void depth_check_kernel(const uint32_t* __restrict__ k32, const uint32_t* __restrict__ gid,
                                   const uint64_t* __restrict__ key_of, int64_t k, int32_t* __restrict__ bad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i + 1 >= k || k32[i] != k32[i + 1]) return;
    const uint32_t g0 = gid[i], g1 = gid[i + 1];
    const uint64_t a = key_of[g0], b = key_of[g1];
    if (a > b || (a == b && g0 > g1)) atomicOr(bad, 1);
}

// ---------------------------------------------------------------- K1b records
// Depth rank s of each kept gaussian: rank_of[g] = s, and its tile count in
// depth order (the emission-offset scan runs in depth order).
__global__ void k1_rank_kernel(const uint32_t* __restrict__ gid, int64_t k, const uint32_t* __restrict__ count_g,
                               int32_t* __restrict__ rank_of, uint32_t* __restrict__ count_s) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= k) return;
    const uint32_t g = gid[s];
    rank_of[g] = (int32_t)s;
    count_s[s] = count_g[g];
}

// ---------------------------------------------------------------- K2 emission
// One warp per 32 consecutive depth ranks: their pairs are one contiguous range of
// emission slots, spread evenly over the lanes (a gaussian's footprint spans 1 to
// hundreds of tiles, so one thread per gaussian diverged); each lane finds the
// owning gaussian of its slot by a shuffle binary search over the warp's prefix of
// counts.  Slot order is the per-gaussian row-major tile order, as before.
// mrec (packed layout): the pair's block mask goes above the scene index, and a
// pair whose footprint reaches no block of its tile gets the key `sentinel`
// (= ntiles), which sorts after every tile and belongs to no tile list.
__global__ void k2_emit_kernel(const uint32_t* __restrict__ gid, const Rect* __restrict__ rect,
                               const uint32_t* __restrict__ offs, int64_t k, int tiles_x,
                               uint32_t* __restrict__ tile_key, uint32_t* __restrict__ emit_g,
                               const MaskRec* __restrict__ mrec, uint32_t sentinel,
                               int64_t k_total = INT64_MAX) {
    const int lane = threadIdx.x & 31;
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) >= k) return;  // whole warp beyond k
    uint32_t g = 0, cnt = 0, w = 1;
    int x0 = 0, y0 = 0;
    if (s < k) {
        g = gid[s];
        const Rect rc = rect[g];
        if (rc.x1 >= rc.x0) {
            w = (uint32_t)(rc.x1 - rc.x0 + 1);
            cnt = w * (uint32_t)(rc.y1 - rc.y0 + 1);
        }
        x0 = rc.x0;
        y0 = rc.y0;
    }
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    const uint32_t excl = incl - cnt;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t base = __shfl_sync(0xffffffffu, s < k ? offs[s] : 0u, 0);
    for (uint32_t p0 = 0; p0 < total; p0 += 32) {
        const uint32_t p = p0 + lane;
        int L = 0;  // last lane with excl <= p
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const uint32_t ex = __shfl_sync(0xffffffffu, excl, (L + step) & 31);
            if (L + step < 32 && ex <= p) L += step;
        }
        const uint32_t exL = __shfl_sync(0xffffffffu, excl, L), wL = __shfl_sync(0xffffffffu, w, L);
        const int x0L = __shfl_sync(0xffffffffu, x0, L), y0L = __shfl_sync(0xffffffffu, y0, L);
        const uint32_t gL = __shfl_sync(0xffffffffu, g, L);
        if (p < total) {
            const uint32_t q = p - exL;
            const uint32_t ty = (uint32_t)y0L + q / wL, tx = (uint32_t)x0L + q % wL;
            RCGS_DCHECK(tx < (uint32_t)tiles_x && gL < (uint32_t)k_total);
            uint32_t key = ty * (uint32_t)tiles_x + tx, val = gL;
            if (mrec) {
                const uint32_t bm = tile_block_mask(mrec[gL], (float)(tx * kTile), (float)(ty * kTile));
                val |= bm << kIdxBits;
                if (bm == 0u) key = sentinel;
            }
            tile_key[base + p] = key;
            emit_g[base + p] = val;
        }
    }
}

// Tile ranges of the sorted pairs (sentinel-keyed pairs: none), and, for scenes
// too large to pack the masks into the values, each pair's block mask.
__global__ void k2_ranges_kernel(const uint32_t* __restrict__ tile_key, const uint32_t* __restrict__ pair_g,
                                 const RasterRec* __restrict__ rec, int tiles_x, uint32_t ntiles, int64_t pairs,
                                 uint2* __restrict__ ranges, uint32_t* __restrict__ pair_m) {
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= pairs) return;
    uint32_t t = tile_key[j];
    if (t >= ntiles) return;
    if (j == 0 || tile_key[j - 1] != t) ranges[t].x = (uint32_t)j;
    if (j == pairs - 1 || tile_key[j + 1] != t) ranges[t].y = (uint32_t)(j + 1);
    if (pair_m == nullptr) return;
    const RasterRec* r = rec + pair_g[j];
    const float2 m = *reinterpret_cast<const float2*>(&r->a);  // the mean's hi parts only
    const int tx = (int)(t % (uint32_t)tiles_x), ty = (int)(t / (uint32_t)tiles_x);
    pair_m[j] = tile_block_mask(make_float4(m.x, m.y, 0.f, 0.f), r->b, r->c, (float)(tx * kTile),
                                (float)(ty * kTile));
}

// Raster work order: tiles by descending entry count (longest-processing-time
// first).  The persistent raster warps pull items in this order, so the heavy
// tiles start early and the tail of the launch is light tiles; in row-major order
// a few dense tiles taken last kept one SM busy for the second half of the
// launch.  Any order gives identical results (items are independent), so a
// single-CTA bucket scatter on count / max * 255 is enough.
__global__ void __launch_bounds__(1024) tile_order_kernel(const uint2* __restrict__ ranges, int ntiles,
                                                          uint32_t* __restrict__ order, uint4* __restrict__ meta) {
    __shared__ uint32_t hist[256];
    __shared__ uint32_t s_max;
    const int t = threadIdx.x;
    if (t < 256) hist[t] = 0;
    if (t == 0) s_max = 1;
    __syncthreads();
    uint32_t mx = 0;
    for (int i = t; i < ntiles; i += blockDim.x) {
        const uint2 r = ranges[i];
        mx = max(mx, r.y - r.x);
    }
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((t & 31) == 0) atomicMax(&s_max, mx);
    __syncthreads();
    const uint64_t m = s_max;
    auto bucket = [&](int i) -> int {  // 0 = heaviest
        const uint2 r = ranges[i];
        return 255 - (int)(((uint64_t)(r.y - r.x) * 255u) / m);
    };
    for (int i = t; i < ntiles; i += blockDim.x) atomicAdd(&hist[bucket(i)], 1u);
    __syncthreads();
    if (t < 32) {  // exclusive scan of the 256 buckets by one warp (8 per lane)
        uint32_t c[8], sum = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            c[j] = hist[8 * t + j];
            sum += c[j];
        }
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (t >= o) incl += y;
        }
        uint32_t run = incl - sum;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            hist[8 * t + j] = run;
            run += c[j];
        }
    }
    __syncthreads();
    // meta: the raster's per-item tile and list range in one 16-byte load (instead of
    // the dependent order -> ranges pair at the start of every work item)
    for (int i = t; i < ntiles; i += blockDim.x) {
        const uint32_t slot = atomicAdd(&hist[bucket(i)], 1u);
        order[slot] = (uint32_t)i;
        const uint2 r = ranges[i];
        meta[slot] = make_uint4((uint32_t)i, r.x, r.y, 0u);
    }
}

// Per-block lists, one CTA (8 warps) per work position: block b's list is the
// tile list's entries (in depth order) whose block mask has bit b, stored at
// blist[8 range.x + b len] (the raster's per-block record slots use the same
// bound), with its length at bcount[8 position + b].  The raster then walks only
// the entries that reach its 8x4 block (on the tile list ~70% of the entries a
// block stepped through were masked out).  Each round covers 256 list entries:
// per warp and block a ballot count, a cross-warp prefix in shared memory, then
// the stable write-out (one warp per tile had made the heaviest tiles' serial
// chunk chains the kernel's duration: 111 us).
__global__ void __launch_bounds__(256) block_lists_kernel(const uint4* __restrict__ meta, int npos,
                                                          const uint32_t* __restrict__ pair_g,
                                                          const uint32_t* __restrict__ pair_m, uint32_t idx_mask,
                                                          uint32_t* __restrict__ blist, uint32_t* __restrict__ bcount,
                                                          const RasterRec* __restrict__ rec, int tiles_x) {
    __shared__ uint32_t s_cnt[8][8];  // [warp][block] counts of the round
    __shared__ uint32_t s_run[8];     // per block: entries written in earlier rounds
    const int w = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (w >= npos) return;
    const uint4 tm = meta[w];
    const uint32_t x0 = tm.y, x1 = tm.z, len = x1 - x0;
    const uint32_t lt = (1u << lane) - 1u;
    if (threadIdx.x < 8) s_run[threadIdx.x] = 0u;
    __syncthreads();
    for (uint32_t c0 = x0; c0 < x1; c0 += 256) {
        const uint32_t j = c0 + 32 * warp + lane;
        uint32_t val = 0, mk = 0;
        if (j < x1) {
            val = pair_g[j];
            mk = pair_m ? pair_m[j] : (val >> kIdxBits);
        }
        const uint32_t g = val & idx_mask;
#ifdef RCGS_CHECKED
        if (j < x1) {  // a dropped (entry, block) must fail the exact per-block test too
            const RasterRec cr = rec[g];
            const int tx = (int)(tm.x % (uint32_t)tiles_x), ty = (int)(tm.x / (uint32_t)tiles_x);
            for (int b = 0; b < 8; ++b) {
                const float bx0 = (float)(tx * kTile + (b & 1) * 8), by0 = (float)(ty * kTile + (b >> 1) * 4);
                RCGS_DCHECK(((mk >> b) & 1u) || !(touches_block(cr.a, bx0, by0) &&
                                                 ellipse_touches_rect(cr.a, cr.b, cr.c, bx0, by0, bx0 + 7.f, by0 + 3.f)));
            }
        }
#endif
        uint32_t bal[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            bal[b] = __ballot_sync(0xffffffffu, j < x1 && ((mk >> b) & 1u));
            if (lane == b) s_cnt[warp][b] = __popc(bal[b]);
        }
        __syncthreads();
        uint32_t base = 0;  // lane b < 8: block b's first slot for this warp
        if (lane < 8) {
            base = s_run[lane];
            for (int q = 0; q < warp; ++q) base += s_cnt[q][lane];
        }
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const uint32_t bb = __shfl_sync(0xffffffffu, base, b);
            if ((bal[b] >> lane) & 1u) blist[8 * (size_t)x0 + (size_t)b * len + bb + __popc(bal[b] & lt)] = g;
        }
        __syncthreads();
        if (threadIdx.x < 8) {
            uint32_t add = 0;
            for (int q = 0; q < 8; ++q) add += s_cnt[q][threadIdx.x];
            s_run[threadIdx.x] += add;
        }
        __syncthreads();
    }
    if (threadIdx.x < 8) bcount[8 * w + threadIdx.x] = s_run[threadIdx.x];
}

// ---------------------------------------------------------------- colour (per step)
// Per-step colour (render.py:209-214), iterated in scene order so the 192-byte SH
// rows are read fully coalesced; the 16-byte result goes to the gaussian's
// depth-rank slot.
__global__ void __launch_bounds__(256, 4) color_kernel(const double* __restrict__ pos, const float4* __restrict__ sh,
                                                      const int32_t* __restrict__ rank_of, int64_t n, Center cen,
                                                      int deg, float4* __restrict__ color) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    if (rank_of[g] < 0) return;  // culled in this view
    // fp32 colour (shmath.cuh), quarters combined in the order the Adam colour
    // epilogue uses, so both give the same bits
    float fx, fy, fz;
    dir_f32(pos[3 * g] - cen.c[0], pos[3 * g + 1] - cen.c[1], pos[3 * g + 2] - cen.c[2], fx, fy, fz);
    float bf[16];
    basis16_rn(fx, fy, fz, deg, bf);
    const float4* row = sh + g * 12;
    float qf[4][3], mf[4][3];
#pragma unroll
    for (int part = 0; part < 4; ++part) {
        float c12[12];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const float4 f = row[3 * part + i];
            c12[4 * i] = f.x;
            c12[4 * i + 1] = f.y;
            c12[4 * i + 2] = f.z;
            c12[4 * i + 3] = f.w;
        }
        color_quarter_f32(bf, c12, part, qf[part], mf[part]);
    }
    int act = 0;
    float col[3];
    bool amb = false;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const float v = __fadd_rn(color_combine_f32(qf[0][ch], qf[1][ch], qf[2][ch], qf[3][ch]), 0.5f);
        amb = amb || color_ambiguous(v, color_combine_f32(mf[0][ch], mf[1][ch], mf[2][ch], mf[3][ch]));
        act |= (v > 0.f) << ch;
        col[ch] = fmaxf(0.f, v);
    }
    if (amb) {  // activation too close to call in fp32: the fp64 colour (exact decision)
        color[g] = color_f64(pos, sh, g, cen, deg);
        return;
    }
    color[g] = make_float4(col[0], col[1], col[2], __int_as_float(act));
}

__global__ void basis_export_kernel(const double* __restrict__ pos, const uint32_t* __restrict__ gid,
                                    const float4* __restrict__ color, int64_t k, Center cen, int deg,
                                    double* __restrict__ basis, uint8_t* __restrict__ active) {
    int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= k) return;
    if (basis) {
        double x, y, z;
        view_dir(pos, gid[s], cen.c, x, y, z);
        double b[16];
        sh_basis16<double>(x, y, z, deg, b);
        for (int i = 0; i < 16; ++i) basis[16 * s + i] = b[i];
    }
    if (active) {
        const int a = __float_as_int(color[gid[s]].w);
        active[3 * s] = a & 1;
        active[3 * s + 1] = (a >> 1) & 1;
        active[3 * s + 2] = (a >> 2) & 1;
    }
}

__global__ void kept_export_kernel(const uint32_t* __restrict__ gid, const double* __restrict__ z,
                                   int64_t k, int64_t* __restrict__ idx_out,
                                   double* __restrict__ z_out) {
    int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= k) return;
    if (idx_out) idx_out[s] = gid[s];
    if (z_out) z_out[s] = z[gid[s]];
}

static int validate_camera(const rcgs_camera* cam) {
    RCGS_CHECK_ARG(cam != nullptr, "camera is null");
    RCGS_CHECK_ARG(cam->width > 0 && cam->height > 0, "intrinsics: non-positive image dimensions");
    RCGS_CHECK_ARG(cam->fx > 0 && cam->fy > 0, "intrinsics: non-positive focal length");
    RCGS_CHECK_ARG((cam->width + kTile - 1) / kTile < 32768 && (cam->height + kTile - 1) / kTile < 32768,
                   "image too large");
    return RCGS_OK;
}

}  // namespace rcgs

using namespace rcgs;

extern "C" int rcgs_scene_create(const double* d_positions, const double* d_rotations,
                                 const double* d_scales, const double* d_opacities, int64_t n,
                                 int sh_degree, void* stream, rcgs_scene** out) {
    RCGS_CHECK_ARG(out != nullptr, "out is null");
    RCGS_CHECK_ARG(n >= 0 && n < (int64_t)0x7fffffff, "scene size %lld out of range", (long long)n);
    RCGS_CHECK_ARG(sh_degree >= 0 && sh_degree <= 3, "sh_degree must be in [0, 3]");
    cudaStream_t s = as_stream(stream);
    rcgs_scene* sc = new rcgs_scene();
    sc->n = n;
    sc->sh_degree = sh_degree;
    int st = RCGS_OK;
    if ((st = dalloc(&sc->pos, 3 * n, s)) || (st = dalloc(&sc->cov3d, 6 * n, s)) ||
        (st = dalloc(&sc->opac, n, s))) {
        dfree(sc->pos, s);
        dfree(sc->cov3d, s);
        dfree(sc->opac, s);
        delete sc;
        return st;
    }
    if (n > 0) {
        RCGS_CUDA(cudaMemcpyAsync(sc->pos, d_positions, 3 * n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        RCGS_CUDA(cudaMemcpyAsync(sc->opac, d_opacities, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
        cov3d_kernel<<<div_up(n, 256), 256, 0, s>>>(d_rotations, d_scales, n, sc->cov3d);
        RCGS_LAUNCH_CHECK();
    }
    *out = sc;
    return RCGS_OK;
}

extern "C" int rcgs_scene_destroy(rcgs_scene* sc, void* stream) {
    if (!sc) return RCGS_OK;
    cudaStream_t s = as_stream(stream);
    dfree(sc->pos, s);
    dfree(sc->cov3d, s);
    dfree(sc->opac, s);
    delete sc;
    return RCGS_OK;
}

static void view_free(rcgs_view* v, cudaStream_t s) {
    dfree(v->gid, s);
    dfree(v->z, s);
    dfree(v->rec, s);
    dfree(v->exact, s);
    dfree(v->offs, s);
    dfree(v->color, s);
    dfree(v->rank_of, s);
    dfree(v->fix, s);
    dfree(v->acc_fx, s);
    dfree(v->pair_g, s);
    dfree(v->pair_m, s);
    dfree(v->ranges, s);
    dfree(v->tile_order, s);
    dfree(v->tile_meta, s);
    dfree(v->blist, s);
    dfree(v->bcount, s);
    dfree(v->work, s);
    release_records(v, s);  // arena ownership, or the view-owned compact copy
    v->wrec_n = v->wrec_s = nullptr;
    v->wrec_w = v->wrec_tf = nullptr;
    v->wrec_valid = false;
}

extern "C" int rcgs_view_destroy(rcgs_view* v, void* stream) {
    if (!v) return RCGS_OK;
    view_free(v, as_stream(stream));
    delete v;
    return RCGS_OK;
}

static int view_build(rcgs_view* v, cudaStream_t s) {
    const rcgs_scene* sc = v->scene;
    const int64_t n = sc->n;
    const int ntiles = v->tiles_x * v->tiles_y;
    RCGS_TRY(dalloc(&v->rank_of, n, s));
    RCGS_TRY(dalloc(&v->fix, n + 1, s));
    RCGS_TRY(dalloc(&v->acc_fx, 3 * n, s));
    if (n > 0) RCGS_CUDA(cudaMemsetAsync(v->acc_fx, 0, 3 * n * sizeof(unsigned long long), s));
    v->acc_dirty = false;
    RCGS_TRY(dalloc(&v->ranges, ntiles, s));
    // the view's persistent work counters (words 0-1) and the build's control words,
    // zeroed by one memset: key min (complemented) / max (u64 words 1, 2), the
    // order-check flag and the long-run count (u32 words 6, 7)
    RCGS_TRY(dalloc(&v->work, 8, s));
    RCGS_CUDA(cudaMemsetAsync(v->work, 0, 8 * sizeof(unsigned), s));
    unsigned long long* minmax = reinterpret_cast<unsigned long long*>(v->work) + 1;
    int32_t* fix_flag = reinterpret_cast<int32_t*>(v->work + 6);
    uint32_t* n_long = v->work + 7;
    v->k = 0;
    v->pairs = 0;
    v->sort_bits = 0;
    if (n == 0) {
        RCGS_CUDA(cudaMemsetAsync(v->fix, 0, sizeof(uint32_t), s));
        RCGS_CUDA(cudaMemsetAsync(v->ranges, 0, ntiles * sizeof(uint2), s));
        RCGS_TRY(dalloc(&v->offs, 1, s));
        RCGS_CUDA(cudaMemsetAsync(v->offs, 0, sizeof(uint32_t), s));
        return RCGS_OK;
    }
    // ---- K1: cull, keys and (for kept gaussians) the records, by scene index
    uint32_t *flag = nullptr, *kpos = nullptr, *kgid = nullptr, *kgid_alt = nullptr, *count_g = nullptr;
    uint64_t *key = nullptr, *kkey = nullptr, *kkey_alt = nullptr;
    Rect* rect = nullptr;
    RCGS_TRY(dalloc(&flag, n, s));
    RCGS_TRY(dalloc(&kpos, n + 1, s));
    RCGS_TRY(dalloc(&key, n, s));
    RCGS_TRY(dalloc(&v->z, n, s));
    RCGS_TRY(dalloc(&v->rec, n, s));
    RCGS_TRY(dalloc(&v->exact, n, s));
    RCGS_TRY(dalloc(&v->color, n, s));
    RCGS_TRY(dalloc(&rect, n, s));
    RCGS_TRY(dalloc(&count_g, n, s));
    static const bool pack_ok = [] {  // RCGS_PAIR_PACK=0: the large-scene layout (tests)
        const char* e = getenv("RCGS_PAIR_PACK");
        return !(e && atoi(e) == 0);
    }();
    v->pair_packed = pack_ok && n < ((int64_t)1 << kIdxBits);
    MaskRec* mrec = nullptr;  // packed layout: per-gaussian block-mask setup for K2 emit
    if (v->pair_packed) RCGS_TRY(dalloc(&mrec, n, s));
    k1_cull_kernel<<<div_up(n > ntiles ? n : (int64_t)ntiles, 256), 256, 0, s>>>(
        sc->pos, sc->cov3d, sc->opac, n, v->cam, v->cfg, flag, key, minmax, v->z, v->rec, v->exact, rect, count_g,
        mrec, v->rank_of, v->ranges, ntiles, v->fix);
    RCGS_LAUNCH_CHECK();
    RCGS_TRY(exclusive_scan_u32(flag, kpos, n, s));
    uint64_t* host = static_cast<uint64_t*>(pinned_scratch(4 * sizeof(uint64_t)));
    RCGS_CHECK_ARG(host != nullptr, "pinned scratch allocation failed");
    uint32_t* hk = reinterpret_cast<uint32_t*>(host + 2);
    RCGS_CUDA(cudaMemcpyAsync(host, minmax, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    RCGS_CUDA(cudaMemcpyAsync(hk, kpos + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    RCGS_CUDA(cudaStreamSynchronize(s));
    const int64_t k = *hk;
    const uint64_t kmin = ~host[0], kmax = host[1];
    v->k = k;
    RCGS_TRY(dalloc(&v->offs, k + 1, s));
    if (k == 0) {
        RCGS_CUDA(cudaMemsetAsync(v->offs, 0, sizeof(uint32_t), s));
        dfree(flag, s);
        dfree(kpos, s);
        dfree(key, s);
        dfree(rect, s);
        dfree(mrec, s);
        dfree(count_g, s);
        return RCGS_OK;
    }
    // ---- stable depth sort over the varying key bits
    // keys relative to the smallest kept key (order preserving): the exponent
    // carry between e.g. [1, 2) and [2, 4) no longer widens the sorted range
    const uint64_t span = kmax - kmin;
    v->sort_bits = span ? 64 - __builtin_clzll(span) : 0;
    const bool k32_path = v->sort_bits <= kDepthKeyBits || !v->full_sort;
    RCGS_TRY(dalloc(&kgid, k, s));
    RCGS_TRY(dalloc(&kgid_alt, k, s));
    if (k32_path) {
        // 4-byte keys holding the top kDepthKeyBits varying bits (3 radix passes;
        // exact when the span has no more bits), written by the compaction, then the
        // tie-run repair of runs with equal truncated keys and the order check
        const int shift = v->sort_bits > kDepthKeyBits ? v->sort_bits - kDepthKeyBits : 0;
        uint32_t *k32 = nullptr, *k32_alt = nullptr;
        RCGS_TRY(dalloc(&k32, k, s));
        RCGS_TRY(dalloc(&k32_alt, k, s));
        compact_k32_kernel<<<div_up(n, 256), 256, 0, s>>>(flag, kpos, key, n, kmin, shift, k32, kgid);
        RCGS_LAUNCH_CHECK();
        dfree(flag, s);
        dfree(kpos, s);
        if (v->sort_bits > 0) {
            RCGS_TRY(radix_sort_u32(&k32, &k32_alt, &kgid, &kgid_alt, false, k,
                                    v->sort_bits < kDepthKeyBits ? v->sort_bits : kDepthKeyBits, s));
            if (shift > 0) {
                const uint32_t max_long = (uint32_t)(k / 33 + 1);
                uint32_t* long_runs = nullptr;
                RCGS_TRY(dalloc(&long_runs, max_long, s));
                depth_fixup_kernel<<<div_up(k, 256), 256, 0, s>>>(k32, kgid, key, k, long_runs, n_long, max_long);
                long_run_sort_kernel<<<128, 1024, 0, s>>>(k32, kgid, key, k, long_runs, n_long, max_long);
                depth_check_kernel<<<div_up(k, 256), 256, 0, s>>>(k32, kgid, key, k, fix_flag);
                dfree(long_runs, s);
            }
            RCGS_LAUNCH_CHECK();
        }
        dfree(k32, s);
        dfree(k32_alt, s);
    } else {
        RCGS_TRY(dalloc(&kkey, k, s));
        RCGS_TRY(dalloc(&kkey_alt, k, s));
        compact_kernel<<<div_up(n, 256), 256, 0, s>>>(flag, kpos, key, n, kkey, kgid);
        RCGS_LAUNCH_CHECK();
        dfree(flag, s);
        dfree(kpos, s);
        key_rebase_kernel<<<div_up(k, 256), 256, 0, s>>>(kkey, k, kmin);
        RCGS_TRY(radix_sort_u64(&kkey, &kkey_alt, &kgid, &kgid_alt, false, k, v->sort_bits, s));
    }
    dfree(key, s);
    dfree(kkey, s);
    dfree(kkey_alt, s);
    dfree(kgid_alt, s);
    // ---- depth ranks: gid[s] (the sorted scene indices), rank_of, counts in depth order
    v->gid = kgid;
    uint32_t* count = nullptr;
    RCGS_TRY(dalloc(&count, k, s));
    k1_rank_kernel<<<div_up(k, 256), 256, 0, s>>>(v->gid, k, count_g, v->rank_of, count);
    RCGS_LAUNCH_CHECK();
    dfree(count_g, s);
    RCGS_TRY(exclusive_scan_u32(count, v->offs, k, s));
    uint32_t* hp = reinterpret_cast<uint32_t*>(host);
    RCGS_CUDA(cudaMemcpyAsync(hp, v->offs + k, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    RCGS_CUDA(cudaMemcpyAsync(hp + 1, fix_flag, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RCGS_CUDA(cudaStreamSynchronize(s));
    const int64_t pairs = hp[0];
    dfree(count, s);
    if (hp[1] != 0) {  // a long tie run needs the full 64-bit key sort: rebuild
        dfree(rect, s);
        dfree(mrec, s);
        return kRetryFullSort;
    }
    v->pairs = pairs;
    if (pairs == 0) {
        dfree(rect, s);
        dfree(mrec, s);
        return RCGS_OK;
    }
    // ---- K2 emit (depth order, values = scene index) + stable tile sort; the sort
    // carries the scene indices themselves, so its output values are the tile lists
    uint32_t *tkey = nullptr, *tkey_alt = nullptr, *emit_g = nullptr, *g_alt = nullptr;
    RCGS_TRY(dalloc(&tkey, pairs, s));
    RCGS_TRY(dalloc(&tkey_alt, pairs, s));
    RCGS_TRY(dalloc(&emit_g, pairs, s));
    RCGS_TRY(dalloc(&g_alt, pairs, s));
    k2_emit_kernel<<<div_up(k, 256), 256, 0, s>>>(v->gid, rect, v->offs, k, v->tiles_x, tkey, emit_g, mrec,
                                                  (uint32_t)ntiles, v->n);
    RCGS_LAUNCH_CHECK();
    dfree(rect, s);
    dfree(mrec, s);
    int tile_bits = 1;
    while ((1 << tile_bits) <= ntiles) ++tile_bits;  // room for the sentinel key ntiles
    RCGS_TRY(radix_sort_u32(&tkey, &tkey_alt, &emit_g, &g_alt, false, pairs, tile_bits, s));
    v->pair_g = emit_g;
    if (!v->pair_packed) RCGS_TRY(dalloc(&v->pair_m, pairs, s));
    k2_ranges_kernel<<<div_up(pairs, 256), 256, 0, s>>>(tkey, emit_g, v->rec, v->tiles_x, (uint32_t)ntiles, pairs,
                                                        v->ranges, v->pair_m);
    RCGS_LAUNCH_CHECK();
    RCGS_TRY(dalloc(&v->tile_order, ntiles, s));
    RCGS_TRY(dalloc(&v->tile_meta, ntiles, s));
    tile_order_kernel<<<1, 1024, 0, s>>>(v->ranges, (int)ntiles, v->tile_order, v->tile_meta);
    RCGS_LAUNCH_CHECK();
    RCGS_TRY(dalloc(&v->blist, 8 * pairs, s));
    RCGS_TRY(dalloc(&v->bcount, 8 * (int64_t)ntiles, s));
    block_lists_kernel<<<ntiles, 256, 0, s>>>(
        v->tile_meta, (int)ntiles, v->pair_g, v->pair_packed ? nullptr : v->pair_m, v->pair_packed ? kIdxMask : 0xffffffffu,
        v->blist, v->bcount, v->rec, v->tiles_x);
    RCGS_LAUNCH_CHECK();
    dfree(g_alt, s);
    dfree(tkey, s);
    dfree(tkey_alt, s);
    return RCGS_OK;
}

extern "C" int rcgs_view_create(const rcgs_scene* scene, const rcgs_camera* cam,
                                const rcgs_raster_config* cfg, void* stream, rcgs_view** out) {
    RCGS_CHECK_ARG(scene != nullptr && cfg != nullptr && out != nullptr, "null argument");
    RCGS_TRY(validate_camera(cam));
    cudaStream_t s = as_stream(stream);
    rcgs_view* v = new rcgs_view();
    v->scene = scene;
    v->cam = *cam;
    v->cfg = *cfg;
    v->n = scene->n;
    v->tiles_x = (cam->width + kTile - 1) / kTile;
    v->tiles_y = (cam->height + kTile - 1) / kTile;
    int st = view_build(v, s);
    if (st == kRetryFullSort) {
        view_free(v, s);
        v->full_sort = true;
        st = view_build(v, s);
    }
    if (st != RCGS_OK) {
        view_free(v, s);
        delete v;
        return st;
    }
    *out = v;
    return RCGS_OK;
}

extern "C" int rcgs_view_info_get(const rcgs_view* v, rcgs_view_info* out) {
    RCGS_CHECK_ARG(v != nullptr && out != nullptr, "null argument");
    out->n_gaussians = v->n;
    out->n_kept = v->k;
    out->n_pairs = v->pairs;
    out->tiles_x = v->tiles_x;
    out->tiles_y = v->tiles_y;
    out->tile_size = kTile;
    out->sort_bits = v->sort_bits;
    return RCGS_OK;
}

extern "C" int rcgs_view_kept(const rcgs_view* v, int64_t* d_index, double* d_depth, void* stream) {
    RCGS_CHECK_ARG(v != nullptr, "null view");
    if (v->k == 0) return RCGS_OK;
    kept_export_kernel<<<div_up(v->k, 256), 256, 0, as_stream(stream)>>>(v->gid, v->z, v->k, d_index, d_depth);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

__global__ void exact_export_kernel(const uint32_t* __restrict__ gid, const ExactRec* __restrict__ exact, int64_t k,
                                    double* __restrict__ out) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= k) return;
    const ExactRec e = exact[gid[s]];
    double* o = out + 6 * s;
    o[0] = e.mx;
    o[1] = e.my;
    o[2] = e.ca;
    o[3] = e.cb;
    o[4] = e.cc;
    o[5] = e.op;
}

extern "C" int rcgs_view_exact(const rcgs_view* v, double* d_out, void* stream) {
    RCGS_CHECK_ARG(v != nullptr && d_out != nullptr, "null argument");
    if (v->k == 0) return RCGS_OK;
    exact_export_kernel<<<div_up(v->k, 256), 256, 0, as_stream(stream)>>>(v->gid, v->exact, v->k, d_out);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

__global__ void unpack_pairs_kernel(const uint32_t* __restrict__ in, int64_t n, uint32_t* __restrict__ out) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) out[j] = in[j] & kIdxMask;
}

extern "C" int rcgs_view_pairs(const rcgs_view* v, uint32_t* d_pair_g, void* stream) {
    RCGS_CHECK_ARG(v != nullptr && d_pair_g != nullptr, "null argument");
    if (v->pairs == 0) return RCGS_OK;
    if (v->pair_packed) {
        unpack_pairs_kernel<<<div_up(v->pairs, 256), 256, 0, as_stream(stream)>>>(v->pair_g, v->pairs, d_pair_g);
        RCGS_LAUNCH_CHECK();
        return RCGS_OK;
    }
    RCGS_CUDA(cudaMemcpyAsync(d_pair_g, v->pair_g, sizeof(uint32_t) * (size_t)v->pairs, cudaMemcpyDeviceToDevice,
                              as_stream(stream)));
    return RCGS_OK;
}

extern "C" int rcgs_view_ranges(const rcgs_view* v, uint32_t* d_ranges, void* stream) {
    RCGS_CHECK_ARG(v != nullptr && d_ranges != nullptr, "null argument");
    RCGS_CUDA(cudaMemcpyAsync(d_ranges, v->ranges, sizeof(uint2) * (size_t)v->tiles_x * v->tiles_y,
                              cudaMemcpyDeviceToDevice, as_stream(stream)));
    return RCGS_OK;
}

extern "C" int rcgs_view_color(rcgs_view* v, const float* d_sh, void* stream) {
    RCGS_CHECK_ARG(v != nullptr, "null view");
    if (v->k == 0) return RCGS_OK;
    RCGS_CHECK_ARG(d_sh != nullptr, "null SH");
    Center c = camera_center(v->cam);
    color_kernel<<<div_up(v->n, 256), 256, 0, as_stream(stream)>>>(
        v->scene->pos, reinterpret_cast<const float4*>(d_sh), v->rank_of, v->n, c, v->scene->sh_degree, v->color);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

extern "C" int rcgs_view_basis(const rcgs_view* v, double* d_basis, uint8_t* d_active, void* stream) {
    RCGS_CHECK_ARG(v != nullptr, "null view");
    if (v->k == 0) return RCGS_OK;
    Center c = camera_center(v->cam);
    basis_export_kernel<<<div_up(v->k, 256), 256, 0, as_stream(stream)>>>(v->scene->pos, v->gid, v->color, v->k, c,
                                                                          v->scene->sh_degree, d_basis, d_active);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

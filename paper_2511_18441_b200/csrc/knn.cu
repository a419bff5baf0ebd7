// Select-from-mask outlier statistics on the GPU:
// knn_mean_distances (selection.py:155-159) -- per point, the mean Euclidean
// distance to its k nearest neighbours (self excluded) -- exactly as scipy's
// cKDTree query + numpy mean produce it:
//   * distances sqrt((dx^2 + dy^2) + dz^2), unfused, correctly rounded sqrt
//     (cKDTree's squared-Minkowski accumulation over dims 0, 1, 2);
//   * the k smallest of them ascending (the (k+1)-th smallest overall, which is
//     the point itself or an identical duplicate at distance 0, is dropped);
//   * their sum in numpy's pairwise order (8 accumulators for 8 < k <= 128, then
//     ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)), tail sequentially),
//     divided by k.
// The search is exact for any grid: a uniform grid of cells of size h (cell
// keys radix-sorted, an open-addressing hash from cell key to its point range),
// one thread per point visiting Chebyshev shells of cells around its own until
// the (k+1)-th best squared distance is no larger than the squared distance to
// the unsearched region.  h only sets the speed: it is re-derived from the
// median (k+1)-NN radius of a sample of points, measured with the same exact
// query on a first grid.
#include <math.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace rcgs {

constexpr int kKnnMaxK = 32;       // k <= 32 (k + 1 <= 33 candidates per point)
constexpr uint64_t kEmptyKey = ~0ull;

struct Grid {
    double lo[3];
    double h, inv_h;
    int64_t dims[3];
    const uint64_t* hkeys;  // hash table keys (kEmptyKey = empty)
    const uint2* hvals;     // [start, end) into the sorted points
    uint64_t hmask;         // table size - 1 (power of two)
    const double* pts;      // (m, 3) sorted by cell
};

constexpr int kKnnLevels = 8;  // grid levels, each 16x coarser
#ifndef RCGS_KNN_MAX_SHELL
#define RCGS_KNN_MAX_SHELL 3
#endif
constexpr int kKnnMaxShell = RCGS_KNN_MAX_SHELL;  // shells searched per level before moving one level up

struct Grids {
    Grid lv[kKnnLevels];
    int n;
};

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

__device__ __forceinline__ int64_t cell_of(double x, double lo, double inv_h, int64_t dim) {
    int64_t c = (int64_t)floor((x - lo) * inv_h);
    return c < 0 ? 0 : (c >= dim ? dim - 1 : c);
}

__device__ __forceinline__ uint64_t cell_key(int64_t cx, int64_t cy, int64_t cz, const int64_t* dims) {
    return ((uint64_t)cx * (uint64_t)dims[1] + (uint64_t)cy) * (uint64_t)dims[2] + (uint64_t)cz;
}

__global__ void knn_bbox_kernel(const double* __restrict__ pts, int64_t m, unsigned long long* __restrict__ mm) {
    // mm[0..2] = min, mm[3..5] = max, as order-preserving uint64 images of the doubles
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
        for (int d = 0; d < 3; ++d) {
            const double v = pts[3 * i + d];
            lo[d] = fmin(lo[d], v);
            hi[d] = fmax(hi[d], v);
        }
    auto ord = [](double v) -> unsigned long long {  // monotone map double -> uint64
        const unsigned long long b = (unsigned long long)__double_as_longlong(v);
        return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    };
    for (int d = 0; d < 3; ++d) {
        unsigned long long a = ord(lo[d]), b = ord(hi[d]);
        for (int o = 16; o > 0; o >>= 1) {
            a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&mm[d], a);
            atomicMax(&mm[3 + d], b);
        }
    }
}

__global__ void knn_keys_kernel(const double* __restrict__ pts, int64_t m, Grid g, uint64_t* __restrict__ keys) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int64_t cx = cell_of(pts[3 * i], g.lo[0], g.inv_h, g.dims[0]);
    const int64_t cy = cell_of(pts[3 * i + 1], g.lo[1], g.inv_h, g.dims[1]);
    const int64_t cz = cell_of(pts[3 * i + 2], g.lo[2], g.inv_h, g.dims[2]);
    keys[i] = cell_key(cx, cy, cz, g.dims);
}

// sorted point coordinates + one hash entry per cell (run of equal keys)
__global__ void knn_cells_kernel(const double* __restrict__ pts, const uint64_t* __restrict__ keys,
                                 const uint32_t* __restrict__ order, int64_t m, double* __restrict__ spts,
                                 uint64_t* __restrict__ hkeys, uint2* __restrict__ hvals, uint64_t hmask) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint32_t o = order[i];
    spts[3 * i] = pts[3 * (int64_t)o];
    spts[3 * i + 1] = pts[3 * (int64_t)o + 1];
    spts[3 * i + 2] = pts[3 * (int64_t)o + 2];
    const uint64_t k = keys[i];
    if (i > 0 && keys[i - 1] == k) return;  // not the first point of its cell
    for (uint64_t slot = mix64(k) & hmask;; slot = (slot + 1) & hmask) {
        const unsigned long long prev = atomicCAS((unsigned long long*)&hkeys[slot], kEmptyKey, k);
        if (prev == kEmptyKey || prev == k) {
            hvals[slot].x = (uint32_t)i;  // the end is filled by knn_ends_kernel
            break;
        }
    }
}

// the last point of each cell completes its hash entry: end = index + 1
__global__ void knn_ends_kernel(const uint64_t* __restrict__ keys, int64_t m, const uint64_t* __restrict__ hkeys,
                                uint2* __restrict__ hvals, uint64_t hmask) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint64_t k = keys[i];
    if (i + 1 < m && keys[i + 1] == k) return;
    for (uint64_t slot = mix64(k) & hmask;; slot = (slot + 1) & hmask)
        if (hkeys[slot] == k) {
            hvals[slot].y = (uint32_t)(i + 1);
            break;
        }
}

__device__ __forceinline__ uint2 lookup(const Grid& g, uint64_t k) {
    for (uint64_t slot = mix64(k) & g.hmask;; slot = (slot + 1) & g.hmask) {
        const uint64_t s = g.hkeys[slot];
        if (s == k) return g.hvals[slot];
        if (s == kEmptyKey) return make_uint2(0u, 0u);
    }
}

// Exact (k+1)-NN squared distances of point p (ascending in best[0..kp1)) on one
// grid level, searching at most `max_shell` Chebyshev shells (-1: unbounded);
// false if the search had to stop before it could prove the result.
template <int KP1, bool kExact>
__device__ __forceinline__ bool knn_level(const Grid& g, double px, double py, double pz, int kp1_rt,
                                          int64_t max_shell, double* best) {
    const int kp1 = kExact ? KP1 : kp1_rt;  // kExact: compile-time indices (registers)
#pragma unroll
    for (int j = 0; j < KP1; ++j) best[j] = INFINITY;
    const int64_t c[3] = {cell_of(px, g.lo[0], g.inv_h, g.dims[0]), cell_of(py, g.lo[1], g.inv_h, g.dims[1]),
                          cell_of(pz, g.lo[2], g.inv_h, g.dims[2])};
    const double p[3] = {px, py, pz};
    int found = 0;
    for (int64_t R = 0;; ++R) {
        if (max_shell >= 0 && R > max_shell) return false;
        for (int64_t dx = -R; dx <= R; ++dx) {
            const int64_t cx = c[0] + dx;
            if (cx < 0 || cx >= g.dims[0]) continue;
            for (int64_t dy = -R; dy <= R; ++dy) {
                const int64_t cy = c[1] + dy;
                if (cy < 0 || cy >= g.dims[1]) continue;
                const bool edge_xy = (dx == -R || dx == R || dy == -R || dy == R);
                for (int64_t dz = -R; dz <= R; dz += (edge_xy ? 1 : (R > 0 ? 2 * R : 1))) {
                    const int64_t cz = c[2] + dz;
                    if (cz < 0 || cz >= g.dims[2]) continue;
                    const uint2 run = lookup(g, cell_key(cx, cy, cz, g.dims));
                    for (uint32_t q = run.x; q < run.y; ++q) {
                        const double ddx = __dsub_rn(g.pts[3 * (int64_t)q], px);
                        const double ddy = __dsub_rn(g.pts[3 * (int64_t)q + 1], py);
                        const double ddz = __dsub_rn(g.pts[3 * (int64_t)q + 2], pz);
                        const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(ddx, ddx), __dmul_rn(ddy, ddy)),
                                                    __dmul_rn(ddz, ddz));
                        if (d2 < best[kp1 - 1]) {  // insert (ascending)
                            double v = d2;
#pragma unroll
                            for (int j = 0; j < KP1; ++j) {
                                if (j < kp1 && v < best[j]) {
                                    const double t = best[j];
                                    best[j] = v;
                                    v = t;
                                }
                            }
                            ++found;
                        }
                    }
                }
            }
        }
        // every point outside the searched cube is at least `bound` away
        double bound = INFINITY;
        bool covers_all = true;
        for (int d = 0; d < 3; ++d) {
            const int64_t lo_c = c[d] - R, hi_c = c[d] + R + 1;
            if (lo_c > 0) {
                bound = fmin(bound, p[d] - (g.lo[d] + (double)lo_c * g.h));
                covers_all = false;
            }
            if (hi_c < g.dims[d]) {
                bound = fmin(bound, (g.lo[d] + (double)hi_c * g.h) - p[d]);
                covers_all = false;
            }
        }
        if (covers_all) return true;
        // conservative by a relative 1e-12 against the rounding of the bound
        const double b = fmax(bound * (1.0 - 1e-12), 0.0);
        if (found >= kp1 && best[kp1 - 1] <= b * b) return true;
    }
}

// Over the levels: a point whose neighbours lie beyond a few shells of the fine
// grid (an isolated outlier) restarts on the next coarser grid; the coarsest
// level (a few cells) is searched without a shell limit.
template <int KP1, bool kExact>
__device__ __forceinline__ void knn_query(const Grids& gs, double px, double py, double pz, int kp1,
                                          double* best) {
    for (int l = 0; l < gs.n; ++l)
        if (knn_level<KP1, kExact>(gs.lv[l], px, py, pz, kp1, l + 1 < gs.n ? kKnnMaxShell : -1, best)) return;
}

// (k+1)-NN squared radius of every `stride`-th sorted point (cell-size sample)
template <int KP1, bool kExact>
__global__ void knn_sample_kernel(Grids gs, int64_t ns, int64_t stride, int k, double* __restrict__ radius2) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ns) return;
    const int64_t q = i * stride;
    const double* pt = gs.lv[0].pts;
    double best[KP1];
    knn_query<KP1, kExact>(gs, pt[3 * q], pt[3 * q + 1], pt[3 * q + 2], k + 1, best);
    radius2[i] = best[kExact ? KP1 - 1 : k];
}

template <int KP1, bool kExact>
__global__ void knn_query_kernel(Grids gs, int64_t m, int k_rt, const uint32_t* __restrict__ order,
                                 double* __restrict__ means) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int k = kExact ? KP1 - 1 : k_rt;
    const double* pt = gs.lv[0].pts;
    double best[KP1];
    knn_query<KP1, kExact>(gs, pt[3 * i], pt[3 * i + 1], pt[3 * i + 2], k + 1, best);
    // distances 1..k ascending, numpy pairwise sum, / k
    double dv[KP1 - 1];
#pragma unroll
    for (int j = 0; j < KP1 - 1; ++j) dv[j] = j < k ? __dsqrt_rn(best[j + 1]) : 0.0;
    double s;
    if (k < 8) {
        s = 0.0;
        for (int j = 0; j < k; ++j) s = __dadd_rn(s, dv[j]);
    } else {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = dv[j];
        int j = 8;
        for (; j + 8 <= k; j += 8)
#pragma unroll
            for (int t = 0; t < 8; ++t) r[t] = __dadd_rn(r[t], dv[j + t]);
        s = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                      __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; j < k; ++j) s = __dadd_rn(s, dv[j]);
    }
    means[order[i]] = __ddiv_rn(s, (double)k);
}

}  // namespace rcgs

using namespace rcgs;

namespace {

int build_grid(const double* d_pts, int64_t m, double h, const double lo[3], const double hi[3], cudaStream_t s,
               Grid* g, uint32_t** order_out, double** spts_out, uint64_t** hkeys_out, uint2** hvals_out) {
    g->h = h;
    g->inv_h = 1.0 / h;
    uint64_t cells = 1;
    for (int d = 0; d < 3; ++d) {
        g->lo[d] = lo[d];
        g->dims[d] = (int64_t)floor((hi[d] - lo[d]) / h) + 1;
        cells *= (uint64_t)g->dims[d];
    }
    RCGS_CHECK_ARG(cells < (1ull << 62), "kNN grid too fine");
    int bits = 1;
    while (bits < 64 && (1ull << bits) < cells) ++bits;
    uint64_t *keys = nullptr, *keys_alt = nullptr;
    uint32_t *order = nullptr, *order_alt = nullptr;
    RCGS_TRY(dalloc(&keys, m, s));
    RCGS_TRY(dalloc(&keys_alt, m, s));
    RCGS_TRY(dalloc(&order, m, s));
    RCGS_TRY(dalloc(&order_alt, m, s));
    knn_keys_kernel<<<div_up(m, 256), 256, 0, s>>>(d_pts, m, *g, keys);
    RCGS_LAUNCH_CHECK();
    RCGS_TRY(radix_sort_u64(&keys, &keys_alt, &order, &order_alt, true, m, bits, s));
    uint64_t tsize = 1;
    while (tsize < 2 * (uint64_t)m) tsize <<= 1;
    double* spts = nullptr;
    uint64_t* hkeys = nullptr;
    uint2* hvals = nullptr;
    RCGS_TRY(dalloc(&spts, 3 * m, s));
    RCGS_TRY(dalloc(&hkeys, (int64_t)tsize, s));
    RCGS_TRY(dalloc(&hvals, (int64_t)tsize, s));
    RCGS_CUDA(cudaMemsetAsync(hkeys, 0xff, tsize * sizeof(uint64_t), s));
    knn_cells_kernel<<<div_up(m, 256), 256, 0, s>>>(d_pts, keys, order, m, spts, hkeys, hvals, tsize - 1);
    knn_ends_kernel<<<div_up(m, 256), 256, 0, s>>>(keys, m, hkeys, hvals, tsize - 1);
    RCGS_LAUNCH_CHECK();
    dfree(keys, s);
    dfree(keys_alt, s);
    dfree(order_alt, s);
    g->hkeys = hkeys;
    g->hvals = hvals;
    g->hmask = tsize - 1;
    g->pts = spts;
    *order_out = order;
    *spts_out = spts;
    *hkeys_out = hkeys;
    *hvals_out = hvals;
    return RCGS_OK;
}

void free_grid(cudaStream_t s, uint32_t* order, double* spts, uint64_t* hkeys, uint2* hvals) {
    dfree(order, s);
    dfree(spts, s);
    dfree(hkeys, s);
    dfree(hvals, s);
}

struct LevelBufs {
    uint32_t* order[kKnnLevels];
    double* spts[kKnnLevels];
    uint64_t* hk[kKnnLevels];
    uint2* hv[kKnnLevels];
};

// grid levels h, 16 h, 256 h, ... up to one of at most 2 cells per dimension
int build_levels(const double* d_pts, int64_t m, double h, const double lo[3], const double hi[3], double ext,
                 cudaStream_t s, Grids* gs, LevelBufs* b) {
    gs->n = 0;
    double hl = h;
    for (int l = 0; l < kKnnLevels; ++l) {
        if (l == kKnnLevels - 1) hl = fmax(hl, ext);  // the last level must be coarse
        RCGS_TRY(build_grid(d_pts, m, hl, lo, hi, s, &gs->lv[l], &b->order[l], &b->spts[l], &b->hk[l], &b->hv[l]));
        gs->n = l + 1;
        if (gs->lv[l].dims[0] <= 2 && gs->lv[l].dims[1] <= 2 && gs->lv[l].dims[2] <= 2) break;
        hl *= 16.0;
    }
    return RCGS_OK;
}

void free_levels(cudaStream_t s, const Grids& gs, LevelBufs* b) {
    for (int l = 0; l < gs.n; ++l) free_grid(s, b->order[l], b->spts[l], b->hk[l], b->hv[l]);
}

int run_query(const Grids& gs, int64_t m, int k, const uint32_t* order, double* means, cudaStream_t s) {
    if (k == 16)  // the reference default (DEFAULT_KNN): all indices compile-time
        knn_query_kernel<17, true><<<div_up(m, 128), 128, 0, s>>>(gs, m, k, order, means);
    else
        knn_query_kernel<kKnnMaxK + 1, false><<<div_up(m, 128), 128, 0, s>>>(gs, m, k, order, means);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

int run_sample(const Grids& gs, int64_t ns, int64_t stride, int k, double* r2, cudaStream_t s) {
    if (k == 16)
        knn_sample_kernel<17, true><<<div_up(ns, 128), 128, 0, s>>>(gs, ns, stride, k, r2);
    else
        knn_sample_kernel<kKnnMaxK + 1, false><<<div_up(ns, 128), 128, 0, s>>>(gs, ns, stride, k, r2);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

}  // namespace

extern "C" int rcgs_knn_mean_distances(const double* d_points, int64_t m, int32_t k, double* d_means,
                                       void* stream) {
    RCGS_CHECK_ARG(d_points != nullptr && d_means != nullptr, "null argument");
    RCGS_CHECK_ARG(k >= 1 && k <= kKnnMaxK, "k must be in [1, %d]", kKnnMaxK);
    RCGS_CHECK_ARG(m > k, "need more than k = %d points, got %lld", k, (long long)m);
    RCGS_CHECK_ARG(m < (1ll << 31), "too many points");
    cudaStream_t s = as_stream(stream);
    // ---- bounding box
    unsigned long long* mm = nullptr;
    RCGS_TRY(dalloc(&mm, 6, s));
    {
        unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
        RCGS_CUDA(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, s));
    }
    knn_bbox_kernel<<<(int)(div_up(m, 256) < 1184 ? div_up(m, 256) : 1184), 256, 0, s>>>(d_points, m, mm);
    RCGS_LAUNCH_CHECK();
    unsigned long long hmm[6];
    RCGS_CUDA(cudaMemcpyAsync(hmm, mm, sizeof(hmm), cudaMemcpyDeviceToHost, s));
    RCGS_CUDA(cudaStreamSynchronize(s));
    dfree(mm, s);
    double lo[3], hi[3];
    for (int d = 0; d < 3; ++d) {
        auto un = [](unsigned long long u) {
            const unsigned long long b = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
            double v;
            memcpy(&v, &b, sizeof(v));
            return v;
        };
        lo[d] = un(hmm[d]);
        hi[d] = un(hmm[3 + d]);
        RCGS_CHECK_ARG(std::isfinite(lo[d]) && std::isfinite(hi[d]), "non-finite points");
    }
    double ext = 0.0;
    for (int d = 0; d < 3; ++d) ext = fmax(ext, hi[d] - lo[d]);
    if (ext <= 0.0) ext = 1.0;
    // ---- pass 1: coarse grid (~8 points per cell if the cloud filled its box), the
    // exact (k+1)-NN radius of a sample of points -> cell size ~ that radius
    double h = ext / fmax(1.0, cbrt((double)m / 8.0));
    {
        Grids gs;
        LevelBufs b;
        RCGS_TRY(build_levels(d_points, m, h, lo, hi, ext, s, &gs, &b));
        const int64_t ns = m < 1024 ? m : 1024;
        double* r2 = nullptr;
        RCGS_TRY(dalloc(&r2, ns, s));
        RCGS_TRY(run_sample(gs, ns, m / ns, k, r2, s));
        std::vector<double> hr2(ns);
        RCGS_CUDA(cudaMemcpyAsync(hr2.data(), r2, sizeof(double) * ns, cudaMemcpyDeviceToHost, s));
        RCGS_CUDA(cudaStreamSynchronize(s));
        dfree(r2, s);
        free_levels(s, gs, &b);
        std::nth_element(hr2.begin(), hr2.begin() + ns / 2, hr2.end());
        const double r = sqrt(hr2[ns / 2]);
        if (r > 0.0 && std::isfinite(r)) h = fmax(r / 1.5, ext * 1e-6);  // <= 1e6 cells per dimension
    }
    // ---- pass 2: the exact query over all points
    const bool dbg = getenv("RCGS_KNN_DEBUG") != nullptr;
    cudaEvent_t e0, e1, e2;
    if (dbg) {
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventCreate(&e2);
        cudaEventRecord(e0, s);
    }
    Grids gs;
    LevelBufs b;
    RCGS_TRY(build_levels(d_points, m, h, lo, hi, ext, s, &gs, &b));
    if (dbg) cudaEventRecord(e1, s);
    RCGS_TRY(run_query(gs, m, k, b.order[0], d_means, s));
    if (dbg) {
        cudaEventRecord(e2, s);
        cudaEventSynchronize(e2);
        float t1 = 0, t2 = 0;
        cudaEventElapsedTime(&t1, e0, e1);
        cudaEventElapsedTime(&t2, e1, e2);
        fprintf(stderr, "knn: m %lld h %.3g levels %d dims0 %lld %lld %lld build %.2f ms query %.2f ms\n",
                (long long)m, h, gs.n, (long long)gs.lv[0].dims[0], (long long)gs.lv[0].dims[1],
                (long long)gs.lv[0].dims[2], t1, t2);
    }
    free_levels(s, gs, &b);
    return RCGS_OK;
}

// Shared helpers for the rcgs CUDA library (sm_100a).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdlib>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/rcgs.h"

namespace rcgs {

constexpr int kTile = 16;                 // 16x16 pixel tiles, one CTA each
constexpr int kTilePixels = kTile * kTile;

void set_error(const char* fmt, ...);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define RCGS_CHECK_ARG(cond, ...)          \
    do {                                   \
        if (!(cond)) {                     \
            ::rcgs::set_error(__VA_ARGS__); \
            return RCGS_EINVAL;            \
        }                                  \
    } while (0)

#define RCGS_CUDA(call)                                                                   \
    do {                                                                                  \
        cudaError_t err__ = (call);                                                       \
        if (err__ != cudaSuccess) {                                                       \
            ::rcgs::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,                  \
                              cudaGetErrorString(err__));                                 \
            return RCGS_ECUDA;                                                            \
        }                                                                                 \
    } while (0)

#define RCGS_LAUNCH_CHECK() RCGS_CUDA(cudaGetLastError())

#define RCGS_TRY(expr)               \
    do {                             \
        int st__ = (expr);           \
        if (st__ != RCGS_OK) return st__; \
    } while (0)

inline unsigned div_up(int64_t a, int64_t b) { return static_cast<unsigned>((a + b - 1) / b); }

// CTAs per SM a persistent main-stream kernel (raster, record streaming, Adam)
// launches: its occupancy limit minus RCGS_PERSIST_RESERVE (default 0), so that
// the side-stream view build finds free CTA slots instead of queueing behind it.
inline int persistent_ctas(int per_sm) {
    static const int reserve = [] {
        const char* e = getenv("RCGS_PERSIST_RESERVE");
        return e ? atoi(e) : 0;
    }();
    const int c = per_sm - reserve;
    return c > 0 ? c : 1;
}

// Keep freed blocks in the device's default pool across stream syncs (the
// default release threshold of 0 returns memory to the driver at every sync,
// which turns each per-view allocation into a map/unmap).
void retain_pool_memory();

// Stream-ordered device allocation from the default memory pool.
template <typename T>
int dalloc(T** p, size_t count, cudaStream_t s) {
    retain_pool_memory();
    *p = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(p), count * sizeof(T), s);
    if (e != cudaSuccess) {
        set_error("cudaMallocAsync(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
        return RCGS_ENOMEM;
    }
    return RCGS_OK;
}

template <typename T>
void dfree(T*& p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
}

// Grow the stream-ordered pool to hold `bytes` (allocate + free) so later
// allocations do not map new physical memory on the timed path.
int pool_reserve(int64_t bytes, cudaStream_t s);

// A zeroed device counter owned by stream `s` (created on first use, never freed),
// for last-block tickets: launches on different streams never share one.
unsigned* stream_ticket(cudaStream_t s);

// Pinned scratch for small device->host readbacks (per thread).
void* pinned_scratch(size_t bytes);

// ---- device scan / radix sort (scan.cu, radix.cu) -------------------------------
// Exclusive scan of n uint32 counts into out (n+1 entries; out[n] = total).
int exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, cudaStream_t s);
// Stable LSD radix sort of (key, value) pairs over key bits [0, end_bit).
// keys/vals are double-buffered: on return *key_cur / *val_cur point at the sorted data.
// vals_in may be null: values then start as the element index.
int radix_sort_u64(uint64_t** key_cur, uint64_t** key_alt, uint32_t** val_cur, uint32_t** val_alt,
                   bool vals_are_index, int64_t n, int end_bit, cudaStream_t s);
void release_records(rcgs_view* v, cudaStream_t s);  // raster.cu: drop or free the view's weight records

int radix_sort_u32(uint32_t** key_cur, uint32_t** key_alt, uint32_t** val_cur, uint32_t** val_alt,
                   bool vals_are_index, int64_t n, int end_bit, cudaStream_t s);

// ---- checked builds (compute-sanitizer is unavailable on this pool) --------------
// `make EXTRA=-DRCGS_CHECKED ...` compiles device-side bound checks on the computed
// indices of the hot kernels (pair / record / scene / sort-destination indices):
// a failed check increments a device counter (no trap, so a bad index is counted,
// not fatal) that rcgs_debug_violations() reads.  Release builds compile them out.
#ifdef RCGS_CHECKED
// one counter per translation unit (no relocatable device code), each TU's host
// reader registered at load time; rcgs_debug_violations sums them
static __device__ unsigned long long g_rcgs_violations = 0;
void register_violation_reader(unsigned long long (*fn)(bool reset));
namespace {
unsigned long long read_violations_tu(bool reset) {
    unsigned long long v = 0;
    cudaMemcpyFromSymbol(&v, g_rcgs_violations, sizeof(v));
    if (reset) {
        const unsigned long long zero = 0;
        cudaMemcpyToSymbol(g_rcgs_violations, &zero, sizeof(zero));
    }
    return v;
}
struct ViolationReg {
    ViolationReg() { register_violation_reader(&read_violations_tu); }
};
static ViolationReg g_violation_reg;
}  // namespace
#define RCGS_DCHECK(cond)                                          \
    do {                                                           \
        if (!(cond)) atomicAdd(&::rcgs::g_rcgs_violations, 1ull); \
    } while (0)
#else
#define RCGS_DCHECK(cond) \
    do {                  \
    } while (0)
#endif

// ---- small device math ----------------------------------------------------------
// world->camera transform exactly as numpy/OpenBLAS evaluates P @ R.T + t
// (oracle/c/rcgs_oracle.c restates it).
__device__ __forceinline__ double cam_coord(const double* R, const double* t, int k, double p0,
                                            double p1, double p2) {
    return __dadd_rn(__fma_rn(p2, R[3 * k + 2], __fma_rn(p1, R[3 * k + 1], __dmul_rn(p0, R[3 * k + 0]))),
                     t[k]);
}

}  // namespace rcgs

// The opaque handles (shared between translation units).
struct rcgs_scene {
    int64_t n;
    int sh_degree;
    double* pos;     // (n,3)
    double* cov3d;   // (n,6): xx, xy, xz, yy, yz, zz
    double* opac;    // (n,)
};

// Raster record of one kept gaussian (rank s), fp32, 48 bytes.  `a` alone is the
// 16-byte cull record (mean + footprint half extents) the raster tests first.
// Powers are in log2 units: power2 = log2(e) * power (render.py:265-269), so
// alpha = op * 2^power2 = 2^(power2 + log2 op).
struct __align__(16) RasterRec {
    float4 a;  // mx_hi, my_hi, half2(ex, ey) bits, log2(opacity)
    float4 b;  // mx_lo, my_lo, p_lo, p_hi     (mean2d = hi + lo; alpha is exactly 0 in fp64 if
               //                               the fp32 power2 < p_lo; [p_lo, p_hi) brackets the gate)
    float4 c;  // nA, nB, nC, 0                 (power2 = nA dx^2 + nB dx dy + nC dy^2 with
               //                                nA = -a/2 log2 e, nB = -b log2 e, nC = -c/2 log2 e)
};

// 8-bit mask of the 8x4 pixel blocks (bit = (y / 4) * 2 + x / 8 within the 16x16
// tile whose top-left pixel is (tx0, ty0)) that the footprint {power2 >= p_lo} of
// record r can reach: the per-block cull of the raster, done once per (gaussian,
// tile) pair at view build.  Q = -power2 = A dx^2 + B dx dy + C dy^2 (PD); for
// each 4-row block row the footprint's x extent over that row band is exact in
// closed form (x_r(dy) concave with its maximiser at dy = -B sqrt(T / (C D)),
// x_l convex, D = 4AC - B^2), compared with the two 8-column blocks.  The
// result must be a superset of the blocks where some pixel has fp64 alpha at or
// above the gate, so every rounding is covered with wide margins: T is raised
// by the cull's evaluation bound (2e-6 of the absolute term sum, which is at
// most (1 + r) / (1 - r) times Q for r = |B| / (2 sqrt(AC)), plus 2e-4 >= the
// raster's 1.5e-4), the extents are widened by 1e-3 relative + 0.02 px, the row
// bands by 0.01 px; near-degenerate footprints (r >= 0.999) and NaN take every
// block.  The raster's checked build re-tests every dropped (entry, block)
// against its exact per-block test.
// Tile-list values: scene index in the low kIdxBits bits and the pair's 8-bit
// block mask above them (scenes below 2^24 gaussians; larger scenes keep plain
// indices and a separate mask array).
constexpr int kIdxBits = 24;
constexpr uint32_t kIdxMask = (1u << kIdxBits) - 1u;

__device__ __forceinline__ float approx_sqrt(float x) {  // MUFU; relative error ~1e-7, x >= 0
    x = fmaxf(x, 1e-30f);
    return x * rsqrtf(x);
}
// Per-gaussian part of the block-mask test (view build, once per kept gaussian):
// m0 = (mx, my, ey, dR), m1 = (B, D, 4AT, 1/(2A)); ey < 0 encodes the special
// cases (-1: every block, -2: none).
struct MaskRec {
    float4 m0, m1;
};

__device__ __forceinline__ MaskRec mask_setup(const float4 ra, const float4 rb, const float4 rc) {
    MaskRec q;
    q.m0 = make_float4(0.f, 0.f, -1.f, 0.f);
    q.m1 = make_float4(0.f, 0.f, 0.f, 0.f);
    const float A = -rc.x, B = -rc.y, C = -rc.z, T0 = -rb.z;
    if (!(A > 0.f && C > 0.f)) return q;
    const float r = fabsf(B) * rsqrtf(4.f * A * C);
    if (!(r < 0.999f) || !(T0 == T0)) return q;
    const float T = T0 + fabsf(T0) * fmaf(2e-6f, __fdividef(1.f + r, 1.f - r), 1e-5f) + 2e-4f;
    if (T < 0.f) {
        q.m0.z = -2.f;
        return q;
    }
    const float D = fmaf(4.f * A, C, -B * B);
    const float AT4 = 4.f * A * T;
    const float ey = approx_sqrt(__fdividef(AT4, D)) * 1.0001f;  // |dy| reach
    const float kq = approx_sqrt(__fdividef(T, C * D));
    q.m0 = make_float4(ra.x + rb.x, ra.y + rb.y, ey, -B * kq);  // dR: maximiser of x_r (x_l: -dR)
    q.m1 = make_float4(B, D, AT4, __fdividef(0.5f, A));
    return q;
}

__device__ __forceinline__ uint32_t tile_block_mask(const MaskRec& q, float tx0, float ty0) {
    const float mx = q.m0.x, my = q.m0.y, ey = q.m0.z, dR = q.m0.w;
    const float B = q.m1.x, D = q.m1.y, AT4 = q.m1.z, inv2A = q.m1.w;
    if (ey < 0.f) return ey == -1.f ? 0xffu : 0u;
    const float dt0 = (ty0 - 0.01f) - my;
    if (dt0 > ey || dt0 + 15.02f < -ey) return 0u;  // no row of the tile in reach
    uint32_t mask = 0u;
#pragma unroll
    for (int by = 0; by < 4; ++by) {
        const float lo = fmaxf(dt0 + 4.f * by, -ey), hi = fminf(dt0 + (4.f * by + 3.02f), ey);
        if (lo > hi) continue;
        const float dr = fminf(fmaxf(dR, lo), hi), dl = fminf(fmaxf(-dR, lo), hi);
        const float xr = (-B * dr + approx_sqrt(fmaf(-D * dr, dr, AT4))) * inv2A;
        const float xl = (-B * dl - approx_sqrt(fmaf(-D * dl, dl, AT4))) * inv2A;
        const float m = fmaf(1e-3f, fabsf(xl) + fabsf(xr), 0.02f);
        const float X0 = (mx + xl) - m, X1 = (mx + xr) + m;
        if (!(X1 < tx0 || X0 > tx0 + 7.f)) mask |= 1u << (2 * by);
        if (!(X1 < tx0 + 8.f || X0 > tx0 + 15.f)) mask |= 2u << (2 * by);
    }
    return mask;
}

__device__ __forceinline__ uint32_t tile_block_mask(const float4 ra, const float4 rb, const float4 rc, float tx0,
                                                    float ty0) {
    return tile_block_mask(mask_setup(ra, rb, rc), tx0, ty0);
}

// Does the cull record's footprint box touch the 8x4 block at (bx0, by0)?
__device__ __forceinline__ bool touches_block(const float4 ra, float bx0, float by0) {
    const unsigned packed = __float_as_uint(ra.z);
    const float ex = __half2float(__ushort_as_half((unsigned short)(packed & 0xffffu)));
    const float ey = __half2float(__ushort_as_half((unsigned short)(packed >> 16)));
    return ra.x + ex >= bx0 && ra.x - ex <= bx0 + 7.f && ra.y + ey >= by0 && ra.y - ey <= by0 + 3.f;
}

// Can the footprint {power2 >= p_lo} reach any point of the rectangle
// [x0, x1] x [y0, y1]?  Q = -power2 is a PSD quadratic of the offset from the
// mean; its minimum over the box is 0 when the mean is inside, else it lies on
// an edge, where the 1-D minimiser is a clamp.  The candidates' fp32 values are
// lowered by their evaluation error bound (2e-6 of the absolute term sum, plus
// 1.5e-4 = 1e-4 natural-log units), so the test only drops entries whose power
// stays below the gate at every pixel of the rectangle -- alpha exactly 0 in
// fp64 there -- and the results do not change.  NaN keeps the entry.
__device__ __forceinline__ bool ellipse_touches_rect(const float4 ra, const float4 rb, const float4 rc, float x0,
                                                     float y0, float x1, float y1) {
    const float X0 = (x0 - ra.x) - rb.x, X1 = (x1 - ra.x) - rb.x;
    const float Y0 = (y0 - ra.y) - rb.y, Y1 = (y1 - ra.y) - rb.y;
    if (X0 <= 0.f && X1 >= 0.f && Y0 <= 0.f && Y1 >= 0.f) return true;
    const float A = -rc.x, B = -rc.y, C = -rc.z;
    const float hA = __fdividef(-0.5f * B, A), hC = __fdividef(-0.5f * B, C);
    auto lower = [&](float dx, float dy) {  // lower bound of Q(dx, dy)
        const float xx = A * dx * dx, yy = C * dy * dy, xy = B * dx * dy;
        return (xx + yy + xy) - fmaf(2e-6f, xx + yy + fabsf(xy), 1.5e-4f);
    };
    auto clampf = [](float v, float lo, float hi) { return fminf(fmaxf(v, lo), hi); };
    float m = lower(X0, clampf(hC * X0, Y0, Y1));
    m = fminf(m, lower(X1, clampf(hC * X1, Y0, Y1)));
    m = fminf(m, lower(clampf(hA * Y0, X0, X1), Y0));
    m = fminf(m, lower(clampf(hA * Y1, X0, X1), Y1));
    return !(m > -rb.z);
}

// Exact (fp64) record for guarded decisions: the reference's own operands.
struct ExactRec {
    double mx, my, ca, cb, cc, op;
};

struct rcgs_view {
    const rcgs_scene* scene;
    rcgs_camera cam;
    rcgs_raster_config cfg;
    int64_t n, k, pairs;
    int tiles_x, tiles_y, sort_bits;
    bool full_sort;       // depth order from the full 64-bit keys (fallback path)
    // per kept rank s (front to back)
    uint32_t* gid;        // (k,) scene index g of depth rank s
    // per gaussian, by scene index g (written for kept gaussians only)
    double* z;            // (n,) view-space z (bit-exact reference depth)
    RasterRec* rec;       // (n,)
    ExactRec* exact;      // (n,)
    uint32_t* offs;       // (k+1,) first emission slot of s; offs[k] = pairs
    float4* color;        // (n,) rgb + active bits (as float 0..7) per step
    int32_t* rank_of;     // (n,) s or -1 (culled)
    uint32_t* fix;        // (n + 1,) {count, g...}: gaussians the Adam colour epilogue left to the fp64 fixup
    unsigned long long* acc_fx;  // (3 n,) the backward's fixed-point sums, zeroed at build (off the optimizer's stream)
    bool acc_dirty;              // acc_fx used since it was zeroed (the next backward clears it first)
    // per pair (sorted by tile, then depth)
    uint32_t* pair_g;     // (pairs,) scene index g
    uint32_t* pair_m;     // (pairs,) tile_block_mask of the pair (8x4 blocks its footprint reaches);
                          // null when packed into pair_g (pair_packed: g | mask << kIdxBits)
    bool pair_packed;
    uint2* ranges;        // (tiles,) [start, end)
    uint32_t* tile_order; // (tiles,) tiles by descending entry count (raster work order)
    uint4* tile_meta;     // (tiles,) per work-order position: {tile, range start, range end, 0}
    uint32_t* blist;      // (8 * pairs,) per-block lists: block b of a tile at 8 range.x + b (range.y - range.x)
    uint32_t* bcount;     // (tiles * 8,) their lengths, by work item (8 work position + block)
    unsigned* work;       // (2,) work-item / exited-warp counters of the persistent launches
    // composite-weight records (rcgs_render_train; geometry + camera only), in the
    // process-wide record arena (raster.cu) while this view owns it
    bool wrec_valid;
    bool wrec_owned;      // records copied out of the arena into view-owned memory
    uint64_t wrec_epoch;
    uint32_t* wrec_off;   // (tiles * 8 + 1,) per-block first record (owned records only)
    uint32_t* wrec_n;     // (tiles * 8,) records per 8x4 block
    uint32_t* wrec_s;     // (8 * pairs,) entry (depth rank) per record slot
    float* wrec_w;        // (8 * pairs, 32) pixel weights per record slot
    float* wrec_tf;       // (H * W,) final transmittance
};

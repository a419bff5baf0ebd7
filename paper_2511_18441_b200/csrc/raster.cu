// K3/K4/K6 tile rasteriser family (render.py:263-398, backward.py:22-40).
//
// Work decomposition.  Pairs are binned per 16x16 tile (preprocess.cu); the
// unit of raster work is one 8x4 pixel block of a tile, handled by ONE warp
// (one pixel per lane).  Warps are persistent and independent: each grabs the
// next block from a global counter, walks its tile's depth-sorted list 32
// entries at a time, culls them against the block with the 16-byte cull record
// (mean + fp64-derived footprint half extents, rounded up), compacts the
// survivors into warp-private shared memory (ballot + popc) and composites
// them front to back.  There is no block-wide barrier anywhere, so a warp
// whose block saturates early simply takes the next block.
//
// Reference semantics (render.py:265-292):
//   alpha = min(0.99, sigma * exp(power)); skip alpha < 1/255;
//   stop *before* the first entry whose T * (1 - alpha) < 1e-4.
//
// Numerics.  The fast path is fp32; every discrete decision is made exactly as
// the fp64 reference makes it:
//   * skip:  alpha >= 1/255 <=> power >= P_g.  power32 < p_lo is certainly
//            skipped, >= p_hi certainly kept; in between the fp64 alpha is
//            recomputed with the reference's operation order.
//   * stop / tau crossing: T is tracked in fp32 with a running relative error
//            bound E; if T * (1 +- 2E) straddles the threshold, the pixel's T is
//            recomputed in fp64 from the start of the tile list (exact cumprod)
//            and fp32 T is resynchronised.
// Entries outside the list or culled for a block have alpha < 1/255 at every
// pixel concerned, which the reference multiplies into T as exactly 1.0.
//
// Modes: FWD image, DEPTH (first tau crossing), BWD (SH backward: per entry a
// warp-shuffle sum of g * w, accumulated per gaussian in 2^-50 fixed point with
// integer atomics -- exact and order independent, hence deterministic), HITS
// (mask statistics), CAPTURE (contribution lists).
#include <cuda_fp16.h>

#include <atomic>
#include <mutex>

#include "common.cuh"

namespace rcgs {

// FWDREC: FWD that also records the composite weights (see `WeightRecords`)
// FWDRGBA: FWD into an RGBA8 viewer frame (separate instantiation, so the
// training / image paths keep their lean epilogue)
enum RasterMode { FWD = 0, DEPTH = 1, BWD = 2, HITS = 3, CAP_COUNT = 4, CAP_WRITE = 5, FWDREC = 6, FWDRGBA = 7 };

constexpr int kWarpsPerCTA = 8;
constexpr int kCTA = 32 * kWarpsPerCTA;
#ifndef RCGS_RASTER_MIN_CTAS
#define RCGS_RASTER_MIN_CTAS 4
#endif
constexpr int kMinCTAs = RCGS_RASTER_MIN_CTAS;  // resident CTAs per SM the register budget targets
// raster_kernel CTA shape: warps are independent (persistent, barrier-free), so
// the CTA size only sets how the per-warp staging buffer is addressed.
#ifndef RCGS_RASTER_WARPS
#define RCGS_RASTER_WARPS 8
#endif
constexpr int kRWarps = RCGS_RASTER_WARPS;
constexpr int kRCTA = 32 * kRWarps;
constexpr int kBlocksPerTile = 8;  // 2 x 4 blocks of 8x4 pixels
constexpr float kLog2e = 1.4426950408889634f;
constexpr double kFixScale = 1125899906842624.0;  // 2^50

// round(v * 2^50) to int64: scaling by a power of two is exact in fp32 (|v| < 2^77
// for a finite product here), so the fp32 round-to-nearest conversion equals
// llrint((double)v * 2^50) with two fp32 instructions instead of three fp64 ones
__device__ __forceinline__ long long to_fixed(float v) {
    return __float2ll_rn(v * 1125899906842624.0f);
}

// Where a composited pixel goes: fp32 HWC / CHW image, or an RGBA8 viewer frame
// (layout 2): the selection overlay (1 - s) img + s hl in fp64 where
// overlay[pix] != 0 (session.py:392-402) then rint(clip(x, 0, 1) * 255) with
// opaque alpha (protocol.py image_to_rgba), bit-identical to doing both on the
// host from the same render.
struct PixelOut {
    float bg0, bg1, bg2;
    int layout;  // 0 HWC, 1 CHW, 2 RGBA8
    float* image;
    float* t_final;
    uint8_t* rgba;
    const uint8_t* overlay;
    double ov_keep, ov_add0, ov_add1, ov_add2;  // 1 - s, s * highlight
};

__device__ __forceinline__ uint8_t to_u8(double x) {
    return (uint8_t)__double2int_rn(__dmul_rn(fmin(fmax(x, 0.0), 1.0), 255.0));
}

template <bool kRgba>
__device__ __forceinline__ void write_pixel(const PixelOut& o, int W, int H, int64_t pix, float acc0, float acc1,
                                            float acc2, float T) {
    const float o0 = fmaf(T, o.bg0, acc0), o1 = fmaf(T, o.bg1, acc1), o2 = fmaf(T, o.bg2, acc2);
    if (!kRgba && o.layout == 0) {
        o.image[3 * pix] = o0;
        o.image[3 * pix + 1] = o1;
        o.image[3 * pix + 2] = o2;
    } else if (!kRgba) {
        const int64_t plane = (int64_t)W * H;
        o.image[pix] = o0;
        o.image[plane + pix] = o1;
        o.image[2 * plane + pix] = o2;
    } else {
        double c0 = o0, c1 = o1, c2 = o2;
        if (o.overlay && o.overlay[pix]) {
            c0 = __dadd_rn(__dmul_rn(o.ov_keep, c0), o.ov_add0);
            c1 = __dadd_rn(__dmul_rn(o.ov_keep, c1), o.ov_add1);
            c2 = __dadd_rn(__dmul_rn(o.ov_keep, c2), o.ov_add2);
        }
        reinterpret_cast<uchar4*>(o.rgba)[pix] = make_uchar4(to_u8(c0), to_u8(c1), to_u8(c2), 255);
    }
    if (o.t_final) o.t_final[pix] = T;
}

struct RasterArgs {
    const uint2* ranges;
    const uint32_t* tile_order;  // work order (nullptr: row-major)
    const uint4* tile_meta;      // per work-order position {tile, range} (nullptr: tile_order + ranges)
    const uint32_t* blist;       // per-block lists (block b of the tile at 8 range.x + b len), or null
    const uint32_t* bcount;      // their lengths, by work item (= 8 work position + block)
    const uint32_t* pair_g;  // tile lists: scene indices in depth order
    const uint32_t* pair_m;  // per list entry: 8x4 blocks of its tile the footprint reaches
                             // (null: packed above the scene index in pair_g)
    uint32_t idx_mask;       // scene-index bits of a pair_g value
    const int32_t* rank_of;  // scene index -> depth rank (capture output)
    const RasterRec* rec;
    const ExactRec* exact;
    const float4* color;
    const uint32_t* gid;
    const double* z;
    unsigned* counter;
    int W, H, tiles_x, n_items;
    int64_t n, pairs;  // scene size and tile-list pairs (checked builds' bounds)
    double alpha_clamp, alpha_skip, t_floor, tau;
    float f_alpha_clamp, f_floor, f_tau;
    float f_gate2;  // log2(alpha_skip): the alpha gate in log2 units
    // FWD
    PixelOut out;
    // DEPTH
    int32_t* cross;
    double* depth;
    // BWD
    const float* grad;
    unsigned long long* acc_fx;  // (k, 3) fixed point
    int32_t* nonfinite;
    // optional work counters (instrumented launches only): evaluated pixel-entry
    // pairs, composited pairs, warp blocks processed, warp blocks skipped,
    // warp-level entry iterations
    unsigned long long* counters;
    uint32_t* trace;  // diagnostics: per work item {t0, t1, smid, iters, evals, exact, resync, tile}
    // HITS
    const uint8_t* mask;
    int32_t* hits;
    unsigned long long* wsum;
    // CAPTURE
    uint32_t* cap_count;
    const uint32_t* cap_offs;
    int64_t* cap_pixel;
    int64_t* cap_kept;
    double* cap_weight;
    // FWDREC: weight records (per (tile, block): count; per record: entry, 32 weights)
    uint32_t* wrec_n;
    uint32_t* wrec_s;
    float* wrec_w;
};

// Instrumentation: when set, raster launches accumulate work counters here.
static unsigned long long* g_counters = nullptr;
static uint32_t* g_trace = nullptr;
static int64_t g_trace_items = 0;

__device__ __forceinline__ uint32_t globaltimer_lo() {
    uint32_t t;
    asm volatile("mov.u32 %0, %%globaltimer_lo;" : "=r"(t));
    return t;
}

__device__ __forceinline__ uint32_t smid() {
    uint32_t r;
    asm("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Persistent launches pull work items from ctr[0]; the last warp to exit resets
// ctr[0..1] for the next launch on the view (ctr[1] counts exited warps), so no
// per-launch allocation or memset is needed.
__device__ __forceinline__ void work_counter_exit(unsigned* ctr, int lane) {
    if (lane == 0 && atomicAdd(&ctr[1], 1u) == gridDim.x * (blockDim.x >> 5) - 1) {
        ctr[0] = 0;
        ctr[1] = 0;
    }
}

// Reference alpha in fp64 with numpy's operation order (render.py:265-271).
__device__ __forceinline__ double exact_alpha(const ExactRec& r, double u, double v, double clamp,
                                              double skip) {
    const double dx = __dsub_rn(u, r.mx), dy = __dsub_rn(v, r.my);
    const double t1 = __dmul_rn(__dmul_rn(__dmul_rn(0.5, r.ca), dx), dx);
    const double t2 = __dmul_rn(__dmul_rn(__dmul_rn(0.5, r.cc), dy), dy);
    const double t3 = __dmul_rn(__dmul_rn(r.cb, dx), dy);
    const double power = __dsub_rn(__dsub_rn(-t1, t2), t3);
    const double al = fmin(clamp, __dmul_rn(r.op, exp(power)));
    return al < skip ? 0.0 : al;
}

__device__ __forceinline__ double exact_alpha_at(const ExactRec* __restrict__ exact, uint32_t s, double u,
                                              double v, double clamp, double skip) {
    return exact_alpha(exact[s], u, v, clamp, skip);
}

// fp32 cull power of a record at pixel (uf, vf) -- one expression shared by the
// per-entry step and the exact re-walk, so both make the same gate decision.
__device__ __forceinline__ float cull_power(const float4 ra, const float4 rb, const float4 rc, float uf, float vf) {
    const float dx = (uf - ra.x) - rb.x;
    const float dy = (vf - ra.y) - rb.y;
    return fmaf(rc.x * dx, dx, fmaf(rc.z * dy, dy, rc.y * dx * dy));
}

// Exact inclusive transmittance of pixel (uf, vf) after list entries [j0, j1]
// (np.cumprod, render.py:278), computed by the whole warp.  Entries below the
// gate (power < p_lo: alpha is exactly 0 in fp64, the same test the per-entry
// step trusts) contribute an exact factor 1 and are skipped; the remaining
// (1 - alpha) factors are multiplied in list order, so every fp64 rounding is
// the reference's.  32 lanes x 4 entries in flight per round instead of one
// lane walking up to a few thousand entries with a dependent fp64 exp each
// (those serial re-walks were the launch tail: one warp busy for 0.7 ms).
__device__ __forceinline__ double warp_exact_T(const uint32_t* __restrict__ pair_g,
                                            const RasterRec* __restrict__ rec,
                                            const ExactRec* __restrict__ exact, double clamp, double skip,
                                            uint32_t j0, uint32_t j1, float uf, float vf, int lane,
                                            uint32_t idx_mask) {
    constexpr int kU = 2;
    const double u = (double)uf, v = (double)vf;
    double T = 1.0;
    for (uint32_t c = j0; c <= j1; c += 32 * kU) {
        uint32_t sv[kU];
#pragma unroll
        for (int q = 0; q < kU; ++q) {
            const uint32_t j = c + q * 32 + lane;
            sv[q] = j <= j1 ? pair_g[j] & idx_mask : 0xffffffffu;
        }
        bool live[kU];
#pragma unroll
        for (int q = 0; q < kU; ++q) {
            live[q] = false;
            if (sv[q] != 0xffffffffu) {
                const RasterRec rr = rec[sv[q]];
                live[q] = !(cull_power(rr.a, rr.b, rr.c, uf, vf) < rr.b.z);
            }
        }
#pragma unroll
        for (int q = 0; q < kU; ++q) {
            double om = 1.0;
            if (live[q]) om = __dsub_rn(1.0, exact_alpha(exact[sv[q]], u, v, clamp, skip));
            unsigned m = __ballot_sync(0xffffffffu, om != 1.0);
            while (m) {
                const int b = __ffs(m) - 1;
                T = __dmul_rn(T, __shfl_sync(0xffffffffu, om, b));
                m &= m - 1;
            }
        }
    }
    return T;
}

// One staged (entry, 8x4 block) pair.  The entry's log2 alpha over the block is
// a quadratic in the pixel's offset (lx, ly) from the block centre:
//   P2 = log2(op) + power2 = qA lx^2 + qB lx ly + qC ly^2 + qD lx + qE ly + qF,
// five FMAs per pixel against per-lane constants, with a rigorous absolute
// error bound eps for this block (staging): the alpha >= 1/255 gate is decided
// in fp32 outside [G2 - eps, G2 + eps) (G2 = log2(1/255)) and in fp64 inside;
// delta = relative error bound of the fp32 alpha.
//
// The raw records of the next 32 list entries (and the pair ids of the chunk
// after) stream into per-lane shared slots with cp.async while the warp
// composites the current chunk, so the dependent gathers pair_g -> rec[s] ->
// colour[s] are off the critical path.
struct WarpStage {
    float4 q0[32];  // qA, qB, qC, qD
    float4 q1[32];  // qE, qF, G2 - eps, G2 + eps
    float4 q2[32];  // colour rgb (fwd modes), delta
    uint32_t g[32], j[32];  // entry: scene index, tile-list position
    float4 ra[32], rb[32], rc[32], rcol[32];  // raw records of the next chunk (lane = entry)
    uint32_t pg[2][32];                       // pair ids (scene indices), double-buffered
    uint32_t pm[2][32];                       // their block masks
};

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
                 "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(smem_dst)),
                 "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One composite step of a pixel (render.py:265-292, 389-397): w = alpha T_before;
// fp32 T with its absolute error bound A (A' = A (1 - alpha) + w delta + 2.4e-7 T';
// delta = relative alpha error); the band tests decide stop (and the tau
// crossing for DEPTH) exactly unless ambiguous.  The outcome is carried as
// values: the composited weight (0 if not composited), next T (-T_final once
// stopped: skipped entries keep it, composited ones stop again), next A, and
// the crossing.  `amb`: the fp32 band straddles a threshold.
struct StepOut {
    float wc, Tn, An;
    bool amb, xc;
};

template <int M>
__device__ __forceinline__ StepOut composite_step(float T, float A, bool live, bool pass, float al, float dl,
                                                  float f_floor, float f_tau) {
    // A skipped entry (alpha 0) gives w = 0 and Tk = T exactly; finished lanes
    // (T <= 0) give w = 0 when skipped and otherwise "stop" again (hi <= 0), so
    // one select per output covers every case.
    StepOut o;
    const float oma = 1.f - al;  // >= 0.01 (alpha clamp)
    const float w = al * T, Tk = T * oma;
    const float Ak = fmaf(A, oma, fmaf(w, dl, 2.4e-7f * Tk));
    const float lo = fmaf(-2.f, Ak, Tk), hi = fmaf(2.f, Ak, Tk);
    const bool stop = pass && hi < f_floor;
    bool amb = pass && !stop && !(lo >= f_floor), xcross = false;
    if (M == DEPTH) {
        xcross = live && pass && hi < f_tau;
        amb = amb || (live && pass && !xcross && !(lo >= f_tau));
    }
    o.wc = stop ? 0.f : w;  // finished lanes: w = 0 (skip) or they stop again
    o.Tn = stop ? fminf(T, -T) : (xcross ? 0.f : Tk);
    o.An = (stop || xcross) ? 0.f : Ak;
    o.amb = amb;
    o.xc = xcross;
    return o;
}

// The slow path of one entry, called by the whole warp (out of line, so the
// fast loop keeps its registers and stays convergent): the exact fp64 alpha for
// the lanes whose fp32 log2 alpha fell in the gate band, then the exact
// transmittance (warp re-walk of the tile list prefix) for every lane whose
// threshold test is ambiguous.  Returns the lane's final outcome; *resync
// counts the re-walks.
struct SlowOut {
    StepOut o;
    uint32_t resync;
};

template <int M>
__device__ __noinline__ SlowOut slow_entry(const uint32_t* __restrict__ pair_g, const RasterRec* __restrict__ rec,
                                           const ExactRec* __restrict__ exact, double clamp, double skip,
                                           double t_floor, double tau, float f_floor, float f_tau, uint32_t g,
                                           uint32_t j, uint32_t j0, float uf, float vf, int lane, float T, float A,
                                           bool live, bool pass, bool gamb, float al, float dl, StepOut cur,
                                           uint32_t idx_mask) {
    uint32_t resync = 0;
    if (gamb) {
        const double a64 = exact_alpha_at(exact, g, (double)uf, (double)vf, clamp, skip);
        pass = a64 != 0.0;
        al = (float)a64;
        dl = 1.2e-7f;  // the fp32 rounding of an exact alpha
        cur = composite_step<M>(T, A, live, pass, al, dl, f_floor, f_tau);
    }
    for (unsigned m = __ballot_sync(0xffffffffu, cur.amb); m; m &= m - 1) {
        const int L = __ffs(m) - 1;
        const float lu = __shfl_sync(0xffffffffu, uf, L), lv = __shfl_sync(0xffffffffu, vf, L);
        const double T64 = warp_exact_T(pair_g, rec, exact, clamp, skip, j0, j, lu, lv, lane, idx_mask);
        if (lane == L) {  // the exact decision (render.py:278-291, 389-397)
            const float w = al * T;
            cur.amb = false;
            if (M == DEPTH && T64 < tau) {
                cur.wc = w;
                cur.Tn = 0.f;
                cur.An = 0.f;
                cur.xc = true;
            } else if (T64 < t_floor) {
                cur.wc = 0.f;
                cur.Tn = fminf(T, -T);
                cur.An = 0.f;
            } else {
                cur.wc = w;
                cur.Tn = (float)T64;
                cur.An = 1.2e-7f * cur.Tn;
            }
        }
        ++resync;
    }
    return SlowOut{cur, resync};
}

// kInstr: the instrumented variant (work counters / per-item trace); production
// launches carry no counter registers or checks in the entry loop.
//
// Per (pixel, entry) the fast path is branch-free: skipped entries (alpha 0)
// leave T and the colour exactly unchanged, finished pixels carry T = 0 (their
// output T is kept in Tout), and everything that needs the exact fp64 answer --
// an alpha inside the gate band, or an fp32 transmittance whose error band
// straddles the stop floor (or tau) -- raises one warp vote per entry that sends
// the warp to the slow path for that entry.
#ifndef RCGS_FWDREC_MIN_CTAS
#define RCGS_FWDREC_MIN_CTAS 3
#endif
template <int M, bool kInstr>
__global__ void __launch_bounds__(kRCTA, (M == FWDREC ? RCGS_FWDREC_MIN_CTAS : kMinCTAs) * 8 / kRWarps)
    raster_kernel(RasterArgs a) {
    constexpr bool kFwd = (M == FWD || M == FWDREC || M == FWDRGBA);
    constexpr int kRow = (M == FWDREC || M == FWDRGBA) ? (int)FWD : M;  // counter row
    __shared__ WarpStage stage_all[kRWarps];
    const int lane = threadIdx.x & 31;
    // The warp index comes from a shuffle: ptxas cannot re-derive a shuffle result
    // from threadIdx / the CTA id at every use, so the staging base stays in a
    // register.
    WarpStage& st = stage_all[kRWarps == 1 ? 0 : __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0)];
    const uint32_t lt_mask = (1u << lane) - 1u;
    // pixel offset from the 8x4 block centre (exact small fp32 values)
    const float lxf = (float)(lane & 7) - 3.5f, lyf = (float)(lane >> 3) - 1.5f;
    const float G2 = a.f_gate2;

    // FWDREC (3 CTAs/SM, 80 registers) takes its work items one ahead: the atomic
    // for the next item is in flight while this one is processed (its round trip
    // was ~7% of the warp samples).  At the 64-register budget of the other modes
    // the extra live value made ptxas rematerialise lane constants inside the
    // entry loop (+24%), so they fetch on demand.
    constexpr bool kAhead = M == FWDREC && RCGS_FWDREC_MIN_CTAS <= 3;
    unsigned nraw = 0;
    if (kAhead && lane == 0) nraw = atomicAdd(a.counter, 1u);
    for (;;) {
        unsigned item = 0;
        if (kAhead) {
            item = __shfl_sync(0xffffffffu, nraw, 0);
            if (item >= (unsigned)a.n_items) break;
            if (lane == 0) nraw = atomicAdd(a.counter, 1u);
        } else {
            if (lane == 0) item = atomicAdd(a.counter, 1u);
            item = __shfl_sync(0xffffffffu, item, 0);
            if (item >= (unsigned)a.n_items) break;
        }
        int tile;
        uint2 range;
        if (a.tile_meta) {
            const uint4 tm = a.tile_meta[item / kBlocksPerTile];
            tile = (int)tm.x;
            range = make_uint2(tm.y, tm.z);
        } else {
            tile = a.tile_order ? (int)a.tile_order[item / kBlocksPerTile] : (int)(item / kBlocksPerTile);
            range = a.ranges[tile];
        }
        const int blk = (int)(item % kBlocksPerTile);
        const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
        const int bx0 = tx * kTile + (blk & 1) * 8, by0 = ty * kTile + (blk >> 1) * 4;
        const int u = bx0 + (lane & 7), v = by0 + (lane >> 3);
        const bool inside = u < a.W && v < a.H;
        const int64_t pix = (int64_t)v * a.W + u;

        // T: fp32 transmittance while the pixel composites (T > 0); once it stops,
        // -T_final (T before the stop entry), and 0 for pixels that never composite.
        // A: the absolute error bound of T vs the fp64 product.
        float T = inside ? 1.f : 0.f, A = 0.f;
        uint32_t n_resync = 0;  // warp-uniform (trace launches)
        float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f;
        int32_t cross = -1;
        uint32_t ncap = 0, cap_base = 0;
        float g0 = 0.f, g1 = 0.f, g2 = 0.f;
        if (M == BWD) {
            if (inside) {
                g0 = a.grad[3 * pix];
                g1 = a.grad[3 * pix + 1];
                g2 = a.grad[3 * pix + 2];
            }
            // sum_p g_p w_ip has no term from this block when all its gradients are 0
            // (the recolor gradient is local to the edited region): skip the block
            if (__all_sync(0xffffffffu, g0 == 0.f && g1 == 0.f && g2 == 0.f)) {
                if (kInstr && a.counters && lane == 0) atomicAdd(&a.counters[5 * kRow + 3], 1ull);
                continue;
            }
        }
        if (kInstr && a.trace && lane == 0) a.trace[8 * (int64_t)item] = globaltimer_lo();
        if (M == HITS && inside && a.mask[pix] == 0) T = 0.f;
        if (M == CAP_WRITE && inside) cap_base = a.cap_offs[pix];

        const float fbx0 = (float)bx0, fby0 = (float)by0;
        const float cxf = fbx0 + 3.5f, cyf = fby0 + 1.5f;
        if (kInstr && M == FWDREC && a.counters) {
            // static list-cull statistics for a two-pixels-per-lane raster (8x8
            // regions): entries passing this 8x4 block's cull, and for the top block
            // of each 8x8 region the entries passing the region's cull (row 5 of the
            // counters: [25] block entries, [26] region entries)
            const bool top = ((blk >> 1) & 1) == 0;
            unsigned cb = 0, cu = 0;
            for (uint32_t j = range.x + lane; j < range.y; j += 32) {
                const uint32_t sj = a.pair_g[j] & a.idx_mask;
                const float4 qa = a.rec[sj].a, qb = a.rec[sj].b, qc = a.rec[sj].c;
                cb += touches_block(qa, fbx0, fby0) &&
                      ellipse_touches_rect(qa, qb, qc, fbx0, fby0, fbx0 + 7.f, fby0 + 3.f);
                if (top) {
                    const unsigned pk = __float_as_uint(qa.z);
                    const float ex = __half2float(__ushort_as_half((unsigned short)(pk & 0xffffu)));
                    const float ey = __half2float(__ushort_as_half((unsigned short)(pk >> 16)));
                    const bool box = qa.x + ex >= fbx0 && qa.x - ex <= fbx0 + 7.f && qa.y + ey >= fby0 &&
                                     qa.y - ey <= fby0 + 7.f;
                    cu += box && ellipse_touches_rect(qa, qb, qc, fbx0, fby0, fbx0 + 7.f, fby0 + 7.f);
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                cb += __shfl_xor_sync(0xffffffffu, cb, o);
                cu += __shfl_xor_sync(0xffffffffu, cu, o);
            }
            if (lane == 0) {
                atomicAdd(&a.counters[25], (unsigned long long)cb);
                atomicAdd(&a.counters[26], (unsigned long long)cu);
            }
        }
        uint32_t n_eval = 0, n_comp = 0, n_iter = 0;
        // FWDREC: this block's record slots, 8 per tile-list entry and block (32-bit:
        // the host checks 8 * pairs < 2^32); every entry the warp composites gets a
        // record (the pixels' weights, 0 where a pixel did not composite).  A shuffle
        // result, so ptxas keeps it in a register.
        const uint32_t rbase =
            __shfl_sync(0xffffffffu, kBlocksPerTile * range.x + (uint32_t)blk * (range.y - range.x), 0);
        // FWDREC: nrec records so far; wp = this lane's weight slot of record nrec
        uint32_t nrec = 0;
        float* wp = M == FWDREC ? a.wrec_w + (size_t)rbase * 32 + lane : nullptr;
        // The list this block walks: its own per-block list (view build: the tile-list
        // entries whose block mask has this block's bit, in order), or the tile list
        // with the mask tested per entry.  Entries left out reach no pixel of the block
        // with alpha >= 1/255, i.e. multiply T by exactly 1 there.
        const bool blists = a.blist != nullptr;
        const uint32_t lo = blists ? 0u : range.x;
        const uint32_t hi = blists ? a.bcount[item] : range.y;
        const uint32_t* const list = blists ? a.blist + rbase : a.pair_g;
        // chunk pipeline: pair ids two chunks ahead, raw records one chunk ahead (each
        // lane copies and later reads only its own slots)
        const bool packed = a.pair_m == nullptr;
        const int mshift = packed ? kIdxBits + blk : blk;
        auto issue_pg = [&](uint32_t cn, int buf) {
            if (cn + lane < hi) {
                cp_async4(&st.pg[buf][lane], list + cn + lane);
                if (!packed && !blists) cp_async4(&st.pm[buf][lane], a.pair_m + cn + lane);
            }
            cp_async_commit();
        };
        auto mask_word = [&](int buf) { return packed ? st.pg[buf][lane] : st.pm[buf][lane]; };
        auto in_block = [&](int buf) { return blists || ((mask_word(buf) >> mshift) & 1u); };
        // raw records only for the entries whose footprint reaches this block
        auto issue_raw = [&](uint32_t cn, int buf) {
            if (cn + lane < hi && in_block(buf)) {
                const uint32_t sn = st.pg[buf][lane] & a.idx_mask;
                cp_async16(&st.ra[lane], &a.rec[sn].a);
                cp_async16(&st.rb[lane], &a.rec[sn].b);
                cp_async16(&st.rc[lane], &a.rec[sn].c);
                if (kFwd) cp_async16(&st.rcol[lane], &a.color[sn]);
            }
            cp_async_commit();
        };
        if (lo < hi) {
            issue_pg(lo, 0);
            issue_pg(lo + 32, 1);
            cp_async_wait<1>();
            issue_raw(lo, 0);
        }
        int buf = 0;
        for (uint32_t c0 = lo; c0 < hi; c0 += 32, buf ^= 1) {
            if (__all_sync(0xffffffffu, !(T > 0.f))) break;
            cp_async_wait<0>();  // this chunk's records (and the next chunk's ids)
            const uint32_t j = c0 + lane;
            bool keep = false;
            uint32_t s = 0;
            float4 ra = make_float4(0.f, 0.f, 0.f, 0.f), rb = ra, rc = ra, rcol = ra;
            if (j < hi) {
                s = st.pg[buf][lane] & a.idx_mask;
                RCGS_DCHECK(s < (uint64_t)a.n);
                // the pair's block mask (view build) is the per-block cull
                keep = in_block(buf);
#ifdef RCGS_CHECKED
                if (!blists) {  // a dropped (entry, block) must fail the exact per-block test too
                    const RasterRec cr = a.rec[s];
                    RCGS_DCHECK(keep || !(touches_block(cr.a, fbx0, fby0) &&
                                          ellipse_touches_rect(cr.a, cr.b, cr.c, fbx0, fby0, fbx0 + 7.f,
                                                               fby0 + 3.f)));
                }
#endif
                if (keep) {
                    ra = st.ra[lane];
                    rb = st.rb[lane];
                    rc = st.rc[lane];
                    if (kFwd) rcol = st.rcol[lane];
                }
            }
            // the slots are consumed: start the next chunk's records and the ids after
            if (c0 + 32 < hi) {
                issue_raw(c0 + 32, buf ^ 1);
                if (c0 + 64 < hi) issue_pg(c0 + 64, buf);
            }
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const int slot = __popc(bal & lt_mask);
                // the entry's quadratic about the block centre and its error bound
                const float mxr = (ra.x - cxf) + rb.x, myr = (ra.y - cyf) + rb.y;
                const float nA = rc.x, nB = rc.y, nC = rc.z, l2op = ra.w;
                const float qD = -fmaf(2.f * nA, mxr, nB * myr);
                const float qE = -fmaf(2.f * nC, myr, nB * mxr);
                const float qF = fmaf(nA * mxr, mxr, fmaf(nB * mxr, myr, fmaf(nC * myr, myr, l2op)));
                // |P2_fp32 - P2| <= 18 u M over the block (u = 2^-24; coefficient
                // rounding, the centred mean, the expansion and the 5-FMA evaluation),
                // M = |qA| X^2 + |qB| X Y + |qC| Y^2 + |log2 op| with X = 3.5 + |mxr|,
                // Y = 1.5 + |myr| bounding every monomial; taken as 2e-6 M + 2e-6
                const float X = 3.5f + fabsf(mxr), Y = 1.5f + fabsf(myr);
                const float Mb = fmaf(fabsf(nA), X * X, fmaf(fabsf(nB), X * Y, fmaf(fabsf(nC), Y * Y, fabsf(l2op))));
                const float eps = fmaf(2e-6f, Mb, 2e-6f);
                st.q0[slot] = make_float4(nA, nB, nC, qD);
                st.q1[slot] = make_float4(qE, qF, G2 - eps, G2 + eps);
                // relative alpha error: ln 2 eps (log2 error) + ex2.approx (< 3e-7)
                const float delta = fmaf(0.6932f, eps, 4e-7f);
                if (kFwd) {
                    st.q2[slot] = make_float4(rcol.x, rcol.y, rcol.z, delta);
                } else {
                    st.q2[slot] = make_float4(0.f, 0.f, 0.f, delta);
                }
                st.g[slot] = s;
                st.j[slot] = j;
                if (M == FWDREC) {  // record ids, one per staged entry
                    RCGS_DCHECK((uint64_t)rbase + nrec + slot < 8ull * (uint64_t)a.pairs &&
                                nrec + slot < range.y - range.x);
                    a.wrec_s[rbase + nrec + slot] = s;
                }
            }
            __syncwarp();
            const int n = __popc(bal);
            float* const wk = wp;  // record k of this chunk: wk[32 k] (one IMAD.WIDE per store)
            // one (pixel, entry) step of staged entry k for this lane
            auto entry = [&](int k) {
                const float4 q0 = st.q0[k], q1 = st.q1[k], q2 = st.q2[k];
                // P2 = lx (qA lx + qB ly + qD) + (ly (qC ly + qE) + qF): five FMAs, two
                // lane constants (each rounding is bounded by the monomial sum M)
                const float P2 = fmaf(lxf, fmaf(q0.x, lxf, fmaf(q0.y, lyf, q0.w)), fmaf(lyf, fmaf(q0.z, lyf, q1.x), q1.y));
                const bool live = T > 0.f;
                const bool pass = P2 >= q1.z;  // false: alpha is certainly 0 (skipped, T x 1 exactly)
                // gate band (finished lanes included: a spurious slow call is harmless)
                const bool gamb = pass && P2 < q1.w;
                // ex2(-inf) = 0: the skip is folded into the exponent (no predicated MUFU)
                const float al = fminf(a.f_alpha_clamp, ex2_approx(pass ? P2 : -INFINITY));
                if (kInstr) {
                    n_eval += live;
                    ++n_iter;
                }
                StepOut o = composite_step<M>(T, A, live, pass, al, q2.w, a.f_floor, a.f_tau);
                if (__any_sync(0xffffffffu, gamb || o.amb)) {
                    const SlowOut so =
                        slow_entry<M>(list, a.rec, a.exact, a.alpha_clamp, a.alpha_skip, a.t_floor, a.tau, a.f_floor,
                                      a.f_tau, st.g[k], st.j[k], lo, cxf + lxf, cyf + lyf, lane, T, A, live, pass,
                                      gamb, al, q2.w, o, a.idx_mask);
                    o = so.o;
                    n_resync += so.resync;
                }
                const float wc = o.wc;
                const bool xc = o.xc;
                const float Tn = o.Tn, An = o.An;
                const bool comp = wc != 0.f;
                if (kInstr) n_comp += comp;
                T = Tn;
                A = An;
                if (M == DEPTH && xc) cross = (int32_t)st.g[k];
                if (kFwd) {
                    acc0 = fmaf(q2.x, wc, acc0);
                    acc1 = fmaf(q2.y, wc, acc1);
                    acc2 = fmaf(q2.z, wc, acc2);
                    if (M == FWDREC) {
                        *reinterpret_cast<float*>(reinterpret_cast<char*>(wk) + (size_t)(uint32_t)k * 128u) = wc;
                    }
                } else if (M == CAP_COUNT) {
                    ncap += comp;
                } else if (M == CAP_WRITE) {
                    if (comp) {
                        const uint32_t o = cap_base + ncap++;
                        RCGS_DCHECK(inside);
                        a.cap_pixel[o] = pix;
                        a.cap_kept[o] = a.rank_of[st.g[k]];  // the API reports depth ranks
                        a.cap_weight[o] = (double)wc;
                    }
                } else if (M == BWD) {
                    // products rounded on their own (no FMA contraction into the tree below), as
                    // in the record-streaming backward
                    float v0 = __fmul_rn(wc, g0), v1 = __fmul_rn(wc, g1), v2 = __fmul_rn(wc, g2);
                    if (__any_sync(0xffffffffu, v0 != 0.f || v1 != 0.f || v2 != 0.f)) {
                        // transposed reduce-scatter of (v0, v1, v2, 0) over the warp: 6
                        // shuffles instead of 15; channel c ends summed in lanes 8c..8c+7
                        const bool h16 = lane & 16, h8 = lane & 8;
                        const float ra_ = __shfl_xor_sync(0xffffffffu, h16 ? v0 : v2, 16);
                        const float rb_ = __shfl_xor_sync(0xffffffffu, h16 ? v1 : 0.f, 16);
                        const float ka = (h16 ? v2 : v0) + ra_, kb = (h16 ? 0.f : v1) + rb_;
                        float val = (h8 ? kb : ka) + __shfl_xor_sync(0xffffffffu, h8 ? ka : kb, 8);
                        val += __shfl_xor_sync(0xffffffffu, val, 4);
                        val += __shfl_xor_sync(0xffffffffu, val, 2);
                        val += __shfl_xor_sync(0xffffffffu, val, 1);
                        if ((lane & 7) == 0 && lane < 24) {
                            if (isfinite(val)) {
                                const long long q = to_fixed(val);
                                atomicAdd(&a.acc_fx[3 * (int64_t)st.g[k] + (lane >> 3)], (unsigned long long)q);
                            } else if (a.nonfinite) {
                                atomicOr(a.nonfinite, 1);
                            }
                        }
                    }
                } else if (M == HITS) {
                    const unsigned hb = __ballot_sync(0xffffffffu, comp);
                    if (hb) {
                        float ws = wc;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) ws += __shfl_xor_sync(0xffffffffu, ws, o);
                        if (lane == 0) {
                            const uint32_t g = st.g[k];
                            atomicAdd(&a.hits[g], __popc(hb));
                            atomicAdd(&a.wsum[g], (unsigned long long)llrint((double)ws * 4294967296.0));
                        }
                    }
                }
            };
            bool all_done = false;
            int k = 0;
            for (; k < n && !all_done; ++k) {
                entry(k);
                all_done = __all_sync(0xffffffffu, !(T > 0.f));  // one vote: cheaper than a cadence test
            }
            nrec += (uint32_t)k;  // entries processed (one record each in FWDREC)
            if (M == FWDREC) wp += (size_t)k * 32;
            __syncwarp();
        }
        cp_async_wait<0>();  // no copy may land in the slots once the next item uses them

        if (kInstr && a.counters) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                n_eval += __shfl_xor_sync(0xffffffffu, n_eval, o);
                n_comp += __shfl_xor_sync(0xffffffffu, n_comp, o);
            }
            if (lane == 0) {
                atomicAdd(&a.counters[5 * kRow + 0], (unsigned long long)n_eval);
                atomicAdd(&a.counters[5 * kRow + 1], (unsigned long long)n_comp);
                atomicAdd(&a.counters[5 * kRow + 2], 1ull);
                atomicAdd(&a.counters[5 * kRow + 4], (unsigned long long)n_iter);
            }
        }
        if (kInstr && a.trace) {
            uint32_t nv = n_eval;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) nv += __shfl_xor_sync(0xffffffffu, nv, o);
            if (lane == 0) {
                uint32_t* tr = a.trace + 8 * (int64_t)item;
                tr[1] = globaltimer_lo();
                tr[2] = smid();
                tr[3] = n_iter;
                tr[4] = nv;
                tr[5] = 0;
                tr[6] = n_resync;
                tr[7] = (uint32_t)tile;
            }
        }
        if (M == FWDREC && lane == 0) {
            a.wrec_n[tile * kBlocksPerTile + blk] = nrec;
            if (kInstr && a.counters) atomicAdd(&a.counters[5 * kRow + 3], (unsigned long long)nrec);
        }
        if (!inside) continue;
        if (kFwd) {
            write_pixel<M == FWDRGBA>(a.out, a.W, a.H, pix, acc0, acc1, acc2, fabsf(T));
        } else if (M == DEPTH) {
            if (a.cross) a.cross[pix] = cross;
            if (a.depth) a.depth[pix] = cross >= 0 ? a.z[cross] : __longlong_as_double(0x7ff0000000000000ll);
        } else if (M == CAP_COUNT) {
            a.cap_count[pix] = ncap;
        }
    }
    work_counter_exit(a.counter, lane);
}

// ---------------------------------------------------------------- weight records
// The composite weights w = alpha * T_before of a view depend on the geometry and
// the camera only, not on the colours an SH-only recolor refits.  FWDREC stores,
// per 8x4 block and per entry iteration in which any pixel composited, the entry
// and the 32 pixel weights (0 where a pixel did not composite).  The backward is
// then a streaming pass over the records (the same products, reduce-scatter and
// fixed-point atomics, in the same entry order: bit-identical to re-traversing),
// and a later render of the same view is an SpMV over them.
struct RecArgs {
    const uint2* ranges;
    const uint32_t* tile_order;
    unsigned* counter;
    int W, H, tiles_x, n_items;
    const uint32_t* wrec_n;
    const uint32_t* wrec_s;
    const float* wrec_w;
    const uint32_t* wrec_off;  // per-block first record (view-owned compact records) or null
    int64_t n;                 // scene size (checked builds' bound)
    // render
    const float4* color;
    const float* t_in;
    PixelOut out;
    // backward
    const float* grad;
    unsigned long long* acc_fx;
    int32_t* nonfinite;
};

// Backward over the recorded weights, latency-hidden.  Each warp walks a static
// stride of the heavy-first block order (no work-counter round trip), and the next
// block's metadata (tile, record range, pixel gradients) is loaded while the
// current block's records stream; record batches are double-buffered.  The per-
// block setup chain (order -> range -> gradients, each a dependent global load)
// was comparable to the ~2-3 record batches a block holds.
struct RecMeta {
    uint32_t base, n;
    float g0, g1, g2;
};

__device__ __forceinline__ RecMeta rec_meta(const RecArgs& a, unsigned item, int tile, int lane) {
    RecMeta m;
    const int blk = (int)(item % kBlocksPerTile);
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int u = tx * kTile + (blk & 1) * 8 + (lane & 7), v = ty * kTile + (blk >> 1) * 4 + (lane >> 3);
    const bool inside = u < a.W && v < a.H;
    const int64_t pix = (int64_t)v * a.W + u;
    m.g0 = inside ? a.grad[3 * pix] : 0.f;
    m.g1 = inside ? a.grad[3 * pix + 1] : 0.f;
    m.g2 = inside ? a.grad[3 * pix + 2] : 0.f;
    const uint2 range = a.ranges[tile];
    m.base = a.wrec_off ? a.wrec_off[tile * kBlocksPerTile + blk]
                        : kBlocksPerTile * range.x + (uint32_t)blk * (range.y - range.x);
    m.n = a.wrec_n[tile * kBlocksPerTile + blk];
    return m;
}

#ifndef RCGS_REC_BWD_CTAS
#define RCGS_REC_BWD_CTAS 4
#endif
// One block's records, all pixel gradients finite: batches of 8 records staged in
// the warp's shared rows (cp.async, double-buffered; rows padded to 36 floats so
// the 4 lanes of each record read conflict-free).  Lane (q, h) = (lane / 4, lane
// % 4) owns record q's pixels h, h + 4, ..., h + 28 and sums w g over them in the
// pairing of the xor-16, 8, 4 stages of the warp butterfly, then the xor-2 / xor-1
// shuffles finish it: the same tree as a plain warp sum of the 32 products, so the
// totals equal the traversal backward's bit for bit (and, with finite g, w = 0
// gives an exact 0 product, as skipping the pixel does).  The sums of channels
// 0 / 1 go through packed FADD2.
// Copy of one 8-record batch of a block into the warp's shared rows `buf` (one
// commit group, empty past the block's end): lane (q, h) copies 32 bytes of record
// q, quarter h.
__device__ __forceinline__ void cp_async16_s(uint32_t dst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async4_s(uint32_t dst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(gsrc) : "memory");
}

// Shared-memory byte addresses of a warp's record rows (2 buffers x 8 rows of 36
// floats) and record ids (2 x 8), computed once per warp.
struct RecSmem {
    uint32_t w, s;
};
constexpr uint32_t kRecRowB = 36 * 4, kRecBufB = 8 * kRecRowB;

__device__ __forceinline__ void rec_bwd_issue(const RecArgs& a, const RecMeta& m, uint32_t r0, RecSmem sm, int buf,
                                              int lane) {
    const int q = lane >> 2, h = lane & 3;
    const uint32_t r = r0 + (uint32_t)q;
    if (r < m.n) {
        const float* src = a.wrec_w + (size_t)(m.base + r) * 32 + 8 * h;
        const uint32_t dst = sm.w + (uint32_t)buf * kRecBufB + (uint32_t)q * kRecRowB + (uint32_t)h * 32u;
        cp_async16_s(dst, src);
        cp_async16_s(dst + 16, src + 4);
    }
    if (lane < 8 && r0 + lane < m.n)
        cp_async4_s(sm.s + (uint32_t)buf * 32u + (uint32_t)lane * 4u, a.wrec_s + m.base + r0 + lane);
    cp_async_commit();
}

// Batch 0 of this block is already in flight in `buf` (issued while the previous
// block's last batch was summed); while this block's last batch is summed, the
// next block's batch 0 goes out (when `nm_pre`), so a warp's record stream does
// not restart at every block (the per-block restart had been ~30% of the stall
// samples).  On return `buf` is the buffer holding the next block's batch 0.
__device__ __forceinline__ void rec_bwd_block(const RecArgs& a, const RecMeta& m, bool nm_pre, const RecMeta& nm,
                                              float (*sw)[8][36], uint32_t (*ss)[8], RecSmem sm, int& buf, int lane) {
    const int q = lane >> 2, h = lane & 3;
    float2 g01[8];
    float g2[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int src = h + 4 * j;
        g01[j] = make_float2(__shfl_sync(0xffffffffu, m.g0, src), __shfl_sync(0xffffffffu, m.g1, src));
        g2[j] = __shfl_sync(0xffffffffu, m.g2, src);
    }
    for (uint32_t r0 = 0; r0 < m.n; r0 += 8, buf ^= 1) {
        if (r0 + 8 < m.n) {
            rec_bwd_issue(a, m, r0 + 8, sm, buf ^ 1, lane);
        } else if (nm_pre) {
            rec_bwd_issue(a, nm, 0, sm, buf ^ 1, lane);
        } else {
            cp_async_commit();  // keeps one group per batch
        }
        cp_async_wait<1>();
        __syncwarp();
        const bool live = r0 + q < m.n;
        float2 p01[8];
        float p2[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float w = live ? sw[buf][q][h + 4 * j] : 0.f;
            // scalar products: a packed FMUL2 here is contracted with the FADD2 below
            p01[j] = make_float2(__fmul_rn(w, g01[j].x), __fmul_rn(w, g01[j].y));
            p2[j] = __fmul_rn(w, g2[j]);  // no FMA contraction into the sums below
        }
        // pixel i = h + 4 j: xor-16 pairs j, j + 4; xor-8 pairs j, j + 2; xor-4 pairs j, j + 1
        float2 a01[4];
        float a2[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            a01[j] = __fadd2_rn(p01[j], p01[j + 4]);
            a2[j] = p2[j] + p2[j + 4];
        }
        const float2 b0 = __fadd2_rn(a01[0], a01[2]), b1 = __fadd2_rn(a01[1], a01[3]);
        float2 c01 = __fadd2_rn(b0, b1);
        float c2 = (a2[0] + a2[2]) + (a2[1] + a2[3]);
        c01.x += __shfl_xor_sync(0xffffffffu, c01.x, 2);
        c01.y += __shfl_xor_sync(0xffffffffu, c01.y, 2);
        c2 += __shfl_xor_sync(0xffffffffu, c2, 2);
        c01.x += __shfl_xor_sync(0xffffffffu, c01.x, 1);
        c01.y += __shfl_xor_sync(0xffffffffu, c01.y, 1);
        c2 += __shfl_xor_sync(0xffffffffu, c2, 1);
        float val = c2;  // selects, not branches
        val = h == 1 ? c01.y : val;
        val = h == 0 ? c01.x : val;
        if (h < 3 && live && val != 0.f) {
            const uint32_t sq = ss[buf][q];
            RCGS_DCHECK(sq < (uint32_t)a.n);
            if (isfinite(val)) {
                atomicAdd(&a.acc_fx[3 * (int64_t)sq + h], (unsigned long long)to_fixed(val));
            } else if (a.nonfinite) {
                atomicOr(a.nonfinite, 1);
            }
        }
        __syncwarp();  // the rows of `buf` are refilled by the issue two batches on
    }
}

__global__ void __launch_bounds__(kCTA, RCGS_REC_BWD_CTAS) rec_bwd_kernel(RecArgs a) {
    const int lane = threadIdx.x & 31;
    __shared__ __align__(16) float s_w[kCTA / 32][2][8][36];
    __shared__ uint32_t s_s[kCTA / 32][2][8];
    float(*sw)[8][36] = s_w[threadIdx.x >> 5];
    uint32_t(*ss)[8] = s_s[threadIdx.x >> 5];
    const RecSmem sm = {(uint32_t)__cvta_generic_to_shared(&sw[0][0][0]), (uint32_t)__cvta_generic_to_shared(&ss[0][0])};
    constexpr int kU = 8;  // records per batch (the 32-value reduce-scatter width)
    const unsigned nw = gridDim.x * (blockDim.x >> 5);
    const unsigned gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    auto tile_of = [&](unsigned item) -> int {
        return a.tile_order ? (int)a.tile_order[item / kBlocksPerTile] : (int)(item / kBlocksPerTile);
    };
    unsigned item = gw;
    if (item >= (unsigned)a.n_items) return;
    RecMeta m = rec_meta(a, item, tile_of(item), lane);
    int ntile = item + nw < (unsigned)a.n_items ? tile_of(item + nw) : 0;
    // a block takes the streamed (fast) path when it has records, a nonzero gradient
    // somewhere and only finite gradients; its batch 0 is then issued ahead
    auto fast = [&](const RecMeta& mm) {
        return mm.n > 0 && !__all_sync(0xffffffffu, mm.g0 == 0.f && mm.g1 == 0.f && mm.g2 == 0.f) &&
               __all_sync(0xffffffffu, isfinite(mm.g0) && isfinite(mm.g1) && isfinite(mm.g2));
    };
    int buf = 0;
    bool pre = fast(m);
    if (pre) rec_bwd_issue(a, m, 0, sm, buf, lane);
    while (true) {
        const unsigned nitem = item + nw;
        const bool has_next = nitem < (unsigned)a.n_items;
        // next block's metadata in flight while this block streams its records
        RecMeta nm = {0u, 0u, 0.f, 0.f, 0.f};
        if (has_next) nm = rec_meta(a, nitem, ntile, lane);
        const int nntile = nitem + nw < (unsigned)a.n_items ? tile_of(nitem + nw) : 0;
        // the gradient is local to the edited region: blocks whose gradients are all
        // 0 have no term
        if (m.n > 0 && !__all_sync(0xffffffffu, m.g0 == 0.f && m.g1 == 0.f && m.g2 == 0.f)) {
            if (pre) {
                const bool npre = has_next && fast(nm);
                rec_bwd_block(a, m, npre, nm, sw, ss, sm, buf, lane);
                pre = npre;
                m = nm;
                if (!has_next) break;
                item = nitem;
                ntile = nntile;
                continue;
            } else {
            // non-finite pixel gradients: a pixel that no record composites (w = 0)
            // must contribute nothing, not 0 * inf
            float w[kU], wn[kU];
            uint32_t sl = 0u, sln = 0u;  // lane q < kU holds record q's scene index
            auto load = [&](uint32_t r0, float* wd, uint32_t& sd) {
#pragma unroll
                for (int q = 0; q < kU; ++q) {
                    const bool ok = r0 + q < m.n;
                    wd[q] = ok ? __ldcs(a.wrec_w + (size_t)(m.base + r0 + q) * 32 + lane) : 0.f;
                }
                sd = (lane < kU && r0 + lane < m.n) ? a.wrec_s[m.base + r0 + lane] : 0u;
                RCGS_DCHECK(!(lane < kU && r0 + lane < m.n) || sd < (uint32_t)a.n);
            };
            load(0, w, sl);
            for (uint32_t r0 = 0; r0 < m.n; r0 += kU) {
                if (r0 + kU < m.n) load(r0 + kU, wn, sln);
                // the kU records' (w g) sums for 3 channels (+1 zero pad) = 32 values,
                // halved across the warp: xor 16, 8, 4, 2, 1 -- the butterfly tree of a
                // plain warp sum (bit-identical totals); lane L ends with record L >> 2,
                // channel L & 3
                float x[32];
#pragma unroll
                for (int q = 0; q < kU; ++q) {
                    const bool comp = w[q] != 0.f;
                    x[4 * q] = comp ? __fmul_rn(w[q], m.g0) : 0.f;
                    x[4 * q + 1] = comp ? __fmul_rn(w[q], m.g1) : 0.f;
                    x[4 * q + 2] = comp ? __fmul_rn(w[q], m.g2) : 0.f;
                    x[4 * q + 3] = 0.f;
                }
#pragma unroll
                for (int h = 16; h >= 1; h >>= 1) {
                    const bool hi = lane & h;
#pragma unroll
                    for (int p = 0; p < h; ++p) {
                        const float send = hi ? x[p] : x[p + h];
                        const float keep = hi ? x[p + h] : x[p];
                        x[p] = keep + __shfl_xor_sync(0xffffffffu, send, h);
                    }
                }
                const float val = x[0];
                const int q = lane >> 2, c = lane & 3;
                const uint32_t sq = __shfl_sync(0xffffffffu, sl, q);
                if (c < 3 && val != 0.f && r0 + q < m.n) {
                    if (isfinite(val)) {
                        atomicAdd(&a.acc_fx[3 * (int64_t)sq + c], (unsigned long long)to_fixed(val));
                    } else if (a.nonfinite) {
                        atomicOr(a.nonfinite, 1);
                    }
                }
#pragma unroll
                for (int u = 0; u < kU; ++u) w[u] = wn[u];
                sl = sln;
            }
            }
        }
        // (this block took no streamed path) issue the next block's batch 0
        cp_async_wait<0>();
        __syncwarp();
        pre = has_next && fast(nm);
        if (pre) rec_bwd_issue(a, nm, 0, sm, buf, lane);
        if (!has_next) break;
        item = nitem;
        m = nm;
        ntile = nntile;
    }
    cp_async_wait<0>();
}

// kMode: 0 SpMV render into an image, 1 backward, 2 SpMV render into an RGBA8 frame
template <int kMode>
__global__ void __launch_bounds__(kCTA) rec_kernel(RecArgs a) {
    constexpr bool kBwd = kMode == 1;
    const int lane = threadIdx.x & 31;
    constexpr int kU = 8;  // records in flight per warp
    for (;;) {
        unsigned item = 0;
        if (lane == 0) item = atomicAdd(a.counter, 1u);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= (unsigned)a.n_items) break;
        const int tile = a.tile_order ? (int)a.tile_order[item / kBlocksPerTile] : (int)(item / kBlocksPerTile);
        const int blk = (int)(item % kBlocksPerTile);
        const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
        const int u = tx * kTile + (blk & 1) * 8 + (lane & 7), v = ty * kTile + (blk >> 1) * 4 + (lane >> 3);
        const bool inside = u < a.W && v < a.H;
        const int64_t pix = (int64_t)v * a.W + u;
        float g0 = 0.f, g1 = 0.f, g2 = 0.f;
        if (kBwd) {
            if (inside) {
                g0 = a.grad[3 * pix];
                g1 = a.grad[3 * pix + 1];
                g2 = a.grad[3 * pix + 2];
            }
            if (__all_sync(0xffffffffu, g0 == 0.f && g1 == 0.f && g2 == 0.f)) continue;
        }
        const uint2 range = a.ranges[tile];
        const uint32_t base = a.wrec_off ? a.wrec_off[tile * kBlocksPerTile + blk]
                                         : kBlocksPerTile * range.x + (uint32_t)blk * (range.y - range.x);
        const uint32_t n = a.wrec_n[tile * kBlocksPerTile + blk];
        float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f;
        for (uint32_t r0 = 0; r0 < n; r0 += kU) {
            float w[kU];
            uint32_t s[kU];
#pragma unroll
            for (int q = 0; q < kU; ++q) {
                const bool ok = r0 + q < n;
                w[q] = ok ? __ldcs(a.wrec_w + (size_t)(base + r0 + q) * 32 + lane) : 0.f;
                s[q] = ok ? a.wrec_s[base + r0 + q] : 0u;
                RCGS_DCHECK(s[q] < (uint32_t)a.n);
            }
#pragma unroll
            for (int q = 0; q < kU; ++q) {
                if (r0 + q >= n) break;
                if (!kBwd) {
                    if (w[q] != 0.f) {
                        const float4 c = a.color[s[q]];
                        acc0 = fmaf(c.x, w[q], acc0);
                        acc1 = fmaf(c.y, w[q], acc1);
                        acc2 = fmaf(c.z, w[q], acc2);
                    }
                }
            }
            if (kBwd) {
                // the kU = 8 records' (w g) sums for 3 channels (+1 zero pad) = 32 values,
                // halved across the warp: xor 16, 8, 4, 2, 1 -- the butterfly tree of a
                // plain warp sum (bit-identical totals), 31 shuffles per 8 records; lane L
                // ends with record L >> 2, channel L & 3
                float x[32];
#pragma unroll
                for (int q = 0; q < kU; ++q) {
                    const bool comp = w[q] != 0.f;
                    x[4 * q] = comp ? __fmul_rn(w[q], g0) : 0.f;
                    x[4 * q + 1] = comp ? __fmul_rn(w[q], g1) : 0.f;
                    x[4 * q + 2] = comp ? __fmul_rn(w[q], g2) : 0.f;
                    x[4 * q + 3] = 0.f;
                }
#pragma unroll
                for (int h = 16; h >= 1; h >>= 1) {
                    const bool hi = lane & h;
#pragma unroll
                    for (int p = 0; p < h; ++p) {
                        const float send = hi ? x[p] : x[p + h];
                        const float keep = hi ? x[p + h] : x[p];
                        x[p] = keep + __shfl_xor_sync(0xffffffffu, send, h);
                    }
                }
                const float val = x[0];
                const int q = lane >> 2, c = lane & 3;
                if (c < 3 && val != 0.f) {
                    if (isfinite(val)) {
                        atomicAdd(&a.acc_fx[3 * (int64_t)s[q] + c], (unsigned long long)to_fixed(val));
                    } else if (a.nonfinite) {
                        atomicOr(a.nonfinite, 1);
                    }
                }
            }
        }
        if (!kBwd && inside) write_pixel<kMode == 2>(a.out, a.W, a.H, pix, acc0, acc1, acc2, a.t_in[pix]);
    }
    work_counter_exit(a.counter, lane);
}

template <int kMode>
static int launch_rec(RecArgs a, cudaStream_t s) {
    static int grid = 0;
    if (grid == 0) {
        int dev = 0, sms = 0, per_sm = 0;
        RCGS_CUDA(cudaGetDevice(&dev));
        RCGS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        RCGS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rec_kernel<1>, kCTA, 0));
        grid = sms * persistent_ctas(per_sm > 0 ? per_sm : 1);
    }
    static const bool dynamic = getenv("RCGS_REC_BWD_DYNAMIC") != nullptr;
    if (kMode == 1 && !dynamic) {
        // static work striding: every launched CTA must be resident at once
        static int bgrid = 0;
        if (bgrid == 0) {
            int dev = 0, sms = 0, per_sm = 0;
            RCGS_CUDA(cudaGetDevice(&dev));
            RCGS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            RCGS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rec_bwd_kernel, kCTA, 0));
            bgrid = sms * persistent_ctas(per_sm > 0 ? per_sm : 1);
        }
        const int blocks = (int)min((int64_t)bgrid, ((int64_t)a.n_items + kWarpsPerCTA - 1) / kWarpsPerCTA);
        if (blocks > 0) rec_bwd_kernel<<<blocks, kCTA, 0, s>>>(a);
        RCGS_LAUNCH_CHECK();
        return RCGS_OK;
    }
    const int blocks = (int)min((int64_t)grid, ((int64_t)a.n_items + kWarpsPerCTA - 1) / kWarpsPerCTA);
    if (blocks > 0) rec_kernel<kMode><<<blocks, kCTA, 0, s>>>(a);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

// One process-wide record arena (per device process): the training path records
// one view at a time on the caller's stream, so the scratch is reused every step
// instead of reserving (and stream-ordered freeing) ~3 GB per view.  It grows
// with plain cudaMalloc/cudaFree (rare; cudaFree synchronises) and is never
// released by views.  A view's records are valid while it is the arena's owner
// at the epoch it recorded in (views are destroyed on other threads, hence the
// atomics).
struct RecordArena {
    std::mutex grow;
    unsigned char* base = nullptr;
    size_t cap = 0;
    std::atomic<const rcgs_view*> owner{nullptr};
    std::atomic<uint64_t> epoch{0};
};
static RecordArena g_arena;

static bool records_valid(const rcgs_view* v) {
    return v->wrec_owned || (v->wrec_valid && g_arena.owner.load() == v && g_arena.epoch.load() == v->wrec_epoch);
}

void release_records(rcgs_view* v, cudaStream_t s) {
    if (v->wrec_owned) {  // view-owned compact copy (rcgs_view_keep_records)
        dfree(v->wrec_n, s);
        dfree(v->wrec_s, s);
        dfree(v->wrec_w, s);
        dfree(v->wrec_tf, s);
        dfree(v->wrec_off, s);
        v->wrec_owned = false;
        return;
    }
    const rcgs_view* expect = v;
    g_arena.owner.compare_exchange_strong(expect, nullptr);
}

// Copy each block's records from the arena layout to a compact layout at the
// scanned per-block offsets (one warp per block).
__global__ void records_compact_kernel(const uint32_t* __restrict__ n_rec, const uint2* __restrict__ ranges,
                                       int n_blocks, const uint32_t* __restrict__ src_s,
                                       const float* __restrict__ src_w, const uint32_t* __restrict__ off,
                                       uint32_t* __restrict__ dst_s, float* __restrict__ dst_w) {
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (b >= n_blocks) return;
    const uint2 range = ranges[b / kBlocksPerTile];
    const uint32_t src = kBlocksPerTile * range.x + (uint32_t)(b % kBlocksPerTile) * (range.y - range.x);
    const uint32_t dst = off[b], n = n_rec[b];
    for (uint32_t r = 0; r < n; ++r) {
        dst_w[(size_t)(dst + r) * 32 + lane] = src_w[(size_t)(src + r) * 32 + lane];
        if (lane == 0) dst_s[dst + r] = src_s[src + r];
    }
}

static RecArgs rec_args(const rcgs_view* v) {
    RecArgs a;
    memset(&a, 0, sizeof(a));
    a.ranges = v->ranges;
    a.tile_order = v->tile_order;
    a.counter = v->work;
    a.W = v->cam.width;
    a.H = v->cam.height;
    a.tiles_x = v->tiles_x;
    a.n_items = v->tiles_x * v->tiles_y * kBlocksPerTile;
    a.wrec_n = v->wrec_n;
    a.wrec_s = v->wrec_s;
    a.wrec_w = v->wrec_w;
    a.wrec_off = v->wrec_owned ? v->wrec_off : nullptr;
    a.n = v->n;
    a.color = v->color;
    a.t_in = v->wrec_tf;
    return a;
}

static RasterArgs base_args(const rcgs_view* v) {
    RasterArgs a;
    memset(&a, 0, sizeof(a));
    a.ranges = v->ranges;
    a.tile_order = v->tile_order;
    a.tile_meta = v->tile_meta;
    a.pair_g = v->pair_g;
    a.pair_m = v->pair_packed ? nullptr : v->pair_m;
    a.blist = v->blist;
    a.bcount = v->bcount;
    a.idx_mask = v->pair_packed ? kIdxMask : 0xffffffffu;
    a.rank_of = v->rank_of;
    a.counter = v->work;
    a.rec = v->rec;
    a.exact = v->exact;
    a.color = v->color;
    a.gid = v->gid;
    a.z = v->z;
    a.W = v->cam.width;
    a.H = v->cam.height;
    a.tiles_x = v->tiles_x;
    a.n_items = v->tiles_x * v->tiles_y * kBlocksPerTile;
    a.n = v->n;
    a.pairs = v->pairs;
    a.alpha_clamp = v->cfg.alpha_clamp;
    a.alpha_skip = v->cfg.alpha_skip;
    a.t_floor = v->cfg.transmittance_floor;
    a.f_alpha_clamp = (float)v->cfg.alpha_clamp;
    a.f_floor = (float)v->cfg.transmittance_floor;
    a.f_gate2 = (float)log2(v->cfg.alpha_skip);
    a.tau = 0.5;
    a.f_tau = 0.5f;
    return a;
}

// Persistent launch: as many CTAs as fit on the device, each warp pulling 8x4
// blocks from a stream-ordered counter.
template <int M>
static int launch(RasterArgs a, cudaStream_t s) {
    static int grid[8] = {0};
    if (grid[M] == 0) {
        int dev = 0, sms = 0, per_sm = 0;
        RCGS_CUDA(cudaGetDevice(&dev));
        RCGS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        RCGS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, raster_kernel<M, false>, kRCTA, 0));
        grid[M] = sms * persistent_ctas(per_sm > 0 ? per_sm : 1);
    }
    a.counters = g_counters;
    a.trace = (g_trace && g_trace_items >= a.n_items) ? g_trace : nullptr;
    const int blocks = (int)min((int64_t)grid[M], ((int64_t)a.n_items + kRWarps - 1) / kRWarps);
    if (blocks > 0) {
        if (a.counters || a.trace)
            raster_kernel<M, true><<<blocks, kRCTA, 0, s>>>(a);
        else
            raster_kernel<M, false><<<blocks, kRCTA, 0, s>>>(a);
    }
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

}  // namespace rcgs

using namespace rcgs;

extern "C" int rcgs_raster_trace(uint32_t* d_trace, int64_t max_items) {
    g_trace = d_trace;
    g_trace_items = d_trace ? max_items : 0;
    return RCGS_OK;
}

extern "C" int rcgs_raster_counters(uint64_t* d_counters30) {
    g_counters = reinterpret_cast<unsigned long long*>(d_counters30);
    return RCGS_OK;
}

// Composite into `out`: an SpMV over the view's recorded weights when it has
// them, else the traversal (FWD).
static int render_into(const rcgs_view* v, const PixelOut& out, cudaStream_t s) {
    if (records_valid(v)) {  // weights recorded by an earlier rcgs_render_train: SpMV
        RecArgs ra = rec_args(v);
        ra.out = out;
        return out.layout == 2 ? launch_rec<2>(ra, s) : launch_rec<0>(ra, s);
    }
    RasterArgs a = base_args(v);
    a.out = out;
    return out.layout == 2 ? launch<FWDRGBA>(a, s) : launch<FWD>(a, s);
}

static PixelOut image_out(const float* h_bg, int layout, float* d_image, float* d_t_final) {
    PixelOut o;
    memset(&o, 0, sizeof(o));
    if (h_bg) {
        o.bg0 = h_bg[0];
        o.bg1 = h_bg[1];
        o.bg2 = h_bg[2];
    }
    o.layout = layout;
    o.image = d_image;
    o.t_final = d_t_final;
    return o;
}

extern "C" int rcgs_render(const rcgs_view* v, const float* h_bg, int layout, float* d_image,
                           float* d_t_final, void* stream) {
    RCGS_CHECK_ARG(v != nullptr && d_image != nullptr, "null argument");
    RCGS_CHECK_ARG(layout == 0 || layout == 1, "unknown layout %d", layout);
    return render_into(v, image_out(h_bg, layout, d_image, d_t_final), as_stream(stream));
}

extern "C" int rcgs_render_rgba(const rcgs_view* v, const uint8_t* d_overlay, const double* h_highlight3,
                                double strength, uint8_t* d_rgba, void* stream) {
    RCGS_CHECK_ARG(v != nullptr && d_rgba != nullptr, "null argument");
    RCGS_CHECK_ARG(d_overlay == nullptr || h_highlight3 != nullptr, "overlay needs a highlight colour");
    PixelOut o;
    memset(&o, 0, sizeof(o));
    o.layout = 2;
    o.rgba = d_rgba;
    o.overlay = d_overlay;
    if (d_overlay) {  // (1 - s) * img + s * highlight, the reference's operand order
        o.ov_keep = 1.0 - strength;
        o.ov_add0 = strength * h_highlight3[0];
        o.ov_add1 = strength * h_highlight3[1];
        o.ov_add2 = strength * h_highlight3[2];
    }
    return render_into(v, o, as_stream(stream));
}

extern "C" int rcgs_render_train(rcgs_view* v, const float* h_bg, int layout, float* d_image, float* d_t_final,
                                 void* stream) {
    RCGS_CHECK_ARG(v != nullptr && d_image != nullptr, "null argument");
    RCGS_CHECK_ARG(layout == 0 || layout == 1, "unknown layout %d", layout);
    if (records_valid(v) || v->pairs == 0) return rcgs_render(v, h_bg, layout, d_image, d_t_final, stream);
    cudaStream_t s = as_stream(stream);
    const int64_t n_items = (int64_t)v->tiles_x * v->tiles_y * kBlocksPerTile;
    const int64_t cap = (int64_t)kBlocksPerTile * v->pairs;  // <= one record per entry and block
    RCGS_CHECK_ARG(cap < ((int64_t)1 << 32), "too many tile-list entries for weight records");
    const int64_t npix = (int64_t)v->cam.width * v->cam.height;
    auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t o_n = 0, o_s = up(o_n + 4 * n_items), o_w = up(o_s + 4 * cap), o_tf = up(o_w + 128 * cap);
    const size_t need = up(o_tf + 4 * npix);
    {
        std::lock_guard<std::mutex> lock(g_arena.grow);
        if (need > g_arena.cap) {
            if (g_arena.base) RCGS_CUDA(cudaFree(g_arena.base));  // synchronises: no use in flight
            g_arena.base = nullptr;
            g_arena.cap = 0;
            const size_t want = need + need / 8;
            RCGS_CUDA(cudaMalloc(&g_arena.base, want));
            g_arena.cap = want;
        }
    }
    v->wrec_n = reinterpret_cast<uint32_t*>(g_arena.base + o_n);
    v->wrec_s = reinterpret_cast<uint32_t*>(g_arena.base + o_s);
    v->wrec_w = reinterpret_cast<float*>(g_arena.base + o_w);
    v->wrec_tf = reinterpret_cast<float*>(g_arena.base + o_tf);
    g_arena.owner.store(v);
    v->wrec_epoch = g_arena.epoch.fetch_add(1) + 1;
    RasterArgs a = base_args(v);
    a.out = image_out(h_bg, layout, d_image, v->wrec_tf);
    a.wrec_n = v->wrec_n;
    a.wrec_s = v->wrec_s;
    a.wrec_w = v->wrec_w;
    RCGS_TRY(launch<FWDREC>(a, s));
    v->wrec_valid = true;
    if (d_t_final)
        RCGS_CUDA(cudaMemcpyAsync(d_t_final, v->wrec_tf, sizeof(float) * v->cam.width * v->cam.height,
                                  cudaMemcpyDeviceToDevice, s));
    return RCGS_OK;
}

extern "C" int rcgs_depth(const rcgs_view* v, double tau, double* d_depth, int32_t* d_cross,
                          void* stream) {
    RCGS_CHECK_ARG(v != nullptr, "null view");
    RCGS_CHECK_ARG(tau > 0.0 && tau < 1.0, "tau must lie in (0, 1)");
    RasterArgs a = base_args(v);
    a.tau = tau;
    a.f_tau = (float)tau;
    a.depth = d_depth;
    a.cross = d_cross;
    return launch<DEPTH>(a, as_stream(stream));
}

extern "C" int rcgs_capture(const rcgs_view* v, int64_t* h_count, int64_t* d_pixel,
                            int64_t* d_kept, double* d_weight, void* stream) {
    RCGS_CHECK_ARG(v != nullptr && h_count != nullptr, "null argument");
    cudaStream_t s = as_stream(stream);
    const int64_t npix = (int64_t)v->cam.width * v->cam.height;
    uint32_t *cnt = nullptr, *offs = nullptr;
    RCGS_TRY(dalloc(&cnt, npix, s));
    RCGS_TRY(dalloc(&offs, npix + 1, s));
    RCGS_CUDA(cudaMemsetAsync(cnt, 0, npix * sizeof(uint32_t), s));
    RasterArgs a = base_args(v);
    a.cap_count = cnt;
    RCGS_TRY(launch<CAP_COUNT>(a, s));
    RCGS_TRY(exclusive_scan_u32(cnt, offs, npix, s));
    uint32_t* host = static_cast<uint32_t*>(pinned_scratch(sizeof(uint32_t)));
    RCGS_CUDA(cudaMemcpyAsync(host, offs + npix, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    RCGS_CUDA(cudaStreamSynchronize(s));
    const int64_t total = *host;
    if (d_pixel && d_kept && d_weight && *h_count >= total) {
        a.cap_offs = offs;
        a.cap_pixel = d_pixel;
        a.cap_kept = d_kept;
        a.cap_weight = d_weight;
        RCGS_TRY(launch<CAP_WRITE>(a, s));
    }
    *h_count = total;
    dfree(cnt, s);
    dfree(offs, s);
    return RCGS_OK;
}

// acc[gid] = active * acc_fx[s] / 2^50 (fixed point -> fp32), zero for culled gaussians.
// acc[g] = fixed-point sums -> fp32, masked by the colour clamp's active channels
// (render.py:211-214); culled gaussians get 0.  Elementwise over the scene.
__global__ void bwd_finish_kernel(const long long* __restrict__ acc_fx, const float4* __restrict__ color,
                                  const int32_t* __restrict__ rank_of, int64_t n, float* __restrict__ acc) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const int act = rank_of[g] >= 0 ? __float_as_int(color[g].w) : 0;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch)
        acc[3 * g + ch] = ((act >> ch) & 1) ? (float)((double)acc_fx[3 * g + ch] / kFixScale) : 0.f;
}

extern "C" int rcgs_view_keep_records(rcgs_view* v, void* stream) {
    RCGS_CHECK_ARG(v != nullptr, "null view");
    if (v->wrec_owned || v->pairs == 0) return RCGS_OK;
    RCGS_CHECK_ARG(records_valid(v), "no weight records to keep (call rcgs_render_train first)");
    cudaStream_t s = as_stream(stream);
    const int n_blocks = v->tiles_x * v->tiles_y * kBlocksPerTile;
    const int64_t npix = (int64_t)v->cam.width * v->cam.height;
    uint32_t *off = nullptr, *rs = nullptr, *ntab = nullptr;
    float *rw = nullptr, *tf = nullptr;
    RCGS_TRY(dalloc(&off, n_blocks + 1, s));
    RCGS_TRY(exclusive_scan_u32(v->wrec_n, off, n_blocks, s));
    uint32_t* host = static_cast<uint32_t*>(pinned_scratch(sizeof(uint32_t)));
    RCGS_CUDA(cudaMemcpyAsync(host, off + n_blocks, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    RCGS_CUDA(cudaStreamSynchronize(s));
    const int64_t total = *host;
    RCGS_TRY(dalloc(&ntab, n_blocks, s));
    RCGS_TRY(dalloc(&rs, total > 0 ? total : 1, s));
    RCGS_TRY(dalloc(&rw, (total > 0 ? total : 1) * 32, s));
    RCGS_TRY(dalloc(&tf, npix, s));
    RCGS_CUDA(cudaMemcpyAsync(ntab, v->wrec_n, sizeof(uint32_t) * n_blocks, cudaMemcpyDeviceToDevice, s));
    RCGS_CUDA(cudaMemcpyAsync(tf, v->wrec_tf, sizeof(float) * npix, cudaMemcpyDeviceToDevice, s));
    records_compact_kernel<<<div_up(n_blocks, 8), 256, 0, s>>>(v->wrec_n, v->ranges, n_blocks, v->wrec_s, v->wrec_w,
                                                              off, rs, rw);
    RCGS_LAUNCH_CHECK();
    release_records(v, s);  // the arena copy is no longer needed
    v->wrec_n = ntab;
    v->wrec_s = rs;
    v->wrec_w = rw;
    v->wrec_tf = tf;
    v->wrec_off = off;
    v->wrec_owned = true;
    v->wrec_valid = true;
    return RCGS_OK;
}

extern "C" int rcgs_backward(const rcgs_view* v, const float* d_grad_image, float* d_acc,
                             int32_t* d_nonfinite, void* stream) {
    RCGS_CHECK_ARG(v != nullptr && d_grad_image != nullptr && d_acc != nullptr, "null argument");
    cudaStream_t s = as_stream(stream);
    if (v->n == 0) return RCGS_OK;
    if (v->k == 0) {
        RCGS_CUDA(cudaMemsetAsync(d_acc, 0, 3 * v->n * sizeof(float), s));
        return RCGS_OK;
    }
    // the view's fixed-point sums by scene index (entries carry g): zeroed when the
    // view was built (on its builder stream), cleared here only for a second backward
    unsigned long long* acc_fx = v->acc_fx;
    if (v->acc_dirty) RCGS_CUDA(cudaMemsetAsync(acc_fx, 0, 3 * v->n * sizeof(unsigned long long), s));
    const_cast<rcgs_view*>(v)->acc_dirty = true;
    if (v->pairs > 0 && records_valid(v)) {  // stream the recorded weights
        RecArgs ra = rec_args(v);
        ra.grad = d_grad_image;
        ra.acc_fx = acc_fx;
        ra.nonfinite = d_nonfinite;
        RCGS_TRY(launch_rec<1>(ra, s));
    } else if (v->pairs > 0) {
        RasterArgs a = base_args(v);
        a.grad = d_grad_image;
        a.acc_fx = acc_fx;
        a.nonfinite = d_nonfinite;
        RCGS_TRY(launch<BWD>(a, s));
    }
    bwd_finish_kernel<<<div_up(v->n, 256), 256, 0, s>>>(reinterpret_cast<const long long*>(acc_fx), v->color,
                                                        v->rank_of, v->n, d_acc);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

extern "C" int rcgs_mask_hits(const rcgs_view* v, const uint8_t* d_mask, int32_t* d_hits,
                              uint64_t* d_wsum, void* stream) {
    RCGS_CHECK_ARG(v != nullptr && d_mask != nullptr && d_hits != nullptr && d_wsum != nullptr,
                   "null argument");
    RasterArgs a = base_args(v);
    a.mask = d_mask;
    a.hits = d_hits;
    a.wsum = reinterpret_cast<unsigned long long*>(d_wsum);
    return launch<HITS>(a, as_stream(stream));
}

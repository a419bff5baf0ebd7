// K3/K4/K6 tile rasteriser family (render.py:263-398, backward.py:22-40).
//
// One CTA per 16x16 tile, one thread per pixel.  The tile's depth-sorted list
// (from preprocess.cu) is streamed through shared memory 256 records at a time
// and composited front to back with the reference semantics:
//   alpha = min(0.99, sigma * exp(power)); skip alpha < 1/255;
//   stop *before* the first entry whose T * (1 - alpha) < 1e-4.
//
// Numerics.  The fast path is fp32.  Every discrete decision is made exactly as
// the fp64 reference would make it:
//   * skip:  alpha >= 1/255 <=> power >= P_g (precomputed per gaussian).  power32
//            below gate.x is certainly skipped, at/above gate.y certainly kept;
//            in between the fp64 alpha is recomputed with the reference's
//            operation order (render.py:265-271).
//   * stop / tau crossing: T is tracked in fp32 together with a running relative
//            error bound E; when T * (1 +- 2E) straddles the threshold, the
//            pixel's T is recomputed in fp64 from the start of the tile list
//            (exact cumprod, render.py:278) and fp32 T is resynchronised.
// Skipped entries multiply T by exactly 1 in the reference, so the tile list
// (footprints padded to contain every alpha >= 1/255 pixel) reproduces the
// dense global-order composite.
//
// Modes: FWD image, DEPTH (first crossing rank), BWD (per-entry partial sums
// of g * w for the SH backward, deterministic: warp shuffle tree -> fixed-order
// sum over warps -> one write per (tile, entry)), HITS (mask statistics),
// CAPTURE (contribution lists).
#include <cuda_fp16.h>

#include "common.cuh"

namespace rcgs {

enum RasterMode { FWD = 0, DEPTH = 1, BWD = 2, HITS = 3, CAP_COUNT = 4, CAP_WRITE = 5 };

constexpr int kNT = kTilePixels;  // 256 threads
constexpr int kWarps = kNT / 32;
constexpr float kLog2e = 1.4426950408889634f;

struct RasterArgs {
    const uint2* ranges;
    const uint32_t* pair_s;
    const uint32_t* pair_e;
    const RasterRec* rec;
    const ExactRec* exact;
    const float4* color;
    const uint32_t* gid;
    const double* z;
    int W, H, tiles_x;
    double alpha_clamp, alpha_skip, t_floor, tau;
    float f_alpha_clamp, f_floor, f_tau;
    // FWD
    float bg0, bg1, bg2;
    int layout;
    float* image;
    float* t_final;
    // DEPTH
    int32_t* cross;
    double* depth;
    // BWD
    const float* grad;
    float* partial;
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
};

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
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

__device__ __noinline__ double exact_alpha_at(const ExactRec* __restrict__ exact, uint32_t s, double u,
                                              double v, double clamp, double skip) {
    return exact_alpha(exact[s], u, v, clamp, skip);
}

// Exact inclusive transmittance after list entries [j0, j1] (np.cumprod, render.py:278).
__device__ __noinline__ double exact_T(const ExactRec* __restrict__ exact,
                                       const uint32_t* __restrict__ pair_s, uint32_t j0, uint32_t j1,
                                       double u, double v, double clamp, double skip) {
    double T = 1.0;
    for (uint32_t j = j0; j <= j1; ++j) {
        const double al = exact_alpha(exact[pair_s[j]], u, v, clamp, skip);
        T = __dmul_rn(T, __dsub_rn(1.0, al));
    }
    return T;
}

struct Pix {
    float uf, vf;
    float T, E;  // fp32 transmittance and its relative error bound vs fp64
};

// Result of one (pixel, entry) step.
enum StepKind { SKIP = 0, COMPOSITE = 1, STOP = 2, CROSS = 3 };

// Evaluate entry j (rank s, staged record r) for a pixel.  On COMPOSITE, *w is
// alpha * T_before and the pixel state advanced.  DEPTH mode returns CROSS at
// the first composited entry with T_inc < tau (the entry index is <= the stop
// index by construction, render.py:389-397).
template <int M>
__device__ __forceinline__ int step(const RasterRec& r, uint32_t s, uint32_t j, uint32_t j0,
                                    Pix& px, const RasterArgs& a, float* w) {
    const float dx = (px.uf - r.mean.x) - r.mean.z;
    const float dy = (px.vf - r.mean.y) - r.mean.w;
    const float power = fmaf(r.conic.x * dx, dx, fmaf(r.conic.z * dy, dy, r.conic.y * dx * dy));
    if (power < r.gate.x) return SKIP;
    float alpha;
    if (power < r.gate.y) {
        const double al = exact_alpha_at(a.exact, s, (double)px.uf, (double)px.vf, a.alpha_clamp, a.alpha_skip);
        if (al == 0.0) return SKIP;
        alpha = (float)al;
    } else {
        alpha = fminf(a.f_alpha_clamp, r.conic.w * ex2_approx(power * kLog2e));
    }
    const float oma = 1.0f - alpha;
    const float Tn = px.T * oma;
    const float delta = fmaf(fabsf(power), r.gate.z + 2e-7f, 6e-7f);
    const float En = fmaf(__fdividef(alpha, oma), delta, px.E + 2.4e-7f);
    float Tkeep = Tn, Ekeep = En;
    double T64 = 0.0;
    bool resynced = false;
    // is the exact inclusive T below the threshold?  (fp32 test, fp64 when ambiguous)
    auto below = [&](float thr_f, double thr_d) -> bool {
        if (Tkeep * (1.0f + 2.0f * Ekeep) < thr_f) return true;
        if (Tkeep * (1.0f - 2.0f * Ekeep) >= thr_f) return false;
        if (!resynced) {
            T64 = exact_T(a.exact, a.pair_s, j0, j, (double)px.uf, (double)px.vf, a.alpha_clamp, a.alpha_skip);
            Tkeep = (float)T64;
            Ekeep = 1.2e-7f;
            resynced = true;
        }
        return T64 < thr_d;
    };
    if (M == DEPTH && below(a.f_tau, a.tau)) return CROSS;
    if (below(a.f_floor, a.t_floor)) return STOP;
    *w = alpha * px.T;
    px.T = Tkeep;
    px.E = Ekeep;
    return COMPOSITE;
}

// Footprint box of a staged record vs the tile's eight 8x4 warp blocks (tile-local
// coordinates): bit w set iff the box may touch warp w's pixels.  The half extents
// are the fp64 footprint widths rounded up to fp16, so the test is conservative.
__device__ __forceinline__ uint32_t warp_block_mask(const RasterRec& r, float x0, float y0) {
    const unsigned packed = __float_as_uint(r.gate.w);
    const float ex = __half2float(__ushort_as_half((unsigned short)(packed & 0xffffu)));
    const float ey = __half2float(__ushort_as_half((unsigned short)(packed >> 16)));
    const float mx = r.mean.x - x0, my = r.mean.y - y0;
    const float lx = mx - ex - 0.01f, hx = mx + ex + 0.01f;
    const float ly = my - ey - 0.01f, hy = my + ey + 0.01f;
    const uint32_t xm = ((lx <= 7.f && hx >= 0.f) ? 1u : 0u) | ((lx <= 15.f && hx >= 8.f) ? 2u : 0u);
    uint32_t m = 0;
#pragma unroll
    for (int by = 0; by < 4; ++by)
        if (ly <= 4.f * by + 3.f && hy >= 4.f * by) m |= xm << (2 * by);
    return m;
}

template <int M>
__global__ void __launch_bounds__(kNT, 3) raster_kernel(RasterArgs a) {
    __shared__ RasterRec srec[kNT];
    __shared__ float4 scol[(M == FWD) ? kNT : 1];
    __shared__ uint32_t ss[kNT];
    __shared__ uint8_t smask[kNT];
    __shared__ uint32_t se[(M == BWD) ? kNT : 1];
    __shared__ float red[(M == BWD) ? kWarps * kNT * 3 : 1];

    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int tile = blockIdx.x;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    // warp w owns the 8x4 block (w & 1, w >> 1) of the 16x16 tile
    const int u = tx * kTile + (warp & 1) * 8 + (lane & 7);
    const int v = ty * kTile + (warp >> 1) * 4 + (lane >> 3);
    const float tile_x0 = (float)(tx * kTile), tile_y0 = (float)(ty * kTile);
    const bool inside = u < a.W && v < a.H;
    const int64_t pix = (int64_t)v * a.W + u;

    Pix px;
    px.uf = (float)u;
    px.vf = (float)v;
    px.T = 1.0f;
    px.E = 0.0f;
    bool done = !inside;
    float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f;
    int32_t cross = -1;
    uint32_t ncap = 0;
    uint32_t cap_base = 0;
    float g0 = 0.f, g1 = 0.f, g2 = 0.f;
    if (M == BWD && inside) {
        g0 = a.grad[3 * pix];
        g1 = a.grad[3 * pix + 1];
        g2 = a.grad[3 * pix + 2];
    }
    if (M == HITS && inside) done = a.mask[pix] == 0;
    if (M == CAP_WRITE && inside) cap_base = a.cap_offs[pix];

    const uint2 range = a.ranges[tile];
    for (uint32_t start = range.x; start < range.y; start += kNT) {
        if (__syncthreads_count(done) == kNT) break;
        const uint32_t cnt = min((uint32_t)kNT, range.y - start);
        if (t < cnt) {
            const uint32_t s = a.pair_s[start + t];
            const RasterRec r = a.rec[s];
            ss[t] = s;
            srec[t] = r;
            smask[t] = (uint8_t)warp_block_mask(r, tile_x0, tile_y0);
            if (M == FWD) scol[t] = a.color[s];
            if (M == BWD) se[t] = a.pair_e[start + t];
        }
        if (M == BWD) {
            for (int i = lane; i < kNT * 3; i += 32) red[warp * kNT * 3 + i] = 0.f;
        }
        __syncthreads();

        // Walk this warp's entries 32 at a time: a ballot over the staged block
        // masks yields the (warp-uniform) list of entries that can reach the block.
        for (uint32_t c0 = 0; c0 < cnt; c0 += 32) {
            const uint32_t kl = c0 + lane;
            unsigned bits = __ballot_sync(0xffffffffu, kl < cnt && ((smask[kl] >> warp) & 1u));
            while (bits) {
                const uint32_t k = c0 + (uint32_t)(__ffs(bits) - 1);
                bits &= bits - 1;
                float w = 0.f;
                int r = SKIP;
                if (!done) {
                    r = step<M>(srec[k], ss[k], start + k, range.x, px, a, &w);
                    if (r == STOP) done = true;
                    if (r == CROSS) {
                        cross = (int32_t)ss[k];
                        done = true;
                    }
                }
                const bool comp = (r == COMPOSITE);
                if (M == FWD) {
                    if (comp) {
                        const float4 c = scol[k];
                        acc0 = fmaf(c.x, w, acc0);
                        acc1 = fmaf(c.y, w, acc1);
                        acc2 = fmaf(c.z, w, acc2);
                    }
                } else if (M == CAP_COUNT) {
                    ncap += comp;
                } else if (M == CAP_WRITE) {
                    if (comp) {
                        const uint32_t o = cap_base + ncap++;
                        a.cap_pixel[o] = pix;
                        a.cap_kept[o] = ss[k];
                        a.cap_weight[o] = (double)w;
                    }
                } else if (M == BWD) {
                    float c0v = comp ? w * g0 : 0.f, c1v = comp ? w * g1 : 0.f, c2v = comp ? w * g2 : 0.f;
                    if (__any_sync(0xffffffffu, c0v != 0.f || c1v != 0.f || c2v != 0.f)) {
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) {
                            c0v += __shfl_xor_sync(0xffffffffu, c0v, o);
                            c1v += __shfl_xor_sync(0xffffffffu, c1v, o);
                            c2v += __shfl_xor_sync(0xffffffffu, c2v, o);
                        }
                        if (lane == 0) {
                            float* rp = red + (warp * kNT + k) * 3;
                            rp[0] = c0v;
                            rp[1] = c1v;
                            rp[2] = c2v;
                        }
                    }
                } else if (M == HITS) {
                    const unsigned bal = __ballot_sync(0xffffffffu, comp);
                    if (bal) {
                        float ws = comp ? w : 0.f;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) ws += __shfl_xor_sync(0xffffffffu, ws, o);
                        if (lane == 0) {
                            const uint32_t g = a.gid[ss[k]];
                            atomicAdd(&a.hits[g], __popc(bal));
                            atomicAdd(&a.wsum[g], (unsigned long long)llrint((double)ws * 4294967296.0));
                        }
                    }
                }
                if (__all_sync(0xffffffffu, done)) bits = 0;
            }
            if (__all_sync(0xffffffffu, done)) break;
        }
        if (M == BWD) {
            __syncthreads();
            if (t < cnt) {
                float s0 = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
                for (int wi = 0; wi < kWarps; ++wi) {
                    const float* rp = red + (wi * kNT + t) * 3;
                    s0 += rp[0];
                    s1 += rp[1];
                    s2 += rp[2];
                }
                float* dst = a.partial + 3 * (int64_t)se[t];
                dst[0] = s0;
                dst[1] = s1;
                dst[2] = s2;
            }
        }
    }

    if (!inside) return;
    if (M == FWD) {
        const float T = px.T;
        const float o0 = fmaf(T, a.bg0, acc0), o1 = fmaf(T, a.bg1, acc1), o2 = fmaf(T, a.bg2, acc2);
        if (a.layout == 0) {
            a.image[3 * pix] = o0;
            a.image[3 * pix + 1] = o1;
            a.image[3 * pix + 2] = o2;
        } else {
            const int64_t plane = (int64_t)a.W * a.H;
            a.image[pix] = o0;
            a.image[plane + pix] = o1;
            a.image[2 * plane + pix] = o2;
        }
        if (a.t_final) a.t_final[pix] = T;
    } else if (M == DEPTH) {
        if (a.cross) a.cross[pix] = cross;
        if (a.depth) a.depth[pix] = cross >= 0 ? a.z[cross] : __longlong_as_double(0x7ff0000000000000ll);
    } else if (M == CAP_COUNT) {
        a.cap_count[pix] = ncap;
    }
}

static RasterArgs base_args(const rcgs_view* v) {
    RasterArgs a;
    memset(&a, 0, sizeof(a));
    a.ranges = v->ranges;
    a.pair_s = v->pair_s;
    a.pair_e = v->pair_e;
    a.rec = v->rec;
    a.exact = v->exact;
    a.color = v->color;
    a.gid = v->gid;
    a.z = v->z;
    a.W = v->cam.width;
    a.H = v->cam.height;
    a.tiles_x = v->tiles_x;
    a.alpha_clamp = v->cfg.alpha_clamp;
    a.alpha_skip = v->cfg.alpha_skip;
    a.t_floor = v->cfg.transmittance_floor;
    a.f_alpha_clamp = (float)v->cfg.alpha_clamp;
    a.f_floor = (float)v->cfg.transmittance_floor;
    a.tau = 0.5;
    a.f_tau = 0.5f;
    return a;
}

template <int M>
static int launch(const RasterArgs& a, const rcgs_view* v, cudaStream_t s) {
    const int ntiles = v->tiles_x * v->tiles_y;
    raster_kernel<M><<<ntiles, kNT, 0, s>>>(a);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

}  // namespace rcgs

using namespace rcgs;

extern "C" int rcgs_render(const rcgs_view* v, const float* h_bg, int layout, float* d_image,
                           float* d_t_final, void* stream) {
    RCGS_CHECK_ARG(v != nullptr && d_image != nullptr, "null argument");
    RCGS_CHECK_ARG(layout == 0 || layout == 1, "unknown layout %d", layout);
    RasterArgs a = base_args(v);
    if (h_bg) {
        a.bg0 = h_bg[0];
        a.bg1 = h_bg[1];
        a.bg2 = h_bg[2];
    }
    a.layout = layout;
    a.image = d_image;
    a.t_final = d_t_final;
    return launch<FWD>(a, v, as_stream(stream));
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
    return launch<DEPTH>(a, v, as_stream(stream));
}

extern "C" int rcgs_capture(const rcgs_view* v, int64_t* h_count, int64_t* d_pixel,
                            int64_t* d_kept, double* d_weight, void* stream) {
    RCGS_CHECK_ARG(v != nullptr && h_count != nullptr, "null argument");
    cudaStream_t s = as_stream(stream);
    const int64_t npix = (int64_t)v->cam.width * v->cam.height;
    uint32_t *cnt = nullptr, *offs = nullptr;
    RCGS_TRY(dalloc(&cnt, npix, s));
    RCGS_TRY(dalloc(&offs, npix + 1, s));
    RasterArgs a = base_args(v);
    a.cap_count = cnt;
    RCGS_TRY(launch<CAP_COUNT>(a, v, s));
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
        RCGS_TRY(launch<CAP_WRITE>(a, v, s));
    }
    *h_count = total;
    dfree(cnt, s);
    dfree(offs, s);
    return RCGS_OK;
}

// Deterministic per-gaussian reduction of the per-(tile, entry) partials:
// acc[gid] = active * sum_{e in [offs[s], offs[s+1])} partial[e] (emission order).
__global__ void bwd_reduce_kernel(const float* __restrict__ partial, const uint32_t* __restrict__ offs,
                                  const float4* __restrict__ color, const uint32_t* __restrict__ gid,
                                  int64_t k, float* __restrict__ acc, int32_t* __restrict__ nonfinite) {
    int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= k) return;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f;
    for (uint32_t e = offs[s]; e < offs[s + 1]; ++e) {
        a0 += partial[3 * (int64_t)e];
        a1 += partial[3 * (int64_t)e + 1];
        a2 += partial[3 * (int64_t)e + 2];
    }
    const int act = __float_as_int(color[s].w);
    a0 = (act & 1) ? a0 : 0.f;
    a1 = (act & 2) ? a1 : 0.f;
    a2 = (act & 4) ? a2 : 0.f;
    const uint32_t g = gid[s];
    acc[3 * (int64_t)g] = a0;
    acc[3 * (int64_t)g + 1] = a1;
    acc[3 * (int64_t)g + 2] = a2;
    if (nonfinite && !(isfinite(a0) && isfinite(a1) && isfinite(a2))) atomicOr(nonfinite, 1);
}

extern "C" int rcgs_backward(const rcgs_view* v, const float* d_grad_image, float* d_acc,
                             int32_t* d_nonfinite, void* stream) {
    RCGS_CHECK_ARG(v != nullptr && d_grad_image != nullptr && d_acc != nullptr, "null argument");
    cudaStream_t s = as_stream(stream);
    if (v->n > 0) RCGS_CUDA(cudaMemsetAsync(d_acc, 0, 3 * v->n * sizeof(float), s));
    if (v->k == 0) return RCGS_OK;
    float* partial = nullptr;
    RCGS_TRY(dalloc(&partial, 3 * (v->pairs > 0 ? v->pairs : 1), s));
    if (v->pairs > 0) {
        RCGS_CUDA(cudaMemsetAsync(partial, 0, 3 * v->pairs * sizeof(float), s));
        RasterArgs a = base_args(v);
        a.grad = d_grad_image;
        a.partial = partial;
        RCGS_TRY(launch<BWD>(a, v, s));
    }
    bwd_reduce_kernel<<<div_up(v->k, 256), 256, 0, s>>>(partial, v->offs, v->color, v->gid, v->k, d_acc,
                                                        d_nonfinite);
    RCGS_LAUNCH_CHECK();
    dfree(partial, s);
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
    return launch<HITS>(a, v, as_stream(stream));
}

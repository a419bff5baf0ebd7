// K5: photometric loss + image gradient (losses.py:68-134), fp64 arithmetic.
//
// total = (1 - lam) * L1 + lam * (1 - SSIM), SSIM with an 11-tap separable
// gaussian (sigma 1.5), zero padding and division by the in-image kernel mass.
// The hand-derived gradient (losses.py:104-115) is linear in five filtered
// maps; by linearity it collapses to three:
//   dSSIM/dy = [F(M1) + 2 y F(M2) + g F(M3)] / n,
//   M1 = (d_mu1 - 2 d_var1 mu1 - d_cov mu2) / mass, M2 = d_var1 / mass,
//   M3 = d_cov / mass.
// Dirty: per 32x32 block, do image and target differ anywhere?
// Pass A: moments of y, g, y^2, g^2, y g (separable filter in shared memory)
//         -> SSIM map, |y - g|, M1..M3 (fp64) and per-block partial sums, for
//         blocks within two blocks of a difference (elsewhere SSIM == 1, L1 == 0).
// Pass B: separable filter of M1..M3 -> gradient within one block of a
//         difference; exact zeros elsewhere and when the images are identical
//         (losses.py:127-130).
// Tail of pass A: the last block to finish reduces the per-block partials in a
//         fixed order -> {l1, ssim, total} (deterministic; formerly a pass C kernel).
// Both filter passes work on 32x32 output tiles (42x42 with the 5-pixel halo),
// one channel at a time; the vertical pass is a register sliding window (each
// thread produces 4 rows of one column from 14 shared-memory rows).
#include <math.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace rcgs {

constexpr int kR = 5;              // window half width
constexpr int kWin = 2 * kR + 1;   // 11
constexpr int kLT = 32;            // output tile edge
constexpr int kLH = kLT + 2 * kR;  // 42
constexpr int kMS = 48;            // pass B: map plane row stride (columns x0 - 8 .. x0 + 39)
constexpr int kMO = 8 - kR;        // pass B: the halo's first column (x0 - 5) within a row
constexpr int kRows = 4;           // output rows per thread in the vertical pass
constexpr int kLNT = 256;          // = kLT * kLT / kRows
#ifndef RCGS_LOSS_HS
#define RCGS_LOSS_HS 4
#endif
constexpr int kHS = RCGS_LOSS_HS;  // adjacent outputs per thread in the horizontal passes
#ifndef RCGS_LOSS_CTAS
#define RCGS_LOSS_CTAS 3
#endif
constexpr int kLossCTAs = RCGS_LOSS_CTAS;  // resident CTAs per SM the filter passes target

struct Window {
    double w[kWin];
};

__device__ __forceinline__ double mass1d(const Window& W, int i, int len) {
    double m = 0.0;
#pragma unroll
    for (int k = 0; k < kWin; ++k) {
        const int j = i + k - kR;
        if (j >= 0 && j < len) m += W.w[k];
    }
    return m;
}

__device__ __forceinline__ void block_sum2(double& a, double& b, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        sh[2 * warp] = a;
        sh[2 * warp + 1] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double x = 0.0, y = 0.0;
        for (int w = 0; w < kLNT / 32; ++w) {
            x += sh[2 * w];
            y += sh[2 * w + 1];
        }
        a = x;
        b = y;
    }
}

// The window in the gradient-map filter type (fp32 for the fp32 entry point).
template <typename F>
struct WindowT {
    F w[kWin];
};

// Vertical 11-tap pass for kRows consecutive output rows of one column from a
// horizontally filtered plane h[kLH][kLT] (rows r0 .. r0 + kRows + 9).
template <typename F, typename Win>
__device__ __forceinline__ void vfilter(const F* __restrict__ h, int r0, int c, const Win& win, F out[kRows]) {
#pragma unroll
    for (int i = 0; i < kRows; ++i) out[i] = F(0);
#pragma unroll
    for (int rr = 0; rr < kRows + kWin - 1; ++rr) {
        const F v = h[(r0 + rr) * kLT + c];
#pragma unroll
        for (int i = 0; i < kRows; ++i) {
            const int k = rr - i;
            if (k >= 0 && k < kWin) out[i] = fma(win.w[k], v, out[i]);
        }
    }
}

// ---------------------------------------------------------------- dirty blocks
// dirty[b] = 1 iff image and target differ anywhere in 32x32 block b.  The
// gradient at a pixel depends on images within 10 px (two 5-px windows), the SSIM
// map within 5 px: blocks farther than one block from every dirty block have an
// exactly-1 SSIM map, zero L1 and a mathematically zero gradient.
template <typename T>
__global__ void __launch_bounds__(kLNT) loss_dirty_kernel(const T* __restrict__ y, const T* __restrict__ g,
                                                          int H, int W, uint8_t* __restrict__ dirty) {
    const int x0 = blockIdx.x * kLT, y0 = blockIdx.y * kLT;
    int d = 0;
    // chunk by chunk with a block vote: a block that differs (most blocks, once the
    // refit is under way) stops after its first chunk; kDU values per thread per
    // chunk (all loads in flight before the compares) keep the votes few
    constexpr int kDU = 4;
    for (int c0 = 0; c0 < kLT * kLT * 3 && !d; c0 += kLNT * kDU) {
        T yv[kDU], gv[kDU];
        bool ok[kDU];
#pragma unroll
        for (int u = 0; u < kDU; ++u) {
            const int i = c0 + u * kLNT + threadIdx.x;
            const int p = i / 3, ch = i - 3 * (i / 3);
            const int gy = y0 + p / kLT, gx = x0 + p % kLT;
            ok[u] = i < kLT * kLT * 3 && gy < H && gx < W;
            const int64_t o = ((int64_t)gy * W + gx) * 3 + ch;
            yv[u] = ok[u] ? y[o] : T(0);
            gv[u] = ok[u] ? g[o] : T(0);
        }
        int di = 0;
#pragma unroll
        for (int u = 0; u < kDU; ++u) di |= ok[u] && yv[u] != gv[u];
        d = __syncthreads_or(di);
    }
    if (threadIdx.x == 0) dirty[blockIdx.y * gridDim.x + blockIdx.x] = (uint8_t)d;
}

__device__ __forceinline__ bool near_dirty(const uint8_t* __restrict__ dirty, int r) {
    const int bx = blockIdx.x, by = blockIdx.y;
    for (int yy = max(0, by - r); yy <= min((int)gridDim.y - 1, by + r); ++yy)
        for (int xx = max(0, bx - r); xx <= min((int)gridDim.x - 1, bx + r); ++xx)
            if (dirty[yy * gridDim.x + xx]) return true;
    return false;
}

// Final reduction of the per-block partials (formerly pass C), run by the last
// pass-A block to finish: a fixed assignment of blocks to threads and a fixed
// reduction tree, so the result is deterministic regardless of which block it is.
struct LossTail {
    unsigned* ticket;  // per-stream counter, zero between launches (the last block resets it)
    double n, lam;
    bool ssim_valid;
    double* out3;
};

__device__ void loss_tail(const double* __restrict__ part, int nb, const LossTail& lt, double* red) {
    __shared__ unsigned s_last;
    __threadfence();  // this block's partial is visible before its ticket
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(lt.ticket, 1u) == (unsigned)nb - 1u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < nb; i += kLNT) {
        a += __ldcg(&part[2 * i]);
        b += __ldcg(&part[2 * i + 1]);
    }
    block_sum2(a, b, red);
    if (threadIdx.x == 0) {
        const double l1 = a / lt.n;
        const double ss = lt.ssim_valid ? b / lt.n : __longlong_as_double(0x7ff8000000000000ll);
        lt.out3[0] = l1;
        lt.out3[1] = ss;
        lt.out3[2] = lt.lam == 0.0 ? l1 : (1.0 - lt.lam) * l1 + lt.lam * (1.0 - ss);
        *lt.ticket = 0u;
    }
}

// 4- or 8-byte asynchronous global -> shared copy (LDGSTS); `in` false zero-fills
template <typename E>
__device__ __forceinline__ void cp_async_elem(E* dst, const E* src, bool in) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(d), "l"(src), "n"(sizeof(E)),
                 "r"(in ? (int)sizeof(E) : 0)
                 : "memory");
}

// 16-byte asynchronous copy; `in` false zero-fills
__device__ __forceinline__ void cp_async16_z(void* dst, const void* src, bool in) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(in ? 16 : 0) : "memory");
}

// ---------------------------------------------------------------- pass A
template <bool SSIM, typename T, typename MT>
__global__ void __launch_bounds__(kLNT, kLossCTAs) loss_pass_a(const T* __restrict__ y, const T* __restrict__ g, int H,
                                                    int W, Window win, MT* __restrict__ maps,
                                                    double* __restrict__ block_part,
                                                    const uint8_t* __restrict__ dirty, LossTail lt) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // input planes in the input type (exact), horizontal sums in fp64
    double* hs = reinterpret_cast<double*>(smem_raw);  // [5][42][32]
    T* iy = reinterpret_cast<T*>(hs + 5 * kLH * kLT);  // [42][42]
    T* ig = iy + kLH * kLH;                            // [42][42]
    __shared__ double red[2 * kLNT / 32];
    __shared__ double mrow[kLT], mcol[kLT];  // in-image kernel mass per output row / column
    const int t = threadIdx.x;
    const int x0 = blockIdx.x * kLT, y0 = blockIdx.y * kLT;
    const int64_t npix = (int64_t)H * W;
    const int c = t % kLT, r0 = (t / kLT) * kRows;
    if (SSIM && t < kLT) mrow[t] = mass1d(win, y0 + t, H);
    if (SSIM && t >= kLT && t < 2 * kLT) mcol[t - kLT] = mass1d(win, x0 + t - kLT, W);

    // Blocks more than two blocks from any difference: L1 = 0 and the SSIM map is
    // exactly 1 (a1 == b1, a2 == b2 bitwise when y == g over the window); their
    // maps are never read by pass B (which only runs within one block of a
    // difference, reading a 5-px halo).
    if (!near_dirty(dirty, SSIM ? 2 : 0)) {
        if (t == 0) {
            const int vw = min(kLT, W - x0), vh = min(kLT, H - y0);
            const int b = blockIdx.y * gridDim.x + blockIdx.x;
            block_part[2 * b] = 0.0;
            block_part[2 * b + 1] = SSIM ? (double)(vw * vh * 3) : 0.0;
        }
        loss_tail(block_part, gridDim.x * gridDim.y, lt, red);
        return;
    }

    double l1 = 0.0, ss = 0.0;
    double inv_mass[kRows];  // 1 / (kernel mass in the image), per output pixel, all channels
    if (SSIM) {
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kRows; ++i) inv_mass[i] = 1.0 / (mrow[r0 + i] * mcol[c]);
    }
    // a channel's y / g planes (with the halo, zero outside the image) stream into
    // iy / ig with async copies: channel 0 up front, channel c + 1 as soon as the
    // horizontal pass of channel c has consumed the planes, so its load overlaps
    // channel c's vertical pass and SSIM algebra
    // (halo row r, column cc) of element i advanced incrementally (no divisions);
    // 32-bit element offsets (the host checks 3 H W < 2^31)
    auto stage = [&](int ch) {
        int r = t / kLH, cc = t - (t / kLH) * kLH;
        for (int i = t; i < kLH * kLH; i += kLNT) {
            const int gy = y0 - kR + r, gx = x0 - kR + cc;
            const bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
            const uint32_t gi = in ? ((uint32_t)gy * (uint32_t)W + (uint32_t)gx) * 3u + (uint32_t)ch : 0u;
            cp_async_elem(iy + i, y + gi, in);
            cp_async_elem(ig + i, g + gi, in);
            cc += kLNT % kLH;
            r += kLNT / kLH;
            if (cc >= kLH) {
                cc -= kLH;
                ++r;
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (SSIM) stage(0);
    for (int ch = 0; ch < 3; ++ch) {
        if (SSIM) {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();
            // horizontal pass: each item a strip of kHS adjacent outputs of one row
            // from a register-resident segment (squares formed once per input) for
            // one of three moment groups -- y (s1, s11), g (s2, s22), y g (s12) --
            // so the 3 x 336 items spread evenly over the 256 threads; every
            // accumulator keeps its k = 0..10 FMA sequence
            constexpr int kP = kLH * kLT;
            constexpr int kHI = kLH * (kLT / kHS);
            for (int i = t; i < 3 * kHI; i += kLNT) {
                const int kind = i / kHI, ii = i - kind * kHI;
                const int r = ii / (kLT / kHS), c0 = (ii % (kLT / kHS)) * kHS;
                double* out = hs + r * kLT + c0;
                if (kind < 2) {
                    const T* src = (kind == 0 ? iy : ig) + r * kLH + c0;  // s1, s11 / s2, s22
                    double x[kHS + kWin - 1], xx[kHS + kWin - 1];
#pragma unroll
                    for (int j = 0; j < kHS + kWin - 1; ++j) {
                        x[j] = (double)src[j];
                        xx[j] = x[j] * x[j];
                    }
#pragma unroll
                    for (int o = 0; o < kHS; ++o) {
                        double s1 = 0, s11 = 0;
#pragma unroll
                        for (int k = 0; k < kWin; ++k) {
                            s1 = fma(win.w[k], x[o + k], s1);
                            s11 = fma(win.w[k], xx[o + k], s11);
                        }
                        out[kind * kP + o] = s1;
                        out[(2 + kind) * kP + o] = s11;
                    }
                } else {
                    const T* sa = iy + r * kLH + c0;  // s12
                    const T* sb = ig + r * kLH + c0;
                    double xy[kHS + kWin - 1];
#pragma unroll
                    for (int j = 0; j < kHS + kWin - 1; ++j) xy[j] = (double)sa[j] * (double)sb[j];
#pragma unroll
                    for (int o = 0; o < kHS; ++o) {
                        double s12 = 0;
#pragma unroll
                        for (int k = 0; k < kWin; ++k) s12 = fma(win.w[k], xy[o + k], s12);
                        out[4 * kP + o] = s12;
                    }
                }
            }
            __syncthreads();
            if (ch + 1 < 3) stage(ch + 1);  // iy / ig are free until the next horizontal pass
        }
        double m[5][kRows];
        if (SSIM) {
#pragma unroll
            for (int q = 0; q < 5; ++q) vfilter<double>(hs + q * kLH * kLT, r0, c, win, m[q]);
        }
        const int gx = x0 + c;
#pragma unroll
        for (int i = 0; i < kRows; ++i) {
            const int gy = y0 + r0 + i;
            if (gy >= H || gx >= W) continue;
            const int64_t o = ((int64_t)gy * W + gx) * 3 + ch;
            const T fy = y[o], fg = g[o];
            l1 += fabs((double)fy - (double)fg);
            if (SSIM) {
                // three fp64 reciprocals replace the reference's divisions (same formulas)
                const double im = inv_mass[i];
                const double mu1 = m[0][i] * im, mu2 = m[1][i] * im;
                const double var1 = m[2][i] * im - mu1 * mu1;
                const double var2 = m[3][i] * im - mu2 * mu2;
                const double cov = m[4][i] * im - mu1 * mu2;
                const double a1 = 2.0 * mu1 * mu2 + 1e-4, a2 = 2.0 * cov + 9e-4;
                const double b1 = mu1 * mu1 + mu2 * mu2 + 1e-4, b2 = var1 + var2 + 9e-4;
                // one fp64 division: 1/(b1 b2), then 1/b1 = b2 * that and 1/b2 = b1 * that
                const double ib = 1.0 / (b1 * b2), ib1 = b2 * ib, ib2 = b1 * ib;
                const double a12 = a1 * a2;
                ss += a12 * ib;
                const double d_mu1 = 2.0 * (mu2 * a2) * ib - 2.0 * mu1 * a12 * ib * ib1;
                const double d_var1 = -a12 * ib * ib2;
                const double d_cov = 2.0 * a1 * ib;
                // channel-planar maps ([map][ch][pixel]) keep pass B's halo loads coalesced
                const int64_t mo = (int64_t)ch * npix + (int64_t)gy * W + gx;
                maps[mo] = (MT)((d_mu1 - 2.0 * d_var1 * mu1 - d_cov * mu2) * im);
                maps[npix * 3 + mo] = (MT)(d_var1 * im);
                maps[2 * npix * 3 + mo] = (MT)(d_cov * im);
            }
        }
        if (SSIM) __syncthreads();  // shared planes are reused by the next channel
    }
    block_sum2(l1, ss, red);
    if (t == 0) {
        const int b = blockIdx.y * gridDim.x + blockIdx.x;
        block_part[2 * b] = l1;
        block_part[2 * b + 1] = ss;
    }
    __syncthreads();  // red[] is reused by the tail
    loss_tail(block_part, gridDim.x * gridDim.y, lt, red);
}

// ---------------------------------------------------------------- pass B
// The separable filter of the three maps runs in MT: fp64 for the fp64 entry
// point, fp32 for the fp32 one (whose maps are already stored in fp32; the
// combination with y and g below stays fp64).
template <bool SSIM, typename T, typename G, typename MT>
__global__ void __launch_bounds__(kLNT, kLossCTAs) loss_pass_b(const T* __restrict__ y, const T* __restrict__ g, int H,
                                                    int W, WindowT<MT> win, double lam,
                                                    const MT* __restrict__ maps,
                                                    const uint8_t* __restrict__ dirty, G* __restrict__ grad) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    MT* hs = reinterpret_cast<MT*>(smem_raw);            // [3][42][32]
    MT* imb = hs + 3 * kLH * kLT;                        // [2][3][42][kMS]: double-buffered map planes
    const int t = threadIdx.x;
    const int x0 = blockIdx.x * kLT, y0 = blockIdx.y * kLT;
    const int64_t npix = (int64_t)H * W;
    const double n = (double)(npix * 3);
    // exact zeros where the gradient is mathematically zero: everywhere when the
    // images are identical (losses.py:127-130), else outside one block of a difference
    // (identical images: no block is dirty, so this is false everywhere)
    const bool any = near_dirty(dirty, SSIM ? 1 : 0);
    const int c = t % kLT, r0 = (t / kLT) * kRows;
    // the next channel's three map planes (with the 5-px halo, zero outside the
    // image) stream into the other buffer while this channel computes
    // Map planes are staged as rows of kMS columns, the halo's first column at kMO:
    // interior tiles of fp32 maps (row starts 16-byte aligned) copy 16-byte chunks
    // of columns x0 - 8 .. x0 + 39 (a third of the copy instructions of element
    // copies), edge tiles copy element by element.
    auto issue = [&](int ch) {
        MT* buf = imb + (ch & 1) * 3 * kLH * kMS;
        const MT* m0 = maps + (int64_t)ch * npix;
        const uint32_t mstride = (uint32_t)(npix * 3);
        const bool vec = sizeof(MT) == 4 && (W & 3) == 0 && x0 >= 8 && x0 + 40 <= W;
        if (vec) {
            for (int i = t; i < kLH * 12; i += kLNT) {
                const int r = i / 12, c4 = i - (i / 12) * 12;
                const int gy = y0 - kR + r;
                const bool in = gy >= 0 && gy < H;
                const uint32_t gi = in ? (uint32_t)gy * (uint32_t)W + (uint32_t)(x0 - 8 + 4 * c4) : 0u;
#pragma unroll
                for (int q = 0; q < 3; ++q) cp_async16_z(buf + q * kLH * kMS + r * kMS + 4 * c4, m0 + q * mstride + gi, in);
            }
        } else {
            int r = t / kLH, cc = t - (t / kLH) * kLH;  // advanced incrementally, as in pass A
            for (int i = t; i < kLH * kLH; i += kLNT) {
                const int gy = y0 - kR + r, gx = x0 - kR + cc;
                const bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
                const uint32_t gi = in ? (uint32_t)gy * (uint32_t)W + (uint32_t)gx : 0u;
#pragma unroll
                for (int q = 0; q < 3; ++q)
                    cp_async_elem(buf + q * kLH * kMS + r * kMS + kMO + cc, m0 + q * mstride + gi, in);
                cc += kLNT % kLH;
                r += kLNT / kLH;
                if (cc >= kLH) {
                    cc -= kLH;
                    ++r;
                }
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (SSIM && any) issue(0);
    const int gx = x0 + c;
    for (int ch = 0; ch < 3; ++ch) {
        // this channel's image / target values, loaded early (used after the filters)
        T fyv[kRows], fgv[kRows];
#pragma unroll
        for (int i = 0; i < kRows; ++i) {
            const int gy = y0 + r0 + i;
            const bool ok = any && gy < H && gx < W;
            const int64_t o = ((int64_t)gy * W + gx) * 3 + ch;
            fyv[i] = ok ? y[o] : T(0);
            fgv[i] = ok ? g[o] : T(0);
        }
        if (SSIM && any) {
            if (ch + 1 < 3) {
                issue(ch + 1);
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            __syncthreads();
            const MT* im = imb + (ch & 1) * 3 * kLH * kMS;
            // horizontal pass in kHS-output strips from register-resident segments
            constexpr int kHI = kLH * (kLT / kHS);
            for (int i = t; i < 3 * kHI; i += kLNT) {  // items (map, row, strip): even spread
                const int q = i / kHI, ii = i - q * kHI;
                const int r = ii / (kLT / kHS), c0 = (ii % (kLT / kHS)) * kHS;
                {
                    const MT* src = im + q * kLH * kMS + r * kMS + kMO + c0;
                    MT x[kHS + kWin - 1];
#pragma unroll
                    for (int j = 0; j < kHS + kWin - 1; ++j) x[j] = src[j];
#pragma unroll
                    for (int o = 0; o < kHS; ++o) {
                        MT s = MT(0);
#pragma unroll
                        for (int k = 0; k < kWin; ++k) s = fma(win.w[k], x[o + k], s);
                        hs[q * kLH * kLT + r * kLT + c0 + o] = s;
                    }
                }
            }
            __syncthreads();
        }
        MT f[3][kRows];
        if (SSIM && any) {
#pragma unroll
            for (int q = 0; q < 3; ++q) vfilter<MT>(hs + q * kLH * kLT, r0, c, win, f[q]);
        }
#pragma unroll
        for (int i = 0; i < kRows; ++i) {
            const int gy = y0 + r0 + i;
            if (gy >= H || gx >= W) continue;
            const int64_t o = ((int64_t)gy * W + gx) * 3 + ch;
            if (!any) {
                grad[o] = G(0);
                continue;
            }
            const T fy = fyv[i], fg = fgv[i];
            // np.sign(y - gt): NaN propagates (a NaN image or target makes the
            // gradient non-finite, so the step is rejected, optimize.py:72-74)
            const double d = (double)fy - (double)fg;
            const double sgn = d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : (d == 0.0 ? 0.0 : d));
            double out = (1.0 - lam) * sgn / n;
            if (SSIM)
                out -= lam * (((double)f[0][i] + 2.0 * (double)fy * (double)f[1][i] + (double)fg * (double)f[2][i]) / n);
            grad[o] = (G)out;
        }
        if (SSIM && any) __syncthreads();
    }
}

static Window make_window() {
    Window w;
    double sum = 0.0;
    for (int i = 0; i < kWin; ++i) {
        const double off = (double)(i - kR);
        w.w[i] = exp(-(off * off) / (2.0 * 1.5 * 1.5));
        sum += w.w[i];
    }
    for (int i = 0; i < kWin; ++i) w.w[i] /= sum;
    return w;
}

}  // namespace rcgs

using namespace rcgs;

// Per-stream zeroed ticket for pass A's tail reduction (the last block resets it, so
// it is zero again for the next launch on that stream; launches on one stream are
// ordered, on different streams they use different tickets).
unsigned* rcgs::stream_ticket(cudaStream_t s) {
    static std::mutex mu;
    static std::unordered_map<cudaStream_t, unsigned*> tickets;
    std::lock_guard<std::mutex> lock(mu);
    auto it = tickets.find(s);
    if (it != tickets.end()) return it->second;
    unsigned* t = nullptr;
    if (cudaMalloc(&t, sizeof(unsigned)) != cudaSuccess || cudaMemset(t, 0, sizeof(unsigned)) != cudaSuccess)
        return nullptr;
    tickets.emplace(s, t);
    return t;
}

// MT: storage type of the three gradient maps between the passes -- fp64 for the
// fp64 entry point, fp32 when the gradient itself is fp32 (halves the maps'
// write + halo-read traffic; every filter sum and the SSIM algebra stay fp64).
template <typename T, typename G, typename MT>
static int loss_grad_impl(const T* d_image, const T* d_target, int32_t height, int32_t width, double lam,
                          double* d_loss3, G* d_grad, void* stream) {
    RCGS_CHECK_ARG(d_image && d_target && d_loss3 && d_grad, "null argument");
    RCGS_CHECK_ARG(height > 0 && width > 0, "expected (H, W, 3) images, got (%d, %d, 3)", height, width);
    RCGS_CHECK_ARG(lam >= 0.0 && lam <= 1.0, "lam must be in [0, 1]");
    RCGS_CHECK_ARG((int64_t)height * width * 9 < ((int64_t)1 << 32), "image too large for 32-bit loss offsets");
    const bool ssim_ok = height >= kWin && width >= kWin;
    RCGS_CHECK_ARG(ssim_ok || lam == 0.0, "images must be at least %dpx on each side for SSIM", kWin);
    cudaStream_t s = as_stream(stream);
    const Window win = make_window();
    const dim3 grid(div_up(width, kLT), div_up(height, kLT));
    const int nb = grid.x * grid.y;
    const int64_t npix = (int64_t)height * width;
    MT* maps = nullptr;
    double* part = nullptr;
    uint8_t* dirty = nullptr;
    RCGS_TRY(dalloc(&part, 2 * nb, s));
    RCGS_TRY(dalloc(&dirty, nb, s));
    LossTail lt;
    lt.ticket = stream_ticket(s);
    RCGS_CHECK_ARG(lt.ticket != nullptr, "loss ticket allocation failed");
    lt.n = (double)(npix * 3);
    lt.lam = lam;
    lt.ssim_valid = ssim_ok;
    lt.out3 = d_loss3;
    loss_dirty_kernel<T><<<grid, kLNT, 0, s>>>(d_image, d_target, height, width, dirty);
    const size_t smem_a = 2 * kLH * kLH * sizeof(T) + 5 * kLH * kLT * sizeof(double);
    const size_t smem_b = 2 * 3 * kLH * kMS * sizeof(MT) + 3 * kLH * kLT * sizeof(MT);
    WindowT<MT> wm;
    for (int k = 0; k < kWin; ++k) wm.w[k] = (MT)win.w[k];
    if (ssim_ok) {
        RCGS_TRY(dalloc(&maps, 3 * npix * 3, s));
        RCGS_CUDA(cudaFuncSetAttribute(loss_pass_a<true, T, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_a));
        RCGS_CUDA(cudaFuncSetAttribute(loss_pass_b<true, T, G, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_b));
        loss_pass_a<true, T, MT><<<grid, kLNT, smem_a, s>>>(d_image, d_target, height, width, win, maps, part, dirty,
                                                            lt);
        RCGS_LAUNCH_CHECK();
        if (lam > 0.0) {
            loss_pass_b<true, T, G, MT><<<grid, kLNT, smem_b, s>>>(d_image, d_target, height, width, wm, lam, maps,
                                                                   dirty, d_grad);
        } else {
            loss_pass_b<false, T, G, MT><<<grid, kLNT, 0, s>>>(d_image, d_target, height, width, wm, lam, maps,
                                                               dirty, d_grad);
        }
        RCGS_LAUNCH_CHECK();
    } else {
        loss_pass_a<false, T, MT><<<grid, kLNT, 0, s>>>(d_image, d_target, height, width, win, nullptr, part,
                                                         dirty, lt);
        loss_pass_b<false, T, G, MT><<<grid, kLNT, 0, s>>>(d_image, d_target, height, width, wm, lam, nullptr,
                                                           dirty, d_grad);
        RCGS_LAUNCH_CHECK();
    }
    dfree(maps, s);
    dfree(part, s);
    dfree(dirty, s);
    return RCGS_OK;
}

extern "C" int rcgs_loss_grad(const float* d_image, const float* d_target, int32_t height, int32_t width,
                              double lam, double* d_loss3, float* d_grad, void* stream) {
    return loss_grad_impl<float, float, float>(d_image, d_target, height, width, lam, d_loss3, d_grad, stream);
}

extern "C" int rcgs_loss_grad_f64(const double* d_image, const double* d_target, int32_t height,
                                  int32_t width, double lam, double* d_loss3, double* d_grad, void* stream) {
    return loss_grad_impl<double, double, double>(d_image, d_target, height, width, lam, d_loss3, d_grad, stream);
}

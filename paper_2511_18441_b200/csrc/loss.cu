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

#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace rcgs {

constexpr int kR = 5;              // window half width
constexpr int kWin = 2 * kR + 1;   // 11
constexpr int kLT = 32;            // output tile edge
constexpr int kLH = kLT + 2 * kR;  // 42
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

// Vertical 11-tap pass for kRows consecutive output rows of one column from a
// horizontally filtered plane h[kLH][kLT] (rows r0 .. r0 + kRows + 9).
__device__ __forceinline__ void vfilter(const double* __restrict__ h, int r0, int c, const Window& win,
                                        double out[kRows]) {
#pragma unroll
    for (int i = 0; i < kRows; ++i) out[i] = 0.0;
#pragma unroll
    for (int rr = 0; rr < kRows + kWin - 1; ++rr) {
        const double v = h[(r0 + rr) * kLT + c];
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
    for (int ch = 0; ch < 3; ++ch) {
        if (SSIM) {
            for (int i = t; i < kLH * kLH; i += kLNT) {
                const int r = i / kLH, cc = i % kLH;
                const int gy = y0 - kR + r, gx = x0 - kR + cc;
                const bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
                const int64_t gi = ((int64_t)gy * W + gx) * 3 + ch;
                iy[i] = in ? y[gi] : T(0);
                ig[i] = in ? g[gi] : T(0);
            }
            __syncthreads();
            // horizontal pass: each thread a strip of kHS adjacent outputs of one row
            // from a register-resident segment (squares formed once per input);
            // every accumulator keeps its k = 0..10 FMA sequence
            constexpr int kP = kLH * kLT;
            for (int i = t; i < kLH * (kLT / kHS); i += kLNT) {
                const int r = i / (kLT / kHS), c0 = (i % (kLT / kHS)) * kHS;
                double* out = hs + r * kLT + c0;
                {
                    const T* src = iy + r * kLH + c0;  // s1, s11 (image)
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
                        out[o] = s1;
                        out[2 * kP + o] = s11;
                    }
                }
                {
                    const T* src = ig + r * kLH + c0;  // s2, s22 (target)
                    double x[kHS + kWin - 1], xx[kHS + kWin - 1];
#pragma unroll
                    for (int j = 0; j < kHS + kWin - 1; ++j) {
                        x[j] = (double)src[j];
                        xx[j] = x[j] * x[j];
                    }
#pragma unroll
                    for (int o = 0; o < kHS; ++o) {
                        double s2 = 0, s22 = 0;
#pragma unroll
                        for (int k = 0; k < kWin; ++k) {
                            s2 = fma(win.w[k], x[o + k], s2);
                            s22 = fma(win.w[k], xx[o + k], s22);
                        }
                        out[kP + o] = s2;
                        out[3 * kP + o] = s22;
                    }
                }
                {
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
        }
        double m[5][kRows];
        if (SSIM) {
#pragma unroll
            for (int q = 0; q < 5; ++q) vfilter(hs + q * kLH * kLT, r0, c, win, m[q]);
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

// 4- or 8-byte asynchronous global -> shared copy (LDGSTS); `in` false zero-fills
template <typename E>
__device__ __forceinline__ void cp_async_elem(E* dst, const E* src, bool in) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(d), "l"(src), "n"(sizeof(E)),
                 "r"(in ? (int)sizeof(E) : 0)
                 : "memory");
}

// ---------------------------------------------------------------- pass B
template <bool SSIM, typename T, typename G, typename MT>
__global__ void __launch_bounds__(kLNT, kLossCTAs) loss_pass_b(const T* __restrict__ y, const T* __restrict__ g, int H,
                                                    int W, Window win, double lam,
                                                    const MT* __restrict__ maps,
                                                    const uint8_t* __restrict__ dirty, G* __restrict__ grad) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* hs = reinterpret_cast<double*>(smem_raw);   // [3][42][32]
    MT* imb = reinterpret_cast<MT*>(hs + 3 * kLH * kLT); // [2][3][42][42]: double-buffered map planes
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
    auto issue = [&](int ch) {
        MT* buf = imb + (ch & 1) * 3 * kLH * kLH;
        for (int i = t; i < kLH * kLH; i += kLNT) {
            const int r = i / kLH, cc = i % kLH;
            const int gy = y0 - kR + r, gx = x0 - kR + cc;
            const bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
            const int64_t gi = in ? (int64_t)ch * npix + (int64_t)gy * W + gx : 0;
#pragma unroll
            for (int q = 0; q < 3; ++q) cp_async_elem(buf + q * kLH * kLH + i, maps + q * npix * 3 + gi, in);
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
            const MT* im = imb + (ch & 1) * 3 * kLH * kLH;
            // horizontal pass in kHS-output strips from register-resident segments
            for (int i = t; i < kLH * (kLT / kHS); i += kLNT) {
                const int r = i / (kLT / kHS), c0 = (i % (kLT / kHS)) * kHS;
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const MT* src = im + q * kLH * kLH + r * kLH + c0;
                    double x[kHS + kWin - 1];
#pragma unroll
                    for (int j = 0; j < kHS + kWin - 1; ++j) x[j] = (double)src[j];
#pragma unroll
                    for (int o = 0; o < kHS; ++o) {
                        double s = 0.0;
#pragma unroll
                        for (int k = 0; k < kWin; ++k) s = fma(win.w[k], x[o + k], s);
                        hs[q * kLH * kLT + r * kLT + c0 + o] = s;
                    }
                }
            }
            __syncthreads();
        }
        double f[3][kRows];
        if (SSIM && any) {
#pragma unroll
            for (int q = 0; q < 3; ++q) vfilter(hs + q * kLH * kLT, r0, c, win, f[q]);
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
            if (SSIM) out -= lam * ((f[0][i] + 2.0 * (double)fy * f[1][i] + (double)fg * f[2][i]) / n);
            grad[o] = (G)out;
        }
        if (SSIM && any) __syncthreads();
    }
}

// ---------------------------------------------------------------- fused loss
// One kernel for the dirty test, pass A and pass B: a CTA walks a strip of kSW
// output columns of one channel down a segment of rows, kB rows per band, with
// rings in shared memory so every row is filtered once per strip:
//   input band j (rows [12j+10, 12j+22) of the segment) -> ring (prefetched with
//   cp.async one band ahead);
//   step 2: vertical 11-tap filter of y, g, y^2, g^2, y g (fp64) for the map rows
//           [12k+5, 12k+17) over kIW input columns (register sliding window);
//   step 3: horizontal filter -> the five moments at kMW map columns -> SSIM map
//           (summed over the strip's own pixels) and the three gradient maps
//           M1..M3 (losses.py:104-115, collapsed as in the header) -> map ring;
//   step 4: separable filter of M1..M3 (MT precision) for the output rows
//           [12i, 12i+12) and the gradient (losses.py:118-134), L1 summed.
// The gradient maps never leave shared memory (pass A wrote and pass B re-read
// three full-image maps), and y / g are read once per strip.
// Exactness where the result is exact in the reference: a map pixel whose
// 11x11 input window has y == g everywhere has SSIM exactly 1 (a1 == b1 and
// a2 == b2 bitwise, so the reference's division is 1); an output pixel whose
// 21x21 window has y == g everywhere gets an exact 0 (the reference leaves
// round-off residue there, and returns exact zeros for identical images,
// losses.py:127-130).  The windows are tracked with per-pixel difference flags
// that go through the same two separable passes (OR instead of FMA).
namespace fl {
constexpr int kSW = 64;                        // output columns per strip
constexpr int kB = 12;                         // rows per band
constexpr int kMW = kSW + 2 * kR;              // 74 map columns (col mc <-> x0 - 5 + mc)
constexpr int kMS = 76;                        // map columns the 4-wide strips of step 3 cover (2 spare)
constexpr int kIW = kMW + 2 * kR;              // 84 input columns (col ic <-> x0 - 10 + ic)
constexpr int kIR = 3 * kB;                    // input ring rows: bands j-1, j and the prefetched j+1
constexpr int kMR = 2 * kB;                    // map ring rows: bands k-1, k
constexpr int kNT = 256;
constexpr int kVG = 4;                         // map rows per thread in step 2 (three row groups)
constexpr int kHS4 = 4;                        // adjacent outputs per thread in the horizontal passes
// bank skew for rows read as 4-wide strips (one pad word per 16)
__host__ __device__ constexpr int skew(int c) { return c + (c >> 4); }
constexpr int kIWs = 92;                       // >= skew(kMS + 2 kR - 1) + 1: the strips read 2 spare columns
constexpr int kMWs = 82;                       // >= skew(kMS - 1) + 1
static_assert(skew(kMS + 2 * kR - 1) < kIWs && skew(kMS - 1) < kMWs, "skewed rows");
constexpr int kVR = 3 * kMWs + 11;             // vmap row stride: 1 mod 32 words (fp32), so the two
                                               // rows of a warp in step 4b use disjoint banks
constexpr int kG4 = 96;                        // step 4a: threads per row group (warp aligned)
constexpr int kR4 = kB / 2;                    // step 4a: rows per thread (two groups)
static_assert(kMW <= kG4 && 2 * kG4 <= kNT, "step 4a mapping");
static_assert(kB % kVG == 0 && (kB / kVG) * kIW <= kNT && (kMS / kHS4) * kB <= kNT && 3 * kMS <= kNT &&
                  (kSW / kHS4) * kB <= kNT,
              "threads");

template <typename T, typename MT>
struct Smem {
    T in_y[kIR][kIW], in_g[kIR][kIW];          // input ring (col ic <-> x0 - 10 + ic)
    double vmom[kB][5][kIWs];                  // step 2 -> 3: vertically filtered moments (skewed)
    MT maps[kMR][3][kMWs];                     // map ring (col mc <-> x0 - 5 + mc, skewed)
    MT vmap[kB][kVR];                          // step 4a -> 4b: [q * kMWs + skew(mc)] per row
    double inv_mcol[kMWs];                     // (skewed)
    uint8_t vd[kB][kIW + 4];                   // (2 spare columns read by the last strip)
    uint8_t mflag[kMR][kMS];                   // map pixel's 11x11 window has a difference
    uint8_t vflag[kB][kMS];                    // step 4a: a flagged map pixel within +-5 rows
    double red[2 * kNT / 32];
};

struct Args {
    int H, W, ch_count;
    int seg_rows, nseg, nstrip;
    double lam, n, inv_n, inv_full;
    bool grad_ssim;
    double* part;                              // 2 per job
    LossTail lt;
};

__device__ __forceinline__ int mod(int a, int m) { return ((a % m) + m) % m; }
__device__ __forceinline__ uint32_t win11(uint32_t bits, int o) { return (bits >> o) & 0x7ffu; }

}  // namespace fl

// W2: the window in MT (float for the fp32 entry point)
template <typename MT>
struct WindowT {
    MT w[kWin];
};

template <typename T, typename G, typename MT>
__global__ void __launch_bounds__(fl::kNT, sizeof(MT) == 4 ? 2 : 1)
    loss_fused_kernel(const T* __restrict__ y, const T* __restrict__ g, Window win, WindowT<MT> wm, fl::Args a,
                      G* __restrict__ grad) {
    using namespace fl;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem<T, MT>& sm = *reinterpret_cast<Smem<T, MT>*>(smem_raw);
    const int t = threadIdx.x;
    // job = (strip, segment, channel), channel fastest: the three channel jobs of a
    // strip read the same lines, adjacent in time (L2)
    const int job = blockIdx.x;
    const int ch = job % 3, seg = (job / 3) % a.nseg, strip = job / (3 * a.nseg);
    const int H = a.H, W = a.W;
    const int x0 = strip * kSW;
    const int R0 = seg * a.seg_rows, R1 = min(H, R0 + a.seg_rows);
    const int nb = (R1 - R0 + kB - 1) / kB;

    if (t < kMS) {
        const int gx = x0 - kR + t;
        sm.inv_mcol[skew(t)] = (t < kMW && gx >= 0 && gx < W) ? 1.0 / mass1d(win, gx, W) : 0.0;
    }
    // the spare columns the last 4-wide strip reads (their outputs are never used)
    for (int e = t; e < kB * 5; e += kNT) {
        const int rr = e / 5, q = e % 5;
        for (int c = kIW; c < kMS + 2 * kR; ++c) sm.vmom[rr][q][skew(c)] = 0.0;
    }
    if (t < kB) {
        for (int c = kIW; c < kIW + 4; ++c) sm.vd[t][c] = 0;
    }
    // input band j: segment rows [12j + 10, 12j + 22) -> ring rows [12 (j mod 3), +12)
    auto load_band = [&](int j) {
        const int rbase = mod(j, 3) * kB;
        for (int e = t; e < kB * kIW; e += kNT) {
            const int rr = e / kIW, ic = e - rr * kIW;
            const int gy = R0 + kB * j + 10 + rr, gx = x0 - 2 * kR + ic;
            const bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
            const int64_t o = in ? ((int64_t)gy * W + gx) * 3 + ch : 0;
            cp_async_elem(&sm.in_y[rbase + rr][ic], y + o, in);
            cp_async_elem(&sm.in_g[rbase + rr][ic], g + o, in);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    double l1 = 0.0, ss = 0.0;

    // step 2 + 3 for map band k (segment rows [12k+5, 12k+17))
    auto map_band = [&](int k) {
        if (t < (kB / kVG) * kIW) {
            const int ic = t % kIW, gp = t / kIW;
            double acc[5][kVG];
#pragma unroll
            for (int q = 0; q < 5; ++q)
#pragma unroll
                for (int o = 0; o < kVG; ++o) acc[q][o] = 0.0;
            uint32_t dbits = 0;
            // ring row of tap 0 of output 0 (segment row 12k + 4gp); rows wrap once at most
            const int rb = mod(kB * k + kVG * gp - 10, kIR);
#pragma unroll
            for (int q = 0; q < kVG + kWin - 1; ++q) {
                const int rr = rb + q >= kIR ? rb + q - kIR : rb + q;
                const T ty = sm.in_y[rr][ic], tg = sm.in_g[rr][ic];
                dbits |= (uint32_t)(ty != tg) << q;
                const double yv = (double)ty, gv = (double)tg;
                const double v[5] = {yv, gv, yv * yv, gv * gv, yv * gv};
#pragma unroll
                for (int o = 0; o < kVG; ++o) {
                    const int kk = q - o;
                    if (kk >= 0 && kk < kWin) {
#pragma unroll
                        for (int m = 0; m < 5; ++m) acc[m][o] = fma(win.w[kk], v[m], acc[m][o]);
                    }
                }
            }
#pragma unroll
            for (int o = 0; o < kVG; ++o) {
                const int rr = kVG * gp + o;
#pragma unroll
                for (int m = 0; m < 5; ++m) sm.vmom[rr][m][skew(ic)] = acc[m][o];
                sm.vd[rr][ic] = win11(dbits, o) != 0u;
            }
        }
        __syncthreads();
        if (t < (kMS / kHS4) * kB) {
            // strips 0..15 of a row in one half-warp (the 8-byte loads of a half-warp
            // are conflict-free on the skewed rows), the 3 remaining strips after them
            const int rr = t < 16 * kB ? t >> 4 : (t - 16 * kB) / 3;
            const int s = t < 16 * kB ? t & 15 : 16 + (t - 16 * kB) % 3;
            const int m = kB * k + 5 + rr;  // segment map row
            const int gy = R0 + m;
            const bool row_in = gy >= 0 && gy < H;
            double mo[5][kHS4];
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                double v[kHS4 + kWin - 1];
#pragma unroll
                for (int j = 0; j < kHS4 + kWin - 1; ++j) v[j] = sm.vmom[rr][q][skew(kHS4 * s + j)];
#pragma unroll
                for (int o = 0; o < kHS4; ++o) {
                    double acc = 0.0;
#pragma unroll
                    for (int kk = 0; kk < kWin; ++kk) acc = fma(win.w[kk], v[o + kk], acc);
                    mo[q][o] = acc;
                }
            }
            uint32_t fbits = 0;
#pragma unroll
            for (int j = 0; j < kHS4 + kWin - 1; ++j) fbits |= (uint32_t)sm.vd[rr][kHS4 * s + j] << j;
            const double inv_mrow =
                !row_in ? 0.0 : (gy >= kR && gy < H - kR) ? a.inv_full : 1.0 / mass1d(win, gy, H);
            const int mrr = mod(m - 5, kMR);
            const bool row_core = m >= 0 && m < R1 - R0;
#pragma unroll
            for (int o = 0; o < kHS4; ++o) {
                const int mc = kHS4 * s + o;
                const int gx = x0 - kR + mc;
                const bool in = row_in && mc < kMW && gx >= 0 && gx < W;
                const bool dirty = win11(fbits, o) != 0u;
                double M1 = 0.0, M2 = 0.0, M3 = 0.0;
                if (in) {
                    const double im = inv_mrow * sm.inv_mcol[skew(mc)];
                    const double mu1 = mo[0][o] * im, mu2 = mo[1][o] * im;
                    const double var1 = mo[2][o] * im - mu1 * mu1;
                    const double var2 = mo[3][o] * im - mu2 * mu2;
                    const double cov = mo[4][o] * im - mu1 * mu2;
                    const double a1 = 2.0 * mu1 * mu2 + 1e-4, a2 = 2.0 * cov + 9e-4;
                    const double b1 = mu1 * mu1 + mu2 * mu2 + 1e-4, b2 = var1 + var2 + 9e-4;
                    const double ib = 1.0 / (b1 * b2), ib1 = b2 * ib, ib2 = b1 * ib;
                    const double a12 = a1 * a2;
                    if (row_core && mc >= kR && mc < kR + kSW) ss += dirty ? a12 * ib : 1.0;
                    const double d_mu1 = 2.0 * (mu2 * a2) * ib - 2.0 * mu1 * a12 * ib * ib1;
                    const double d_var1 = -a12 * ib * ib2;
                    const double d_cov = 2.0 * a1 * ib;
                    M1 = (d_mu1 - 2.0 * d_var1 * mu1 - d_cov * mu2) * im;
                    M2 = d_var1 * im;
                    M3 = d_cov * im;
                }
                sm.maps[mrr][0][skew(mc)] = (MT)M1;
                sm.maps[mrr][1][skew(mc)] = (MT)M2;
                sm.maps[mrr][2][skew(mc)] = (MT)M3;
                sm.mflag[mrr][mc] = in && dirty;
            }
        }
    };

    // prologue: input bands -2, -1 (and 0 prefetched), map band -1
    load_band(-2);
    load_band(-1);
    load_band(0);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    map_band(-1);
    for (int i = 0; i < nb; ++i) {
        load_band(i + 1);  // into band i-2's slot (last read in iteration i-1)
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();  // band i landed; map band i-1 written
        map_band(i);
        __syncthreads();
        // step 4a: vertical filter of the maps for output rows [12i, 12i+12)
        if (a.grad_ssim && t < 2 * kG4 && t % kG4 < kMW) {
            const int mc = t % kG4, gp = t / kG4;  // rows kR4 gp .. kR4 gp + kR4 - 1
            MT f[3][kR4];
#pragma unroll
            for (int q = 0; q < 3; ++q)
#pragma unroll
                for (int o = 0; o < kR4; ++o) f[q][o] = MT(0);
            uint32_t fb = 0;
            const int mb = mod(kB * i + kR4 * gp - kR - 5, kMR);  // ring row of segment map row 12i + 6gp - 5
#pragma unroll
            for (int q = 0; q < kR4 + kWin - 1; ++q) {
                const int mr = mb + q >= kMR ? mb + q - kMR : mb + q;
                const MT v0 = sm.maps[mr][0][skew(mc)], v1 = sm.maps[mr][1][skew(mc)], v2 = sm.maps[mr][2][skew(mc)];
                fb |= (uint32_t)sm.mflag[mr][mc] << q;
#pragma unroll
                for (int o = 0; o < kR4; ++o) {
                    const int kk = q - o;
                    if (kk >= 0 && kk < kWin) {
                        f[0][o] = fma(wm.w[kk], v0, f[0][o]);
                        f[1][o] = fma(wm.w[kk], v1, f[1][o]);
                        f[2][o] = fma(wm.w[kk], v2, f[2][o]);
                    }
                }
            }
#pragma unroll
            for (int o = 0; o < kR4; ++o) {
#pragma unroll
                for (int q = 0; q < 3; ++q) sm.vmap[kR4 * gp + o][q * kMWs + skew(mc)] = f[q][o];
                sm.vflag[kR4 * gp + o][mc] = win11(fb, o) != 0u;
            }
        }
        __syncthreads();
        // step 4b: horizontal filter + gradient for output rows [12i, 12i+12)
        if (t < (kSW / kHS4) * kB) {
            const int rr = t / (kSW / kHS4), s = t % (kSW / kHS4);
            const int r = kB * i + rr;
            const int gy = R0 + r;
            if (gy < R1) {
                double f[3][kHS4];
                uint32_t fb = 0;
                if (a.grad_ssim) {
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        MT v[kHS4 + kWin - 1];
#pragma unroll
                        for (int j = 0; j < kHS4 + kWin - 1; ++j) v[j] = sm.vmap[rr][q * kMWs + skew(kHS4 * s + j)];
#pragma unroll
                        for (int o = 0; o < kHS4; ++o) {
                            MT acc = MT(0);
#pragma unroll
                            for (int kk = 0; kk < kWin; ++kk) acc = fma(wm.w[kk], v[o + kk], acc);
                            f[q][o] = (double)acc;
                        }
                    }
#pragma unroll
                    for (int j = 0; j < kHS4 + kWin - 1; ++j) fb |= (uint32_t)sm.vflag[rr][kHS4 * s + j] << j;
                }
                const int ir = mod(r - 10, kIR);
                const double cl1 = (1.0 - a.lam) * a.inv_n, cs = a.lam * a.inv_n;
#pragma unroll
                for (int o = 0; o < kHS4; ++o) {
                    const int c = kHS4 * s + o;
                    const int gx = x0 + c;
                    if (gx >= W) continue;
                    const T fy = sm.in_y[ir][c + 2 * kR], fg = sm.in_g[ir][c + 2 * kR];
                    const double d = (double)fy - (double)fg;
                    l1 += fabs(d);
                    // np.sign(y - gt): NaN propagates (optimize.py:72-74 rejects the step)
                    const double sgn = d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : (d == 0.0 ? 0.0 : d));
                    double out = cl1 * sgn;
                    if (a.grad_ssim) {
                        if (win11(fb, o) == 0u) {
                            out = 0.0;  // 21x21 window without a difference: exactly zero
                        } else {
                            out -= cs * (f[0][o] + 2.0 * (double)fy * f[1][o] + (double)fg * f[2][o]);
                        }
                    }
                    grad[((int64_t)gy * W + gx) * 3 + ch] = (G)out;
                }
            }
        }
        __syncthreads();  // vmom / vmap / ring slots are reused by the next band
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    block_sum2(l1, ss, sm.red);
    if (t == 0) {
        a.part[2 * job] = l1;
        a.part[2 * job + 1] = ss;
    }
    __syncthreads();
    loss_tail(a.part, gridDim.x, a.lt, sm.red);
}

// Images smaller than the SSIM window (lam must be 0): L1 and its sign gradient.
template <typename T, typename G>
__global__ void __launch_bounds__(kLNT) loss_l1_kernel(const T* __restrict__ y, const T* __restrict__ g, int64_t n3,
                                                       double* __restrict__ part, G* __restrict__ grad, LossTail lt) {
    __shared__ double red[2 * kLNT / 32];
    double l1 = 0.0, zero = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)kLNT + threadIdx.x; i < n3; i += (int64_t)gridDim.x * kLNT) {
        const double d = (double)y[i] - (double)g[i];
        l1 += fabs(d);
        const double sgn = d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : (d == 0.0 ? 0.0 : d));
        grad[i] = (G)((1.0 - lt.lam) * sgn / lt.n);
    }
    block_sum2(l1, zero, red);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = l1;
        part[2 * blockIdx.x + 1] = 0.0;
    }
    __syncthreads();
    loss_tail(part, gridDim.x, lt, red);
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
    const size_t smem_b = 2 * 3 * kLH * kLH * sizeof(MT) + 3 * kLH * kLT * sizeof(double);
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
            loss_pass_b<true, T, G, MT><<<grid, kLNT, smem_b, s>>>(d_image, d_target, height, width, win, lam, maps,
                                                                   dirty, d_grad);
        } else {
            loss_pass_b<false, T, G, MT><<<grid, kLNT, 0, s>>>(d_image, d_target, height, width, win, lam, maps,
                                                               dirty, d_grad);
        }
        RCGS_LAUNCH_CHECK();
    } else {
        loss_pass_a<false, T, MT><<<grid, kLNT, 0, s>>>(d_image, d_target, height, width, win, nullptr, part,
                                                         dirty, lt);
        loss_pass_b<false, T, G, MT><<<grid, kLNT, 0, s>>>(d_image, d_target, height, width, win, lam, nullptr,
                                                           dirty, d_grad);
        RCGS_LAUNCH_CHECK();
    }
    dfree(maps, s);
    dfree(part, s);
    dfree(dirty, s);
    return RCGS_OK;
}

// The fused path (default; RCGS_LOSS_LEGACY=1 selects the three-kernel path above
// for A/B measurements).
static bool loss_legacy() {
    static const bool v = [] {
        const char* e = getenv("RCGS_LOSS_LEGACY");
        return e && atoi(e) != 0;
    }();
    return v;
}

template <typename T, typename G, typename MT>
static int loss_fused_impl(const T* d_image, const T* d_target, int32_t height, int32_t width, double lam,
                           double* d_loss3, G* d_grad, void* stream) {
    RCGS_CHECK_ARG(d_image && d_target && d_loss3 && d_grad, "null argument");
    RCGS_CHECK_ARG(height > 0 && width > 0, "expected (H, W, 3) images, got (%d, %d, 3)", height, width);
    RCGS_CHECK_ARG(lam >= 0.0 && lam <= 1.0, "lam must be in [0, 1]");
    const bool ssim_ok = height >= kWin && width >= kWin;
    RCGS_CHECK_ARG(ssim_ok || lam == 0.0, "images must be at least %dpx on each side for SSIM", kWin);
    cudaStream_t s = as_stream(stream);
    const Window win = make_window();
    const int64_t npix = (int64_t)height * width;
    LossTail lt;
    lt.ticket = stream_ticket(s);
    RCGS_CHECK_ARG(lt.ticket != nullptr, "loss ticket allocation failed");
    lt.n = (double)(npix * 3);
    lt.lam = lam;
    lt.ssim_valid = ssim_ok;
    lt.out3 = d_loss3;
    double* part = nullptr;
    if (!ssim_ok) {
        const int nb = (int)std::min<int64_t>(div_up(npix * 3, kLNT), 1024);
        RCGS_TRY(dalloc(&part, 2 * nb, s));
        loss_l1_kernel<T, G><<<nb, kLNT, 0, s>>>(d_image, d_target, npix * 3, part, d_grad, lt);
        RCGS_LAUNCH_CHECK();
        dfree(part, s);
        return RCGS_OK;
    }
    using SM = fl::Smem<T, MT>;
    auto kern = loss_fused_kernel<T, G, MT>;
    static int slots = 0;  // resident CTAs on the device (per instantiation)
    if (slots == 0) {
        RCGS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SM)));
        int dev = 0, sms = 0, per_sm = 0;
        RCGS_CUDA(cudaGetDevice(&dev));
        RCGS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        RCGS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, fl::kNT, sizeof(SM)));
        slots = std::max(1, sms * per_sm);
    }
    fl::Args a;
    a.H = height;
    a.W = width;
    a.ch_count = 3;
    a.nstrip = (int)div_up(width, fl::kSW);
    // row segments: about one wave of (strip, segment, channel) jobs over the
    // resident CTA slots (each segment re-filters one 12-row band above it)
    const int bands = (int)div_up(height, fl::kB);
    const int want = std::max(1, std::min(bands, slots / (3 * a.nstrip)));
    static const int max_seg_bands = [] {
        const char* e = getenv("RCGS_LOSS_SEG_BANDS");
        return e ? std::max(1, atoi(e)) : 1 << 20;
    }();
    const int seg_bands = std::min((int)div_up(bands, want), max_seg_bands);
    a.seg_rows = seg_bands * fl::kB;
    a.nseg = (int)div_up(height, a.seg_rows);
    a.lam = lam;
    a.n = lt.n;
    a.inv_n = 1.0 / lt.n;
    double full = 0.0;
    for (int k = 0; k < kWin; ++k) full += win.w[k];
    a.inv_full = 1.0 / full;
    a.grad_ssim = lam > 0.0;
    const int jobs = a.nstrip * a.nseg * 3;
    RCGS_TRY(dalloc(&part, 2 * jobs, s));
    a.part = part;
    a.lt = lt;
    WindowT<MT> wm;
    for (int k = 0; k < kWin; ++k) wm.w[k] = (MT)win.w[k];
    kern<<<jobs, fl::kNT, sizeof(SM), s>>>(d_image, d_target, win, wm, a, d_grad);
    RCGS_LAUNCH_CHECK();
    dfree(part, s);
    return RCGS_OK;
}

extern "C" int rcgs_loss_grad(const float* d_image, const float* d_target, int32_t height, int32_t width,
                              double lam, double* d_loss3, float* d_grad, void* stream) {
    if (loss_legacy())
        return loss_grad_impl<float, float, float>(d_image, d_target, height, width, lam, d_loss3, d_grad, stream);
    return loss_fused_impl<float, float, float>(d_image, d_target, height, width, lam, d_loss3, d_grad, stream);
}

extern "C" int rcgs_loss_grad_f64(const double* d_image, const double* d_target, int32_t height,
                                  int32_t width, double lam, double* d_loss3, double* d_grad, void* stream) {
    if (loss_legacy())
        return loss_grad_impl<double, double, double>(d_image, d_target, height, width, lam, d_loss3, d_grad, stream);
    return loss_fused_impl<double, double, double>(d_image, d_target, height, width, lam, d_loss3, d_grad, stream);
}

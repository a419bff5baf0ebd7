// Stereo depth from re-rendered baselines on the GPU (
// stereo.py:61-219): ZNCC block matching with sub-pixel refinement and the
// left-right check, then disparity -> depth, H/V fusion and the gaussian-depth
// backfill.  Bit-exact to the reference given the same images:
//
// * The (2r+1)^2 box means are scipy.ndimage.uniform_filter(mode="nearest")
//   (scipy 1.18.1, the reference's dependency): per axis (0 then 1) a running
//   SUM over each line -- tmp = sum of the first window in order, then
//   tmp += (new - old) -- with every output tmp / size.  Each line is walked
//   sequentially by one thread, so the rounding sequence is scipy's.
// * Shifting the right image along x copies columns, so the vertical pass of a
//   shifted image is the vertical pass of the unshifted one at column max(x-d,0):
//   only the left*shifted products need a vertical pass per disparity.
// * Per-disparity volumes are laid out [y][x][d]: the threads of a warp walk 32
//   consecutive disparities of the same line, so every step's loads and stores
//   are contiguous.
// * All arithmetic is IEEE fp64 without contraction (-ffp-contract=off is not
//   enough for device code: every op below is an explicit __d*_rn intrinsic).
#include "common.cuh"

namespace rcgs {

struct StereoDims {
    int h, w;      // oriented image (rows matched along x)
    int nd;        // max_disparity + 1 (score entries per pixel)
    int nde;       // min(nd, w): disparities that can be valid
    int nw;        // warps of 32 disparities per row (ceil(nde / 32))
    int r;         // window radius
    double size;   // 2r + 1
    double inv;    // RN(1 / size)
    double floor_v, floor_sq, lr_tol;
};

__device__ __forceinline__ int clampi(int i, int n) { return i < 0 ? 0 : (i >= n ? n - 1 : i); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// RN(t / size) without the general division routine: q = RN(t * RN(1/size)) is
// faithful, the remainder t - q*size is exact in one fma, and RN(q + rem/size
// estimate) is the correctly rounded quotient (Markstein's correction step);
// rcgs_stereo_div_check verifies it against __ddiv_rn on the GPU.
__device__ __forceinline__ double div_size(double t, double size, double inv) {
    const double q = __dmul_rn(t, inv);
    const double rem = __fma_rn(-q, size, t);
    return __fma_rn(rem, inv, q);
}

// Gray planes in the matching orientation (transpose: rows of the match are the
// image columns, stereo.py:207-209): P0 = gray(left), P1 = gray(right),
// P2 = mirror(gray(right)), P3 = mirror(gray(left)) (the LR pass, stereo.py:143).
// gray = mean over channels, numpy order ((r + g) + b) / 3 (stereo.py:87-94).
template <typename T>
__global__ void stereo_gray_kernel(const T* __restrict__ left, const T* __restrict__ right, int ch_l, int ch_r,
                                   int transpose, StereoDims sd, double* __restrict__ planes) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t np = (int64_t)sd.h * sd.w;
    if (i >= np) return;
    const int y = (int)(i / sd.w), x = (int)(i - (int64_t)y * sd.w);
    const int64_t src = transpose ? ((int64_t)x * sd.h + y) : i;  // source image is (H, W) = oriented^T
    auto gray = [&](const T* img, int ch) {
        const T* p = img + src * ch;
        if (ch == 1) return (double)p[0];
        double s = (double)p[0];
        for (int c = 1; c < ch; ++c) s = dadd(s, (double)p[c]);
        return ddiv(s, (double)ch);
    };
    const double gl = gray(left, ch_l), gr = gray(right, ch_r);
    const int64_t mi = (int64_t)y * sd.w + (sd.w - 1 - x);
    planes[i] = gl;
    planes[np + i] = gr;
    planes[2 * np + mi] = gr;
    planes[3 * np + mi] = gl;
}

// One line of scipy's uniform_filter1d(mode="nearest"): tmp = sum of the first
// window (in order), then tmp += (new - old); every output is tmp / size.  val(i)
// reads the line at a clamped index.  Loads are issued kU steps ahead of the
// dependent adds so the walk is bound by the add chain, not by load latency.
template <int kU, class Val, class Emit>
__device__ __forceinline__ void box_line(int n, const StereoDims& sd, Val val, Emit emit) {
    double tmp = 0.0;
    for (int j = -sd.r; j <= sd.r; ++j) tmp = dadd(tmp, val(j));
    emit(0, div_size(tmp, sd.size, sd.inv));
    int i = 1;
    for (; i + kU <= n; i += kU) {
        double vn[kU], vo[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            vn[u] = val(i + u + sd.r);
            vo[u] = val(i + u - sd.r - 1);
        }
        asm volatile("" ::: "memory");  // keep the kU loads in flight together (ptxas sinks them otherwise)
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            tmp = dadd(tmp, dsub(vn[u], vo[u]));
            emit(i + u, div_size(tmp, sd.size, sd.inv));
        }
    }
    for (; i < n; ++i) {
        tmp = dadd(tmp, dsub(val(i + sd.r), val(i - sd.r - 1)));
        emit(i, div_size(tmp, sd.size, sd.inv));
    }
}

// The same line walk with the line streamed through a private shared-memory ring
// by cp.async (8-byte copies, kGA groups of kC elements in flight): the copies
// cannot be sunk next to their use by the compiler, so the walk is bound by the
// add chain even with few lines in flight.  Element k of the stream is the line
// at clamp(k - r); ring slot k % kR, thread stride `ts` (conflict-free).
// Requires kR > 2r + 1 + (kGA + 1) * kC (old values are read from the ring).
constexpr int kRing = 64, kRingC = 8, kRingGA = 4;

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}

__host__ __device__ constexpr int ring_max_radius() { return (kRing - 2 - (kRingGA + 1) * kRingC) / 2; }

template <class Addr, class Xf, class Emit>
__device__ __forceinline__ void box_line_ring(int n, const StereoDims& sd, Addr addr, Xf xf, double* ring, int ts,
                                              Emit emit) {
    const int total = n + 2 * sd.r;
    auto issue = [&](int g) {
#pragma unroll
        for (int u = 0; u < kRingC; ++u) {
            const int k = g * kRingC + u;
            if (k < total) cp_async8(ring + (k % kRing) * ts, addr(clampi(k - sd.r, n)));
        }
        asm volatile("cp.async.commit_group;" ::: "memory");  // one group per call keeps the count uniform
    };
    auto e = [&](int k) { return xf(ring[(k % kRing) * ts]); };
#pragma unroll 1
    for (int g = 0; g < kRingGA; ++g) issue(g);
    double tmp = 0.0;
    const int last = 2 * sd.r;
    const int groups = (total + kRingC - 1) / kRingC;
#pragma unroll 1
    for (int g = 0; g < groups; ++g) {
        issue(g + kRingGA);
        asm volatile("cp.async.wait_group %0;" ::"n"(kRingGA) : "memory");
#pragma unroll
        for (int u = 0; u < kRingC; ++u) {
            const int k = g * kRingC + u;
            if (k >= total) break;
            if (k <= last) {
                tmp = dadd(tmp, e(k));
                if (k == last) emit(0, div_size(tmp, sd.size, sd.inv));
            } else {
                tmp = dadd(tmp, dsub(e(k), e(k - last - 1)));
                emit(k - last, div_size(tmp, sd.size, sd.inv));
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Vertical running box of A, A*A, B, B*B (thread per (column, plane)).
// blockIdx.y = pass (0: left/right, 1: mirrored right/left); gray planes 2p, 2p+1.
__global__ void __launch_bounds__(64) stereo_vbox_planes_kernel(const double* __restrict__ planes, StereoDims sd, double* __restrict__ v4) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 4 * sd.w) return;
    const int64_t np = (int64_t)sd.h * sd.w;
    const int k = i / sd.w, x = i - k * sd.w;
    const double* src = planes + (2 * blockIdx.y + (k >> 1)) * np;
    const bool sq = k & 1;
    double* out = v4 + (4 * blockIdx.y + k) * np + x;
    __shared__ double ring[kRing * 64];
    if (sd.r <= ring_max_radius()) {
        box_line_ring(sd.h, sd, [&](int y) { return src + (int64_t)y * sd.w + x; },
                      [&](double v) { return sq ? dmul(v, v) : v; }, ring + threadIdx.x, 64,
                      [&](int y, double m) { out[(int64_t)y * sd.w] = m; });
        return;
    }
    box_line<32>(sd.h, sd, [&](int y) {
        const double v = src[(int64_t)clampi(y, sd.h) * sd.w + x];
        return sq ? dmul(v, v) : v;
    }, [&](int y, double m) { out[(int64_t)y * sd.w] = m; });
}

// Horizontal running box of the vertical planes VA, VA2 -> box(A), box(A*A)
// (thread per (row, plane)).
__global__ void __launch_bounds__(64) stereo_hbox_left_kernel(const double* __restrict__ v4, StereoDims sd, double* __restrict__ mu_ex) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 2 * sd.h) return;
    const int64_t np = (int64_t)sd.h * sd.w;
    const int k = i / sd.h, y = i - k * sd.h;
    const double* line = v4 + (4 * blockIdx.y + k) * np + (int64_t)y * sd.w;
    double* out = mu_ex + (2 * blockIdx.y + k) * np + (int64_t)y * sd.w;
    __shared__ double ring[kRing * 64];
    if (sd.r <= ring_max_radius()) {
        box_line_ring(sd.w, sd, [&](int x) { return line + x; }, [](double v) { return v; }, ring + threadIdx.x, 64,
                      [&](int x, double m) { out[x] = m; });
        return;
    }
    box_line<32>(sd.w, sd, [&](int x) { return line[clampi(x, sd.w)]; }, [&](int x, double m) { out[x] = m; });
}

// Vertical running box of A * shift_d(B) for every disparity, written [y][x][d]
// (thread per (column, d), d fastest).  shift_d(B)[y, x] = B[y, max(x - d, 0)]
// (stereo.py:110-112).
__global__ void stereo_vbox_products_kernel(const double* __restrict__ planes, StereoDims sd,
                                            double* __restrict__ vab_all) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)sd.w * sd.nde) return;
    const int64_t np = (int64_t)sd.h * sd.w;
    const double* A = planes + (2 * blockIdx.y) * np;
    const double* B = planes + (2 * blockIdx.y + 1) * np;
    double* vab = vab_all + blockIdx.y * np * sd.nd;
    const int x = (int)(i / sd.nde), d = (int)(i - (int64_t)x * sd.nde);
    const int xs = x - d > 0 ? x - d : 0;
    const int64_t pitch = (int64_t)sd.w * sd.nd;  // one row of the volume
    double* out = vab + (int64_t)x * sd.nd + d;
    box_line<8>(sd.h, sd, [&](int y) {
        const int64_t row = (int64_t)clampi(y, sd.h) * sd.w;
        return dmul(A[row + x], B[row + xs]);
    }, [&](int y, double m) { out[(int64_t)y * pitch] = m; });
}

// Per (pixel, warp of 32 disparities): the warp's first maximum and the scores
// around it -- enough to finish np.argmax + the parabolic refinement without the
// (nd, H, W) score volume.
struct ScorePart {
    double best_d, s_best, s_prev, s_next, s_first, s_last;
};

__device__ __forceinline__ bool better(double a, int da, double b, int db) {  // np.argmax order
    const bool na = isnan(a), nb = isnan(b);
    if (na || nb) return na && (!nb || da < db);
    return a > b || (a == b && da < db);
}

// One (row, disparity) walk of the horizontal pass: running boxes of shift_d(VB),
// shift_d(VB2) and V(A*shift_d(B)) along the row and the ZNCC score at every x
// (stereo.py:113-117).  init() sums the first window; score(x, pab_new) advances
// to x (x > 0) and returns the score, -2 where invalid.
struct ScoreWalk {
    const double *vb, *vb2, *mul, *exl, *pab;
    int d, da;
    bool active;
    double t1, t2, t3;
    const StereoDims* sd;

    __device__ __forceinline__ int sh(int x) const {  // column of the shifted image's vertical box (nearest)
        const int c = clampi(x, sd->w) - da;
        return c > 0 ? c : 0;
    }
    __device__ __forceinline__ double pv(int x) const { return pab[(int64_t)clampi(x, sd->w) * sd->nd]; }
    __device__ __forceinline__ void init() {
        t1 = t2 = t3 = 0.0;
        for (int j = -sd->r; j <= sd->r; ++j) {
            const int c = sh(j);
            t1 = dadd(t1, vb[c]);
            t2 = dadd(t2, vb2[c]);
            t3 = dadd(t3, pv(j));
        }
    }
    __device__ __forceinline__ double score(int x, double pnew) {
        if (x > 0) {
            const int cn = sh(x + sd->r), co = sh(x - sd->r - 1);
            t1 = dadd(t1, dsub(vb[cn], vb[co]));
            t2 = dadd(t2, dsub(vb2[cn], vb2[co]));
            t3 = dadd(t3, dsub(pnew, pv(x - sd->r - 1)));
        }
        const double mu_r = div_size(t1, sd->size, sd->inv), ex_r2 = div_size(t2, sd->size, sd->inv);
        const double ex_ab = div_size(t3, sd->size, sd->inv);
        const double mu_l = mul[x];
        const double var_l = dsub(exl[x], dmul(mu_l, mu_l));
        const double var_r = dsub(ex_r2, dmul(mu_r, mu_r));
        const double cov = dsub(ex_ab, dmul(mu_l, mu_r));
        if (!(active && var_l >= sd->floor_v && var_r >= sd->floor_v && x >= d)) return -2.0;
        const double p = dmul(var_l, var_r);
        return ddiv(cov, __dsqrt_rn(p < sd->floor_sq ? sd->floor_sq : p));  // np.maximum keeps a NaN
    }
};

// Horizontal pass + per-warp argmax epilogue.  A warp walks 32 consecutive
// disparities of one row (lanes with d >= nde carry the reference's -2), so its
// loads of the [y][x][d] volume are contiguous; the scores of 32 consecutive x
// are staged in shared memory ([d][x], padded) and each lane then scans the 32
// disparities of one pixel -- no per-step shuffles.  (Packing a lone last
// disparity of 32 rows into one warp, lane = row, was tried: those warps walk
// uncoalesced and became the critical path, 2.5x slower.)
constexpr int kHsWarps = 4;

__global__ void __launch_bounds__(32 * kHsWarps) stereo_hscore_kernel(const double* __restrict__ v4_all,
                                                                      const double* __restrict__ mu_ex_all,
                                                                      const double* __restrict__ vab_all, StereoDims sd,
                                                                      ScorePart* __restrict__ parts_all) {
    __shared__ double stage[kHsWarps][32][33];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t np = (int64_t)sd.h * sd.w;
    const double* v4 = v4_all + 4 * blockIdx.y * np;
    const double* mu_ex = mu_ex_all + 2 * blockIdx.y * np;
    const double* vab = vab_all + blockIdx.y * np * sd.nd;
    ScorePart* parts = parts_all + blockIdx.y * np * sd.nw;
    ScoreWalk wk;
    wk.sd = &sd;
    if (gw >= (int64_t)sd.h * sd.nw) return;  // whole warps exit together
    const int y = (int)(gw / sd.nw);
    wk.d = (int)(gw - (int64_t)y * sd.nw) * 32 + lane;
    wk.active = wk.d < sd.nde;
    wk.da = wk.active ? wk.d : 0;  // inactive lanes read valid memory, results unused
    wk.vb = v4 + 2 * np + (int64_t)y * sd.w;
    wk.vb2 = v4 + 3 * np + (int64_t)y * sd.w;
    wk.mul = mu_ex + (int64_t)y * sd.w;
    wk.exl = mu_ex + np + (int64_t)y * sd.w;
    wk.pab = vab + (int64_t)y * sd.w * sd.nd + wk.da;
    wk.init();
    const int wi = wk.d >> 5;
    ScorePart* out = parts + (int64_t)y * sd.w * sd.nw + wi;
    double(*st)[33] = stage[wl];
    for (int x0 = 0; x0 < sd.w; x0 += 32) {
#pragma unroll 1
        for (int u0 = 0; u0 < 32; u0 += 8) {
            double pn[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) pn[u] = wk.pv(x0 + u0 + u + sd.r);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int x = x0 + u0 + u;
                st[lane][u0 + u] = x < sd.w ? wk.score(x, pn[u]) : -2.0;
            }
        }
        __syncwarp();
        const int x = x0 + lane;
        if (x < sd.w) {  // lane = pixel: first maximum over this warp's 32 disparities
            double bv = st[0][lane];
            int bl = 0;
            for (int k = 1; k < 32; ++k) {
                const double v = st[k][lane];
                if (better(v, k, bv, bl)) {
                    bv = v;
                    bl = k;
                }
            }
            ScorePart pr;
            pr.best_d = (double)(wi * 32 + bl);
            pr.s_best = bv;
            pr.s_prev = st[bl > 0 ? bl - 1 : 0][lane];
            pr.s_next = st[bl < 31 ? bl + 1 : 31][lane];
            pr.s_first = st[0][lane];
            pr.s_last = st[31][lane];
            out[(int64_t)x * sd.nw] = pr;
        }
        __syncwarp();
    }
}

// Finish np.argmax over all disparities and the parabolic refinement of
// stereo.py:121-139 from the per-warp parts.  Scores of d >= nde are -2
// (stereo.py:107-108), as the lanes that produced them.
__global__ void stereo_best_kernel(const ScorePart* __restrict__ parts, StereoDims sd, double* __restrict__ disp) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t np = (int64_t)sd.h * sd.w;
    if (i >= np) return;
    const ScorePart* p = parts + (blockIdx.y * np + i) * sd.nw;
    disp += blockIdx.y * np;
    int wb = 0;
    ScorePart b = p[0];
    for (int k = 1; k < sd.nw; ++k) {
        const ScorePart c = p[k];
        if (better(c.s_best, (int)c.best_d, b.s_best, (int)b.best_d)) {
            b = c;
            wb = k;
        }
    }
    int best = (int)b.best_d;
    const double s0 = b.s_best;
    if (best >= sd.nd) best = sd.nd - 1;  // cannot happen (-2 ties resolve to lower d); defensive
    const int dmax = sd.nd - 1;
    double out = s0 <= -2.0 ? -1.0 : (double)best;
    const int lane = best - wb * 32;
    const double sm = best == 0 ? s0 : (lane > 0 ? b.s_prev : p[wb - 1].s_last);
    double sp;
    if (best >= dmax) sp = s0;
    else if (best + 1 >= sd.nde) sp = -2.0;
    else sp = lane < 31 ? b.s_next : p[wb + 1].s_first;
    const bool refinable = best > 0 && best < dmax && sm > -2.0 && sp > -2.0 && s0 > -2.0;
    const double den = dsub(dadd(sm, sp), dmul(2.0, s0));
    if (refinable && den < -1e-12) {
        double delta = ddiv(dmul(0.5, dsub(sm, sp)), den);
        delta = delta < -0.5 ? -0.5 : (delta > 0.5 ? 0.5 : delta);
        out = dadd((double)best, delta);
    }
    disp[i] = out;
}

// Self-check of div_size against the IEEE division on pseudo-random operands.
__global__ void stereo_div_check_kernel(double size, double inv, int64_t n, uint64_t seed,
                                        unsigned long long* mismatches) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t z = seed + (uint64_t)i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    // mantissa random, exponent in [2^-40, 2^24), sign random
    const uint64_t e = 1023 - 40 + (z >> 58) % 64;
    const double t = __longlong_as_double((long long)((z & 0x000FFFFFFFFFFFFFull) | (e << 52) | ((z >> 57) & 1) << 63));
    if (div_size(t, size, inv) != ddiv(t, size)) atomicAdd(mismatches, 1ull);
}

// Left-right consistency (stereo.py:151-161) and the un-transpose to (H, W).
__global__ void stereo_lr_kernel(const double* __restrict__ dl, const double* __restrict__ dr_mirror, StereoDims sd,
                                 int transpose, double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)sd.h * sd.w) return;
    const int y = (int)(i / sd.w), x = (int)(i - (int64_t)y * sd.w);
    const double d = dl[i];
    double res = -1.0;
    if (d >= 0.0) {
        const double pf = rint(dsub((double)x, d));
        if (pf >= 0.0 && pf < (double)sd.w) {
            const int p = (int)pf;
            const double pd = dr_mirror[(int64_t)y * sd.w + (sd.w - 1 - p)];
            if (pd >= 0.0 && fabs(dsub(d, pd)) <= sd.lr_tol) res = d;
        }
    }
    out[transpose ? ((int64_t)x * sd.h + y) : i] = res;
}

// depth = fx * baseline / disparity where disparity > min (else +inf), H/V fused by
// minimum, holes backfilled from the gaussian depth (stereo.py:164-219).
__global__ void stereo_depth_kernel(const double* __restrict__ disp_h, const double* __restrict__ disp_v, int64_t n,
                                    double fxb, double fyb, double min_disp, const double* __restrict__ fallback,
                                    double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    const double a = disp_h[i], b = disp_v[i];
    const double dh = a > min_disp ? ddiv(fxb, a) : inf;
    const double dv = b > min_disp ? ddiv(fyb, b) : inf;
    double f = dh < dv ? dh : dv;  // np.minimum (no NaN can occur: disparities are finite)
    if (fallback && !isfinite(f)) f = fallback[i];
    out[i] = f;
}

int stereo_match_impl(const void* left, const void* right, int height, int width, int ch_l, int ch_r, int elem_bytes,
                      int transpose, int max_disparity, int radius, double floor_v, double floor_sq, double lr_tol,
                      double* disp, cudaStream_t s) {
    StereoDims sd;
    sd.h = transpose ? width : height;
    sd.w = transpose ? height : width;
    sd.nd = max_disparity + 1;
    sd.nde = sd.nd < sd.w ? sd.nd : sd.w;
    sd.nw = (sd.nde + 31) / 32;
    sd.r = radius;
    sd.size = (double)(2 * radius + 1);
    sd.inv = 1.0 / sd.size;
    sd.floor_v = floor_v;
    sd.floor_sq = floor_sq;
    sd.lr_tol = lr_tol;
    const int64_t np = (int64_t)sd.h * sd.w;
    const int64_t nvol = np * sd.nd;
    // both passes (left/right and the mirrored right/left of the LR check) run in
    // the same launches (blockIdx.y), so the sequential line walks have twice the
    // independent lines in flight
    double *planes = nullptr, *v4 = nullptr, *muex = nullptr, *vab = nullptr, *dd = nullptr;
    ScorePart* parts = nullptr;
    int rc = RCGS_OK;
    if ((rc = dalloc(&planes, 4 * np, s)) || (rc = dalloc(&v4, 8 * np, s)) || (rc = dalloc(&muex, 4 * np, s)) ||
        (rc = dalloc(&vab, 2 * nvol, s)) || (rc = dalloc(&parts, 2 * np * sd.nw, s)) || (rc = dalloc(&dd, 2 * np, s)))
        goto done;
    {
        const int T = 256;
        if (elem_bytes == 4)
            stereo_gray_kernel<float><<<div_up(np, T), T, 0, s>>>((const float*)left, (const float*)right, ch_l,
                                                                  ch_r, transpose, sd, planes);
        else
            stereo_gray_kernel<double><<<div_up(np, T), T, 0, s>>>((const double*)left, (const double*)right,
                                                                   ch_l, ch_r, transpose, sd, planes);
        stereo_vbox_planes_kernel<<<dim3(div_up(4 * sd.w, 64), 2), 64, 0, s>>>(planes, sd, v4);
        stereo_hbox_left_kernel<<<dim3(div_up(2 * sd.h, 64), 2), 64, 0, s>>>(v4, sd, muex);
        stereo_vbox_products_kernel<<<dim3(div_up((int64_t)sd.w * sd.nde, T), 2), T, 0, s>>>(planes, sd, vab);
        stereo_hscore_kernel<<<dim3(div_up((int64_t)sd.h * sd.nw * 32, 32 * kHsWarps), 2), 32 * kHsWarps, 0, s>>>(
            v4, muex, vab, sd, parts);
        stereo_best_kernel<<<dim3(div_up(np, T), 2), T, 0, s>>>(parts, sd, dd);
        stereo_lr_kernel<<<div_up(np, T), T, 0, s>>>(dd, dd + np, sd, transpose, disp);
        rc = cudaGetLastError() == cudaSuccess ? RCGS_OK : RCGS_ECUDA;
        if (rc) set_error("stereo kernels failed to launch");
    }
done:
    dfree(planes, s);
    dfree(v4, s);
    dfree(muex, s);
    dfree(vab, s);
    dfree(parts, s);
    dfree(dd, s);
    return rc;
}

}  // namespace rcgs

using namespace rcgs;

extern "C" int rcgs_stereo_match(const void* d_left, const void* d_right, int32_t height, int32_t width,
                                 int32_t channels_left, int32_t channels_right, int32_t elem_bytes, int32_t transpose, int32_t max_disparity,
                                 int32_t window_radius, double variance_floor, double variance_floor_sq,
                                 double lr_tolerance, double* d_disparity, void* stream) {
    RCGS_CHECK_ARG(d_left && d_right && d_disparity, "null argument");
    RCGS_CHECK_ARG(height > 0 && width > 0, "empty stereo image %dx%d", height, width);
    RCGS_CHECK_ARG(channels_left >= 1 && channels_right >= 1, "channels must be >= 1");
    RCGS_CHECK_ARG(elem_bytes == 4 || elem_bytes == 8, "elements must be float32 or float64");
    RCGS_CHECK_ARG(max_disparity >= 0 && window_radius >= 0, "negative max_disparity / window_radius");
    return stereo_match_impl(d_left, d_right, height, width, channels_left, channels_right, elem_bytes, transpose != 0, max_disparity,
                             window_radius, variance_floor, variance_floor_sq, lr_tolerance, d_disparity,
                             as_stream(stream));
}

extern "C" int rcgs_stereo_div_check(int32_t size, int64_t n, uint64_t seed, int64_t* h_mismatches, void* stream) {
    RCGS_CHECK_ARG(size >= 1 && n >= 0 && h_mismatches, "bad arguments");
    cudaStream_t s = as_stream(stream);
    unsigned long long* cnt = nullptr;
    RCGS_TRY(dalloc(&cnt, 1, s));
    RCGS_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
    if (n > 0) {
        stereo_div_check_kernel<<<div_up(n, 256), 256, 0, s>>>((double)size, 1.0 / (double)size, n, seed, cnt);
        RCGS_LAUNCH_CHECK();
    }
    unsigned long long h = 0;
    RCGS_CUDA(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
    RCGS_CUDA(cudaStreamSynchronize(s));
    dfree(cnt, s);
    *h_mismatches = (int64_t)h;
    return RCGS_OK;
}

extern "C" int rcgs_stereo_depth(const double* d_disp_h, const double* d_disp_v, int64_t n, double fx_baseline,
                                 double fy_baseline, double min_disparity, const double* d_fallback, double* d_depth,
                                 void* stream) {
    RCGS_CHECK_ARG(d_disp_h && d_disp_v && d_depth, "null argument");
    if (n > 0) {
        stereo_depth_kernel<<<div_up(n, 256), 256, 0, as_stream(stream)>>>(d_disp_h, d_disp_v, n, fx_baseline,
                                                                          fy_baseline, min_disparity, d_fallback,
                                                                          d_depth);
        RCGS_LAUNCH_CHECK();
    }
    return RCGS_OK;
}

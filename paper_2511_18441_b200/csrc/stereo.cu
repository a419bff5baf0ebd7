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
    int r;         // window radius
    double size;   // 2r + 1
    double floor_v, floor_sq, lr_tol;
};

__device__ __forceinline__ int clampi(int i, int n) { return i < 0 ? 0 : (i >= n ? n - 1 : i); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// Gray planes in the matching orientation (transpose: rows of the match are the
// image columns, stereo.py:207-209): P0 = gray(left), P1 = gray(right),
// P2 = mirror(gray(right)), P3 = mirror(gray(left)) (the LR pass, stereo.py:143).
// gray = mean over channels, numpy order ((r + g) + b) / 3 (stereo.py:87-94).
template <typename T>
__global__ void stereo_gray_kernel(const T* __restrict__ left, const T* __restrict__ right, int ch_l, int ch_r,
                                   int transpose,
                                   StereoDims sd, double* __restrict__ planes) {
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

// Vertical running box of A, A*A, B, B*B (thread per (column, plane)).
__global__ void stereo_vbox_planes_kernel(const double* __restrict__ A, const double* __restrict__ B, StereoDims sd,
                                          double* __restrict__ out4) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 4 * sd.w) return;
    const int k = i / sd.w, x = i - k * sd.w;
    const double* src = k < 2 ? A : B;
    const bool sq = k & 1;
    double* out = out4 + (int64_t)k * sd.h * sd.w;
    auto val = [&](int y) {
        const double v = src[(int64_t)clampi(y, sd.h) * sd.w + x];
        return sq ? dmul(v, v) : v;
    };
    double tmp = 0.0;
    for (int j = -sd.r; j <= sd.r; ++j) tmp = dadd(tmp, val(j));
    out[x] = ddiv(tmp, sd.size);
    for (int y = 1; y < sd.h; ++y) {
        tmp = dadd(tmp, dsub(val(y + sd.r), val(y - sd.r - 1)));
        out[(int64_t)y * sd.w + x] = ddiv(tmp, sd.size);
    }
}

// Horizontal running box of the vertical planes VA, VA2 -> box(A), box(A*A)
// (thread per (row, plane)).
__global__ void stereo_hbox_left_kernel(const double* __restrict__ v4, StereoDims sd, double* __restrict__ mu_ex) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 2 * sd.h) return;
    const int k = i / sd.h, y = i - k * sd.h;
    const double* line = v4 + (int64_t)k * sd.h * sd.w + (int64_t)y * sd.w;
    double* out = mu_ex + (int64_t)k * sd.h * sd.w + (int64_t)y * sd.w;
    auto val = [&](int x) { return line[clampi(x, sd.w)]; };
    double tmp = 0.0;
    for (int j = -sd.r; j <= sd.r; ++j) tmp = dadd(tmp, val(j));
    out[0] = ddiv(tmp, sd.size);
    for (int x = 1; x < sd.w; ++x) {
        tmp = dadd(tmp, dsub(val(x + sd.r), val(x - sd.r - 1)));
        out[x] = ddiv(tmp, sd.size);
    }
}

// Vertical running box of A * shift_d(B) for every disparity, written [y][x][d]
// (thread per (column, d), d fastest).  shift_d(B)[y, x] = B[y, max(x - d, 0)]
// (stereo.py:110-112).
__global__ void stereo_vbox_products_kernel(const double* __restrict__ A, const double* __restrict__ B, StereoDims sd,
                                            double* __restrict__ vab) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)sd.w * sd.nde) return;
    const int x = (int)(i / sd.nde), d = (int)(i - (int64_t)x * sd.nde);
    const int xs = x - d > 0 ? x - d : 0;
    auto val = [&](int y) {
        const int64_t row = (int64_t)clampi(y, sd.h) * sd.w;
        return dmul(A[row + x], B[row + xs]);
    };
    const int64_t pitch = (int64_t)sd.w * sd.nd;  // one row of the volume
    double* out = vab + (int64_t)x * sd.nd + d;
    double tmp = 0.0;
    for (int j = -sd.r; j <= sd.r; ++j) tmp = dadd(tmp, val(j));
    out[0] = ddiv(tmp, sd.size);
    for (int y = 1; y < sd.h; ++y) {
        tmp = dadd(tmp, dsub(val(y + sd.r), val(y - sd.r - 1)));
        out[(int64_t)y * pitch] = ddiv(tmp, sd.size);
    }
}

// Horizontal running boxes of shift_d(VB), shift_d(VB2) and V(A*shift_d(B)) along
// each row, with the ZNCC score of every (x, d) (stereo.py:113-117); thread per
// (row, d), d fastest.  Scores are written [y][x][d].
__global__ void stereo_hscore_kernel(const double* __restrict__ v4, const double* __restrict__ mu_ex,
                                     const double* __restrict__ vab, StereoDims sd, double* __restrict__ scores) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)sd.h * sd.nde) return;
    const int y = (int)(i / sd.nde), d = (int)(i - (int64_t)y * sd.nde);
    const int64_t np = (int64_t)sd.h * sd.w;
    const double* vb = v4 + 2 * np + (int64_t)y * sd.w;
    const double* vb2 = v4 + 3 * np + (int64_t)y * sd.w;
    const double* mul = mu_ex + (int64_t)y * sd.w;
    const double* exl = mu_ex + np + (int64_t)y * sd.w;
    const double* pab = vab + (int64_t)y * sd.w * sd.nd + d;
    double* out = scores + (int64_t)y * sd.w * sd.nd + d;
    auto sh = [&](int x) {  // column of the shifted image's vertical box at x (nearest-extended)
        const int c = clampi(x, sd.w) - d;
        return c > 0 ? c : 0;
    };
    double t1 = 0.0, t2 = 0.0, t3 = 0.0;
    for (int j = -sd.r; j <= sd.r; ++j) {
        const int c = sh(j);
        t1 = dadd(t1, vb[c]);
        t2 = dadd(t2, vb2[c]);
        t3 = dadd(t3, pab[(int64_t)clampi(j, sd.w) * sd.nd]);
    }
    for (int x = 0; x < sd.w; ++x) {
        if (x > 0) {
            const int cn = sh(x + sd.r), co = sh(x - sd.r - 1);
            t1 = dadd(t1, dsub(vb[cn], vb[co]));
            t2 = dadd(t2, dsub(vb2[cn], vb2[co]));
            t3 = dadd(t3, dsub(pab[(int64_t)clampi(x + sd.r, sd.w) * sd.nd],
                               pab[(int64_t)clampi(x - sd.r - 1, sd.w) * sd.nd]));
        }
        const double mu_r = ddiv(t1, sd.size), ex_r2 = ddiv(t2, sd.size), ex_ab = ddiv(t3, sd.size);
        const double mu_l = mul[x];
        const double var_l = dsub(exl[x], dmul(mu_l, mu_l));
        const double var_r = dsub(ex_r2, dmul(mu_r, mu_r));
        const double cov = dsub(ex_ab, dmul(mu_l, mu_r));
        const bool ok = var_l >= sd.floor_v && var_r >= sd.floor_v && x >= d;
        const double p = dmul(var_l, var_r);
        const double den = __dsqrt_rn(p < sd.floor_sq ? sd.floor_sq : p);  // np.maximum keeps a NaN
        out[(int64_t)x * sd.nd] = ok ? ddiv(cov, den) : -2.0;
    }
}

// argmax over d (first maximum; np.argmax also stops at the first NaN) and the
// parabolic refinement of stereo.py:121-139.  Entries d >= w are -2 (stereo.py:107-108).
__device__ __forceinline__ double score_at(const double* s, int d, const StereoDims& sd) {
    return d < sd.nde ? s[d] : -2.0;
}

__global__ void stereo_best_kernel(const double* __restrict__ scores, StereoDims sd, double* __restrict__ disp) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)sd.h * sd.w) return;
    const double* s = scores + i * sd.nd;
    int best = 0;
    double s0 = score_at(s, 0, sd);
    if (!isnan(s0)) {
        for (int d = 1; d < sd.nd; ++d) {
            const double v = score_at(s, d, sd);
            if (isnan(v)) {
                best = d;
                s0 = v;
                break;
            }
            if (v > s0) {
                best = d;
                s0 = v;
            }
        }
    }
    double out = s0 <= -2.0 ? -1.0 : (double)best;
    const int dmax = sd.nd - 1;
    const double sm = score_at(s, best - 1 > 0 ? best - 1 : 0, sd);
    const double sp = score_at(s, best + 1 < dmax ? best + 1 : dmax, sd);
    const bool refinable = best > 0 && best < dmax && sm > -2.0 && sp > -2.0 && s0 > -2.0;
    const double den = dsub(dadd(sm, sp), dmul(2.0, s0));
    if (refinable && den < -1e-12) {
        double delta = ddiv(dmul(0.5, dsub(sm, sp)), den);
        delta = delta < -0.5 ? -0.5 : (delta > 0.5 ? 0.5 : delta);
        out = dadd((double)best, delta);
    }
    disp[i] = out;
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
    sd.r = radius;
    sd.size = (double)(2 * radius + 1);
    sd.floor_v = floor_v;
    sd.floor_sq = floor_sq;
    sd.lr_tol = lr_tol;
    const int64_t np = (int64_t)sd.h * sd.w;
    const int64_t nvol = np * sd.nd;
    double *planes = nullptr, *v4 = nullptr, *muex = nullptr, *vab = nullptr, *scores = nullptr, *dl = nullptr,
           *drm = nullptr;
    int rc = RCGS_OK;
    if ((rc = dalloc(&planes, 4 * np, s)) || (rc = dalloc(&v4, 4 * np, s)) || (rc = dalloc(&muex, 2 * np, s)) ||
        (rc = dalloc(&vab, nvol, s)) || (rc = dalloc(&scores, nvol, s)) || (rc = dalloc(&dl, np, s)) ||
        (rc = dalloc(&drm, np, s)))
        goto done;
    {
        const int T = 256;
        if (elem_bytes == 4)
            stereo_gray_kernel<float><<<div_up(np, T), T, 0, s>>>((const float*)left, (const float*)right, ch_l,
                                                                  ch_r, transpose, sd, planes);
        else
            stereo_gray_kernel<double><<<div_up(np, T), T, 0, s>>>((const double*)left, (const double*)right,
                                                                   ch_l, ch_r, transpose, sd, planes);
        for (int pass = 0; pass < 2; ++pass) {  // pass 0: (left, right); pass 1: mirrored (right, left)
            const double* A = planes + (2 * pass) * np;
            const double* B = planes + (2 * pass + 1) * np;
            stereo_vbox_planes_kernel<<<div_up(4 * sd.w, 128), 128, 0, s>>>(A, B, sd, v4);
            stereo_hbox_left_kernel<<<div_up(2 * sd.h, 128), 128, 0, s>>>(v4, sd, muex);
            stereo_vbox_products_kernel<<<div_up((int64_t)sd.w * sd.nde, T), T, 0, s>>>(A, B, sd, vab);
            stereo_hscore_kernel<<<div_up((int64_t)sd.h * sd.nde, 128), 128, 0, s>>>(v4, muex, vab, sd, scores);
            stereo_best_kernel<<<div_up(np, T), T, 0, s>>>(scores, sd, pass ? drm : dl);
        }
        stereo_lr_kernel<<<div_up(np, T), T, 0, s>>>(dl, drm, sd, transpose, disp);
        rc = cudaGetLastError() == cudaSuccess ? RCGS_OK : RCGS_ECUDA;
        if (rc) set_error("stereo kernels failed to launch");
    }
done:
    dfree(planes, s);
    dfree(v4, s);
    dfree(muex, s);
    dfree(vab, s);
    dfree(scores, s);
    dfree(dl, s);
    dfree(drm, s);
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

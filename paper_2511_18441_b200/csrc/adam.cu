// K7: SH gradient expansion fused with Adam (backward.py:36-40, optimize.py:59-83).
//
// The per-view backward (raster.cu) leaves one fp32 3-vector per gaussian,
// acc[i, ch] = active * sum_p g[p, ch] w_ip.  The dense (N, 16, 3) gradient is
// basis_k(dir_i) * acc[i, ch]; it is never materialised: one thread per float4
// of the 48 coefficients runs Adam with fully coalesced 16-byte SH / m / v
// accesses and rebuilds the (at most two) SH basis rows it needs in fp32.
// A device-side reject flag (non-finite gradient, optimize.py:72-74) skips the
// update, and the device step counter feeds the bias corrections, so a
// sequence of steps needs no host synchronisation.
#include <math.h>

#include "common.cuh"
#include "shmath.cuh"

namespace rcgs {

constexpr int kMaxViews = 16;

struct AccViews {
    const float* acc[kMaxViews];
    double cen[kMaxViews][3];
    int n;
};

struct AdamHyper {
    float lr_dc, lr_rest, b1, b2, eps;
};

__device__ __forceinline__ void adam4(float4& p, float4& m, float4& v, const float g[4], int f0,
                                      const AdamHyper& h, float inv_bc1, float inv_bc2) {
    float* pp = &p.x;
    float* mm = &m.x;
    float* vv = &v.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int k = (f0 + j) / 3;
        const float lr = k == 0 ? h.lr_dc : h.lr_rest;
        mm[j] = h.b1 * mm[j] + (1.0f - h.b1) * g[j];
        vv[j] = h.b2 * vv[j] + (1.0f - h.b2) * g[j] * g[j];
        const float mh = mm[j] * inv_bc1, vh = vv[j] * inv_bc2;
        pp[j] -= __fdividef(lr * mh, sqrtf(vh) + h.eps);
    }
}

// Bias corrections 1/(1 - beta^t) for t = step + 1, once per launch (fp64 pow).
__global__ void adam_prep_kernel(const int64_t* __restrict__ step, double db1, double db2,
                                 float2* __restrict__ inv) {
    const double t = (double)(*step + 1);
    *inv = make_float2((float)(1.0 / (1.0 - pow(db1, t))), (float)(1.0 / (1.0 - pow(db2, t))));
}

// One thread per float4 of a gaussian's 48 coefficients (12 per gaussian, fully
// coalesced SH / m / v traffic).  Each thread rebuilds the few SH basis rows it
// needs in fp32 from the fp64 view direction (cheap next to the 96 bytes it
// moves), so there is no shared-memory staging and no block barrier.
__global__ void __launch_bounds__(256) adam_fused_kernel(
    const double* __restrict__ pos, int64_t n, int deg, float4* __restrict__ sh, float4* __restrict__ m,
    float4* __restrict__ v, AccViews views, AdamHyper h, const float2* __restrict__ bc,
    const int32_t* __restrict__ reject) {
    if (reject && *reject) return;
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;  // n * 12 < 2^32 (checked on host)
    if (q >= (uint32_t)n * 12u) return;
    const uint32_t g = q / 12u;
    const int c4 = (int)(q - g * 12u);
    const int k0 = (4 * c4) / 3;  // the 4 coefficients span rows k0 and k0 + 1 at most
    // the 48 bytes of state this thread updates, loaded first (in flight during the
    // basis math) with streaming hints: touched once per step, keep L2 for the raster
    float4 p = __ldcs(sh + q), mm = __ldcs(m + q), vv = __ldcs(v + q);
    const double px = pos[3 * g], py = pos[3 * g + 1], pz = pos[3 * g + 2];
    float gr[4] = {0.f, 0.f, 0.f, 0.f};
    for (int vi = 0; vi < views.n; ++vi) {
        float x = (float)(px - views.cen[vi][0]), y = (float)(py - views.cen[vi][1]),
              z = (float)(pz - views.cen[vi][2]);
        const float inv = rsqrtf(x * x + y * y + z * z);
        x *= inv;
        y *= inv;
        z *= inv;
        // branch-free: every basis row in registers, then predicated selects of k0, k0 + 1
        const float xx = x * x, yy = y * y, zz = z * z;
        const float d1 = deg >= 1 ? 1.f : 0.f, d2 = deg >= 2 ? 1.f : 0.f, d3 = deg >= 3 ? 1.f : 0.f;
        const float r0 = 0.28209479177387814f;
        const float r1 = d1 * -0.4886025119029199f * y, r2 = d1 * 0.4886025119029199f * z;
        const float r3 = d1 * -0.4886025119029199f * x;
        const float r4 = d2 * 1.0925484305920792f * (x * y), r5 = d2 * -1.0925484305920792f * (y * z);
        const float r6 = d2 * 0.31539156525252005f * (2.f * zz - xx - yy);
        const float r7 = d2 * -1.0925484305920792f * (x * z), r8 = d2 * 0.5462742152960396f * (xx - yy);
        const float r9 = d3 * -0.5900435899266435f * y * (3.f * xx - yy);
        const float r10 = d3 * 2.890611442640554f * (x * y) * z;
        const float r11 = d3 * -0.4570457994644658f * y * (4.f * zz - xx - yy);
        const float r12 = d3 * 0.3731763325901154f * z * (2.f * zz - 3.f * xx - 3.f * yy);
        const float r13 = d3 * -0.4570457994644658f * x * (4.f * zz - xx - yy);
        const float r14 = d3 * 1.445305721320277f * z * (xx - yy);
        const float r15 = d3 * -0.5900435899266435f * x * (xx - 3.f * yy);
#define RCGS_PICK(kk)                                                                           \
    ((kk) == 0 ? r0 : (kk) == 1 ? r1 : (kk) == 2 ? r2 : (kk) == 3 ? r3 : (kk) == 4 ? r4 :         \
     (kk) == 5 ? r5 : (kk) == 6 ? r6 : (kk) == 7 ? r7 : (kk) == 8 ? r8 : (kk) == 9 ? r9 :         \
     (kk) == 10 ? r10 : (kk) == 11 ? r11 : (kk) == 12 ? r12 : (kk) == 13 ? r13 : (kk) == 14 ? r14 \
                                                                                : (kk) == 15 ? r15 : 0.f)
        const float b0 = RCGS_PICK(k0), b1 = RCGS_PICK(k0 + 1);
#undef RCGS_PICK
        const float* a = views.acc[vi] + 3 * (size_t)g;
        const float a0 = a[0], a1 = a[1], a2 = a[2];
        // element 4 c4 + j has row (4 c4 + j) / 3 and channel (4 c4 + j) % 3; c4 % 3
        // fixes the pattern: 0 -> (k0: ch 0,1,2; k0+1: ch 0), 1 -> (k0: 1,2; k0+1: 0,1),
        // 2 -> (k0: 2; k0+1: 0,1,2)
        const int r = c4 % 3;
        const float e0 = r == 0 ? b0 * a0 : (r == 1 ? b0 * a1 : b0 * a2);
        const float e1 = r == 0 ? b0 * a1 : (r == 1 ? b0 * a2 : b1 * a0);
        const float e2 = r == 0 ? b0 * a2 : (r == 1 ? b1 * a0 : b1 * a1);
        const float e3 = r == 0 ? b1 * a0 : (r == 1 ? b1 * a1 : b1 * a2);
        gr[0] += e0;
        gr[1] += e1;
        gr[2] += e2;
        gr[3] += e3;
    }
    if (views.n > 1) {
        const float invn = 1.0f / (float)views.n;
#pragma unroll
        for (int j = 0; j < 4; ++j) gr[j] *= invn;
    }
    const float2 ibc = *bc;
    adam4(p, mm, vv, gr, 4 * c4, h, ibc.x, ibc.y);
    __stcs(sh + q, p);
    __stcs(m + q, mm);
    __stcs(v + q, vv);
}

__global__ void adam_dense_kernel(float4* __restrict__ p, float4* __restrict__ m, float4* __restrict__ v,
                                  const float4* __restrict__ grad, int64_t nq, AdamHyper h,
                                  const float2* __restrict__ bc, const int32_t* __restrict__ reject) {
    if (reject && *reject) return;
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const float2 ibc = *bc;
    const float4 g4 = grad[q];
    const float gr[4] = {g4.x, g4.y, g4.z, g4.w};
    float4 pp = p[q], mm = m[q], vv = v[q];
    adam4(pp, mm, vv, gr, 4 * (int)(q % 12), h, ibc.x, ibc.y);
    p[q] = pp;
    m[q] = mm;
    v[q] = vv;
}

__global__ void step_commit_kernel(const int32_t* __restrict__ reject, int64_t* __restrict__ step) {
    if (!(reject && *reject)) *step += 1;
}

__global__ void sh_grad_kernel(const double* __restrict__ pos, int64_t n, int deg,
                               const float* __restrict__ acc, Center cen, float* __restrict__ grad) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    double x, y, z;
    view_dir(pos, g, cen.c, x, y, z);
    double b[16];
    sh_basis16<double>(x, y, z, deg, b);
    const float a0 = acc[3 * g], a1 = acc[3 * g + 1], a2 = acc[3 * g + 2];
    float* o = grad + 48 * g;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        o[3 * k] = (float)(b[k] * a0);
        o[3 * k + 1] = (float)(b[k] * a1);
        o[3 * k + 2] = (float)(b[k] * a2);
    }
}

__global__ void nonfinite_kernel(const float* __restrict__ x, int64_t count, int32_t* __restrict__ flag) {
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(x[i]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

static AdamHyper hyper(const rcgs_adam_config* c) {
    AdamHyper h;
    h.lr_dc = (float)c->lr_dc;
    h.lr_rest = (float)c->lr_rest;
    h.b1 = (float)c->beta1;
    h.b2 = (float)c->beta2;
    h.eps = (float)c->eps;
    return h;
}

}  // namespace rcgs

using namespace rcgs;

extern "C" int rcgs_adam_fused(const rcgs_scene* sc, float* d_sh, float* d_m, float* d_v,
                               const float* const* h_d_accs, const double* h_centers, int32_t n_views,
                               const rcgs_adam_config* cfg, const int32_t* d_reject, int64_t* d_step,
                               void* stream) {
    RCGS_CHECK_ARG(sc && d_sh && d_m && d_v && h_d_accs && h_centers && cfg && d_step, "null argument");
    RCGS_CHECK_ARG(n_views >= 1 && n_views <= kMaxViews, "views per step must be in [1, %d]", kMaxViews);
    RCGS_CHECK_ARG(sc->n < (int64_t)357913941, "scene too large for 32-bit Adam indexing");
    cudaStream_t s = as_stream(stream);
    if (sc->n > 0) {
        AccViews av;
        av.n = n_views;
        for (int i = 0; i < n_views; ++i) {
            av.acc[i] = h_d_accs[i];
            for (int j = 0; j < 3; ++j) av.cen[i][j] = h_centers[3 * i + j];
        }
        float2* bc = nullptr;
        RCGS_TRY(dalloc(&bc, 1, s));
        adam_prep_kernel<<<1, 1, 0, s>>>(d_step, cfg->beta1, cfg->beta2, bc);
        adam_fused_kernel<<<div_up(sc->n * 12, 256), 256, 0, s>>>(
            sc->pos, sc->n, sc->sh_degree, reinterpret_cast<float4*>(d_sh), reinterpret_cast<float4*>(d_m),
            reinterpret_cast<float4*>(d_v), av, hyper(cfg), bc, d_reject);
        RCGS_LAUNCH_CHECK();
        dfree(bc, s);
    }
    step_commit_kernel<<<1, 1, 0, s>>>(d_reject, d_step);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

extern "C" int rcgs_adam_dense(float* d_params, float* d_m, float* d_v, const float* d_grads, int64_t n,
                               const rcgs_adam_config* cfg, const int32_t* d_reject, int64_t* d_step,
                               void* stream) {
    RCGS_CHECK_ARG(d_params && d_m && d_v && d_grads && cfg && d_step, "null argument");
    cudaStream_t s = as_stream(stream);
    const int64_t nq = n * 12;
    if (nq > 0) {
        float2* bc = nullptr;
        RCGS_TRY(dalloc(&bc, 1, s));
        adam_prep_kernel<<<1, 1, 0, s>>>(d_step, cfg->beta1, cfg->beta2, bc);
        adam_dense_kernel<<<div_up(nq, 256), 256, 0, s>>>(
            reinterpret_cast<float4*>(d_params), reinterpret_cast<float4*>(d_m), reinterpret_cast<float4*>(d_v),
            reinterpret_cast<const float4*>(d_grads), nq, hyper(cfg), bc, d_reject);
        RCGS_LAUNCH_CHECK();
        dfree(bc, s);
    }
    step_commit_kernel<<<1, 1, 0, s>>>(d_reject, d_step);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

extern "C" int rcgs_sh_grad(const rcgs_scene* sc, const float* d_acc, const double* h_center3, float* d_grad,
                            void* stream) {
    RCGS_CHECK_ARG(sc && d_acc && h_center3 && d_grad, "null argument");
    if (sc->n == 0) return RCGS_OK;
    Center c;
    for (int j = 0; j < 3; ++j) c.c[j] = h_center3[j];
    sh_grad_kernel<<<div_up(sc->n, 256), 256, 0, as_stream(stream)>>>(sc->pos, sc->n, sc->sh_degree, d_acc, c,
                                                                       d_grad);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

extern "C" int rcgs_nonfinite_check(const float* d_x, int64_t count, int32_t* d_flag, void* stream) {
    RCGS_CHECK_ARG(d_flag != nullptr, "null flag");
    if (count <= 0) return RCGS_OK;
    unsigned blocks = div_up(count, 256);
    if (blocks > 4096) blocks = 4096;
    nonfinite_kernel<<<blocks, 256, 0, as_stream(stream)>>>(d_x, count, d_flag);
    RCGS_LAUNCH_CHECK();
    return RCGS_OK;
}

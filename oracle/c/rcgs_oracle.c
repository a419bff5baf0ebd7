/* Plain-C restatement of the exact-decision arithmetic of the reference path.
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * numpy evaluates `P @ R.T + t` (render.py:175, selection.py:193) through
 * OpenBLAS; on x86-64 hosts the per-coordinate result equals the fused chain
 *     fma(p2, R[k][2], fma(p1, R[k][1], p0 * R[k][0])) + t[k]
 * (SURVEY.md 0.4).  The CUDA kernels use the same chain (csrc/common.cuh
 * cam_coord); tests/test_oracle_golden.py checks this C function against numpy
 * on the host that runs the tests, which pins the claim per host.
 * Compiled with -ffp-contract=off so only the explicit fma() calls fuse.
 */
#include <math.h>
#include <stdint.h>

void rcgs_oracle_view_transform(const double* pts, int64_t n, const double* R, const double* t,
                                double* out) {
    for (int64_t i = 0; i < n; ++i) {
        const double p0 = pts[3 * i], p1 = pts[3 * i + 1], p2 = pts[3 * i + 2];
        for (int k = 0; k < 3; ++k)
            out[3 * i + k] = fma(p2, R[3 * k + 2], fma(p1, R[3 * k + 1], p0 * R[3 * k + 0])) + t[k];
    }
}

/* selection.py:184-206: nearest pixel (round half even) + occlusion visibility. */
void rcgs_oracle_project_points(const double* pts, int64_t n, const double* R, const double* t,
                                double fx, double fy, double cx, double cy, int32_t width,
                                int32_t height, const double* depth, double tol, int64_t* pu,
                                int64_t* pv, uint8_t* vis) {
    for (int64_t i = 0; i < n; ++i) {
        double c[3];
        rcgs_oracle_view_transform(pts + 3 * i, 1, R, t, c);
        pu[i] = -1;
        pv[i] = -1;
        vis[i] = 0;
        if (!(c[2] > 0)) continue;
        const double u = fx * c[0] / c[2] + cx, v = fy * c[1] / c[2] + cy;
        pu[i] = (int64_t)nearbyint(u);
        pv[i] = (int64_t)nearbyint(v);
        if (pu[i] < 0 || pu[i] >= width || pv[i] < 0 || pv[i] >= height) continue;
        vis[i] = c[2] <= depth[pv[i] * width + pu[i]] * (1.0 + tol);
    }
}

/* render.py:95-100 compute_covariance + scene.py:98-112 quaternion_to_rotation:
 * elementwise numpy ops (plain), then the stacked matmul m @ m^T, which numpy
 * runs through OpenBLAS dgemm = the same fused chain as above (checked against
 * numpy by tests/test_oracle_golden.py).  Output (n, 6): xx xy xz yy yz zz. */
void rcgs_oracle_cov3d(const double* rot, const double* scale, int64_t n, double* out) {
    for (int64_t g = 0; g < n; ++g) {
        const double w = rot[4 * g], x = rot[4 * g + 1], y = rot[4 * g + 2], z = rot[4 * g + 3];
        double r[3][3];
        r[0][0] = 1 - 2 * (y * y + z * z);
        r[0][1] = 2 * (x * y - w * z);
        r[0][2] = 2 * (x * z + w * y);
        r[1][0] = 2 * (x * y + w * z);
        r[1][1] = 1 - 2 * (x * x + z * z);
        r[1][2] = 2 * (y * z - w * x);
        r[2][0] = 2 * (x * z - w * y);
        r[2][1] = 2 * (y * z + w * x);
        r[2][2] = 1 - 2 * (x * x + y * y);
        double m[3][3];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) m[i][j] = r[i][j] * scale[3 * g + j];
        double s[3][3];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) s[i][j] = fma(m[i][2], m[j][2], fma(m[i][1], m[j][1], m[i][0] * m[j][0]));
        double* o = out + 6 * g;
        o[0] = s[0][0];
        o[1] = s[0][1];
        o[2] = s[0][2];
        o[3] = s[1][1];
        o[4] = s[1][2];
        o[5] = s[2][2];
    }
}

/* render.py:172-214 per gaussian, every fp64 value that feeds a discrete
 * decision: z, mean2d, the dilated cov2d (a, b, c), det, the 3-sigma viewport
 * test, and the conic (c, -b, a) / det.
 *   jac (plain ops), t = jac @ R (stacked matmul: the fused chain, with jac's
 *   structural zeros multiplied in), cov2 = einsum("nij,njk,nlk->nil", t, S, t)
 *   = sum over j (outer) and k (inner) of (t_ij * S_jk) * t_lk accumulated
 *   left to right (numpy's einsum sum-of-products loop; checked bit-exact).
 * out (n, 12): kept, z, mx, my, a, b, c, det, ca, cb, cc, radius. */
void rcgs_oracle_project_exact(const double* pos, const double* cov3d, int64_t n, const double* R,
                               const double* t, double fx, double fy, double cx, double cy, int32_t width,
                               int32_t height, double near_clip, double dilation, double sigmas, double* out) {
    for (int64_t g = 0; g < n; ++g) {
        double* o = out + 12 * g;
        double c3[3];
        rcgs_oracle_view_transform(pos + 3 * g, 1, R, t, c3);
        const double x = c3[0], y = c3[1], z = c3[2];
        for (int q = 0; q < 12; ++q) o[q] = 0.0;
        o[1] = z;
        if (!(z > near_clip)) continue;
        const double mx = fx * x / z + cx, my = fy * y / z + cy;
        double jac[2][3] = {{fx / z, 0.0, -fx * x / (z * z)}, {0.0, fy / z, -fy * y / (z * z)}};
        double tt[2][3];
        for (int i = 0; i < 2; ++i)
            for (int k = 0; k < 3; ++k)
                tt[i][k] = fma(jac[i][2], R[6 + k], fma(jac[i][1], R[3 + k], jac[i][0] * R[k]));
        const double* S6 = cov3d + 6 * g;
        const double S[3][3] = {{S6[0], S6[1], S6[2]}, {S6[1], S6[3], S6[4]}, {S6[2], S6[4], S6[5]}};
        double cv[2][2];
        for (int i = 0; i < 2; ++i)
            for (int l = 0; l < 2; ++l) {
                double acc = 0.0;
                for (int j = 0; j < 3; ++j)
                    for (int k = 0; k < 3; ++k) acc = acc + (tt[i][j] * S[j][k]) * tt[l][k];
                cv[i][l] = acc;
            }
        const double a = cv[0][0] + dilation, b = cv[0][1], c = cv[1][1] + dilation;
        const double det = a * c - b * b;
        const double mid = 0.5 * (a + c);
        const double lam = mid + sqrt(fmax(mid * mid - det, 0.0));
        const double radius = sigmas * sqrt(lam);
        const double w1 = width - 1, h1 = height - 1;
        const int kept = (det > 0) && (mx + radius >= 0) && (mx - radius <= w1) && (my + radius >= 0) &&
                         (my - radius <= h1);
        o[0] = kept;
        o[2] = mx;
        o[3] = my;
        o[4] = a;
        o[5] = b;
        o[6] = c;
        o[7] = det;
        o[8] = c / det;
        o[9] = -b / det;
        o[10] = a / det;
        o[11] = radius;
    }
}

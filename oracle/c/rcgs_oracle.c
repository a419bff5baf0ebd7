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

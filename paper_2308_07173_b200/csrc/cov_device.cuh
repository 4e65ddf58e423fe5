// cov_device.cuh -- GICP plane-regularised covariance from a 3x3 scatter (device).
//
// Paper: each point is a Gaussian p_i ~ N(p_i, C_i) whose C_i is
// estimated from its neighbours (l.404, l.413). Regularisation (DESIGN.md reading
// R7): eigenvalues of S replaced by (eps, 1, 1) ascending, i.e.
//   C = I - (1 - eps) n n^T,  n = eigenvector of the smallest eigenvalue of S;
// n = +z when S == 0 (all neighbours coincide, reading R11).
//
// Numerics: the scatter is accumulated in fp32 relative to
// the first neighbour (exact differences for nearby points, two passes); the
// eigen problem is solved in fp64: smallest root of the characteristic cubic by
// monotone Newton from 0, eigenvector as the largest cross product of two rows of
// S - lambda I. No trigonometry, no iteration-count dependence on the spectrum
// beyond the (rare) double-root case.
#pragma once

#include <cuda_runtime.h>

namespace gicp {

__device__ __forceinline__ void plane_cov(float s00, float s01, float s02, float s11, float s12, float s22, float eps,
                                          float out[6]) {
    double a00 = s00, a01 = s01, a02 = s02, a11 = s11, a12 = s12, a22 = s22;
    const double mx = fmax(fmax(fmax(fabs(a00), fabs(a01)), fmax(fabs(a02), fabs(a11))), fmax(fabs(a12), fabs(a22)));
    double nx = 0.0, ny = 0.0, nz = 1.0;
    if (mx > 0.0) {
        const double inv = 1.0 / mx;
        a00 *= inv;
        a01 *= inv;
        a02 *= inv;
        a11 *= inv;
        a12 *= inv;
        a22 *= inv;
        // p(l) = l^3 - c2 l^2 + c1 l - c0, roots = eigenvalues
        const double c2 = a00 + a11 + a22;
        const double c1 = a00 * a11 + a00 * a22 + a11 * a22 - a01 * a01 - a02 * a02 - a12 * a12;
        const double c0 = a00 * (a11 * a22 - a12 * a12) - a01 * (a01 * a22 - a12 * a02) + a02 * (a01 * a12 - a11 * a02);
        // p is concave and increasing left of the smallest root: Newton from 0 is monotone
        double l = 0.0;
        for (int it = 0; it < 64; ++it) {
            const double p = ((l - c2) * l + c1) * l - c0;
            const double dp = (3.0 * l - 2.0 * c2) * l + c1;
            if (!(dp > 0.0)) break;
            // left of the root p < 0; p >= 0 means rounding noise at the root (the
            // iterate would oscillate by an ulp instead of reaching a fixed point)
            if (!(p < 0.0)) break;
            const double ln = l - p / dp;
            if (ln == l) break;
            l = ln;
        }
        const double r0x = a00 - l, r0y = a01, r0z = a02;
        const double r1x = a01, r1y = a11 - l, r1z = a12;
        const double r2x = a02, r2y = a12, r2z = a22 - l;
        // cross products of row pairs
        double vx = r0y * r1z - r0z * r1y, vy = r0z * r1x - r0x * r1z, vz = r0x * r1y - r0y * r1x;
        double d = vx * vx + vy * vy + vz * vz;
        {
            const double wx = r0y * r2z - r0z * r2y, wy = r0z * r2x - r0x * r2z, wz = r0x * r2y - r0y * r2x;
            const double e = wx * wx + wy * wy + wz * wz;
            if (e > d) {
                vx = wx;
                vy = wy;
                vz = wz;
                d = e;
            }
        }
        {
            const double wx = r1y * r2z - r1z * r2y, wy = r1z * r2x - r1x * r2z, wz = r1x * r2y - r1y * r2x;
            const double e = wx * wx + wy * wy + wz * wz;
            if (e > d) {
                vx = wx;
                vy = wy;
                vz = wz;
                d = e;
            }
        }
        if (d > 1e-28) {
            const double r = rsqrt(d);
            nx = vx * r;
            ny = vy * r;
            nz = vz * r;
        } else {
            // S - lambda I has rank <= 1 (lambda1 ~ lambda2): any unit n orthogonal to
            // the dominant row is an eigenvector of the smallest eigenvalue
            double bx = r0x, by = r0y, bz = r0z, bn = bx * bx + by * by + bz * bz;
            const double n1 = r1x * r1x + r1y * r1y + r1z * r1z, n2 = r2x * r2x + r2y * r2y + r2z * r2z;
            if (n1 > bn) {
                bx = r1x;
                by = r1y;
                bz = r1z;
                bn = n1;
            }
            if (n2 > bn) {
                bx = r2x;
                by = r2y;
                bz = r2z;
                bn = n2;
            }
            if (bn > 1e-28) {
                // cross with the axis least aligned with b
                const double ax = fabs(bx), ay = fabs(by), az = fabs(bz);
                double ex = 0, ey = 0, ez = 0;
                if (ax <= ay && ax <= az)
                    ex = 1;
                else if (ay <= az)
                    ey = 1;
                else
                    ez = 1;
                vx = by * ez - bz * ey;
                vy = bz * ex - bx * ez;
                vz = bx * ey - by * ex;
                const double r = rsqrt(vx * vx + vy * vy + vz * vz);
                nx = vx * r;
                ny = vy * r;
                nz = vz * r;
            }
        }
        // one Newton step on the norm (rsqrt is approximate in fp64)
        const double nn = nx * nx + ny * ny + nz * nz;
        const double corr = 1.5 - 0.5 * nn;
        nx *= corr;
        ny *= corr;
        nz *= corr;
    }
    const double w = 1.0 - (double)eps;
    out[0] = (float)(1.0 - w * nx * nx);
    out[1] = (float)(-w * nx * ny);
    out[2] = (float)(-w * nx * nz);
    out[3] = (float)(1.0 - w * ny * ny);
    out[4] = (float)(-w * ny * nz);
    out[5] = (float)(1.0 - w * nz * nz);
}

}  // namespace gicp

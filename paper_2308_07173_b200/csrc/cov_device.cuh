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

// Full symmetric 3x3 eigen decomposition in fp64 for the clamp regularisations
// (reading R21): lam1 by monotone Newton from 0 (as plane_cov), lam3 by
// monotone Newton from the Gershgorin upper bound (p is convex and increasing
// right of the largest root), lam2 = trace - lam1 - lam3; v1 and v3 as the
// largest cross product of two rows of S - lam I, v3 re-orthogonalised against
// v1, v2 = v3 x v1. Where eigenvalues are (nearly) equal the split of the
// eigenspace is arbitrary but the clamped C = sum lam'_i v_i v_i^T is not.
// reg 1: lam' = max(lam, eps) (absolute, m^2); reg 2: lam' = max(lam / lam3, eps).
__device__ __forceinline__ void null_vector(double a00, double a01, double a02, double a11, double a12, double a22,
                                            double l, double& nx, double& ny, double& nz) {
    const double r0x = a00 - l, r0y = a01, r0z = a02;
    const double r1x = a01, r1y = a11 - l, r1z = a12;
    const double r2x = a02, r2y = a12, r2z = a22 - l;
    double vx = r0y * r1z - r0z * r1y, vy = r0z * r1x - r0x * r1z, vz = r0x * r1y - r0y * r1x;
    double d = vx * vx + vy * vy + vz * vz;
    {
        const double wx = r0y * r2z - r0z * r2y, wy = r0z * r2x - r0x * r2z, wz = r0x * r2y - r0y * r2x;
        const double e = wx * wx + wy * wy + wz * wz;
        if (e > d) { vx = wx; vy = wy; vz = wz; d = e; }
    }
    {
        const double wx = r1y * r2z - r1z * r2y, wy = r1z * r2x - r1x * r2z, wz = r1x * r2y - r1y * r2x;
        const double e = wx * wx + wy * wy + wz * wz;
        if (e > d) { vx = wx; vy = wy; vz = wz; d = e; }
    }
    if (d > 1e-28) {
        const double r = 1.0 / sqrt(d);
        nx = vx * r;
        ny = vy * r;
        nz = vz * r;
        return;
    }
    // rank <= 1: any unit vector orthogonal to the dominant row
    double bx = r0x, by = r0y, bz = r0z, bn = bx * bx + by * by + bz * bz;
    const double n1 = r1x * r1x + r1y * r1y + r1z * r1z, n2 = r2x * r2x + r2y * r2y + r2z * r2z;
    if (n1 > bn) { bx = r1x; by = r1y; bz = r1z; bn = n1; }
    if (n2 > bn) { bx = r2x; by = r2y; bz = r2z; bn = n2; }
    if (!(bn > 1e-28)) {  // S - l I == 0: every direction
        nx = 0.0; ny = 0.0; nz = 1.0;
        return;
    }
    const double ax = fabs(bx), ay = fabs(by), az = fabs(bz);
    double ex = 0, ey = 0, ez = 0;
    if (ax <= ay && ax <= az) ex = 1; else if (ay <= az) ey = 1; else ez = 1;
    vx = by * ez - bz * ey;
    vy = bz * ex - bx * ez;
    vz = bx * ey - by * ex;
    const double r = 1.0 / sqrt(vx * vx + vy * vy + vz * vz);
    nx = vx * r;
    ny = vy * r;
    nz = vz * r;
}

__device__ __forceinline__ void clamp_cov(float s00, float s01, float s02, float s11, float s12, float s22, int reg,
                                          float eps, float out[6]) {
    double a00 = s00, a01 = s01, a02 = s02, a11 = s11, a12 = s12, a22 = s22;
    const double mx = fmax(fmax(fmax(fabs(a00), fabs(a01)), fmax(fabs(a02), fabs(a11))), fmax(fabs(a12), fabs(a22)));
    if (!(mx > 0.0)) {  // S == 0: every eigenvalue clamps to eps
        out[0] = eps; out[1] = 0.f; out[2] = 0.f; out[3] = eps; out[4] = 0.f; out[5] = eps;
        return;
    }
    const double inv = 1.0 / mx;
    a00 *= inv; a01 *= inv; a02 *= inv; a11 *= inv; a12 *= inv; a22 *= inv;
    const double c2 = a00 + a11 + a22;
    const double c1 = a00 * a11 + a00 * a22 + a11 * a22 - a01 * a01 - a02 * a02 - a12 * a12;
    const double c0 = a00 * (a11 * a22 - a12 * a12) - a01 * (a01 * a22 - a12 * a02) + a02 * (a01 * a12 - a11 * a02);
    auto P = [&](double l) { return ((l - c2) * l + c1) * l - c0; };
    auto dP = [&](double l) { return (3.0 * l - 2.0 * c2) * l + c1; };
    double l1 = 0.0;
    for (int it = 0; it < 64; ++it) {
        const double p = P(l1), dp = dP(l1);
        if (!(p < 0.0) || !(dp > 0.0)) break;
        const double ln = l1 - p / dp;
        if (ln == l1) break;
        l1 = ln;
    }
    double l3 = fmax(fmax(fabs(a00) + fabs(a01) + fabs(a02), fabs(a01) + fabs(a11) + fabs(a12)),
                     fabs(a02) + fabs(a12) + fabs(a22));
    for (int it = 0; it < 64; ++it) {
        const double p = P(l3), dp = dP(l3);
        if (!(p > 0.0) || !(dp > 0.0)) break;
        const double ln = l3 - p / dp;
        if (ln == l3) break;
        l3 = ln;
    }
    const double l2 = fmin(fmax(c2 - l1 - l3, l1), l3);
    double v1x, v1y, v1z, v3x, v3y, v3z;
    null_vector(a00, a01, a02, a11, a12, a22, l1, v1x, v1y, v1z);
    null_vector(a00, a01, a02, a11, a12, a22, l3, v3x, v3y, v3z);
    {
        const double d = v3x * v1x + v3y * v1y + v3z * v1z;
        v3x -= d * v1x; v3y -= d * v1y; v3z -= d * v1z;
        double nn = v3x * v3x + v3y * v3y + v3z * v3z;
        if (!(nn > 1e-20)) {  // v3 parallel to v1 (isotropic case): any orthogonal direction
            const double ax = fabs(v1x), ay = fabs(v1y), az = fabs(v1z);
            double ex = 0, ey = 0, ez = 0;
            if (ax <= ay && ax <= az) ex = 1; else if (ay <= az) ey = 1; else ez = 1;
            v3x = v1y * ez - v1z * ey; v3y = v1z * ex - v1x * ez; v3z = v1x * ey - v1y * ex;
            nn = v3x * v3x + v3y * v3y + v3z * v3z;
        }
        const double r = 1.0 / sqrt(nn);
        v3x *= r; v3y *= r; v3z *= r;
    }
    const double v2x = v3y * v1z - v3z * v1y, v2y = v3z * v1x - v3x * v1z, v2z = v3x * v1y - v3y * v1x;
    double w1, w2, w3;
    if (reg == 1) {  // absolute eigenvalues (undo the normalisation)
        w1 = fmax(l1 * mx, (double)eps);
        w2 = fmax(l2 * mx, (double)eps);
        w3 = fmax(l3 * mx, (double)eps);
    } else {
        w1 = fmax(l1 / l3, (double)eps);
        w2 = fmax(l2 / l3, (double)eps);
        w3 = 1.0;
    }
    auto C = [&](double ax, double ay, double bx, double by, double cx, double cy) {
        return w1 * ax * ay + w2 * bx * by + w3 * cx * cy;
    };
    out[0] = (float)C(v1x, v1x, v2x, v2x, v3x, v3x);
    out[1] = (float)C(v1x, v1y, v2x, v2y, v3x, v3y);
    out[2] = (float)C(v1x, v1z, v2x, v2z, v3x, v3z);
    out[3] = (float)C(v1y, v1y, v2y, v2y, v3y, v3y);
    out[4] = (float)C(v1y, v1z, v2y, v2z, v3y, v3z);
    out[5] = (float)C(v1z, v1z, v2z, v2z, v3z, v3z);
}

}  // namespace gicp

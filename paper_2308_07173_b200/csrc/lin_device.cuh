// lin_device.cuh -- the per-correspondence GICP terms shared by the 1-NN
// linearisation (linearize.cu) and the voxelized one (vgicp.cu).
//
// Paper: d = q - T p (eq_trans_err), M = (C^q + R C^p R^T)^-1
// (l.388-402, readings R1/R2), J = [skew(p' - c) | -I] for the pivoted left
// perturbation (R13): H += J^T M J (21), b += J^T M d (6), e += d^T M d.
#pragma once

#include "gicp_internal.cuh"

namespace gicp {

constexpr int kLinAcc = 28;  // H(21) b(6) e(1)

// per-pair terms for the residual d (fp32) at the transformed point pp: t[0..26]
// = H (21), b (6) (not written when ERROR_ONLY), returns the cost term e (fp32)
template <bool ERROR_ONLY>
__device__ __forceinline__ float point_terms(const Pose& P, const double pp[3], const float dx, const float dy,
                                             const float dz, const float cp[6], const float cq[6], float t[27]) {
    // A = C^q + R C^p R^T
    const float* R = P.Rf;
    const float C[9] = {cp[0], cp[1], cp[2], cp[1], cp[3], cp[4], cp[2], cp[4], cp[5]};
    float RC[9];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) RC[3 * a + b] = R[3 * a] * C[b] + R[3 * a + 1] * C[3 + b] + R[3 * a + 2] * C[6 + b];
    float A[6];  // upper: 00 01 02 11 12 22
    A[0] = cq[0] + (RC[0] * R[0] + RC[1] * R[1] + RC[2] * R[2]);
    A[1] = cq[1] + (RC[0] * R[3] + RC[1] * R[4] + RC[2] * R[5]);
    A[2] = cq[2] + (RC[0] * R[6] + RC[1] * R[7] + RC[2] * R[8]);
    A[3] = cq[3] + (RC[3] * R[3] + RC[4] * R[4] + RC[5] * R[5]);
    A[4] = cq[4] + (RC[3] * R[6] + RC[4] * R[7] + RC[5] * R[8]);
    A[5] = cq[5] + (RC[6] * R[6] + RC[7] * R[7] + RC[8] * R[8]);
    // M = A^-1 by the adjugate (A SPD, cond <= 1/eps)
    const float m00 = A[3] * A[5] - A[4] * A[4];
    const float m01 = A[2] * A[4] - A[1] * A[5];
    const float m02 = A[1] * A[4] - A[2] * A[3];
    const float m11 = A[0] * A[5] - A[2] * A[2];
    const float m12 = A[1] * A[2] - A[0] * A[4];
    const float m22 = A[0] * A[3] - A[1] * A[1];
    const float det = A[0] * m00 + A[1] * m01 + A[2] * m02;
    const float id = 1.0f / det;
    const float M00 = m00 * id, M01 = m01 * id, M02 = m02 * id, M11 = m11 * id, M12 = m12 * id, M22 = m22 * id;
    const float mdx = M00 * dx + M01 * dy + M02 * dz;
    const float mdy = M01 * dx + M11 * dy + M12 * dz;
    const float mdz = M02 * dx + M12 * dy + M22 * dz;
    const float et = dx * mdx + dy * mdy + dz * mdz;
    if (ERROR_ONLY) return et;
    // lever arm about the pivot (fp64 difference, then fp32)
    const float px = (float)(pp[0] - P.c[0]), py = (float)(pp[1] - P.c[1]), pz = (float)(pp[2] - P.c[2]);
    // P = skew(p') = [[0,-z,y],[z,0,-x],[-y,x,0]];  MP = M P
    const float MP00 = M01 * pz - M02 * py, MP01 = -M00 * pz + M02 * px, MP02 = M00 * py - M01 * px;
    const float MP10 = M11 * pz - M12 * py, MP11 = -M01 * pz + M12 * px, MP12 = M01 * py - M11 * px;
    const float MP20 = M12 * pz - M22 * py, MP21 = -M02 * pz + M22 * px, MP22 = M02 * py - M12 * px;
    // H_ww = P^T (M P), P^T = -P: rows of P^T: [0, z, -y], [-z, 0, x], [y, -x, 0]
    const float H00 = pz * MP10 - py * MP20;
    const float H01 = pz * MP11 - py * MP21;
    const float H02 = pz * MP12 - py * MP22;
    const float H11 = -pz * MP01 + px * MP21;
    const float H12 = -pz * MP02 + px * MP22;
    const float H22 = py * MP02 - px * MP12;
    // H_wv = -P^T M = (M P)^T  (since P^T M = -(M P)^T ... with M symmetric: (MP)^T = P^T M)
    // J = [P | -I]: J^T M J = [[P^T M P, -P^T M], [-M P, M]]; -P^T M = -(MP)^T
    const float H03 = -MP00, H04 = -MP10, H05 = -MP20;
    const float H13 = -MP01, H14 = -MP11, H15 = -MP21;
    const float H23 = -MP02, H24 = -MP12, H25 = -MP22;
    // b = J^T M d = [P^T M d; -M d];  P^T (Md) = -p' x Md
    const float b0 = pz * mdy - py * mdz;
    const float b1 = -pz * mdx + px * mdz;
    const float b2 = py * mdx - px * mdy;
    const float v[27] = {H00, H01, H02, H03, H04, H05, H11, H12, H13, H14, H15, H22,   H23,   H24,
                         H25, M00, M01, M02, M11, M12, M22, b0,  b1,  b2,  -mdx, -mdy, -mdz};
#pragma unroll
    for (int c = 0; c < 27; ++c) t[c] = v[c];
    return et;
}

// the same terms added to the fp64 acc (times w when WEIGHTED: the voxel size N of
// VGICP); returns the cost term this pair added
template <bool ERROR_ONLY, bool WEIGHTED = false>
__device__ __forceinline__ double accumulate_terms(const Pose& P, const double pp[3], const float dx, const float dy,
                                                 const float dz, const float cp[6], const float cq[6],
                                                 double acc[kLinAcc], const double w = 1.0) {
    float t[27];
    const float e = point_terms<ERROR_ONLY>(P, pp, dx, dy, dz, cp, cq, t);
    const double et = WEIGHTED ? w * (double)e : (double)e;
    acc[27] += et;
    if constexpr (!ERROR_ONLY) {
#pragma unroll
        for (int c = 0; c < 27; ++c) acc[c] += WEIGHTED ? w * (double)t[c] : (double)t[c];
    }
    return et;
}


}  // namespace gicp

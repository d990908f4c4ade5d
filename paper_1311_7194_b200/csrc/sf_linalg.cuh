// sf_linalg.cuh — small dense linear algebra of the ICP solve, host/device.
//
//   eigendecompose_sym6   cyclic Jacobi (registration.cpp:125-165). The reference forms
//                         the full plane rotation and evaluates m = rot^T * m * rot and
//                         v = v * rot as dense 6x6 products; the products only touch rows
//                         /columns p and q (the other terms are exact zeros), so the
//                         updates below are the same values in the same summation order.
//   solve_gated           eigen-gated spectral solve + unshrink (registration.cpp:167-193)
//   nearest_rotation      polar factor U V^T via two-sided Jacobi SVD with 2x2 real
//                         Jacobi steps, descending singular values (pose.cpp:20-29; the
//                         SVD algorithm is Eigen's JacobiSVD as restated in
//                         oracle/shim/Eigen/Dense)
//   apply_motion          small-angle rotation -> nearest rotation -> compose (pose.cpp:31-43)
#pragma once

#include "sf_common.cuh"

namespace sf {

// Row-major 6x6 helpers (the reference's Matrix<double,6,6> is column-major; only the
// summation order matters and it is reproduced explicitly below).
struct Eig6 {
    double values[6];   // ascending
    double vectors[36]; // column-major: vectors[c*6 + r]
};

// All loops over fixed index ranges are fully unrolled so m and v live in registers.
SF_HD void eigendecompose_sym6(const double* a /* row-major 6x6 */, Eig6& out) {
    double m[6][6], v[6][6];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            m[i][j] = 0.5 * (a[i * 6 + j] + a[j * 6 + i]);
            v[i][j] = i == j ? 1.0 : 0.0;
        }
    // m.norm(): column-major left-to-right sum of squares
    double sq = m[0][0] * m[0][0];
#pragma unroll
    for (int c = 0; c < 6; ++c)
#pragma unroll
        for (int r = 0; r < 6; ++r) {
            if (c == 0 && r == 0) continue;
            sq = sq + m[r][c] * m[r][c];
        }
    const double nrm = sqrt(sq);
    const double scl = (1.0 < nrm) ? nrm : 1.0;  // std::max(1.0, m.norm())
    const double tol = 1e-12 * scl;
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = 0.0;
#pragma unroll
        for (int p = 0; p < 6; ++p)
#pragma unroll
            for (int q = p + 1; q < 6; ++q) off += m[p][q] * m[p][q];
        if (sqrt(off) <= tol) break;
#pragma unroll
        for (int p = 0; p < 6; ++p) {
#pragma unroll
            for (int q = p + 1; q < 6; ++q) {
                const double apq = m[p][q];
                if (!(fabs(apq) <= tol / 30.0)) {
                    const double theta = (m[q][q] - m[p][p]) / (2.0 * apq);
                    const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                    const double c = 1.0 / sqrt(t * t + 1.0);
                    const double s = t * c;
                    // m1 = rot^T * m: rows p, q
#pragma unroll
                    for (int j = 0; j < 6; ++j) {
                        const double mp = m[p][j], mq = m[q][j];
                        m[p][j] = c * mp + (-s) * mq;
                        m[q][j] = s * mp + c * mq;
                    }
                    // m = m1 * rot: columns p, q
#pragma unroll
                    for (int i = 0; i < 6; ++i) {
                        const double mp = m[i][p], mq = m[i][q];
                        m[i][p] = mp * c + mq * (-s);
                        m[i][q] = mp * s + mq * c;
                    }
                    // v = v * rot
#pragma unroll
                    for (int i = 0; i < 6; ++i) {
                        const double vp = v[i][p], vq = v[i][q];
                        v[i][p] = vp * c + vq * (-s);
                        v[i][q] = vp * s + vq * c;
                    }
                }
            }
        }
    }
    // std::sort by diagonal (libstdc++ insertion sort for n <= 16: stable), on a register copy
    double d[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) d[i] = m[i][i];
    int order[6] = {0, 1, 2, 3, 4, 5};
    for (int i = 1; i < 6; ++i) {
        const int val = order[i];
        double dv = 0.0;
#pragma unroll
        for (int k = 0; k < 6; ++k)
            if (k == val) dv = d[k];
        int j = i;
        while (j > 0) {
            double dp = 0.0;
            const int o = order[j - 1];
#pragma unroll
            for (int k = 0; k < 6; ++k)
                if (k == o) dp = d[k];
            if (!(dv < dp)) break;
            order[j] = o;
            --j;
        }
        order[j] = val;
    }
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        const int o = order[i];
#pragma unroll
        for (int k = 0; k < 6; ++k)
            if (k == o) {
                out.values[i] = d[k];
#pragma unroll
                for (int r = 0; r < 6; ++r) out.vectors[i * 6 + r] = v[r][k];
            }
    }
}

#ifdef __CUDACC__
// Warp-cooperative eigendecompose_sym6 (call with all 32 lanes of one warp). Lane i < 6
// owns row i of m and of v; a rotation broadcasts the pre-rotation rows p and q, lanes p
// and q form rot^T * m for their rows, then every lane applies * rot to its columns p, q
// and to its row of v. Each element sees the same operations in the same order as the
// sequential version above, so the results are bit-identical; the critical path shrinks
// from ~36 dependent updates per rotation to ~4. `a` is row-major 6x6 (shared memory),
// `out` is written by lanes 0..5.
__device__ __forceinline__ void eigendecompose_sym6_warp(const double* a, Eig6* out) {
    constexpr unsigned kFull = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int r = lane < 6 ? lane : 0;
    double m[6], v[6];
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        m[j] = 0.5 * (a[r * 6 + j] + a[j * 6 + r]);
        v[j] = r == j ? 1.0 : 0.0;
    }
    double sq = 0.0;
#pragma unroll
    for (int c = 0; c < 6; ++c)
#pragma unroll
        for (int rr = 0; rr < 6; ++rr) {
            const double x = 0.5 * (a[rr * 6 + c] + a[c * 6 + rr]);
            sq = (c == 0 && rr == 0) ? x * x : sq + x * x;
        }
    const double nrm = sqrt(sq);
    const double scl = (1.0 < nrm) ? nrm : 1.0;
    const double tol = 1e-12 * scl;
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = 0.0;
#pragma unroll
        for (int p = 0; p < 6; ++p)
#pragma unroll
            for (int q = p + 1; q < 6; ++q) {
                const double mpq = __shfl_sync(kFull, m[q], p);
                off += mpq * mpq;
            }
        if (sqrt(off) <= tol) break;
#pragma unroll
        for (int p = 0; p < 6; ++p) {
#pragma unroll
            for (int q = p + 1; q < 6; ++q) {
                double rp[6], rq[6];
#pragma unroll
                for (int j = 0; j < 6; ++j) {
                    rp[j] = __shfl_sync(kFull, m[j], p);
                    rq[j] = __shfl_sync(kFull, m[j], q);
                }
                const double apq = rp[q];
                if (!(fabs(apq) <= tol / 30.0)) {
                    const double theta = (rq[q] - rp[p]) / (2.0 * apq);
                    const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                    const double c = 1.0 / sqrt(t * t + 1.0);
                    const double s = t * c;
                    if (r == p) {
#pragma unroll
                        for (int j = 0; j < 6; ++j) m[j] = c * rp[j] + (-s) * rq[j];
                    } else if (r == q) {
#pragma unroll
                        for (int j = 0; j < 6; ++j) m[j] = s * rp[j] + c * rq[j];
                    }
                    const double mp = m[p], mq = m[q];
                    m[p] = mp * c + mq * (-s);
                    m[q] = mp * s + mq * c;
                    const double vp = v[p], vq = v[q];
                    v[p] = vp * c + vq * (-s);
                    v[q] = vp * s + vq * c;
                }
            }
        }
    }
    double d[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) d[k] = __shfl_sync(kFull, m[k], k);
    int order[6] = {0, 1, 2, 3, 4, 5};  // stable insertion sort, as the sequential version
    for (int i = 1; i < 6; ++i) {
        const int val = order[i];
        double dv = 0.0;
#pragma unroll
        for (int k = 0; k < 6; ++k)
            if (k == val) dv = d[k];
        int j = i;
        while (j > 0) {
            double dp = 0.0;
            const int o = order[j - 1];
#pragma unroll
            for (int k = 0; k < 6; ++k)
                if (k == o) dp = d[k];
            if (!(dv < dp)) break;
            order[j] = o;
            --j;
        }
        order[j] = val;
    }
    if (lane < 6) {
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            const int o = order[i];
#pragma unroll
            for (int k = 0; k < 6; ++k)
                if (k == o) {
                    if (lane == 0) out->values[i] = d[k];
                    out->vectors[i * 6 + lane] = v[k];
                }
        }
    }
}
#endif

// ---- 3x3 Jacobi SVD (Eigen JacobiSVD restated) ------------------------------------
struct Rot2 {
    double c, s;
};
SF_HD Rot2 rot_mul(Rot2 a, Rot2 b) { return Rot2{a.c * b.c - a.s * b.s, a.c * b.s + a.s * b.c}; }
SF_HD Rot2 rot_t(Rot2 a) { return Rot2{a.c, -a.s}; }

SF_HD void make_jacobi(double x, double y, double z, Rot2& j) {
    const double deno = 2.0 * fabs(y);
    if (deno < 2.2250738585072014e-308) {
        j.c = 1.0;
        j.s = 0.0;
        return;
    }
    const double tau = (x - z) / deno;
    const double w = sqrt(tau * tau + 1.0);
    double t;
    if (tau > 0.0) t = 1.0 / (tau + w);
    else t = 1.0 / (tau - w);
    const double sign_t = t > 0.0 ? 1.0 : -1.0;
    const double n = 1.0 / sqrt(t * t + 1.0);
    j.s = -sign_t * (y / fabs(y)) * fabs(t) * n;
    j.c = n;
}

// m is row-major 3x3: m[r][c]
SF_HD void real_2x2_jacobi_svd(const double (*mat)[3], int p, int q, Rot2& jl, Rot2& jr) {
    double m00 = mat[p][p], m01 = mat[p][q], m10 = mat[q][p], m11 = mat[q][q];
    Rot2 rot1;
    const double t = m00 + m11;
    const double d = m10 - m01;
    if (fabs(d) < 2.2250738585072014e-308) {
        rot1.s = 0.0;
        rot1.c = 1.0;
    } else {
        const double u = t / d;
        const double tmp = sqrt(1.0 + u * u);
        rot1.s = 1.0 / tmp;
        rot1.c = u / tmp;
    }
    {
        const double a0 = m00, a1 = m01, b0 = m10, b1 = m11;
        m00 = rot1.c * a0 + rot1.s * b0;
        m01 = rot1.c * a1 + rot1.s * b1;
        m10 = -rot1.s * a0 + rot1.c * b0;
        m11 = -rot1.s * a1 + rot1.c * b1;
        (void)m10;
    }
    make_jacobi(m00, m01, m11, jr);
    jl = rot_mul(rot1, rot_t(jr));
}

SF_HD void apply_left3(double (*m)[3], int p, int q, Rot2 j) {
    for (int k = 0; k < 3; ++k) {
        const double xi = m[p][k], yi = m[q][k];
        m[p][k] = j.c * xi + j.s * yi;
        m[q][k] = -j.s * xi + j.c * yi;
    }
}
SF_HD void apply_right3(double (*m)[3], int p, int q, Rot2 j) {
    for (int k = 0; k < 3; ++k) {
        const double xi = m[k][p], yi = m[k][q];
        m[k][p] = j.c * xi - j.s * yi;
        m[k][q] = j.s * xi + j.c * yi;
    }
}

// nearest_rotation (pose.cpp:20-29)
SF_HD m33 nearest_rotation(const m33& a) {
    double work[3][3], u[3][3], v[3][3];
    double scl = fabs(a.m[0]);
    // cwiseAbs().maxCoeff() in column-major order
    for (int c = 0; c < 3; ++c)
        for (int r = 0; r < 3; ++r) {
            const double x = fabs(a.m[r * 3 + c]);
            scl = scl < x ? x : scl;
        }
    if (scl == 0.0) scl = 1.0;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            work[r][c] = a.m[r * 3 + c] / scl;
            u[r][c] = r == c ? 1.0 : 0.0;
            v[r][c] = r == c ? 1.0 : 0.0;
        }
    const double considerAsZero = 2.2250738585072014e-308;
    const double precision = 2.0 * 2.220446049250313e-16;
    double maxDiag = fabs(work[0][0]);
    maxDiag = maxDiag < fabs(work[1][1]) ? fabs(work[1][1]) : maxDiag;
    maxDiag = maxDiag < fabs(work[2][2]) ? fabs(work[2][2]) : maxDiag;
    bool finished = false;
    int sweeps = 0;
    while (!finished && sweeps < 64) {
        finished = true;
        ++sweeps;
#pragma unroll
        for (int p = 1; p < 3; ++p) {
#pragma unroll
            for (int q = 0; q < p; ++q) {
                const double pm = precision * maxDiag;
                const double threshold = considerAsZero < pm ? pm : considerAsZero;
                if (fabs(work[p][q]) > threshold || fabs(work[q][p]) > threshold) {
                    finished = false;
                    Rot2 jl, jr;
                    real_2x2_jacobi_svd(work, p, q, jl, jr);
                    apply_left3(work, p, q, jl);
                    apply_right3(u, p, q, rot_t(jl));
                    apply_right3(work, p, q, jr);
                    apply_right3(v, p, q, jr);
                    const double a_pp = fabs(work[p][p]), a_qq = fabs(work[q][q]);
                    const double mx = a_pp < a_qq ? a_qq : a_pp;
                    maxDiag = maxDiag < mx ? mx : maxDiag;
                }
            }
        }
    }
    double sv[3];
    for (int i = 0; i < 3; ++i) {
        const double aii = work[i][i];
        sv[i] = fabs(aii);
        if (aii < 0.0)
            for (int k = 0; k < 3; ++k) u[k][i] = -u[k][i];
    }
    for (int i = 0; i < 3; ++i) sv[i] = sv[i] * scl;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        // first maximum of sv[i..2] (Eigen maxCoeff(&pos)), swapped into place
        int pos = i;
        double best = sv[i];
#pragma unroll
        for (int k = i + 1; k < 3; ++k)
            if (sv[k] > best) {
                pos = k;
                best = sv[k];
            }
#pragma unroll
        for (int c = i + 1; c < 3; ++c) {
            if (c != pos) continue;
            const double t = sv[i];
            sv[i] = sv[c];
            sv[c] = t;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                double x = u[k][i];
                u[k][i] = u[k][c];
                u[k][c] = x;
                x = v[k][i];
                v[k][i] = v[k][c];
                v[k][c] = x;
            }
        }
    }
    m33 U, V;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            U.m[r * 3 + c] = u[r][c];
            V.m[r * 3 + c] = v[r][c];
        }
    m33 R = mm(U, mt(V));
    // determinant (shim order, grid-independent): m(0,0)*(m11*m22 - m21*m12) - m10*(...) + m20*(...)
    const double* M = R.m;
    auto at = [&](int r, int c) { return M[r * 3 + c]; };
    const double det = at(0, 0) * (at(1, 1) * at(2, 2) - at(2, 1) * at(1, 2)) -
                       at(1, 0) * (at(0, 1) * at(2, 2) - at(2, 1) * at(0, 2)) +
                       at(2, 0) * (at(0, 1) * at(1, 2) - at(1, 1) * at(0, 2));
    if (det < 0.0) {
        m33 flip;
        for (int i = 0; i < 9; ++i) flip.m[i] = 0.0;
        flip.m[0] = 1.0;
        flip.m[4] = 1.0;
        flip.m[8] = -1.0;
        R = mm(mm(U, flip), mt(V));
    }
    return R;
}

// apply_motion (pose.cpp:31-43)
SF_HD Pose apply_motion(const Pose& pose, d3 r, d3 t) {
    const double a = r.x, b = r.y, g = r.z;
    m33 lin;
    lin.m[0] = 1.0;
    lin.m[1] = -g;
    lin.m[2] = b;
    lin.m[3] = g;
    lin.m[4] = 1.0;
    lin.m[5] = -a;
    lin.m[6] = -b;
    lin.m[7] = a;
    lin.m[8] = 1.0;
    Pose corr;
    corr.R = nearest_rotation(lin);
    corr.t = t;
    return compose(corr, pose);
}

// apply_motion with the polar factor in closed form. The small-angle matrix is I + [w]x
// (w = r); (I + W)^T (I + W) = I - W^2 has eigenvalue 1 along w and 1 + |w|^2 across it, so
// its nearest rotation U V^T = (I + W) (I - W^2)^(-1/2) = k (I + W) + m w w^T with
// k = 1 / sqrt(1 + |w|^2), m = 1 / (sqrt(1 + |w|^2) (1 + sqrt(1 + |w|^2))) (W w = 0).
// Equal to the SVD route up to rounding (the polar factor of a non-singular matrix is
// unique); one sqrt and two divisions instead of Jacobi SVD sweeps.
SF_HD Pose apply_motion_fast(const Pose& pose, d3 r, d3 t) {
    const double a = r.x, b = r.y, g = r.z;
    const double x = (a * a + b * b) + g * g;
    const double sq = sqrt(1.0 + x);
    const double k = 1.0 / sq, m = 1.0 / (sq * (1.0 + sq));
    Pose corr;
    corr.R.m[0] = k + m * a * a;
    corr.R.m[1] = -k * g + m * a * b;
    corr.R.m[2] = k * b + m * a * g;
    corr.R.m[3] = k * g + m * b * a;
    corr.R.m[4] = k + m * b * b;
    corr.R.m[5] = -k * a + m * b * g;
    corr.R.m[6] = -k * b + m * g * a;
    corr.R.m[7] = k * a + m * g * b;
    corr.R.m[8] = k + m * g * g;
    corr.t = t;
    return compose(corr, pose);
}

#ifdef __CUDACC__
// Jacobi eigendecomposition of a symmetric 6x6 by one warp with the parallel (round-robin)
// ordering: each sweep is 5 rounds of 3 disjoint rotations, applied together (disjoint plane
// rotations commute), so a sweep has 5 dependent rotation steps instead of 15. Same
// rotation formula, thresholds and stopping rule as registration.cpp:125-165; the ordering
// changes rounding only (the device ICP is tolerance-checked). Lane i < 6
// owns row i of m and of v. Output as eigendecompose_sym6 (ascending, stable order).
__device__ __forceinline__ void eigendecompose_sym6_warp_rr(const double* a, Eig6* out) {
    constexpr unsigned kFull = 0xffffffffu;
    // partner of lane i in round r (perfect matchings of K6)
    constexpr int kPartner[5][6] = {{1, 0, 3, 2, 5, 4}, {2, 4, 0, 5, 1, 3}, {3, 5, 4, 0, 2, 1},
                                    {4, 3, 5, 1, 0, 2}, {5, 2, 1, 4, 3, 0}};
    const int lane = threadIdx.x & 31;
    const int r = lane < 6 ? lane : 0;
    double m[6], v[6];
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        m[j] = 0.5 * (a[r * 6 + j] + a[j * 6 + r]);
        v[j] = r == j ? 1.0 : 0.0;
    }
    double sq = 0.0;
#pragma unroll
    for (int c = 0; c < 6; ++c)
#pragma unroll
        for (int rr = 0; rr < 6; ++rr) {
            const double x = 0.5 * (a[rr * 6 + c] + a[c * 6 + rr]);
            sq = (c == 0 && rr == 0) ? x * x : sq + x * x;
        }
    const double nrm = sqrt(sq);
    const double tol = 1e-12 * ((1.0 < nrm) ? nrm : 1.0);
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = 0.0;  // sum of squares above the diagonal, same value in every lane
#pragma unroll
        for (int p = 0; p < 6; ++p)
#pragma unroll
            for (int q = p + 1; q < 6; ++q) {
                const double mpq = __shfl_sync(kFull, m[q], p);
                off += mpq * mpq;
            }
        if (sqrt(off) <= tol) break;
#pragma unroll
        for (int rd = 0; rd < 5; ++rd) {
            // my pair (p, q), p < q; lanes >= 6 mirror lane 0
            int j = 0;
#pragma unroll
            for (int i = 0; i < 6; ++i)
                if (r == i) j = kPartner[rd][i];
            const int p = r < j ? r : j;
            double mrow_j[6];
#pragma unroll
            for (int k = 0; k < 6; ++k) mrow_j[k] = __shfl_sync(kFull, m[k], j);
            // app, aqq, apq from my row and the partner's row
            double mine_rr = 0.0, mine_rj = 0.0, part_jj = 0.0;
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                if (k == r) mine_rr = m[k];
                if (k == j) mine_rj = m[k];
                if (k == j) part_jj = mrow_j[k];
            }
            const double app = r == p ? mine_rr : part_jj, aqq = r == p ? part_jj : mine_rr;
            double apq = mine_rj;  // row p, column q: owned by lane p
            {
                double part_jr = 0.0;
#pragma unroll
                for (int k = 0; k < 6; ++k)
                    if (k == r) part_jr = mrow_j[k];
                if (r != p) apq = part_jr;
            }
            double c = 1.0, s = 0.0;
            if (!(fabs(apq) <= tol / 30.0)) {
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                c = 1.0 / sqrt(t * t + 1.0);
                s = t * c;
            }
            // rows: rot^T * m for my row (p: c*row_p - s*row_q; q: s*row_p + c*row_q)
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                const double mp = r == p ? m[k] : mrow_j[k], mq = r == p ? mrow_j[k] : m[k];
                m[k] = r == p ? c * mp + (-s) * mq : s * mp + c * mq;
            }
            // columns: (rot^T m) * rot and v * rot; every lane needs all three pairs' (c, s)
#pragma unroll
            for (int pp = 0; pp < 6; ++pp) {
                const int qq = kPartner[rd][pp];
                if (qq < pp) continue;
                const double cp = __shfl_sync(kFull, c, pp), sp = __shfl_sync(kFull, s, pp);
                const double xp = m[pp], xq = m[qq];
                m[pp] = xp * cp + xq * (-sp);
                m[qq] = xp * sp + xq * cp;
                const double vp = v[pp], vq = v[qq];
                v[pp] = vp * cp + vq * (-sp);
                v[qq] = vp * sp + vq * cp;
            }
        }
    }
    double d[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) d[k] = __shfl_sync(kFull, m[k], k);
    int order[6] = {0, 1, 2, 3, 4, 5};
    for (int i = 1; i < 6; ++i) {
        const int val = order[i];
        double dv = 0.0;
#pragma unroll
        for (int k = 0; k < 6; ++k)
            if (k == val) dv = d[k];
        int j = i;
        while (j > 0) {
            double dp = 0.0;
            const int o = order[j - 1];
#pragma unroll
            for (int k = 0; k < 6; ++k)
                if (k == o) dp = d[k];
            if (!(dv < dp)) break;
            order[j] = o;
            --j;
        }
        order[j] = val;
    }
    if (lane < 6) {
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            const int o = order[i];
#pragma unroll
            for (int k = 0; k < 6; ++k)
                if (k == o) {
                    if (lane == 0) out->values[i] = d[k];
                    out->vectors[i * 6 + lane] = v[k];
                }
        }
    }
}
#endif

}  // namespace sf

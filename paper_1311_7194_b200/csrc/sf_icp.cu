// sf_icp.cu — projective point-to-plane ICP on the device (registration.cpp:17-224).
//
// Every iteration is ONE launch with device-side control (no host round trip):
//   k_icp_step  per source pixel: projective association + distance / normal rejection
//               (registration.cpp:17-50), then the 21 + 6 + 1 normal-equation sums in
//               unshrunk form (double-double TwoSum accumulators) and the shrink bounding box
//               (registration.cpp:52-123); CTA partials in a fixed order. The last CTA merges
//               them, raises TrackingLost below 10 matches (registration.cpp:202-204), forms
//               the shrink (centre / scale) and applies it to the sums as a linear map; one
//               warp runs the Jacobi 6x6 (rows across lanes, bit-identical to the sequential
//               sweep), one thread the gated solve, unshrink, apply_motion and the
//               convergence test (registration.cpp:125-220).
// Under CUDA-graph capture (tracker) the iterations are a conditional WHILE node: the body
// repeats until converged / lost / max_iterations, decided on the device. Issued eagerly,
// a converged / failed state makes the remaining iterations' kernels exit at once.
// Partials are merged in a fixed order, so results are deterministic run to run.
//
// Parity: the association is FP64 in the reference order (the same matches). The normal
// equations differ from the reference's by rounding only: tree instead of sequential Kahan
// summation, and shrink applied to the sums instead of to each match (~1e-15 relative);
// pose parity is asserted at 1e-6.
#include <algorithm>
#include <functional>
#include <cmath>
#include <cstdlib>
#include <string>

#include "sf_icp.cuh"
#include "sf_linalg.cuh"

namespace sf {

#ifdef SF_DIAG_ICP_TAIL  // timing diagnostics: timestamps of the last step's tail
__device__ unsigned long long g_icp_dbg[8];
#define SF_ICP_STAMP(i) (g_icp_dbg[i] = globaltimer_ns())
extern "C" int sf_debug_icp_tail(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, g_icp_dbg, 8 * sizeof(unsigned long long));
}
#else
#define SF_ICP_STAMP(i) ((void)0)
#endif

// COND: the launch sits in a graph with the device-side iteration loop and drives its
// condition. (Separate instantiations: kernels that call the device graph API are not
// profiled by Nsight Compute, so the eager / fixed-sequence form must not contain the call.)
template <bool COND>
__global__ void k_icp_init(IcpState* st, const double* __restrict__ initial12, const int* dead, int max_iterations,
                           cudaGraphConditionalHandle cond) {
    icp_state_init(st, initial12, dead && *dead);
    if constexpr (COND) cudaGraphSetConditional(cond, (!st->done && max_iterations > 0) ? 1u : 0u);
}

// Returns true in every thread of the CTA that finished last (all partials visible).
__device__ __forceinline__ bool last_cta(unsigned int* counter) {
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (s_last) __threadfence();
    return s_last;
}

// solve_gated + apply_motion + convergence (registration.cpp:175-212), one thread.
// The eigendecomposition of the normal matrix is done before, by one warp (e).
__device__ __noinline__ void solve_finalize(IcpState* st, const double* s_sum, const Eig6& e,
                                            const IcpParamsDev& prm, bool exact_motion = false) {
    const int iter = st->iterations;  // iterations completed before this one
    double b[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) b[i] = s_sum[21 + i];
    const double res_sq = s_sum[27];
    const unsigned long long cnt = st->cur_count;
    const double n_pairs = static_cast<double>(cnt);
    st->pair_count = cnt;
    st->residual_rms = sqrt(dmax(0.0, res_sq) / n_pairs);
    double x[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        st->eigenvalues[i] = e.values[i];
        const bool keep = e.values[i] / n_pairs > prm.theta;
        st->gated[i] = keep ? 1 : 0;
        if (keep) {
            const double* vcol = e.vectors + i * 6;
            double vb = vcol[0] * b[0];
#pragma unroll
            for (int r = 1; r < 6; ++r) vb = vb + vcol[r] * b[r];
            const double sc = vb / e.values[i];
#pragma unroll
            for (int r = 0; r < 6; ++r) x[r] = x[r] + vcol[r] * sc;
        }
    }
#pragma unroll
    for (int i = 0; i < 36; ++i) st->eigenvectors[i] = e.vectors[i];
    double xn = x[0] * x[0];
#pragma unroll
    for (int r = 1; r < 6; ++r) xn = xn + x[r] * x[r];
    st->shrunk_norm = sqrt(xn);
    // unshrink_motion (registration.cpp:167-173)
    const d3 s = st->scale, c = st->center;
    const d3 r = mk((1.0 / s.x) * x[0], (1.0 / s.y) * x[1], (1.0 / s.z) * x[2]);
    const d3 t = sub(mk(x[3], x[4], x[5]), cross(r, c));
    st->motion_r = r;
    st->motion_t = t;
    // apply_motion (pose.cpp:31-43): the reference's SVD route, or its closed form (same polar
    // factor up to rounding)
    st->delta = exact_motion ? apply_motion(st->delta, r, t) : apply_motion_fast(st->delta, r, t);
    st->eig_pending = 0;  // eigenpairs computed by this path
    st->iterations = iter + 1;
    if (st->shrunk_norm < prm.eps) st->done = 1;
}

// Fast path of solve_gated (registration.cpp:175-193). When every eigenvalue of A passes the
// gate lambda_i / N > theta, the gated solution sum_i v_i (v_i . b) / lambda_i is A^-1 b. A
// Cholesky factorisation of A - c I succeeding certifies lambda_min(A) > c - |E| (backward
// stability, |E| <= 7 eps |A|_F); c = theta N (1 + 1e-9) + 64 eps |A|_F leaves room for the
// reference's own eigenvalue rounding, so the reference gates every direction in too. Then
// x = A^-1 b by a second Cholesky (same solution up to rounding). Returns false (Jacobi path)
// otherwise. One thread.
// The two factorisations run on two lanes: pass 0 the shifted one (the certificate), pass 1
// the unshifted one and the two triangular solves (x). The fast path holds when both succeed.
__device__ __noinline__ bool fast_gated_solve(const double* s_fin, double n_pairs, double theta, int pass, double* x) {
    double A[6][6];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int j = i; j < 6; ++j) A[i][j] = A[j][i] = s_fin[i * 6 - i * (i - 1) / 2 + (j - i)];
    double sh = 0.0;
    if (pass == 0) {
        double fro = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i)
#pragma unroll
            for (int j = 0; j < 6; ++j) fro += A[i][j] * A[i][j];
        fro = sqrt(fro);
        sh = theta * n_pairs * (1.0 + 1e-9) + 64.0 * 2.220446049250313e-16 * fro;
    }
    double L[6][6], invd[6];
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        double s = A[j][j] - sh;
#pragma unroll
        for (int k = 0; k < j; ++k) s -= L[j][k] * L[j][k];
        if (!(s > 0.0)) return false;
        // 1/sqrt(s) and sqrt(s) = s / sqrt(s) from one reciprocal square root (a few ulps; the
        // certificate's shift leaves 64 eps |A|_F for 7 eps |A|_F of backward error)
        const double inv = rsqrt(s), d = s * inv;
        L[j][j] = d;
        invd[j] = inv;
#pragma unroll
        for (int i = j + 1; i < 6; ++i) {
            double t = A[i][j];
#pragma unroll
            for (int k = 0; k < j; ++k) t -= L[i][k] * L[j][k];
            L[i][j] = t * inv;
        }
    }
    if (pass == 0) return true;
    double y[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) {  // L y = b
        double t = s_fin[21 + i];
#pragma unroll
        for (int k = 0; k < i; ++k) t -= L[i][k] * y[k];
        y[i] = t * invd[i];  // reciprocal of the pivot from the factorisation (ulp-level vs t / L[i][i])
    }
#pragma unroll
    for (int i = 5; i >= 0; --i) {  // L^T x = y
        double t = y[i];
#pragma unroll
        for (int k = i + 1; k < 6; ++k) t -= L[k][i] * x[k];
        x[i] = t * invd[i];
    }
    return true;
}

// Gated solution x (fast path) -> the rest of solve_gated + apply_motion + convergence.
__device__ __noinline__ void finalize_motion(IcpState* st, const double* s_fin, const double* x, const IcpParamsDev& prm) {
    const int iter = st->iterations;
    const unsigned long long cnt = st->cur_count;
    st->pair_count = cnt;
    st->residual_rms = sqrt(dmax(0.0, s_fin[27]) / static_cast<double>(cnt));
    for (int i = 0; i < 6; ++i) st->gated[i] = 1;
    for (int i = 0; i < 21; ++i) st->A_last[i] = s_fin[i];
    st->eig_pending = 1;
    double xn = x[0] * x[0];
#pragma unroll
    for (int r = 1; r < 6; ++r) xn = xn + x[r] * x[r];
    st->shrunk_norm = sqrt(xn);
    const d3 is = st->inv_scale, c = st->center;  // inv_scale = 1.0 / scale (set with it)
    const d3 r = mk(is.x * x[0], is.y * x[1], is.z * x[2]);
    const d3 t = sub(mk(x[3], x[4], x[5]), cross(r, c));
    st->motion_r = r;
    st->motion_t = t;
    st->delta = apply_motion_fast(st->delta, r, t);
    st->iterations = iter + 1;
    if (st->shrunk_norm < prm.eps) st->done = 1;
}

// Deferred eigendecomposition of the last iteration's normal matrix (GatedSolution
// eigenvalues / eigenvectors for IcpResult and the frame metrics). One warp.
__global__ void k_icp_report(IcpState* st) {
    if (!st->eig_pending) return;
    __shared__ double s_A[36];
    __shared__ Eig6 s_eig;
    const int lane = threadIdx.x & 31;
    for (int i = lane; i < 36; i += 32) {
        const int r = i / 6, c = i % 6;
        const int a = r <= c ? r : c, b = r <= c ? c : r;
        s_A[i] = st->A_last[a * 6 - a * (a - 1) / 2 + (b - a)];
    }
    __syncwarp();
    eigendecompose_sym6_warp_rr(s_A, &s_eig);
    __syncwarp();
    if (lane < 6) st->eigenvalues[lane] = s_eig.values[lane];
    for (int i = lane; i < 36; i += 32) st->eigenvectors[i] = s_eig.vectors[i];
    if (lane == 0) st->eig_pending = 0;
}

#ifndef SF_ICP_STEP_THREADS
#define SF_ICP_STEP_THREADS 256
#endif
#ifndef SF_ICP_STEP_CTAS
#define SF_ICP_STEP_CTAS 296
#endif
constexpr int kStepThreads = SF_ICP_STEP_THREADS;  // k_icp_step: threads per CTA
constexpr int kStepCtas = SF_ICP_STEP_CTAS;  // fixed => deterministic reduction tree
static_assert(kStepCtas <= kIcpCtas, "partial buffers hold kIcpCtas CTAs");
// CTA-reduction transpose [kSums][kStepThreads / 32 segments][33]: the padding puts the 32-value
// segments that the merge threads of one warp walk in lockstep on different banks
constexpr int kSegStride = 33, kSumStride = (kStepThreads / 32) * kSegStride;
constexpr int kStepSmem = kSums * kSumStride * static_cast<int>(sizeof(double));
constexpr int kMergeLanes = kStepThreads / kSums;  // threads per sum in the final merge (252 of 256 busy)

// match_points association for source pixel i (registration.cpp:17-50).
__device__ __forceinline__ bool associate(int i, const float* __restrict__ src, const float* __restrict__ src_n,
                                          const float* __restrict__ tgt, const float* __restrict__ tgt_n,
                                          const Intr& si, const Intr& ti, const IcpParamsDev& prm, const Pose& delta,
                                          d3& p, d3& q, d3& nn) {
    const int u = i % si.w, v = i / si.w;
    const float sd = src[i];
    const float snx = src_n[3 * i], sny = src_n[3 * i + 1], snz = src_n[3 * i + 2];
    if (!(sd > 0.0f && (snx * snx + sny * sny) + snz * snz > 0.0f)) return false;
    p = apply(delta, unproject(si, u, v, sd));
    double pu, pv;
    if (!project(ti, p, pu, pv)) return false;
    const int tu = ref_lround_int(pu), tv = ref_lround_int(pv);
    if (!(tu >= 0 && tv >= 0 && tu < ti.w && tv < ti.h)) return false;
    const int j = tv * ti.w + tu;
    const float td = tgt[j];
    const float tnx = tgt_n[3 * j], tny = tgt_n[3 * j + 1], tnz = tgt_n[3 * j + 2];
    if (!(td > 0.0f && (tnx * tnx + tny * tny) + tnz * tnz > 0.0f)) return false;
    q = unproject(ti, tu, tv, td);
    if (sqnorm(sub(p, q)) > prm.max_dist_sq) return false;
    nn = mk(tnx, tny, tnz);
    const d3 ns = mv(delta.R, mk(snx, sny, snz));
    return !(dot(ns, nn) < prm.cos_max);
}

__host__ __device__ constexpr int packed_index(int i, int j) {  // upper triangle of 6x6, row-major, i <= j
    return i * 6 - i * (i - 1) / 2 + (j - i);
}

// The solve of one iteration from its merged unshrunk sums (one warp; lanes of warp 0).
// st->center / scale / inv_scale / cur_count are set. Shrink as a linear map on the sums,
// gated solve (certified Cholesky fast path, else the warp Jacobi), pose update,
// convergence, and the loop condition. `counter` (the last-CTA ticket) is reset.
template <bool COND>
__device__ __noinline__ void solve_from_sums(IcpState* st, double* s_sum, double* s_fin, const IcpParamsDev& prm,
                                             unsigned int* counter, cudaGraphConditionalHandle cond) {
    const int lane = threadIdx.x & 31;
    // ---- shrink as a linear map on the sums: A = L S6 L^T, b = -L t6, with
    // L = [[D, -D C], [0, I]], D = diag(1/s), C = [c]x (one thread, fully unrolled: the 36
    // entries are independent, so the latency overlaps).
    if (lane == 0) {
        const d3 c = st->center, inv = st->inv_scale;
        const double C[3][3] = {{0.0, -c.z, c.y}, {c.z, 0.0, -c.x}, {-c.y, c.x, 0.0}};
        const double D[3] = {inv.x, inv.y, inv.z};
        double S[6][6];
#pragma unroll
        for (int i = 0; i < 6; ++i)
#pragma unroll
            for (int j = i; j < 6; ++j) S[i][j] = S[j][i] = s_sum[packed_index(i, j)];
        // G = S L^T restricted to what is needed: G[k][j] = sum_l S[k][l] L[j][l]
        double G[6][6];
#pragma unroll
        for (int k = 0; k < 6; ++k) {
#pragma unroll
            for (int j = 0; j < 3; ++j) {  // L[j] = (D_j e_j, -D_j C[j])
                double t = S[k][j];
#pragma unroll
                for (int l = 0; l < 3; ++l) t -= S[k][3 + l] * C[j][l];
                G[k][j] = D[j] * t;
            }
#pragma unroll
            for (int j = 3; j < 6; ++j) G[k][j] = S[k][j];
        }
#pragma unroll
        for (int i = 0; i < 6; ++i)
#pragma unroll
            for (int j = i; j < 6; ++j) {
                double a;
                if (i < 3) {
                    a = G[i][j];
#pragma unroll
                    for (int l = 0; l < 3; ++l) a -= C[i][l] * G[3 + l][j];
                    a *= D[i];
                } else {
                    a = G[i][j];
                }
                s_fin[packed_index(i, j)] = a;
            }
        const double* T = s_sum + 21;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            double t = T[i];
#pragma unroll
            for (int l = 0; l < 3; ++l) t -= C[i][l] * T[3 + l];
            s_fin[21 + i] = -(D[i] * t);
        }
#pragma unroll
        for (int i = 3; i < 6; ++i) s_fin[21 + i] = -T[i];
        s_fin[27] = s_sum[27];
    }
    __syncwarp();
    if (lane == 0) SF_ICP_STAMP(2);
    double x[6];
    const bool ok = lane < 2 && fast_gated_solve(s_fin, static_cast<double>(st->cur_count), prm.theta, lane, x);
    const bool s_fast = (__ballot_sync(0xffffffffu, ok) & 3u) == 3u;
    if (lane == 1) {
        SF_ICP_STAMP(3);
        if (s_fast) {
            finalize_motion(st, s_fin, x, prm);
            SF_ICP_STAMP(4);
            *counter = 0;
            st->t_end = globaltimer_ns();
            if constexpr (COND)
                cudaGraphSetConditional(cond, (!st->done && st->iterations < prm.max_iterations) ? 1u : 0u);
        }
    }
    __syncwarp();
    if (s_fast) return;
    __shared__ double s_A[36];
    __shared__ Eig6 s_eig;
    for (int i = lane; i < 36; i += 32) {
        const int r = i / 6, cc = i % 6;
        s_A[i] = s_fin[r <= cc ? packed_index(r, cc) : packed_index(cc, r)];
    }
    __syncwarp();
    eigendecompose_sym6_warp_rr(s_A, &s_eig);
    __syncwarp();
    if (lane == 0) {
        solve_finalize(st, s_fin, s_eig, prm);
        *counter = 0;
        st->t_end = globaltimer_ns();
        if constexpr (COND)
            cudaGraphSetConditional(cond, (!st->done && st->iterations < prm.max_iterations) ? 1u : 0u);
    }}

// One ICP iteration (registration.cpp:17-123 + 175-212) in one launch.
//
// The reference shrinks the matches (centre c, scale s from their bounding box) before it
// assembles A = sum row row^T, b = -sum row d with row = (s^-1 (p - c) x n, n) and
// d = (s (p^ - q^)) . n. Both are linear in the unshrunk sums: row = L (p x n, n) with
// L = [[S^-1, -S^-1 [c]x], [0, I]] and d = (p - q) . n, so A = L S6 L^T, b = -L t6 where
// S6 = sum r r^T, t6 = sum r d over r = (p x n, n). Every CTA therefore accumulates the 28
// unshrunk sums (double-double) together with the bounding box in the same pass as the
// association, and the last CTA to finish merges the partials in a fixed order, forms c, s,
// applies L (~1e-15 relative: the same result as shrinking first, up to rounding), runs the
// warp-parallel Jacobi and the gated solve. No match records go through HBM.
//
// PARTIAL (sharded ICP, north star "27-float allreduce"): the pass covers only the source
// pixels [pix0, pix1) of this rank, and the last CTA writes the rank's merged partial sums,
// box and count to `rec` instead of solving; the ranks' records are then all-reduced and
// k_icp_solve_ranks solves (identically on every rank).
template <bool COND, bool PARTIAL = false>
__global__ void __launch_bounds__(kStepThreads, 512 / kStepThreads)
    k_icp_step(const float* __restrict__ src, const float* __restrict__ src_n, const float* __restrict__ tgt,
               const float* __restrict__ tgt_n, Intr si, Intr ti, IcpParamsDev prm, IcpState* st,
               double* __restrict__ part_bbox, unsigned long long* __restrict__ part_count, DD* __restrict__ part,
               unsigned int* counter, cudaGraphConditionalHandle cond, int pix0 = 0, int pix1 = 0x7fffffff,
               IcpRankPartial* rec = nullptr) {
    extern __shared__ double s_red[];  // [kSums][segments][kSegStride]
    if (threadIdx.x == 0 && st->bodies == 0) atomicCAS(&st->t_step0, 0ull, globaltimer_ns());
    if (st->done) {  // converged / lost: end the device-side loop
        if constexpr (COND && !PARTIAL) {
            if (blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0u);
        }
        return;
    }
    const Pose delta = st->delta;
    const int n = min(si.w * si.h, pix1);
    const int tid = threadIdx.x;
    // per-thread partial sums in plain FP64 (a thread adds ~4 matches); double-double from the
    // CTA reduction on
    double acc[kSums];
#pragma unroll
    for (int k = 0; k < kSums; ++k) acc[k] = 0.0;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    unsigned long long cnt = 0;
    for (int i = pix0 + blockIdx.x * blockDim.x + tid; i < n; i += gridDim.x * blockDim.x) {
        d3 p, q, nn;
        if (!associate(i, src, src_n, tgt, tgt_n, si, ti, prm, delta, p, q, nn)) continue;
        const d3 pxn = cross(p, nn);
        const double r[6] = {pxn.x, pxn.y, pxn.z, nn.x, nn.y, nn.z};
        const double d = dot(sub(p, q), nn);
        int k = 0;
#pragma unroll
        for (int a = 0; a < 6; ++a)
#pragma unroll
            for (int b = a; b < 6; ++b, ++k) acc[k] += r[a] * r[b];
#pragma unroll
        for (int a = 0; a < 6; ++a) acc[21 + a] += r[a] * d;
        acc[27] += d * d;
        const double pp[3] = {p.x, p.y, p.z}, qq[3] = {q.x, q.y, q.z};
#pragma unroll
        for (int a = 0; a < 3; ++a) {  // shrink's bounding box (registration.cpp:54-59)
            lo[a] = dmin(dmin(lo[a], pp[a]), qq[a]);
            hi[a] = dmax(dmax(hi[a], pp[a]), qq[a]);
        }
        ++cnt;
    }
    // ---- CTA reduction: box and count by shuffles (exact in any order); the 28 sums by a
    // shared-memory transpose in a fixed order (thread order within 32-thread segments).
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            lo[a] = dmin(lo[a], __shfl_down_sync(0xffffffffu, lo[a], off));
            hi[a] = dmax(hi[a], __shfl_down_sync(0xffffffffu, hi[a], off));
        }
        cnt += __shfl_down_sync(0xffffffffu, cnt, off);
    }
    __shared__ double s_b[kStepThreads / 32][6];
    __shared__ unsigned long long s_c[kStepThreads / 32];
    const int lane = tid & 31, wid = tid >> 5;
    if (lane == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            s_b[wid][a] = lo[a];
            s_b[wid][3 + a] = hi[a];
        }
        s_c[wid] = cnt;
    }
#pragma unroll
    for (int k = 0; k < kSums; ++k) s_red[k * kSumStride + (tid >> 5) * kSegStride + (tid & 31)] = acc[k];
    __syncthreads();
    constexpr int kSeg = kStepThreads / 32;  // 8 segments of 32 threads per sum
    __shared__ DD s_seg[kSums][kSeg];
    if (tid < kSums * kSeg) {
        const double* row = s_red + (tid / kSeg) * kSumStride + (tid % kSeg) * kSegStride;
        DD seg{row[0], 0.0};
        for (int t = 1; t < 32; ++t) dd_add(seg, row[t]);
        s_seg[tid / kSeg][tid % kSeg] = seg;
    }
    if (tid == 0) {
        for (int w = 1; w < kStepThreads / 32; ++w) {
            for (int a = 0; a < 3; ++a) {
                s_b[0][a] = dmin(s_b[0][a], s_b[w][a]);
                s_b[0][3 + a] = dmax(s_b[0][3 + a], s_b[w][3 + a]);
            }
            s_c[0] += s_c[w];
        }
        for (int a = 0; a < 6; ++a) part_bbox[blockIdx.x * 6 + a] = s_b[0][a];
        part_count[blockIdx.x] = s_c[0];
    }
    __syncthreads();
    if (tid < kSums) {
        DD a = s_seg[tid][0];
        for (int j = 1; j < kSeg; ++j) dd_merge(a, s_seg[tid][j]);
        part[blockIdx.x * kSums + tid] = a;
    }
    if (!last_cta(counter)) return;
    if (tid == 0) SF_ICP_STAMP(0);

    // ---- last CTA: merge the partials (fixed order) --------------------------------------
    // The box / count partials and the 28 double-double sums are loaded and reduced in one pass
    // (independent loads in flight together), then thread 0 finishes the box while 28 threads
    // finish the sums.
    const int nparts = gridDim.x;
    __shared__ int s_lost;
    constexpr int L = kMergeLanes, kBatch = 17;  // partials in flight per thread (two L2 round trips)
    __shared__ DD s_m[kSums][L];
    __shared__ double s_sum[kSums], s_fin[kSums];
    double b[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    unsigned long long c = 0;
    for (int p = tid; p < nparts; p += blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            b[a] = dmin(b[a], __ldcg(&part_bbox[p * 6 + a]));
            b[3 + a] = dmax(b[3 + a], __ldcg(&part_bbox[p * 6 + 3 + a]));
        }
        c += __ldcg(&part_count[p]);
    }
    if (tid < kSums * L) {
        const int k = tid % kSums, j = tid / kSums;
        const double2* vp = reinterpret_cast<const double2*>(part);
        DD a{0.0, 0.0};
        bool first = true;
        for (int p0 = j; p0 < nparts; p0 += kBatch * L) {
            double2 v[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const int p = p0 + u * L;
                v[u] = p < nparts ? __ldcg(&vp[p * kSums + k]) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                if (p0 + u * L >= nparts) break;
                const DD x{v[u].x, v[u].y};
                if (first) {
                    a = x;
                    first = false;
                } else {
                    dd_merge(a, x);
                }
            }
        }
        s_m[k][j] = a;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            b[a] = dmin(b[a], __shfl_down_sync(0xffffffffu, b[a], off));
            b[3 + a] = dmax(b[3 + a], __shfl_down_sync(0xffffffffu, b[3 + a], off));
        }
        c += __shfl_down_sync(0xffffffffu, c, off);
    }
    __syncthreads();  // s_b / s_c reuse; s_m complete
    if (lane == 0) {
        for (int a = 0; a < 6; ++a) s_b[wid][a] = b[a];
        s_c[wid] = c;
    }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < kStepThreads / 32; ++w) {
            for (int a = 0; a < 3; ++a) {
                s_b[0][a] = dmin(s_b[0][a], s_b[w][a]);
                s_b[0][3 + a] = dmax(s_b[0][3 + a], s_b[w][3 + a]);
            }
            s_c[0] += s_c[w];
        }
        const unsigned long long total = s_c[0];
        if constexpr (PARTIAL) {
            rec->count = static_cast<double>(total);
            for (int a = 0; a < 3; ++a) {
                rec->box[a] = s_b[0][a];
                rec->box[3 + a] = -s_b[0][3 + a];  // max as a min of the negation: one MIN all-reduce
            }
        } else {
            if (st->bodies == 0) st->t_assoc0 = globaltimer_ns();
            st->bodies += 1;
            s_lost = total < 10 ? 1 : 0;
            if (total < 10) {  // TrackingLost (registration.cpp:202-204)
                st->lost = 1;
                st->lost_count = total;
                st->done = 1;
            } else {
                st->matches = total;
                st->cur_count = total;
                // shrink centre / scale (registration.cpp:54-64)
                const d3 l = mk(s_b[0][0], s_b[0][1], s_b[0][2]), hh = mk(s_b[0][3], s_b[0][4], s_b[0][5]);
                const d3 cc = scale(0.5, add(l, hh));
                const d3 ext = sub(hh, l);
                const d3 sc = mk(dmax(ext.x, prm.floor), dmax(ext.y, prm.floor), dmax(ext.z, prm.floor));
                st->center = cc;
                st->scale = sc;
                st->inv_scale = mk(1.0 / sc.x, 1.0 / sc.y, 1.0 / sc.z);
            }
        }
    }
    if (tid >= 32 && tid < 32 + kSums) {  // a warp other than thread 0's: overlaps the box work
        const int k = tid - 32;
        DD a = s_m[k][0];
        for (int j = 1; j < L; ++j) dd_merge(a, s_m[k][j]);
        if constexpr (PARTIAL) {
            rec->sums[2 * k] = a.hi;
            rec->sums[2 * k + 1] = a.lo;
        } else {
            s_sum[k] = a.hi + a.lo;
        }
    }
    __syncthreads();
    if constexpr (PARTIAL) {
        if (tid == 0) *counter = 0;
        return;
    } else {
        if (s_lost) {
            if (tid == 0) {
                *counter = 0;
                if constexpr (COND) cudaGraphSetConditional(cond, 0u);
            }
            return;
        }
    }
    if (tid == 0) SF_ICP_STAMP(1);
    if (tid >= 32) return;
    solve_from_sums<COND>(st, s_sum, s_fin, prm, counter, cond);
}

// Sharded ICP: merge the ranks' records (local ranks in rank order; after an NCCL all-reduce
// a single record holding the sums), then the same TrackingLost test, shrink and solve as
// k_icp_step's last CTA. One warp.
template <bool COND>
__global__ void __launch_bounds__(32, 1)
    k_icp_solve_ranks(IcpState* st, const IcpRankPartial* __restrict__ recs, int nrec, IcpParamsDev prm,
                      unsigned int* counter, cudaGraphConditionalHandle cond) {
    const int lane = threadIdx.x;
    if (st->done) {
        if constexpr (COND) {
            if (lane == 0) cudaGraphSetConditional(cond, 0u);
        }
        return;
    }
    __shared__ double s_sum[kSums], s_fin[kSums];
    __shared__ int s_lost;
    if (lane < kSums) {
        DD a{recs[0].sums[2 * lane], recs[0].sums[2 * lane + 1]};
        for (int r = 1; r < nrec; ++r) dd_merge(a, DD{recs[r].sums[2 * lane], recs[r].sums[2 * lane + 1]});
        s_sum[lane] = a.hi + a.lo;
    }
    if (lane == 0) {
        double b[6];
        double cnt = 0.0;
        for (int a = 0; a < 6; ++a) b[a] = INFINITY;
        for (int r = 0; r < nrec; ++r) {
            for (int a = 0; a < 6; ++a) b[a] = dmin(b[a], recs[r].box[a]);
            cnt += recs[r].count;
        }
        const unsigned long long total = static_cast<unsigned long long>(cnt);
        if (st->bodies == 0) st->t_assoc0 = globaltimer_ns();
        st->bodies += 1;
        s_lost = total < 10 ? 1 : 0;
        if (total < 10) {  // TrackingLost (registration.cpp:202-204)
            st->lost = 1;
            st->lost_count = total;
            st->done = 1;
        } else {
            st->matches = total;
            st->cur_count = total;
            const d3 l = mk(b[0], b[1], b[2]), hh = mk(-b[3], -b[4], -b[5]);
            const d3 ext = sub(hh, l);
            const d3 sc = mk(dmax(ext.x, prm.floor), dmax(ext.y, prm.floor), dmax(ext.z, prm.floor));
            st->center = scale(0.5, add(l, hh));  // registration.cpp:60-63
            st->scale = sc;
            st->inv_scale = mk(1.0 / sc.x, 1.0 / sc.y, 1.0 / sc.z);
        }
    }
    __syncwarp();
    if (s_lost) {
        if constexpr (COND) {
            if (lane == 0) cudaGraphSetConditional(cond, 0u);
        }
        return;
    }
    solve_from_sums<COND>(st, s_sum, s_fin, prm, counter, cond);
}

// ---------------------------------------------------------------------------------
// Reference-order reduction (sf_match_params.reduction == 1): bit-identical to the
// reference's icp(). Per iteration three launches:
//   k_icp_exact_match  association (the same `associate`), matches compacted in row-major
//                      order: CTA b owns the contiguous pixel range [b * chunk, (b+1) * chunk)
//                      and appends its matches in pixel order (ballot + CTA prefix); the
//                      shrink's bounding box (min / max: exact in any order) and the counts;
//                      the last CTA forms centre / scale (registration.cpp:52-64) or raises
//                      TrackingLost (registration.cpp:202-204)
//   k_icp_exact_terms  per match, the shrunk match and the 28 addends of assemble in the
//                      reference's arithmetic (registration.cpp:65-70, 104-113), stored in
//                      global match order
//   k_icp_exact_solve  one warp: lane k runs the reference's Kahan accumulator k over the
//                      addends in match order (registration.cpp:79-89, 107-113) — the same
//                      sequence of floating-point operations, so the same sums — then the
//                      cyclic Jacobi (eigendecompose_sym6_warp, same rotation order), the
//                      spectral gated solve, unshrink and apply_motion with the SVD polar
//                      factor (registration.cpp:125-212, pose.cpp:20-43).
// The Kahan chains are sequential (4 dependent FP64 adds per match and sum), so an iteration
// costs ~matches x the FP64 add latency; the tree path (default) is the fast one.
// ---------------------------------------------------------------------------------
constexpr int kExactCtas = kIcpCtas;

__host__ __device__ inline int exact_chunk(int n) {  // pixels per CTA range (multiple of 32)
    return ((n + kExactCtas - 1) / kExactCtas + 31) & ~31;
}

template <bool COND>
__global__ void __launch_bounds__(kIcpThreads, 1)
    k_icp_exact_match(const float* __restrict__ src, const float* __restrict__ src_n, const float* __restrict__ tgt,
                      const float* __restrict__ tgt_n, Intr si, Intr ti, IcpParamsDev prm, IcpState* st,
                      MatchRec* __restrict__ rec, double* __restrict__ part_bbox,
                      unsigned long long* __restrict__ part_count, unsigned int* counter,
                      cudaGraphConditionalHandle cond) {
    if (threadIdx.x == 0 && st->bodies == 0) atomicCAS(&st->t_step0, 0ull, globaltimer_ns());
    if (st->done) {
        if constexpr (COND) {
            if (blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0u);
        }
        return;
    }
    const Pose delta = st->delta;
    const int n = si.w * si.h;
    const int chunk = exact_chunk(n);
    const int begin = blockIdx.x * chunk, end = min(n, begin + chunk);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int kWarps = kIcpThreads / 32;
    __shared__ unsigned int s_wcnt[kWarps];
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    unsigned int base = 0;  // matches this CTA appended so far
    for (int r0 = begin; r0 < end; r0 += kIcpThreads) {
        const int i = r0 + tid;
        d3 p, q, nn;
        const bool ok = i < end && associate(i, src, src_n, tgt, tgt_n, si, ti, prm, delta, p, q, nn);
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        if (lane == 0) s_wcnt[wid] = __popc(bal);
        __syncthreads();
        unsigned int off = base, tot = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const unsigned int c = s_wcnt[w];
            off += w < wid ? c : 0u;
            tot += c;
        }
        if (ok) {
            MatchRec m;
            m.p[0] = p.x, m.p[1] = p.y, m.p[2] = p.z;
            m.q[0] = q.x, m.q[1] = q.y, m.q[2] = q.z;
            m.n[0] = nn.x, m.n[1] = nn.y, m.n[2] = nn.z;
            rec[begin + off + __popc(bal & ((1u << lane) - 1u))] = m;
            const double pp[3] = {p.x, p.y, p.z}, qq[3] = {q.x, q.y, q.z};
#pragma unroll
            for (int a = 0; a < 3; ++a) {  // shrink's bounding box (registration.cpp:54-59)
                lo[a] = dmin(dmin(lo[a], pp[a]), qq[a]);
                hi[a] = dmax(dmax(hi[a], pp[a]), qq[a]);
            }
        }
        base += tot;
        __syncthreads();  // s_wcnt reuse
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            lo[a] = dmin(lo[a], __shfl_down_sync(0xffffffffu, lo[a], off));
            hi[a] = dmax(hi[a], __shfl_down_sync(0xffffffffu, hi[a], off));
        }
    __shared__ double s_b[kWarps][6];
    if (lane == 0)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            s_b[wid][a] = lo[a];
            s_b[wid][3 + a] = hi[a];
        }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < kWarps; ++w)
            for (int a = 0; a < 3; ++a) {
                s_b[0][a] = dmin(s_b[0][a], s_b[w][a]);
                s_b[0][3 + a] = dmax(s_b[0][3 + a], s_b[w][3 + a]);
            }
        for (int a = 0; a < 6; ++a) part_bbox[blockIdx.x * 6 + a] = s_b[0][a];
        part_count[blockIdx.x] = base;
    }
    if (!last_cta(counter)) return;
    if (tid == 0) {
        double b[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
        unsigned long long total = 0;
        for (int c = 0; c < static_cast<int>(gridDim.x); ++c) {
            for (int a = 0; a < 3; ++a) {
                b[a] = dmin(b[a], __ldcg(&part_bbox[c * 6 + a]));
                b[3 + a] = dmax(b[3 + a], __ldcg(&part_bbox[c * 6 + 3 + a]));
            }
            total += __ldcg(&part_count[c]);
        }
        if (st->bodies == 0) st->t_assoc0 = globaltimer_ns();
        st->bodies += 1;
        if (total < 10) {  // TrackingLost (registration.cpp:202-204)
            st->lost = 1;
            st->lost_count = total;
            st->done = 1;
            if constexpr (COND) cudaGraphSetConditional(cond, 0u);
        } else {
            st->matches = total;
            st->cur_count = total;
            // shrink centre / scale (registration.cpp:60-63)
            const d3 l = mk(b[0], b[1], b[2]), hh = mk(b[3], b[4], b[5]);
            const d3 ext = sub(hh, l);
            const d3 sc = mk(dmax(ext.x, prm.floor), dmax(ext.y, prm.floor), dmax(ext.z, prm.floor));
            st->center = scale(0.5, add(l, hh));
            st->scale = sc;
            st->inv_scale = mk(1.0 / sc.x, 1.0 / sc.y, 1.0 / sc.z);
        }
        *counter = 0;
    }
}

// The 28 addends of assemble for every match, in global match order (CTA ranges in order).
__global__ void __launch_bounds__(kIcpThreads)
    k_icp_exact_terms(const IcpState* __restrict__ st, const MatchRec* __restrict__ rec,
                      const unsigned long long* __restrict__ part_count, int n, double* __restrict__ terms) {
    if (st->done) return;
    const int b = blockIdx.x;
    const unsigned long long cnt = part_count[b];
    __shared__ unsigned long long s_off;
    if (threadIdx.x < 32) {  // matches of the ranges before this one
        unsigned long long o = 0;
        for (int c = threadIdx.x; c < b; c += 32) o += part_count[c];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) o += __shfl_down_sync(0xffffffffu, o, off);
        if (threadIdx.x == 0) s_off = o;
    }
    __syncthreads();
    const d3 c = st->center, s = st->scale, inv = st->inv_scale;
    const MatchRec* r = rec + static_cast<size_t>(b) * exact_chunk(n);
    double* out = terms + s_off * kSums;
    for (unsigned long long j = threadIdx.x; j < cnt; j += blockDim.x) {
        const MatchRec m = r[j];
        const d3 p = mk(m.p[0], m.p[1], m.p[2]), q = mk(m.q[0], m.q[1], m.q[2]), nn = mk(m.n[0], m.n[1], m.n[2]);
        // ShrunkMatch (registration.cpp:65-69)
        const d3 ph = cmul(inv, sub(p, c)), qh = cmul(inv, sub(q, c));
        const d3 ch = cmul(inv, sub(cross(p, nn), cross(c, nn)));
        // assemble's row and residual (registration.cpp:104-106)
        const double row[6] = {ch.x, ch.y, ch.z, nn.x, nn.y, nn.z};
        const double d = dot(cmul(s, sub(ph, qh)), nn);
        double* t = out + j * kSums;
        int k = 0;
#pragma unroll
        for (int a = 0; a < 6; ++a)
#pragma unroll
            for (int bb = a; bb < 6; ++bb, ++k) t[k] = row[a] * row[bb];
#pragma unroll
        for (int a = 0; a < 6; ++a) t[21 + a] = -row[a] * d;
        t[27] = d * d;
    }
}

// The reference's Compensated::add (registration.cpp:79-89).
__device__ __forceinline__ void kahan_add(double& sum, double& carry, double value) {
    const double y = value - carry;
    const double t = sum + y;
    carry = (t - sum) - y;
    sum = t;
}

template <bool COND>
__global__ void __launch_bounds__(32, 1)
    k_icp_exact_solve(IcpState* st, const double* __restrict__ terms, IcpParamsDev prm,
                      cudaGraphConditionalHandle cond) {
    const int lane = threadIdx.x;
    if (st->done) {  // lost in this iteration's match (or earlier)
        if constexpr (COND) {
            if (lane == 0) cudaGraphSetConditional(cond, 0u);
        }
        return;
    }
    const unsigned long long total = st->cur_count;
    double sum = 0.0, carry = 0.0;
    // The addends stream through shared memory in a cp.async pipeline (kStages batches of kB
    // matches in flight), so the loop runs at the latency of the dependent Kahan chain.
    constexpr int kB = 32, kStages = 4;
    constexpr int kStageBytes = kB * kSums * 8;  // 7168 B, a multiple of 16
    __shared__ __align__(16) double s_t[kStages][kB * kSums];
    const unsigned long long nbatch = (total + kB - 1) / kB;
    auto issue = [&](unsigned long long b) {
        if (b < nbatch) {
            const unsigned long long m0 = b * kB;
            const int bytes = static_cast<int>(total - m0 < kB ? total - m0 : kB) * kSums * 8;
            const char* g = reinterpret_cast<const char*>(terms + m0 * kSums);
            const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(s_t[b % kStages]));
            for (int off = lane * 16; off < bytes; off += 32 * 16)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sbase + off), "l"(g + off) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    static_assert(kStageBytes % 16 == 0, "stage size");
#pragma unroll
    for (int b = 0; b < kStages - 1; ++b) issue(b);
    for (unsigned long long b = 0; b < nbatch; ++b) {
        asm volatile("cp.async.wait_group %0;" ::"n"(kStages - 2) : "memory");
        __syncwarp();
        const double* x = s_t[b % kStages];
        const int nm = static_cast<int>(total - b * kB < kB ? total - b * kB : kB);
        if (lane < kSums) {
            if (nm == kB) {
#pragma unroll
                for (int j = 0; j < kB; ++j) kahan_add(sum, carry, x[j * kSums + lane]);
            } else {
                for (int j = 0; j < nm; ++j) kahan_add(sum, carry, x[j * kSums + lane]);
            }
        }
        __syncwarp();  // stage b % kStages is free again
        issue(b + kStages - 1);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __shared__ double s_sum[kSums];
    __shared__ double s_A[36];
    __shared__ Eig6 s_eig;
    if (lane < kSums) s_sum[lane] = sum;
    __syncwarp();
    for (int i = lane; i < 36; i += 32) {  // eq.A from the upper-triangle sums (registration.cpp:115-120)
        const int r = i / 6, cc = i % 6;
        s_A[i] = s_sum[r <= cc ? packed_index(r, cc) : packed_index(cc, r)];
    }
    __syncwarp();
    eigendecompose_sym6_warp(s_A, &s_eig);
    __syncwarp();
    if (lane == 0) {
        solve_finalize(st, s_sum, s_eig, prm, true);
        st->t_end = globaltimer_ns();
        if constexpr (COND)
            cudaGraphSetConditional(cond, (!st->done && st->iterations < prm.max_iterations) ? 1u : 0u);
    }
}

// One reference-order iteration: the three launches (eager, or inside a capture).
template <bool COND>
static void issue_exact_iteration(IcpWork& wk, const float* src, const float* src_n, const float* tgt,
                                  const float* tgt_n, const Intr& si, const Intr& ti, const IcpParamsDev& prm,
                                  cudaStream_t s, cudaGraphConditionalHandle cond) {
    const int n = si.w * si.h;
    k_icp_exact_match<COND><<<kExactCtas, kIcpThreads, 0, s>>>(src, src_n, tgt, tgt_n, si, ti, prm, wk.st, wk.rec,
                                                                wk.part_bbox, wk.part_count, wk.counters + 1, cond);
    SF_LAUNCH_CHECK();
    k_icp_exact_terms<<<kExactCtas, kIcpThreads, 0, s>>>(wk.st, wk.rec, wk.part_count, n, wk.terms);
    SF_LAUNCH_CHECK();
    k_icp_exact_solve<COND><<<1, 32, 0, s>>>(wk.st, wk.terms, prm, cond);
    SF_LAUNCH_CHECK();
}

IcpParamsDev make_icp_params(const sf_match_params& p) {
    IcpParamsDev d;
    d.cos_max = std::cos(p.max_normal_angle);          // registration.cpp:25
    d.max_dist_sq = p.max_distance * p.max_distance;   // registration.cpp:26
    d.eps = p.convergence_epsilon;
    d.theta = p.eigen_threshold;
    d.floor = p.shrink_floor;
    d.max_iterations = p.max_iterations;
    d.exact = p.reduction == 1 ? 1 : 0;
    return d;
}

// Launch the whole ICP: init + the iterations (match, assemble).
// Under stream capture the iterations become a conditional WHILE node of the graph being
// captured: the body {match, assemble} repeats while the assemble's last CTA keeps the
// condition set (not converged, not lost, fewer than max_iterations), so a frame launches
// 1 + 2 x iterations kernels. Issued eagerly, it is the fixed sequence of max_iterations
// (match, assemble) pairs whose kernels exit at once after convergence.
// *device_loop (optional) reports which form was used; the loop form adds only the init
// launch to *launches (the caller adds 2 x IcpState::bodies after the fact).
void launch_icp(IcpWork& wk, const float* src, const float* src_n, const float* tgt, const float* tgt_n,
                const Intr& si, const Intr& ti, const double* d_initial, const IcpParamsDev& prm, cudaStream_t s,
                uint64_t* launches, const int* dead, bool* device_loop, bool state_ready) {
    SF_CUDA(cudaFuncSetAttribute(k_icp_step<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStepSmem));
    SF_CUDA(cudaFuncSetAttribute(k_icp_step<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStepSmem));
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    SF_CUDA(cudaStreamIsCapturing(s, &cs));
    // SF_ICP_DEVICE_LOOP=0 keeps the fixed launch sequence under capture too (Nsight Compute
    // does not profile kernels inside conditional graph nodes).
    static const bool loop_enabled = [] {
        const char* e = std::getenv("SF_ICP_DEVICE_LOOP");
        return !(e && e[0] == '0');
    }();
    const bool loop = loop_enabled && cs == cudaStreamCaptureStatusActive && prm.max_iterations > 0;
    if (device_loop) *device_loop = loop;
    if (prm.exact) wk.ensure_exact();
    if (!loop) {
        uint64_t cnt = 0;
        if (!state_ready) {
            k_icp_init<false><<<1, 1, 0, s>>>(wk.st, d_initial, dead, prm.max_iterations, 0);
            SF_LAUNCH_CHECK();
            cnt = 1;
        }
        for (int it = 0; it < prm.max_iterations; ++it) {
            if (prm.exact) {
                issue_exact_iteration<false>(wk, src, src_n, tgt, tgt_n, si, ti, prm, s, 0);
                cnt += 3;
                continue;
            }
            k_icp_step<false><<<kStepCtas, kStepThreads, kStepSmem, s>>>(src, src_n, tgt, tgt_n, si, ti, prm, wk.st,
                                                                        wk.part_bbox, wk.part_count, wk.part,
                                                                        wk.counters, 0);
            SF_LAUNCH_CHECK();
            cnt += 1;
        }
        if (launches) *launches += cnt;
        return;
    }
    cudaGraph_t g = nullptr;
    SF_CUDA(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, nullptr, nullptr));
    cudaGraphConditionalHandle cond;
    SF_CUDA(cudaGraphConditionalHandleCreate(&cond, g, 0, 0));
    if (state_ready) {
        // first iteration as a plain node: it sets the condition for the loop of the others
        // (the loop-entry latency of the conditional node is paid only by multi-iteration frames)
        if (prm.exact)
            issue_exact_iteration<true>(wk, src, src_n, tgt, tgt_n, si, ti, prm, s, cond);
        else
            k_icp_step<true><<<kStepCtas, kStepThreads, kStepSmem, s>>>(src, src_n, tgt, tgt_n, si, ti, prm, wk.st,
                                                                       wk.part_bbox, wk.part_count, wk.part,
                                                                       wk.counters, cond);
    } else {
        k_icp_init<true><<<1, 1, 0, s>>>(wk.st, d_initial, dead, prm.max_iterations, cond);
        if (launches) *launches += 1;
    }
    SF_LAUNCH_CHECK();
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    SF_CUDA(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &ndeps));
    cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    SF_CUDA(cudaGraphAddNode(&node, g, deps, ndeps, &cp));
    SF_CUDA(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    if (!wk.body_stream) SF_CUDA(cudaStreamCreateWithFlags(&wk.body_stream, cudaStreamNonBlocking));
    cudaStream_t bs = wk.body_stream;
    SF_CUDA(cudaStreamBeginCaptureToGraph(bs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    if (prm.exact) {
        try {
            issue_exact_iteration<true>(wk, src, src_n, tgt, tgt_n, si, ti, prm, bs, cond);
        } catch (...) {
            cudaGraph_t g2 = nullptr;
            cudaStreamEndCapture(bs, &g2);
            throw;
        }
    } else {
        k_icp_step<true><<<kStepCtas, kStepThreads, kStepSmem, bs>>>(src, src_n, tgt, tgt_n, si, ti, prm, wk.st,
                                                                    wk.part_bbox, wk.part_count, wk.part,
                                                                    wk.counters, cond);
    }
    const cudaError_t le = cudaGetLastError();
    cudaGraph_t captured = nullptr;
    const cudaError_t ee = cudaStreamEndCapture(bs, &captured);
    SF_CUDA(le);
    SF_CUDA(ee);
}

// Sharded ICP (north star: "ICP partial sums combined with a 27-float allreduce"): per
// iteration every local rank's PARTIAL pass over its slice of the source pixels, the reduction
// of the ranks' records (`reduce`: nothing for in-process ranks, whose records the solve merges
// in rank order; NCCL all-reduces for one rank per process), then k_icp_solve_ranks, identical
// on every rank. Under capture with allow_loop the iterations are a conditional WHILE node as
// in launch_icp; otherwise max_iterations bodies are issued and converged ones exit at once.
void launch_icp_ranks(IcpWork& wk, const float* src, const float* src_n, const float* tgt, const float* tgt_n,
                      const Intr& I, const double* d_initial, const IcpParamsDev& prm, int rank0, int nlocal,
                      int world, IcpRankPartial* recs, int nrec, const std::function<void(cudaStream_t)>& reduce,
                      bool allow_loop, cudaStream_t s, uint64_t* launches, const int* dead, bool* device_loop) {
    SF_CUDA(cudaFuncSetAttribute(k_icp_step<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStepSmem));
    SF_CUDA(cudaFuncSetAttribute(k_icp_step<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStepSmem));
    const int n = I.w * I.h;
    auto body = [&](cudaStream_t bs, bool cond_on, cudaGraphConditionalHandle cond) {
        for (int i = 0; i < nlocal; ++i) {
            const int r = rank0 + i;
            const int p0 = static_cast<int>(static_cast<long long>(n) * r / world);
            const int p1 = static_cast<int>(static_cast<long long>(n) * (r + 1) / world);
            if (cond_on)
                k_icp_step<true, true><<<kStepCtas, kStepThreads, kStepSmem, bs>>>(
                    src, src_n, tgt, tgt_n, I, I, prm, wk.st, wk.part_bbox, wk.part_count, wk.part, wk.counters + 2,
                    cond, p0, p1, recs + i);
            else
                k_icp_step<false, true><<<kStepCtas, kStepThreads, kStepSmem, bs>>>(
                    src, src_n, tgt, tgt_n, I, I, prm, wk.st, wk.part_bbox, wk.part_count, wk.part, wk.counters + 2,
                    0, p0, p1, recs + i);
            SF_LAUNCH_CHECK();
        }
        reduce(bs);
        if (cond_on) k_icp_solve_ranks<true><<<1, 32, 0, bs>>>(wk.st, recs, nrec, prm, wk.counters + 3, cond);
        else k_icp_solve_ranks<false><<<1, 32, 0, bs>>>(wk.st, recs, nrec, prm, wk.counters + 3, 0);
        SF_LAUNCH_CHECK();
    };
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    SF_CUDA(cudaStreamIsCapturing(s, &cs));
    const bool loop = allow_loop && cs == cudaStreamCaptureStatusActive && prm.max_iterations > 0;
    if (device_loop) *device_loop = loop;
    if (!loop) {
        k_icp_init<false><<<1, 1, 0, s>>>(wk.st, d_initial, dead, prm.max_iterations, 0);
        SF_LAUNCH_CHECK();
        for (int it = 0; it < prm.max_iterations; ++it) body(s, false, 0);
        if (launches) *launches += 1 + static_cast<uint64_t>(prm.max_iterations) * (nlocal + 1);
        return;
    }
    cudaGraph_t g = nullptr;
    SF_CUDA(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, nullptr, nullptr));
    cudaGraphConditionalHandle cond;
    SF_CUDA(cudaGraphConditionalHandleCreate(&cond, g, 0, 0));
    k_icp_init<true><<<1, 1, 0, s>>>(wk.st, d_initial, dead, prm.max_iterations, cond);
    SF_LAUNCH_CHECK();
    if (launches) *launches += 1;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    SF_CUDA(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &ndeps));
    cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    SF_CUDA(cudaGraphAddNode(&node, g, deps, ndeps, &cp));
    SF_CUDA(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
    if (!wk.body_stream) SF_CUDA(cudaStreamCreateWithFlags(&wk.body_stream, cudaStreamNonBlocking));
    cudaStream_t bs = wk.body_stream;
    SF_CUDA(cudaStreamBeginCaptureToGraph(bs, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal));
    try {
        body(bs, true, cond);
    } catch (...) {
        cudaGraph_t g2 = nullptr;
        cudaStreamEndCapture(bs, &g2);
        throw;
    }
    cudaGraph_t captured = nullptr;
    SF_CUDA(cudaStreamEndCapture(bs, &captured));
}

void launch_icp_report(IcpWork& wk, cudaStream_t s, uint64_t* launches) {
    k_icp_report<<<1, 32, 0, s>>>(wk.st);
    SF_LAUNCH_CHECK();
    if (launches) *launches += 1;
}

void fill_icp_result(const IcpState& st, sf_icp_result* out) {
    memset(out, 0, sizeof(*out));
    pose_to12(st.delta, out->delta);
    out->iterations = st.iterations;
    out->matches = st.matches;
    out->motion_r[0] = st.motion_r.x;
    out->motion_r[1] = st.motion_r.y;
    out->motion_r[2] = st.motion_r.z;
    out->motion_t[0] = st.motion_t.x;
    out->motion_t[1] = st.motion_t.y;
    out->motion_t[2] = st.motion_t.z;
    for (int i = 0; i < 6; ++i) {
        out->eigenvalues[i] = st.eigenvalues[i];
        out->gated_mask[i] = st.gated[i];
    }
    for (int i = 0; i < 36; ++i) out->eigenvectors[i] = st.eigenvectors[i];
    out->residual_rms = st.residual_rms;
    out->shrunk_motion_norm = st.shrunk_norm;
    out->pair_count = st.pair_count;
}

}  // namespace sf

using namespace sf;

extern "C" int sf_icp(const sf_frame* source, const float* source_normals, const sf_frame* target,
                      const float* target_normals, const double initial[12], const sf_match_params* params,
                      sf_icp_result* result, void* stream) {
    return guarded([&]() -> int {
        if (!source || !target || !target_normals || !initial || !params || !result)
            throw Error(SF_INVALID_ARGUMENT, "sf_icp: null argument");
        const sf_intrinsics& si = source->intrinsics;
        const sf_intrinsics& ti = target->intrinsics;
        if (si.width != ti.width || si.height != ti.height)
            throw Error(SF_INVALID_ARGUMENT, "match: frames must share intrinsics");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        static thread_local IcpWork wk;
        wk.ensure(si.width, si.height);
        const size_t n = static_cast<size_t>(si.width) * si.height;
        const float *d_src = source->depth, *d_tgt = target->depth, *d_tn = target_normals,
                    *d_sn = source_normals;
        if (!source->on_device) {
            SF_CUDA(cudaMemcpyAsync(wk.src, source->depth, n * sizeof(float), cudaMemcpyHostToDevice, s));
            d_src = wk.src;
            if (source_normals) {
                SF_CUDA(cudaMemcpyAsync(wk.src_n_in, source_normals, 3 * n * sizeof(float), cudaMemcpyHostToDevice, s));
                d_sn = wk.src_n_in;
            }
        }
        if (!target->on_device) {
            SF_CUDA(cudaMemcpyAsync(wk.tgt, target->depth, n * sizeof(float), cudaMemcpyHostToDevice, s));
            SF_CUDA(cudaMemcpyAsync(wk.tgt_n, target_normals, 3 * n * sizeof(float), cudaMemcpyHostToDevice, s));
            d_tgt = wk.tgt;
            d_tn = wk.tgt_n;
        }
        const Intr SI = to_intr(si), TI = to_intr(ti);
        if (!d_sn) {  // compute_normals(source, params.normal_options) (registration.cpp:218)
            launch_compute_normals(d_src, si.width, si.height, SI, params->normal_sigma0, params->normal_spatial_scale,
                                   wk.src_normals, s, nullptr, nullptr);
            d_sn = wk.src_normals;
        }
        SF_CUDA(cudaMemcpyAsync(wk.initial, initial, 12 * sizeof(double), cudaMemcpyHostToDevice, s));
        const IcpParamsDev prm = make_icp_params(*params);
        launch_icp(wk, d_src, d_sn, d_tgt, d_tn, SI, TI, wk.initial, prm, s, nullptr, nullptr);
        launch_icp_report(wk, s, nullptr);
        IcpState hs;
        SF_CUDA(cudaMemcpyAsync(&hs, wk.st, sizeof(hs), cudaMemcpyDeviceToHost, s));
        SF_CUDA(cudaStreamSynchronize(s));
        if (hs.lost)
            throw Error(SF_TRACKING_LOST, "icp: only " + std::to_string(hs.lost_count) + " correspondences");
        fill_icp_result(hs, result);
        if (prm.max_iterations <= 0) pose_to12(pose_from12(initial), result->delta);
        return SF_OK;
    });
}

// sf_icp.cu — projective point-to-plane ICP on the device (registration.cpp:17-224).
//
// Every iteration is two launches with device-side control (no host round trip):
//   k_icp_match     per source pixel: projective association + distance / normal
//                   rejection (registration.cpp:17-50); match record to HBM/L2; per-CTA
//                   bbox (min/max of p and q) and count. The last CTA to finish merges the
//                   partials -> shrink centre / scale (registration.cpp:52-74), or
//                   TrackingLost below 10 matches (registration.cpp:202-204).
//   k_icp_assemble  per match: shrunk row (c_hat, n), d; 21 + 6 + 1 compensated sums
//                   (double-double TwoSum accumulators), warp shuffle -> CTA partials
//                   (registration.cpp:76-123). The last CTA merges the partials in a fixed
//                   order; one warp runs the Jacobi 6x6 (rows across lanes, bit-identical to
//                   the sequential sweep), one thread the gated solve, unshrink, apply_motion
//                   and the convergence test (registration.cpp:125-220).
// Under CUDA-graph capture (tracker) the iterations are a conditional WHILE node: the body
// repeats until converged / lost / max_iterations, decided on the device. Issued eagerly,
// a converged / failed state makes the remaining iterations' kernels exit at once.
// Partials are merged in a fixed order, so results are deterministic run to run.
//
// Parity: the association and every per-match quantity are FP64 in the reference order.
// The only deviation is the summation order of the 28 sums (tree instead of sequential
// Kahan); both are within ~1 ulp of the exact sum, pose parity is asserted at 1e-6.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "sf_icp.cuh"
#include "sf_linalg.cuh"

namespace sf {

__global__ void k_icp_init(IcpState* st, const double* __restrict__ initial12, const int* dead, int max_iterations,
                           int use_cond, cudaGraphConditionalHandle cond) {
    IcpState z;
    memset(&z, 0, sizeof(z));
    z.delta = pose_from12(initial12);
    z.done = (dead && *dead) ? 1 : 0;
    *st = z;
    if (use_cond) cudaGraphSetConditional(cond, (!z.done && max_iterations > 0) ? 1u : 0u);
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

// shrink's centre / scale (registration.cpp:54-64) from the bbox partials (min/max and
// integer counts are exact in any order).
__device__ void bbox_finalize(IcpState* st, const double* __restrict__ part_bbox,
                              const unsigned long long* __restrict__ part_count, int nparts, const IcpParamsDev& prm) {
    double b[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    unsigned long long cnt = 0;
    for (int p = threadIdx.x; p < nparts; p += blockDim.x) {
        const volatile double* pb = part_bbox + p * 6;
        for (int a = 0; a < 3; ++a) {
            b[a] = dmin(b[a], pb[a]);
            b[3 + a] = dmax(b[3 + a], pb[3 + a]);
        }
        cnt += ((const volatile unsigned long long*)part_count)[p];
    }
    for (int off = 16; off > 0; off >>= 1) {
        for (int a = 0; a < 3; ++a) {
            b[a] = dmin(b[a], __shfl_down_sync(0xffffffffu, b[a], off));
            b[3 + a] = dmax(b[3 + a], __shfl_down_sync(0xffffffffu, b[3 + a], off));
        }
        cnt += __shfl_down_sync(0xffffffffu, cnt, off);
    }
    __shared__ double s_b[kIcpThreads / 32][6];
    __shared__ unsigned long long s_c[kIcpThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        for (int a = 0; a < 6; ++a) s_b[wid][a] = b[a];
        s_c[wid] = cnt;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int k = 1; k < (int)(blockDim.x / 32); ++k) {
        for (int a = 0; a < 3; ++a) {
            s_b[0][a] = dmin(s_b[0][a], s_b[k][a]);
            s_b[0][3 + a] = dmax(s_b[0][3 + a], s_b[k][3 + a]);
        }
        s_c[0] += s_c[k];
    }
    cnt = s_c[0];
    if (cnt < 10) {
        st->lost = 1;
        st->lost_count = cnt;
        st->done = 1;
        return;
    }
    st->matches = cnt;
    st->cur_count = cnt;
    const d3 l = mk(s_b[0][0], s_b[0][1], s_b[0][2]), hh = mk(s_b[0][3], s_b[0][4], s_b[0][5]);
    const d3 c = scale(0.5, add(l, hh));
    const d3 ext = sub(hh, l);
    const d3 s = mk(dmax(ext.x, prm.floor), dmax(ext.y, prm.floor), dmax(ext.z, prm.floor));  // cwiseMax(floor)
    st->center = c;
    st->scale = s;
    st->inv_scale = mk(1.0 / s.x, 1.0 / s.y, 1.0 / s.z);
}

// match_points (registration.cpp:17-50) + bbox partials of shrink (registration.cpp:54-59)
__global__ void __launch_bounds__(kIcpThreads)
    k_icp_match(const float* __restrict__ src, const float* __restrict__ src_n, const float* __restrict__ tgt,
                const float* __restrict__ tgt_n, Intr si, Intr ti, IcpParamsDev prm, IcpState* st,
                MatchRec* __restrict__ rec, uint8_t* __restrict__ flag, double* __restrict__ part_bbox,
                unsigned long long* __restrict__ part_count, unsigned int* counter) {
    if (st->done) return;
    const Pose delta = st->delta;
    const int w = si.w, h = si.h;
    const int n = w * h;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    unsigned long long cnt = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int u = i % w, v = i / w;
        uint8_t ok = 0;
        const float sd = src[i];
        const float snx = src_n[3 * i], sny = src_n[3 * i + 1], snz = src_n[3 * i + 2];
        if (sd > 0.0f && (snx * snx + sny * sny) + snz * snz > 0.0f) {
            const d3 p = apply(delta, unproject(si, u, v, sd));
            double pu, pv;
            if (project(ti, p, pu, pv)) {
                const int tu = ref_lround_int(pu), tv = ref_lround_int(pv);
                if (tu >= 0 && tv >= 0 && tu < ti.w && tv < ti.h) {
                    const int j = tv * ti.w + tu;
                    const float td = tgt[j];
                    const float tnx = tgt_n[3 * j], tny = tgt_n[3 * j + 1], tnz = tgt_n[3 * j + 2];
                    if (td > 0.0f && (tnx * tnx + tny * tny) + tnz * tnz > 0.0f) {
                        const d3 q = unproject(ti, tu, tv, td);
                        if (!(sqnorm(sub(p, q)) > prm.max_dist_sq)) {
                            const d3 nn = mk(tnx, tny, tnz);
                            const d3 ns = mv(delta.R, mk(snx, sny, snz));
                            if (!(dot(ns, nn) < prm.cos_max)) {
                                ok = 1;
                                MatchRec r;
                                r.p[0] = p.x;
                                r.p[1] = p.y;
                                r.p[2] = p.z;
                                r.q[0] = q.x;
                                r.q[1] = q.y;
                                r.q[2] = q.z;
                                r.n[0] = nn.x;
                                r.n[1] = nn.y;
                                r.n[2] = nn.z;
                                rec[i] = r;
                                const double pp[3] = {p.x, p.y, p.z}, qq[3] = {q.x, q.y, q.z};
                                for (int a = 0; a < 3; ++a) {
                                    lo[a] = dmin(dmin(lo[a], pp[a]), qq[a]);
                                    hi[a] = dmax(dmax(hi[a], pp[a]), qq[a]);
                                }
                                ++cnt;
                            }
                        }
                    }
                }
            }
        }
        flag[i] = ok;
    }
    // CTA reduction (min/max are exact: order-free)
    for (int off = 16; off > 0; off >>= 1) {
        for (int a = 0; a < 3; ++a) {
            lo[a] = dmin(lo[a], __shfl_down_sync(0xffffffffu, lo[a], off));
            hi[a] = dmax(hi[a], __shfl_down_sync(0xffffffffu, hi[a], off));
        }
        cnt += __shfl_down_sync(0xffffffffu, cnt, off);
    }
    __shared__ double s_b[kIcpThreads / 32][6];
    __shared__ unsigned long long s_c[kIcpThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        for (int a = 0; a < 3; ++a) {
            s_b[wid][a] = lo[a];
            s_b[wid][3 + a] = hi[a];
        }
        s_c[wid] = cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < kIcpThreads / 32; ++k) {
            for (int a = 0; a < 3; ++a) {
                s_b[0][a] = dmin(s_b[0][a], s_b[k][a]);
                s_b[0][3 + a] = dmax(s_b[0][3 + a], s_b[k][3 + a]);
            }
            s_c[0] += s_c[k];
        }
        for (int a = 0; a < 6; ++a) part_bbox[blockIdx.x * 6 + a] = s_b[0][a];
        part_count[blockIdx.x] = s_c[0];
    }
    if (last_cta(counter)) {
        if (threadIdx.x == 0) st->bodies += 1;
        bbox_finalize(st, part_bbox, part_count, gridDim.x, prm);
        if (threadIdx.x == 0) *counter = 0;
    }
}

// solve_gated + apply_motion + convergence (registration.cpp:175-212), one thread.
// The eigendecomposition of the normal matrix is done before, by one warp (e).
__device__ __noinline__ void solve_finalize(IcpState* st, const double* s_sum, const Eig6& e,
                                            const IcpParamsDev& prm) {
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
    st->delta = apply_motion(st->delta, r, t);
    st->iterations = iter + 1;
    if (st->shrunk_norm < prm.eps) st->done = 1;
}

constexpr int kMergeLanes = kIcpThreads / kSums;  // threads per sum in the final merge (252 of 256 busy)

// assemble (registration.cpp:93-123) on the shrunk matches (registration.cpp:65-72).
__global__ void __launch_bounds__(kIcpThreads)
    k_icp_assemble(IcpState* st, const MatchRec* __restrict__ rec, const uint8_t* __restrict__ flag, int n,
                   DD* __restrict__ part, unsigned int* counter, IcpParamsDev prm, int use_cond,
                   cudaGraphConditionalHandle cond) {
    if (st->done) {  // converged / lost (possibly in this iteration's match pass): end the loop
        if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(cond, 0u);
        return;
    }
    const d3 c = st->center, inv = st->inv_scale, scl = st->scale;
    DD acc[kSums];
#pragma unroll
    for (int k = 0; k < kSums; ++k) acc[k] = DD{0.0, 0.0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (!flag[i]) continue;
        const MatchRec r = rec[i];
        const d3 p = mk(r.p[0], r.p[1], r.p[2]), q = mk(r.q[0], r.q[1], r.q[2]), nn = mk(r.n[0], r.n[1], r.n[2]);
        const d3 p_hat = cmul(inv, sub(p, c));
        const d3 q_hat = cmul(inv, sub(q, c));
        const d3 c_hat = cmul(inv, sub(cross(p, nn), cross(c, nn)));
        const double row[6] = {c_hat.x, c_hat.y, c_hat.z, nn.x, nn.y, nn.z};
        const double d = dot(cmul(scl, sub(p_hat, q_hat)), nn);
        int k = 0;
#pragma unroll
        for (int a = 0; a < 6; ++a)
#pragma unroll
            for (int b = a; b < 6; ++b, ++k) dd_add(acc[k], row[a] * row[b]);
#pragma unroll
        for (int a = 0; a < 6; ++a) dd_add(acc[21 + a], -row[a] * d);
        dd_add(acc[27], d * d);
    }
    // warp tree
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int k = 0; k < kSums; ++k) {
            DD o;
            o.hi = __shfl_down_sync(0xffffffffu, acc[k].hi, off);
            o.lo = __shfl_down_sync(0xffffffffu, acc[k].lo, off);
            dd_merge(acc[k], o);
        }
    }
    __shared__ DD s_acc[kIcpThreads / 32][kSums];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0)
        for (int k = 0; k < kSums; ++k) s_acc[wid][k] = acc[k];
    __syncthreads();
    if (threadIdx.x < kSums) {
        DD a = s_acc[0][threadIdx.x];
        for (int w = 1; w < kIcpThreads / 32; ++w) dd_merge(a, s_acc[w][threadIdx.x]);
        part[blockIdx.x * kSums + threadIdx.x] = a;
    }
    if (!last_cta(counter)) return;
    // Fixed-order merge of all CTA partials: sum k, lane j takes partials j, j+L, ... The
    // loads go straight to L2 (ld.cg, after last_cta's fence) in batches of kBatch so their
    // latencies overlap; the merge order is fixed, so the result is deterministic.
    constexpr int L = kMergeLanes, kBatch = 8;
    __shared__ DD s_m[kSums][L];
    __shared__ double s_sum[kSums];
    const int nparts = gridDim.x;
    if (threadIdx.x < kSums * L) {
        const int k = threadIdx.x % kSums, j = threadIdx.x / kSums;
        const double2* vp = reinterpret_cast<const double2*>(part);
        DD a{0.0, 0.0};
        bool first = true;
        for (int p0 = j; p0 < nparts; p0 += kBatch * L) {
            double2 b[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                const int p = p0 + u * L;
                b[u] = p < nparts ? __ldcg(&vp[p * kSums + k]) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < kBatch; ++u) {
                if (p0 + u * L >= nparts) break;
                const DD x{b[u].x, b[u].y};
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
    __syncthreads();
    if (threadIdx.x < kSums) {
        DD a = s_m[threadIdx.x][0];
        for (int j = 1; j < kMergeLanes; ++j) dd_merge(a, s_m[threadIdx.x][j]);
        s_sum[threadIdx.x] = a.hi + a.lo;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        __shared__ double s_A[36];
        __shared__ Eig6 s_eig;
        for (int i = threadIdx.x; i < 36; i += 32) {
            const int r = i / 6, c = i % 6, lo = r < c ? r : c, hi = r < c ? c : r;
            s_A[i] = s_sum[lo * 6 - lo * (lo - 1) / 2 + (hi - lo)];  // packed upper triangle, row-major
        }
        __syncwarp();
        eigendecompose_sym6_warp(s_A, &s_eig);
        __syncwarp();
        if (threadIdx.x == 0) {
            solve_finalize(st, s_sum, s_eig, prm);
            *counter = 0;
            if (use_cond) cudaGraphSetConditional(cond, (!st->done && st->iterations < prm.max_iterations) ? 1u : 0u);
        }
    }
}

IcpParamsDev make_icp_params(const sf_match_params& p) {
    IcpParamsDev d;
    d.cos_max = std::cos(p.max_normal_angle);          // registration.cpp:25
    d.max_dist_sq = p.max_distance * p.max_distance;   // registration.cpp:26
    d.eps = p.convergence_epsilon;
    d.theta = p.eigen_threshold;
    d.floor = p.shrink_floor;
    d.max_iterations = p.max_iterations;
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
                uint64_t* launches, const int* dead, bool* device_loop) {
    const int n = si.w * si.h;
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
    if (!loop) {
        k_icp_init<<<1, 1, 0, s>>>(wk.st, d_initial, dead, prm.max_iterations, 0, 0);
        SF_LAUNCH_CHECK();
        uint64_t cnt = 1;
        for (int it = 0; it < prm.max_iterations; ++it) {
            k_icp_match<<<kIcpCtas, kIcpThreads, 0, s>>>(src, src_n, tgt, tgt_n, si, ti, prm, wk.st, wk.rec, wk.flag,
                                                         wk.part_bbox, wk.part_count, wk.counters);
            k_icp_assemble<<<kIcpCtas, kIcpThreads, 0, s>>>(wk.st, wk.rec, wk.flag, n, wk.part, wk.counters + 1, prm,
                                                            0, 0);
            SF_LAUNCH_CHECK();
            cnt += 2;
        }
        if (launches) *launches += cnt;
        return;
    }
    cudaGraph_t g = nullptr;
    SF_CUDA(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, nullptr, nullptr));
    cudaGraphConditionalHandle cond;
    SF_CUDA(cudaGraphConditionalHandleCreate(&cond, g, 0, 0));
    k_icp_init<<<1, 1, 0, s>>>(wk.st, d_initial, dead, prm.max_iterations, 1, cond);
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
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    if (!wk.body_stream) SF_CUDA(cudaStreamCreateWithFlags(&wk.body_stream, cudaStreamNonBlocking));
    cudaStream_t bs = wk.body_stream;
    SF_CUDA(cudaStreamBeginCaptureToGraph(bs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    k_icp_match<<<kIcpCtas, kIcpThreads, 0, bs>>>(src, src_n, tgt, tgt_n, si, ti, prm, wk.st, wk.rec, wk.flag,
                                                  wk.part_bbox, wk.part_count, wk.counters);
    k_icp_assemble<<<kIcpCtas, kIcpThreads, 0, bs>>>(wk.st, wk.rec, wk.flag, n, wk.part, wk.counters + 1, prm, 1,
                                                     cond);
    const cudaError_t le = cudaGetLastError();
    cudaGraph_t captured = nullptr;
    const cudaError_t ee = cudaStreamEndCapture(bs, &captured);
    SF_CUDA(le);
    SF_CUDA(ee);
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

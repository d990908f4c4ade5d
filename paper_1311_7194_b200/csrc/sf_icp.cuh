// sf_icp.cuh — ICP device state shared by sf_icp.cu and the tracker.
#pragma once

#include <functional>

#include "sf_internal.h"

namespace sf {

constexpr int kIcpThreads = 256;
constexpr int kIcpCtas = 296;  // 2 per SM; fixed => deterministic reduction tree
constexpr int kSums = 28;      // 21 upper(A) + 6 b + 1 residual

struct DD {
    double hi, lo;
};
__device__ __forceinline__ void dd_add(DD& a, double x) {
    const double s = a.hi + x;
    const double bb = s - a.hi;
    const double e = (a.hi - (s - bb)) + (x - bb);
    a.hi = s;
    a.lo += e;
}
__device__ __forceinline__ void dd_merge(DD& a, const DD& b) {
    const double s = a.hi + b.hi;
    const double bb = s - a.hi;
    const double e = (a.hi - (s - bb)) + (b.hi - bb);
    a.hi = s;
    a.lo = (a.lo + b.lo) + e;
}

struct IcpState {
    Pose delta;
    int done;       // converged or failed: later iterations are no-ops
    int lost;       // TrackingLost raised
    int iterations;
    int bodies;     // iterations whose step kernel ran (device-side loop: one launch each)
    unsigned long long matches;       // matches of the last completed iteration
    unsigned long long lost_count;    // match count that triggered TrackingLost
    d3 center, scale, inv_scale;      // shrink of the current iteration
    unsigned long long cur_count;
    // GatedSolution of the last iteration
    double eigenvalues[6];
    double eigenvectors[36];
    int gated[6];
    double residual_rms, shrunk_norm;
    unsigned long long pair_count;
    d3 motion_r, motion_t;
    // Fast gated solve (every eigenvalue certified above the gate): the eigendecomposition of
    // the last iteration's normal matrix is deferred to k_icp_report (off the critical path).
    int eig_pending;
    double A_last[21];  // packed upper triangle of the last iteration's (shrunk) normal matrix
    unsigned long long t_begin, t_end;  // device clock (ns): state init, end of the last solve
    unsigned long long t_step0, t_assoc0;  // first step: first CTA start, association done (tail start)
};

// One rank's share of an iteration's normal equations (sharded ICP): the 28 unshrunk sums as
// double-double pairs, the match count, the box as (lo, -hi) so that one MIN all-reduce
// combines it. An NCCL SUM over sums[] + count and a MIN over box[] merge the ranks.
struct IcpRankPartial {
    double sums[2 * kSums];
    double count;
    double box[6];
    double pad;
};

struct IcpParamsDev {
    double max_dist_sq, cos_max, eps, theta, floor;
    int max_iterations;
    int exact;  // sf_match_params.reduction == 1: the reference's summation order
};

// One correspondence of match_points (registration.hpp PointMatch), reference-order path.
struct MatchRec {
    double p[3], q[3], n[3];
};

// Scratch for one ICP (owned by the caller: stand-alone API or tracker).
struct IcpWork {
    int w = 0, h = 0;
    double* part_bbox = nullptr;
    unsigned long long* part_count = nullptr;
    DD* part = nullptr;
    IcpState* st = nullptr;
    float* src_normals = nullptr;
    float *src = nullptr, *tgt = nullptr, *tgt_n = nullptr, *src_n_in = nullptr;
    double* initial = nullptr;
    unsigned int* counters = nullptr;  // "last CTA" tickets of the two fused reductions
    // reference-order reduction (allocated on first use): row-major-compacted matches per
    // CTA range, and the 28 per-match terms in match order
    MatchRec* rec = nullptr;
    double* terms = nullptr;
    void ensure_exact() {
        if (rec) return;
        const size_t n = static_cast<size_t>(w) * h;
        SF_CUDA(cudaMalloc(&rec, n * sizeof(MatchRec)));
        SF_CUDA(cudaMalloc(&terms, n * kSums * sizeof(double)));
    }
    void ensure(int W, int H) {
        if (W == w && H == h && st) return;
        release();
        const size_t n = static_cast<size_t>(W) * H;
        SF_CUDA(cudaMalloc(&counters, 4 * sizeof(unsigned int)));
        SF_CUDA(cudaMemset(counters, 0, 4 * sizeof(unsigned int)));
        SF_CUDA(cudaMalloc(&part_bbox, kIcpCtas * 6 * sizeof(double)));
        SF_CUDA(cudaMalloc(&part_count, kIcpCtas * sizeof(unsigned long long)));
        SF_CUDA(cudaMalloc(&part, kIcpCtas * kSums * sizeof(DD)));
        SF_CUDA(cudaMalloc(&st, sizeof(IcpState)));
        SF_CUDA(cudaMemset(st, 0, sizeof(IcpState)));  // fields a path never writes are snapshotted whole
        SF_CUDA(cudaMalloc(&src_normals, 3 * n * sizeof(float)));
        SF_CUDA(cudaMalloc(&src, n * sizeof(float)));
        SF_CUDA(cudaMalloc(&tgt, n * sizeof(float)));
        SF_CUDA(cudaMalloc(&tgt_n, 3 * n * sizeof(float)));
        SF_CUDA(cudaMalloc(&src_n_in, 3 * n * sizeof(float)));
        SF_CUDA(cudaMalloc(&initial, 12 * sizeof(double)));
        w = W;
        h = H;
    }
    void release() {
        void* p[] = {part_bbox, part_count, part, st, src_normals, src, tgt, tgt_n, src_n_in, initial,
                     counters, rec, terms};
        for (void* q : p)
            if (q) cudaFree(q);
        rec = nullptr;
        terms = nullptr;
        counters = nullptr;
        part_bbox = nullptr;
        part_count = nullptr;
        part = nullptr;
        st = nullptr;
        src_normals = src = tgt = tgt_n = src_n_in = nullptr;
        initial = nullptr;
        w = h = 0;
    }
    cudaStream_t body_stream = nullptr;  // captures the body of the device-side iteration loop
    ~IcpWork() {
        release();
        if (body_stream) cudaStreamDestroy(body_stream);
    }
};

IcpParamsDev make_icp_params(const sf_match_params& p);
// state_ready: the caller already initialised wk.st (icp_state_init in one of its kernels), so
// the ICP starts with its first step; under capture the first step is a plain kernel node and
// only later iterations run in the conditional WHILE node.
void launch_icp(IcpWork& wk, const float* src, const float* src_n, const float* tgt, const float* tgt_n,
                const Intr& si, const Intr& ti, const double* d_initial, const IcpParamsDev& prm, cudaStream_t s,
                uint64_t* launches, const int* dead, bool* device_loop = nullptr, bool state_ready = false);

// IcpState for a new ICP from the initial delta (one thread).
__device__ inline void icp_state_init(IcpState* st, const double* initial12, bool dead) {
    IcpState z;
    memset(&z, 0, sizeof(z));
    z.delta = pose_from12(initial12);
    z.done = dead ? 1 : 0;
    z.t_begin = globaltimer_ns();
    *st = z;
}
void fill_icp_result(const IcpState& st, sf_icp_result* out);
// Sharded ICP: partial sums over pixel slices per local rank, `reduce` across processes (NCCL),
// replicated solve (sf_icp.cu). recs: nlocal records (this process's ranks); nrec: records the
// solve merges after `reduce` (nlocal in-process, 1 after an all-reduce across processes).
void launch_icp_ranks(IcpWork& wk, const float* src, const float* src_n, const float* tgt, const float* tgt_n,
                      const Intr& I, const double* d_initial, const IcpParamsDev& prm, int rank0, int nlocal,
                      int world, IcpRankPartial* recs, int nrec, const std::function<void(cudaStream_t)>& reduce,
                      bool allow_loop, cudaStream_t s, uint64_t* launches, const int* dead, bool* device_loop);
// Eigenpairs of the last iteration when the fast gated solve deferred them (one warp).
void launch_icp_report(IcpWork& wk, cudaStream_t s, uint64_t* launches);

}  // namespace sf

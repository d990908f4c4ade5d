// sf_tracker.cu — the fused frame: run()'s per-frame body (pipeline.cpp:233-301) on the
// device, captured once into a CUDA graph and replayed per frame.
//
// Track step (pipeline.cpp:257-287):
//   raycast(grid, current_pose)                  -> model depth + normals   (render.cpp)
//   initial_delta = compose(invert(current), current)   (initial_transform_hook without
//                                                         an external delta, registration.cpp:222-224)
//   icp(captured, model depth, model normals, initial_delta)   (source normals from
//                                                         match.normal_options, registration.cpp:216-220)
//   estimated = compose(current, delta); current = estimated
//   fuse_frame(grid, captured, estimated)
// Ground-truth step (and the first frame): fuse at the given pose.
// TrackingLost / PoolExhausted set a device "dead" flag: the rest of the frame and every
// later step become no-ops, mirroring run()'s break (pipeline.cpp:289-299).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "sf_icp.cuh"
#include "sf_linalg.cuh"
#include "sf_sample.cuh"

namespace sf {

struct TrackerDev {
    int dead;
    int status;
    int registered;
    int frame;
    int died_at;  // frame whose TrackingLost / PoolExhausted set `dead` (-1: none)
    int pad_;
};

// run()'s catch blocks end the loop at the failing frame (pipeline.cpp:289-299).
__device__ __forceinline__ void mark_dead(TrackerDev* td, int status) {
    td->dead = 1;
    td->status = status;
    td->died_at = td->frame;
}

// Everything a frame's metrics are decoded from (host side: pinned, mapped).
struct TrackerFetch {
    double cur[12];
    double fuse_pose[12];
    TrackerDev td;
    FrameCounters ctr;
    RayCounters rs;
    IcpState icp;
};

template <typename T>
__device__ __forceinline__ void copy_words(T* dst, const T* src, int tid, int nthreads) {
    static_assert(sizeof(T) % 8 == 0, "8-byte words");
    const unsigned long long* s = reinterpret_cast<const unsigned long long*>(src);
    volatile unsigned long long* d = reinterpret_cast<volatile unsigned long long*>(dst);
    for (int i = tid; i < static_cast<int>(sizeof(T) / 8); i += nthreads) d[i] = s[i];
}

// Frame metrics snapshot written straight to mapped pinned memory (all threads of one CTA).
__device__ inline void snapshot_body(TrackerFetch* dst, const double* __restrict__ cur,
                                     const double* __restrict__ fuse_pose, const TrackerDev* td,
                                     const FrameCounters* ctr, const RayCounters* __restrict__ rs,
                                     const IcpState* __restrict__ icp) {
    const int t = threadIdx.x, n = blockDim.x;
    volatile double* dc = dst->cur;
    volatile double* dp = dst->fuse_pose;
    if (t < 12) {
        dc[t] = cur[t];
        dp[t] = fuse_pose[t];
    }
    copy_words(&dst->td, td, t, n);
    copy_words(&dst->ctr, ctr, t, n);
    copy_words(&dst->rs, rs, t, n);
    copy_words(&dst->icp, icp, t, n);
}
__global__ void k_tracker_snapshot(TrackerFetch* dst, const double* __restrict__ cur,
                                   const double* __restrict__ fuse_pose, const TrackerDev* __restrict__ td,
                                   const FrameCounters* __restrict__ ctr, const RayCounters* __restrict__ rs,
                                   const IcpState* __restrict__ icp) {
    snapshot_body(dst, cur, fuse_pose, td, ctr, rs, icp);
}

// Where a step's last kernel leaves the frame's metrics: one of two mapped pinned snapshots
// (by step parity, counted on the device in TrackerDev::frame) read by sf_tracker_fetch_frame.
struct SnapTargets {
    TrackerFetch* slot[2];
    const double* cur;
    const double* fuse_pose;
    const RayCounters* rs;
    const IcpState* icp;
};
__device__ inline void finish_snapshot(const SnapTargets& st, TrackerDev* td, const FrameCounters* ctr) {
    __syncthreads();  // thread 0's final counter / status writes
    snapshot_body(st.slot[td->frame & 1], st.cur, st.fuse_pose, td, ctr, st.rs, st.icp);
    __syncthreads();
    if (threadIdx.x == 0) td->frame += 1;
}

__global__ void k_tracker_begin_track(const double* __restrict__ cur, const double* __restrict__ external,
                                      double* __restrict__ init_delta, RayCounters* rstats, TrackerDev* td) {
    if (td->dead) return;
    // initial_pose = initial_transform_hook(current, external) = external ? compose(current,
    // *external) : current (registration.cpp:222-224); initial_delta = compose(invert(current),
    // initial_pose) (pipeline.cpp:262-267)
    const Pose c = pose_from12(cur);
    const Pose init = external ? compose(c, pose_from12(external)) : c;
    const Pose d = compose(invert(c), init);
    pose_to12(d, init_delta);
    RayCounters z{0, 0, 0, 0};
    *rstats = z;
    td->registered = 0;  // set again once ICP succeeds (pipeline.cpp:274)
}

__global__ void k_tracker_after_icp(double* __restrict__ cur, double* __restrict__ fuse_pose, const IcpState* st,
                                    TrackerDev* td, int orthonormalize) {
    if (td->dead) return;
    if (st->lost) {
        mark_dead(td, SF_TRACKING_LOST);
        return;
    }
    Pose est = compose(pose_from12(cur), st->delta);  // pipeline.cpp:282
    if (orthonormalize) est.R = nearest_rotation(est.R);
    pose_to12(est, cur);
    pose_to12(est, fuse_pose);
    td->registered = 1;
}

// One warp: begin_track (lane 0) and the raycast's frame constants at the current pose.
__global__ void k_tracker_begin_track_consts(VolParams P, Intr cam, const double* __restrict__ cur,
                                             const double* __restrict__ external, double* __restrict__ init_delta,
                                             RayCounters* rstats, TrackerDev* td, FrameConsts* fc,
                                             IcpState* icp) {
    if (threadIdx.x == 0) {
        if (!td->dead) {
            const Pose c = pose_from12(cur);
            const Pose init = external ? compose(c, pose_from12(external)) : c;
            pose_to12(compose(invert(c), init), init_delta);
            RayCounters z{0, 0, 0, 0};
            *rstats = z;
            td->registered = 0;  // set again once ICP succeeds (pipeline.cpp:274)
        }
        icp_state_init(icp, init_delta, td->dead != 0);  // the frame's ICP starts from init_delta
    }
    frame_consts_warp(P, cam, cur, fc);
}

// One warp: the pose update after ICP (lane 0, as k_tracker_after_icp), then the fusion's
// frame constants at that pose and its counter reset (launch_fuse's first two kernels).
__global__ void k_tracker_after_icp_fuse_begin(double* __restrict__ cur, double* __restrict__ fuse_pose,
                                               const IcpState* st, TrackerDev* td, int orthonormalize, VolParams P,
                                               Intr cam, FrameConsts* fc, FrameCounters* ctr, const VolCounters* vc) {
    if (threadIdx.x == 0 && !td->dead) {
        if (st->lost) {
            mark_dead(td, SF_TRACKING_LOST);
        } else {
            Pose est = compose(pose_from12(cur), st->delta);  // pipeline.cpp:282
            if (orthonormalize) est.R = nearest_rotation(est.R);
            pose_to12(est, cur);
            pose_to12(est, fuse_pose);
            td->registered = 1;
        }
    }
    __syncwarp();
    frame_consts_warp(P, cam, fuse_pose, fc);
    if (threadIdx.x == 0) fuse_begin_body(ctr, vc, &td->dead);
}

// fuse_finalize + tracker finish
__global__ void k_tracker_fuse_finish(FrameCounters* ctr, const VolCounters* vc, TrackerDev* td, SnapTargets snap) {
    if (threadIdx.x == 0) {
        fuse_finalize_body(ctr, vc);
        if (!td->dead && ctr->exhausted) mark_dead(td, SF_POOL_EXHAUSTED);
    }
    finish_snapshot(snap, td, ctr);
}

__global__ void k_tracker_begin_gt(const double* __restrict__ gt, double* __restrict__ cur,
                                   double* __restrict__ fuse_pose, RayCounters* rstats, TrackerDev* td, int set_current) {
    if (td->dead) return;
    for (int i = 0; i < 12; ++i) {
        fuse_pose[i] = gt[i];
        if (set_current) cur[i] = gt[i];
    }
    RayCounters z{0, 0, 0, 0};
    *rstats = z;
    td->registered = 0;
}

__global__ void k_tracker_finish(const FrameCounters* ctr, TrackerDev* td, SnapTargets snap) {
    if (threadIdx.x == 0 && !td->dead && ctr->exhausted) mark_dead(td, SF_POOL_EXHAUSTED);
    finish_snapshot(snap, td, ctr);
}

}  // namespace sf

using namespace sf;

// The captured frame (and its sigma plane) into the tracker's buffers: one launch for both.
__global__ void k_copy_frame(float4* __restrict__ d0, const float4* __restrict__ s0, float4* __restrict__ d1,
                             const float4* __restrict__ s1, size_t n4) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
        d0[i] = __ldg(&s0[i]);
        if (d1) d1[i] = __ldg(&s1[i]);
    }
}
// Returns true when it launched the kernel (false: plain copies for unaligned buffers).
static bool launch_copy_frame(float* d0, const float* s0, float* d1, const float* s1, size_t n, cudaStream_t s) {
    const bool vec = n % 4 == 0 && (reinterpret_cast<uintptr_t>(s0) & 15) == 0 &&
                     (!d1 || (reinterpret_cast<uintptr_t>(s1) & 15) == 0);
    if (!vec) {  // unaligned user buffers: plain copies
        SF_CUDA(cudaMemcpyAsync(d0, s0, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
        if (d1) SF_CUDA(cudaMemcpyAsync(d1, s1, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
        return false;
    }
    k_copy_frame<<<148 * 2, 256, 0, s>>>(reinterpret_cast<float4*>(d0), reinterpret_cast<const float4*>(s0),
                                         reinterpret_cast<float4*>(d1), reinterpret_cast<const float4*>(s1), n / 4);
    SF_LAUNCH_CHECK();
    return true;
}

// A host pose (12 doubles) into device memory through the kernel's parameters: no
// host-to-device copy from pageable memory on the step's stream.
struct Pose12 {
    double v[12];
};
__global__ void k_set_pose12(double* __restrict__ dst, Pose12 p) {
    if (threadIdx.x < 12) dst[threadIdx.x] = p.v[threadIdx.x];
}

struct sf_tracker {
    sf_volume* vol = nullptr;
    sf_tracker_config cfg{};
    Intr cam{};
    FuseParams fp{};
    FuseParams fp_sigma{};
    IcpParamsDev icp_prm{};
    FrameBuffers fb;
    IcpWork icp;
    double* d_cur = nullptr;
    double* d_init_delta = nullptr;
    double* d_gt = nullptr;
    FrameConsts* d_rc_fc = nullptr;
    float *d_ts = nullptr, *d_te = nullptr, *d_model_depth = nullptr, *d_model_normals = nullptr;
    float *d_cap = nullptr, *d_cap_sigma = nullptr;
    RayCounters* d_rstats = nullptr;
    int* d_ray_list = nullptr;  // active rays of the model raycast
    RayBracket* d_brackets = nullptr;  // stage-1 brackets (refine pass)
    TrackerDev* d_td = nullptr;
    // host-side
    int frames = 0;
    int last_mode = 0;
    bool last_registered = false;
    uint64_t last_launches = 0;
    cudaStream_t capture_stream = nullptr;  // graphs are captured here (the legacy stream cannot capture)
    cudaStream_t side_stream = nullptr;     // graph branch: deferred ICP eigenpairs, parallel to the fuse
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_prep_fork = nullptr, ev_prep_join = nullptr;
    // Streaming host frames: the H2D copy of frame k runs on copy_stream into stage[k % 2]
    // while frame k-1 computes; each frame's metrics are snapshotted into snap[k % 2].
    cudaStream_t copy_stream = nullptr;
    float* d_stage[2] = {nullptr, nullptr};
    float* d_stage_sigma[2] = {nullptr, nullptr};
    cudaEvent_t ev_staged[2] = {nullptr, nullptr}, ev_stage_free[2] = {nullptr, nullptr};
    cudaEvent_t ev_snap[2] = {nullptr, nullptr};
    cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // stage timing (graph nodes)
    int stage_events = 2;  // 2: all stage events, 1: integrate pair only, 0: none
    void mark(int i, cudaStream_t s) {
        if (stage_events == 2 || (stage_events == 1 && (i == 3 || i == 4))) record_event(ev[i], s);
    }
    cudaGraphExec_t graph[3][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};  // [mode][sigma]
    uint64_t graph_kernels[3][2] = {{0, 0}, {0, 0}, {0, 0}};
    bool graph_icp_loop[3][2] = {{false, false}, {false, false}, {false, false}};
    bool issue_icp_loop = false;  // set by issue(): ICP iterations run as a device-side loop
    bool last_icp_loop = false;
    // pinned fetch staging (also the per-frame snapshot layout)
    using Fetch = TrackerFetch;
    uint64_t extra_launches = 0;  // kernels of the current step outside the frame graph
    TrackerFetch* snap_dev[2] = {nullptr, nullptr};  // device views of snap[0..1]
    Fetch* h = nullptr;
    Fetch* snap = nullptr;  // pinned [2]: per-frame metric snapshots (streaming)
    struct SnapMeta {
        int frame, mode;
        uint64_t launches;
        bool icp_loop;
    } snap_meta[2] = {};

    // device buffers -> pinned host f (asynchronous on s)
    SnapTargets snap_targets() const {
        SnapTargets t;
        t.slot[0] = snap_dev[0];
        t.slot[1] = snap_dev[1];
        t.cur = d_cur;
        t.fuse_pose = fb.pose;
        t.rs = d_rstats;
        t.icp = icp.st;
        return t;
    }
    // The frame's metrics into pinned host memory: one kernel storing through the mapped
    // pointer (six separate device-to-host copies cost ~20 us of stream latency per step).
    void copy_metrics(Fetch* f, cudaStream_t s) {
        Fetch* df = nullptr;
        SF_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&df), f, 0));
        k_tracker_snapshot<<<1, 128, 0, s>>>(df, d_cur, fb.pose, d_td, fb.ctr, d_rstats, icp.st);
        SF_LAUNCH_CHECK();
    }
    void decode(const Fetch* f, int frame, int mode, uint64_t launches, bool icp_loop, sf_frame_metrics* out) const;

    ~sf_tracker() {
        cudaSetDevice(vol ? vol->device : 0);
        for (auto& row : graph)
            for (auto& g : row)
                if (g) cudaGraphExecDestroy(g);
        void* p[] = {d_cur, d_init_delta, d_gt, d_rc_fc, d_ts, d_te, d_model_depth, d_model_normals, d_cap,
                     d_cap_sigma, d_rstats, d_td, d_ray_list, d_brackets};
        for (void* q : p)
            if (q) cudaFree(q);
        if (h) cudaFreeHost(h);
        if (capture_stream) cudaStreamDestroy(capture_stream);
        if (side_stream) cudaStreamDestroy(side_stream);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (ev_prep_fork) cudaEventDestroy(ev_prep_fork);
        if (ev_prep_join) cudaEventDestroy(ev_prep_join);
        if (copy_stream) cudaStreamDestroy(copy_stream);
        for (int i = 0; i < 2; ++i) {
            if (d_stage[i]) cudaFree(d_stage[i]);
            if (d_stage_sigma[i]) cudaFree(d_stage_sigma[i]);
            if (ev_staged[i]) cudaEventDestroy(ev_staged[i]);
            if (ev_stage_free[i]) cudaEventDestroy(ev_stage_free[i]);
            if (ev_snap[i]) cudaEventDestroy(ev_snap[i]);
        }
        if (snap) cudaFreeHost(snap);
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
    }

    // The frame's launch sequence (captured into a graph or issued directly).
    uint64_t issue(int mode, bool has_sigma, cudaStream_t s) {
        uint64_t n = 0;
        const int* dead = &d_td->dead;
        const FuseParams& p = has_sigma ? fp_sigma : fp;
        const float* sig = has_sigma ? d_cap_sigma : nullptr;
        mark(0, s);
        issue_icp_loop = false;
        bool joined = true;
        bool prep_done = false, merged = false;
        if (mode == 0 || mode == 3) {
            // Branch: everything that depends only on the captured frame (ICP source normals,
            // the fusion's normals / edge mask / per-pixel factors) runs beside the raycast.
            SF_CUDA(cudaEventRecord(ev_prep_fork, s));
            SF_CUDA(cudaStreamWaitEvent(side_stream, ev_prep_fork, 0));
            launch_compute_normals(d_cap, cam.w, cam.h, cam, cfg.match.normal_sigma0, cfg.match.normal_spatial_scale,
                                   icp.src_normals, side_stream, &n, dead);
            launch_fuse_prep(*vol, fb, cam, d_cap, sig, p, side_stream, &n, dead);
            SF_CUDA(cudaEventRecord(ev_prep_join, side_stream));
            prep_done = true;
            k_tracker_begin_track_consts<<<1, 32, 0, s>>>(vol->P, cam, d_cur, mode == 3 ? d_gt : nullptr,
                                                          d_init_delta, d_rstats, d_td, d_rc_fc, icp.st);
            SF_LAUNCH_CHECK();
            ++n;
            launch_ray_bounds(*vol, d_rc_fc, cam, d_ts, d_te, s, &n, dead, d_ray_list, d_rstats, d_model_depth,
                              d_model_normals);
            launch_raycast(*vol, d_rc_fc, cam, d_ts, d_te, d_model_depth, d_model_normals, d_rstats, s, &n, dead,
                           d_ray_list, d_brackets);
            mark(1, s);
            SF_CUDA(cudaStreamWaitEvent(s, ev_prep_join, 0));
            launch_icp(icp, d_cap, icp.src_normals, d_model_depth, d_model_normals, cam, cam, d_init_delta, icp_prm, s,
                       &n, dead, &issue_icp_loop, true);
            k_tracker_after_icp_fuse_begin<<<1, 32, 0, s>>>(d_cur, fb.pose, icp.st, d_td, cfg.orthonormalize, vol->P,
                                                            cam, fb.fc, fb.ctr, vol->d_vc);
            SF_LAUNCH_CHECK();
            ++n;
            merged = true;
            // the deferred eigenpairs of the last ICP iteration run beside the fuse
            SF_CUDA(cudaEventRecord(ev_fork, s));
            SF_CUDA(cudaStreamWaitEvent(side_stream, ev_fork, 0));
            launch_icp_report(icp, side_stream, &n);
            SF_CUDA(cudaEventRecord(ev_join, side_stream));
            joined = false;
            mark(2, s);
        } else {
            k_tracker_begin_gt<<<1, 1, 0, s>>>(d_gt, d_cur, fb.pose, d_rstats, d_td, mode == 1 ? 1 : 0);
            SF_LAUNCH_CHECK();
            ++n;
            mark(1, s);
            mark(2, s);
        }
        FuseEvents fe;
        fe.before_integrate = stage_events ? ev[3] : nullptr;
        fe.after_integrate = stage_events ? ev[4] : nullptr;
        launch_fuse(*vol, fb, cam, d_cap, sig, p, s, false, &n, dead, &fe, prep_done, merged);
        if (!joined) {
            SF_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
            joined = true;
        }
        if (merged) k_tracker_fuse_finish<<<1, 128, 0, s>>>(fb.ctr, vol->d_vc, d_td, snap_targets());
        else k_tracker_finish<<<1, 128, 0, s>>>(fb.ctr, d_td, snap_targets());
        SF_LAUNCH_CHECK();
        ++n;
        mark(5, s);
        return n;
    }
};

extern "C" {

int sf_tracker_create(sf_volume_t vol, const sf_tracker_config* config, const double initial_pose[12],
                      sf_tracker_t* out) {
    return guarded([&]() -> int {
        if (!vol || !config || !initial_pose || !out) throw Error(SF_INVALID_ARGUMENT, "sf_tracker_create: null");
        SF_CUDA(cudaSetDevice(vol->device));
        auto t = std::make_unique<sf_tracker>();
        t->vol = vol;
        t->cfg = *config;
        t->cam = to_intr(config->camera);
        t->fp = resolve_fuse_params(*vol, config->fusion, false);
        t->fp_sigma = resolve_fuse_params(*vol, config->fusion, true);
        t->icp_prm = make_icp_params(config->match);
        const int w = config->camera.width, h = config->camera.height;
        if (w <= 0 || h <= 0) throw Error(SF_INVALID_ARGUMENT, "intrinsics: non-positive image size");
        ensure_frame_buffers(*vol, t->fb, w, h);
        t->icp.ensure(w, h);
        if (t->icp_prm.exact) t->icp.ensure_exact();  // not allowed later, inside the graph capture
        const size_t n = static_cast<size_t>(w) * h;
        SF_CUDA(cudaMalloc(&t->d_cur, 12 * sizeof(double)));
        SF_CUDA(cudaMalloc(&t->d_init_delta, 12 * sizeof(double)));
        SF_CUDA(cudaMalloc(&t->d_gt, 12 * sizeof(double)));
        SF_CUDA(cudaMalloc(&t->d_rc_fc, sizeof(FrameConsts)));
        SF_CUDA(cudaMalloc(&t->d_ts, n * sizeof(float)));
        SF_CUDA(cudaMalloc(&t->d_te, n * sizeof(float)));
        SF_CUDA(cudaMalloc(&t->d_model_depth, n * sizeof(float)));
        SF_CUDA(cudaMalloc(&t->d_model_normals, 3 * n * sizeof(float)));
        SF_CUDA(cudaMalloc(&t->d_cap, n * sizeof(float)));
        SF_CUDA(cudaMalloc(&t->d_cap_sigma, n * sizeof(float)));
        SF_CUDA(cudaMalloc(&t->d_rstats, sizeof(RayCounters)));
        SF_CUDA(cudaMalloc(&t->d_ray_list, n * sizeof(int)));
        SF_CUDA(cudaMalloc(&t->d_brackets, n * sizeof(RayBracket)));

        SF_CUDA(cudaMalloc(&t->d_td, sizeof(TrackerDev)));
        const TrackerDev td0{0, 0, 0, 0, -1, 0};
        SF_CUDA(cudaMemcpy(t->d_td, &td0, sizeof(TrackerDev), cudaMemcpyHostToDevice));
        SF_CUDA(cudaMemset(t->d_rstats, 0, sizeof(RayCounters)));
        SF_CUDA(cudaMemset(t->d_init_delta, 0, 12 * sizeof(double)));
        SF_CUDA(cudaMemcpy(t->d_cur, initial_pose, 12 * sizeof(double), cudaMemcpyHostToDevice));
        SF_CUDA(cudaMallocHost(&t->h, sizeof(sf_tracker::Fetch)));
        for (auto& e : t->ev) SF_CUDA(cudaEventCreate(&e));
        SF_CUDA(cudaStreamCreateWithFlags(&t->side_stream, cudaStreamNonBlocking));
        SF_CUDA(cudaStreamCreateWithFlags(&t->copy_stream, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            SF_CUDA(cudaMalloc(&t->d_stage[i], n * sizeof(float)));
            SF_CUDA(cudaMalloc(&t->d_stage_sigma[i], n * sizeof(float)));
            SF_CUDA(cudaEventCreateWithFlags(&t->ev_staged[i], cudaEventDisableTiming));
            SF_CUDA(cudaEventCreateWithFlags(&t->ev_stage_free[i], cudaEventDisableTiming));
            SF_CUDA(cudaEventCreateWithFlags(&t->ev_snap[i], cudaEventDisableTiming));
        }
        SF_CUDA(cudaMallocHost(&t->snap, 2 * sizeof(sf_tracker::Fetch)));
        std::memset(t->snap, 0, 2 * sizeof(sf_tracker::Fetch));
        for (int i = 0; i < 2; ++i)
            SF_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&t->snap_dev[i]), &t->snap[i], 0));
        SF_CUDA(cudaEventCreateWithFlags(&t->ev_fork, cudaEventDisableTiming));
        SF_CUDA(cudaEventCreateWithFlags(&t->ev_join, cudaEventDisableTiming));
        SF_CUDA(cudaEventCreateWithFlags(&t->ev_prep_fork, cudaEventDisableTiming));
        SF_CUDA(cudaEventCreateWithFlags(&t->ev_prep_join, cudaEventDisableTiming));
        std::memset(t->h, 0, sizeof(sf_tracker::Fetch));
        *out = t.release();
        return SF_OK;
    });
}

int sf_tracker_destroy(sf_tracker_t tr) {
    delete tr;
    return SF_OK;
}

int sf_tracker_step(sf_tracker_t tr, const sf_frame* captured, int32_t mode, const double gt_pose[12], void* stream) {
    return guarded([&]() -> int {
        if (!tr || !captured) throw Error(SF_INVALID_ARGUMENT, "sf_tracker_step: null argument");
        if (captured->intrinsics.width != tr->cam.w || captured->intrinsics.height != tr->cam.h)
            throw Error(SF_INVALID_ARGUMENT, "sf_tracker_step: frame size differs from the tracker camera");
        if ((mode == 1 || mode == 2) && !gt_pose)
            throw Error(SF_INVALID_ARGUMENT, "sf_tracker_step: this mode needs a pose argument");
        if (mode < 0 || mode > 2) throw Error(SF_INVALID_ARGUMENT, "sf_tracker_step: unknown mode");
        if (mode != 1 && tr->frames > 0) require_codes(*tr->vol, "tracking (raycast of the model)");
        SF_CUDA(cudaSetDevice(tr->vol->device));
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const size_t n = static_cast<size_t>(tr->cam.w) * tr->cam.h;
        const bool has_sigma = captured->sigma != nullptr;
        tr->extra_launches = 0;
        const int slot = tr->frames & 1;
        if (captured->on_device) {
            tr->extra_launches +=
                launch_copy_frame(tr->d_cap, captured->depth, has_sigma ? tr->d_cap_sigma : nullptr, captured->sigma, n, s);
        } else {
            // Host frame: the H2D copy runs on the copy stream into a staging buffer, so it
            // overlaps the previous frame's compute; the frame then starts with a D2D copy.
            SF_CUDA(cudaStreamWaitEvent(tr->copy_stream, tr->ev_stage_free[slot], 0));
            SF_CUDA(cudaMemcpyAsync(tr->d_stage[slot], captured->depth, n * sizeof(float), cudaMemcpyHostToDevice,
                                    tr->copy_stream));
            if (has_sigma)
                SF_CUDA(cudaMemcpyAsync(tr->d_stage_sigma[slot], captured->sigma, n * sizeof(float),
                                        cudaMemcpyHostToDevice, tr->copy_stream));
            SF_CUDA(cudaEventRecord(tr->ev_staged[slot], tr->copy_stream));
            SF_CUDA(cudaStreamWaitEvent(s, tr->ev_staged[slot], 0));
            tr->extra_launches += launch_copy_frame(tr->d_cap, tr->d_stage[slot], has_sigma ? tr->d_cap_sigma : nullptr,
                                                    tr->d_stage_sigma[slot], n, s);
            SF_CUDA(cudaEventRecord(tr->ev_stage_free[slot], s));
        }
        // First frame: fuse at the current (initial) pose without registration (pipeline.cpp:250-252).
        // internal modes: 0 track, 1 ground truth, 2 fuse at current (first frame), 3 track with
        // an external initial delta (tracking.mode = icp_with_hook, pipeline.cpp:262-266)
        int eff = mode == 2 ? 3 : mode;
        if (mode != 1 && tr->frames == 0) eff = 2;  // fuse at current, keep current
        if (eff == 1 || eff == 3) {
            Pose12 g;
            for (int i = 0; i < 12; ++i) g.v[i] = gt_pose[i];
            k_set_pose12<<<1, 32, 0, s>>>(tr->d_gt, g);
            SF_LAUNCH_CHECK();
            tr->extra_launches += 1;
        }
        if (eff == 2) SF_CUDA(cudaMemcpyAsync(tr->d_gt, tr->d_cur, 12 * sizeof(double), cudaMemcpyDeviceToDevice, s));
        const int gmode = eff == 0 ? 0 : eff == 1 ? 1 : 2;
        const int sidx = has_sigma ? 1 : 0;
        if (tr->cfg.use_graphs && eff != 2) {
            cudaGraphExec_t& ge = tr->graph[gmode][sidx];
            if (!ge) {
                cudaGraph_t g;
                uint64_t issued = 0;
                if (!tr->capture_stream) SF_CUDA(cudaStreamCreateWithFlags(&tr->capture_stream, cudaStreamNonBlocking));
                cudaStream_t cs = tr->capture_stream;
                SF_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
                try {
                    issued = tr->issue(eff, has_sigma, cs);
                } catch (...) {
                    cudaStreamEndCapture(cs, &g);
                    throw;
                }
                SF_CUDA(cudaStreamEndCapture(cs, &g));
                SF_CUDA(cudaGraphInstantiate(&ge, g, 0));
                // kernels issued into the top-level graph (the ICP loop body is counted per
                // iteration at fetch time)
                tr->graph_kernels[gmode][sidx] = issued;
                tr->graph_icp_loop[gmode][sidx] = tr->issue_icp_loop;
                SF_CUDA(cudaGraphDestroy(g));
            }
            SF_CUDA(cudaGraphLaunch(ge, s));
            tr->last_launches = tr->graph_kernels[gmode][sidx];
            tr->last_icp_loop = tr->graph_icp_loop[gmode][sidx];
        } else {
            tr->last_launches = tr->issue(eff, has_sigma, s);
            tr->last_icp_loop = tr->issue_icp_loop;
        }
        tr->last_mode = eff;
        // metric snapshot of this frame (read by sf_tracker_fetch_frame without waiting for
        // frames issued later)
        // (the step's last kernel wrote this frame's metric snapshot into snap[slot])
        tr->last_launches += tr->extra_launches;  // the frame copy / pose kernels
        SF_CUDA(cudaEventRecord(tr->ev_snap[slot], s));
        tr->snap_meta[slot] = {tr->frames, eff, tr->last_launches, tr->last_icp_loop};
        ++tr->frames;
        return SF_OK;
    });
}

int sf_tracker_set_pose(sf_tracker_t tr, const double pose[12], void* stream) {
    return guarded([&]() -> int {
        if (!tr || !pose) throw Error(SF_INVALID_ARGUMENT, "sf_tracker_set_pose: null argument");
        SF_CUDA(cudaSetDevice(tr->vol->device));
        Pose12 g;
        for (int i = 0; i < 12; ++i) g.v[i] = pose[i];
        k_set_pose12<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(tr->d_cur, g);
        SF_LAUNCH_CHECK();
        return SF_OK;
    });
}

void sf_tracker::decode(const Fetch* f, int frame, int mode, uint64_t launches, bool icp_loop,
                        sf_frame_metrics* out) const {
    std::memset(out, 0, sizeof(*out));
    out->frame = frame;
    out->status = f->td.status;
    out->registered = (mode == 0 || mode == 3) ? f->td.registered : 0;
    std::memcpy(out->pose, f->fuse_pose, sizeof(out->pose));
    // The frame that ended the run carries what run()'s catch block pushes (pipeline.cpp:289-299):
    // TrackingLost -> not registered, default (identity) estimated pose, no fusion stats;
    // PoolExhausted -> the registration, but default FusionStats (fuse_frame threw).
    const bool died_here = f->td.dead && f->td.died_at == frame;
    const bool lost_here = died_here && f->td.status == SF_TRACKING_LOST;
    const bool exhausted_here = died_here && f->td.status == SF_POOL_EXHAUSTED;
    if (lost_here) {
        out->registered = 0;
        for (int i = 0; i < 12; ++i) out->pose[i] = (i == 0 || i == 4 || i == 8) ? 1.0 : 0.0;
    }
    if (out->registered) {
        out->iterations = f->icp.iterations;
        out->matches = f->icp.matches;
        out->residual_rms = f->icp.residual_rms;
        for (int i = 0; i < 6; ++i) {
            out->lambda_over_n[i] = f->icp.eigenvalues[i] / static_cast<double>(f->icp.pair_count);
            out->gated_mask[i] = f->icp.gated[i];
        }
    }
    const uint64_t nn = vol->P.N, m = vol->P.M;
    if (!lost_here && !exhausted_here) {
        out->fusion.voxels_updated = f->ctr.voxels_updated;
        out->fusion.blocks_allocated_now = f->ctr.alloc_now - f->ctr.alloc_before;
        out->fusion.blocks_total = f->ctr.alloc_now;
        out->fusion.memory_bytes = 2ull * f->ctr.alloc_now * m * m * m + 4ull * nn * nn * nn;
    }
    out->raycast.sample_steps = f->rs.sample_steps;
    out->raycast.hit_pixels = f->rs.hit_pixels;
    out->raycast.rays_with_bounds = f->rs.rays_with_bounds;
    out->ray_dda_cells = f->rs.dda_cells;
    out->ray_refine_samples = f->rs.refine_samples;
    out->blocks_processed = static_cast<uint64_t>(f->ctr.limit) + f->ctr.n_update;
    if (f->ctr.skip) out->blocks_processed = 0;
    out->voxels_visited = out->blocks_processed * m * m * m;
    out->exact_voxels = f->ctr.exact_voxels;
    out->integrate_ns = f->ctr.t_end > f->ctr.t_begin ? f->ctr.t_end - f->ctr.t_begin : 0;
#ifdef SF_DIAG_ICP_ASSOC  // timing diagnostics: the first step's association phase only
    out->icp_ns = f->icp.t_step0 && f->icp.t_assoc0 > f->icp.t_step0 ? f->icp.t_assoc0 - f->icp.t_step0 : 0;
#else
    out->icp_ns = f->icp.t_step0 && f->icp.t_end > f->icp.t_step0 ? f->icp.t_end - f->icp.t_step0 : 0;
#endif
    out->icp_steps = f->icp.bodies;
    out->kernel_launches = launches;
    // device-side ICP loop: one launch per iteration body (three in the reference-order mode)
    if (icp_loop) out->kernel_launches += static_cast<uint64_t>(f->icp.bodies) * (icp_prm.exact ? 3u : 1u);
}

int sf_tracker_fetch(sf_tracker_t tr, sf_frame_metrics* out, void* stream) {
    return guarded([&]() -> int {
        if (!tr || !out) throw Error(SF_INVALID_ARGUMENT, "sf_tracker_fetch: null argument");
        SF_CUDA(cudaSetDevice(tr->vol->device));
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        tr->copy_metrics(tr->h, s);
        SF_CUDA(cudaStreamSynchronize(s));
        tr->decode(tr->h, tr->frames - 1, tr->last_mode, tr->last_launches, tr->last_icp_loop, out);
        return SF_OK;
    });
}

int sf_tracker_fetch_frame(sf_tracker_t tr, int32_t frame, sf_frame_metrics* out) {
    return guarded([&]() -> int {
        if (!tr || !out) throw Error(SF_INVALID_ARGUMENT, "sf_tracker_fetch_frame: null argument");
        if (frame < 0 || frame >= tr->frames || frame < tr->frames - 2)
            throw Error(SF_OUT_OF_RANGE, "sf_tracker_fetch_frame: only the last two frames are kept");
        SF_CUDA(cudaSetDevice(tr->vol->device));
        const int slot = frame & 1;
        const auto& mt = tr->snap_meta[slot];
        SF_CUDA(cudaEventSynchronize(tr->ev_snap[slot]));
        // the device picked the snapshot slot by its own frame counter: it must be this frame's
        if (mt.frame != frame || tr->snap[slot].td.frame != frame)
            throw Error(SF_LOGIC_ERROR, "sf_tracker_fetch_frame: snapshot slot holds another frame "
                                        "(a step failed after its launch)");
        tr->decode(&tr->snap[slot], mt.frame, mt.mode, mt.launches, mt.icp_loop, out);
        return SF_OK;
    });
}

int sf_tracker_stage_times(sf_tracker_t tr, float ms[5]) {
    return guarded([&]() -> int {
        if (!tr || !ms) throw Error(SF_INVALID_ARGUMENT, "sf_tracker_stage_times: null argument");
        const int pairs[5][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 4}, {0, 5}};
        for (int i = 0; i < 5; ++i) {
            const bool have = tr->stage_events == 2 || (tr->stage_events == 1 && i == 3);
            ms[i] = -1.0f;  // stage not recorded
            if (have) SF_CUDA(cudaEventElapsedTime(&ms[i], tr->ev[pairs[i][0]], tr->ev[pairs[i][1]]));
        }
        return SF_OK;
    });
}

int sf_tracker_set_stage_timing(sf_tracker_t tr, int32_t level) {
    return guarded([&]() -> int {
        if (!tr || level < 0 || level > 2) throw Error(SF_INVALID_ARGUMENT, "sf_tracker_set_stage_timing: bad level");
        if (level == tr->stage_events) return SF_OK;
        SF_CUDA(cudaSetDevice(tr->vol->device));
        SF_CUDA(cudaDeviceSynchronize());
        for (auto& row : tr->graph)
            for (auto& g : row) {
                if (g) SF_CUDA(cudaGraphExecDestroy(g));
                g = nullptr;
            }
        tr->stage_events = level;
        return SF_OK;
    });
}

int sf_tracker_device_pose(sf_tracker_t tr, const double** device_pose) {
    return guarded([&]() -> int {
        if (!tr || !device_pose) throw Error(SF_INVALID_ARGUMENT, "sf_tracker_device_pose: null argument");
        *device_pose = tr->d_cur;
        return SF_OK;
    });
}

int sf_tracker_io_bytes(sf_tracker_t tr, int32_t has_sigma, uint64_t* h2d, uint64_t* d2h) {
    return guarded([&]() -> int {
        if (!tr || !h2d || !d2h) throw Error(SF_INVALID_ARGUMENT, "sf_tracker_io_bytes: null argument");
        const uint64_t n = static_cast<uint64_t>(tr->cam.w) * tr->cam.h;
        *h2d = n * sizeof(float) * (has_sigma ? 2 : 1);
        using F = sf_tracker::Fetch;  // the per-frame metric snapshot read back by fetch
        *d2h = sizeof(F::cur) + sizeof(F::fuse_pose) + sizeof(F::td) + sizeof(F::ctr) + sizeof(F::rs) + sizeof(F::icp);
        return SF_OK;
    });
}

int sf_tracker_last_launch_count(sf_tracker_t tr, uint64_t* count) {
    return guarded([&]() -> int {
        if (!tr || !count) throw Error(SF_INVALID_ARGUMENT, "sf_tracker_last_launch_count: null argument");
        *count = tr->last_launches;
        return SF_OK;
    });
}

}  // extern "C"

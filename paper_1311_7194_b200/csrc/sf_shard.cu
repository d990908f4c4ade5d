// sf_shard.cu — halo exchange of a spatially sharded block pool.
//
// Rank r integrates the blocks it owns (owner = hash of the 8^3-block brick, shard_owner).
// For the raycast to be exact on the union of ranks, every trilinear sample the reference
// takes near a brick face must be evaluable on the rank owning its base voxel: the stage-1
// bracket (two samples 0.5 delta apart), the secant samples between them and the six
// gradient samples (+-1 voxel) all lie within 3 voxels of that base voxel. So every rank
// mirrors, read-only, the blocks of other ranks that touch one of its bricks (26-neighbour
// adjacency, one block = M >= 4 voxels deep). After each integrate:
//   k_pack_halo   the processed blocks bordering another rank's brick -> (key, payload) records
//   (all-gather of the records across ranks: NCCL in the caller)
//   k_apply_halo  records bordering this rank's bricks -> allocated (first sight) + copied
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <vector>

#include "sf_icp.cuh"
#include "sf_internal.h"
#include "sf_linalg.cuh"
#include "sf_sample.cuh"

namespace sf {

__device__ __forceinline__ void key_xyz(const VolParams& P, int key, int& bx, int& by, int& bz) {
    bx = key % P.N;
    by = (key / P.N) % P.N;
    bz = key / (P.N * P.N);
}

// Does any of the 26 neighbours of (bx, by, bz) (inside the grid) belong to a brick of rank
// `r` (match == true) / of a rank other than `r` (match == false)? Only blocks on a brick
// face have neighbours in another brick.
__device__ bool neighbour_owner(const VolParams& P, int bx, int by, int bz, int r, bool match) {
    const int bm = (1 << P.shard_shift) - 1;
    const int fx = bx & bm, fy = by & bm, fz = bz & bm;
    if (fx != 0 && fx != bm && fy != 0 && fy != bm && fz != 0 && fz != bm) {
        // interior of its brick: all neighbours share the brick's owner
        const bool own = shard_owner(bx, by, bz, P.shard_shift, P.shard_world) == r;
        return match ? own : !own;
    }
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                if (!dx && !dy && !dz) continue;
                const int x = bx + dx, y = by + dy, z = bz + dz;
                if (x < 0 || y < 0 || z < 0 || x >= P.N || y >= P.N || z >= P.N) continue;
                const bool own = shard_owner(x, y, z, P.shard_shift, P.shard_world) == r;
                if (own == match) return true;
            }
    return false;
}

struct HaloCounters {
    unsigned int packed, applied, exhausted, pad;
};

// One warp per processed block of the last integrate (work list of fuse_frame).
__global__ void k_pack_halo(VolParams P, const int2* __restrict__ work, const FrameCounters* __restrict__ ctr,
                            const uint16_t* __restrict__ payload, int32_t* __restrict__ keys_out,
                            uint4* __restrict__ pay_out, uint64_t cap, HaloCounters* hc) {
    // (hc is zeroed by the caller; an overflow leaves packed > cap: the receivers take the
    // first cap records and the frame reports halo_overflow)
    const uint32_t limit = ctr->limit, upd_base = ctr->upd_base;
    const uint32_t n = ctr->skip ? 0u : limit + ctr->n_update;
    const int lane = threadIdx.x & 31;
    const uint32_t warps = gridDim.x * (blockDim.x / 32);
    const int vec = P.M3 / 8;  // uint4 per block (M^3 * 2 B / 16 B)
    for (uint32_t i = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; i < n; i += warps) {
        const int2 wk = i < limit ? work[i] : work[upd_base + (i - limit)];
        const uint32_t slot = static_cast<uint32_t>(wk.x) & 0x7fffffffu;
        int bx, by, bz;
        key_xyz(P, wk.y, bx, by, bz);
        uint32_t idx = 0;
        if (lane == 0) {
            idx = neighbour_owner(P, bx, by, bz, P.shard_rank, false) ? atomicAdd(&hc->packed, 1u) : 0xffffffffu;
        }
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if (idx == 0xffffffffu || idx >= cap) continue;
        if (lane == 0) keys_out[idx] = wk.y;
        const uint4* src = reinterpret_cast<const uint4*>(payload + (size_t)slot * P.M3);
        for (int j = lane; j < vec; j += 32) pay_out[(size_t)idx * vec + j] = src[j];
    }
}

// One warp per received record; records of blocks that border this rank's bricks are
// mirrored (allocated on first sight: free-list pop, table / index / occupancy update).
// n_dev (optional): the record count is the sender's device counter (min(packed, n)).
__global__ void k_apply_halo(VolParams P, const int32_t* __restrict__ keys, const uint4* __restrict__ pays,
                             uint64_t n, int32_t* __restrict__ table, const int32_t* __restrict__ free_list,
                             int32_t* __restrict__ slot_key, uint32_t* __restrict__ occ, uint16_t* __restrict__ payload,
                             VolCounters* vc, HaloCounters* hc, const HaloCounters* n_dev = nullptr,
                             const int* dead = nullptr) {
    if (dead && *dead) return;
    if (n_dev && n_dev->packed < n) n = n_dev->packed;
    const int lane = threadIdx.x & 31;
    const uint64_t warps = gridDim.x * (blockDim.x / 32);
    const int vec = P.M3 / 8;
    for (uint64_t i = blockIdx.x * (uint64_t)(blockDim.x / 32) + threadIdx.x / 32; i < n; i += warps) {
        const int key = keys[i];
        int slot = -1;
        if (lane == 0 && key >= 0 && static_cast<uint64_t>(key) < P.table_size) {
            int bx, by, bz;
            key_xyz(P, key, bx, by, bz);
            if (!shard_owns(P, bx, by, bz) && neighbour_owner(P, bx, by, bz, P.shard_rank, true)) {
                slot = table[key];
                if (slot == kEmpty) {
                    const unsigned long long top = atomicAdd(&vc->free_top, ~0ull);  // pop
                    if (top == 0) {
                        atomicAdd(&vc->free_top, 1ull);
                        atomicAdd(&hc->exhausted, 1u);
                        slot = -1;
                    } else {
                        slot = free_list[top - 1];
                        table[key] = slot;
                        slot_key[slot] = key;
                        occ_set(P, occ, static_cast<uint64_t>(key));
                        atomicAdd(&vc->allocated_count, 1ull);
                        atomicAdd(&vc->halo_count, 1ull);
                        atomicMax(&vc->high_water, static_cast<unsigned long long>(slot) + 1ull);
                    }
                }
                if (slot >= 0) atomicAdd(&hc->applied, 1u);
            }
        }
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (slot < 0) continue;
        uint4* dst = reinterpret_cast<uint4*>(payload + (size_t)slot * P.M3);
        for (int j = lane; j < vec; j += 32) dst[j] = pays[i * vec + j];
    }
}


// =========================================================================================
// Sharded fused frame: run()'s per-frame body (pipeline.cpp:233-301) over a
// block pool partitioned across ranks, issued as ONE CUDA graph per frame with the exchanges
// inside it. Ranks are either in-process (LOCAL: several volumes on this GPU, exchanges are
// kernels over their buffers; how the algorithm is tested on one B200) or one per process
// (NCCL: all-reduce / all-gather on the stream, captured into the graph). Per frame:
//   ray bounds per rank over its own blocks -> MIN/MAX all-reduce = the single-volume bounds;
//   each rank marches ONLY the rays its own bounds meet (its active list), from the global
//   bounds; nearest-depth composite; ICP on the composite, either replicated on every rank or
//   (icp_mode 1) as partial sums over pixel slices combined by an all-reduce (the north star's
//   27-float reduction); pose update; fuse per rank (owned blocks only); halo exchange of the
//   processed blocks bordering other ranks' bricks through fixed-capacity buffers (device-side
//   counts, no host synchronisation).
// =========================================================================================
constexpr int kMaxLocalRanks = 8;

struct ShardDev {
    int dead, status, registered, frame;
};
struct ShardSnapshot {  // written to mapped pinned memory by the frame's last kernel
    double pose[12];
    ShardDev sd;
    IcpState icp;
    unsigned long long voxels_updated, owned_blocks, hit_pixels, halo_records, halo_overflow, exhausted;
};
template <typename T>
struct RankArr {
    T p[kMaxLocalRanks];
};

// min of t_start / max of t_end over in-process ranks: the global ray bounds
__global__ void k_bounds_minmax_local(RankArr<const float*> ts, RankArr<const float*> te, int R, int n, float* gts,
                                      float* gte, const int* dead) {
    if (*dead) return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        float a = ts.p[0][i], b = te.p[0][i];
        for (int r = 1; r < R; ++r) {
            a = fminf(a, ts.p[r][i]);
            b = fmaxf(b, te.p[r][i]);
        }
        gts[i] = a;
        gte[i] = b;
    }
}
// Nearest-depth composite over in-process ranks: the key order of k_composite_key (depth bits,
// a rank with a normal before one without, then the lower rank); the winner's maps are copied.
__global__ void k_composite_local(RankArr<const float*> depth, RankArr<const float*> normals, int R, int n,
                                  float* out_d, float* out_n, unsigned long long* hits, const int* dead) {
    if (*dead) return;
    unsigned long long h = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        long long best = 0x7fffffffffffffffLL;
        int win = -1;
        for (int r = 0; r < R; ++r) {
            const float d = depth.p[r][i];
            if (!(d > 0.0f)) continue;
            const float* nm = normals.p[r] + 3 * i;
            const bool no_normal = nm[0] == 0.0f && nm[1] == 0.0f && nm[2] == 0.0f;
            const long long k = (static_cast<long long>(__float_as_uint(d)) << 32) |
                                (static_cast<long long>(no_normal) << 31) | static_cast<long long>(r);
            if (k < best) {
                best = k;
                win = r;
            }
        }
        if (win >= 0) {
            out_d[i] = depth.p[win][i];
            for (int c = 0; c < 3; ++c) out_n[3 * i + c] = normals.p[win][3 * i + c];
            ++h;
        } else {
            out_d[i] = 0.0f;
            out_n[3 * i] = out_n[3 * i + 1] = out_n[3 * i + 2] = 0.0f;
        }
    }
    for (int off = 16; off > 0; off >>= 1) h += __shfl_down_sync(0xffffffffu, h, off);
    if ((threadIdx.x & 31) == 0 && h) atomicAdd(hits, h);
}
// Active-ray list of the GLOBAL bounds (march_all_rays: every rank marches every bounded ray).
__global__ void k_list_from_global(const float* __restrict__ ts, const float* __restrict__ te, int n, int* list,
                                   RayCounters* ctr, const int* dead) {
    if (*dead) return;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool act = i < n && ts[i] <= te[i];
    const unsigned bal = __ballot_sync(0xffffffffu, act);
    const int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (bal) {
        const int leader = __ffs(bal) - 1;
        if (lane == leader) base = atomicAdd(&ctr->listed, static_cast<unsigned long long>(__popc(bal)));
        base = __shfl_sync(0xffffffffu, base, leader);
    }
    if (act) list[base + __popc(bal & ((1u << lane) - 1u))] = i;
}
__global__ void k_reset_listed(RankArr<RayCounters*> rs, int R) {
    if (threadIdx.x < R) rs.p[threadIdx.x]->listed = 0;
}
__global__ void k_count_hits(const float* depth, int n, unsigned long long* hits, const int* dead) {
    if (*dead) return;
    unsigned long long h = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) h += depth[i] > 0.0f;
    for (int off = 16; off > 0; off >>= 1) h += __shfl_down_sync(0xffffffffu, h, off);
    if ((threadIdx.x & 31) == 0 && h) atomicAdd(hits, h);
}

// Frame set-up of a tracked frame: initial delta (pipeline.cpp:262-267), ICP state, the
// raycast's frame constants at the current pose, per-rank ray counters zeroed.
__global__ void k_shard_begin_track(VolParams P, Intr cam, const double* __restrict__ cur,
                                    const double* __restrict__ external, double* __restrict__ init_delta,
                                    RankArr<RayCounters*> rstats, int R, ShardDev* sd, FrameConsts* fc, IcpState* icp,
                                    unsigned long long* frame_ctr) {
    if (threadIdx.x == 0) {
        if (!sd->dead) {
            const Pose c = pose_from12(cur);
            const Pose init = external ? compose(c, pose_from12(external)) : c;
            pose_to12(compose(invert(c), init), init_delta);
            sd->registered = 0;
        }
        for (int r = 0; r < R; ++r) *rstats.p[r] = RayCounters{0, 0, 0, 0, 0};
        for (int k = 0; k < 6; ++k) frame_ctr[k] = 0;
        icp_state_init(icp, init_delta, sd->dead != 0);
    }
    frame_consts_warp(P, cam, cur, fc);
}
// Pose update after ICP (pipeline.cpp:282) and the fuse pose into every rank's frame buffers.
__global__ void k_shard_after_icp(double* __restrict__ cur, double* __restrict__ fuse_pose, const IcpState* st,
                                  ShardDev* sd, int orthonormalize, RankArr<double*> rank_pose, int R) {
    if (threadIdx.x != 0 || sd->dead) return;
    if (st->lost) {
        sd->dead = 1;
        sd->status = SF_TRACKING_LOST;
        return;
    }
    Pose est = compose(pose_from12(cur), st->delta);
    if (orthonormalize) est.R = nearest_rotation(est.R);
    pose_to12(est, cur);
    pose_to12(est, fuse_pose);
    for (int r = 0; r < R; ++r) pose_to12(est, rank_pose.p[r]);
    sd->registered = 1;
}
__global__ void k_shard_begin_gt(const double* __restrict__ gt, double* __restrict__ cur, double* __restrict__ fuse_pose,
                                 ShardDev* sd, int set_current, RankArr<double*> rank_pose, int R,
                                 unsigned long long* frame_ctr) {
    if (threadIdx.x != 0) return;
    for (int k = 0; k < 6; ++k) frame_ctr[k] = 0;
    if (sd->dead) return;
    for (int i = 0; i < 12; ++i) {
        fuse_pose[i] = gt[i];
        if (set_current) cur[i] = gt[i];
    }
    for (int r = 0; r < R; ++r)
        for (int i = 0; i < 12; ++i) rank_pose.p[r][i] = gt[i];
    sd->registered = 0;
}
// After the per-rank fuse: this process's statistics into frame_ctr[0..5] = {voxels_updated,
// owned blocks, (hits), halo records, halo overflow, exhausted}; PoolExhausted ends the run.
__global__ void k_shard_fuse_done(RankArr<const FrameCounters*> ctr, RankArr<const VolCounters*> vc,
                                  RankArr<const HaloCounters*> hc, int R, unsigned long long cap,
                                  unsigned long long* frame_ctr, ShardDev* sd) {
    if (threadIdx.x != 0) return;
    unsigned long long vu = 0, owned = 0, halo = 0, over = 0, ex = 0;
    for (int r = 0; r < R; ++r) {
        vu += ctr.p[r]->voxels_updated;
        owned += vc.p[r]->allocated_count - vc.p[r]->halo_count;
        if (ctr.p[r]->exhausted) ex += 1;
        if (hc.p[r]) {
            halo += hc.p[r]->packed;
            if (hc.p[r]->packed > cap) over += hc.p[r]->packed - cap;
        }
    }
    frame_ctr[0] = vu;
    frame_ctr[1] = owned;
    frame_ctr[3] = halo;
    frame_ctr[4] = over;
    frame_ctr[5] = ex;
}
__global__ void k_shard_snapshot(ShardSnapshot* dst, const double* fuse_pose, ShardDev* sd, const IcpState* icp,
                                 const unsigned long long* frame_ctr) {
    if (threadIdx.x != 0) return;
    if (!sd->dead && frame_ctr[5]) {
        sd->dead = 1;
        sd->status = SF_POOL_EXHAUSTED;
    }
    volatile ShardSnapshot* d = dst;
    for (int i = 0; i < 12; ++i) d->pose[i] = fuse_pose[i];
    d->sd.dead = sd->dead;
    d->sd.status = sd->status;
    d->sd.registered = sd->registered;
    d->sd.frame = sd->frame;
    const unsigned long long* s = reinterpret_cast<const unsigned long long*>(icp);
    volatile unsigned long long* t = reinterpret_cast<volatile unsigned long long*>(&dst->icp);
    for (int i = 0; i < static_cast<int>(sizeof(IcpState) / 8); ++i) t[i] = s[i];
    d->voxels_updated = frame_ctr[0];
    d->owned_blocks = frame_ctr[1];
    d->hit_pixels = frame_ctr[2];
    d->halo_records = frame_ctr[3];
    d->halo_overflow = frame_ctr[4];
    d->exhausted = frame_ctr[5];
    sd->frame += 1;
}
struct Pose12Arg {
    double v[12];
};
__global__ void k_shard_set_pose(double* dst, Pose12Arg p) {
    if (threadIdx.x < 12) dst[threadIdx.x] = p.v[threadIdx.x];
}

// NCCL, resolved at run time (no link-time dependency of the library on it).
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
    const char* (*GetErrorString)(ncclResult_t);
};
static NcclApi* nccl_api() {
    static NcclApi api{};
    static bool tried = false, ok = false;
    if (!tried) {
        tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
            api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
            api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
            api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
            api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(h, "ncclAllGather"));
            api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
            ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.AllGather &&
                 api.GetErrorString;
        }
    }
    if (!ok) throw Error(SF_UNSUPPORTED, "NCCL (libnccl.so.2) is not available");
    return &api;
}
#define SF_STATUS(call)                                                    \
    do {                                                                   \
        const int rc_ = (call);                                            \
        if (rc_ != SF_OK) throw ::sf::Error(rc_, sf_last_error());         \
    } while (0)
#define SF_NCCL(call)                                                                                        \
    do {                                                                                                     \
        ncclResult_t r_ = (call);                                                                            \
        if (r_ != ncclSuccess)                                                                               \
            throw ::sf::Error(SF_CUDA_ERROR,                                                                 \
                              std::string("NCCL error ") + ::sf::nccl_api()->GetErrorString(r_) + " in " #call); \
    } while (0)

struct ShardRank {
    sf_volume* vol = nullptr;
    FrameBuffers fb;
    float *ts = nullptr, *te = nullptr, *depth = nullptr, *normals = nullptr;
    int* list = nullptr;
    RayBracket* brackets = nullptr;
    RayCounters* rstats = nullptr;
    int32_t* halo_keys = nullptr;
    uint4* halo_pays = nullptr;
    HaloCounters* hc = nullptr;      // this rank's packed-record counters
    HaloCounters* hc_in = nullptr;   // records applied from the other ranks
};

}  // namespace sf

struct sf_shard_tracker {
    int world = 1, nlocal = 1, rank0 = 0;
    bool nccl = false;
    ncclComm_t comm = nullptr;
    std::vector<std::unique_ptr<sf::ShardRank>> ranks;
    sf_shard_tracker_config cfg{};
    sf::Intr cam{};
    sf::FuseParams fp{}, fp_sigma{};
    sf::IcpParamsDev icp_prm{};
    sf::IcpWork icp;
    sf::IcpRankPartial* d_recs = nullptr;
    double *d_cur = nullptr, *d_init_delta = nullptr, *d_gt = nullptr, *d_fuse_pose = nullptr;
    sf::FrameConsts* d_rc_fc = nullptr;
    float *d_cap = nullptr, *d_cap_sigma = nullptr, *d_gts = nullptr, *d_gte = nullptr;
    float *d_comp_depth = nullptr, *d_comp_normals = nullptr;
    long long* d_key = nullptr;
    sf::ShardDev* d_sd = nullptr;
    unsigned long long* d_frame_ctr = nullptr;  // [6]
    int32_t* g_keys = nullptr;                  // NCCL: all ranks' halo records
    uint4* g_pays = nullptr;
    sf::HaloCounters* g_hc = nullptr;
    sf::ShardSnapshot* snap = nullptr;  // pinned, mapped
    sf::ShardSnapshot* snap_dev = nullptr;
    cudaStream_t capture_stream = nullptr, side_stream = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaGraphExec_t graph[3][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};
    uint64_t graph_kernels[3][2] = {};
    bool graph_icp_loop[3][2] = {};
    int frames = 0, last_mode = 0;
    uint64_t last_launches = 0;
    bool last_icp_loop = false, issue_icp_loop = false;
    int device = 0;
    bool march_all_rays = false;  // SF_SHARD_ALL_RAYS=1: every rank marches every bounded ray (A/B check)

    sf::VolParams P0() const { return ranks[0]->vol->P; }
    size_t npx() const { return static_cast<size_t>(cam.w) * cam.h; }

    template <typename T, typename F>
    sf::RankArr<T> arr(F f) const {
        sf::RankArr<T> a{};
        for (int i = 0; i < nlocal; ++i) a.p[i] = f(*ranks[i]);
        return a;
    }

    void allreduce(const void* send, void* recv, size_t n, ncclDataType_t t, ncclRedOp_t op, cudaStream_t s) {
        SF_NCCL(::sf::nccl_api()->AllReduce(send, recv, n, t, op, comm, s));
    }

    uint64_t issue(int mode, bool has_sigma, cudaStream_t s);
    ~sf_shard_tracker();
};

using namespace sf;

uint64_t sf_shard_tracker::issue(int mode, bool has_sigma, cudaStream_t s) {
    uint64_t n = 0;
    const int* dead = &d_sd->dead;
    const FuseParams& p = has_sigma ? fp_sigma : fp;
    const float* sig = has_sigma ? d_cap_sigma : nullptr;
    const int np = static_cast<int>(npx());
    const int R = nlocal;
    issue_icp_loop = false;
    auto rank_pose = arr<double*>([](ShardRank& r) { return r.fb.pose; });
    if (mode == 0 || mode == 3) {
        k_shard_begin_track<<<1, 32, 0, s>>>(P0(), cam, d_cur, mode == 3 ? d_gt : nullptr, d_init_delta,
                                             arr<RayCounters*>([](ShardRank& r) { return r.rstats; }), R, d_sd,
                                             d_rc_fc, icp.st, d_frame_ctr);
        SF_LAUNCH_CHECK();
        ++n;
        // source normals of the captured frame (ICP) on a parallel branch
        SF_CUDA(cudaEventRecord(ev_fork, s));
        SF_CUDA(cudaStreamWaitEvent(side_stream, ev_fork, 0));
        launch_compute_normals(d_cap, cam.w, cam.h, cam, cfg.base.match.normal_sigma0,
                               cfg.base.match.normal_spatial_scale, icp.src_normals, side_stream, &n, dead);
        SF_CUDA(cudaEventRecord(ev_join, side_stream));
        // 1. ray bounds over each rank's own blocks (+ its active-ray list)
        for (auto& r : ranks)
            launch_ray_bounds(*r->vol, d_rc_fc, cam, r->ts, r->te, s, &n, dead, r->list, r->rstats, r->depth,
                              r->normals);
        // 2. global bounds = MIN / MAX over the ranks
        const float *gts = ranks[0]->ts, *gte = ranks[0]->te;
        if (nccl) {
            allreduce(ranks[0]->ts, ranks[0]->ts, npx(), ncclFloat32, ncclMin, s);
            allreduce(ranks[0]->te, ranks[0]->te, npx(), ncclFloat32, ncclMax, s);
        } else if (R > 1) {
            k_bounds_minmax_local<<<148 * 4, 256, 0, s>>>(arr<const float*>([](ShardRank& r) { return r.ts; }),
                                                         arr<const float*>([](ShardRank& r) { return r.te; }), R, np,
                                                         d_gts, d_gte, dead);
            SF_LAUNCH_CHECK();
            ++n;
            gts = d_gts;
            gte = d_gte;
        }
        // 3. each rank marches only the rays its own blocks meet, from the global bounds
        if (march_all_rays) {
            k_reset_listed<<<1, 32, 0, s>>>(arr<RayCounters*>([](ShardRank& r) { return r.rstats; }), R);
            SF_LAUNCH_CHECK();
            for (auto& r : ranks) {
                k_list_from_global<<<(np + 255) / 256, 256, 0, s>>>(gts, gte, np, r->list, r->rstats, dead);
                SF_LAUNCH_CHECK();
            }
            n += 1 + R;
        }
        for (auto& r : ranks)
            launch_raycast(*r->vol, d_rc_fc, cam, gts, gte, r->depth, r->normals, r->rstats, s, &n, dead, r->list,
                           r->brackets);
        // 4. nearest-depth composite
        const float *cd = d_comp_depth, *cn = d_comp_normals;
        if (nccl) {
            SF_STATUS(sf_composite_key(ranks[0]->depth, ranks[0]->normals, npx(), rank0, reinterpret_cast<int64_t*>(d_key), s));
            allreduce(d_key, d_key, npx(), ncclInt64, ncclMin, s);
            SF_STATUS(sf_composite_select(reinterpret_cast<const int64_t*>(d_key), npx(), rank0, ranks[0]->depth, ranks[0]->normals, s));
            allreduce(ranks[0]->depth, ranks[0]->depth, npx(), ncclInt32, ncclSum, s);
            allreduce(ranks[0]->normals, ranks[0]->normals, 3 * npx(), ncclInt32, ncclSum, s);
            k_count_hits<<<148 * 2, 256, 0, s>>>(ranks[0]->depth, np, d_frame_ctr + 2, dead);
            SF_LAUNCH_CHECK();
            n += 3;
            cd = ranks[0]->depth;
            cn = ranks[0]->normals;
        } else {
            k_composite_local<<<148 * 4, 256, 0, s>>>(arr<const float*>([](ShardRank& r) { return r.depth; }),
                                                     arr<const float*>([](ShardRank& r) { return r.normals; }), R, np,
                                                     d_comp_depth, d_comp_normals, d_frame_ctr + 2, dead);
            SF_LAUNCH_CHECK();
            ++n;
        }
        SF_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
        // 5. ICP on the composite: replicated, or partial sums all-reduced
        if (cfg.icp_mode == 1) {
            auto reduce = [&](cudaStream_t bs) {
                if (!nccl) return;
                allreduce(d_recs->sums, d_recs->sums, 2 * kSums + 1, ncclFloat64, ncclSum, bs);  // sums + count
                allreduce(d_recs->box, d_recs->box, 6, ncclFloat64, ncclMin, bs);
            };
            launch_icp_ranks(icp, d_cap, icp.src_normals, cd, cn, cam, d_init_delta, icp_prm, rank0, R, world, d_recs,
                             nccl ? 1 : R, reduce, !nccl, s, &n, dead, &issue_icp_loop);
        } else {
            launch_icp(icp, d_cap, icp.src_normals, cd, cn, cam, cam, d_init_delta, icp_prm, s, &n, dead,
                       &issue_icp_loop, true);
        }
        k_shard_after_icp<<<1, 32, 0, s>>>(d_cur, d_fuse_pose, icp.st, d_sd, cfg.base.orthonormalize, rank_pose, R);
        SF_LAUNCH_CHECK();
        ++n;
    } else {
        k_shard_begin_gt<<<1, 1, 0, s>>>(d_gt, d_cur, d_fuse_pose, d_sd, mode == 1 ? 1 : 0, rank_pose, R,
                                         d_frame_ctr);
        SF_LAUNCH_CHECK();
        ++n;
    }
    // 6. fuse on every rank (owned blocks only)
    for (auto& r : ranks) launch_fuse(*r->vol, r->fb, cam, d_cap, sig, p, s, false, &n, dead);
    // 7. halo exchange
    const uint64_t cap = cfg.halo_capacity;
    const int vec = P0().M3 / 8;
    if (world > 1) {
        for (auto& r : ranks) {
            SF_CUDA(cudaMemsetAsync(r->hc, 0, sizeof(HaloCounters), s));
            SF_CUDA(cudaMemsetAsync(r->hc_in, 0, sizeof(HaloCounters), s));
            k_pack_halo<<<148 * 4, 256, 0, s>>>(r->vol->P, r->fb.work, r->fb.ctr, r->vol->d_payload, r->halo_keys,
                                                r->halo_pays, cap, r->hc);
            SF_LAUNCH_CHECK();
            ++n;
        }
        auto apply = [&](ShardRank& dst, const int32_t* keys, const uint4* pays, const HaloCounters* cnt) {
            Volume& v = *dst.vol;
            k_apply_halo<<<148 * 4, 256, 0, s>>>(v.P, keys, pays, cap, v.d_table, v.d_free_list, v.d_slot_key, v.d_occ,
                                                 v.d_payload, v.d_vc, dst.hc_in, cnt, dead);
            SF_LAUNCH_CHECK();
            ++n;
        };
        if (nccl) {
            ShardRank& r = *ranks[0];
            SF_NCCL(nccl_api()->AllGather(r.halo_keys, g_keys, cap, ncclInt32, comm, s));
            SF_NCCL(nccl_api()->AllGather(r.halo_pays, g_pays, cap * vec * 16, ncclUint8, comm, s));
            SF_NCCL(nccl_api()->AllGather(r.hc, g_hc, sizeof(HaloCounters) / 4, ncclUint32, comm, s));
            for (int q = 0; q < world; ++q)
                if (q != rank0) apply(r, g_keys + q * cap, g_pays + q * cap * vec, g_hc + q);
        } else {
            for (int i = 0; i < R; ++i)
                for (int q = 0; q < R; ++q)
                    if (q != i) apply(*ranks[i], ranks[q]->halo_keys, ranks[q]->halo_pays, ranks[q]->hc);
        }
    }
    // 8. statistics and the frame's metric snapshot
    k_shard_fuse_done<<<1, 32, 0, s>>>(arr<const FrameCounters*>([](ShardRank& r) { return r.fb.ctr; }),
                                       arr<const VolCounters*>([](ShardRank& r) { return r.vol->d_vc; }),
                                       arr<const HaloCounters*>([&](ShardRank& r) {
                                           return world > 1 ? r.hc : static_cast<HaloCounters*>(nullptr);
                                       }),
                                       R, cap, d_frame_ctr, d_sd);
    SF_LAUNCH_CHECK();
    ++n;
    if (nccl) {
        // hits are already global (composite); sum the others over the processes
        allreduce(d_frame_ctr, d_frame_ctr, 2, ncclUint64, ncclSum, s);
        allreduce(d_frame_ctr + 3, d_frame_ctr + 3, 3, ncclUint64, ncclSum, s);
    }
    k_shard_snapshot<<<1, 32, 0, s>>>(snap_dev, d_fuse_pose, d_sd, icp.st, d_frame_ctr);
    SF_LAUNCH_CHECK();
    ++n;
    return n;
}

sf_shard_tracker::~sf_shard_tracker() {
    cudaSetDevice(device);
    for (auto& row : graph)
        for (auto& g : row)
            if (g) cudaGraphExecDestroy(g);
    for (auto& r : ranks) {
        void* p[] = {r->ts, r->te, r->depth, r->normals, r->list, r->brackets, r->rstats, r->halo_keys, r->halo_pays,
                     r->hc, r->hc_in};
        for (void* q : p)
            if (q) cudaFree(q);
    }
    void* p[] = {d_recs, d_cur, d_init_delta, d_gt, d_fuse_pose, d_rc_fc, d_cap, d_cap_sigma, d_gts, d_gte,
                 d_comp_depth, d_comp_normals, d_key, d_sd, d_frame_ctr, g_keys, g_pays, g_hc};
    for (void* q : p)
        if (q) cudaFree(q);
    if (snap) cudaFreeHost(snap);
    if (capture_stream) cudaStreamDestroy(capture_stream);
    if (side_stream) cudaStreamDestroy(side_stream);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (comm) nccl_api()->CommDestroy(comm);
}

static void shard_tracker_init(sf_shard_tracker* t, const sf_shard_tracker_config* config, const double* pose) {
    const sf_tracker_config& c = config->base;
    Volume& v0 = *t->ranks[0]->vol;
    t->device = v0.device;
    t->cfg = *config;
    if (const char* e = std::getenv("SF_SHARD_ALL_RAYS")) t->march_all_rays = e[0] == '1';
    if (t->cfg.halo_capacity == 0) t->cfg.halo_capacity = 16384;
    t->cam = to_intr(c.camera);
    t->fp = resolve_fuse_params(v0, c.fusion, false);
    t->fp_sigma = resolve_fuse_params(v0, c.fusion, true);
    t->icp_prm = make_icp_params(c.match);
    if (t->icp_prm.exact) throw Error(SF_UNSUPPORTED, "sharded tracker: reference-order ICP reduction not supported");
    const int w = c.camera.width, h = c.camera.height;
    if (w <= 0 || h <= 0) throw Error(SF_INVALID_ARGUMENT, "intrinsics: non-positive image size");
    const size_t n = static_cast<size_t>(w) * h;
    t->icp.ensure(w, h);
    const uint64_t cap = t->cfg.halo_capacity;
    for (auto& rp : t->ranks) {
        ShardRank& r = *rp;
        if (r.vol->P.M3 % 8 != 0) throw Error(SF_INVALID_ARGUMENT, "sharded tracker: M^3 must be a multiple of 8");
        require_codes(*r.vol, "sharded tracker");
        ensure_frame_buffers(*r.vol, r.fb, w, h);
        SF_CUDA(cudaMalloc(&r.ts, n * sizeof(float)));
        SF_CUDA(cudaMalloc(&r.te, n * sizeof(float)));
        SF_CUDA(cudaMalloc(&r.depth, n * sizeof(float)));
        SF_CUDA(cudaMalloc(&r.normals, 3 * n * sizeof(float)));
        SF_CUDA(cudaMalloc(&r.list, n * sizeof(int)));
        SF_CUDA(cudaMalloc(&r.brackets, n * sizeof(RayBracket)));
        SF_CUDA(cudaMalloc(&r.rstats, sizeof(RayCounters)));
        SF_CUDA(cudaMemset(r.rstats, 0, sizeof(RayCounters)));
        if (t->world > 1) {
            SF_CUDA(cudaMalloc(&r.halo_keys, cap * sizeof(int32_t)));
            SF_CUDA(cudaMalloc(&r.halo_pays, cap * (r.vol->P.M3 / 8) * sizeof(uint4)));
            SF_CUDA(cudaMalloc(&r.hc, sizeof(HaloCounters)));
            SF_CUDA(cudaMalloc(&r.hc_in, sizeof(HaloCounters)));
        }
    }
    SF_CUDA(cudaMalloc(&t->d_recs, kMaxLocalRanks * sizeof(IcpRankPartial)));
    SF_CUDA(cudaMalloc(&t->d_cur, 12 * sizeof(double)));
    SF_CUDA(cudaMalloc(&t->d_init_delta, 12 * sizeof(double)));
    SF_CUDA(cudaMalloc(&t->d_gt, 12 * sizeof(double)));
    SF_CUDA(cudaMalloc(&t->d_fuse_pose, 12 * sizeof(double)));
    SF_CUDA(cudaMalloc(&t->d_rc_fc, sizeof(FrameConsts)));
    SF_CUDA(cudaMalloc(&t->d_cap, n * sizeof(float)));
    SF_CUDA(cudaMalloc(&t->d_cap_sigma, n * sizeof(float)));
    SF_CUDA(cudaMalloc(&t->d_gts, n * sizeof(float)));
    SF_CUDA(cudaMalloc(&t->d_gte, n * sizeof(float)));
    SF_CUDA(cudaMalloc(&t->d_comp_depth, n * sizeof(float)));
    SF_CUDA(cudaMalloc(&t->d_comp_normals, 3 * n * sizeof(float)));
    SF_CUDA(cudaMalloc(&t->d_key, n * sizeof(long long)));
    SF_CUDA(cudaMalloc(&t->d_sd, sizeof(ShardDev)));
    SF_CUDA(cudaMemset(t->d_sd, 0, sizeof(ShardDev)));
    SF_CUDA(cudaMalloc(&t->d_frame_ctr, 8 * sizeof(unsigned long long)));
    SF_CUDA(cudaMemset(t->d_frame_ctr, 0, 8 * sizeof(unsigned long long)));
    if (t->nccl && t->world > 1) {
        const int vec = v0.P.M3 / 8;
        SF_CUDA(cudaMalloc(&t->g_keys, t->world * cap * sizeof(int32_t)));
        SF_CUDA(cudaMalloc(&t->g_pays, t->world * cap * vec * sizeof(uint4)));
        SF_CUDA(cudaMalloc(&t->g_hc, t->world * sizeof(HaloCounters)));
    }
    SF_CUDA(cudaMemcpy(t->d_cur, pose, 12 * sizeof(double), cudaMemcpyHostToDevice));
    SF_CUDA(cudaMallocHost(&t->snap, sizeof(ShardSnapshot)));
    std::memset(t->snap, 0, sizeof(ShardSnapshot));
    SF_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&t->snap_dev), t->snap, 0));
    SF_CUDA(cudaStreamCreateWithFlags(&t->side_stream, cudaStreamNonBlocking));
    SF_CUDA(cudaEventCreateWithFlags(&t->ev_fork, cudaEventDisableTiming));
    SF_CUDA(cudaEventCreateWithFlags(&t->ev_join, cudaEventDisableTiming));
}

extern "C" {

int sf_shard_pack_halo(sf_volume_t v, int32_t* keys, uint16_t* payloads, uint64_t cap, uint32_t* count,
                       void* stream) {
    return guarded([&]() -> int {
        if (v) require_codes(*v, "shard halo");
        if (!v || !count || (cap && (!keys || !payloads))) throw Error(SF_INVALID_ARGUMENT, "sf_shard_pack_halo: null");
        if (v->P.shard_world <= 1) throw Error(SF_LOGIC_ERROR, "sf_shard_pack_halo: volume is not sharded");
        if (v->P.M3 % 8 != 0) throw Error(SF_INVALID_ARGUMENT, "sf_shard_pack_halo: M^3 must be a multiple of 8");
        if (!v->fb.ctr) throw Error(SF_LOGIC_ERROR, "sf_shard_pack_halo: no integrate on this volume yet");
        SF_CUDA(cudaSetDevice(v->device));
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        HaloCounters* hc = nullptr;
        SF_CUDA(cudaMallocAsync(&hc, sizeof(HaloCounters), s));
        SF_CUDA(cudaMemsetAsync(hc, 0, sizeof(HaloCounters), s));
        k_pack_halo<<<148 * 4, 256, 0, s>>>(v->P, v->fb.work, v->fb.ctr, v->d_payload, keys,
                                            reinterpret_cast<uint4*>(payloads), cap, hc);
        SF_LAUNCH_CHECK();
        HaloCounters h{};
        SF_CUDA(cudaMemcpyAsync(&h, hc, sizeof(h), cudaMemcpyDeviceToHost, s));
        SF_CUDA(cudaFreeAsync(hc, s));
        SF_CUDA(cudaStreamSynchronize(s));
        *count = h.packed;
        if (h.packed > cap) throw Error(SF_OUT_OF_RANGE, "sf_shard_pack_halo: record capacity too small");
        return SF_OK;
    });
}

int sf_shard_apply_halo(sf_volume_t v, const int32_t* keys, const uint16_t* payloads, uint64_t n, uint32_t* applied,
                        void* stream) {
    return guarded([&]() -> int {
        if (!v || (n && (!keys || !payloads))) throw Error(SF_INVALID_ARGUMENT, "sf_shard_apply_halo: null");
        if (v->P.shard_world <= 1) throw Error(SF_LOGIC_ERROR, "sf_shard_apply_halo: volume is not sharded");
        SF_CUDA(cudaSetDevice(v->device));
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        HaloCounters* hc = nullptr;
        SF_CUDA(cudaMallocAsync(&hc, sizeof(HaloCounters), s));
        SF_CUDA(cudaMemsetAsync(hc, 0, sizeof(HaloCounters), s));
        if (n) {
            k_apply_halo<<<148 * 4, 256, 0, s>>>(v->P, keys, reinterpret_cast<const uint4*>(payloads), n, v->d_table,
                                                 v->d_free_list, v->d_slot_key, v->d_occ, v->d_payload, v->d_vc, hc);
            SF_LAUNCH_CHECK();
        }
        HaloCounters h{};
        SF_CUDA(cudaMemcpyAsync(&h, hc, sizeof(h), cudaMemcpyDeviceToHost, s));
        SF_CUDA(cudaFreeAsync(hc, s));
        SF_CUDA(cudaStreamSynchronize(s));
        if (applied) *applied = h.applied;
        if (h.exhausted)
            throw Error(SF_POOL_EXHAUSTED, "grid: payload pool exhausted (" + std::to_string(v->P.capacity) +
                                               " blocks) while mirroring halo blocks");
        return SF_OK;
    });
}


int sf_nccl_unique_id(uint8_t out[128]) {
    return guarded([&]() -> int {
        if (!out) throw Error(SF_INVALID_ARGUMENT, "sf_nccl_unique_id: null");
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
        ncclUniqueId id;
        SF_NCCL(nccl_api()->GetUniqueId(&id));
        std::memcpy(out, &id, sizeof(id));
        return SF_OK;
    });
}

int sf_shard_tracker_create_local(sf_volume_t* volumes, int32_t count, const sf_shard_tracker_config* config,
                                  const double initial_pose[12], sf_shard_tracker_t* out) {
    return guarded([&]() -> int {
        if (!volumes || !config || !initial_pose || !out || count < 1)
            throw Error(SF_INVALID_ARGUMENT, "sf_shard_tracker_create_local: null argument");
        if (count > kMaxLocalRanks) throw Error(SF_INVALID_ARGUMENT, "sf_shard_tracker_create_local: at most 8 ranks");
        auto t = std::make_unique<sf_shard_tracker>();
        t->world = count;
        t->nlocal = count;
        for (int i = 0; i < count; ++i) {
            if (!volumes[i]) throw Error(SF_INVALID_ARGUMENT, "sf_shard_tracker_create_local: null volume");
            const VolParams& P = volumes[i]->P;
            if (count > 1 && (P.shard_world != count || P.shard_rank != i))
                throw Error(SF_INVALID_ARGUMENT,
                            "sf_shard_tracker_create_local: volume i must be sharded as rank i of count");
            if (volumes[i]->device != volumes[0]->device)
                throw Error(SF_INVALID_ARGUMENT, "sf_shard_tracker_create_local: volumes on different devices");
            auto r = std::make_unique<ShardRank>();
            r->vol = volumes[i];
            t->ranks.push_back(std::move(r));
        }
        SF_CUDA(cudaSetDevice(volumes[0]->device));
        shard_tracker_init(t.get(), config, initial_pose);
        *out = t.release();
        return SF_OK;
    });
}

int sf_shard_tracker_create_nccl(sf_volume_t volume, const uint8_t nccl_id[128], int32_t rank, int32_t world,
                                 const sf_shard_tracker_config* config, const double initial_pose[12],
                                 sf_shard_tracker_t* out) {
    return guarded([&]() -> int {
        if (!volume || !nccl_id || !config || !initial_pose || !out)
            throw Error(SF_INVALID_ARGUMENT, "sf_shard_tracker_create_nccl: null argument");
        if (world < 1 || rank < 0 || rank >= world)
            throw Error(SF_INVALID_ARGUMENT, "sf_shard_tracker_create_nccl: need 0 <= rank < world");
        if (world > 1 && (volume->P.shard_world != world || volume->P.shard_rank != rank))
            throw Error(SF_INVALID_ARGUMENT, "sf_shard_tracker_create_nccl: the volume must be sharded as rank of world");
        auto t = std::make_unique<sf_shard_tracker>();
        t->world = world;
        t->nlocal = 1;
        t->rank0 = rank;
        t->nccl = true;
        auto r = std::make_unique<ShardRank>();
        r->vol = volume;
        t->ranks.push_back(std::move(r));
        SF_CUDA(cudaSetDevice(volume->device));
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        SF_NCCL(nccl_api()->CommInitRank(&t->comm, world, id, rank));
        shard_tracker_init(t.get(), config, initial_pose);
        *out = t.release();
        return SF_OK;
    });
}

int sf_shard_tracker_destroy(sf_shard_tracker_t tr) {
    delete tr;
    return SF_OK;
}

int sf_shard_tracker_step(sf_shard_tracker_t tr, const sf_frame* captured, int32_t mode, const double gt_pose[12],
                          void* stream) {
    return guarded([&]() -> int {
        if (!tr || !captured) throw Error(SF_INVALID_ARGUMENT, "sf_shard_tracker_step: null argument");
        if (captured->intrinsics.width != tr->cam.w || captured->intrinsics.height != tr->cam.h)
            throw Error(SF_INVALID_ARGUMENT, "sf_shard_tracker_step: frame size differs from the tracker camera");
        if ((mode == 1 || mode == 2) && !gt_pose)
            throw Error(SF_INVALID_ARGUMENT, "sf_shard_tracker_step: this mode needs a pose argument");
        if (mode < 0 || mode > 2) throw Error(SF_INVALID_ARGUMENT, "sf_shard_tracker_step: unknown mode");
        SF_CUDA(cudaSetDevice(tr->device));
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const size_t n = tr->npx();
        const bool has_sigma = captured->sigma != nullptr;
        const cudaMemcpyKind k = captured->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        SF_CUDA(cudaMemcpyAsync(tr->d_cap, captured->depth, n * sizeof(float), k, s));
        if (has_sigma) SF_CUDA(cudaMemcpyAsync(tr->d_cap_sigma, captured->sigma, n * sizeof(float), k, s));
        int eff = mode == 2 ? 3 : mode;
        if (mode != 1 && tr->frames == 0) eff = 2;  // first frame: fuse at the current pose (pipeline.cpp:250-252)
        uint64_t extra = 0;
        if (eff == 1 || eff == 3) {
            Pose12Arg g;
            for (int i = 0; i < 12; ++i) g.v[i] = gt_pose[i];
            k_shard_set_pose<<<1, 32, 0, s>>>(tr->d_gt, g);
            SF_LAUNCH_CHECK();
            extra = 1;
        }
        if (eff == 2) SF_CUDA(cudaMemcpyAsync(tr->d_gt, tr->d_cur, 12 * sizeof(double), cudaMemcpyDeviceToDevice, s));
        const int gmode = eff == 0 ? 0 : eff == 1 ? 1 : 2;
        const int sidx = has_sigma ? 1 : 0;
        if (tr->cfg.base.use_graphs && eff != 2) {
            cudaGraphExec_t& ge = tr->graph[gmode][sidx];
            if (!ge) {
                if (!tr->capture_stream) SF_CUDA(cudaStreamCreateWithFlags(&tr->capture_stream, cudaStreamNonBlocking));
                cudaStream_t cs = tr->capture_stream;
                cudaGraph_t g;
                uint64_t issued = 0;
                SF_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
                try {
                    issued = tr->issue(eff, has_sigma, cs);
                } catch (...) {
                    cudaStreamEndCapture(cs, &g);
                    throw;
                }
                SF_CUDA(cudaStreamEndCapture(cs, &g));
                SF_CUDA(cudaGraphInstantiate(&ge, g, 0));
                SF_CUDA(cudaGraphDestroy(g));
                tr->graph_kernels[gmode][sidx] = issued;
                tr->graph_icp_loop[gmode][sidx] = tr->issue_icp_loop;
            }
            SF_CUDA(cudaGraphLaunch(ge, s));
            tr->last_launches = tr->graph_kernels[gmode][sidx] + extra;
            tr->last_icp_loop = tr->graph_icp_loop[gmode][sidx];
        } else {
            tr->last_launches = tr->issue(eff, has_sigma, s) + extra;
            tr->last_icp_loop = tr->issue_icp_loop;
        }
        tr->last_mode = eff;
        ++tr->frames;
        return SF_OK;
    });
}

int sf_shard_tracker_set_pose(sf_shard_tracker_t tr, const double pose[12], void* stream) {
    return guarded([&]() -> int {
        if (!tr || !pose) throw Error(SF_INVALID_ARGUMENT, "sf_shard_tracker_set_pose: null argument");
        SF_CUDA(cudaSetDevice(tr->device));
        Pose12Arg g;
        for (int i = 0; i < 12; ++i) g.v[i] = pose[i];
        k_shard_set_pose<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(tr->d_cur, g);
        SF_LAUNCH_CHECK();
        return SF_OK;
    });
}

int sf_shard_tracker_fetch(sf_shard_tracker_t tr, sf_shard_frame_metrics* out, void* stream) {
    return guarded([&]() -> int {
        if (!tr || !out) throw Error(SF_INVALID_ARGUMENT, "sf_shard_tracker_fetch: null argument");
        SF_CUDA(cudaSetDevice(tr->device));
        SF_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
        const ShardSnapshot& f = *tr->snap;
        std::memset(out, 0, sizeof(*out));
        out->frame = tr->frames - 1;
        out->status = f.sd.status;
        const bool tracked = tr->last_mode == 0 || tr->last_mode == 3;
        out->registered = tracked ? f.sd.registered : 0;
        std::memcpy(out->pose, f.pose, sizeof(out->pose));
        if (out->registered) {
            out->iterations = f.icp.iterations;
            out->matches = f.icp.matches;
        }
        out->voxels_updated = f.voxels_updated;
        out->blocks_total = f.owned_blocks;
        out->hit_pixels = f.hit_pixels;
        out->halo_records = f.halo_records;
        out->halo_overflow = f.halo_overflow;
        out->icp_steps = tracked ? f.icp.bodies : 0;
        out->kernel_launches = tr->last_launches;
        if (tr->last_icp_loop && tracked)
            out->kernel_launches += static_cast<uint64_t>(f.icp.bodies) *
                                    (tr->cfg.icp_mode == 1 ? static_cast<uint64_t>(tr->nlocal) + 1 : 1u);
        return SF_OK;
    });
}

}  // extern "C"

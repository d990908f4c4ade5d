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
#include "sf_internal.h"

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
__global__ void k_apply_halo(VolParams P, const int32_t* __restrict__ keys, const uint4* __restrict__ pays,
                             uint64_t n, int32_t* __restrict__ table, const int32_t* __restrict__ free_list,
                             int32_t* __restrict__ slot_key, uint32_t* __restrict__ occ, uint16_t* __restrict__ payload,
                             VolCounters* vc, HaloCounters* hc) {
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

}  // namespace sf

using namespace sf;

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

}  // extern "C"

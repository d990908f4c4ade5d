// sf_fusion.cu — fuse_frame on the device (fusion.cpp:25-376, grid.cpp:174-269).
//
// Per frame (all launches asynchronous, no host round trip):
//   k_frame_consts     1 thread: camera_from_world, frustum SAT axes + intervals   (grid.cpp:228-259)
//   k_normals          compute_normals with the fusion options                     (camera.cpp:44-76, fusion.cpp:33-36)
//   k_edge             depth-edge mask                                              (fusion.cpp:40-62)
//   k_pixel_meas       5x5 near-edge dilation + every per-pixel factor of the
//                      measurement (sigma, p_k, w_k, grazing reject)                (fusion.cpp:63-70, 148-171)
//   k_block_keys_set   surface samples -> block keys (FP64), deduplicated in an N^3-bit set,
//                      new keys (EMPTY in the table) split off                     (fusion.cpp:190-206)
//   k_alloc_visible    ordered slot assignment (rank among the new keys == position in
//                      std::set<BlockLess> order == sequential free-list pops; PoolExhausted
//                      key / prefix semantics; fusion.cpp:294-299,369; grid.cpp:87-100)
//                      beside the SAT frustum test + 9 probes over the other allocated
//                      blocks (grid.cpp:174-269; fusion.cpp:211-233)
//   (select_update_blocks exports the ordered lists: k_block_keys, CUB radix sort +
//    unique == std::set order (fusion.cpp:177-183,193), k_visible)
//   k_integrate        per voxel: project, band test, filter, quantize              (fusion.cpp:81-173, 237-272, 300-364)
//   k_fuse_finalize    FusionStats                                                  (fusion.cpp:372-375)
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <vector>

#include "sf_internal.h"
#include "sf_sample.cuh"

#include <type_traits>

namespace sf {

constexpr int kThreads = 256;
constexpr int kPersistentCtas = 148 * 8;
#ifndef SF_ALLOC_CTAS
#define SF_ALLOC_CTAS (148 * 4)
#endif
constexpr int kAllocCtas = SF_ALLOC_CTAS;  // k_alloc_visible: rank CTAs + visibility CTAs (last-CTA epilogue)

// ---------------------------------------------------------------------------------
// frame setup (one warp: hull points, corner rays and SAT axes computed lane-parallel)
// ---------------------------------------------------------------------------------
__global__ void k_frame_consts(VolParams P, Intr intr, const double* __restrict__ pose12, FrameConsts* fc) {
    if (blockIdx.x != 0) return;
    frame_consts_warp(P, intr, pose12, fc);
}

// Zero the per-frame counters; a set dead flag (tracker: tracking lost / pool exhausted
// earlier) turns every later kernel of the frame into a no-op.
__global__ void k_fuse_begin(FrameCounters* ctr, const VolCounters* vc, const int* dead) { fuse_begin_body(ctr, vc, dead); }

// ---------------------------------------------------------------------------------
// frame preparation
// ---------------------------------------------------------------------------------
__device__ __forceinline__ bool px_valid(const float* depth, int w, int h, int u, int v) {
    return u >= 0 && v >= 0 && u < w && v < h && depth[(size_t)v * w + u] > 0.0f;
}

// compute_normals (camera.cpp:44-76)
__global__ void k_normals(const float* __restrict__ depth, int w, int h, Intr intr, double sigma0, double spatial,
                          float* __restrict__ normals, const int* dead) {
    if (dead && *dead) return;
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    const int v = blockIdx.y * blockDim.y + threadIdx.y;
    if (u >= w || v >= h) return;
    float* out = normals + 3 * ((size_t)v * w + u);
    float nx = 0.f, ny = 0.f, nz = 0.f;
    if (u >= 1 && u + 1 < w && v >= 1 && v + 1 < h) {
        const float z = px_valid(depth, w, h, u, v) ? depth[(size_t)v * w + u] : 0.0f;
        if (z > 0.0f) {
            const float zl = depth[(size_t)v * w + u - 1];
            const float zr = depth[(size_t)v * w + u + 1];
            const float zu = depth[(size_t)(v - 1) * w + u];
            const float zd = depth[(size_t)(v + 1) * w + u];
            if (!(zl <= 0.0f || zr <= 0.0f || zu <= 0.0f || zd <= 0.0f)) {
                const double threshold = 3.0 * sigma0 * double(z) * double(z) + 2.0 * spatial;
                if (!(fabsf(zl - z) > threshold || fabsf(zr - z) > threshold || fabsf(zu - z) > threshold ||
                      fabsf(zd - z) > threshold)) {
                    const d3 du = sub(unproject(intr, u + 1, v, zr), unproject(intr, u - 1, v, zl));
                    const d3 dv = sub(unproject(intr, u, v + 1, zd), unproject(intr, u, v - 1, zu));
                    d3 n = cross(du, dv);
                    const double len = sqrt(sqnorm(n));
                    if (len > 0.0) {
                        n = divs(n, len);
                        if (dot(n, unproject(intr, u, v, z)) > 0.0) n = neg(n);
                        nx = (float)n.x;
                        ny = (float)n.y;
                        nz = (float)n.z;
                    }
                }
            }
        }
    }
    out[0] = nx;
    out[1] = ny;
    out[2] = nz;
}

// Edge mask (fusion.cpp:44-62)
__global__ void k_edge(const float* __restrict__ depth, int w, int h, double sigma0, uint8_t* __restrict__ edge,
                       const int* dead) {
    if (dead && *dead) return;
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    const int v = blockIdx.y * blockDim.y + threadIdx.y;
    if (u >= w || v >= h) return;
    uint8_t e = 0;
    if (!px_valid(depth, w, h, u, v)) {
        e = 1;
    } else {
        const float z = depth[(size_t)v * w + u];
        const double jump = 3.0 * sigma0 * double(z) * double(z) + 0.02 * double(z);
        bool is_edge = u == 0 || v == 0 || u == w - 1 || v == h - 1;
        for (int k = 0; !is_edge && k < 4; ++k) {
            const int nu = u + (k == 0 ? 1 : k == 1 ? -1 : 0);
            const int nv = v + (k == 2 ? 1 : k == 3 ? -1 : 0);
            if (!px_valid(depth, w, h, nu, nv) || fabsf(depth[(size_t)nv * w + nu] - z) > jump) is_edge = true;
        }
        e = is_edge ? 1 : 0;
    }
    edge[(size_t)v * w + u] = e;
}

// Per-pixel measurement factors (fusion.cpp:148-171) + near-edge dilation (fusion.cpp:63-70).
// Everything after the band test in estimate_measurement depends only on the chosen pixel.
__global__ void k_pixel_meas(const float* __restrict__ depth, const float* __restrict__ sigma, int w, int h,
                             Intr intr, FuseParams fp, const float* __restrict__ normals,
                             const uint8_t* __restrict__ edge, double* __restrict__ pix_var,
                             double* __restrict__ pix_w, uint8_t* __restrict__ pix_ok, double* __restrict__ pix_dm,
                             float2* __restrict__ pix_f, double* __restrict__ pix_q, const int* dead) {
    if (dead && *dead) return;
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    const int v = blockIdx.y * blockDim.y + threadIdx.y;
    if (u >= w || v >= h) return;
    const size_t idx = (size_t)v * w + u;
    uint8_t ok = 0;
    double var = 0.0, wk = 0.0, qual = 1.0;
    if (px_valid(depth, w, h, u, v)) {
        const double measured = depth[idx];
        const double sg = fp.has_sigma && sigma[idx] > 0.0f ? static_cast<double>(sigma[idx])
                                                             : fp.sigma0 * measured * measured;
        var = dmax(sg * sg, fp.min_variance);
        wk = fp.w_fixed;
        ok = 1;
        if (fp.downweight) {
            double quality = 0.3;
            const float fx = normals[3 * idx], fy = normals[3 * idx + 1], fz = normals[3 * idx + 2];
            if ((fx * fx + fy * fy) + fz * fz > 0.0f) {
                const d3 ray = normalized(unproject(intr, u, v, 1.0));
                quality = fabs(dot(mk((double)fx, (double)fy, (double)fz), ray));
            }
            bool near = false;
            for (int dv = -2; !near && dv <= 2; ++dv)
                for (int du = -2; !near && du <= 2; ++du) {
                    const int nu = u + du, nv = v + dv;
                    if (nu >= 0 && nv >= 0 && nu < w && nv < h && edge[(size_t)nv * w + nu]) near = true;
                }
            if (near) quality *= 0.5;
            qual = quality;
            if (quality < 0.2) {
                ok = 0;
            } else {
                wk *= quality;
                var /= quality;
            }
        }
    }
    pix_var[idx] = var;
    pix_q[idx] = qual;
    pix_w[idx] = wk;
    pix_ok[idx] = ok;
    pix_dm[idx] = ok ? (double)depth[idx] : 0.0;
    pix_f[idx] = make_float2(ok ? depth[idx] : 0.0f, static_cast<float>(fp.mode == 2 ? var : wk));
}

// ---------------------------------------------------------------------------------
// block keys, allocation
// ---------------------------------------------------------------------------------
__global__ void k_block_keys(VolParams P, const FrameConsts* __restrict__ fc, const float* __restrict__ depth,
                             int w, int h, int stride, int su, int sv, uint32_t* __restrict__ keys, uint32_t sentinel,
                             const uint32_t* skip) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= su * sv) return;
    uint32_t k0 = sentinel, k1 = sentinel, k2 = sentinel;
    const int u = (i % su) * stride;
    const int v = (i / su) * stride;
    if (!*skip && px_valid(depth, w, h, u, v)) {
        const Intr& intr = fc->intr;
        const Pose& pose = fc->pose;
        const d3 dir_cam = normalized(unproject(intr, u, v, 1.0));
        const d3 dir = mv(pose.R, dir_cam);
        const double t_hit = (double)depth[(size_t)v * w + u] / dir_cam.z;
        const double offs[3] = {-fc->delta, 0.0, fc->delta};
        uint32_t out[3];
        for (int k = 0; k < 3; ++k) {
            const d3 x = add(pose.t, scale(t_hit + offs[k], dir));
            // block_of_point (grid.cpp:283-287)
            const int bx = ref_floor_int((x.x - P.ox) / P.block_side);
            const int by = ref_floor_int((x.y - P.oy) / P.block_side);
            const int bz = ref_floor_int((x.z - P.oz) / P.block_side);
            const bool in = bx >= 0 && by >= 0 && bz >= 0 && bx < P.N && by < P.N && bz < P.N && shard_owns(P, bx, by, bz);
            out[k] = in ? static_cast<uint32_t>(table_index(P, bx, by, bz)) : sentinel;
        }
        k0 = out[0];
        k1 = out[1];
        k2 = out[2];
    }
    keys[3 * i + 0] = k0;
    keys[3 * i + 1] = k1;
    keys[3 * i + 2] = k2;
}

__global__ void k_list_len(FrameCounters* ctr, const uint32_t* __restrict__ uniq, uint32_t sentinel) {
    const uint32_t n = ctr->n_unique;
    const uint32_t len = (n > 0 && uniq[n - 1] == sentinel) ? n - 1 : n;
    ctr->n_list = len;
    ctr->limit = len;
}

// ---------------------------------------------------------------------------------
// Fuse-path allocation without a global sort.
//
// Only two things depend on the ORDER of the reference's std::set allocate list: which slot
// a new block receives (the r-th new key in (z,y,x) order takes the r-th pop of the free
// list) and, on PoolExhausted, which prefix of the list is processed (keys below the first
// unallocatable one). Integration itself is per block and order-free. So the keys are
// deduplicated through an N^3-bit set (atomicOr), the new ones are ranked among themselves
// by counting (rank = #{new keys < k}: exact, deterministic, O(n_new^2 / threads) and
// n_new is small after the first frame), and the work list is built in any order.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t warp_append(bool pred, uint32_t* counter) {
    const unsigned am = __activemask();
    const unsigned bal = __ballot_sync(am, pred);
    const int lane = threadIdx.x & 31;
    uint32_t base = 0;
    if (bal) {
        const int leader = __ffs(bal) - 1;
        if (lane == leader) base = atomicAdd(counter, static_cast<uint32_t>(__popc(bal)));
        base = __shfl_sync(am, base, leader);
    }
    return base + __popc(bal & ((1u << lane) - 1u));
}

// block_of_point keys of the surface samples (fusion.cpp:187-209), deduplicated in the key set.
// The first inserter of a key also classifies it: an existing block's work item is written
// at once (item j = its position in the unordered allocate set); a new key (EMPTY table
// entry) is appended to the new-key list with j, and gets its slot in k_alloc_visible.
__global__ void k_block_keys_set(VolParams P, const FrameConsts* __restrict__ fc, const float* __restrict__ depth,
                                 int w, int h, int stride, int su, int sv, uint32_t* __restrict__ keybits,
                                 uint32_t* __restrict__ uniq, FrameCounters* ctr, const int32_t* __restrict__ table,
                                 uint32_t* __restrict__ new_keys, uint32_t* __restrict__ new_idx,
                                 int2* __restrict__ work) {
    pdl_wait();
    if (ctr->skip) return;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool in_range = i < su * sv;
    const int u = in_range ? (i % su) * stride : 0;
    const int v = in_range ? (i / su) * stride : 0;
    const bool valid = in_range && px_valid(depth, w, h, u, v);
    d3 dir = mk(0, 0, 0);
    double t_hit = 0.0;
    if (valid) {
        const Intr& intr = fc->intr;
        const d3 dir_cam = normalized(unproject(intr, u, v, 1.0));
        dir = mv(fc->pose.R, dir_cam);
        t_hit = (double)depth[(size_t)v * w + u] / dir_cam.z;
    }
    // (x - origin) / block_side correctly rounded: RN(1/b) product + one fma-residual step
    // (Markstein), as the reference's division (grid.cpp:283-287)
    auto div_block = [&](double a) {
        const double q = a * P.inv_block_side;
        return fma(fma(-q, P.block_side, a), P.inv_block_side, q);
    };
    const double offs[3] = {-fc->delta, 0.0, fc->delta};
    uint32_t keys[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        keys[k] = 0xffffffffu;
        if (valid) {
            const d3 x = add(fc->pose.t, scale(t_hit + offs[k], dir));
            const int bx = ref_floor_int(div_block(x.x - P.ox));
            const int by = ref_floor_int(div_block(x.y - P.oy));
            const int bz = ref_floor_int(div_block(x.z - P.oz));
            if (bx >= 0 && by >= 0 && bz >= 0 && bx < P.N && by < P.N && bz < P.N && shard_owns(P, bx, by, bz))
                keys[k] = static_cast<uint32_t>(table_index(P, bx, by, bz));
        }
    }
    // the three insertions, then the fresh keys' table reads, are independent of each other
    bool fresh[3];
    int32_t slot[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        fresh[k] = false;
        if (keys[k] != 0xffffffffu) {
            const uint32_t bit = 1u << (keys[k] & 31);
            fresh[k] = !(atomicOr(&keybits[keys[k] >> 5], bit) & bit);
        }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) slot[k] = fresh[k] ? table[keys[k]] : kEmpty;
    // one warp-wide reservation per list: inclusive scan of {fresh count, new count}
    uint32_t nf = 0, nn = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        nf += fresh[k] ? 1u : 0u;
        nn += (fresh[k] && slot[k] == kEmpty) ? 1u : 0u;
    }
    uint32_t sc = nf | (nn << 16);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, sc, off);
        if (lane >= off) sc += o;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, sc, 31);
    uint32_t base_f = 0, base_n = 0;
    if (lane == 0 && (tot & 0xffffu)) base_f = atomicAdd(&ctr->n_unique, tot & 0xffffu);
    if (lane == 1 && (tot >> 16)) base_n = atomicAdd(&ctr->n_new, tot >> 16);
    base_f = __shfl_sync(0xffffffffu, base_f, 0);
    base_n = __shfl_sync(0xffffffffu, base_n, 1);
    uint32_t j = base_f + (sc & 0xffffu) - nf, q = base_n + (sc >> 16) - nn;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (!fresh[k]) continue;
        const uint32_t key = keys[k];
        uniq[j] = key;
        if (slot[k] == kEmpty) {
            new_keys[q] = key;
            new_idx[q] = j;
            work[j] = make_int2(static_cast<int32_t>(0x80000000u), static_cast<int32_t>(key));
            ++q;
        } else {
            work[j] = make_int2(slot[k], static_cast<int32_t>(key));
        }
        ++j;
    }
}

// Conservative: the block's bounding sphere lies strictly inside the frustum (margins far
// above rounding), hence the exact SAT (grid.cpp:228-269) would report an intersection.
__device__ __forceinline__ bool block_surely_inside(const VolParams& P, const FrameConsts* __restrict__ fc, d3 lo) {
    const double hs = 0.5 * P.block_side;
    const d3 c = apply(fc->inv, add(lo, mk(hs, hs, hs)));
    const double r = hs * 1.7320508075688772 * (1.0 + 1e-9) + 1e-12;
    if (!(c.z - r > fc->intr.near_plane * (1.0 + 1e-9) && c.z + r < fc->intr.far_plane * (1.0 - 1e-9))) return false;
#pragma unroll
    for (int f = 0; f < 4; ++f)
        if (!(dot(fc->side_n[f], c) > r)) return false;
    return true;
}

// Visible allocated blocks outside the allocate set (membership from the key set): exact
// frustum SAT + 9 probes (grid.cpp:174-269; fusion.cpp:211-233).
__device__ __forceinline__ bool block_visible(const VolParams& P, const FrameConsts* __restrict__ fc, int32_t key,
                                              const float* __restrict__ depth, int w, int h) {
    int bx, by, bz;
    if (P.nshift >= 0) {
        bx = key & (P.N - 1);
        by = (key >> P.nshift) & (P.N - 1);
        bz = key >> (2 * P.nshift);
    } else {
        bx = key % P.N;
        by = (key / P.N) % P.N;
        bz = key / (P.N * P.N);
    }
    const d3 lo = block_min_corner(P, bx, by, bz);
    const double side = P.block_side;
    const d3 hi = add(lo, mk(side, side, side));
    // a sharded volume integrates only its own blocks (mirrored halo blocks are read-only)
    if (!shard_owns(P, bx, by, bz) || !(block_surely_inside(P, fc, lo) || frustum_intersects_block(P, fc, lo, hi)))
        return false;
    const Intr& intr = fc->intr;
    for (int k = 0; k < 9; ++k) {
        const d3 probe = k == 8 ? add(lo, mk(0.5 * side, 0.5 * side, 0.5 * side))
                                : add(lo, mk(k & 1 ? side : 0.0, k & 2 ? side : 0.0, k & 4 ? side : 0.0));
        const d3 xc = apply(fc->inv, probe);
        double pu, pv;
        if (!project(intr, xc, pu, pv)) continue;
        const int u = ref_lround_int(pu);
        const int v = ref_lround_int(pv);
        if (!(u >= 0 && v >= 0 && u < w && v < h)) continue;
        const float d = depth[(size_t)v * w + u];
        if (!(d > 0.0f) || xc.z <= d + fc->delta) return true;
    }
    return false;
}

// One launch, two roles, then a last-CTA epilogue:
//  - CTAs [0, kRankCtas): ordered slots for the new keys. rank = #{new keys < key} (one warp
//    per kRankKeys keys, lanes over the list) is the key's position among the new keys in
//    std::set<BlockLess> order, so its slot is the rank-th pop of the free list — what the
//    reference's lazy allocate_block calls in list order produce (fusion.cpp:294-299;
//    grid.cpp:87-100); rank == free_top is the PoolExhausted key (fusion.cpp:369).
//  - the other CTAs: the update list over the blocks allocated before this frame (slots
//    below the frame's starting high-water mark). It does not depend on the allocation:
//    slots (re)used this frame hold keys of the allocate set, which the key set excludes.
//  - last CTA: counters; on PoolExhausted the processed allocate prefix (keys below the
//    exhaustion key) is compacted to the front of the work list and the update list dropped.
constexpr int kRankCtas = 148;
constexpr int kRankKeys = 4;
__global__ void __launch_bounds__(256)
    k_alloc_visible(VolParams P, const FrameConsts* __restrict__ fc, FrameCounters* ctr, VolCounters* vc,
                    const uint32_t* __restrict__ new_keys, const uint32_t* __restrict__ new_idx,
                    int32_t* __restrict__ table, const int32_t* __restrict__ free_list, int32_t* __restrict__ slot_key,
                    uint32_t* __restrict__ occ, const uint32_t* __restrict__ uniq, const uint32_t* __restrict__ keybits,
                    const float* __restrict__ depth, int w, int h, int2* __restrict__ work) {
    pdl_wait();
    __shared__ bool s_last;
    __shared__ uint32_t s_wsum[8];
    if (ctr->skip) return;
    const uint32_t n = ctr->n_new, n_unique = ctr->n_unique;
    const unsigned long long top = vc->free_top;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (blockIdx.x < kRankCtas) {
        const uint32_t nw = kRankCtas * (blockDim.x >> 5);
        for (uint32_t g = blockIdx.x * (blockDim.x >> 5) + warp; g * kRankKeys < n; g += nw) {
            uint32_t kq[kRankKeys], rank[kRankKeys];
#pragma unroll
            for (int t = 0; t < kRankKeys; ++t) {
                const uint32_t q = g * kRankKeys + t;
                kq[t] = q < n ? new_keys[q] : 0u;
                rank[t] = 0;
            }
            for (uint32_t j = lane; j < n; j += 32) {
                const uint32_t x = new_keys[j];
#pragma unroll
                for (int t = 0; t < kRankKeys; ++t) rank[t] += x < kq[t] ? 1u : 0u;
            }
#pragma unroll
            for (int t = 0; t < kRankKeys; ++t) {
                const uint32_t r = __reduce_add_sync(0xffffffffu, rank[t]);
                const uint32_t q = g * kRankKeys + t;
                if (lane == t && q < n) {
                    const uint32_t key = kq[t];
                    if (r < top) {
                        const int32_t slot = free_list[top - 1 - r];
                        table[key] = slot;
                        slot_key[slot] = static_cast<int32_t>(key);
                        occ_set(P, occ, key);
                        atomicMax(&vc->high_water, (unsigned long long)slot + 1ull);
                        work[new_idx[q]] = make_int2(static_cast<int32_t>(static_cast<uint32_t>(slot) | 0x80000000u),
                                                     static_cast<int32_t>(key));
                    } else if (r == top) {
                        ctr->exhaust_key = key;  // PoolExhausted at this key (fusion.cpp:369)
                    }
                }
            }
        }
    } else {
        const unsigned long long hw = ctr->hw_before;
        const uint32_t stride = (gridDim.x - kRankCtas) * blockDim.x;
        for (unsigned long long s = (blockIdx.x - kRankCtas) * (unsigned long long)blockDim.x + threadIdx.x; s < hw;
             s += stride) {
            const int32_t key = slot_key[s];
            const bool vis = key >= 0 && !((keybits[key >> 5] >> (key & 31)) & 1u) &&
                             block_visible(P, fc, key, depth, w, h);
            const uint32_t j = warp_append(vis, &ctr->n_update);
            if (vis) work[n_unique + j] = make_int2(static_cast<int32_t>(s), key);
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&ctr->tickets, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const bool exhausted = n > top;
    if (threadIdx.x == 0) {
        const unsigned long long got = n < top ? n : top;
        vc->free_top = top - got;
        vc->allocated_count += got;
        ctr->exhausted = exhausted ? 1u : 0u;
        if (!exhausted) ctr->exhaust_key = 0xffffffffu;
        ctr->n_list = n_unique;
        ctr->upd_base = n_unique;
        if (!exhausted) ctr->limit = n_unique;
        else ctr->n_update = 0;  // the update list is never reached
    }
    if (!exhausted) return;
    // PoolExhausted: keep the items of keys below the exhaustion key (all of them have slots:
    // a new key below it has a smaller rank), compacted in place in chunk order.
    const uint32_t ex_key = *(volatile uint32_t*)&ctr->exhaust_key;
    uint32_t pos = 0;
    for (uint32_t base = 0; base < n_unique; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        int2 it = make_int2(0, 0);
        bool take = false;
        if (i < n_unique) {
            it = work[i];
            take = static_cast<uint32_t>(it.y) < ex_key;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        if (lane == 0) s_wsum[warp] = __popc(bal);
        __syncthreads();
        uint32_t off = pos;
        for (int k = 0; k < warp; ++k) off += s_wsum[k];
        uint32_t tot = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) tot += s_wsum[k];
        if (take) work[off + __popc(bal & ((1u << lane) - 1u))] = it;
        pos += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) ctr->limit = pos;
}

// ---------------------------------------------------------------------------------
// visibility: exact SAT + probes over every allocated block
// ---------------------------------------------------------------------------------
__device__ __forceinline__ bool in_sorted(const uint32_t* __restrict__ a, uint32_t n, uint32_t key) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        const uint32_t x = a[mid];
        if (x < key) lo = mid + 1;
        else hi = mid;
    }
    return lo < n && a[lo] == key;
}

__global__ void k_visible(VolParams P, const FrameConsts* __restrict__ fc, FrameCounters* ctr,
                          const VolCounters* __restrict__ vc, const int32_t* __restrict__ slot_key,
                          const uint32_t* __restrict__ uniq, const float* __restrict__ depth, int w, int h,
                          int2* __restrict__ work, uint32_t* __restrict__ export_keys, int export_only) {
    if (ctr->skip || (!export_only && ctr->exhausted)) return;
    const unsigned long long hw = vc->high_water;
    const uint32_t n_list = ctr->n_list;
    const uint32_t base = ctr->limit;
    const Intr& intr = fc->intr;
    for (unsigned long long s = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; s < hw;
         s += (unsigned long long)gridDim.x * blockDim.x) {
        const int32_t key = slot_key[s];
        if (key < 0) continue;
        if (in_sorted(uniq, n_list, static_cast<uint32_t>(key))) continue;  // in the allocate set
        const int bx = key % P.N, by = (key / P.N) % P.N, bz = key / (P.N * P.N);
        if (!shard_owns(P, bx, by, bz)) continue;  // mirrored halo block of another rank
        const d3 lo = block_min_corner(P, bx, by, bz);
        const double side = P.block_side;
        const d3 hi = add(lo, mk(side, side, side));
        if (!block_surely_inside(P, fc, lo) && !frustum_intersects_block(P, fc, lo, hi)) continue;
        bool visible = false;
        for (int i = 0; i < 9 && !visible; ++i) {
            const d3 probe = i == 8 ? add(lo, mk(0.5 * side, 0.5 * side, 0.5 * side))
                                    : add(lo, mk(i & 1 ? side : 0.0, i & 2 ? side : 0.0, i & 4 ? side : 0.0));
            const d3 xc = apply(fc->inv, probe);
            double pu, pv;
            if (!project(intr, xc, pu, pv)) continue;
            const int u = ref_lround_int(pu);
            const int v = ref_lround_int(pv);
            if (!(u >= 0 && v >= 0 && u < w && v < h)) continue;
            const float d = depth[(size_t)v * w + u];
            if (!(d > 0.0f) || xc.z <= d + fc->delta) visible = true;
        }
        if (!visible) continue;
        const uint32_t j = atomicAdd(&ctr->n_update, 1u);
        if (export_only) export_keys[j] = static_cast<uint32_t>(key);
        else work[base + j] = make_int2(static_cast<int32_t>(s), key);
    }
}

// Work item i: the allocate part [0, limit), then the update part [upd_base, upd_base + n_update).
__device__ __forceinline__ int2 work_at(const int2* __restrict__ work, uint32_t limit, uint32_t upd_base, uint32_t i) {
    return i < limit ? work[i] : work[upd_base + (i - limit)];
}
// The key set must be empty for the next frame: clear the words of this frame's keys (the
// work-list pass, its only reader, has finished).
__device__ __forceinline__ void clear_keybits(const FrameCounters* ctr, const uint32_t* __restrict__ uniq,
                                              uint32_t* __restrict__ keybits) {
    const uint32_t n = ctr->n_unique;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        keybits[uniq[i] >> 5] = 0u;
}

// ---------------------------------------------------------------------------------
// per-voxel integration
// ---------------------------------------------------------------------------------
// log2(v) to ~0.01 for positive normal v, from the exponent and a quadratic in the
// mantissa (integer + FP64 pipe only).
__device__ __forceinline__ double approx_log2(double v) {
    const long long b = __double_as_longlong(v);
    const int e = static_cast<int>((b >> 52) & 0x7ff) - 1023;
    const double m = __longlong_as_double((b & 0x000fffffffffffffLL) | 0x3ff0000000000000LL) - 1.0;
    return i2d_exact(e) + m * (1.3465 - 0.3465 * m);
}
// Variance-mode aux code #{k in 1..255 : value >= thresh[k]} (thresholds ascending, each an
// exact reference encode boundary): guess from the log-scale formula of grid.cpp:42-45,
// then walk to the exact answer (almost always zero or one step).
__device__ __forceinline__ int aux_var_code(const VolParams& P, const double* s_thr, double value) {
    if (value != value) return 0;  // NaN: every comparison fails
    const double vc = dclamp(value, P.aux_p_min, P.aux_p_max);
    const double gs = dclamp((approx_log2(vc) - P.aux_lg_pmin) * P.aux_lg_scale, 0.0, 255.0);
    int g = static_cast<int>(static_cast<unsigned int>(__double_as_longlong(gs + kMagic52)));
    while (g < 255 && value >= s_thr[g + 1]) ++g;
    while (g > 0 && !(value >= s_thr[g])) --g;
    return g;
}

__device__ __forceinline__ uint8_t aux_encode_dev(const VolParams& P, const double* s_thr, double value) {
    if (P.aux_mode == 0) {
        const double clamped = dclamp(value, 0.0, P.aux_w_max);
        return static_cast<uint8_t>(static_cast<long long>(llround(clamped / P.aux_w_max * 255.0)));
    }
    return static_cast<uint8_t>(aux_var_code(P, s_thr, value));
}

// ---------------------------------------------------------------------------------
// FP64 filter rules and payload encoding (fusion.cpp:237-272, 353-361), shared by the
// generic kernel and the exact fallback of the row kernel. The `approx` variants replace the
// one division by a Newton-refined reciprocal and certify the resulting decisions.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ bool approx_rcp(double z, double& r) {
    if (!(fabs(z) > 1e-30 && fabs(z) < 1e30)) return false;
    double x;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(x) : "d"(z));  // MUFU.RCP64H, ~20 bits
    x = fma(x, fma(-z, x, 1.0), x);                          // ~40 bits
    x = fma(x, fma(-z, x, 1.0), x);                          // ~full precision
    x = fma(x, fma(-z, x, 1.0), x);
    r = x;
    return true;
}
// lround decision certain when the interval [a - e, a + e] holds no rounding boundary.
// Conversion-free (certain_lround_fast): the XU pipe was this kernel's limiter.
__device__ __forceinline__ bool certain_lround(double a, int& out) {
    return certain_lround_fast(a, 1e-9 + 1e-12 * fabs(a), out);
}
// Variance-mode aux code from an approximate value: certain unless within 1e-12 relative of
// a threshold (each threshold is an exact reference encode boundary).
__device__ __forceinline__ bool certain_aux_var(const VolParams& P, const double* s_thr, double a, double a_err,
                                                int& out) {
    const int lo = aux_var_code(P, s_thr, a);
    out = lo;
    const double m = 1e-12 * fabs(a) + 100.0 * a_err + 1e-300;
    if (lo > 0 && !(a - m >= s_thr[lo])) return false;
    if (lo < 255 && !(a + m < s_thr[lo + 1])) return false;
    return true;
}

// Filter rules (fusion.cpp:237-272); `approx` replaces the one division by a reciprocal.
template <int MODE>
__device__ __forceinline__ bool filter_rule(bool has_prior, double prior_t, double prior_a, double tsdf_k, double pk,
                                            double wk, const FuseParams& fp, bool approx, double& new_t,
                                            double& new_a, double& a_err) {
    a_err = 0.0;  // absolute error bound of new_a on the approx path
    if (MODE == 0) {
        new_t = has_prior ? (1.0 - wk) * prior_t + wk * tsdf_k : tsdf_k;
        new_a = wk;
    } else if (MODE == 1) {
        if (!has_prior) {
            new_t = tsdf_k;
            new_a = wk;
        } else {
            const double num = prior_a * prior_t + wk * tsdf_k, den = prior_a + wk;
            double r;
            if (approx) {
                if (!approx_rcp(den, r)) return false;
                new_t = num * r;
            } else {
                new_t = num / den;
            }
            new_a = dmin(prior_a + wk, fp.w_max);
        }
    } else {
        if (!has_prior) {
            new_t = tsdf_k;
            new_a = pk;
        } else {
            const double predicted = prior_a + fp.q;
            const double den = predicted + pk;
            double gain, r;
            if (approx) {
                if (!approx_rcp(den, r)) return false;
                gain = predicted * r;
            } else {
                gain = predicted / den;
            }
            new_t = prior_t + gain * (tsdf_k - prior_t);
            new_a = (1.0 - gain) * predicted;
            // 1 - gain cancels when gain ~ 1: |gain' - gain| <= 4 ulp(gain) propagates as an
            // absolute error ~4.5e-16 * predicted, independent of new_a's magnitude.
            if (approx) a_err = 1e-15 * predicted;
        }
    }
    return true;
}

// Payload code of a filter result. approx: decisions must be certain (else return false).
__device__ __forceinline__ bool encode_cell(const VolParams& P, const double* s_thr, double new_t, double new_a,
                                            double a_err, bool approx, double inv_delta, double inv_wmax,
                                            uint16_t& out) {
    const double delta = P.delta;
    if (!approx) {
        if (fabs(new_t) > delta) {
            out = kChiPayload;
        } else {
            const int8_t code = quantize_tsdf(new_t, delta);
            const uint8_t ac = aux_encode_dev(P, s_thr, new_a);
            out = static_cast<uint16_t>(static_cast<uint8_t>(code)) | static_cast<uint16_t>(ac << 8);
        }
        return true;
    }
    const double at = fabs(new_t);
    const double tol = 1e-12 * delta;
    if (!(fabs(at - delta) > tol)) return false;  // chi cut too close to call
    if (at > delta) {
        out = kChiPayload;
        return true;
    }
    int code, ac;
    if (!certain_lround(dclamp(new_t, -delta, delta) * inv_delta * (double)kTsdfCodeRange, code)) return false;
    if (P.aux_mode == 0) {
        if (!certain_lround(dclamp(new_a, 0.0, P.aux_w_max) * inv_wmax * 255.0, ac)) return false;
    } else {
        if (!certain_aux_var(P, s_thr, new_a, a_err, ac)) return false;
    }
    out = static_cast<uint16_t>(static_cast<uint8_t>(static_cast<int8_t>(code))) |
          static_cast<uint16_t>(static_cast<uint8_t>(ac) << 8);
    return true;
}

// ---------------------------------------------------------------------------------
// Row-compacted integrate (M = 4 or 8): the roofline kernel. Bit-exact by certification.
//
// Only rounding DECISIONS of the reference reach the stored state: z > 0, the pixel
// lround(u), lround(v) (fusion.cpp:92-93), the band cut |T| > delta (fusion.cpp:145), the
// chi cut |T'| > delta and the tsdf / aux codes (fusion.cpp:353-361). Everything in between
// is evaluated in FP32 with a rigorous error bound, and a decision is accepted only when the
// value is farther than that bound from the decision boundary; otherwise the voxel is
// recomputed by the reference's FP64 path (`exact_voxel`, probability ~1e-3 per voxel).
//
// Phase 1 (one thread per x-row of M voxels): one vector load of the row's payload (16 B at
// M = 8), the row origin in camera space in FP64 (x_c = R^T(voxel_center - t), the
// reference's order), then per voxel x_c = origin + lx * voxel * R^T e_x in FP32, projection
// with a hardware reciprocal, certified pixel rounding, one float2 gather {depth, p_k} and the
// band test on T = (d - z_hi) - (z_lo + lx dz) (double-float row origin: error ~1e-9 m).
// Voxels in the band are compacted into a shared-memory queue (uncertain ones at its top).
// Phase 2: the CTA drains the queue densely (no divergence between in-band and free-space
// voxels): Kalman / weighted / simple update in FP32, certified quantisation, 2 B store.
// Error bounds and margins: DESIGN.md §3.2.
// ---------------------------------------------------------------------------------
constexpr float kMagic23 = 12582912.0f;  // 1.5 * 2^23
// std::lround(a) when certain under margin e; requires |a| < 2^22 (callers clamp).
__device__ __forceinline__ bool certain_lround_f(float a, float e, int& out) {
    const float t = __fadd_rn(a, kMagic23);
    const float n = __fsub_rn(t, kMagic23);
    const float d = __fsub_rn(a, n);  // exact: |a - n| <= 1/2, both multiples of ulp(a)
    out = __float_as_int(t) - __float_as_int(kMagic23);
    return fabsf(d) < 0.5f - e;
}
__device__ __forceinline__ float rcp_approx_f(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));  // MUFU.RCP, <= 1 ulp
    return r;
}
// log2(v) to ~0.01 for positive normal v (exponent + quadratic in the mantissa).
__device__ __forceinline__ float approx_log2_f(float v) {
    const int b = __float_as_int(v);
    const float m = __int_as_float((b & 0x007fffff) | 0x3f800000) - 1.0f;
    return static_cast<float>((b >> 23) - 127) + m * (1.3465f - 0.3465f * m);
}

// Per-frame constants of the row kernel, computed once per CTA into shared memory.
struct RowShared {
    double R[9], t[3];  // world -> camera (invert(pose)): x_c = R x + t, the reference's order
    double ox, oy, oz, voxel;
    float Dxf, Dyf, Dzf;      // x_c step per voxel along x: voxel * R e_x
    float fxf, fyf, cxf, cyf;
    float Fmax, Wpix, Mvox;   // max(fx, fy), max(w, h) + 2, M * voxel
    float thr_in, thr_out;    // band test: |T| certainly inside / outside delta
    float k127, ecode;        // 127 / delta; tsdf-code margin (code units)
    float q, w_max, k255w, lg_pmin, lg_scale;
    float thr_lo, thr_hi;     // clamp range of the variance code guess
    float delta_f, echi;      // float payload: chi cut |T'| > delta certain outside delta +- echi
    double cx, cy;            // principal point (pixel-boundary planes of small-footprint rows)
    double eT;                // |T_f32 - T_ref| bound (m) of the phase-1 measurement
    int lut_shift, lut_base, lut_n;  // variance-code lookup (AuxTables::lut; lut_n = 0: log-scale guess)
    int axis, lstep;          // row axis (0 x, 1 y, 2 z: the block axis closest to the optical axis), its l stride
};

// Row axis of a frame: the block axis with the largest camera-z component (x on ties).
__device__ __forceinline__ int row_axis(const Pose& inv) {
    int ax = 0;
    if (fabs(inv.R.m[7]) > fabs(inv.R.m[6 + ax])) ax = 1;
    if (fabs(inv.R.m[8]) > fabs(inv.R.m[6 + ax])) ax = 2;
    return ax;
}
// Per-frame constants of the row kernels (one thread).
template <int M>
__device__ void row_kernel_init(const VolParams& P, const FrameConsts* __restrict__ fc, const FuseParams& fp,
                                const AuxTables* __restrict__ aux, RowShared& sh, VolParams& sP, FuseParams& sFp,
                                float* s_thr) {
    sh.lut_shift = aux->lut_shift;
    sh.lut_base = aux->lut_base;
    sh.lut_n = aux->lut_n;
    s_thr[0] = -INFINITY;
    s_thr[257] = s_thr[258] = s_thr[259] = INFINITY;
    sP = P;
    sFp = fp;
    const Pose inv = fc->inv;
    const Intr intr = fc->intr;
    for (int i = 0; i < 9; ++i) sh.R[i] = inv.R.m[i];
    sh.t[0] = inv.t.x;
    sh.t[1] = inv.t.y;
    sh.t[2] = inv.t.z;
    sh.ox = P.ox;
    sh.oy = P.oy;
    sh.oz = P.oz;
    sh.voxel = P.voxel;
    // rows along the block axis with the largest camera-z component (x on ties)
    const int ax = row_axis(inv);
    sh.axis = ax;
    sh.lstep = ax == 0 ? 1 : ax == 1 ? M : M * M;
    sh.Dxf = static_cast<float>(P.voxel * inv.R.m[ax]);
    sh.Dyf = static_cast<float>(P.voxel * inv.R.m[3 + ax]);
    sh.Dzf = static_cast<float>(P.voxel * inv.R.m[6 + ax]);
    sh.cx = intr.cx;
    sh.cy = intr.cy;
    sh.fxf = static_cast<float>(intr.fx);
    sh.fyf = static_cast<float>(intr.fy);
    sh.cxf = static_cast<float>(intr.cx);
    sh.cyf = static_cast<float>(intr.cy);
    sh.Fmax = static_cast<float>(dmax(intr.fx, intr.fy));
    sh.Wpix = static_cast<float>(intr.w > intr.h ? intr.w : intr.h) + 2.0f;
    sh.Mvox = static_cast<float>(M * P.voxel);
    // T error bound (m) for rows with z < 16 m: double-float row origin, lx * dz, and the
    // (Sterbenz-exact in the band) subtraction d - z_hi
    const double delta = P.delta;
    // |T_f32 - T_ref| <= 2^-24 ((M-1) voxel [Dzf] + (M-1) voxel [fma] + |d - Azh| + |T| [two
    // subtractions] + (M-1) voxel) + 2^-40 [the reference's own FP64 x_c vs the row model],
    // with |d - Azh|, |T| <= delta + (M-1) voxel inside the decision region; x 1.25 slack
    const double eT = 1.25 * 0x1p-23 * (delta + 1.5 * (M - 1) * P.voxel) + 0x1p-40;
    sh.eT = eT;
    sh.thr_out = static_cast<float>((delta + eT) * 1.000001);
    sh.thr_in = static_cast<float>((delta - eT) * 0.999999);
    sh.k127 = static_cast<float>(kTsdfCodeRange / delta);
    // code margin: the measurement's eT (gain <= 1) plus the FP32 filter's own error
    // (<= 2.4e-4 code units: rounded inputs, rcp.approx, three roundings; x 1.5 slack)
    sh.ecode = static_cast<float>(3.6e-4 + 1.5 * eT * (kTsdfCodeRange / delta));
    sh.q = static_cast<float>(fp.q);
    sh.w_max = static_cast<float>(P.aux_w_max);
    sh.k255w = static_cast<float>(255.0 / P.aux_w_max);
    sh.lg_pmin = static_cast<float>(P.aux_lg_pmin);
    sh.lg_scale = static_cast<float>(P.aux_lg_scale);
    sh.thr_lo = static_cast<float>(P.aux_p_min * 0.5);
    sh.thr_hi = static_cast<float>(P.aux_p_max * 2.0);
    // float payload chi cut: T' carries the measurement's eT (gain <= 1) and the FP32 filter
    // error (a few ulp of delta); float(delta) itself is within 2^-24 delta
    sh.delta_f = static_cast<float>(delta);
    sh.echi = static_cast<float>(2.0 * eT + 4e-6 * delta);
}
// Phase-2 update of one in-band voxel in FP32; false when a decision is not certain.
template <int MODE>
__device__ __forceinline__ bool approx_update(uint32_t cell, float tk, float pf, const RowShared& rc,
                                              const float* s_tdec, const float* s_adec, const float* s_thr,
                                              const uint2* s_lut, uint32_t& out) {
    const int code = static_cast<int>(static_cast<int8_t>(cell & 0xFF));
    const bool has_prior = code != kChiCode;
    const float pt = s_tdec[code + 128], pa = s_adec[cell >> 8];
    float nt, na, pred = 0.0f;
    // filters (fusion.cpp:237-272)
    if (MODE == 0) {
        nt = has_prior ? (1.0f - pf) * pt + pf * tk : tk;
        na = pf;
    } else if (MODE == 1) {
        nt = has_prior ? (pa * pt + pf * tk) * rcp_approx_f(pa + pf) : tk;
        na = has_prior ? fminf(pa + pf, rc.w_max) : pf;
    } else {
        pred = has_prior ? pa + rc.q : 0.0f;
        const float gain = pred * rcp_approx_f(pred + pf);
        nt = has_prior ? pt + gain * (tk - pt) : tk;
        na = has_prior ? pf * gain : pf;  // pf * gain == (1 - gain) * predicted, without the cancellation
    }
    // chi cut and tsdf code (grid.cpp:20-23; |nt| <= delta so the clamp is the identity)
    const float a = nt * rc.k127;
    const float aa = fabsf(a);
    if (!(fabsf(aa - 127.0f) > rc.ecode)) return false;
    if (aa > 127.0f) {
        out = kChiPayload;
        return true;
    }
    int tc;
    if (!certain_lround_f(a, rc.ecode, tc)) return false;
    int ac;
    if (MODE == 2) {
        // #{k : na >= thresh[k]} (thresholds = exact reference encode boundaries). Margin:
        // FP32 evaluation (<= 2e-6 relative) + the reference's own cancellation in
        // (1 - gain) * predicted (<= 1e-15 * predicted) + float thresholds (2^-24).
        const float m = 3e-6f * na + 1e-15f * pred;
        if (rc.lut_n > 0) {
            // the bucket of na's float bits holds at most one threshold: code = #below + (na >= it)
            if (!(na >= 0.0f)) return false;
            const int b = min(max(static_cast<int>(__float_as_uint(na) >> rc.lut_shift) - rc.lut_base, 0), rc.lut_n - 1);
            const uint2 e = s_lut[b];
            const int g = static_cast<int>(e.y) + (na >= __uint_as_float(e.x) ? 1 : 0);
            if (!(na - m >= s_thr[g + 1]) && g > 0) return false;   // thresh[g]
            if (!(na + m < s_thr[g + 2]) && g < 255) return false;  // thresh[g + 1]
            out = static_cast<uint32_t>(static_cast<uint8_t>(tc)) | (static_cast<uint32_t>(g) << 8);
            return true;
        }
        // The log-scale guess is within 0.1 code of the encode formula, so the code is one of
        // round(guess) - 1 .. + 1: two comparisons settle it (s_thr is shifted by one with
        // -inf / +inf sentinels so every index below is in range).
        const float vc = fminf(fmaxf(na, rc.thr_lo), rc.thr_hi);
        const float gs = fminf(fmaxf((approx_log2_f(vc) - rc.lg_pmin) * rc.lg_scale, 0.0f), 255.0f);
        const int gr = __float_as_int(__fadd_rn(gs, kMagic23)) - __float_as_int(kMagic23);
        const float t_m1 = s_thr[gr], t_0 = s_thr[gr + 1], t_p1 = s_thr[gr + 2], t_p2 = s_thr[gr + 3];
        // thresholds of codes gr-1 .. gr+2 (s_thr[k + 1] = thresh[k])
        if (!(na >= t_m1) || !(na < t_p2)) return false;  // guess off by more than one: exact path
        const bool ge0 = na >= t_0, ge1 = na >= t_p1;
        const int g = gr - 1 + static_cast<int>(ge0) + static_cast<int>(ge1);
        const float lo = ge1 ? t_p1 : ge0 ? t_0 : t_m1;   // thresh[g]
        const float hi = ge1 ? t_p2 : ge0 ? t_p1 : t_0;   // thresh[g + 1]
        if (!(na - m >= lo) && g > 0) return false;
        if (!(na + m < hi) && g < 255) return false;
        ac = g;
    } else {
        if (!certain_lround_f(fminf(fmaxf(na, 0.0f), rc.w_max) * rc.k255w, 1e-3f, ac)) return false;
    }
    out = static_cast<uint32_t>(static_cast<uint8_t>(tc)) | (static_cast<uint32_t>(ac) << 8);
    return true;
}

// Second chance for a voxel whose FP32 update was not certain (codes): the filter rule in FP64
// on the same phase-1 inputs (T with its bound eT, p_k / w_k rounded to float), the decisions
// certified against that input error only (no FP32 filter error): ~4x fewer voxels reach the
// full FP64 path (exact_voxel), which re-derives the measurement from the projection.
// Errors of the FP64 results vs the reference's: new_t <= eT (gain <= 1) + 2 delta 2^-25 (p_k
// rounding through the gain, |T - prior| <= 2 delta) + FP64 rounding; new_a relative <= 2^-24
// (d ln new_a / d ln p_k <= 1) + the reference's own cancellation a_err (filter_rule).
template <int MODE>
__device__ __noinline__ bool refine_update(const VolParams& P, const FuseParams& fp, const AuxTables* __restrict__ aux,
                                           uint32_t cell, float tk, float pf, double eT, uint32_t& out) {
    const int code = static_cast<int>(static_cast<int8_t>(cell & 0xFF));
    const bool has_prior = code != kChiCode;
    const double pt = has_prior ? aux->tsdf_decode[code + 128] : 0.0;
    const double pa = has_prior ? aux->aux_decode[cell >> 8] : 0.0;
    double nt, na, a_err;
    if (!filter_rule<MODE>(has_prior, pt, pa, static_cast<double>(tk), MODE == 2 ? static_cast<double>(pf) : 0.0,
                           MODE == 2 ? 0.0 : static_cast<double>(pf), fp, true, nt, na, a_err))
        return false;
    const double delta = P.delta;
    const double et = 1.5 * (eT + 0x1p-24 * delta) + 1e-15 * delta;
    const double at = fabs(nt);
    if (!(fabs(at - delta) > et)) return false;
    if (at > delta) {
        out = kChiPayload;
        return true;
    }
    int tc, ac;
    if (!certain_lround_fast(nt * (kTsdfCodeRange / delta), et * (kTsdfCodeRange / delta) + 1e-9, tc)) return false;
    const double ea = 1.5 * (0x1p-23 * fabs(na) + a_err) + 1e-300;
    if (P.aux_mode == 0) {
        const double k = 255.0 / P.aux_w_max;
        if (!certain_lround_fast(dclamp(na, 0.0, P.aux_w_max) * k, ea * k + 1e-9, ac)) return false;
    } else {
        ac = aux_var_code(P, aux->aux_thresh, na);
        if (ac > 0 && !(na - ea >= aux->aux_thresh[ac])) return false;
        if (ac < 255 && !(na + ea < aux->aux_thresh[ac + 1])) return false;
    }
    out = static_cast<uint32_t>(static_cast<uint8_t>(static_cast<int8_t>(tc))) | (static_cast<uint32_t>(ac) << 8);
    return true;
}

// The reference's FP64 path for one voxel (fusion.cpp:81-173, 237-364): the payload code,
// or -1 when there is no measurement.
template <int MODE>
__device__ __noinline__ int exact_voxel(const VolParams& P, const FrameConsts* __restrict__ fc, const FuseParams& fp,
                                        const AuxTables* __restrict__ aux, int key, int l, uint32_t cell,
                                        const double* __restrict__ pix_dm, const double* __restrict__ pix_var,
                                        const double* __restrict__ pix_w) {
    const int N = P.N, M = P.M;
    const int bx = key % N, by = (key / N) % N, bz = key / (N * N);
    const int lx = l % M, ly = (l / M) % M, lz = l / (M * M);
    const d3 xc = apply(fc->inv, voxel_center(P, bx * M + lx, by * M + ly, bz * M + lz));
    double pu, pv;
    if (!project(fc->intr, xc, pu, pv)) return -1;
    const int u = ref_lround_int(pu), v = ref_lround_int(pv);
    if (!(u >= 0 && v >= 0 && u < fc->intr.w && v < fc->intr.h)) return -1;
    const size_t pix = (size_t)v * fc->intr.w + u;
    const double dm = pix_dm[pix];  // depth where the pixel passes every per-pixel test, else 0
    if (!(dm > 0.0)) return -1;
    const double tsdf_k = dm - xc.z;
    if (fabs(tsdf_k) > P.delta) return -1;
    const int8_t code = static_cast<int8_t>(cell & 0xFF);
    const bool has_prior = code != kChiCode;
    const double prior_t = has_prior ? aux->tsdf_decode[(int)code + 128] : 0.0;
    const double prior_a = has_prior ? aux->aux_decode[cell >> 8] : 0.0;
    double new_t, new_a, a_err;
    filter_rule<MODE>(has_prior, prior_t, prior_a, tsdf_k, MODE == 2 ? pix_var[pix] : 0.0,
                      MODE == 2 ? 0.0 : pix_w[pix], fp, false, new_t, new_a, a_err);
    uint16_t out;
    encode_cell(P, aux->aux_thresh, new_t, new_a, 0.0, false, 1.0 / P.delta, 1.0 / P.aux_w_max, out);
    return out;
}

// Float payload (block-sparse FloatShadowGrid semantics, grid.hpp:77-88; fusion.cpp:313-318,
// 350-362): phase-2 update of one in-band voxel in FP32 from its float prior. The stored value
// only has to meet the value tolerance (1e-5), but the chi cut |T'| > delta is a decision:
// false when it is not certain (then the FP64 path decides).
template <int MODE>
__device__ __forceinline__ bool approx_update_f2(float2 prior, float tk, float pf, const RowShared& rc, float2& out) {
    const bool has_prior = prior.x < INFINITY;  // !FloatShadowGrid::is_chi
    const float pt = prior.x, pa = prior.y;
    float nt, na;
    if (MODE == 0) {
        nt = has_prior ? (1.0f - pf) * pt + pf * tk : tk;
        na = pf;
    } else if (MODE == 1) {
        nt = has_prior ? (pa * pt + pf * tk) * rcp_approx_f(pa + pf) : tk;
        na = has_prior ? fminf(pa + pf, rc.w_max) : pf;
    } else {
        const float pred = pa + rc.q;
        const float gain = pred * rcp_approx_f(pred + pf);
        nt = has_prior ? pt + gain * (tk - pt) : tk;
        na = has_prior ? pf * gain : pf;  // == (1 - gain) * predicted, without the cancellation
    }
    const float at = fabsf(nt);
    if (!(fabsf(at - rc.delta_f) > rc.echi)) return false;
    out = at > rc.delta_f ? make_float2(INFINITY, 0.0f) : make_float2(nt, na);
    return true;
}

// The reference's FP64 path for one voxel with a float prior (fusion.cpp:81-173, 237-272,
// 313-318, 357-361): false when there is no measurement.
template <int MODE>
__device__ __noinline__ bool exact_voxel_f2(const VolParams& P, const FrameConsts* __restrict__ fc, const FuseParams& fp,
                                            int key, int l, float2 prior, const double* __restrict__ pix_dm,
                                            const double* __restrict__ pix_var, const double* __restrict__ pix_w,
                                            float2& out) {
    const int N = P.N, M = P.M;
    const int bx = key % N, by = (key / N) % N, bz = key / (N * N);
    const int lx = l % M, ly = (l / M) % M, lz = l / (M * M);
    const d3 xc = apply(fc->inv, voxel_center(P, bx * M + lx, by * M + ly, bz * M + lz));
    double pu, pv;
    if (!project(fc->intr, xc, pu, pv)) return false;
    const int u = ref_lround_int(pu), v = ref_lround_int(pv);
    if (!(u >= 0 && v >= 0 && u < fc->intr.w && v < fc->intr.h)) return false;
    const size_t pix = (size_t)v * fc->intr.w + u;
    const double dm = pix_dm[pix];
    if (!(dm > 0.0)) return false;
    const double tsdf_k = dm - xc.z;
    if (fabs(tsdf_k) > P.delta) return false;
    const bool has_prior = prior.x < INFINITY;
    double new_t, new_a, a_err;
    filter_rule<MODE>(has_prior, has_prior ? (double)prior.x : 0.0, has_prior ? (double)prior.y : 0.0, tsdf_k,
                      MODE == 2 ? pix_var[pix] : 0.0, MODE == 2 ? 0.0 : pix_w[pix], fp, false, new_t, new_a, a_err);
    out = fabs(new_t) > P.delta ? make_float2(INFINITY, 0.0f) : make_float2((float)new_t, (float)new_a);
    return true;
}

constexpr int kRowThreads = 256;
#ifndef SF_ROW_CTAS
#define SF_ROW_CTAS 3
#endif
constexpr int kRowCtasPerSm = SF_ROW_CTAS;
constexpr uint32_t kGrabUnits = 4;  // 32-row units a warp takes per atomic (before the tail)
constexpr uint32_t kTailUnitsPerWarp = 8;  // single-unit grabs once this much work per warp remains
#ifndef SF_STATIC_PCT
#define SF_STATIC_PCT 50
#endif
constexpr uint32_t kStaticPct = SF_STATIC_PCT;  // share of the row units dealt out statically
#ifndef SF_SLAB  // M = 8: half-block slab kernel (k_integrate_slab) instead of k_integrate_rows
#define SF_SLAB 1
#endif
#ifndef SF_DIAG_TIMES  // timing diagnostics (tools/slab_times.py): per-warp timeline of k_integrate_slab
#define SF_DIAG_TIMES 0
#endif

template <int MS>
struct RowVec;
template <>
struct RowVec<3> {
    using T = uint4;
    __device__ static uint32_t cell(const uint4& r, int lx) {
        const uint32_t w = lx < 2 ? r.x : lx < 4 ? r.y : lx < 6 ? r.z : r.w;
        return (lx & 1) ? (w >> 16) : (w & 0xFFFF);
    }
    __device__ static uint4 chi() { return make_uint4(0x00800080u, 0x00800080u, 0x00800080u, 0x00800080u); }
    __device__ static uint4 gather(const uint16_t* c, int stride) {  // a row along y or z
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = c[(2 * k) * stride] | (static_cast<uint32_t>(c[(2 * k + 1) * stride]) << 16);
        return make_uint4(w[0], w[1], w[2], w[3]);
    }
};
template <>
struct RowVec<2> {
    using T = uint2;
    __device__ static uint32_t cell(const uint2& r, int lx) {
        const uint32_t w = lx < 2 ? r.x : r.y;
        return (lx & 1) ? (w >> 16) : (w & 0xFFFF);
    }
    __device__ static uint2 chi() { return make_uint2(0x00800080u, 0x00800080u); }
    __device__ static uint2 gather(const uint16_t* c, int stride) {
        return make_uint2(c[0] | (static_cast<uint32_t>(c[stride]) << 16),
                          c[2 * stride] | (static_cast<uint32_t>(c[3 * stride]) << 16));
    }
};

// Per-warp ring of queued voxels: >= 31 left over + 32 rows x M new entries, a power of two.
template <int MS>
struct RowRing {
    // >= 31 left over + the new entries between drains (M = 8 drains after each half-row)
    static constexpr int kEntries = (MS == 3 && kRowCtasPerSm <= 3) ? 512 : 256;
    static constexpr size_t kBytes = (kRowThreads / 32) * kEntries * sizeof(uint4);
};

// P2: the float2 {tsdf, aux} payload layout (SF_PAYLOAD_FLOAT2) instead of the 2-byte codes.
template <int MODE, int MS, bool P2>
__global__ void __launch_bounds__(kRowThreads, kRowCtasPerSm)
    k_integrate_rows(VolParams P, const FrameConsts* __restrict__ fc, FuseParams fp, const int2* __restrict__ work,
                     FrameCounters* __restrict__ ctr, const AuxTables* __restrict__ aux,
                     const float2* __restrict__ pix_f, const double* __restrict__ pix_dm,
                     const double* __restrict__ pix_var, const double* __restrict__ pix_w,
                     const int32_t* __restrict__ slot_key, uint16_t* __restrict__ payload,
                     float2* __restrict__ fpay, const uint32_t* __restrict__ uniq, uint32_t* __restrict__ keybits) {
    pdl_wait();
    constexpr int M = 1 << MS, M3 = M * M * M, RPB = M * M;
    constexpr int kRing = RowRing<MS>::kEntries;
    using RV = RowVec<MS>;
    __shared__ float s_tdec[256], s_adec[256], s_thr[260];  // s_thr[k + 1] = thresh[k]; +-inf sentinels
    __shared__ uint2 s_lut[(P2 || MODE != 2) ? 1 : kAuxLut];  // variance-code lookup (codes, Kalman)
    extern __shared__ uint4 s_ring[];  // per warp kRing entries: {slot, l | cell << 9 | exact << 31, T, p}
    __shared__ RowShared sh;
    __shared__ VolParams sP;  // by reference into the (noinline) exact path without a stack copy
    __shared__ FuseParams sFp;
    if (ctr->skip) return;
    if (threadIdx.x == 0) atomicMin(&ctr->t_begin, globaltimer_ns());
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        s_tdec[i] = aux->tsdf_decode_f[i];
        s_adec[i] = aux->aux_decode_f[i];
        s_thr[i + 1] = aux->aux_thresh_f[i];
    }
    if (!P2 && MODE == 2)
        for (int i = threadIdx.x; i < aux->lut_n; i += blockDim.x) s_lut[i] = aux->lut[i];
    if (threadIdx.x == 0) row_kernel_init<M>(P, fc, fp, aux, sh, sP, sFp, s_thr);
    clear_keybits(ctr, uniq, keybits);
    __syncthreads();
    const uint32_t limit = ctr->limit, upd_base = ctr->upd_base;
    const unsigned long long n_rows = ((unsigned long long)limit + ctr->n_update) * RPB;
    const int w = fc->intr.w, h = fc->intr.h, N = P.N;
    const int lane = threadIdx.x & 31;
    uint4* ring = s_ring + (threadIdx.x >> 5) * kRing;
    uint32_t head = 0, tail = 0;  // warp-uniform ring cursors (monotone; index & (kRing - 1))
    uint32_t updated = 0, exact = 0;
    // Phase 2 on ring entries [head, head + n): lanes take one entry each.
    auto drain = [&](uint32_t n) {
        if (lane < n) {
            const uint4 e = ring[(head + lane) & (kRing - 1)];
            const uint32_t l = e.y & 0x1FF, cell = (e.y >> 9) & 0xFFFF;
            if constexpr (P2) {
                float2* cellp = fpay + (size_t)e.x * M3 + l;
                const float2 prior = *cellp;
                float2 out;
                bool have = true;
                if ((e.y >> 31) || !approx_update_f2<MODE>(prior, __uint_as_float(e.z), __uint_as_float(e.w), sh, out)) {
                    ++exact;
                    have = exact_voxel_f2<MODE>(sP, fc, sFp, slot_key[e.x], static_cast<int>(l), prior, pix_dm, pix_var,
                                                pix_w, out);
                }
                if (have) {
                    *cellp = out;
                    ++updated;
                }
            } else {
                uint32_t out;
                int code = 0;
                if ((e.y >> 31) || !approx_update<MODE>(cell, __uint_as_float(e.z), __uint_as_float(e.w), sh, s_tdec,
                                                        s_adec, s_thr, s_lut, out)) {
                    ++exact;
                    code = exact_voxel<MODE>(sP, fc, sFp, aux, slot_key[e.x], static_cast<int>(l), cell, pix_dm,
                                             pix_var, pix_w);
                    out = static_cast<uint32_t>(code);
                }
                if (code >= 0) {
                    payload[(size_t)e.x * M3 + l] = static_cast<uint16_t>(out);
                    ++updated;
                }
            }
        }
        head += n;
    };
    // Guided dynamic scheduling in units of 32 rows: kGrabUnits per atomic while plenty of work
    // remains, single units for the tail (the last grabs decide when the kernel ends).
    const uint32_t n_units = static_cast<uint32_t>((n_rows + 31) / 32);
    const uint32_t tail_units = gridDim.x * (kRowThreads / 32) * kTailUnitsPerWarp;
    // The first kStaticPct % of the units are dealt out statically (contiguous runs per warp,
    // no atomics); the rest is grabbed dynamically.
    const uint32_t n_warps = gridDim.x * (kRowThreads / 32);
    const uint32_t gwarp = blockIdx.x * (kRowThreads / 32) + (threadIdx.x >> 5);
    const uint32_t s_per_warp = static_cast<uint32_t>((static_cast<unsigned long long>(n_units) * kStaticPct) /
                                                      (100ull * n_warps));
    const uint32_t dyn_base = s_per_warp * n_warps;
    uint32_t s_next = gwarp * s_per_warp;
    const uint32_t s_end = s_next + s_per_warp;
    uint32_t seen = dyn_base;
    for (;;) {
        uint32_t grab, units;
        if (s_next < s_end) {
            grab = s_next;
            units = min(kGrabUnits, s_end - s_next);
            s_next += units;
        } else {
            const uint32_t step = seen + tail_units < n_units ? kGrabUnits : 1u;
            uint32_t g = 0;
            if (lane == 0) g = atomicAdd(&ctr->row_chunks, step);
            grab = dyn_base + __shfl_sync(0xffffffffu, g, 0);
            seen = grab + step;
            if (grab >= n_units) break;
            units = min(step, n_units - grab);
        }
        const unsigned long long grab_row = (unsigned long long)grab * 32;
        for (uint32_t sub = 0; sub < units; ++sub) {
            // ---------------- phase 1: one row per lane ----------------
            // Rows run along the block axis closest to the optical axis (sh.axis, chosen per
            // frame), so a row's voxels project to a tiny pixel footprint. Row set-up
            // (divergent), then a converged loop over the row's M voxels in which every lane
            // evaluates its voxel and in-band / uncertain voxels are appended to the warp's ring
            // right away (one ballot per voxel position: nothing held in registers).
            const unsigned long long row = grab_row + sub * 32 + lane;
            uint32_t slot = 0, rbase = 0;
            typename RV::T cells = RV::chi();
            bool fast = false, exact_row = false, small = false;
            float Axf = 0.f, Ayf = 0.f, Azh = 1.f, Azl = 0.f, half = -1.f;
            // small-footprint rows: pixel-boundary planes s(l) = s0 + l ds (> 0: the upper
            // column / row) with margins, and the (up to) 2 x 2 candidate pixels' {depth, p_k}
            float su0 = -1e30f, dsu = 0.f, mu = 0.f, sv0 = -1e30f, dsv = 0.f, mv = 0.f;
            float2 c00 = make_float2(0.f, 0.f), c10 = c00, c01 = c00, c11 = c00;
            const int lstep = sh.lstep;
            if (row < n_rows) {
                const uint32_t item = static_cast<uint32_t>(row >> (2 * MS));
                const int r = static_cast<int>(row & (RPB - 1));
                const int2 wk = work_at(work, limit, upd_base, item);
                slot = static_cast<uint32_t>(wk.x) & 0x7fffffffu;
                const bool fresh = (static_cast<uint32_t>(wk.x) >> 31) != 0;
                const int key = wk.y;
                int bx, by, bz;
                if (P.nshift >= 0) {
                    bx = key & (N - 1);
                    by = (key >> P.nshift) & (N - 1);
                    bz = key >> (2 * P.nshift);
                } else {
                    bx = key % N;
                    by = (key / N) % N;
                    bz = key / (N * N);
                }
                // the row's first voxel (local coordinates; the row coordinate is 0)
                const int ri = r & (M - 1), rj = r >> MS;
                int l0x, l0y, l0z;
                if (sh.axis == 0) {
                    l0x = 0, l0y = ri, l0z = rj;
                } else if (sh.axis == 1) {
                    l0x = ri, l0y = 0, l0z = rj;
                } else {
                    l0x = ri, l0y = rj, l0z = 0;
                }
                rbase = static_cast<uint32_t>(l0x + (l0y << MS) + (l0z << (2 * MS)));
                if constexpr (P2) {
                    if (fresh) {  // newly allocated block: chi (+inf, 0) (grid.hpp:77-88)
                        float2* f0 = fpay + (size_t)slot * M3 + rbase;
                        if (lstep == 1) {
                            float4* frow = reinterpret_cast<float4*>(f0);
#pragma unroll
                            for (int j = 0; j < M / 2; ++j) frow[j] = make_float4(INFINITY, 0.0f, INFINITY, 0.0f);
                        } else {
#pragma unroll
                            for (int j = 0; j < M; ++j) f0[j * lstep] = make_float2(INFINITY, 0.0f);
                        }
                    }
                } else {
                    uint16_t* c0 = payload + (size_t)slot * M3 + rbase;
                    if (lstep == 1) {
                        typename RV::T* prow = reinterpret_cast<typename RV::T*>(c0);
                        if (fresh) *prow = RV::chi();  // newly allocated block: chi-initialised (grid.cpp:87-100)
                        else cells = *prow;
                    } else if (fresh) {
#pragma unroll
                        for (int j = 0; j < M; ++j) c0[j * lstep] = kChiPayload;
                    } else {
                        cells = RV::gather(c0, lstep);
                    }
                }
                // row origin x_c = R (voxel_center) + t in FP64 (voxel_center, grid.cpp:271-273)
                const double vx = sh.ox + (i2d_exact((bx << MS) + l0x) + 0.5) * sh.voxel;
                const double vy = sh.oy + (i2d_exact((by << MS) + l0y) + 0.5) * sh.voxel;
                const double vz = sh.oz + (i2d_exact((bz << MS) + l0z) + 0.5) * sh.voxel;
                const double Ax = ((sh.R[0] * vx + sh.R[1] * vy) + sh.R[2] * vz) + sh.t[0];
                const double Ay = ((sh.R[3] * vx + sh.R[4] * vy) + sh.R[5] * vz) + sh.t[1];
                const double Az = ((sh.R[6] * vx + sh.R[7] * vy) + sh.R[8] * vz) + sh.t[2];
                Axf = static_cast<float>(Ax);
                Ayf = static_cast<float>(Ay);
                Azh = static_cast<float>(Az);
                Azl = static_cast<float>(Az - static_cast<double>(Azh));
                const float zend = fmaf(static_cast<float>(M - 1), sh.Dzf, Azh);
                const float zlo = fminf(Azh, zend) - 1e-6f, zhi = fmaxf(Azh, zend) + 1e-6f;
                const float rzlo = rcp_approx_f(zlo);
                const float X = fmaxf(fabsf(Axf), fabsf(Ayf)) + sh.Mvox, Z = fabsf(Azh) + sh.Mvox;
                const float Xq = sh.Fmax * X * rzlo;  // >= |u - cx|, |v - cy| over the row
                fast = zlo > 1e-3f && zhi < 16.0f && Xq < 2097152.0f;
                // pixel-rounding margin of the row; |u|, |v| < 2^22 guaranteed
                if (fast) {
                    const float eu = 1.6f * (0x1p-23f * Xq * (2.5f + Z * rzlo) + 0x1p-24f * sh.Wpix);
                    half = 0.5f - eu;
                    // Footprint: u, v are monotone along the row (z > 0), so every voxel's true
                    // pixel column lies in lround([min(u0, u1) - eu, max(u0, u1) + eu]).
                    const float r0 = rcp_approx_f(Azh), r1 = rcp_approx_f(zend);
                    const float xe = fmaf(static_cast<float>(M - 1), sh.Dxf, Axf);
                    const float ye = fmaf(static_cast<float>(M - 1), sh.Dyf, Ayf);
                    const float u0 = fmaf(sh.fxf, Axf * r0, sh.cxf), u1 = fmaf(sh.fxf, xe * r1, sh.cxf);
                    const float v0 = fmaf(sh.fyf, Ayf * r0, sh.cyf), v1 = fmaf(sh.fyf, ye * r1, sh.cyf);
                    const float slack = eu + 1e-3f;
                    const int cu0 = static_cast<int>(floorf(fminf(u0, u1) - slack + 0.5f));
                    const int cu1 = static_cast<int>(floorf(fmaxf(u0, u1) + slack + 0.5f));
                    const int cv0 = static_cast<int>(floorf(fminf(v0, v1) - slack + 0.5f));
                    const int cv1 = static_cast<int>(floorf(fmaxf(v0, v1) + slack + 0.5f));
                    small = cu1 - cu0 <= 1 && cv1 - cv0 <= 1;
                    if (small) {
                        // boundary between columns cu0 and cu0 + 1 at u = cu0 + 1/2: the sign of
                        // s = fx x - (cu0 + 1/2 - cx) z (z > 0), affine along the row. Error of
                        // its FP32 evaluation (inputs rounded once, products, the fma chain):
                        // <= 2^-24 * 6 * (fx X + |b| Z + M voxel (fx + |b|)), plus 1e-9 for the
                        // reference's own FP64 rounding of x_c and u.
                        if (cu1 > cu0) {
                            const float b = static_cast<float>((static_cast<double>(cu0) + 0.5) - sh.cx);
                            su0 = fmaf(sh.fxf, Axf, -(b * Azh));
                            dsu = fmaf(sh.fxf, sh.Dxf, -(b * sh.Dzf));
                            mu = 0x1p-24f * 6.0f *
                                     (sh.fxf * X + fabsf(b) * Z + sh.Mvox * (sh.fxf + fabsf(b))) + 1e-9f;
                        }
                        if (cv1 > cv0) {
                            const float b = static_cast<float>((static_cast<double>(cv0) + 0.5) - sh.cy);
                            sv0 = fmaf(sh.fyf, Ayf, -(b * Azh));
                            dsv = fmaf(sh.fyf, sh.Dyf, -(b * sh.Dzf));
                            mv = 0x1p-24f * 6.0f *
                                     (sh.fyf * X + fabsf(b) * Z + sh.Mvox * (sh.fyf + fabsf(b))) + 1e-9f;
                        }
                        // candidate pixels (outside the image: no measurement, fusion.cpp:93-95)
                        const bool u0in = cu0 >= 0 && cu0 < w, u1in = cu1 > cu0 && cu1 >= 0 && cu1 < w;
                        const bool v0in = cv0 >= 0 && cv0 < h, v1in = cv1 > cv0 && cv1 >= 0 && cv1 < h;
                        if (u0in && v0in) c00 = pix_f[cv0 * w + cu0];
                        if (u1in && v0in) c10 = pix_f[cv0 * w + cu1];
                        if (u0in && v1in) c01 = pix_f[cv1 * w + cu0];
                        if (u1in && v1in) c11 = pix_f[cv1 * w + cu1];
                    }
                } else {
                    // row near / across the camera plane, or very far: exact path for all its voxels
                    exact_row = !(zhi < -1e-3f);
                }
            }
            const float Dxf = sh.Dxf, Dyf = sh.Dyf, Dzf = sh.Dzf;
            const float fxf = sh.fxf, fyf = sh.fyf, cxf = sh.cxf, cyf = sh.cyf;
            const float thr_in = sh.thr_in, thr_out = sh.thr_out;
            const unsigned lt_mask = (1u << lane) - 1u;
            // every lane small (or without work): the plane-test loop, else the general one
            const bool warp_small = __all_sync(0xffffffffu, small || (!fast && !exact_row));
            if (warp_small) {
#pragma unroll
                for (int lx = 0; lx < M; ++lx) {
                    const float fl = static_cast<float>(lx);
                    const float su = fmaf(fl, dsu, su0), sv = fmaf(fl, dsv, sv0);
                    const bool iu = su > 0.0f, iv = sv > 0.0f;
                    const bool cert = fabsf(su) > mu && fabsf(sv) > mv;
                    const float2 px = iv ? (iu ? c11 : c01) : (iu ? c10 : c00);
                    const float t = (px.x - Azh) - (lx == 0 ? Azl : fmaf(fl, Dzf, Azl));
                    const float at = fabsf(t);
                    const bool meas = small && px.x > 0.0f;
                    const bool in = meas && cert && at < thr_in;
                    const bool unc = small && (!cert || (meas && !(at < thr_in) && !(at > thr_out)));
                    const bool q = in || unc;
                    const unsigned bal = __ballot_sync(0xffffffffu, q);
                    if (q) {
                        const uint32_t meta = (rbase + lx * lstep) | (P2 ? 0u : (RV::cell(cells, lx) << 9)) |
                                              (unc ? 0x80000000u : 0u);
                        ring[(tail + __popc(bal & lt_mask)) & (kRing - 1)] =
                            make_uint4(slot, meta, __float_as_uint(t), __float_as_uint(px.y));
                    }
                    tail += __popc(bal);
                    if (kRing < 32 * M + 31 && lx == M / 2 - 1) {  // half-row drain (small ring)
                        __syncwarp();
                        while (tail - head >= 32) drain(32);
                        __syncwarp();
                    }
                }
            } else {
#pragma unroll
                for (int lx = 0; lx < M; ++lx) {
                    // explicit fma: one rounding per coordinate (the bounds above assume <= 2)
                    const float xf = lx == 0 ? Axf : fmaf(static_cast<float>(lx), Dxf, Axf);
                    const float yf = lx == 0 ? Ayf : fmaf(static_cast<float>(lx), Dyf, Ayf);
                    const float zf = lx == 0 ? Azh : fmaf(static_cast<float>(lx), Dzf, Azh);
                    const float rz = rcp_approx_f(zf);
                    const float uf = fmaf(fxf, xf * rz, cxf), vf = fmaf(fyf, yf * rz, cyf);
                    const float tu = __fadd_rn(uf, kMagic23), tv = __fadd_rn(vf, kMagic23);
                    const bool cert = fabsf(__fsub_rn(uf, __fsub_rn(tu, kMagic23))) < half &&
                                      fabsf(__fsub_rn(vf, __fsub_rn(tv, kMagic23))) < half;
                    const uint32_t u = static_cast<uint32_t>(__float_as_int(tu) - __float_as_int(kMagic23));
                    const uint32_t v = static_cast<uint32_t>(__float_as_int(tv) - __float_as_int(kMagic23));
                    const bool inimg = fast && cert && u < (uint32_t)w && v < (uint32_t)h;
                    const float2 px = pix_f[inimg ? v * (uint32_t)w + u : 0u];
                    const float t = (px.x - Azh) - (lx == 0 ? Azl : fmaf(static_cast<float>(lx), Dzf, Azl));
                    const float at = fabsf(t);
                    const bool meas = inimg && px.x > 0.0f;
                    const bool in = meas && at < thr_in;
                    const bool unc = exact_row || (fast && (!cert || (meas && !(at < thr_in) && !(at > thr_out))));
                    const bool q = in || unc;
                    const unsigned bal = __ballot_sync(0xffffffffu, q);
                    if (q) {
                        const uint32_t meta = (rbase + lx * lstep) | (P2 ? 0u : (RV::cell(cells, lx) << 9)) |
                                              (unc ? 0x80000000u : 0u);
                        ring[(tail + __popc(bal & lt_mask)) & (kRing - 1)] =
                            make_uint4(slot, meta, __float_as_uint(t), __float_as_uint(px.y));
                    }
                    tail += __popc(bal);
                    if (kRing < 32 * M + 31 && lx == M / 2 - 1) {  // half-row drain (small ring)
                        __syncwarp();
                        while (tail - head >= 32) drain(32);
                        __syncwarp();
                    }
                }
            }
            __syncwarp();  // ring entries and the fresh rows' chi stores before the drain
            // ---------------- phase 2: drain full rounds ----------------
            while (tail - head >= 32) drain(32);
            __syncwarp();  // drained slots may be refilled by the next compaction
        }
    }
    drain(tail - head);
    for (int off = 16; off > 0; off >>= 1) {
        updated += __shfl_down_sync(0xffffffffu, updated, off);
        exact += __shfl_down_sync(0xffffffffu, exact, off);
    }
    if (lane == 0 && updated) atomicAdd(&ctr->voxels_updated, (unsigned long long)updated);
    if (lane == 0 && exact) atomicAdd(&ctr->exact_voxels, (unsigned long long)exact);
    if (lane == 0) atomicMax(&ctr->t_end, globaltimer_ns());
}

// ---------------------------------------------------------------------------------
// Half-block slab integrate (M = 8): the roofline kernel.
//
// Same certified decisions and FP32 evaluation as k_integrate_rows; what
// changes is the data movement. A warp's unit of work is 32 rows of one block = a half-block
// slab of 256 voxels, which is 32 contiguous x-rows of the payload (16 B each for codes, 64 B
// for float2). The slab is copied HBM -> shared memory with cp.async one unit ahead (work
// items two units ahead), phase 1 classifies voxels from registers and queues in-band ones by
// slab position, phase 2 updates them in shared memory (no global latency in the update), and
// the slab goes back to HBM as coalesced 16-byte stores. Fresh blocks are filled with chi in
// shared memory instead of being read.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

#if SF_DIAG_TIMES  // timing diagnostics: per warp {kernel entry, first unit, last unit end, units}
__device__ unsigned long long g_slab_dbg[148 * 4 * 8 * 4];
#endif
#ifndef SF_SLAB_PF
#define SF_SLAB_PF 1
#endif
constexpr bool kSlabPrefetch = SF_SLAB_PF;
#ifndef SF_REFINE
#define SF_REFINE 1
#endif
constexpr bool kRefine = SF_REFINE;  // FP64 filter on the phase-1 inputs before the full FP64 path  // work items two units ahead (else one)
constexpr int kSlabVox = 256;   // voxels per unit (32 rows of M = 8)
// CTAs per SM of the slab kernel: codes 3 (80 registers; issue-bound, more warps pay), float2 2
// (128 registers: no rematerialisation; the smaller instruction stream is latency-bound anyway)
template <bool P2>
constexpr int kSlabCtas = P2 ? 2 : kRowCtasPerSm;
constexpr int kSlabRing = 256;  // queued voxels per warp: one unit's worth, drained per unit
template <bool P2>
struct SlabSmem {
    using Cell = typename std::conditional<P2, float2, uint16_t>::type;
    static constexpr size_t kRingBytes = (kRowThreads / 32) * kSlabRing * sizeof(uint4);
    static constexpr size_t kSlabBytes = (kRowThreads / 32) * 2 * kSlabVox * sizeof(Cell);
    static constexpr size_t kBytes = kRingBytes + kSlabBytes;
};

// Offset (voxels, inside the block) of x-row q of unit half h: the slab is z in [4h, 4h + 4)
// for rows along x or y, y in [4h, 4h + 4) for rows along z.
__device__ __forceinline__ int slab_xrow(int axis, int h, int q) {
    return axis == 2 ? 64 * (q >> 2) + 32 * h + 8 * (q & 3) : 256 * h + 8 * q;
}

template <int MODE, bool P2>
__global__ void __launch_bounds__(kRowThreads, kSlabCtas<P2>)
    k_integrate_slab(VolParams P, const FrameConsts* __restrict__ fc, FuseParams fp, const int2* __restrict__ work,
                     FrameCounters* __restrict__ ctr, const AuxTables* __restrict__ aux,
                     const float2* __restrict__ pix_f, const double* __restrict__ pix_dm,
                     const double* __restrict__ pix_var, const double* __restrict__ pix_w,
                     uint16_t* __restrict__ payload, float2* __restrict__ fpay, const uint32_t* __restrict__ uniq,
                     uint32_t* __restrict__ keybits) {
    pdl_wait();
    constexpr int M = 8, MS = 3, M3 = 512;
    using Cell = typename SlabSmem<P2>::Cell;
    __shared__ float s_tdec[256], s_adec[256], s_thr[260];  // s_thr[k + 1] = thresh[k]; +-inf sentinels
    __shared__ uint2 s_lut[(P2 || MODE != 2) ? 1 : kAuxLut];  // variance-code lookup (codes, Kalman)
    extern __shared__ __align__(128) uint4 s_dyn[];  // rings (uint4 {pos | exact << 31, T, p, 0}), then the slabs
    __shared__ RowShared sh;
    __shared__ VolParams sP;
    __shared__ FuseParams sFp;
    if (ctr->skip) return;
#if SF_DIAG_TIMES
    const unsigned long long t_entry = globaltimer_ns();
    unsigned long long t_first = 0, n_done = 0;
#endif
    if (threadIdx.x == 0) atomicMin(&ctr->t_begin, globaltimer_ns());
    // The first units' work items and slab copies are issued before the per-frame constants are
    // set up (they need only the row axis), so their latency overlaps the prologue.
    const uint32_t limit = ctr->limit, upd_base = ctr->upd_base;
    const uint32_t n_units = (limit + ctr->n_update) * 2u;
    const int w = fc->intr.w, h = fc->intr.h, N = P.N;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint4* ring = s_dyn + warp * kSlabRing;
    Cell* slabs = reinterpret_cast<Cell*>(reinterpret_cast<char*>(s_dyn) + SlabSmem<P2>::kRingBytes) +
                  warp * 2 * kSlabVox;
    const int axis = row_axis(fc->inv);
    // slab position of this lane's row: voxel l at pos0 + l * pstride (x-row q holds 8 voxels)
    const int pstride = axis == 0 ? 1 : axis == 1 ? 8 : 32;
    const int pos0 = axis == 0 ? 8 * lane : axis == 1 ? 64 * (lane >> 3) + (lane & 7) : 8 * (lane >> 3) + (lane & 7);
    uint32_t updated = 0, exact = 0;

    // ---- unit supply: a static share per warp, then guided dynamic grabs ----
    const uint32_t n_warps = gridDim.x * (kRowThreads / 32);
    const uint32_t gwarp = blockIdx.x * (kRowThreads / 32) + warp;
    const uint32_t s_per_warp =
        static_cast<uint32_t>((static_cast<unsigned long long>(n_units) * kStaticPct) / (100ull * n_warps));
    const uint32_t dyn_base = s_per_warp * n_warps;
    const uint32_t tail_units = n_warps * kTailUnitsPerWarp;
    uint32_t s_next = gwarp * s_per_warp;
    const uint32_t s_end = s_next + s_per_warp;
    uint32_t d_lo = 0, d_hi = 0, seen = dyn_base;
    bool done = false;
    auto take = [&]() -> uint32_t {
        if (s_next < s_end) return s_next++;
        if (d_lo < d_hi) return d_lo++;
        if (done) return n_units;
        const uint32_t step = seen + tail_units < n_units ? kGrabUnits : 1u;
        uint32_t g = 0;
        if (lane == 0) g = atomicAdd(&ctr->row_chunks, step);
        g = dyn_base + __shfl_sync(0xffffffffu, g, 0);
        seen = g + step;
        if (g >= n_units) {
            done = true;
            return n_units;
        }
        d_lo = g + 1;
        d_hi = min(g + step, n_units);
        return g;
    };
    auto load_item = [&](uint32_t u) -> int2 {
        return u < n_units ? work_at(work, limit, upd_base, u >> 1) : make_int2(0, 0);
    };
    // Slab of unit u into buffer b: cp.async of this lane's x-row, or chi for a fresh block.
    // float2: 16-byte chunk c = lane + 32 j of the slab is quarter (c & 3) of x-row c >> 2, so a
    // warp's accesses are consecutive in shared memory (no bank conflicts) and in global memory.
    auto issue_slab = [&](uint32_t u, int2 wk, int b) {
        if (u >= n_units) return;
        const uint32_t slot = static_cast<uint32_t>(wk.x) & 0x7fffffffu;
        const bool fresh_blk = (static_cast<uint32_t>(wk.x) >> 31) != 0;  // chi (grid.cpp:87-100, grid.hpp:77-88)
        if constexpr (P2) {
            uint4* d4 = reinterpret_cast<uint4*>(slabs + b * kSlabVox) + lane;
            // chunk j: x-row (lane >> 2) + 8 j, whose offset is linear in j (64 voxels per step
            // for rows along x or y, 128 for rows along z)
            const float2* g = fpay + (size_t)slot * M3 + slab_xrow(axis, static_cast<int>(u & 1), lane >> 2) +
                              2 * (lane & 3);
            const int gstep = axis == 2 ? 128 : 64;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (fresh_blk)
                    d4[32 * j] = make_uint4(__float_as_uint(INFINITY), 0u, __float_as_uint(INFINITY), 0u);
                else
                    cp_async16(d4 + 32 * j, g + j * gstep);
            }
        } else {
            Cell* dst = slabs + b * kSlabVox + 8 * lane;
            if (fresh_blk)
                *reinterpret_cast<uint4*>(dst) = make_uint4(0x00800080u, 0x00800080u, 0x00800080u, 0x00800080u);
            else
                cp_async16(dst, payload + (size_t)slot * M3 + slab_xrow(axis, static_cast<int>(u & 1), lane));
        }
    };

    uint32_t u0 = take();
    int2 wk0 = load_item(u0);
    uint32_t u1 = take();
    int2 wk1 = load_item(u1);
    issue_slab(u0, wk0, 0);
    cp_async_commit();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        s_tdec[i] = aux->tsdf_decode_f[i];
        s_adec[i] = aux->aux_decode_f[i];
        s_thr[i + 1] = aux->aux_thresh_f[i];
    }
    if (!P2 && MODE == 2)
        for (int i = threadIdx.x; i < aux->lut_n; i += blockDim.x) s_lut[i] = aux->lut[i];
    if (threadIdx.x == 0) row_kernel_init<M>(P, fc, fp, aux, sh, sP, sFp, s_thr);
    __syncthreads();
    for (int it = 0; u0 < n_units; ++it) {
        uint32_t u2 = n_units;
        int2 wk2 = make_int2(0, 0);
        if (kSlabPrefetch) {
            u2 = take();
            wk2 = load_item(u2);  // consumed by the next iteration's issue
        }
        issue_slab(u1, wk1, (it + 1) & 1);
        cp_async_commit();
        cp_async_wait<1>();  // this unit's slab has landed (the next one may still be in flight)
        __syncwarp();
        Cell* slab = slabs + (it & 1) * kSlabVox;
#if SF_DIAG_TIMES
        if (it == 0) t_first = globaltimer_ns();
        ++n_done;
#endif
        const uint32_t slot = static_cast<uint32_t>(wk0.x) & 0x7fffffffu;
        const bool fresh = (static_cast<uint32_t>(wk0.x) >> 31) != 0;
        const int key = wk0.y;
        const int hh = static_cast<int>(u0 & 1);
        // ---------------- phase 1: one row per lane (as k_integrate_rows) ----------------
        uint32_t tail = 0;
        {
            bool fast = false, exact_row = false, small = false;
            float Axf = 0.f, Ayf = 0.f, Azh = 1.f, Azl = 0.f, half = -1.f;
            float su0 = -1e30f, dsu = 0.f, mu = 0.f, sv0 = -1e30f, dsv = 0.f, mv = 0.f;
            float2 c00 = make_float2(0.f, 0.f), c10 = c00, c01 = c00, c11 = c00;
            int bx, by, bz;
            if (P.nshift >= 0) {
                bx = key & (N - 1);
                by = (key >> P.nshift) & (N - 1);
                bz = key >> (2 * P.nshift);
            } else {
                bx = key % N;
                by = (key / N) % N;
                bz = key / (N * N);
            }
            const int r = 32 * hh + lane;
            const int ri = r & (M - 1), rj = r >> MS;
            int l0x, l0y, l0z;
            if (axis == 0) {
                l0x = 0, l0y = ri, l0z = rj;
            } else if (axis == 1) {
                l0x = ri, l0y = 0, l0z = rj;
            } else {
                l0x = ri, l0y = rj, l0z = 0;
            }
            // row origin x_c = R (voxel_center) + t in FP64 (voxel_center, grid.cpp:271-273)
            const double vx = sh.ox + (i2d_exact((bx << MS) + l0x) + 0.5) * sh.voxel;
            const double vy = sh.oy + (i2d_exact((by << MS) + l0y) + 0.5) * sh.voxel;
            const double vz = sh.oz + (i2d_exact((bz << MS) + l0z) + 0.5) * sh.voxel;
            const double Ax = ((sh.R[0] * vx + sh.R[1] * vy) + sh.R[2] * vz) + sh.t[0];
            const double Ay = ((sh.R[3] * vx + sh.R[4] * vy) + sh.R[5] * vz) + sh.t[1];
            const double Az = ((sh.R[6] * vx + sh.R[7] * vy) + sh.R[8] * vz) + sh.t[2];
            Axf = static_cast<float>(Ax);
            Ayf = static_cast<float>(Ay);
            Azh = static_cast<float>(Az);
            Azl = static_cast<float>(Az - static_cast<double>(Azh));
            const float zend = fmaf(static_cast<float>(M - 1), sh.Dzf, Azh);
            const float zlo = fminf(Azh, zend) - 1e-6f, zhi = fmaxf(Azh, zend) + 1e-6f;
            const float rzlo = rcp_approx_f(zlo);
            const float X = fmaxf(fabsf(Axf), fabsf(Ayf)) + sh.Mvox, Z = fabsf(Azh) + sh.Mvox;
            const float Xq = sh.Fmax * X * rzlo;  // >= |u - cx|, |v - cy| over the row
            fast = zlo > 1e-3f && zhi < 16.0f && Xq < 2097152.0f;
            if (fast) {
                // pixel-rounding margin of the row and its pixel footprint
                const float eu = 1.6f * (0x1p-23f * Xq * (2.5f + Z * rzlo) + 0x1p-24f * sh.Wpix);
                half = 0.5f - eu;
                const float r0 = rcp_approx_f(Azh), r1 = rcp_approx_f(zend);
                const float xe = fmaf(static_cast<float>(M - 1), sh.Dxf, Axf);
                const float ye = fmaf(static_cast<float>(M - 1), sh.Dyf, Ayf);
                const float u0f = fmaf(sh.fxf, Axf * r0, sh.cxf), u1f = fmaf(sh.fxf, xe * r1, sh.cxf);
                const float v0f = fmaf(sh.fyf, Ayf * r0, sh.cyf), v1f = fmaf(sh.fyf, ye * r1, sh.cyf);
                const float slack = eu + 1e-3f;
                const int cu0 = static_cast<int>(floorf(fminf(u0f, u1f) - slack + 0.5f));
                const int cu1 = static_cast<int>(floorf(fmaxf(u0f, u1f) + slack + 0.5f));
                const int cv0 = static_cast<int>(floorf(fminf(v0f, v1f) - slack + 0.5f));
                const int cv1 = static_cast<int>(floorf(fmaxf(v0f, v1f) + slack + 0.5f));
                small = cu1 - cu0 <= 1 && cv1 - cv0 <= 1;
                if (small) {
                    // pixel-boundary planes (see k_integrate_rows)
                    if (cu1 > cu0) {
                        const float b = static_cast<float>((static_cast<double>(cu0) + 0.5) - sh.cx);
                        su0 = fmaf(sh.fxf, Axf, -(b * Azh));
                        dsu = fmaf(sh.fxf, sh.Dxf, -(b * sh.Dzf));
                        mu = 0x1p-24f * 6.0f * (sh.fxf * X + fabsf(b) * Z + sh.Mvox * (sh.fxf + fabsf(b))) + 1e-9f;
                    }
                    if (cv1 > cv0) {
                        const float b = static_cast<float>((static_cast<double>(cv0) + 0.5) - sh.cy);
                        sv0 = fmaf(sh.fyf, Ayf, -(b * Azh));
                        dsv = fmaf(sh.fyf, sh.Dyf, -(b * sh.Dzf));
                        mv = 0x1p-24f * 6.0f * (sh.fyf * X + fabsf(b) * Z + sh.Mvox * (sh.fyf + fabsf(b))) + 1e-9f;
                    }
                    const bool u0in = cu0 >= 0 && cu0 < w, u1in = cu1 > cu0 && cu1 >= 0 && cu1 < w;
                    const bool v0in = cv0 >= 0 && cv0 < h, v1in = cv1 > cv0 && cv1 >= 0 && cv1 < h;
                    if (u0in && v0in) c00 = pix_f[cv0 * w + cu0];
                    if (u1in && v0in) c10 = pix_f[cv0 * w + cu1];
                    if (u0in && v1in) c01 = pix_f[cv1 * w + cu0];
                    if (u1in && v1in) c11 = pix_f[cv1 * w + cu1];
                }
            } else {
                exact_row = !(zhi < -1e-3f);
            }
            const float Dxf = sh.Dxf, Dyf = sh.Dyf, Dzf = sh.Dzf;
            const float fxf = sh.fxf, fyf = sh.fyf, cxf = sh.cxf, cyf = sh.cyf;
            const float thr_in = sh.thr_in, thr_out = sh.thr_out;
            const unsigned lt_mask = (1u << lane) - 1u;
            const bool warp_small = __all_sync(0xffffffffu, small || (!fast && !exact_row));
            if (warp_small) {
                // d - z_hi per candidate pixel; no measurement (no depth, or a lane without a
                // small row) -> +1e30, which every voxel finds out of band
                const float tb00 = small && c00.x > 0.0f ? c00.x - Azh : 1e30f;
                const float tb10 = small && c10.x > 0.0f ? c10.x - Azh : 1e30f;
                const float tb01 = small && c01.x > 0.0f ? c01.x - Azh : 1e30f;
                const float tb11 = small && c11.x > 0.0f ? c11.x - Azh : 1e30f;
#pragma unroll
                for (int lx = 0; lx < M; ++lx) {
                    const float fl = static_cast<float>(lx);
                    const float su = fmaf(fl, dsu, su0), sv = fmaf(fl, dsv, sv0);
                    const bool iu = su > 0.0f, iv = sv > 0.0f;
                    const bool cert = fabsf(su) > mu && fabsf(sv) > mv;  // lanes without a small row: su0, sv0 = -1e30
                    const float tb = iv ? (iu ? tb11 : tb01) : (iu ? tb10 : tb00);
                    const float t = tb - (lx == 0 ? Azl : fmaf(fl, Dzf, Azl));
                    const bool gt = fabsf(t) > thr_out;
                    // in: cert && |t| < thr_in; uncertain: !cert, or |t| between the thresholds
                    const bool q = !cert || !gt;
                    const unsigned bal = __ballot_sync(0xffffffffu, q);
                    if (q) {
                        const bool unc = !cert || !(fabsf(t) < thr_in);
                        const float pk = iv ? (iu ? c11.y : c01.y) : (iu ? c10.y : c00.y);
                        ring[tail + __popc(bal & lt_mask)] =
                            make_uint4(static_cast<uint32_t>(pos0 + lx * pstride) | (unc ? 0x80000000u : 0u),
                                       __float_as_uint(t), __float_as_uint(pk), 0u);
                    }
                    tail += __popc(bal);
                }
            } else {
#pragma unroll
                for (int lx = 0; lx < M; ++lx) {
                    const float xf = lx == 0 ? Axf : fmaf(static_cast<float>(lx), Dxf, Axf);
                    const float yf = lx == 0 ? Ayf : fmaf(static_cast<float>(lx), Dyf, Ayf);
                    const float zf = lx == 0 ? Azh : fmaf(static_cast<float>(lx), Dzf, Azh);
                    const float rz = rcp_approx_f(zf);
                    const float uf = fmaf(fxf, xf * rz, cxf), vf = fmaf(fyf, yf * rz, cyf);
                    const float tu = __fadd_rn(uf, kMagic23), tv = __fadd_rn(vf, kMagic23);
                    const bool cert = fabsf(__fsub_rn(uf, __fsub_rn(tu, kMagic23))) < half &&
                                      fabsf(__fsub_rn(vf, __fsub_rn(tv, kMagic23))) < half;
                    const uint32_t u = static_cast<uint32_t>(__float_as_int(tu) - __float_as_int(kMagic23));
                    const uint32_t v = static_cast<uint32_t>(__float_as_int(tv) - __float_as_int(kMagic23));
                    const bool inimg = fast && cert && u < (uint32_t)w && v < (uint32_t)h;
                    const float2 px = pix_f[inimg ? v * (uint32_t)w + u : 0u];
                    const float t = (px.x - Azh) - (lx == 0 ? Azl : fmaf(static_cast<float>(lx), Dzf, Azl));
                    const float at = fabsf(t);
                    const bool meas = inimg && px.x > 0.0f;
                    const bool in = meas && at < thr_in;
                    const bool unc = exact_row || (fast && (!cert || (meas && !(at < thr_in) && !(at > thr_out))));
                    const bool q = in || unc;
                    const unsigned bal = __ballot_sync(0xffffffffu, q);
                    if (q)
                        ring[tail + __popc(bal & lt_mask)] =
                            make_uint4(static_cast<uint32_t>(pos0 + lx * pstride) | (unc ? 0x80000000u : 0u),
                                       __float_as_uint(t), __float_as_uint(px.y), 0u);
                    tail += __popc(bal);
                }
            }
        }
        __syncwarp();  // ring entries before the drain
        // ---------------- phase 2: update the queued voxels in shared memory ----------------
        bool wrote = false;
        for (uint32_t head = 0; head < tail; head += 32) {
            if (head + lane < tail) {
                const uint4 e = ring[head + lane];
                const int pos = static_cast<int>(e.x & 0xFFu);
                Cell* cellp = slab + pos;
                const bool unc = (e.x >> 31) != 0;
                if constexpr (P2) {
                    const float2 prior = *cellp;
                    float2 out;
                    bool have = true;
                    if (unc || !approx_update_f2<MODE>(prior, __uint_as_float(e.y), __uint_as_float(e.z), sh, out)) {
                        ++exact;
                        const int l = slab_xrow(axis, hh, pos >> 3) + (pos & 7);
                        have = exact_voxel_f2<MODE>(sP, fc, sFp, key, l, prior, pix_dm, pix_var, pix_w, out);
                    }
                    if (have) {
                        *cellp = out;
                        ++updated;
                        wrote = true;
                    }
                } else {
                    const uint32_t cell = *cellp;
                    uint32_t out;
                    int code = 0;
                    if (unc || (!approx_update<MODE>(cell, __uint_as_float(e.y), __uint_as_float(e.z), sh, s_tdec,
                                                     s_adec, s_thr, s_lut, out) &&
                                !(kRefine && refine_update<MODE>(sP, sFp, aux, cell, __uint_as_float(e.y),
                                                                 __uint_as_float(e.z), sh.eT, out)))) {
                        ++exact;
                        const int l = slab_xrow(axis, hh, pos >> 3) + (pos & 7);
                        code = exact_voxel<MODE>(sP, fc, sFp, aux, key, l, cell, pix_dm, pix_var, pix_w);
                        out = static_cast<uint32_t>(code);
                    }
                    if (code >= 0) {
                        *cellp = static_cast<uint16_t>(out);
                        ++updated;
                        wrote = true;
                    }
                }
            }
        }
        // ---------------- write-back: 32 x-rows, coalesced 16-byte stores ----------------
        if (__any_sync(0xffffffffu, wrote) || fresh) {
            __syncwarp();
            if constexpr (P2) {
                const uint4* s4 = reinterpret_cast<const uint4*>(slab) + lane;
                float2* g = fpay + (size_t)slot * M3 + slab_xrow(axis, hh, lane >> 2) + 2 * (lane & 3);
                const int gstep = axis == 2 ? 128 : 64;
#pragma unroll
                for (int j = 0; j < 4; ++j) *reinterpret_cast<uint4*>(g + j * gstep) = s4[32 * j];
            } else {
                const uint4* s4 = reinterpret_cast<const uint4*>(slab + 8 * lane);
                *reinterpret_cast<uint4*>(payload + (size_t)slot * M3 + slab_xrow(axis, hh, lane)) = s4[0];
            }
        }
        __syncwarp();  // ring and slab reuse
        u0 = u1;
        wk0 = wk1;
        if (kSlabPrefetch) {
            u1 = u2;
            wk1 = wk2;
        } else {
            u1 = take();
            wk1 = load_item(u1);
        }
    }
    cp_async_wait<0>();
    clear_keybits(ctr, uniq, keybits);  // in the tail, where warps run out of units
#if SF_DIAG_TIMES
    if (lane == 0 && gwarp < 148 * 4 * 8) {
        unsigned long long* d = g_slab_dbg + 4 * gwarp;
        d[0] = t_entry;
        d[1] = t_first;
        d[2] = globaltimer_ns();
        d[3] = n_done;
    }
#endif
    for (int off = 16; off > 0; off >>= 1) {
        updated += __shfl_down_sync(0xffffffffu, updated, off);
        exact += __shfl_down_sync(0xffffffffu, exact, off);
    }
    if (lane == 0 && updated) atomicAdd(&ctr->voxels_updated, (unsigned long long)updated);
    if (lane == 0 && exact) atomicAdd(&ctr->exact_voxels, (unsigned long long)exact);
    if (lane == 0) atomicMax(&ctr->t_end, globaltimer_ns());
}
#if SF_DIAG_TIMES
extern "C" int sf_debug_slab_times(unsigned long long* out, int n) {
    return (int)cudaMemcpyFromSymbol(out, g_slab_dbg, n * sizeof(unsigned long long));
}
#endif

// ---- measurement refinement (fusion.cpp:99-143) ---------------------------------------
// glibc's hypot (dbl-64, the non-FMA build of Borges' corrected algorithm used by the
// reference's libm; checked against libm on 5e4 random pairs, tests/test_oracle_cpu.py):
// not correctly rounded, so the exact operation sequence matters.
__device__ __forceinline__ double glibc_hypot_kernel(double ax, double ay) {
    double h = sqrt(ax * ax + ay * ay);
    double t1, t2;
    if (h <= 2.0 * ay) {
        const double delta = h - ay;
        t1 = ax * (2.0 * delta - ax);
        t2 = (delta - 2.0 * (ax - ay)) * delta;
    } else {
        const double delta = h - ax;
        t1 = 2.0 * delta * (ax - 2.0 * ay);
        t2 = (4.0 * delta - ay) * ay + delta * delta;
    }
    h -= (t1 + t2) / (2.0 * h);
    return h;
}
__device__ double glibc_hypot(double x, double y) {
    if (!isfinite(x) || !isfinite(y)) {
        if (isinf(x) || isinf(y)) return INFINITY;
        return x + y;
    }
    x = fabs(x);
    y = fabs(y);
    double ax = x < y ? y : x, ay = x < y ? x : y;
    constexpr double kScale = 0x1p-600, kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54;
    if (ax > kLarge) {
        if (ay <= ax * kEps) return ax + ay;
        return glibc_hypot_kernel(ax * kScale, ay * kScale) / kScale;
    }
    if (ay < kTiny) {
        if (ax >= ay / kEps) return ax + ay;
        return glibc_hypot_kernel(ax / kScale, ay / kScale) * kScale;
    }
    if (ay <= ax * kEps) return ax + ay;
    return glibc_hypot_kernel(ax, ay);
}
// bilinear depth (fusion.cpp:102-112)
__device__ double depth_interp(const float* __restrict__ depth, int w, int h, double uu, double vv) {
    const int u0 = ref_floor_int(uu), v0 = ref_floor_int(vv);
    if (!(u0 >= 0 && v0 >= 0 && u0 < w && v0 < h) || !(u0 + 1 >= 0 && v0 + 1 >= 0 && u0 + 1 < w && v0 + 1 < h))
        return 0.0;
    const float d00 = depth[(size_t)v0 * w + u0], d10 = depth[(size_t)v0 * w + u0 + 1];
    const float d01 = depth[(size_t)(v0 + 1) * w + u0], d11 = depth[(size_t)(v0 + 1) * w + u0 + 1];
    if (d00 <= 0.0f || d10 <= 0.0f || d01 <= 0.0f || d11 <= 0.0f) return 0.0;
    const double fu = uu - u0, fv = vv - v0;
    return (d00 * (1.0 - fu) + d10 * fu) * (1.0 - fv) + (d01 * (1.0 - fu) + d11 * fu) * fv;
}
__device__ double refine_dist_sq(const float* __restrict__ depth, const Intr& I, double uu, double vv, d3 xc) {
    const double d = depth_interp(depth, I.w, I.h, uu, vv);
    if (d <= 0.0) return INFINITY;
    return sqnorm(sub(unproject(I, uu, vv, d), xc));
}
// Sub-pixel descent (fusion.cpp:113-141). Returns true when it moved the measurement: then
// (u, v), measured and tsdf_k are the refined ones.
__device__ __noinline__ bool refine_measurement(const float* __restrict__ depth, const Intr& I, int steps, double pu,
                                                double pv, d3 xc, int& u, int& v, double& measured, double& tsdf_k) {
    double cu = pu, cv = pv;
    double best = refine_dist_sq(depth, I, cu, cv, xc);
    if (!isfinite(best)) return false;
    const double hh = 0.5;  // gradient probe and step length, pixels
    for (int step = 0; step < steps; ++step) {
        const double gu = refine_dist_sq(depth, I, cu + hh, cv, xc) - refine_dist_sq(depth, I, cu - hh, cv, xc);
        const double gv = refine_dist_sq(depth, I, cu, cv + hh, xc) - refine_dist_sq(depth, I, cu, cv - hh, xc);
        const double norm = glibc_hypot(gu, gv);
        if (!isfinite(norm) || norm == 0.0) break;
        const double nu = cu - hh * gu / norm;
        const double nv = cv - hh * gv / norm;
        const double cand = refine_dist_sq(depth, I, nu, nv, xc);
        if (!(cand < best)) break;
        best = cand;
        cu = nu;
        cv = nv;
    }
    const double d_here = depth_interp(depth, I.w, I.h, cu, cv);
    if (!(d_here > 0.0)) return false;
    u = ref_lround_int(cu);
    v = ref_lround_int(cv);
    measured = d_here;
    tsdf_k = (d_here >= xc.z ? 1.0 : -1.0) * sqrt(best);
    return true;
}

template <int MODE, bool FLOATP>
__global__ void __launch_bounds__(kThreads)
    k_integrate(VolParams P, const FrameConsts* __restrict__ fc, FuseParams fp, const int2* __restrict__ work,
                const FrameCounters* __restrict__ ctr, const AuxTables* __restrict__ aux,
                const float* __restrict__ depth, const double* __restrict__ pix_var, const double* __restrict__ pix_w,
                const uint8_t* __restrict__ pix_ok, uint16_t* __restrict__ payload, float2* __restrict__ fpayload,
                unsigned long long* __restrict__ voxels_updated, const uint32_t* __restrict__ uniq,
                uint32_t* __restrict__ keybits, const float* __restrict__ sigma, const double* __restrict__ pix_q) {
    __shared__ double s_tdec[256], s_adec[256], s_thr[256];
    if (ctr->skip) return;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        s_tdec[i] = aux->tsdf_decode[i];
        s_adec[i] = aux->aux_decode[i];
        s_thr[i] = aux->aux_thresh[i];
    }
    __syncthreads();
    const Pose inv = fc->inv;
    const Intr intr = fc->intr;
    const double delta = P.delta;
    const int w = intr.w, h = intr.h;
    clear_keybits(ctr, uniq, keybits);
    const uint32_t limit = ctr->limit, upd_base = ctr->upd_base;
    const unsigned long long n_work = (unsigned long long)limit + ctr->n_update;
    const unsigned long long total = n_work * (unsigned long long)P.M3;
    const int M = P.M, MM = P.M * P.M, N = P.N;
    unsigned long long updated = 0;
    for (unsigned long long g = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; g < total;
         g += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long item = g / (unsigned)P.M3;
        const int l = static_cast<int>(g - item * (unsigned)P.M3);
        const int2 wk = work_at(work, limit, upd_base, static_cast<uint32_t>(item));
        const uint32_t slot = static_cast<uint32_t>(wk.x) & 0x7fffffffu;
        const bool fresh = (static_cast<uint32_t>(wk.x) >> 31) != 0;
        const int key = wk.y;
        const int bx = key % N, by = (key / N) % N, bz = key / (N * N);
        const int lx = l % M, ly = (l / M) % M, lz = l / MM;
        const size_t pidx = (size_t)slot * P.M3 + l;
        // estimate_measurement (fusion.cpp:81-99, 145)
        const d3 xc = apply(inv, voxel_center(P, bx * M + lx, by * M + ly, bz * M + lz));
        bool meas = false;
        double tsdf_k = 0.0;
        size_t pix = 0;
        double pu, pv;
        bool refined = false;
        double r_var = 0.0, r_w = 0.0;
        if (project(intr, xc, pu, pv)) {
            int u = ref_lround_int(pu);
            int v = ref_lround_int(pv);
            if (u >= 0 && v >= 0 && u < w && v < h) {
                pix = (size_t)v * w + u;
                const float d = depth[pix];
                if (d > 0.0f) {
                    double measured = d;
                    tsdf_k = measured - xc.z;
                    if (fp.refine > 0)
                        refined = refine_measurement(depth, intr, fp.refine, pu, pv, xc, u, v, measured, tsdf_k);
                    if (!refined) {
                        meas = !(fabs(tsdf_k) > delta) && pix_ok[pix];
                    } else if (!(fabs(tsdf_k) > delta)) {
                        // measurement at the refined pixel with the interpolated depth (fusion.cpp:147-171)
                        pix = (size_t)v * w + u;
                        const double sg = fp.has_sigma && sigma[pix] > 0.0f ? static_cast<double>(sigma[pix])
                                                                             : fp.sigma0 * measured * measured;
                        r_var = dmax(sg * sg, fp.min_variance);
                        r_w = fp.w_fixed;
                        meas = true;
                        if (fp.downweight) {
                            const double q = pix_q[pix];
                            if (q < 0.2) {
                                meas = false;
                            } else {
                                r_w *= q;
                                r_var /= q;
                            }
                        }
                    }
                }
            }
        }
        if (!meas) {
            if (fresh) {
                payload[pidx] = kChiPayload;
                if (FLOATP) fpayload[pidx] = make_float2(INFINITY, 0.0f);
            }
            continue;
        }
        // prior (fusion.cpp:311-322)
        bool has_prior;
        double prior_t = 0.0, prior_a = 0.0;
        if (FLOATP) {
            const float2 f = fresh ? make_float2(INFINITY, 0.0f) : fpayload[pidx];
            has_prior = f.x < INFINITY;  // !FloatShadowGrid::is_chi
            if (has_prior) {
                prior_t = f.x;
                prior_a = f.y;
            }
        } else {
            const uint16_t cell = fresh ? kChiPayload : payload[pidx];
            const int8_t code = static_cast<int8_t>(cell & 0xFF);
            has_prior = code != kChiCode;
            if (has_prior) {
                prior_t = s_tdec[(int)code + 128];
                prior_a = s_adec[cell >> 8];
            }
        }
        // filters (fusion.cpp:237-272)
        double new_t, new_a;
        if (MODE == 0) {  // simple
            const double wk_ = refined ? r_w : pix_w[pix];
            new_t = has_prior ? (1.0 - wk_) * prior_t + wk_ * tsdf_k : tsdf_k;
            new_a = wk_;
        } else if (MODE == 1) {  // weighted
            const double wk_ = refined ? r_w : pix_w[pix];
            if (!has_prior) {
                new_t = tsdf_k;
                new_a = wk_;
            } else {
                new_t = (prior_a * prior_t + wk_ * tsdf_k) / (prior_a + wk_);
                new_a = dmin(prior_a + wk_, fp.w_max);
            }
        } else {  // kalman
            const double pk = refined ? r_var : pix_var[pix];
            if (!has_prior) {
                new_t = tsdf_k;
                new_a = pk;
            } else {
                const double predicted = prior_a + fp.q;
                const double gain = predicted / (predicted + pk);
                new_t = prior_t + gain * (tsdf_k - prior_t);
                new_a = (1.0 - gain) * predicted;
            }
        }
        const bool chi = fabs(new_t) > delta;
        uint16_t out = kChiPayload;
        if (!chi) {
            const int8_t code = quantize_tsdf(new_t, delta);
            const uint8_t ac = aux_encode_dev(P, s_thr, new_a);
            out = static_cast<uint16_t>(static_cast<uint8_t>(code)) | static_cast<uint16_t>(ac << 8);
        }
        payload[pidx] = out;
        if (FLOATP) fpayload[pidx] = chi ? make_float2(INFINITY, 0.0f) : make_float2((float)new_t, (float)new_a);
        ++updated;
    }
    // voxels_updated: warp reduction, one atomic per warp
    for (int off = 16; off > 0; off >>= 1) updated += __shfl_down_sync(0xffffffffu, updated, off);
    if ((threadIdx.x & 31) == 0 && updated) atomicAdd(voxels_updated, updated);
}

__global__ void k_fuse_finalize(FrameCounters* ctr, const VolCounters* vc) { fuse_finalize_body(ctr, vc); }

// ---------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------
static uint32_t sentinel_of(const VolParams& P) { return static_cast<uint32_t>(P.table_size); }
static int end_bit_of(const VolParams& P) {
    const uint32_t s = sentinel_of(P);
    int b = 1;
    while (b < 32 && (s >> b) != 0) ++b;
    return b;
}

size_t cub_temp_bytes_needed(uint32_t key_cap) {
    size_t a = 0, b = 0, c = 0;
    SF_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, a, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)key_cap, 0, 32));
    SF_CUDA(cub::DeviceSelect::Unique(nullptr, b, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                      (int)key_cap));
    SF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, c, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)key_cap));
    return std::max({a, b, c, (size_t)256});
}

void launch_consts(const VolParams& P, const Intr& intr, const double* d_pose, FrameConsts* d_fc, cudaStream_t s,
                   uint64_t* launches) {
    k_frame_consts<<<1, 32, 0, s>>>(P, intr, d_pose, d_fc);
    SF_LAUNCH_CHECK();
    if (launches) *launches += 1;
}

void launch_compute_normals(const float* depth, int w, int h, const Intr& intr, double sigma0, double spatial_scale,
                            float* normals, cudaStream_t s, uint64_t* launches, const int* dead_flag) {
    const dim3 blk(32, 8), grd((w + 31) / 32, (h + 7) / 8);
    k_normals<<<grd, blk, 0, s>>>(depth, w, h, intr, sigma0, spatial_scale, normals, dead_flag);
    SF_LAUNCH_CHECK();
    if (launches) *launches += 1;
}

FuseParams resolve_fuse_params(const Volume& v, const sf_fusion_params& p, bool has_sigma) {
    // FusionParams::validate (fusion.cpp:12-17) and the mode/aux checks (fusion.cpp:279-283)
    if (!(p.w_fixed > 0.0) || p.w_fixed > 1.0) throw Error(SF_INVALID_ARGUMENT, "fusion: w_fixed must be in (0, 1]");
    if (!(p.w_max > 0.0)) throw Error(SF_INVALID_ARGUMENT, "fusion: w_max must be positive");
    if (p.sigma0 < 0.0) throw Error(SF_INVALID_ARGUMENT, "fusion: sigma0 must be >= 0");
    if (p.refinement_steps < 0) throw Error(SF_INVALID_ARGUMENT, "fusion: negative refinement_steps");
    if (p.mode == 2 && v.aux.mode != 1) throw Error(SF_INVALID_ARGUMENT, "fusion: Kalman mode needs a variance-mode grid");
    if (p.mode != 2 && v.aux.mode != 0)
        throw Error(SF_INVALID_ARGUMENT, "fusion: weight-mode grid required for this fusion mode");
    if (p.mode < 0 || p.mode > 2) throw Error(SF_INVALID_ARGUMENT, "fusion: unknown mode");
    FuseParams f{};
    f.mode = p.mode;
    f.w_fixed = p.w_fixed;
    f.w_max = p.w_max;
    const double delta = v.P.delta;
    if (p.process_variance >= 0.0) {
        f.q = p.process_variance;
    } else {  // FusionParams::resolved_q (fusion.cpp:19-23)
        const double step = 0.1 * delta / kTsdfCodeRange;
        f.q = step * step;
    }
    f.sigma0 = p.sigma0;
    f.min_variance = p.min_variance;
    f.downweight = p.edge_downweight ? 1 : 0;
    f.has_sigma = has_sigma ? 1 : 0;
    f.refine = p.refinement_steps;
    return f;
}

template <int MODE, int MS, bool P2>
static void launch_integrate_rows(Volume& v, FrameBuffers& fb, const FuseParams& fp, cudaStream_t s) {
    static_assert(RowRing<MS>::kBytes <= 200 * 1024, "ring exceeds shared memory");
    static bool configured = false;  // per instantiation
    if (!configured) {
        SF_CUDA(cudaFuncSetAttribute(k_integrate_rows<MODE, MS, P2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)RowRing<MS>::kBytes));
        configured = true;
    }
    launch_pdl(k_integrate_rows<MODE, MS, P2>, dim3(148 * kRowCtasPerSm), dim3(kRowThreads), RowRing<MS>::kBytes, s,
               v.P, fb.fc, fp, fb.work, fb.ctr, v.d_aux, fb.pix_f, fb.pix_dm, fb.pix_var, fb.pix_w, v.d_slot_key,
               v.d_payload, v.d_fpayload, fb.keys_unique, v.d_keybits);
}

template <int MODE, bool P2>
static void launch_integrate_slab(Volume& v, FrameBuffers& fb, const FuseParams& fp, cudaStream_t s) {
    static bool configured = false;  // per instantiation
    if (!configured) {
        SF_CUDA(cudaFuncSetAttribute(k_integrate_slab<MODE, P2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)SlabSmem<P2>::kBytes));
        configured = true;
    }
    launch_pdl(k_integrate_slab<MODE, P2>, dim3(148 * kSlabCtas<P2>), dim3(kRowThreads), SlabSmem<P2>::kBytes, s,
               v.P, fb.fc, fp, fb.work, fb.ctr, v.d_aux, fb.pix_f, fb.pix_dm, fb.pix_var, fb.pix_w, v.d_payload,
               v.d_fpayload, fb.keys_unique, v.d_keybits);
}

// Frame prep of fuse_frame (depends only on the frame): normals with the fusion options
// (sigma0, spatial_scale = 0.25 * delta; fusion.cpp:33-36), edge mask, per-pixel measurement
// factors (fusion.cpp:40-72, 148-171).
void launch_fuse_prep(Volume& v, FrameBuffers& fb, const Intr& intr, const float* depth, const float* sigma,
                      const FuseParams& fp, cudaStream_t s, uint64_t* launches, const int* dead) {
    const int w = fb.w, h = fb.h;
    const dim3 blk2(32, 8), grd2((w + 31) / 32, (h + 7) / 8);
    uint64_t n = 0;
    if (fp.downweight) {
        k_normals<<<grd2, blk2, 0, s>>>(depth, w, h, intr, fp.sigma0, 0.25 * v.P.delta, fb.normals, dead);
        SF_LAUNCH_CHECK();
        k_edge<<<grd2, blk2, 0, s>>>(depth, w, h, fp.sigma0, fb.edge, dead);
        SF_LAUNCH_CHECK();
        n += 2;
    }
    k_pixel_meas<<<grd2, blk2, 0, s>>>(depth, sigma, w, h, intr, fp, fb.normals, fb.edge, fb.pix_var, fb.pix_w,
                                        fb.pix_ok, fb.pix_dm, fb.pix_f, fb.pix_q, dead);
    SF_LAUNCH_CHECK();
    n += 1;
    if (launches) *launches += n;
}

void launch_fuse(Volume& v, FrameBuffers& fb, const Intr& intr, const float* depth, const float* sigma,
                 const FuseParams& fp, cudaStream_t s, bool export_only, uint64_t* launches, const int* dead_flag,
                 const FuseEvents* events, bool prep_done, bool caller_brackets) {
    const int w = fb.w, h = fb.h;
    const VolParams& P = v.P;
    uint64_t n = 0;
    if (!caller_brackets) {  // else the caller ran frame_consts_warp + fuse_begin_body in its own kernel
        launch_consts(P, intr, fb.pose, fb.fc, s, &n);
        k_fuse_begin<<<1, 1, 0, s>>>(fb.ctr, v.d_vc, dead_flag);
        SF_LAUNCH_CHECK();
        n += 1;
    }
    const int* dead = reinterpret_cast<const int*>(&fb.ctr->skip);
    if (!export_only && !prep_done) launch_fuse_prep(v, fb, intr, depth, sigma, fp, s, &n, dead);
    const int su = (w + fb.stride - 1) / fb.stride, sv = (h + fb.stride - 1) / fb.stride;
    if (export_only) {
        // select_update_blocks: the ordered lists themselves are the output -> sorted
        // unique allocate list (CUB), update list by the same visibility test.
        const uint32_t sentinel = sentinel_of(P);
        k_block_keys<<<(su * sv + kThreads - 1) / kThreads, kThreads, 0, s>>>(P, fb.fc, depth, w, h, fb.stride, su,
                                                                              sv, fb.keys, sentinel, &fb.ctr->skip);
        SF_LAUNCH_CHECK();
        size_t tb = fb.cub_temp_bytes;
        SF_CUDA(cub::DeviceRadixSort::SortKeys(fb.cub_temp, tb, fb.keys, fb.keys_sorted, (int)fb.key_cap, 0,
                                               end_bit_of(P), s));
        tb = fb.cub_temp_bytes;
        SF_CUDA(cub::DeviceSelect::Unique(fb.cub_temp, tb, fb.keys_sorted, fb.keys_unique, &fb.ctr->n_unique,
                                          (int)fb.key_cap, s));
        k_list_len<<<1, 1, 0, s>>>(fb.ctr, fb.keys_unique, sentinel);
        SF_LAUNCH_CHECK();
        k_visible<<<kPersistentCtas, kThreads, 0, s>>>(P, fb.fc, fb.ctr, v.d_vc, v.d_slot_key, fb.keys_unique, depth,
                                                       w, h, fb.work, fb.keys /* reused as export buffer */, 1);
        SF_LAUNCH_CHECK();
        n += 3 + 4;  // keys + list_len + visible + (sort, unique: >= 4 CUB kernels)
    } else {
        // fuse_frame: unordered key set + ranked new keys + work list (no global sort)
        launch_pdl(k_block_keys_set, dim3((su * sv + kThreads - 1) / kThreads), dim3(kThreads), 0, s, P, fb.fc, depth,
                   w, h, fb.stride, su, sv, v.d_keybits, fb.keys_unique, fb.ctr, v.d_table, fb.ranks, fb.flags,
                   fb.work);
        SF_LAUNCH_CHECK();
        launch_pdl(k_alloc_visible, dim3(kAllocCtas), dim3(kThreads), 0, s, P, fb.fc, fb.ctr, v.d_vc, fb.ranks,
                   fb.flags, v.d_table, v.d_free_list, v.d_slot_key, v.d_occ, fb.keys_unique, v.d_keybits, depth, w,
                   h, fb.work);
        SF_LAUNCH_CHECK();
        n += 2;
    }
    if (!export_only) {
        unsigned long long* vu = &fb.ctr->voxels_updated;
#define SF_INTEGRATE(MODE, FP)                                                                                    \
    k_integrate<MODE, FP><<<kPersistentCtas, kThreads, 0, s>>>(P, fb.fc, fp, fb.work, fb.ctr, v.d_aux, depth,       \
                                                               fb.pix_var, fb.pix_w, fb.pix_ok, v.d_payload,        \
                                                               v.d_fpayload, vu, fb.keys_unique, v.d_keybits, sigma,     \
                                                               fb.pix_q)
        const bool fpl = v.d_fpayload != nullptr;
        if (events && events->before_integrate) record_event(events->before_integrate, s);
        const bool rows_ok = (P.mshift == 3 || P.mshift == 2) && v.h_aux.fp32_ok && fp.refine == 0;
        const bool fast = v.layout == SF_PAYLOAD_CODES && rows_ok;
        const bool fast_f2 = v.layout == SF_PAYLOAD_FLOAT2 && rows_ok;
#if SF_SLAB
#define SF_INTEGRATE_ROWS(MODE, MS) \
    (MS == 3 ? launch_integrate_slab<MODE, false>(v, fb, fp, s) : launch_integrate_rows<MODE, MS, false>(v, fb, fp, s))
#define SF_INTEGRATE_ROWS_F2(MODE, MS) \
    (MS == 3 ? launch_integrate_slab<MODE, true>(v, fb, fp, s) : launch_integrate_rows<MODE, MS, true>(v, fb, fp, s))
#else
#define SF_INTEGRATE_ROWS(MODE, MS) launch_integrate_rows<MODE, MS, false>(v, fb, fp, s)
#define SF_INTEGRATE_ROWS_F2(MODE, MS) launch_integrate_rows<MODE, MS, true>(v, fb, fp, s)
#endif
        if (fast_f2) {
            if (P.mshift == 3) {
                if (fp.mode == 0) SF_INTEGRATE_ROWS_F2(0, 3);
                else if (fp.mode == 1) SF_INTEGRATE_ROWS_F2(1, 3);
                else SF_INTEGRATE_ROWS_F2(2, 3);
            } else {
                if (fp.mode == 0) SF_INTEGRATE_ROWS_F2(0, 2);
                else if (fp.mode == 1) SF_INTEGRATE_ROWS_F2(1, 2);
                else SF_INTEGRATE_ROWS_F2(2, 2);
            }
        } else if (fast) {
            if (P.mshift == 3) {
                if (fp.mode == 0) SF_INTEGRATE_ROWS(0, 3);
                else if (fp.mode == 1) SF_INTEGRATE_ROWS(1, 3);
                else SF_INTEGRATE_ROWS(2, 3);
            } else {
                if (fp.mode == 0) SF_INTEGRATE_ROWS(0, 2);
                else if (fp.mode == 1) SF_INTEGRATE_ROWS(1, 2);
                else SF_INTEGRATE_ROWS(2, 2);
            }
        } else if (fp.mode == 0) {
            if (fpl) SF_INTEGRATE(0, true);
            else SF_INTEGRATE(0, false);
        } else if (fp.mode == 1) {
            if (fpl) SF_INTEGRATE(1, true);
            else SF_INTEGRATE(1, false);
        } else {
            if (fpl) SF_INTEGRATE(2, true);
            else SF_INTEGRATE(2, false);
        }
#undef SF_INTEGRATE
#undef SF_INTEGRATE_ROWS
#undef SF_INTEGRATE_ROWS_F2
        SF_LAUNCH_CHECK();
        if (events && events->after_integrate) record_event(events->after_integrate, s);
        n += 1;
        if (!caller_brackets) {
            k_fuse_finalize<<<1, 1, 0, s>>>(fb.ctr, v.d_vc);
            SF_LAUNCH_CHECK();
            n += 1;
        }
    }
    if (launches) *launches += n;
}

static void validate_intrinsics(const sf_intrinsics& i) {
    // Intrinsics::validate (camera.cpp:9-14)
    if (i.width <= 0 || i.height <= 0) throw Error(SF_INVALID_ARGUMENT, "intrinsics: non-positive image size");
    if (i.fx <= 0.0 || i.fy <= 0.0) throw Error(SF_INVALID_ARGUMENT, "intrinsics: non-positive focal length");
    if (!(i.near_plane > 0.0) || !(i.near_plane < i.far_plane))
        throw Error(SF_INVALID_ARGUMENT, "intrinsics: need 0 < near < far");
}

// Stage a frame (host or device pointers) into device memory; returns device pointers.
static void stage_frame(FrameBuffers& fb, const sf_frame& f, cudaStream_t s, const float** d_depth,
                        const float** d_sigma) {
    const size_t n = static_cast<size_t>(f.intrinsics.width) * f.intrinsics.height;
    if (f.on_device) {
        *d_depth = f.depth;
        *d_sigma = f.sigma;
        return;
    }
    SF_CUDA(cudaMemcpyAsync(fb.depth, f.depth, n * sizeof(float), cudaMemcpyHostToDevice, s));
    *d_depth = fb.depth;
    *d_sigma = nullptr;
    if (f.sigma) {
        SF_CUDA(cudaMemcpyAsync(fb.sigma, f.sigma, n * sizeof(float), cudaMemcpyHostToDevice, s));
        *d_sigma = fb.sigma;
    }
}

}  // namespace sf

using namespace sf;

extern "C" {

int sf_integrate(sf_volume_t v, const sf_frame* frame, const double pose[12], const sf_fusion_params* params,
                 sf_fusion_stats* stats, void* stream) {
    return guarded([&]() -> int {
        if (!v || !frame || !pose || !params) throw Error(SF_INVALID_ARGUMENT, "sf_integrate: null argument");
        SF_CUDA(cudaSetDevice(v->device));
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        validate_intrinsics(frame->intrinsics);
        const FuseParams fp = resolve_fuse_params(*v, *params, frame->sigma != nullptr);
        ensure_frame_buffers(*v, v->fb, frame->intrinsics.width, frame->intrinsics.height);
        FrameBuffers& fb = v->fb;
        const float *d_depth, *d_sigma;
        stage_frame(fb, *frame, s, &d_depth, &d_sigma);
        SF_CUDA(cudaMemcpyAsync(fb.pose, pose, 12 * sizeof(double), cudaMemcpyHostToDevice, s));
        const Intr intr = to_intr(frame->intrinsics);
        launch_fuse(*v, fb, intr, d_depth, d_sigma, fp, s, false, nullptr, nullptr);
        SF_CUDA(cudaMemcpyAsync(fb.h_ctr, fb.ctr, sizeof(FrameCounters), cudaMemcpyDeviceToHost, s));
        SF_CUDA(cudaStreamSynchronize(s));
        const FrameCounters& c = *fb.h_ctr;
        if (stats) {
            const uint64_t nn = v->P.N, m = v->P.M;
            stats->voxels_updated = c.voxels_updated;
            stats->blocks_allocated_now = c.alloc_now - c.alloc_before;
            stats->blocks_total = c.alloc_now;
            stats->memory_bytes = 2ull * c.alloc_now * m * m * m + 4ull * nn * nn * nn;
        }
        if (c.exhausted)
            throw Error(SF_POOL_EXHAUSTED, "grid: payload pool exhausted (" + std::to_string(v->P.capacity) +
                                               " blocks); increase pool capacity or lower resolution");
        return SF_OK;
    });
}

int sf_select_update_blocks(sf_volume_t v, const sf_frame* frame, const double pose[12], int32_t* allocate_xyz,
                            uint64_t* allocate_count, int32_t* update_xyz, uint64_t* update_count, void* stream) {
    return guarded([&]() -> int {
        SF_CUDA(cudaSetDevice(v->device));
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        validate_intrinsics(frame->intrinsics);
        ensure_frame_buffers(*v, v->fb, frame->intrinsics.width, frame->intrinsics.height);
        FrameBuffers& fb = v->fb;
        const float *d_depth, *d_sigma;
        stage_frame(fb, *frame, s, &d_depth, &d_sigma);
        SF_CUDA(cudaMemcpyAsync(fb.pose, pose, 12 * sizeof(double), cudaMemcpyHostToDevice, s));
        const Intr intr = to_intr(frame->intrinsics);
        FuseParams fp{};
        launch_fuse(*v, fb, intr, d_depth, d_sigma, fp, s, true, nullptr, nullptr);
        SF_CUDA(cudaMemcpyAsync(fb.h_ctr, fb.ctr, sizeof(FrameCounters), cudaMemcpyDeviceToHost, s));
        SF_CUDA(cudaStreamSynchronize(s));
        const FrameCounters c = *fb.h_ctr;
        if (c.n_list > *allocate_count || c.n_update > *update_count)
            throw Error(SF_OUT_OF_RANGE, "select_update_blocks: output capacity");
        std::vector<uint32_t> a(c.n_list), u(c.n_update);
        if (c.n_list) SF_CUDA(cudaMemcpy(a.data(), fb.keys_unique, a.size() * 4, cudaMemcpyDeviceToHost));
        if (c.n_update) SF_CUDA(cudaMemcpy(u.data(), fb.keys, u.size() * 4, cudaMemcpyDeviceToHost));
        std::sort(u.begin(), u.end());  // occupied_blocks_in_frustum walks the table in order
        const uint32_t N = v->P.N;
        auto put = [&](uint32_t key, int32_t* out) {
            out[0] = key % N;
            out[1] = (key / N) % N;
            out[2] = key / (N * N);
        };
        for (size_t i = 0; i < a.size(); ++i) put(a[i], allocate_xyz + 3 * i);
        for (size_t i = 0; i < u.size(); ++i) put(u[i], update_xyz + 3 * i);
        *allocate_count = a.size();
        *update_count = u.size();
        return SF_OK;
    });
}

int sf_compute_normals(const sf_frame* frame, double sigma0, double spatial_scale, float* normals_xyz,
                       int32_t out_on_device, void* stream) {
    return guarded([&]() -> int {
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        validate_intrinsics(frame->intrinsics);
        const int w = frame->intrinsics.width, h = frame->intrinsics.height;
        const size_t n = static_cast<size_t>(w) * h;
        float* d_depth = nullptr;
        float* d_out = nullptr;
        const float* src = frame->depth;
        if (!frame->on_device) {
            SF_CUDA(cudaMallocAsync(&d_depth, n * sizeof(float), s));
            SF_CUDA(cudaMemcpyAsync(d_depth, frame->depth, n * sizeof(float), cudaMemcpyHostToDevice, s));
            src = d_depth;
        }
        float* dst = normals_xyz;
        if (!out_on_device) {
            SF_CUDA(cudaMallocAsync(&d_out, 3 * n * sizeof(float), s));
            dst = d_out;
        }
        launch_compute_normals(src, w, h, to_intr(frame->intrinsics), sigma0, spatial_scale, dst, s, nullptr,
                               nullptr);
        if (!out_on_device)
            SF_CUDA(cudaMemcpyAsync(normals_xyz, d_out, 3 * n * sizeof(float), cudaMemcpyDeviceToHost, s));
        if (d_depth) SF_CUDA(cudaFreeAsync(d_depth, s));
        if (d_out) SF_CUDA(cudaFreeAsync(d_out, s));
        SF_CUDA(cudaStreamSynchronize(s));
        return SF_OK;
    });
}

}  // extern "C"

// sf_sample.cuh — trilinear TSDF sampling on the device (render.cpp:12-63), shared by the
// raycast (sf_render.cu) and marching cubes (sf_mesh.cu). FP64 in the reference's order.
#pragma once

#include "sf_internal.h"

namespace sf {

__device__ __forceinline__ bool occupied(const uint32_t* __restrict__ occ, uint64_t ti) {
    return (__ldg(&occ[ti >> 5]) >> (ti & 31)) & 1u;
}

// voxel_code + sample_tsdf (render.cpp:12-48). Returns false for nullopt.
struct Sampler {
    VolParams P;
    const int32_t* __restrict__ table;
    const uint16_t* __restrict__ payload;
    const uint32_t* __restrict__ occ;
    const double* tdec;  // shared-memory LUT, index code + 128

    __device__ __forceinline__ int blk(int x) const { return P.mshift >= 0 ? (x >> P.mshift) : x / P.M; }

    __device__ __forceinline__ bool code(int x, int y, int z, double& out) const {
        const int M = P.M;
        const int bx = blk(x), by = blk(y), bz = blk(z);
        const int32_t slot = __ldg(&table[table_index(P, bx, by, bz)]);
        if (slot == kEmpty) return false;
        const int lx = x - bx * M, ly = y - by * M, lz = z - bz * M;
        const uint16_t pl = __ldg(&payload[(size_t)slot * P.M3 + (lz * M + ly) * M + lx]);
        const int8_t c = static_cast<int8_t>(pl & 0xFF);
        if (c == kChiCode) return false;
        out = tdec[(int)c + 128];
        return true;
    }

    // a / voxel correctly rounded: q = RN(a * RN(1/voxel)) is within 1 ulp, and one
    // fma-residual correction gives RN(a / voxel) (Markstein's theorem), FP64 pipe only.
    __device__ __forceinline__ double div_voxel(double a) const {
        const double q = a * P.inv_voxel;
        const double r = fma(-q, P.voxel, a);
        return fma(r, P.inv_voxel, q);
    }

    __device__ bool sample(d3 p, double& out) const {
        const double gx = div_voxel(p.x - P.ox) - 0.5;
        const double gy = div_voxel(p.y - P.oy) - 0.5;
        const double gz = div_voxel(p.z - P.oz) - 0.5;
        // |g| >= 2^30 (or NaN) lies outside [0, res - 1) whatever floor gives
        constexpr double kLim = 1073741824.0;
        if (!(fabs(gx) < kLim && fabs(gy) < kLim && fabs(gz) < kLim)) return false;
        int bx, by, bz;
        const double flx = floor_exact(gx, bx), fly = floor_exact(gy, by), flz = floor_exact(gz, bz);
        const int res = P.res;
        if (bx < 0 || by < 0 || bz < 0 || bx + 1 >= res || by + 1 >= res || bz + 1 >= res) return false;
        // The base corner's block EMPTY => voxel_code fails => nullopt (render.cpp:14-15,39):
        // decided from the 1-bit occupancy map without touching the 4-byte table.
        if (!occupied(occ, table_index(P, blk(bx), blk(by), blk(bz)))) return false;
        const double fx = gx - flx, fy = gy - fly, fz = gz - flz;
        double c[8];
        if (P.mshift >= 0) {
            // All 8 table reads issued together, then all 8 payload reads (no dependent
            // branch between loads); any EMPTY block or chi corner => nullopt.
            const int ms = P.mshift, mm = P.M - 1, N = P.N;
            const int lx = bx & mm, ly = by & mm, lz = bz & mm;
            uint16_t pl[8];
            bool ok = true;
            if (lx != mm && ly != mm && lz != mm) {
                // all eight corners in the base block (7/8)^3 of the time: one table read
                const int32_t slot = __ldg(&table[((size_t)(bz >> ms) * N + (by >> ms)) * N + (bx >> ms)]);
                if (slot == kEmpty) return false;
                const uint16_t* b = payload + (size_t)slot * P.M3 + (((lz << ms) + ly) << ms) + lx;
                const int M = P.M, MM = M * M;
                pl[0] = __ldg(b);
                pl[1] = __ldg(b + 1);
                pl[2] = __ldg(b + M);
                pl[3] = __ldg(b + M + 1);
                pl[4] = __ldg(b + MM);
                pl[5] = __ldg(b + MM + 1);
                pl[6] = __ldg(b + MM + M);
                pl[7] = __ldg(b + MM + M + 1);
            } else {
                const int bxs[2] = {bx >> ms, (bx + 1) >> ms}, lxs[2] = {lx, (bx + 1) & mm};
                const int bys[2] = {by >> ms, (by + 1) >> ms}, lys[2] = {ly, (by + 1) & mm};
                const int bzs[2] = {bz >> ms, (bz + 1) >> ms}, lzs[2] = {lz, (bz + 1) & mm};
                int32_t s[8];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    s[i] = __ldg(&table[((size_t)bzs[i >> 2] * N + bys[(i >> 1) & 1]) * N + bxs[i & 1]]);
#pragma unroll
                for (int i = 0; i < 8; ++i) ok = ok && s[i] != kEmpty;
                if (!ok) return false;
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    pl[i] = __ldg(&payload[(size_t)s[i] * P.M3 + (((lzs[i >> 2] << ms) + lys[(i >> 1) & 1]) << ms) +
                                           lxs[i & 1]]);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int8_t cc = static_cast<int8_t>(pl[i] & 0xFF);
                ok = ok && cc != kChiCode;
                c[i] = tdec[(int)cc + 128];
            }
            if (!ok) return false;
        } else {
            for (int i = 0; i < 8; ++i)
                if (!code(bx + (i & 1), by + ((i >> 1) & 1), bz + ((i >> 2) & 1), c[i])) return false;
        }
        const double x0 = c[0] + (c[1] - c[0]) * fx;
        const double x1 = c[2] + (c[3] - c[2]) * fx;
        const double x2 = c[4] + (c[5] - c[4]) * fx;
        const double x3 = c[6] + (c[7] - c[6]) * fx;
        const double y0 = x0 + (x1 - x0) * fy;
        const double y1 = x2 + (x3 - x2) * fy;
        out = y0 + (y1 - y0) * fz;
        return true;
    }

    // sample() for the refinement near a known surface: no occupancy early-out (the table is
    // authoritative: same result), and the slot of the last single-block sample is cached, so
    // successive samples in the same block cost one L1-resident payload read.
    __device__ bool sample_near(d3 p, double& out, int64_t& ckey, int32_t& cslot) const {
        if (P.mshift < 0) return sample(p, out);
        const double gx = div_voxel(p.x - P.ox) - 0.5;
        const double gy = div_voxel(p.y - P.oy) - 0.5;
        const double gz = div_voxel(p.z - P.oz) - 0.5;
        constexpr double kLim = 1073741824.0;
        if (!(fabs(gx) < kLim && fabs(gy) < kLim && fabs(gz) < kLim)) return false;
        int bx, by, bz;
        const double flx = floor_exact(gx, bx), fly = floor_exact(gy, by), flz = floor_exact(gz, bz);
        const int res = P.res;
        if (bx < 0 || by < 0 || bz < 0 || bx + 1 >= res || by + 1 >= res || bz + 1 >= res) return false;
        const double fx = gx - flx, fy = gy - fly, fz = gz - flz;
        // One branch-free path for every corner layout (the 1-, 2-, 4- and 8-block cases would
        // diverge within a warp). The base corner's block slot comes from the cache or one
        // table read; a corner whose +1 step crosses into the next block along some axis reads
        // that block's slot — those reads do not depend on the base one, so every table read
        // and then every payload read of the sample is in flight at once. Any EMPTY block or
        // chi corner gives nullopt (render.cpp:14-15, 39), as in sample(). Table indices fit
        // int32 (N^3 < 2^31, checked at volume creation).
        const int ms = P.mshift, mm = P.M - 1, N = P.N;
        const int lx = bx & mm, ly = by & mm, lz = bz & mm;
        const bool cx = lx == mm, cy = ly == mm, cz = lz == mm;
        const int kb = ((bz >> ms) * N + (by >> ms)) * N + (bx >> ms);
        const int32_t sb = kb == ckey ? cslot : __ldg(&table[kb]);
        const int NN = N * N;
        bool ok = true;
        double c[8];
        uint16_t pl[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const bool ox = (i & 1) && cx, oy = ((i >> 1) & 1) && cy, oz = (i >> 2) && cz;
            const int32_t sl = (ox || oy || oz) ? __ldg(&table[kb + (ox ? 1 : 0) + (oy ? N : 0) + (oz ? NN : 0)]) : sb;
            const int vx = ox ? 0 : lx + (i & 1), vy = oy ? 0 : ly + ((i >> 1) & 1), vz = oz ? 0 : lz + (i >> 2);
            ok = ok && sl != kEmpty;
            pl[i] = sl != kEmpty ? __ldg(&payload[((size_t)sl << (3 * ms)) + (((vz << ms) + vy) << ms) + vx])
                                 : static_cast<uint16_t>(kChiPayload);
        }
        ckey = kb;  // cache the base corner's block
        cslot = sb;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int8_t cc = static_cast<int8_t>(pl[i] & 0xFF);
            ok = ok && cc != kChiCode;
            c[i] = tdec[(int)cc + 128];
        }
        if (!ok) return false;
        const double x0 = c[0] + (c[1] - c[0]) * fx;
        const double x1 = c[2] + (c[3] - c[2]) * fx;
        const double x2 = c[4] + (c[5] - c[4]) * fx;
        const double x3 = c[6] + (c[7] - c[6]) * fx;
        const double y0 = x0 + (x1 - x0) * fy;
        const double y1 = x2 + (x3 - x2) * fy;
        out = y0 + (y1 - y0) * fz;
        return true;
    }

    // The 8 decoded corners of the last voxel cell sampled by sample_cached (or its nullopt).
    struct CellCache {
        int bx = -1, by = -1, bz = -1;
        bool ok = false;
        double c[8];
    };
    // sample_near for the secant iterations of one ray: once the bracket is inside one voxel
    // cell, successive samples share the cell's 8 corners, which are reused instead of
    // reloaded (same corner values, same fractions, same arithmetic: bit-identical).
    __device__ bool sample_cached(d3 p, double& out, int64_t& ckey, int32_t& cslot, CellCache& cc) const {
        if (P.mshift < 0) return sample(p, out);
        const double gx = div_voxel(p.x - P.ox) - 0.5;
        const double gy = div_voxel(p.y - P.oy) - 0.5;
        const double gz = div_voxel(p.z - P.oz) - 0.5;
        constexpr double kLim = 1073741824.0;
        if (!(fabs(gx) < kLim && fabs(gy) < kLim && fabs(gz) < kLim)) return false;
        int bx, by, bz;
        const double flx = floor_exact(gx, bx), fly = floor_exact(gy, by), flz = floor_exact(gz, bz);
        const int res = P.res;
        if (bx < 0 || by < 0 || bz < 0 || bx + 1 >= res || by + 1 >= res || bz + 1 >= res) return false;
        const double fx = gx - flx, fy = gy - fly, fz = gz - flz;
        if (bx != cc.bx || by != cc.by || bz != cc.bz) {
            const int ms = P.mshift, mm = P.M - 1, N = P.N;
            const int lx = bx & mm, ly = by & mm, lz = bz & mm;
            const bool cx = lx == mm, cy = ly == mm, cz = lz == mm;
            const int kb = ((bz >> ms) * N + (by >> ms)) * N + (bx >> ms);
            const int32_t sb = kb == ckey ? cslot : __ldg(&table[kb]);
            const int NN = N * N;
            bool ok = true;
            uint16_t pl[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const bool ox = (i & 1) && cx, oy = ((i >> 1) & 1) && cy, oz = (i >> 2) && cz;
                const int32_t sl =
                    (ox || oy || oz) ? __ldg(&table[kb + (ox ? 1 : 0) + (oy ? N : 0) + (oz ? NN : 0)]) : sb;
                const int vx = ox ? 0 : lx + (i & 1), vy = oy ? 0 : ly + ((i >> 1) & 1), vz = oz ? 0 : lz + (i >> 2);
                ok = ok && sl != kEmpty;
                pl[i] = sl != kEmpty ? __ldg(&payload[((size_t)sl << (3 * ms)) + (((vz << ms) + vy) << ms) + vx])
                                     : static_cast<uint16_t>(kChiPayload);
            }
            ckey = kb;
            cslot = sb;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int8_t code = static_cast<int8_t>(pl[i] & 0xFF);
                ok = ok && code != kChiCode;
                cc.c[i] = tdec[(int)code + 128];
            }
            cc.bx = bx;
            cc.by = by;
            cc.bz = bz;
            cc.ok = ok;
        }
        if (!cc.ok) return false;
        const double* c = cc.c;
        const double x0 = c[0] + (c[1] - c[0]) * fx;
        const double x1 = c[2] + (c[3] - c[2]) * fx;
        const double x2 = c[4] + (c[5] - c[4]) * fx;
        const double x3 = c[6] + (c[7] - c[6]) * fx;
        const double y0 = x0 + (x1 - x0) * fy;
        const double y1 = x2 + (x3 - x2) * fy;
        out = y0 + (y1 - y0) * fz;
        return true;
    }

    // sample_tsdf_gradient (render.cpp:50-63) with the six samples independent of each other
    // (issued together instead of one after the other; the reference's early exit on a
    // nullopt only skips samples whose values would be discarded: same result).
    __device__ bool gradient_par(d3 p, double h, d3& g, int64_t ckey, int32_t cslot) const {
        double v[6];
        bool ok[6];
        const d3 q[6] = {mk(p.x + h, p.y, p.z), mk(p.x - h, p.y, p.z), mk(p.x, p.y + h, p.z),
                         mk(p.x, p.y - h, p.z), mk(p.x, p.y, p.z + h), mk(p.x, p.y, p.z - h)};
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            int64_t k = ckey;
            int32_t sl = cslot;
            ok[i] = sample_near(q[i], v[i], k, sl);
        }
        if (!(ok[0] && ok[1] && ok[2] && ok[3] && ok[4] && ok[5])) return false;
        g = mk((v[0] - v[1]) / (2.0 * h), (v[2] - v[3]) / (2.0 * h), (v[4] - v[5]) / (2.0 * h));
        return true;
    }

    // sample_tsdf_gradient (render.cpp:50-63) with the near-surface sampler
    __device__ bool gradient_near(d3 p, double h, d3& g, int64_t& ckey, int32_t& cslot) const {
        double a, b;
        if (!sample_near(mk(p.x + h, p.y, p.z), a, ckey, cslot) || !sample_near(mk(p.x - h, p.y, p.z), b, ckey, cslot))
            return false;
        const double gx = (a - b) / (2.0 * h);
        if (!sample_near(mk(p.x, p.y + h, p.z), a, ckey, cslot) || !sample_near(mk(p.x, p.y - h, p.z), b, ckey, cslot))
            return false;
        const double gy = (a - b) / (2.0 * h);
        if (!sample_near(mk(p.x, p.y, p.z + h), a, ckey, cslot) || !sample_near(mk(p.x, p.y, p.z - h), b, ckey, cslot))
            return false;
        const double gz = (a - b) / (2.0 * h);
        g = mk(gx, gy, gz);
        return true;
    }

    // sample_tsdf_gradient (render.cpp:50-63)
    __device__ bool gradient(d3 p, double h, d3& g) const {
        double a, b;
        if (!sample(mk(p.x + h, p.y, p.z), a) || !sample(mk(p.x - h, p.y, p.z), b)) return false;
        const double gx = (a - b) / (2.0 * h);
        if (!sample(mk(p.x, p.y + h, p.z), a) || !sample(mk(p.x, p.y - h, p.z), b)) return false;
        const double gy = (a - b) / (2.0 * h);
        if (!sample(mk(p.x, p.y, p.z + h), a) || !sample(mk(p.x, p.y, p.z - h), b)) return false;
        const double gz = (a - b) / (2.0 * h);
        g = mk(gx, gy, gz);
        return true;
    }
};


// Exact convex SAT of the camera frustum against a block (grid.cpp:174-269).
__device__ inline bool frustum_intersects_block(const VolParams& P, const FrameConsts* __restrict__ fc, d3 lo, d3 hi) {
    // box axes: the box projection is exactly [lo_a, hi_a]
    const double blo[3] = {lo.x, lo.y, lo.z}, bhi[3] = {hi.x, hi.y, hi.z};
    for (int k = 0; k < 3; ++k) {
        if (fc->sat_hi[k] < blo[k] || bhi[k] < fc->sat_lo[k]) return false;
    }
    for (int k = 3; k < kSatAxes; ++k) {
        if (!fc->sat_valid[k]) continue;
        const d3 a = fc->sat_axis[k];
        double mn = INFINITY, mx = -INFINITY;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const d3 p = mk(i & 1 ? hi.x : lo.x, i & 2 ? hi.y : lo.y, i & 4 ? hi.z : lo.z);
            const double d = dot(a, p);
            mn = dmin(mn, d);
            mx = dmax(mx, d);
        }
        if (fc->sat_hi[k] < mn || mx < fc->sat_lo[k]) return false;
    }
    return true;
}

// ---- per-frame setup shared by the fusion and tracker kernels -------------------------
// frame constants: one warp (hull points, corner rays and SAT axes lane-parallel)
__device__ inline void frame_consts_warp(const VolParams& P, const Intr& intr, const double* __restrict__ pose12,
                                  FrameConsts* fc) {
    const int lane = threadIdx.x & 31;
    __shared__ d3 s_pts[8], s_rays[4];
    __shared__ Pose s_pose;
    if (lane == 0) {
        const Pose pose = pose_from12(pose12);
        s_pose = pose;
        fc->pose = pose;
        fc->inv = invert(pose);
        fc->intr = intr;
        fc->delta = P.delta;
    }
    __syncwarp();
    const Pose pose = s_pose;
    // Frustum hull and separating axes, exactly as occupied_blocks_in_frustum builds them
    // (grid.cpp:228-262): hull points near/far x v x u, corner rays, 26 candidate axes.
    const double us[2] = {-0.5, intr.w - 0.5};
    const double vs[2] = {-0.5, intr.h - 0.5};
    if (lane < 8) {
        const double zs[2] = {intr.near_plane, intr.far_plane};
        s_pts[lane] = apply(pose, unproject(intr, us[lane & 1], vs[(lane >> 1) & 1], zs[lane >> 2]));
    } else if (lane < 12) {
        const int r = lane - 8;  // r00, r10, r01, r11
        s_rays[r] = normalized(mv(pose.R, unproject(intr, us[r & 1], vs[r >> 1], 1.0)));
    } else if (lane < 16) {
        // side face through the camera centre and two image corners, in the camera frame,
        // oriented so the optical axis is inside
        const int f = lane - 12;  // top (v = -0.5), bottom, left (u = -0.5), right
        const d3 a = f < 2 ? unproject(intr, us[0], vs[f], 1.0) : unproject(intr, us[f - 2], vs[0], 1.0);
        const d3 b = f < 2 ? unproject(intr, us[1], vs[f], 1.0) : unproject(intr, us[f - 2], vs[1], 1.0);
        d3 nrm = normalized(cross(a, b));
        if (nrm.z < 0.0) nrm = neg(nrm);
        fc->side_n[f] = nrm;
    }
    __syncwarp();
    if (lane < kSatAxes) {
        const d3 r00 = s_rays[0], r10 = s_rays[1], r01 = s_rays[2], r11 = s_rays[3];
        const d3 box_axes[3] = {mk(1, 0, 0), mk(0, 1, 0), mk(0, 0, 1)};
        d3 ax;
        if (lane < 3) ax = box_axes[lane];
        else if (lane == 3) ax = col(pose.R, 2);  // optical axis
        else if (lane == 4) ax = cross(r00, r10);  // top
        else if (lane == 5) ax = cross(r11, r01);  // bottom
        else if (lane == 6) ax = cross(r01, r00);  // left
        else if (lane == 7) ax = cross(r10, r11);  // right
        else {
            const int e = (lane - 8) / 3, b = (lane - 8) % 3;
            const d3 edges[6] = {r00, r10, r01, r11, col(pose.R, 0), col(pose.R, 1)};
            ax = cross(edges[e], box_axes[b]);
        }
        fc->sat_axis[lane] = ax;
        fc->sat_valid[lane] = !(sqnorm(ax) < 1e-18);
        double lo = INFINITY, hi = -INFINITY;
        for (int i = 0; i < 8; ++i) {
            const double d = dot(ax, s_pts[i]);
            lo = dmin(lo, d);
            hi = dmax(hi, d);
        }
        fc->sat_lo[lane] = lo;
        fc->sat_hi[lane] = hi;
    }
}

// Zero the per-frame counters; a set dead flag turns the frame's later kernels into no-ops.
__device__ inline void fuse_begin_body(FrameCounters* ctr, const VolCounters* vc, const int* dead) {
    FrameCounters z;
    memset(&z, 0, sizeof(z));
    z.alloc_before = vc->allocated_count - vc->halo_count;  // owned blocks only
    z.skip = dead ? static_cast<uint32_t>(*dead != 0) : 0u;
    z.t_begin = ~0ull;
    z.hw_before = vc->high_water;
    *ctr = z;
}
__device__ inline void fuse_finalize_body(FrameCounters* ctr, const VolCounters* vc) {
    ctr->alloc_now = vc->allocated_count - vc->halo_count;
}
}  // namespace sf

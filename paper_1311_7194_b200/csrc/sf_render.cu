// sf_render.cu — sparse-volume raycasting on the device (render.cpp:12-250).
//
//   k_ray_bounds  per pixel: slab clip + Amanatides-Woo DDA over the N^3 block lattice,
//                 occupancy read from the 1-bit/block bitmap (N^3/8 bytes, L2 resident)
//                 instead of the 4-byte offset table; first/last occupied cell -> float
//                 [t_start, t_end]                                     (render.cpp:65-153)
//   k_raycast     per pixel: stage-1 march on the sequential double t lattice, secant /
//                 bisection stage 2, 6-sample gradient normal          (render.cpp:160-250)
// All arithmetic is FP64 in the reference's order (no contraction), so depth, normals and
// the stage-1 sample count are bit-identical to the CPU path.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sf_internal.h"
#include "sf_sample.cuh"

namespace sf {


// ---- exact skipping along one DDA axis -----------------------------------------------
// An axis of the DDA is the sequence s_0 = tm, s_{k+1} = RN(s_k + td), tm, td > 0. Inside
// one binade [2^e, 2^(e+1)) every sum is a multiple of the same ulp u, so
// s_{k+1} = s_k + rint(td / u) * u as long as the result stays in the binade: the sequence is
// an arithmetic progression in integer mantissa units, and one real addition carries it
// into the next binade. (When td / u is a half-integer the sum is a rounding tie; RNE makes
// the first result even and every later increment the even neighbour, again constant.)
// seq_below counts the terms < X in O(binades) and returns the exact bits the sequential
// additions would produce for the first term >= X and the last term < X.
// floor(a / b) for 0 <= a < 2^53, 0 < b < 2^53: FP64 estimate, then exact integer correction
// (a 64-bit integer division is a long software sequence on the GPU).
__device__ __forceinline__ long long floor_div_53(long long a, long long b) {
    const double bd = static_cast<double>(b);
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(bd));
    r = fma(r, fma(-bd, r, 1.0), r);
    r = fma(r, fma(-bd, r, 1.0), r);
    long long j = static_cast<long long>(static_cast<double>(a) * r);
    while (j > 0 && j * b > a) --j;
    while ((j + 1) * b <= a) ++j;
    return j;
}

struct SeqPos {
    long long k;  // number of terms < X
    double at;    // s_k (first term >= X)
    double prev;  // s_{k-1}, or -inf when k == 0
};
__device__ __forceinline__ bool seq_below(double t, double d, double X, long long kmax, SeqPos& out) {
    constexpr long long kMantMask = (1LL << 52) - 1;
    long long K = 0;
    double prev = -INFINITY;
    for (int guard = 0; guard < 48; ++guard) {
        if (!(t < X)) {
            out = SeqPos{K, t, prev};
            return true;
        }
        if (K > kmax) return false;
        const long long tb = __double_as_longlong(t);
        const int e = static_cast<int>((tb >> 52) & 0x7ff);
        if (e < 64 || e > 1900) return false;
        const double q = d * __longlong_as_double(static_cast<long long>(1075 - e + 1023) << 52);  // td / ulp(t)
        if (!(q < 1125899906842624.0)) {  // td >= 2^50 ulps: one plain step
            prev = t;
            t = t + d;
            ++K;
            continue;
        }
        const double qt = q + kMagic52, qr = qt - kMagic52;
        long long k = (__double_as_longlong(qt) & kMantMask) - (1LL << 51);  // rint(q)
        const long long m = (tb & kMantMask) | (1LL << 52);
        if (fabs(q - qr) == 0.5) {  // tie
            if (m & 1) {            // odd start: one real step makes it even
                prev = t;
                t = t + d;
                ++K;
                continue;
            }
            const long long k0 = static_cast<long long>(floor(q));
            k = k0 + (k0 & 1);
        }
        if (k <= 0) return false;  // the sequence does not move
        constexpr long long kLim = (1LL << 53) - 1;  // largest mantissa integer of the binade
        const long long xb = __double_as_longlong(X);
        if (static_cast<int>((xb >> 52) & 0x7ff) == e) {
            const long long mx = (xb & kMantMask) | (1LL << 52);
            const long long cnt = floor_div_53(mx - m + k - 1, k);  // #{j >= 0 : m + j k < mx}
            if (m + cnt * k <= kLim) {  // the first term >= X is still in this binade
                out = SeqPos{K + cnt, __longlong_as_double(tb + cnt * k), __longlong_as_double(tb + (cnt - 1) * k)};
                return out.k <= kmax;
            }
        }
        const long long room = floor_div_53(kLim - m, k);  // in-binade steps j: m + j k <= kLim
        prev = __longlong_as_double(tb + room * k);  // every in-binade term is < X
        t = prev + d;                                // the real addition into the next binade
        K += room + 1;
    }
    return false;
}

// DDA state of render.cpp:103-144.
struct Dda {
    int cx, cy, cz, sx, sy, sz;
    double tmx, tmy, tmz, tdx, tdy, tdz;
    double t_in;
};
// Take every step with tm < T at once (the sequential loop takes them in tm order, ties
// x before y before z; the state after all steps below T does not depend on that order).
// Only valid when no cell visited before T can be occupied (the caller guarantees it).
// Returns false (state untouched) when a sequence is out of the fast path's domain.
__device__ __forceinline__ bool dda_jump(Dda& s, double T) {
    SeqPos px{0, s.tmx, -INFINITY}, py{0, s.tmy, -INFINITY}, pz{0, s.tmz, -INFINITY};
    constexpr long long kMax = 1 << 24;
    if (s.sx != 0 && !seq_below(s.tmx, s.tdx, T, kMax, px)) return false;
    if (s.sy != 0 && !seq_below(s.tmy, s.tdy, T, kMax, py)) return false;
    if (s.sz != 0 && !seq_below(s.tmz, s.tdz, T, kMax, pz)) return false;
    s.cx += s.sx * static_cast<int>(px.k);
    s.cy += s.sy * static_cast<int>(py.k);
    s.cz += s.sz * static_cast<int>(pz.k);
    s.tmx = px.at;
    s.tmy = py.at;
    s.tmz = pz.at;
    s.t_in = dmax(s.t_in, dmax(px.prev, dmax(py.prev, pz.prev)));  // time of the last step taken
    return true;
}

// Cheap conservative pre-test of pixel (u, v)'s ray: false only if the ray surely misses the
// occupied box grown by one block between the near and far planes, in which case the exact
// path below rejects it too (its slab clip and grown-box test are the same geometry, evaluated
// exactly). Evaluated on the unnormalised ray x(s) = t + s R (du, dv, 1), whose camera depth
// is s, with the box grown by a margin far above the rounding of either evaluation — no
// square root and no division per ray (the exact path has a dozen). Most rays of a frame
// miss the object.
__device__ __forceinline__ bool may_meet_occupied(const VolParams& P, const FrameConsts* __restrict__ fc,
                                                  const uint32_t* __restrict__ occ, int u, int v, double inv_fx,
                                                  double inv_fy) {
    const int* bb = occ_bbox(P, occ);
    if (bb[0] > bb[3]) return false;  // nothing allocated: the exact path finds nothing either
    const Intr& intr = fc->intr;
    const Pose& pose = fc->pose;
    const double du = (u - intr.cx) * inv_fx, dv = (v - intr.cy) * inv_fy;
    const d3 wv = mv(pose.R, mk(du, dv, 1.0));
    const double wd[3] = {wv.x, wv.y, wv.z}, org[3] = {pose.t.x, pose.t.y, pose.t.z};
    const double box_lo[3] = {P.ox, P.oy, P.oz};
    const double margin = 1e-7 * P.box_side + 1e-9;
    double slo = intr.near_plane * (1.0 - 1e-9), shi = intr.far_plane * (1.0 + 1e-9);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double wlo = box_lo[a] + (double)(bb[a] - 1) * P.block_side - margin;
        const double whi = box_lo[a] + (double)(bb[3 + a] + 2) * P.block_side + margin;
        if (fabs(wd[a]) < 1e-12) {
            if (org[a] < wlo || org[a] > whi) return false;
            continue;
        }
        double r;  // ~1/wd[a] (two Newton steps on the hardware estimate: far below the margins)
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(wd[a]));
        r = fma(r, fma(-wd[a], r, 1.0), r);
        r = fma(r, fma(-wd[a], r, 1.0), r);
        const double s0 = (wlo - org[a]) * r, s1 = (whi - org[a]) * r;
        slo = dmax(slo, dmin(s0, s1));
        shi = dmin(shi, dmax(s0, s1));
    }
    return slo <= shi * (1.0 + 1e-9) + 1e-12;
}

// Ray bounds of pixel (u, v) (render.cpp:65-153): writes t_start / t_end; true when the ray
// has bounds (!bounds.empty(u, v)).
__device__ __forceinline__ bool bounds_pixel(const VolParams& P, const FrameConsts* __restrict__ fc,
                                             const uint32_t* __restrict__ occ, const VolCounters* __restrict__ vc,
                                             const uint32_t* __restrict__ s_coarse, float* __restrict__ t_start,
                                             float* __restrict__ t_end, int w, double jump_cells,
                                             int u, int v, double inv_fx,
                                             double inv_fy, unsigned long long& cells) {
    const size_t idx = (size_t)v * w + u;
    float ts = INFINITY, te = -INFINITY;
    if (vc->allocated_count != 0 && may_meet_occupied(P, fc, occ, u, v, inv_fx, inv_fy)) {
        const Intr& intr = fc->intr;
        const Pose& pose = fc->pose;
        const int n = P.N;
        const double side = P.block_side;
        const double box_lo[3] = {P.ox, P.oy, P.oz};
        const double box_hi[3] = {P.ox + P.box_side, P.oy + P.box_side, P.oz + P.box_side};
        const double org[3] = {pose.t.x, pose.t.y, pose.t.z};
        const d3 dir_cam = normalized(unproject(intr, u, v, 1.0));
        const d3 dv3 = mv(pose.R, dir_cam);
        const double dir[3] = {dv3.x, dv3.y, dv3.z};
        double lo = intr.near_plane / dir_cam.z;
        double hi = intr.far_plane / dir_cam.z;
        for (int a = 0; a < 3; ++a) {
            if (fabs(dir[a]) < 1e-15) {
                if (org[a] < box_lo[a] || org[a] > box_hi[a]) {
                    lo = 1.0;
                    hi = 0.0;
                    break;
                }
                continue;
            }
            double t0 = (box_lo[a] - org[a]) / dir[a];
            double t1 = (box_hi[a] - org[a]) / dir[a];
            if (t0 > t1) {
                const double tmp = t0;
                t0 = t1;
                t1 = tmp;
            }
            lo = dmax(lo, t0);
            hi = dmin(hi, t1);
        }
        // Conservative reject: a ray missing the occupied bounding box (grown by one block)
        // meets no allocated block, so its DDA would find nothing.
        const int* bb = occ_bbox(P, occ);
        const int bx0 = bb[0], by0 = bb[1], bz0 = bb[2], bx1 = bb[3], by1 = bb[4], bz1 = bb[5];
        double t_grown = -INFINITY;  // entry time into the occupied box grown by one block
        if (lo <= hi && bx0 <= bx1) {
            double rlo = lo, rhi = hi;
            const int bl[3] = {bx0, by0, bz0}, bh[3] = {bx1, by1, bz1};
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const double wlo = box_lo[a] + (double)(bl[a] - 1) * side;
                const double whi = box_lo[a] + (double)(bh[a] + 2) * side;
                if (fabs(dir[a]) < 1e-300) {
                    if (org[a] < wlo || org[a] > whi) rhi = -INFINITY;
                    continue;
                }
                double t0 = (wlo - org[a]) / dir[a], t1 = (whi - org[a]) / dir[a];
                if (t0 > t1) {
                    const double tmp = t0;
                    t0 = t1;
                    t1 = tmp;
                }
                rlo = dmax(rlo, t0);
                rhi = dmin(rhi, t1);
            }
            if (!(rlo <= rhi)) lo = 1.0, hi = 0.0;
            t_grown = rlo;
        }
        if (lo <= hi && bx0 <= bx1) {
            // Scalar (register-resident) Amanatides-Woo state; same operations as render.cpp:103-144.
            const double ex = org[0] + lo * dir[0], ey = org[1] + lo * dir[1], ez = org[2] + lo * dir[2];
            auto clampc = [n](int c) { return c < 0 ? 0 : (n - 1 < c ? n - 1 : c); };  // std::clamp(c, 0, n-1)
            int cx = clampc(ref_floor_int((ex - box_lo[0]) / side));
            int cy = clampc(ref_floor_int((ey - box_lo[1]) / side));
            int cz = clampc(ref_floor_int((ez - box_lo[2]) / side));
            auto init_axis = [&](double d, double blo, int c, double e, int& st, double& tm, double& td) {
                if (d > 1e-15) {
                    st = 1;
                    tm = lo + (blo + (double)(c + 1) * side - e) / d;
                    td = side / d;
                } else if (d < -1e-15) {
                    st = -1;
                    tm = lo + (blo + (double)c * side - e) / d;
                    td = -side / d;
                } else {
                    st = 0;
                    tm = INFINITY;
                    td = INFINITY;
                }
            };
            {
                // cells of the reference DDA (render.cpp:103-144) from the entry cell to the cell
                // at min(hi, box exit): one per plane crossing + 1 (for the roofline count only)
                const double hx = org[0] + hi * dir[0], hy = org[1] + hi * dir[1], hz = org[2] + hi * dir[2];
                const int qx = clampc(ref_floor_int((hx - box_lo[0]) / side));
                const int qy = clampc(ref_floor_int((hy - box_lo[1]) / side));
                const int qz = clampc(ref_floor_int((hz - box_lo[2]) / side));
                cells += 1ull + static_cast<unsigned>(abs(qx - cx)) + static_cast<unsigned>(abs(qy - cy)) +
                         static_cast<unsigned>(abs(qz - cz));
            }
            Dda s;
            s.cx = cx;
            s.cy = cy;
            s.cz = cz;
            init_axis(dir[0], box_lo[0], cx, ex, s.sx, s.tmx, s.tdx);
            init_axis(dir[1], box_lo[1], cy, ey, s.sy, s.tmy, s.tdy);
            init_axis(dir[2], box_lo[2], cz, ez, s.sz, s.tmz, s.tdz);
            s.t_in = lo;
            double first = INFINITY, last = -INFINITY;
            const double td_min = dmin(s.tdx, dmin(s.tdy, s.tdz));
            // Skip the run-up to the occupied box: every cell entered before the ray reaches
            // the box grown by one block lies outside the occupied box.
            if (t_grown > lo + 4.0 * td_min) dda_jump(s, t_grown);
            const double sb_side = side * (1 << kCoarseShift);
            int declined_cc = -1;  // coarse cell whose skip was judged too short to jump
            // Loop state derived from the cells (recomputed after a jump, stepped otherwise):
            //  r* = steps left on an axis before the ray leaves the occupied box in its direction
            //       of travel (no later cell can be allocated: cells move monotonically per axis,
            //       so first/last are final there); the original loop tests all three per step,
            //       only the stepped axis can change;
            //  in-box test r* <= w*; table index and coarse cell kept incrementally.
            const int wx = bx1 - bx0, wy = by1 - by0, wz = bz1 - bz0;
            const int kx = s.sx, ky = s.sy * n, kz = s.sz * n * n;  // N^3 < 2^31 (N <= 1024)
            const double inv_dir[3] = {1.0 / dir[0], 1.0 / dir[1], 1.0 / dir[2]};
            int rx, ry, rz, cc, key;
            uint32_t cbit;
            auto derive = [&]() {
                rx = s.sx > 0 ? bx1 - s.cx : s.cx - bx0;
                ry = s.sy > 0 ? by1 - s.cy : s.cy - by0;
                rz = s.sz > 0 ? bz1 - s.cz : s.cz - bz0;
                key = (s.cz * n + s.cy) * n + s.cx;
                cc = ((s.cz >> kCoarseShift) * P.Nc + (s.cy >> kCoarseShift)) * P.Nc + (s.cx >> kCoarseShift);
                cbit = (s_coarse[cc >> 5] >> (cc & 31)) & 1u;
            };
            // an axis that does not move must lie inside the box, else no cell ever is
            // (sx == 0: r = c - b0 must be in [0, w])
            auto outside = [&]() {
                return rx < 0 || ry < 0 || rz < 0 || (s.sx == 0 && rx > wx) || (s.sy == 0 && ry > wy) ||
                       (s.sz == 0 && rz > wz);
            };
            bool live = s.cx >= 0 && s.cx < n && s.cy >= 0 && s.cy < n && s.cz >= 0 && s.cz < n;
            if (live) {
                derive();
                live = !outside();
            }
            uint32_t pend_word = 0, pend_bit = 0;  // occupancy probe of the previous step
        double pend_tin = 0.0, pend_tout = 0.0;
        while (live && s.t_in <= hi) {
                const int axis = s.tmx <= s.tmy ? (s.tmx <= s.tmz ? 0 : 2) : (s.tmy <= s.tmz ? 1 : 2);
                const double tm = axis == 0 ? s.tmx : (axis == 1 ? s.tmy : s.tmz);
                if (!cbit && cc != declined_cc) {
                    // Super-block never held a block: jump to a quarter cell before the ray
                    // leaves it (the cells visited up to then are inside it, hence empty).
                    const int sbx = s.cx >> kCoarseShift, sby = s.cy >> kCoarseShift, sbz = s.cz >> kCoarseShift;
                    const double ox_ = box_lo[0] + sbx * sb_side, oy_ = box_lo[1] + sby * sb_side,
                                 oz_ = box_lo[2] + sbz * sb_side;
                    // exit time through the reciprocal: the quarter-cell margin of T below
                    // absorbs its rounding (a few ulps of t)
                    double t_exit = INFINITY;
                    if (s.sx != 0) t_exit = dmin(t_exit, ((s.sx > 0 ? ox_ + sb_side : ox_) - org[0]) * inv_dir[0]);
                    if (s.sy != 0) t_exit = dmin(t_exit, ((s.sy > 0 ? oy_ + sb_side : oy_) - org[1]) * inv_dir[1]);
                    if (s.sz != 0) t_exit = dmin(t_exit, ((s.sz > 0 ? oz_ + sb_side : oz_) - org[2]) * inv_dir[2]);
                    const double T = dmin(t_exit, hi) - 0.25 * td_min;
                    // a jump costs a few hundred instructions: worth it past ~16 plain steps
                    if (T > tm + jump_cells * td_min && dda_jump(s, T)) {
                        if (s.cx < 0 || s.cx >= n || s.cy < 0 || s.cy >= n || s.cz < 0 || s.cz >= n) break;
                        derive();
                        if (outside()) break;
                        continue;
                    }
                    declined_cc = cc;  // short crossing: plain steps through it (no occupancy reads)
                }
                // Occupancy of the cell (only inside a super-block that ever held a block;
                // cbit set implies cc != declined_cc). The word is consumed one step later,
                // so its load overlaps the next DDA step instead of stalling this one.
                {
                    const bool probe = cbit && rx <= wx && ry <= wy && rz <= wz;
                    const uint32_t word = probe ? __ldg(&occ[static_cast<uint32_t>(key) >> 5]) : 0u;
                    if ((pend_word >> pend_bit) & 1u) {  // t_in and t_out never decrease along the ray
                        if (first == INFINITY) first = pend_tin;
                        last = pend_tout;
                    }
                    pend_word = word;
                    pend_bit = static_cast<uint32_t>(key) & 31u;
                    pend_tin = s.t_in;
                    pend_tout = dmin(tm, hi);
                }
                s.t_in = tm;
                // step the axis with the smallest tm (branch-free: the lanes of a warp step
                // different axes)
                const bool a0 = axis == 0, a1 = axis == 1, a2 = axis == 2;
                const int cxo = s.cx, cyo = s.cy, czo = s.cz;
                s.cx += a0 ? s.sx : 0;
                s.cy += a1 ? s.sy : 0;
                s.cz += a2 ? s.sz : 0;
                rx -= a0 ? 1 : 0;
                ry -= a1 ? 1 : 0;
                rz -= a2 ? 1 : 0;
                if ((rx | ry | rz) < 0) break;
                const double tn = tm + (a0 ? s.tdx : (a1 ? s.tdy : s.tdz));
                s.tmx = a0 ? tn : s.tmx;
                s.tmy = a1 ? tn : s.tmy;
                s.tmz = a2 ? tn : s.tmz;
                key += a0 ? kx : (a1 ? ky : kz);
                if (((cxo ^ s.cx) | (cyo ^ s.cy) | (czo ^ s.cz)) >> kCoarseShift) {  // crossed into another super-block
                    cc = ((s.cz >> kCoarseShift) * P.Nc + (s.cy >> kCoarseShift)) * P.Nc + (s.cx >> kCoarseShift);
                    cbit = (s_coarse[cc >> 5] >> (cc & 31)) & 1u;
                }
            }
            if ((pend_word >> pend_bit) & 1u) {
                if (first == INFINITY) first = pend_tin;
                last = pend_tout;
            }
            if (first <= last) {
                ts = (float)dmax(first, lo);
                te = (float)dmin(last, hi);
            }
        }
    }
    t_start[idx] = ts;
    t_end[idx] = te;
    return ts <= te;
}

__device__ __forceinline__ void write_empty(float* __restrict__ depth_out, float* __restrict__ normals_out, size_t idx) {
    depth_out[idx] = 0.0f;
    normals_out[3 * idx] = 0.0f;
    normals_out[3 * idx + 1] = 0.0f;
    normals_out[3 * idx + 2] = 0.0f;
}

// Coarse occupancy (1 bit per 16^3 blocks) staged in shared memory: the DDA only reads the
// fine bitmap (L2) inside super-blocks that ever held a block. Exact: a clear coarse bit
// implies every block of the super-block is EMPTY.
__device__ __forceinline__ void stage_coarse(const VolParams& P, const uint32_t* __restrict__ occ, uint32_t* s_coarse) {
    const uint64_t nc = P.Nc;
    const int cwords = static_cast<int>((nc * nc * nc + 31) / 32);
    for (int i = threadIdx.x; i < cwords; i += blockDim.x) s_coarse[i] = __ldg(&occ[P.occ_fine_words + i]);
}

__global__ void __launch_bounds__(256, 2) k_ray_bounds(VolParams P, const FrameConsts* __restrict__ fc, const uint32_t* __restrict__ occ,
                             const VolCounters* __restrict__ vc, float* __restrict__ t_start,
                             float* __restrict__ t_end, int w, int h, const int* dead, int* __restrict__ ray_list,
                             RayCounters* list_ctr, float* __restrict__ depth_out, float* __restrict__ normals_out,
                             double jump_cells, uint32_t* __restrict__ sched, const uint32_t* __restrict__ order) {
    pdl_wait();
    extern __shared__ uint32_t s_coarse[];
    if (dead && *dead) return;
    stage_coarse(P, occ, s_coarse);
    __syncthreads();
    // Persistent CTAs; each warp takes 8x4-pixel patches from a counter (neighbouring rays have
    // similar DDA lengths, so fewer lanes idle in the step loop; dynamic patches balance the
    // SMs: ray cost varies by orders of magnitude across the image). Patches are handed out
    // centre first (`order`): the long rays usually sit in the middle of the image.
    const int ln = threadIdx.x & 31;
    const int pw = (w + 7) >> 3, n_patches = pw * ((h + 3) >> 2);
    const double inv_fx = 1.0 / fc->intr.fx, inv_fy = 1.0 / fc->intr.fy;
    unsigned long long cells = 0;
    for (;;) {
        int patch = 0;
        if (ln == 0) patch = static_cast<int>(atomicAdd(&sched[0], 1u));
        patch = __shfl_sync(0xffffffffu, patch, 0);
        if (patch >= n_patches) break;
        patch = static_cast<int>(__ldg(&order[patch]));
        const int u = (patch % pw) * 8 + (ln & 7);
        const int v = (patch / pw) * 4 + (ln >> 3);
        if (u >= w || v >= h) continue;
        const bool act = bounds_pixel(P, fc, occ, vc, s_coarse, t_start, t_end, w, jump_cells, u, v, inv_fx,
                                      inv_fy, cells);
        if (ray_list) {
            // Active-ray list for the march (warp-aggregated append); inactive pixels get the
            // empty raycast result here.
            const int idx = v * w + u;
            if (!act) write_empty(depth_out, normals_out, idx);
            const unsigned am = __activemask();
            const unsigned bal = __ballot_sync(am, act);
            unsigned long long base = 0;
            if (bal) {
                const int leader = __ffs(bal) - 1;
                if (ln == leader) base = atomicAdd(&list_ctr->listed, static_cast<unsigned long long>(__popc(bal)));
                base = __shfl_sync(am, base, leader);
            }
            if (act) ray_list[base + __popc(bal & ((1u << ln) - 1u))] = idx;
        }
    }
    if (list_ctr) {
        for (int off = 16; off > 0; off >>= 1) cells += __shfl_down_sync(0xffffffffu, cells, off);
        if (ln == 0 && cells) atomicAdd(&list_ctr->dda_cells, cells);
    }
    // last CTA out resets the counters for the next launch
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(&sched[1], 1u) == gridDim.x - 1) {
        sched[0] = 0;
        sched[1] = 0;
    }
}

// One ray per group of G lanes (G = 8: four rays per warp). Stage 1 evaluates G consecutive
// points of the reference's sequential t lattice at once (lane k walks the same additions
// t += step, so every t is bit-identical), then finds the first sign change in lattice
// order with ballots/shuffles: "previous sample" is the last VALID sample before it, as in
// render.cpp:185-207, carried across groups. Samples past the bracket are discarded
// (sampling is pure), so results and the stage-1 step count equal the reference's.
// Stage 2 runs redundantly in all G lanes (same addresses: broadcast loads); the six
// gradient samples run one per lane.
// Stage 1 of the raycast for pixel idx (render.cpp:160-208) by a group of G lanes: appends the
// bracket of the first + -> - crossing to the refine list, else writes the empty result.
template <int G>
__device__ __forceinline__ void march_ray(const VolParams& P, const FrameConsts* __restrict__ fc,
                                          const int32_t* __restrict__ table, const uint16_t* __restrict__ payload,
                                          const uint32_t* __restrict__ occ, const double* s_tdec,
                                          const float* __restrict__ t_start, const float* __restrict__ t_end,
                                          float* __restrict__ depth_out, float* __restrict__ normals_out,
                                          RayCounters* stats, int w, RayBracket* __restrict__ brackets, int idx,
                                          unsigned long long& steps, unsigned long long& with_bounds) {
    const int lane = threadIdx.x & 31;
    const int g = lane & (G - 1);
    const int gbase = lane & ~(G - 1);
    const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u)) << gbase;
    auto group_bits = [&](bool pred) { return (__ballot_sync(gmask, pred) & gmask) >> gbase; };
    const int u = idx % w, v = idx / w;
    float out_d = 0.0f, nx = 0.f, ny = 0.f, nz = 0.f;
    bool bracket_out = false;
    RayBracket br{};
    const float fs = t_start[idx], fe = t_end[idx];
    if (fs <= fe) {  // !bounds.empty(u, v)
        with_bounds += 1;
        const Sampler S{P, table, payload, occ, s_tdec};
        const Intr& intr = fc->intr;
        const Pose& pose = fc->pose;
        const double coarse_step = 0.5 * P.delta;
        const d3 dir_cam = normalized(unproject(intr, u, v, 1.0));
        const d3 dir = mv(pose.R, dir_cam);
        const double t1 = fe;
        bool carry = false, bracketed = false;
        double carry_t = 0.0, carry_val = 0.0;
        double hit_a = 0.0, hit_b = 0.0, val_a = 0.0, val_b = 0.0;
        double t_base = fs;
        for (;;) {
            double t = t_base;
            bool has = true, fin = false;
            for (int k = 0; k < g; ++k) {
                if (t >= t1) {
                    has = false;
                    break;
                }
                t += coarse_step;
            }
            if (has && t >= t1) {
                fin = true;
                t = t1;
            }
            double val = 0.0;
            const bool valid = has && S.sample(add(pose.t, scale(t, dir)), val);
            const unsigned vm = group_bits(valid), fm = group_bits(fin), hm = group_bits(has);
            const unsigned below = vm & ((1u << g) - 1u);
            const int pl = below ? 31 - __clz(below) : 0;
            double pv = __shfl_sync(gmask, val, pl, G), pt = __shfl_sync(gmask, t, pl, G);
            bool hp = below != 0;
            if (!hp) {
                hp = carry;
                pv = carry_val;
                pt = carry_t;
            }
            const unsigned hit = group_bits(valid && hp && pv > 0.0 && val < 0.0);
            if (hit) {
                const int hl = __ffs(hit) - 1;
                hit_a = __shfl_sync(gmask, pt, hl, G);
                val_a = __shfl_sync(gmask, pv, hl, G);
                hit_b = __shfl_sync(gmask, t, hl, G);
                val_b = __shfl_sync(gmask, val, hl, G);
                steps += hl + 1;
                bracketed = true;
                break;
            }
            steps += __popc(hm);
            if (fm || hm != (G == 32 ? 0xffffffffu : (1u << G) - 1u)) break;
            if (vm) {
                const int ll = 31 - __clz(vm);
                carry = true;
                carry_t = __shfl_sync(gmask, t, ll, G);
                carry_val = __shfl_sync(gmask, val, ll, G);
            }
            t_base = __shfl_sync(gmask, t, G - 1, G) + coarse_step;
        }
        if (bracketed && g == 0) {
            bracket_out = true;
            br = RayBracket{hit_a, hit_b, val_a, val_b, idx, 0};
        }
    }
    // Rays with a bracket go to the one-thread-per-ray refine pass (stage 2 + normal); the
    // others get the empty result here.
    const unsigned am = __activemask();
    const unsigned bal = __ballot_sync(am, bracket_out);
    unsigned long long base = 0;
    if (bal) {
        const int leader = __ffs(bal) - 1;
        if (lane == leader) base = atomicAdd(&stats->brackets, static_cast<unsigned long long>(__popc(bal)));
        base = __shfl_sync(am, base, leader);
    }
    if (bracket_out) {
        brackets[base + __popc(bal & ((1u << lane) - 1u))] = br;
    } else if (g == 0) {
        depth_out[idx] = out_d;
        normals_out[3 * idx] = nx;
        normals_out[3 * idx + 1] = ny;
        normals_out[3 * idx + 2] = nz;
    }
}

#ifndef SF_RAYCAST_CTAS
#define SF_RAYCAST_CTAS 3
#endif
template <int G>
__global__ void __launch_bounds__(256, SF_RAYCAST_CTAS)
    k_raycast(VolParams P, const FrameConsts* __restrict__ fc, const int32_t* __restrict__ table,
              const uint16_t* __restrict__ payload, const uint32_t* __restrict__ occ, const AuxTables* __restrict__ aux,
              const float* __restrict__ t_start, const float* __restrict__ t_end, float* __restrict__ depth_out,
              float* __restrict__ normals_out, RayCounters* stats, int w, int h, const int* dead,
              const int* __restrict__ ray_list, RayBracket* __restrict__ brackets) {
    pdl_wait();
    static_assert(G >= 8 && G <= 32 && (G & (G - 1)) == 0, "group of 8..32 lanes");
    (void)h;
    constexpr int kRaysPerCta = 256 / G;
    __shared__ double s_tdec[256];
    if (dead && *dead) return;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_tdec[i] = aux->tsdf_decode[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int g = lane & (G - 1);
    unsigned long long steps = 0, with_bounds = 0;
    const unsigned long long n_rays = stats->listed;
    for (unsigned long long r = (unsigned long long)blockIdx.x * kRaysPerCta + threadIdx.x / G; r < n_rays;
         r += (unsigned long long)gridDim.x * kRaysPerCta) {  // uniform within the group
        march_ray<G>(P, fc, table, payload, occ, s_tdec, t_start, t_end, depth_out, normals_out, stats, w, brackets,
                     ray_list[r], steps, with_bounds);
    }
    if (g != 0) steps = with_bounds = 0;  // per-ray values are replicated in the group
    // RaycastStats: warp reduction, one atomic per warp and counter.
    for (int off = 16; off > 0; off >>= 1) {
        steps += __shfl_down_sync(0xffffffffu, steps, off);
        with_bounds += __shfl_down_sync(0xffffffffu, with_bounds, off);
    }
    if (lane == 0 && stats) {
        if (steps) atomicAdd(&stats->sample_steps, steps);
        if (with_bounds) atomicAdd(&stats->rays_with_bounds, with_bounds);
    }
}

// Stage 2 + gradient normal of one bracketed ray (render.cpp:209-246); returns 1 for a hit.
__device__ __forceinline__ unsigned refine_ray(const Sampler& S, const VolParams& P, const FrameConsts* __restrict__ fc,
                                               const RayBracket& b, float* __restrict__ depth_out,
                                               float* __restrict__ normals_out, int w,
                                               unsigned long long& samples) {
    const Intr& intr = fc->intr;
    const Pose& pose = fc->pose;
    const double vox = P.voxel;
    const double fine_tol = 0.01 * vox;
    unsigned hits = 0;
    const int idx = b.idx;
    const int u = idx % w, v = idx / w;
    const d3 dir_cam = normalized(unproject(intr, u, v, 1.0));
    const d3 dir = mv(pose.R, dir_cam);
    double hit_a = b.a, hit_b = b.b, val_a = b.va, val_b = b.vb;
    float out_d = 0.0f, nx = 0.f, ny = 0.f, nz = 0.f;
    int64_t ckey = -1;
    int32_t cslot = kEmpty;
    Sampler::CellCache cell;
    int iter = 0;
    for (; iter < 48 && hit_b - hit_a > fine_tol; ++iter) {
        double t_new = hit_b - val_b * (hit_b - hit_a) / (val_b - val_a);
        if (!(t_new > hit_a) || !(t_new < hit_b)) t_new = 0.5 * (hit_a + hit_b);
        double val;
#ifndef SF_REFINE_CACHE
#define SF_REFINE_CACHE 1
#endif
#if SF_REFINE_CACHE
        if (!S.sample_cached(add(pose.t, scale(t_new, dir)), val, ckey, cslot, cell)) {
#else
        if (!S.sample_near(add(pose.t, scale(t_new, dir)), val, ckey, cslot)) {
#endif
            hit_a = t_new;
            val_a = dmax(val_a, 1e-12);
            continue;
        }
        if (val > 0.0) {
            hit_a = t_new;
            val_a = val;
        } else {
            hit_b = t_new;
            val_b = val;
        }
    }
    samples += iter;
    double root;
    if (val_b != val_a) {
        const double interp = hit_b - val_b * (hit_b - hit_a) / (val_b - val_a);
        root = dclamp(interp, hit_a, hit_b);
    } else {
        root = 0.5 * (hit_a + hit_b);
    }
    const double dd = root * dir_cam.z;
    if (!(dd < intr.near_plane || dd > intr.far_plane)) {
        out_d = (float)dd;
        hits += 1;
        samples += 6;
        // sample_tsdf_gradient (render.cpp:50-63)
        const d3 p = add(pose.t, scale(root, dir));
        d3 gr;
#ifndef SF_GRAD_PAR
#define SF_GRAD_PAR 0
#endif
#if SF_GRAD_PAR
        if (S.gradient_par(p, vox, gr, ckey, cslot) && sqnorm(gr) > 0.0) {
#else
        if (S.gradient_near(p, vox, gr, ckey, cslot) && sqnorm(gr) > 0.0) {
#endif
            // world_to_cam * grad.normalized()  (render.cpp:242-245)
            const d3 n_cam = mv(mt(pose.R), normalized(gr));
            nx = (float)n_cam.x;
            ny = (float)n_cam.y;
            nz = (float)n_cam.z;
        }
    }
    depth_out[idx] = out_d;
    normals_out[3 * idx] = nx;
    normals_out[3 * idx + 1] = ny;
    normals_out[3 * idx + 2] = nz;
    return hits;
}

// Stage 2 (secant / bisection to 0.01 voxel, render.cpp:209-233) and the gradient normal
// (render.cpp:236-246) for every bracketed ray: one thread per ray (the sequential secant
// iterations have no parallelism within a ray; the six gradient samples are independent).
__global__ void __launch_bounds__(256)
    k_raycast_refine(VolParams P, const FrameConsts* __restrict__ fc, const int32_t* __restrict__ table,
                     const uint16_t* __restrict__ payload, const uint32_t* __restrict__ occ,
                     const AuxTables* __restrict__ aux, const RayBracket* __restrict__ brackets,
                     float* __restrict__ depth_out, float* __restrict__ normals_out, RayCounters* stats, int w,
                     const int* dead) {
    pdl_wait();
    __shared__ double s_tdec[256];
    if (dead && *dead) return;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_tdec[i] = aux->tsdf_decode[i];
    __syncthreads();
    const Sampler S{P, table, payload, occ, s_tdec};
    const unsigned long long n = stats->brackets;
    unsigned long long hits = 0, samples = 0;
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        hits += refine_ray(S, P, fc, brackets[i], depth_out, normals_out, w, samples);
    }
    for (int off = 16; off > 0; off >>= 1) {
        hits += __shfl_down_sync(0xffffffffu, hits, off);
        samples += __shfl_down_sync(0xffffffffu, samples, off);
    }
    if ((threadIdx.x & 31) == 0 && hits) atomicAdd(&stats->hit_pixels, hits);
    if ((threadIdx.x & 31) == 0 && samples) atomicAdd(&stats->refine_samples, samples);
}

// Minimum number of DDA cells an exact skip must save (a jump costs a few hundred
// instructions; shorter crossings of empty super-blocks are stepped without occupancy reads).
constexpr double kRayJumpCells = 16.0;

// Patch order of k_ray_bounds: 8x4 patches sorted by the distance of their centre to the
// image centre (built once per image size, outside graph capture: ensure_frame_buffers).
void ensure_patch_order(Volume& v, int w, int h) {
    if (w == v.order_w && h == v.order_h) return;
    const int pw = (w + 7) >> 3, ph = (h + 3) >> 2;
    std::vector<uint32_t> idx(static_cast<size_t>(pw) * ph);
    std::vector<double> dist(idx.size());
    for (int y = 0; y < ph; ++y)
        for (int x = 0; x < pw; ++x) {
            const double dx = (x * 8 + 4) - 0.5 * w, dy = (y * 4 + 2) - 0.5 * h;
            idx[static_cast<size_t>(y) * pw + x] = static_cast<uint32_t>(y * pw + x);
            dist[static_cast<size_t>(y) * pw + x] = dx * dx + dy * dy;
        }
    std::stable_sort(idx.begin(), idx.end(), [&](uint32_t a, uint32_t b) { return dist[a] < dist[b]; });
    if (v.d_patch_order) SF_CUDA(cudaFree(v.d_patch_order));
    v.d_patch_order = nullptr;
    SF_CUDA(cudaMalloc(&v.d_patch_order, idx.size() * sizeof(uint32_t)));
    SF_CUDA(cudaMemcpy(v.d_patch_order, idx.data(), idx.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    v.order_w = w;
    v.order_h = h;
}

void launch_ray_bounds(Volume& v, const FrameConsts* d_fc, const Intr& intr, float* t_start, float* t_end,
                       cudaStream_t s, uint64_t* launches, const int* dead_flag, int* ray_list,
                       RayCounters* list_ctr, float* depth, float* normals) {
    ensure_patch_order(v, intr.w, intr.h);
    const dim3 blk(256), grd(148 * 2);
    const uint64_t nc = v.P.Nc;
    const size_t smem = ((nc * nc * nc + 31) / 32) * sizeof(uint32_t);
    if (smem > 48 * 1024) SF_CUDA(cudaFuncSetAttribute(k_ray_bounds, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    launch_pdl(k_ray_bounds, grd, blk, smem, s, v.P, d_fc, v.d_occ, v.d_vc, t_start, t_end, intr.w, intr.h,
               dead_flag, ray_list, list_ctr, depth, normals, kRayJumpCells, v.d_sched, v.d_patch_order);
    SF_LAUNCH_CHECK();
    if (launches) *launches += 1;
}

// Active-ray list from caller-supplied bounds (raycast(..., bounds), render.hpp:61-63);
// pixels with empty bounds get the empty raycast result.
__global__ void k_list_from_bounds(const float* __restrict__ t_start, const float* __restrict__ t_end, int n,
                                   int* __restrict__ ray_list, RayCounters* list_ctr, float* __restrict__ depth_out,
                                   float* __restrict__ normals_out) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const bool act = idx < n && t_start[idx] <= t_end[idx];
    if (idx < n && !act) {
        depth_out[idx] = 0.0f;
        normals_out[3 * idx] = 0.0f;
        normals_out[3 * idx + 1] = 0.0f;
        normals_out[3 * idx + 2] = 0.0f;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, act);
    const int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (bal) {
        const int leader = __ffs(bal) - 1;
        if (lane == leader) base = atomicAdd(&list_ctr->listed, static_cast<unsigned long long>(__popc(bal)));
        base = __shfl_sync(0xffffffffu, base, leader);
    }
    if (act) ray_list[base + __popc(bal & ((1u << lane) - 1u))] = idx;
}

// Composite of per-rank raycasts (sf_gpu.h): nearest depth wins, a rank with a normal wins
// ties against one without, then the lower rank.
__global__ void k_composite_key(const float* __restrict__ depth, const float* __restrict__ normals, uint64_t n,
                                int rank, long long* __restrict__ key) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float d = depth[i];
    long long k = 0x7fffffffffffffffLL;
    if (d > 0.0f) {
        const bool no_normal = normals[3 * i] == 0.0f && normals[3 * i + 1] == 0.0f && normals[3 * i + 2] == 0.0f;
        k = (static_cast<long long>(__float_as_uint(d)) << 32) | (static_cast<long long>(no_normal) << 31) |
            static_cast<long long>(rank);
    }
    key[i] = k;
}
__global__ void k_composite_select(const long long* __restrict__ key, uint64_t n, int rank, float* __restrict__ depth,
                                   float* __restrict__ normals) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long k = key[i];
    const bool win = k != 0x7fffffffffffffffLL && static_cast<int>(k & 0x7fffffff) == rank;
    if (!win) {
        depth[i] = 0.0f;
        normals[3 * i] = 0.0f;
        normals[3 * i + 1] = 0.0f;
        normals[3 * i + 2] = 0.0f;
    }
}

void launch_raycast(Volume& v, const FrameConsts* d_fc, const Intr& intr, const float* t_start, const float* t_end,
                    float* depth, float* normals, RayCounters* d_stats, cudaStream_t s, uint64_t* launches,
                    const int* dead_flag, const int* ray_list, RayBracket* brackets) {
    constexpr int G = 8;  // lanes per ray: 32 rays per 256-thread CTA, persistent over the list
    const dim3 blk(256), grd(148 * SF_RAYCAST_CTAS);
    launch_pdl(k_raycast<G>, grd, blk, 0, s, v.P, d_fc, v.d_table, v.d_payload, v.d_occ, v.d_aux, t_start, t_end,
               depth, normals, d_stats, intr.w, intr.h, dead_flag, ray_list, brackets);
    SF_LAUNCH_CHECK();
    // one warp per CTA: the ~30 k bracketed rays spread over all SMs (latency-bound, few warps)
#ifndef SF_REFINE_CTAS
#define SF_REFINE_CTAS 16
#endif
#ifndef SF_REFINE_THREADS
#define SF_REFINE_THREADS 32
#endif
    launch_pdl(k_raycast_refine, dim3(148 * SF_REFINE_CTAS), dim3(SF_REFINE_THREADS), 0, s, v.P, d_fc, v.d_table, v.d_payload, v.d_occ,
               v.d_aux, brackets, depth, normals, d_stats, intr.w, dead_flag);
    SF_LAUNCH_CHECK();
    if (launches) *launches += 2;
}

// Scratch for the stand-alone raycast API.
struct RayScratch {
    int w = 0, h = 0;
    float *ts = nullptr, *te = nullptr, *depth = nullptr, *normals = nullptr;
    int* list = nullptr;
    RayBracket* brackets = nullptr;
    FrameConsts* fc = nullptr;
    double* pose = nullptr;
    RayCounters* stats = nullptr;
    void ensure(int W, int H) {
        if (W == w && H == h && ts) return;
        release();
        const size_t n = static_cast<size_t>(W) * H;
        SF_CUDA(cudaMalloc(&ts, n * sizeof(float)));
        SF_CUDA(cudaMalloc(&te, n * sizeof(float)));
        SF_CUDA(cudaMalloc(&depth, n * sizeof(float)));
        SF_CUDA(cudaMalloc(&normals, 3 * n * sizeof(float)));
        SF_CUDA(cudaMalloc(&fc, sizeof(FrameConsts)));
        SF_CUDA(cudaMalloc(&pose, 12 * sizeof(double)));
        SF_CUDA(cudaMalloc(&stats, sizeof(RayCounters)));
        SF_CUDA(cudaMalloc(&list, n * sizeof(int)));
        SF_CUDA(cudaMalloc(&brackets, n * sizeof(RayBracket)));
        w = W;
        h = H;
    }
    void release() {
        void* p[] = {ts, te, depth, normals, fc, pose, stats, list, brackets};
        for (void* q : p)
            if (q) cudaFree(q);
        ts = te = depth = normals = nullptr;
        list = nullptr;
        brackets = nullptr;
        fc = nullptr;
        pose = nullptr;
        stats = nullptr;
        w = h = 0;
    }
};

static void validate_intr(const sf_intrinsics& i) {
    if (i.width <= 0 || i.height <= 0) throw Error(SF_INVALID_ARGUMENT, "intrinsics: non-positive image size");
    if (i.fx <= 0.0 || i.fy <= 0.0) throw Error(SF_INVALID_ARGUMENT, "intrinsics: non-positive focal length");
    if (!(i.near_plane > 0.0) || !(i.near_plane < i.far_plane))
        throw Error(SF_INVALID_ARGUMENT, "intrinsics: need 0 < near < far");
}

}  // namespace sf

using namespace sf;

static RayScratch& ray_scratch() {
    static thread_local RayScratch rs;
    return rs;
}

extern "C" {

int sf_ray_bounds(sf_volume_t v, const double pose[12], const sf_intrinsics* intr, float* t_start, float* t_end,
                  int32_t out_on_device, void* stream) {
    return guarded([&]() -> int {
        SF_CUDA(cudaSetDevice(v->device));
        validate_intr(*intr);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        RayScratch& rs = ray_scratch();
        rs.ensure(intr->width, intr->height);
        const Intr I = to_intr(*intr);
        SF_CUDA(cudaMemcpyAsync(rs.pose, pose, 12 * sizeof(double), cudaMemcpyHostToDevice, s));
        launch_consts(v->P, I, rs.pose, rs.fc, s, nullptr);
        float* ts = out_on_device ? t_start : rs.ts;
        float* te = out_on_device ? t_end : rs.te;
        launch_ray_bounds(*v, rs.fc, I, ts, te, s, nullptr, nullptr);
        const size_t n = static_cast<size_t>(intr->width) * intr->height;
        if (!out_on_device) {
            SF_CUDA(cudaMemcpyAsync(t_start, rs.ts, n * sizeof(float), cudaMemcpyDeviceToHost, s));
            SF_CUDA(cudaMemcpyAsync(t_end, rs.te, n * sizeof(float), cudaMemcpyDeviceToHost, s));
        }
        SF_CUDA(cudaStreamSynchronize(s));
        return SF_OK;
    });
}

int sf_raycast(sf_volume_t v, const double pose[12], const sf_intrinsics* intr, float* depth, float* normals_xyz,
               int32_t out_on_device, sf_raycast_stats* stats, void* stream) {
    return guarded([&]() -> int {
        if (v) require_codes(*v, "raycast");
        SF_CUDA(cudaSetDevice(v->device));
        validate_intr(*intr);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        RayScratch& rs = ray_scratch();
        rs.ensure(intr->width, intr->height);
        const Intr I = to_intr(*intr);
        SF_CUDA(cudaMemcpyAsync(rs.pose, pose, 12 * sizeof(double), cudaMemcpyHostToDevice, s));
        SF_CUDA(cudaMemsetAsync(rs.stats, 0, sizeof(RayCounters), s));
        launch_consts(v->P, I, rs.pose, rs.fc, s, nullptr);
        float* d = out_on_device ? depth : rs.depth;
        float* nm = out_on_device ? normals_xyz : rs.normals;
        launch_ray_bounds(*v, rs.fc, I, rs.ts, rs.te, s, nullptr, nullptr, rs.list, rs.stats, d, nm);
        launch_raycast(*v, rs.fc, I, rs.ts, rs.te, d, nm, rs.stats, s, nullptr, nullptr, rs.list, rs.brackets);
        const size_t n = static_cast<size_t>(intr->width) * intr->height;
        if (!out_on_device) {
            SF_CUDA(cudaMemcpyAsync(depth, rs.depth, n * sizeof(float), cudaMemcpyDeviceToHost, s));
            SF_CUDA(cudaMemcpyAsync(normals_xyz, rs.normals, 3 * n * sizeof(float), cudaMemcpyDeviceToHost, s));
        }
        RayCounters c{};
        SF_CUDA(cudaMemcpyAsync(&c, rs.stats, sizeof(c), cudaMemcpyDeviceToHost, s));
        SF_CUDA(cudaStreamSynchronize(s));
        if (stats) {
            stats->sample_steps = c.sample_steps;
            stats->hit_pixels = c.hit_pixels;
            stats->rays_with_bounds = c.rays_with_bounds;
        }
        return SF_OK;
    });
}

int sf_raycast_with_bounds(sf_volume_t v, const double pose[12], const sf_intrinsics* intr, const float* t_start,
                           const float* t_end, float* depth, float* normals_xyz, int32_t on_device,
                           sf_raycast_stats* stats, void* stream) {
    return guarded([&]() -> int {
        if (v) require_codes(*v, "raycast");
        if (!v || !pose || !intr || !t_start || !t_end || !depth || !normals_xyz)
            throw Error(SF_INVALID_ARGUMENT, "sf_raycast_with_bounds: null argument");
        SF_CUDA(cudaSetDevice(v->device));
        validate_intr(*intr);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        RayScratch& rs = ray_scratch();
        rs.ensure(intr->width, intr->height);
        const Intr I = to_intr(*intr);
        const size_t n = static_cast<size_t>(intr->width) * intr->height;
        SF_CUDA(cudaMemcpyAsync(rs.pose, pose, 12 * sizeof(double), cudaMemcpyHostToDevice, s));
        SF_CUDA(cudaMemsetAsync(rs.stats, 0, sizeof(RayCounters), s));
        launch_consts(v->P, I, rs.pose, rs.fc, s, nullptr);
        const float* ts = t_start;
        const float* te = t_end;
        if (!on_device) {
            SF_CUDA(cudaMemcpyAsync(rs.ts, t_start, n * sizeof(float), cudaMemcpyHostToDevice, s));
            SF_CUDA(cudaMemcpyAsync(rs.te, t_end, n * sizeof(float), cudaMemcpyHostToDevice, s));
            ts = rs.ts;
            te = rs.te;
        }
        float* d = on_device ? depth : rs.depth;
        float* nm = on_device ? normals_xyz : rs.normals;
        k_list_from_bounds<<<(int)((n + 255) / 256), 256, 0, s>>>(ts, te, (int)n, rs.list, rs.stats, d, nm);
        SF_LAUNCH_CHECK();
        launch_raycast(*v, rs.fc, I, ts, te, d, nm, rs.stats, s, nullptr, nullptr, rs.list, rs.brackets);
        if (!on_device) {
            SF_CUDA(cudaMemcpyAsync(depth, rs.depth, n * sizeof(float), cudaMemcpyDeviceToHost, s));
            SF_CUDA(cudaMemcpyAsync(normals_xyz, rs.normals, 3 * n * sizeof(float), cudaMemcpyDeviceToHost, s));
        }
        RayCounters c{};
        SF_CUDA(cudaMemcpyAsync(&c, rs.stats, sizeof(c), cudaMemcpyDeviceToHost, s));
        SF_CUDA(cudaStreamSynchronize(s));
        if (stats) {
            stats->sample_steps = c.sample_steps;
            stats->hit_pixels = c.hit_pixels;
            stats->rays_with_bounds = c.rays_with_bounds;
        }
        return SF_OK;
    });
}

int sf_composite_key(const float* depth, const float* normals_xyz, uint64_t n, int32_t rank, int64_t* key,
                     void* stream) {
    return guarded([&]() -> int {
        if (!depth || !normals_xyz || !key || rank < 0) throw Error(SF_INVALID_ARGUMENT, "sf_composite_key: bad argument");
        if (n == 0) return SF_OK;
        k_composite_key<<<(unsigned)((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
            depth, normals_xyz, n, rank, reinterpret_cast<long long*>(key));
        SF_LAUNCH_CHECK();
        return SF_OK;
    });
}

int sf_composite_select(const int64_t* key, uint64_t n, int32_t rank, float* depth, float* normals_xyz,
                        void* stream) {
    return guarded([&]() -> int {
        if (!depth || !normals_xyz || !key || rank < 0)
            throw Error(SF_INVALID_ARGUMENT, "sf_composite_select: bad argument");
        if (n == 0) return SF_OK;
        k_composite_select<<<(unsigned)((n + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
            reinterpret_cast<const long long*>(key), n, rank, depth, normals_xyz);
        SF_LAUNCH_CHECK();
        return SF_OK;
    });
}

}  // extern "C"

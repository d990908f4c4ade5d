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
#include <vector>

#include "sf_internal.h"

namespace sf {

__device__ __forceinline__ bool occupied(const uint32_t* __restrict__ occ, uint64_t ti) {
    return (__ldg(&occ[ti >> 5]) >> (ti & 31)) & 1u;
}

__global__ void k_ray_bounds(VolParams P, const FrameConsts* __restrict__ fc, const uint32_t* __restrict__ occ,
                             const VolCounters* __restrict__ vc, float* __restrict__ t_start,
                             float* __restrict__ t_end, int w, int h, const int* dead) {
    // Coarse occupancy (1 bit per 16^3 blocks) staged in shared memory: the DDA only reads
    // the fine bitmap (L2) inside super-blocks that ever held a block. Exact: a clear coarse
    // bit implies every block of the super-block is EMPTY.
    extern __shared__ uint32_t s_coarse[];
    if (dead && *dead) return;
    {
        const int tid = threadIdx.y * blockDim.x + threadIdx.x;
        const uint64_t nc = P.Nc;
        const int cwords = static_cast<int>((nc * nc * nc + 31) / 32);
        for (int i = tid; i < cwords; i += blockDim.x * blockDim.y) s_coarse[i] = __ldg(&occ[P.occ_fine_words + i]);
        __syncthreads();
    }
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    const int v = blockIdx.y * blockDim.y + threadIdx.y;
    if (u >= w || v >= h) return;
    const size_t idx = (size_t)v * w + u;
    float ts = INFINITY, te = -INFINITY;
    if (vc->allocated_count != 0) {
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
            int sx, sy, sz;
            double tmx, tmy, tmz, tdx, tdy, tdz;
            init_axis(dir[0], box_lo[0], cx, ex, sx, tmx, tdx);
            init_axis(dir[1], box_lo[1], cy, ey, sy, tmy, tdy);
            init_axis(dir[2], box_lo[2], cz, ez, sz, tmz, tdz);
            double first = INFINITY, last = -INFINITY;
            double t_in = lo;
            while (t_in <= hi) {
                // Past the occupied box in the direction of travel: no later cell can be
                // allocated (cells move monotonically per axis), so first/last are final.
                if ((sx >= 0 && cx > bx1) || (sx <= 0 && cx < bx0) || (sy >= 0 && cy > by1) || (sy <= 0 && cy < by0) ||
                    (sz >= 0 && cz > bz1) || (sz <= 0 && cz < bz0))
                    break;
                const int axis = tmx <= tmy ? (tmx <= tmz ? 0 : 2) : (tmy <= tmz ? 1 : 2);
                const double tm = axis == 0 ? tmx : (axis == 1 ? tmy : tmz);
                const double t_out = dmin(tm, hi);
                if (cx >= bx0 && cx <= bx1 && cy >= by0 && cy <= by1 && cz >= bz0 && cz <= bz1) {
                    const int cc = ((cz >> kCoarseShift) * P.Nc + (cy >> kCoarseShift)) * P.Nc + (cx >> kCoarseShift);
                    if (((s_coarse[cc >> 5] >> (cc & 31)) & 1u) && occupied(occ, table_index(P, cx, cy, cz))) {
                        first = dmin(first, t_in);
                        last = dmax(last, t_out);
                    }
                }
                t_in = tm;
                if (axis == 0) {
                    cx += sx;
                    if (cx < 0 || cx >= n) break;
                    tmx += tdx;
                } else if (axis == 1) {
                    cy += sy;
                    if (cy < 0 || cy >= n) break;
                    tmy += tdy;
                } else {
                    cz += sz;
                    if (cz < 0 || cz >= n) break;
                    tmz += tdz;
                }
            }
            if (first <= last) {
                ts = (float)dmax(first, lo);
                te = (float)dmin(last, hi);
            }
        }
    }
    t_start[idx] = ts;
    t_end[idx] = te;
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

    __device__ bool sample(d3 p, double& out) const {
        const double gx = (p.x - P.ox) / P.voxel - 0.5;
        const double gy = (p.y - P.oy) / P.voxel - 0.5;
        const double gz = (p.z - P.oz) / P.voxel - 0.5;
        const int bx = ref_floor_int(gx), by = ref_floor_int(gy), bz = ref_floor_int(gz);
        const int res = P.res;
        if (bx < 0 || by < 0 || bz < 0 || bx + 1 >= res || by + 1 >= res || bz + 1 >= res) return false;
        // The base corner's block EMPTY => voxel_code fails => nullopt (render.cpp:14-15,39):
        // decided from the 1-bit occupancy map without touching the 4-byte table.
        if (!occupied(occ, table_index(P, blk(bx), blk(by), blk(bz)))) return false;
        const double fx = gx - (double)bx, fy = gy - (double)by, fz = gz - (double)bz;
        double c[8];
        for (int i = 0; i < 8; ++i)
            if (!code(bx + (i & 1), by + ((i >> 1) & 1), bz + ((i >> 2) & 1), c[i])) return false;
        const double x0 = c[0] + (c[1] - c[0]) * fx;
        const double x1 = c[2] + (c[3] - c[2]) * fx;
        const double x2 = c[4] + (c[5] - c[4]) * fx;
        const double x3 = c[6] + (c[7] - c[6]) * fx;
        const double y0 = x0 + (x1 - x0) * fy;
        const double y1 = x2 + (x3 - x2) * fy;
        out = y0 + (y1 - y0) * fz;
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

__global__ void __launch_bounds__(256)
    k_raycast(VolParams P, const FrameConsts* __restrict__ fc, const int32_t* __restrict__ table,
              const uint16_t* __restrict__ payload, const uint32_t* __restrict__ occ, const AuxTables* __restrict__ aux,
              const float* __restrict__ t_start, const float* __restrict__ t_end, float* __restrict__ depth_out,
              float* __restrict__ normals_out, RayCounters* stats, int w, int h, const int* dead) {
    __shared__ double s_tdec[256];
    if (dead && *dead) return;
    const int tid = threadIdx.y * blockDim.x + threadIdx.x;
    for (int i = tid; i < 256; i += blockDim.x * blockDim.y) s_tdec[i] = aux->tsdf_decode[i];
    __syncthreads();
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    const int v = blockIdx.y * blockDim.y + threadIdx.y;
    unsigned long long steps = 0, hits = 0, with_bounds = 0;
    if (u < w && v < h) {
        const size_t idx = (size_t)v * w + u;
        float out_d = 0.0f, nx = 0.f, ny = 0.f, nz = 0.f;
        const float fs = t_start[idx], fe = t_end[idx];
        if (fs <= fe) {  // !bounds.empty(u, v)
            with_bounds = 1;
            const Sampler S{P, table, payload, occ, s_tdec};
            const Intr& intr = fc->intr;
            const Pose& pose = fc->pose;
            const double vox = P.voxel;
            const double coarse_step = 0.5 * P.delta;
            const double fine_tol = 0.01 * vox;
            const d3 dir_cam = normalized(unproject(intr, u, v, 1.0));
            const d3 dir = mv(pose.R, dir_cam);
            const double t0 = fs, t1 = fe;
            double prev_t = 0.0, prev_val = 0.0;
            bool have_prev = false, bracketed = false;
            double hit_a = 0.0, hit_b = 0.0, val_a = 0.0, val_b = 0.0;
            for (double t = t0;; t += coarse_step) {
                const bool final_sample = t >= t1;
                if (final_sample) t = t1;
                ++steps;
                double val;
                if (S.sample(add(pose.t, scale(t, dir)), val)) {
                    if (have_prev && prev_val > 0.0 && val < 0.0) {
                        hit_a = prev_t;
                        val_a = prev_val;
                        hit_b = t;
                        val_b = val;
                        bracketed = true;
                        break;
                    }
                    have_prev = true;
                    prev_t = t;
                    prev_val = val;
                }
                if (final_sample) break;
            }
            if (bracketed) {
                double root = hit_b;
                for (int iter = 0; iter < 48 && hit_b - hit_a > fine_tol; ++iter) {
                    double t_new = hit_b - val_b * (hit_b - hit_a) / (val_b - val_a);
                    if (!(t_new > hit_a) || !(t_new < hit_b)) t_new = 0.5 * (hit_a + hit_b);
                    double val;
                    if (!S.sample(add(pose.t, scale(t_new, dir)), val)) {
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
                if (val_b != val_a) {
                    const double interp = hit_b - val_b * (hit_b - hit_a) / (val_b - val_a);
                    root = dclamp(interp, hit_a, hit_b);
                } else {
                    root = 0.5 * (hit_a + hit_b);
                }
                const double dd = root * dir_cam.z;
                if (!(dd < intr.near_plane || dd > intr.far_plane)) {
                    out_d = (float)dd;
                    hits = 1;
                    d3 g;
                    if (S.gradient(add(pose.t, scale(root, dir)), vox, g) && sqnorm(g) > 0.0) {
                        // world_to_cam * grad.normalized()  (render.cpp:242-245)
                        const d3 n_cam = mv(mt(pose.R), normalized(g));
                        nx = (float)n_cam.x;
                        ny = (float)n_cam.y;
                        nz = (float)n_cam.z;
                    }
                }
            }
        }
        depth_out[idx] = out_d;
        normals_out[3 * idx] = nx;
        normals_out[3 * idx + 1] = ny;
        normals_out[3 * idx + 2] = nz;
    }
    // RaycastStats: warp reduction, one atomic per warp and counter.
    for (int off = 16; off > 0; off >>= 1) {
        steps += __shfl_down_sync(0xffffffffu, steps, off);
        hits += __shfl_down_sync(0xffffffffu, hits, off);
        with_bounds += __shfl_down_sync(0xffffffffu, with_bounds, off);
    }
    if ((tid & 31) == 0 && stats) {
        if (steps) atomicAdd(&stats->sample_steps, steps);
        if (hits) atomicAdd(&stats->hit_pixels, hits);
        if (with_bounds) atomicAdd(&stats->rays_with_bounds, with_bounds);
    }
}

void launch_ray_bounds(Volume& v, const FrameConsts* d_fc, const Intr& intr, float* t_start, float* t_end,
                       cudaStream_t s, uint64_t* launches, const int* dead_flag) {
    const dim3 blk(32, 8), grd((intr.w + 31) / 32, (intr.h + 7) / 8);
    const uint64_t nc = v.P.Nc;
    const size_t smem = ((nc * nc * nc + 31) / 32) * sizeof(uint32_t);
    if (smem > 48 * 1024) SF_CUDA(cudaFuncSetAttribute(k_ray_bounds, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_ray_bounds<<<grd, blk, smem, s>>>(v.P, d_fc, v.d_occ, v.d_vc, t_start, t_end, intr.w, intr.h, dead_flag);
    SF_LAUNCH_CHECK();
    if (launches) *launches += 1;
}

void launch_raycast(Volume& v, const FrameConsts* d_fc, const Intr& intr, const float* t_start, const float* t_end,
                    float* depth, float* normals, RayCounters* d_stats, cudaStream_t s, uint64_t* launches,
                    const int* dead_flag) {
    const dim3 blk(32, 4), grd((intr.w + 31) / 32, (intr.h + 3) / 4);
    k_raycast<<<grd, blk, 0, s>>>(v.P, d_fc, v.d_table, v.d_payload, v.d_occ, v.d_aux, t_start, t_end, depth, normals,
                                  d_stats, intr.w, intr.h, dead_flag);
    SF_LAUNCH_CHECK();
    if (launches) *launches += 1;
}

// Scratch for the stand-alone raycast API.
struct RayScratch {
    int w = 0, h = 0;
    float *ts = nullptr, *te = nullptr, *depth = nullptr, *normals = nullptr;
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
        w = W;
        h = H;
    }
    void release() {
        void* p[] = {ts, te, depth, normals, fc, pose, stats};
        for (void* q : p)
            if (q) cudaFree(q);
        ts = te = depth = normals = nullptr;
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
        SF_CUDA(cudaSetDevice(v->device));
        validate_intr(*intr);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        RayScratch& rs = ray_scratch();
        rs.ensure(intr->width, intr->height);
        const Intr I = to_intr(*intr);
        SF_CUDA(cudaMemcpyAsync(rs.pose, pose, 12 * sizeof(double), cudaMemcpyHostToDevice, s));
        SF_CUDA(cudaMemsetAsync(rs.stats, 0, sizeof(RayCounters), s));
        launch_consts(v->P, I, rs.pose, rs.fc, s, nullptr);
        launch_ray_bounds(*v, rs.fc, I, rs.ts, rs.te, s, nullptr, nullptr);
        float* d = out_on_device ? depth : rs.depth;
        float* nm = out_on_device ? normals_xyz : rs.normals;
        launch_raycast(*v, rs.fc, I, rs.ts, rs.te, d, nm, rs.stats, s, nullptr, nullptr);
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

}  // extern "C"

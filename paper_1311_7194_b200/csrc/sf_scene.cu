// sf_scene.cu — synthetic depth input (scene.cpp:13-147), the input side of the benches.
//
// Sphere tracing runs on the device, one thread per pixel, FP64 in the reference order, so
// noise-free frames are bit-identical to render_synthetic_depth. The Gaussian noise of a
// noisy frame is a sequential draw over hit pixels in row-major order
// (std::mt19937_64 + std::normal_distribution, scene.cpp:111-138); it is applied on the
// host with the same standard library, so noisy frames match the reference bit for bit too.
#include <cmath>
#include <random>
#include <vector>

#include "sf_internal.h"

namespace sf {

struct SceneDev {
    int ns, np, nb;
    const double* spheres;  // cx cy cz r
    const double* planes;   // nx ny nz offset (normalised)
    const double* boxes;    // cx cy cz hx hy hz (axis-aligned, identity rotation)
};

__device__ double scene_sdf(const SceneDev& S, d3 x) {
    double best = INFINITY;
    for (int i = 0; i < S.ns; ++i) {
        const double* s = S.spheres + 4 * i;
        const double d = sqrt(sqnorm(sub(x, mk(s[0], s[1], s[2])))) - s[3];
        best = dmin(best, d);
    }
    for (int i = 0; i < S.np; ++i) {
        const double* p = S.planes + 4 * i;
        const double d = dot(mk(p[0], p[1], p[2]), x) - p[3];
        best = dmin(best, d);
    }
    for (int i = 0; i < S.nb; ++i) {
        const double* b = S.boxes + 6 * i;
        // local = R^T (x - t) with R = identity (scene.cpp:21-26)
        m33 I;
        for (int k = 0; k < 9; ++k) I.m[k] = (k % 4 == 0) ? 1.0 : 0.0;
        const d3 local = mv(mt(I), sub(x, mk(b[0], b[1], b[2])));
        const d3 q = sub(mk(fabs(local.x), fabs(local.y), fabs(local.z)), mk(b[3], b[4], b[5]));
        const d3 outside = mk(dmax(q.x, 0.0), dmax(q.y, 0.0), dmax(q.z, 0.0));
        double mx = q.x;
        mx = mx < q.y ? q.y : mx;
        mx = mx < q.z ? q.z : mx;
        const double d = sqrt(sqnorm(outside)) + dmin(mx, 0.0);
        best = dmin(best, d);
    }
    return best;
}

__global__ void k_sphere_trace(SceneDev S, Pose pose, Intr intr, int max_steps, double tolerance,
                               double* __restrict__ out) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    const int v = blockIdx.y * blockDim.y + threadIdx.y;
    if (u >= intr.w || v >= intr.h) return;
    const d3 dir_cam = normalized(unproject(intr, u, v, 1.0));
    const d3 dir = mv(pose.R, dir_cam);
    const double t_near = intr.near_plane / dir_cam.z;
    const double t_far = intr.far_plane / dir_cam.z;
    double t = t_near, depth = 0.0;
    for (int step = 0; step < max_steps && t <= t_far; ++step) {
        const d3 x = add(pose.t, scale(t, dir));
        const double d = scene_sdf(S, x);
        if (d < tolerance) {
            depth = t * dir_cam.z;
            break;
        }
        t += d;
    }
    out[(size_t)v * intr.w + u] = depth;
}

}  // namespace sf

using namespace sf;

extern "C" int sf_render_synthetic_depth(const sf_scene* scene, const double pose[12], const sf_intrinsics* intr,
                                         double noise_sigma0, uint64_t noise_seed, int32_t max_steps,
                                         double tolerance_scale, double domain_size, float* depth_host,
                                         float* sigma_host) {
    return guarded([&]() -> int {
        if (intr->width <= 0 || intr->height <= 0)
            throw Error(SF_INVALID_ARGUMENT, "intrinsics: non-positive image size");
        const size_t n = static_cast<size_t>(intr->width) * intr->height;
        const bool noisy = noise_sigma0 > 0.0;
        std::fill(depth_host, depth_host + n, 0.0f);
        if (sigma_host) std::fill(sigma_host, sigma_host + n, 0.0f);
        const int ns = scene->sphere_count, np = scene->plane_count, nb = scene->box_count;
        if (ns + np + nb == 0) return SF_OK;
        // AnalyticScene::add_plane normalisation (scene.cpp:53-57), add_sphere/add_box checks.
        std::vector<double> planes(4 * np);
        for (int i = 0; i < np; ++i) {
            const double* p = scene->planes + 4 * i;
            const double len = std::sqrt((p[0] * p[0] + p[1] * p[1]) + p[2] * p[2]);
            if (!(len > 0.0)) throw Error(SF_INVALID_ARGUMENT, "scene: plane normal must be nonzero");
            planes[4 * i + 0] = p[0] / len;
            planes[4 * i + 1] = p[1] / len;
            planes[4 * i + 2] = p[2] / len;
            planes[4 * i + 3] = p[3] / len;
        }
        for (int i = 0; i < ns; ++i)
            if (!(scene->spheres[4 * i + 3] > 0.0))
                throw Error(SF_INVALID_ARGUMENT, "scene: sphere radius must be positive");
        double *d_s = nullptr, *d_p = nullptr, *d_b = nullptr, *d_out = nullptr;
        SF_CUDA(cudaMalloc(&d_s, std::max(1, 4 * ns) * sizeof(double)));
        SF_CUDA(cudaMalloc(&d_p, std::max(1, 4 * np) * sizeof(double)));
        SF_CUDA(cudaMalloc(&d_b, std::max(1, 6 * nb) * sizeof(double)));
        SF_CUDA(cudaMalloc(&d_out, n * sizeof(double)));
        if (ns) SF_CUDA(cudaMemcpy(d_s, scene->spheres, 4 * ns * sizeof(double), cudaMemcpyHostToDevice));
        if (np) SF_CUDA(cudaMemcpy(d_p, planes.data(), 4 * np * sizeof(double), cudaMemcpyHostToDevice));
        if (nb) SF_CUDA(cudaMemcpy(d_b, scene->boxes, 6 * nb * sizeof(double), cudaMemcpyHostToDevice));
        SceneDev S{ns, np, nb, d_s, d_p, d_b};
        const Intr I = to_intr(*intr);
        const double tolerance = tolerance_scale * domain_size;
        const dim3 blk(32, 4), grd((I.w + 31) / 32, (I.h + 3) / 4);
        k_sphere_trace<<<grd, blk>>>(S, pose_from12(pose), I, max_steps, tolerance, d_out);
        SF_LAUNCH_CHECK();
        std::vector<double> depth(n);
        SF_CUDA(cudaMemcpy(depth.data(), d_out, n * sizeof(double), cudaMemcpyDeviceToHost));
        cudaFree(d_s);
        cudaFree(d_p);
        cudaFree(d_b);
        cudaFree(d_out);
        std::mt19937_64 rng(noise_seed);
        std::normal_distribution<double> gauss(0.0, 1.0);
        for (size_t i = 0; i < n; ++i) {
            double d = depth[i];
            if (d <= 0.0) continue;
            if (noisy) {
                const double sigma = noise_sigma0 * d * d;
                d += sigma * gauss(rng);
                if (sigma_host) sigma_host[i] = static_cast<float>(sigma);
            }
            if (d < intr->near_plane || d > intr->far_plane) {
                if (noisy && sigma_host) sigma_host[i] = 0.0f;
                continue;
            }
            depth_host[i] = static_cast<float>(d);
        }
        return SF_OK;
    });
}

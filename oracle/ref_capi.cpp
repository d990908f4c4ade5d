// C-ABI wrapper around the UNMODIFIED reference library — TEST INFRASTRUCTURE ONLY.
//
// Built with the reference sources into oracle/_ref/libsfref.so (oracle/Makefile). Each
// sfref_* function has the signature of the matching sf_* entry point in include/sf_gpu.h
// and forwards to the reference's public C++ API, so tests (and bench.py's reference /
// cpu_baseline legs) can run the reference and the CUDA path on identical inputs.
#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "../include/sf_gpu.h"
#include "sparsefusion/camera.hpp"
#include "sparsefusion/fusion.hpp"
#include "sparsefusion/frame_io.hpp"
#include "sparsefusion/grid.hpp"
#include "sparsefusion/marching_cubes.hpp"
#include "sparsefusion/pose.hpp"
#include "sparsefusion/registration.hpp"
#include "sparsefusion/render.hpp"
#include "sparsefusion/scene.hpp"

using namespace sparsefusion;

struct sfref_volume {
    std::unique_ptr<SparseTsdfGrid> grid;
};
struct sfref_mesh {
    Mesh mesh;
};

namespace {

thread_local std::string g_error;

int fail(int code, const std::string& msg) {
    g_error = msg;
    return code;
}

template <typename F>
int guarded(F&& f) {
    try {
        g_error.clear();
        return f();
    } catch (const PoolExhausted& e) {
        return fail(SF_POOL_EXHAUSTED, e.what());
    } catch (const TrackingLost& e) {
        return fail(SF_TRACKING_LOST, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(SF_INVALID_ARGUMENT, e.what());
    } catch (const std::out_of_range& e) {
        return fail(SF_OUT_OF_RANGE, e.what());
    } catch (const std::logic_error& e) {
        return fail(SF_LOGIC_ERROR, e.what());
    } catch (const std::exception& e) {
        return fail(SF_IO_ERROR, e.what());
    }
}

GridConfig to_config(const sf_grid_config* c) {
    GridConfig g;
    g.blocks_per_axis = c->blocks_per_axis;
    g.voxels_per_block_axis = c->voxels_per_block_axis;
    g.box_origin = Eigen::Vector3d(c->box_origin[0], c->box_origin[1], c->box_origin[2]);
    g.box_side = c->box_side;
    g.truncation = c->truncation;
    return g;
}

AuxQuantization to_aux(const sf_aux_quant* a) {
    AuxQuantization q;
    if (!a) return q;
    q.mode = a->mode == 0 ? AuxMode::Weight : AuxMode::Variance;
    q.w_max = a->w_max;
    q.p_min = a->p_min;
    q.p_max = a->p_max;
    return q;
}

Intrinsics to_intr(const sf_intrinsics* i) {
    Intrinsics r;
    r.width = i->width;
    r.height = i->height;
    r.fx = i->fx;
    r.fy = i->fy;
    r.cx = i->cx;
    r.cy = i->cy;
    r.near_plane = i->near_plane;
    r.far_plane = i->far_plane;
    return r;
}

Pose to_pose(const double* p) {
    Pose pose;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) pose.rotation(r, c) = p[r * 3 + c];
    pose.translation = Eigen::Vector3d(p[9], p[10], p[11]);
    return pose;
}

void from_pose(const Pose& pose, double* p) {
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) p[r * 3 + c] = pose.rotation(r, c);
    for (int i = 0; i < 3; ++i) p[9 + i] = pose.translation[i];
}

DepthFrame to_frame(const sf_frame* f) {
    DepthFrame d(to_intr(&f->intrinsics));
    const std::size_t n = d.pixel_count();
    std::memcpy(d.depth.data(), f->depth, n * sizeof(float));
    if (f->sigma) d.sigma.assign(f->sigma, f->sigma + n);
    return d;
}

NormalMap to_normals(const float* xyz, int w, int h) {
    NormalMap m(w, h);
    for (std::size_t i = 0; i < m.normals.size(); ++i)
        m.normals[i] = Eigen::Vector3f(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
    return m;
}

void from_normals(const NormalMap& m, float* xyz) {
    for (std::size_t i = 0; i < m.normals.size(); ++i)
        for (int k = 0; k < 3; ++k) xyz[3 * i + k] = m.normals[i][k];
}

FusionParams to_fusion(const sf_fusion_params* p) {
    FusionParams f;
    f.mode = p->mode == 0 ? FusionMode::Simple : p->mode == 1 ? FusionMode::Weighted : FusionMode::Kalman;
    f.w_fixed = p->w_fixed;
    f.w_max = p->w_max;
    f.process_variance = p->process_variance;
    f.sigma0 = p->sigma0;
    f.delta = p->delta;
    f.refinement_steps = p->refinement_steps;
    f.edge_downweight = p->edge_downweight != 0;
    f.min_variance = p->min_variance;
    return f;
}

MatchParams to_match(const sf_match_params* p) {
    MatchParams m;
    m.max_distance = p->max_distance;
    m.max_normal_angle = p->max_normal_angle;
    m.max_iterations = p->max_iterations;
    m.convergence_epsilon = p->convergence_epsilon;
    m.eigen_threshold = p->eigen_threshold;
    m.shrink_floor = p->shrink_floor;
    m.normal_options.sigma0 = p->normal_sigma0;
    m.normal_options.spatial_scale = p->normal_spatial_scale;
    return m;
}

void from_icp(const IcpResult& r, sf_icp_result* out) {
    std::memset(out, 0, sizeof(*out));
    from_pose(r.delta, out->delta);
    out->iterations = r.iterations;
    out->matches = r.matches;
    for (int i = 0; i < 3; ++i) {
        out->motion_r[i] = r.solution.motion.r[i];
        out->motion_t[i] = r.solution.motion.t[i];
    }
    for (int i = 0; i < 6; ++i) {
        out->eigenvalues[i] = r.solution.eigenvalues[i];
        out->gated_mask[i] = r.solution.gated_mask[i] ? 1 : 0;
        for (int k = 0; k < 6; ++k) out->eigenvectors[i * 6 + k] = r.solution.eigenvectors(k, i);
    }
    out->residual_rms = r.solution.residual_rms;
    out->shrunk_motion_norm = r.solution.shrunk_motion_norm;
    out->pair_count = r.solution.pair_count;
}

AnalyticScene to_scene(const sf_scene* s) {
    AnalyticScene scene;
    for (int i = 0; i < s->sphere_count; ++i) {
        const double* p = s->spheres + 4 * i;
        scene.add_sphere({p[0], p[1], p[2]}, p[3]);
    }
    for (int i = 0; i < s->plane_count; ++i) {
        const double* p = s->planes + 4 * i;
        scene.add_plane({p[0], p[1], p[2]}, p[3]);
    }
    for (int i = 0; i < s->box_count; ++i) {
        const double* p = s->boxes + 6 * i;
        Pose pose;
        pose.translation = {p[0], p[1], p[2]};
        scene.add_box(pose, {p[3], p[4], p[5]});
    }
    return scene;
}

}  // namespace

extern "C" {

const char* sfref_last_error(void) { return g_error.c_str(); }

int sfref_volume_create(const sf_grid_config* config, uint64_t pool_capacity, const sf_aux_quant* aux,
                        int32_t /*device*/, sfref_volume** out) {
    return guarded([&]() -> int {
        auto v = std::make_unique<sfref_volume>();
        v->grid = std::make_unique<SparseTsdfGrid>(to_config(config), pool_capacity, to_aux(aux));
        *out = v.release();
        return SF_OK;
    });
}

int sfref_volume_destroy(sfref_volume* v) {
    delete v;
    return SF_OK;
}

int sfref_volume_get_info(sfref_volume* v, sf_volume_info* out) {
    const SparseTsdfGrid& g = *v->grid;
    std::memset(out, 0, sizeof(*out));
    const GridConfig& c = g.config();
    out->config.blocks_per_axis = c.blocks_per_axis;
    out->config.voxels_per_block_axis = c.voxels_per_block_axis;
    for (int i = 0; i < 3; ++i) out->config.box_origin[i] = c.box_origin[i];
    out->config.box_side = c.box_side;
    out->config.truncation = c.truncation;
    out->aux.mode = g.aux_quantization().mode == AuxMode::Weight ? 0 : 1;
    out->aux.w_max = g.aux_quantization().w_max;
    out->aux.p_min = g.aux_quantization().p_min;
    out->aux.p_max = g.aux_quantization().p_max;
    out->delta = g.delta();
    out->voxel_size = g.voxel_size();
    out->pool_capacity = g.pool_capacity();
    out->allocated_count = g.allocated_count();
    out->memory_bytes = g.memory_bytes();
    return SF_OK;
}

int sfref_volume_allocate_block(sfref_volume* v, const int32_t bc[3], int32_t* slot_out) {
    return guarded([&]() -> int {
        *slot_out = v->grid->allocate_block(Eigen::Vector3i(bc[0], bc[1], bc[2]));
        return SF_OK;
    });
}

int sfref_volume_free_block(sfref_volume* v, const int32_t bc[3]) {
    return guarded([&]() -> int {
        v->grid->free_block(Eigen::Vector3i(bc[0], bc[1], bc[2]));
        return SF_OK;
    });
}

int sfref_volume_block_slot(sfref_volume* v, const int32_t bc[3], int32_t* slot_out) {
    return guarded([&]() -> int {
        *slot_out = v->grid->block_slot(Eigen::Vector3i(bc[0], bc[1], bc[2]));
        return SF_OK;
    });
}

int sfref_volume_read_voxel(sfref_volume* v, const int32_t vc[3], int32_t* is_chi, double* tsdf, double* aux) {
    return guarded([&]() -> int {
        const auto r = v->grid->read_voxel(Eigen::Vector3i(vc[0], vc[1], vc[2]));
        *is_chi = r ? 0 : 1;
        *tsdf = r ? r->tsdf : 0.0;
        *aux = r ? r->aux : 0.0;
        return SF_OK;
    });
}

int sfref_volume_write_voxel(sfref_volume* v, const int32_t vc[3], int32_t tsdf_is_chi, double tsdf, double aux) {
    return guarded([&]() -> int {
        std::optional<double> t;
        if (!tsdf_is_chi) t = tsdf;
        v->grid->write_voxel(Eigen::Vector3i(vc[0], vc[1], vc[2]), t, aux);
        return SF_OK;
    });
}

int sfref_volume_read_table(sfref_volume* v, int32_t* table) {
    const SparseTsdfGrid& g = *v->grid;
    const std::size_t n = g.config().blocks_per_axis;
    std::fill(table, table + n * n * n, SparseTsdfGrid::kEmpty);
    for (const Eigen::Vector3i& bc : g.allocated_blocks())
        table[(static_cast<std::size_t>(bc.z()) * n + bc.y()) * n + bc.x()] = g.block_slot(bc);
    return SF_OK;
}

int sfref_volume_read_payload(sfref_volume* v, uint64_t first, uint64_t count, uint16_t* out) {
    const SparseTsdfGrid& g = *v->grid;
    if (first + count > g.pool_capacity()) return fail(SF_OUT_OF_RANGE, "payload range");
    const std::size_t vpb = g.voxels_per_block();
    for (uint64_t s = 0; s < count; ++s) {
        const auto p = g.block_payload(static_cast<int32_t>(first + s));
        std::memcpy(out + s * vpb, p.data(), vpb * sizeof(uint16_t));
    }
    return SF_OK;
}

int sfref_volume_write_payload(sfref_volume* v, uint64_t first, uint64_t count, const uint16_t* in) {
    SparseTsdfGrid& g = *v->grid;
    if (first + count > g.pool_capacity()) return fail(SF_OUT_OF_RANGE, "payload range");
    const std::size_t vpb = g.voxels_per_block();
    for (uint64_t s = 0; s < count; ++s) {
        auto p = g.block_payload(static_cast<int32_t>(first + s));
        std::memcpy(p.data(), in + s * vpb, vpb * sizeof(uint16_t));
    }
    return SF_OK;
}

int sfref_volume_check_consistency(sfref_volume* v) {
    return guarded([&]() -> int {
        v->grid->check_consistency();
        return SF_OK;
    });
}

int sfref_volume_save_snapshot(sfref_volume* v, const char* path) {
    return guarded([&]() -> int {
        v->grid->save_snapshot(path);
        return SF_OK;
    });
}

int sfref_volume_load_snapshot(const char* path, uint64_t pool_capacity, int32_t, sfref_volume** out) {
    return guarded([&]() -> int {
        auto v = std::make_unique<sfref_volume>();
        v->grid = std::make_unique<SparseTsdfGrid>(SparseTsdfGrid::load_snapshot(path, pool_capacity));
        *out = v.release();
        return SF_OK;
    });
}

// Dense float shadow (grid.hpp:77-88): oracle for the float payload mode, <= 128^3.
int sfref_volume_enable_shadow(sfref_volume* v) {
    return guarded([&]() -> int {
        v->grid->enable_shadow();
        return SF_OK;
    });
}

int sfref_volume_read_shadow(sfref_volume* v, float* tsdf, float* aux) {
    if (!v->grid->has_shadow()) return fail(SF_LOGIC_ERROR, "no shadow");
    const FloatShadowGrid& s = v->grid->shadow();
    std::memcpy(tsdf, s.tsdf.data(), s.tsdf.size() * sizeof(float));
    std::memcpy(aux, s.aux.data(), s.aux.size() * sizeof(float));
    return SF_OK;
}

int sfref_integrate(sfref_volume* v, const sf_frame* frame, const double pose[12],
                    const sf_fusion_params* params, sf_fusion_stats* stats, void*) {
    return guarded([&]() -> int {
        const DepthFrame f = to_frame(frame);
        const FusionStats s = fuse_frame(*v->grid, f, to_pose(pose), to_fusion(params));
        if (stats) {
            stats->voxels_updated = s.voxels_updated;
            stats->blocks_allocated_now = s.blocks_allocated_now;
            stats->blocks_total = s.blocks_total;
            stats->memory_bytes = s.memory_bytes;
        }
        return SF_OK;
    });
}

int sfref_select_update_blocks(sfref_volume* v, const sf_frame* frame, const double pose[12],
                               int32_t* alloc_xyz, uint64_t* alloc_count, int32_t* upd_xyz,
                               uint64_t* upd_count, void*) {
    return guarded([&]() -> int {
        const DepthFrame f = to_frame(frame);
        const UpdateLists lists = select_update_blocks(*v->grid, f, to_pose(pose));
        if (lists.allocate.size() > *alloc_count || lists.update.size() > *upd_count)
            return fail(SF_OUT_OF_RANGE, "select_update_blocks: output capacity");
        for (std::size_t i = 0; i < lists.allocate.size(); ++i)
            for (int k = 0; k < 3; ++k) alloc_xyz[3 * i + k] = lists.allocate[i][k];
        for (std::size_t i = 0; i < lists.update.size(); ++i)
            for (int k = 0; k < 3; ++k) upd_xyz[3 * i + k] = lists.update[i][k];
        *alloc_count = lists.allocate.size();
        *upd_count = lists.update.size();
        return SF_OK;
    });
}

int sfref_ray_bounds(sfref_volume* v, const double pose[12], const sf_intrinsics* intr, float* t_start,
                     float* t_end, int32_t, void*) {
    return guarded([&]() -> int {
        const RayBounds b = compute_ray_bounds(*v->grid, to_pose(pose), to_intr(intr));
        std::memcpy(t_start, b.t_start.data(), b.t_start.size() * sizeof(float));
        std::memcpy(t_end, b.t_end.data(), b.t_end.size() * sizeof(float));
        return SF_OK;
    });
}

int sfref_raycast(sfref_volume* v, const double pose[12], const sf_intrinsics* intr, float* depth,
                  float* normals_xyz, int32_t, sf_raycast_stats* stats, void*) {
    return guarded([&]() -> int {
        const RaycastResult r = raycast(*v->grid, to_pose(pose), to_intr(intr));
        std::memcpy(depth, r.depth.depth.data(), r.depth.depth.size() * sizeof(float));
        from_normals(r.normals, normals_xyz);
        if (stats) {
            stats->sample_steps = r.stats.sample_steps;
            stats->hit_pixels = r.stats.hit_pixels;
            stats->rays_with_bounds = r.stats.rays_with_bounds;
        }
        return SF_OK;
    });
}

int sfref_compute_normals(const sf_frame* frame, double sigma0, double spatial_scale, float* normals_xyz,
                          int32_t, void*) {
    return guarded([&]() -> int {
        NormalOptions o;
        o.sigma0 = sigma0;
        o.spatial_scale = spatial_scale;
        from_normals(compute_normals(to_frame(frame), o), normals_xyz);
        return SF_OK;
    });
}

int sfref_icp(const sf_frame* source, const float* source_normals, const sf_frame* target,
              const float* target_normals, const double initial[12], const sf_match_params* params,
              sf_icp_result* result, void*) {
    return guarded([&]() -> int {
        const DepthFrame s = to_frame(source);
        const DepthFrame t = to_frame(target);
        const int w = t.intrinsics.width, h = t.intrinsics.height;
        const NormalMap tn = to_normals(target_normals, w, h);
        IcpResult r;
        if (source_normals)
            r = icp(s, to_normals(source_normals, w, h), t, tn, to_pose(initial), to_match(params));
        else
            r = icp(s, t, tn, to_pose(initial), to_match(params));
        from_icp(r, result);
        return SF_OK;
    });
}

// Per-voxel measurement (fusion.cpp:81-173) for KAT-style probes.
int sfref_estimate_measurement(const sf_frame* frame, const double pose[12], const double voxel_center[3],
                               const sf_fusion_params* params, int32_t* is_chi, double* tsdf,
                               double* variance, double* weight) {
    return guarded([&]() -> int {
        const DepthFrame f = to_frame(frame);
        FusionParams p = to_fusion(params);
        const MeasurementSample s = estimate_measurement(
            f, to_pose(pose), Eigen::Vector3d(voxel_center[0], voxel_center[1], voxel_center[2]), p);
        *is_chi = s.tsdf ? 0 : 1;
        *tsdf = s.tsdf ? *s.tsdf : 0.0;
        *variance = s.variance;
        *weight = s.weight;
        return SF_OK;
    });
}

int sfref_render_synthetic_depth(const sf_scene* scene, const double pose[12], const sf_intrinsics* intr,
                                 double noise_sigma0, uint64_t noise_seed, int32_t max_steps,
                                 double tolerance_scale, double domain_size, float* depth,
                                 float* sigma) {
    return guarded([&]() -> int {
        NoiseModel noise{noise_sigma0, noise_seed};
        SphereTraceOptions trace{max_steps, tolerance_scale, domain_size};
        const DepthFrame f =
            render_synthetic_depth(to_scene(scene), to_pose(pose), to_intr(intr), noise, trace);
        std::memcpy(depth, f.depth.data(), f.depth.size() * sizeof(float));
        if (sigma) {
            if (f.has_sigma()) std::memcpy(sigma, f.sigma.data(), f.sigma.size() * sizeof(float));
            else std::memset(sigma, 0, f.depth.size() * sizeof(float));
        }
        return SF_OK;
    });
}

int sfref_orbit_trajectory(const double target[3], double radius, int32_t frames, const double axis[3],
                           double start_angle, double arc, double* poses_out) {
    return guarded([&]() -> int {
        const auto poses = orbit_trajectory(Eigen::Vector3d(target[0], target[1], target[2]), radius, frames,
                                            Eigen::Vector3d(axis[0], axis[1], axis[2]), start_angle, arc);
        for (std::size_t i = 0; i < poses.size(); ++i) from_pose(poses[i], poses_out + 12 * i);
        return SF_OK;
    });
}

int sfref_compose(const double a[12], const double b[12], double out[12]) {
    from_pose(compose(to_pose(a), to_pose(b)), out);
    return SF_OK;
}

int sfref_invert(const double a[12], double out[12]) {
    from_pose(invert(to_pose(a)), out);
    return SF_OK;
}

int sfref_apply_motion(const double pose[12], const double r[3], const double t[3], double out[12]) {
    SmallMotion m;
    m.r = Eigen::Vector3d(r[0], r[1], r[2]);
    m.t = Eigen::Vector3d(t[0], t[1], t[2]);
    from_pose(apply_motion(to_pose(pose), m), out);
    return SF_OK;
}

// One run() frame body (pipeline.cpp:250-287) without acquisition, for the fused-frame
// reference timing and tracking parity: track = raycast(current) -> icp -> compose -> fuse.
// mode 0: track; 1: fuse at current_pose; 2: track with external initial delta (icp_with_hook).
int sfref_pipeline_frame(sfref_volume* v, const sf_frame* captured, const sf_intrinsics* camera,
                         const sf_fusion_params* fparams, const sf_match_params* mparams, int32_t mode,
                         const double* external, double current_pose[12], sf_fusion_stats* stats,
                         int32_t* iterations, uint64_t* matches) {
    return guarded([&]() -> int {
        const DepthFrame f = to_frame(captured);
        Pose current = to_pose(current_pose);
        *iterations = 0;
        *matches = 0;
        if (mode == 0 || mode == 2) {
            const RaycastResult rendered = raycast(*v->grid, current, to_intr(camera));
            std::optional<Pose> ext;
            if (mode == 2) ext = to_pose(external);
            const Pose initial_pose = initial_transform_hook(current, ext);
            const Pose initial_delta = compose(invert(current), initial_pose);
            const IcpResult r = icp(f, rendered.depth, rendered.normals, initial_delta, to_match(mparams));
            *iterations = r.iterations;
            *matches = r.matches;
            current = compose(current, r.delta);
            from_pose(current, current_pose);
        }
        const FusionStats s = fuse_frame(*v->grid, f, current, to_fusion(fparams));
        if (stats) {
            stats->voxels_updated = s.voxels_updated;
            stats->blocks_allocated_now = s.blocks_allocated_now;
            stats->blocks_total = s.blocks_total;
            stats->memory_bytes = s.memory_bytes;
        }
        return SF_OK;
    });
}

int sfref_marching_cubes(sfref_volume* v, const double region_pose[12], const sf_intrinsics* region_intrinsics,
                         uint64_t batch_memory_budget, sfref_mesh** out, void*) {
    return guarded([&]() -> int {
        MarchingCubesOptions o;
        if (region_pose) o.region = FrustumRegion{to_pose(region_pose), to_intr(region_intrinsics)};
        if (batch_memory_budget) o.batch_memory_budget = batch_memory_budget;
        auto m = std::make_unique<sfref_mesh>();
        m->mesh = marching_cubes(*v->grid, o);
        *out = m.release();
        return SF_OK;
    });
}

int sfref_mesh_counts(sfref_mesh* m, uint64_t* vertices, uint64_t* triangles) {
    if (vertices) *vertices = m->mesh.vertices.size();
    if (triangles) *triangles = m->mesh.triangles.size();
    return SF_OK;
}

int sfref_mesh_read(sfref_mesh* m, float* vertices_xyz, float* normals_xyz, uint32_t* triangles, int32_t, void*) {
    for (size_t i = 0; i < m->mesh.vertices.size(); ++i)
        for (int k = 0; k < 3; ++k) {
            if (vertices_xyz) vertices_xyz[3 * i + k] = m->mesh.vertices[i][k];
            if (normals_xyz) normals_xyz[3 * i + k] = m->mesh.normals[i][k];
        }
    for (size_t i = 0; i < m->mesh.triangles.size(); ++i)
        for (int k = 0; k < 3; ++k)
            if (triangles) triangles[3 * i + k] = m->mesh.triangles[i][k];
    return SF_OK;
}

int sfref_mesh_destroy(sfref_mesh* m) {
    delete m;
    return SF_OK;
}

int sfref_dfrm_write(const char* path, const sf_frame* frame) {
    return guarded([&]() -> int {
        write_dfrm(to_frame(frame), path);
        return SF_OK;
    });
}

int sfref_dfrm_read(const char* path, sf_intrinsics* intrinsics, float* depth, float* sigma, int32_t* has_sigma,
                    int32_t) {
    return guarded([&]() -> int {
        const DepthFrame f = read_dfrm(path);
        intrinsics->width = f.intrinsics.width;
        intrinsics->height = f.intrinsics.height;
        intrinsics->fx = f.intrinsics.fx;
        intrinsics->fy = f.intrinsics.fy;
        intrinsics->cx = f.intrinsics.cx;
        intrinsics->cy = f.intrinsics.cy;
        intrinsics->near_plane = f.intrinsics.near_plane;
        intrinsics->far_plane = f.intrinsics.far_plane;
        if (!depth) return SF_OK;
        std::memcpy(depth, f.depth.data(), f.depth.size() * sizeof(float));
        if (has_sigma) *has_sigma = f.has_sigma() ? 1 : 0;
        if (f.has_sigma() && sigma) std::memcpy(sigma, f.sigma.data(), f.sigma.size() * sizeof(float));
        return SF_OK;
    });
}

// write_trajectory / read_trajectory (frame_io.cpp:81-126), same conventions as sf_trajectory_*
int sfref_trajectory_write(const char* path, const int32_t* frame_index, const double* poses12, uint64_t count) {
    return guarded([&]() -> int {
        std::vector<TrajectoryEntry> t(count);
        for (uint64_t i = 0; i < count; ++i) {
            t[i].frame_index = frame_index[i];
            t[i].pose = to_pose(poses12 + 12 * i);
        }
        write_trajectory(t, path);
        return SF_OK;
    });
}

int sfref_trajectory_read(const char* path, int32_t* frame_index, double* poses12, uint64_t* count) {
    return guarded([&]() -> int {
        const std::vector<TrajectoryEntry> t = read_trajectory(path);
        if (frame_index && poses12) {
            if (t.size() > *count) return SF_OUT_OF_RANGE;
            for (size_t i = 0; i < t.size(); ++i) {
                frame_index[i] = t[i].frame_index;
                from_pose(t[i].pose, poses12 + 12 * i);
            }
        }
        *count = t.size();
        return SF_OK;
    });
}

}  // extern "C"

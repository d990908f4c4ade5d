// sparsefusion_adapter.cpp — the reference library's hot-path entry points, namespace
// `sparsefusion`, implemented over the C-ABI of include/sf_gpu.h (libsf_gpu.so, sm_100a).
//
// Drop-in contract: a program written against the reference headers
// (/root/reference/proj/include/sparsefusion/*.hpp, unchanged) links this translation unit
// ahead of the reference's own objects; the definitions below replace the reference's
//   fuse_frame, select_update_blocks             (fusion.hpp:71-72, 102-103)
//   compute_ray_bounds, raycast (both overloads) (render.hpp:38-39, 61-63)
//   icp (both overloads)                         (registration.hpp:120-124)
//   compute_normals                              (camera.hpp:90)
//   marching_cubes                               (marching_cubes.hpp:42)
// and every other symbol (grid storage, scalar helpers, scene, I/O, pipeline) stays the
// reference's. The reference's SparseTsdfGrid keeps its host storage (the header fixes its
// layout: offset table, payload pool, free list as std::vector members), so each call mirrors
// the grid into a device volume (sf_volume_import_state: table, pool, free-list stack, and the
// float shadow when enabled), runs the CUDA path, and — for fuse_frame — writes the device
// state back (also on PoolExhausted, whose partial state the reference defines,
// fusion.cpp:369). Errors come back as the reference's exception types and messages.
//
// Built by `make conformance` only where the reference headers exist; the reference's test
// suites (proj/tests/*.cpp, unmodified) are linked against it (tests/test_gpu_conformance.py).
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "sparsefusion/camera.hpp"
#include "sparsefusion/fusion.hpp"
#include "sparsefusion/grid.hpp"
#include "sparsefusion/marching_cubes.hpp"
#include "sparsefusion/registration.hpp"
#include "sparsefusion/render.hpp"
#include "sf_gpu.h"

namespace {

using sparsefusion::SparseTsdfGrid;

// Read/write access to SparseTsdfGrid's private storage without touching the reference
// header: a pointer-to-member named in an explicit template instantiation is exempt from
// access checking ([temp.explicit]/14), and the friend function hands it out.
template <typename Tag, typename Tag::type M>
struct Expose {
    friend typename Tag::type member(Tag) { return M; }
};
struct TableTag {
    using type = std::vector<std::int32_t> SparseTsdfGrid::*;
    friend type member(TableTag);
};
struct PoolTag {
    using type = std::vector<sparsefusion::VoxelPayload> SparseTsdfGrid::*;
    friend type member(PoolTag);
};
struct FreeTag {
    using type = std::vector<std::int32_t> SparseTsdfGrid::*;
    friend type member(FreeTag);
};
struct CountTag {
    using type = std::size_t SparseTsdfGrid::*;
    friend type member(CountTag);
};
template struct Expose<TableTag, &SparseTsdfGrid::offset_table_>;
template struct Expose<PoolTag, &SparseTsdfGrid::payload_pool_>;
template struct Expose<FreeTag, &SparseTsdfGrid::free_list_>;
template struct Expose<CountTag, &SparseTsdfGrid::allocated_count_>;

static_assert(sizeof(sparsefusion::VoxelPayload) == 2, "payload cell = {int8 tsdf, uint8 aux}");

// sf_status -> the reference's exception types (grid.cpp:14-17,83,90-92,139; registration.cpp:202-204)
[[noreturn]] void raise(int status) {
    const std::string msg = sf_last_error();
    switch (status) {
        case SF_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case SF_OUT_OF_RANGE: throw std::out_of_range(msg);
        case SF_LOGIC_ERROR: throw std::logic_error(msg);
        case SF_POOL_EXHAUSTED: throw sparsefusion::PoolExhausted(msg);
        case SF_TRACKING_LOST: throw sparsefusion::TrackingLost(msg);
        default: throw std::runtime_error(msg.empty() ? "sf_gpu: status " + std::to_string(status) : msg);
    }
}
void check(int status) {
    if (status != SF_OK) raise(status);
}

sf_intrinsics to_c(const sparsefusion::Intrinsics& i) {
    return sf_intrinsics{i.width, i.height, i.fx, i.fy, i.cx, i.cy, i.near_plane, i.far_plane};
}
sf_frame to_c(const sparsefusion::DepthFrame& f) {
    sf_frame c{};
    c.intrinsics = to_c(f.intrinsics);
    c.depth = f.depth.data();
    c.sigma = f.has_sigma() ? f.sigma.data() : nullptr;
    c.on_device = 0;
    return c;
}
void to_c(const sparsefusion::Pose& p, double out[12]) {
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) out[r * 3 + c] = p.rotation(r, c);
    for (int i = 0; i < 3; ++i) out[9 + i] = p.translation[i];
}
sparsefusion::Pose from_c(const double p[12]) {
    sparsefusion::Pose o;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) o.rotation(r, c) = p[r * 3 + c];
    o.translation = Eigen::Vector3d(p[9], p[10], p[11]);
    return o;
}
sf_match_params to_c(const sparsefusion::MatchParams& m) {
    sf_match_params c{};
    c.max_distance = m.max_distance;
    c.max_normal_angle = m.max_normal_angle;
    c.max_iterations = m.max_iterations;
    c.convergence_epsilon = m.convergence_epsilon;
    c.eigen_threshold = m.eigen_threshold;
    c.shrink_floor = m.shrink_floor;
    c.normal_sigma0 = m.normal_options.sigma0;
    c.normal_spatial_scale = m.normal_options.spatial_scale;
    c.reduction = 0;  // tree-ordered sums (pose within ~1e-15 of the reference per call)
    return c;
}
sparsefusion::NormalMap normals_from(const std::vector<float>& xyz, int w, int h) {
    sparsefusion::NormalMap n(w, h);
    for (std::size_t i = 0; i < n.normals.size(); ++i)
        n.normals[i] = Eigen::Vector3f(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
    return n;
}
std::vector<float> normals_to(const sparsefusion::NormalMap& n) {
    std::vector<float> out(3 * n.normals.size());
    for (std::size_t i = 0; i < n.normals.size(); ++i)
        for (int k = 0; k < 3; ++k) out[3 * i + k] = n.normals[i][k];
    return out;
}

// The grid mirrored into a device volume for the duration of one call.
class DeviceGrid {
public:
    DeviceGrid(const SparseTsdfGrid& g, bool shadow) : grid_(g), shadow_(shadow && g.has_shadow()) {
        const sparsefusion::GridConfig& gc = g.config();
        sf_grid_config c{};
        c.blocks_per_axis = gc.blocks_per_axis;
        c.voxels_per_block_axis = gc.voxels_per_block_axis;
        for (int i = 0; i < 3; ++i) c.box_origin[i] = gc.box_origin[i];
        c.box_side = gc.box_side;
        c.truncation = gc.truncation;
        const sparsefusion::AuxQuantization& aq = g.aux_quantization();
        sf_aux_quant a{aq.mode == sparsefusion::AuxMode::Weight ? 0 : 1, aq.w_max, aq.p_min, aq.p_max};
        check(sf_volume_create(&c, g.pool_capacity(), &a, 0, &v_));
        const auto& table = g.*member(TableTag{});
        const auto& pool = g.*member(PoolTag{});
        const auto& free_list = g.*member(FreeTag{});
        check(sf_volume_import_state(v_, table.data(), reinterpret_cast<const std::uint16_t*>(pool.data()),
                                     g.pool_capacity(), free_list.data(), free_list.size()));
        if (shadow_) {
            check(sf_volume_enable_float_payload(v_));
            std::vector<float> f(2 * g.voxels_per_block() * g.pool_capacity());
            for_each_shadow_voxel([&](std::size_t slot_voxel, std::size_t dense) {
                f[2 * slot_voxel] = g.shadow().tsdf[dense];
                f[2 * slot_voxel + 1] = g.shadow().aux[dense];
            });
            check(sf_volume_write_float_payload(v_, 0, g.pool_capacity(), f.data()));
        }
    }
    ~DeviceGrid() {
        if (v_) sf_volume_destroy(v_);
    }
    DeviceGrid(const DeviceGrid&) = delete;
    DeviceGrid& operator=(const DeviceGrid&) = delete;
    sf_volume_t get() const { return v_; }

    // device state -> the host grid (after fuse_frame)
    void write_back(SparseTsdfGrid& g) {
        auto& table = g.*member(TableTag{});
        auto& pool = g.*member(PoolTag{});
        auto& free_list = g.*member(FreeTag{});
        check(sf_volume_read_table(v_, table.data()));
        check(sf_volume_read_payload(v_, 0, g.pool_capacity(), reinterpret_cast<std::uint16_t*>(pool.data())));
        std::uint64_t n = 0;
        check(sf_volume_read_free_list(v_, nullptr, &n));
        free_list.resize(n);
        check(sf_volume_read_free_list(v_, free_list.data(), &n));
        sf_volume_info info{};
        check(sf_volume_get_info(v_, &info));
        g.*member(CountTag{}) = info.allocated_count;
        if (shadow_) {
            std::vector<float> f(2 * g.voxels_per_block() * g.pool_capacity());
            check(sf_volume_read_float_payload(v_, 0, g.pool_capacity(), f.data()));
            for_each_shadow_voxel([&](std::size_t slot_voxel, std::size_t dense) {
                g.shadow().tsdf[dense] = f[2 * slot_voxel];
                g.shadow().aux[dense] = f[2 * slot_voxel + 1];
            });
        }
    }

private:
    // (slot-major voxel index, dense shadow index) of every voxel of every allocated block
    template <typename F>
    void for_each_shadow_voxel(F&& f) const {
        const int m = grid_.config().voxels_per_block_axis;
        for (const Eigen::Vector3i& bc : grid_.allocated_blocks()) {
            const std::int32_t slot = grid_.block_slot(bc);
            for (int z = 0; z < m; ++z)
                for (int y = 0; y < m; ++y)
                    for (int x = 0; x < m; ++x) {
                        const Eigen::Vector3i l(x, y, z);
                        f(static_cast<std::size_t>(slot) * grid_.voxels_per_block() + grid_.local_index(l),
                          grid_.shadow().index(bc * m + l));
                    }
        }
    }
    const SparseTsdfGrid& grid_;
    bool shadow_;
    sf_volume_t v_ = nullptr;
};

}  // namespace

namespace sparsefusion {

// fuse_frame (fusion.hpp:102-103; fusion.cpp:274-376) -> sf_integrate
FusionStats fuse_frame(SparseTsdfGrid& grid, const DepthFrame& frame, const Pose& pose, const FusionParams& params) {
    params.validate();
    if (params.mode == FusionMode::Kalman && grid.aux_quantization().mode != AuxMode::Variance)
        throw std::invalid_argument("fusion: Kalman mode needs a variance-mode grid");
    if (params.mode != FusionMode::Kalman && grid.aux_quantization().mode != AuxMode::Weight)
        throw std::invalid_argument("fusion: weight-mode grid required for this fusion mode");
    DeviceGrid d(grid, true);
    const sf_frame f = to_c(frame);
    double p12[12];
    to_c(pose, p12);
    sf_fusion_params fp{};
    fp.mode = params.mode == FusionMode::Simple ? 0 : params.mode == FusionMode::Weighted ? 1 : 2;
    fp.w_fixed = params.w_fixed;
    fp.w_max = params.w_max;
    fp.process_variance = params.process_variance;
    fp.sigma0 = params.sigma0;
    fp.delta = params.delta;
    fp.refinement_steps = params.refinement_steps;
    fp.edge_downweight = params.edge_downweight ? 1 : 0;
    fp.min_variance = params.min_variance;
    sf_fusion_stats st{};
    const int rc = sf_integrate(d.get(), &f, p12, &fp, &st, nullptr);
    if (rc == SF_OK || rc == SF_POOL_EXHAUSTED) d.write_back(grid);  // partial state on exhaustion
    check(rc);
    FusionStats out;
    out.voxels_updated = st.voxels_updated;
    out.blocks_allocated_now = st.blocks_allocated_now;
    out.blocks_total = st.blocks_total;
    out.memory_bytes = st.memory_bytes;
    return out;
}

// select_update_blocks (fusion.hpp:71-72; fusion.cpp:187-235) -> sf_select_update_blocks
UpdateLists select_update_blocks(const SparseTsdfGrid& grid, const DepthFrame& frame, const Pose& pose) {
    DeviceGrid d(grid, false);
    const sf_frame f = to_c(frame);
    double p12[12];
    to_c(pose, p12);
    std::uint64_t na = 3ull * frame.depth.size() + 16, nu = grid.pool_capacity() + 16;
    std::vector<std::int32_t> a(3 * na), u(3 * nu);
    check(sf_select_update_blocks(d.get(), &f, p12, a.data(), &na, u.data(), &nu, nullptr));
    UpdateLists out;
    for (std::uint64_t i = 0; i < na; ++i) out.allocate.emplace_back(a[3 * i], a[3 * i + 1], a[3 * i + 2]);
    for (std::uint64_t i = 0; i < nu; ++i) out.update.emplace_back(u[3 * i], u[3 * i + 1], u[3 * i + 2]);
    return out;
}

// compute_ray_bounds (render.hpp:38-39; render.cpp:65-153) -> sf_ray_bounds
RayBounds compute_ray_bounds(const SparseTsdfGrid& grid, const Pose& pose, const Intrinsics& intrinsics) {
    intrinsics.validate();
    DeviceGrid d(grid, false);
    double p12[12];
    to_c(pose, p12);
    const sf_intrinsics ic = to_c(intrinsics);
    RayBounds b(intrinsics.width, intrinsics.height);
    check(sf_ray_bounds(d.get(), p12, &ic, b.t_start.data(), b.t_end.data(), 0, nullptr));
    return b;
}

namespace {
RaycastResult raycast_impl(const SparseTsdfGrid& grid, const Pose& pose, const Intrinsics& intrinsics,
                           const RayBounds* bounds) {
    intrinsics.validate();
    DeviceGrid d(grid, false);
    double p12[12];
    to_c(pose, p12);
    const sf_intrinsics ic = to_c(intrinsics);
    RaycastResult r{DepthFrame(intrinsics), NormalMap(intrinsics.width, intrinsics.height), {}};
    std::vector<float> n(3 * r.depth.depth.size());
    sf_raycast_stats st{};
    if (bounds) {
        if (bounds->width != intrinsics.width || bounds->height != intrinsics.height)
            throw std::invalid_argument("raycast: bounds size does not match the intrinsics");
        check(sf_raycast_with_bounds(d.get(), p12, &ic, bounds->t_start.data(), bounds->t_end.data(),
                                     r.depth.depth.data(), n.data(), 0, &st, nullptr));
    } else {
        check(sf_raycast(d.get(), p12, &ic, r.depth.depth.data(), n.data(), 0, &st, nullptr));
    }
    r.normals = normals_from(n, intrinsics.width, intrinsics.height);
    r.stats.sample_steps = st.sample_steps;
    r.stats.hit_pixels = st.hit_pixels;
    r.stats.rays_with_bounds = st.rays_with_bounds;
    return r;
}
}  // namespace

// raycast (render.hpp:61-63; render.cpp:155-250) -> sf_raycast / sf_raycast_with_bounds
RaycastResult raycast(const SparseTsdfGrid& grid, const Pose& pose, const Intrinsics& intrinsics,
                      const RayBounds& bounds) {
    return raycast_impl(grid, pose, intrinsics, &bounds);
}
RaycastResult raycast(const SparseTsdfGrid& grid, const Pose& pose, const Intrinsics& intrinsics) {
    return raycast_impl(grid, pose, intrinsics, nullptr);
}

// compute_normals (camera.hpp:90; camera.cpp:44-76) -> sf_compute_normals
NormalMap compute_normals(const DepthFrame& frame, const NormalOptions& opts) {
    const sf_frame f = to_c(frame);
    std::vector<float> n(3 * frame.depth.size());
    check(sf_compute_normals(&f, opts.sigma0, opts.spatial_scale, n.data(), 0, nullptr));
    return normals_from(n, frame.intrinsics.width, frame.intrinsics.height);
}

namespace {
IcpResult icp_impl(const DepthFrame& source, const NormalMap* source_normals, const DepthFrame& target,
                   const NormalMap& target_normals, const Pose& initial, const MatchParams& params) {
    if (source.intrinsics.width != target.intrinsics.width || source.intrinsics.height != target.intrinsics.height)
        throw std::invalid_argument("match: frames must share intrinsics");
    const sf_frame s = to_c(source), t = to_c(target);
    const std::vector<float> tn = normals_to(target_normals);
    std::vector<float> sn;
    if (source_normals) sn = normals_to(*source_normals);
    double p12[12];
    to_c(initial, p12);
    const sf_match_params mp = to_c(params);
    sf_icp_result r{};
    check(sf_icp(&s, source_normals ? sn.data() : nullptr, &t, tn.data(), p12, &mp, &r, nullptr));
    IcpResult out;
    out.delta = from_c(r.delta);
    out.iterations = r.iterations;
    out.matches = r.matches;
    GatedSolution& g = out.solution;
    g.motion.r = Eigen::Vector3d(r.motion_r[0], r.motion_r[1], r.motion_r[2]);
    g.motion.t = Eigen::Vector3d(r.motion_t[0], r.motion_t[1], r.motion_t[2]);
    for (int i = 0; i < 6; ++i) {
        g.eigenvalues[i] = r.eigenvalues[i];
        g.gated_mask[i] = r.gated_mask[i] != 0;
        for (int k = 0; k < 6; ++k) g.eigenvectors(k, i) = r.eigenvectors[i * 6 + k];
    }
    g.residual_rms = r.residual_rms;
    g.shrunk_motion_norm = r.shrunk_motion_norm;
    g.pair_count = r.pair_count;
    return out;
}
}  // namespace

// icp (registration.hpp:120-124; registration.cpp:195-220) -> sf_icp
IcpResult icp(const DepthFrame& source, const NormalMap& source_normals, const DepthFrame& target,
              const NormalMap& target_normals, const Pose& initial, const MatchParams& params) {
    return icp_impl(source, &source_normals, target, target_normals, initial, params);
}
IcpResult icp(const DepthFrame& source, const DepthFrame& target, const NormalMap& target_normals,
              const Pose& initial, const MatchParams& params) {
    return icp_impl(source, nullptr, target, target_normals, initial, params);
}

// marching_cubes (marching_cubes.hpp:42; marching_cubes.cpp:74-196) -> sf_marching_cubes
Mesh marching_cubes(const SparseTsdfGrid& grid, const MarchingCubesOptions& options) {
    DeviceGrid d(grid, false);
    double p12[12];
    sf_intrinsics ic{};
    if (options.region) {
        to_c(options.region->pose, p12);
        ic = to_c(options.region->intrinsics);
    }
    sf_mesh_t m = nullptr;
    check(sf_marching_cubes(d.get(), options.region ? p12 : nullptr, options.region ? &ic : nullptr,
                            options.batch_memory_budget, &m, nullptr));
    std::uint64_t nv = 0, nt = 0;
    const int rc = sf_mesh_counts(m, &nv, &nt);
    Mesh out;
    std::vector<float> v(3 * nv), n(3 * nv);
    std::vector<std::uint32_t> t(3 * nt);
    const int rc2 = rc == SF_OK ? sf_mesh_read(m, v.data(), n.data(), t.data(), 0, nullptr) : rc;
    sf_mesh_destroy(m);
    check(rc2);
    out.vertices.resize(nv);
    out.normals.resize(nv);
    out.triangles.resize(nt);
    for (std::uint64_t i = 0; i < nv; ++i) {
        out.vertices[i] = Eigen::Vector3f(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
        out.normals[i] = Eigen::Vector3f(n[3 * i], n[3 * i + 1], n[3 * i + 2]);
    }
    for (std::uint64_t i = 0; i < nt; ++i) out.triangles[i] = {t[3 * i], t[3 * i + 1], t[3 * i + 2]};
    return out;
}

}  // namespace sparsefusion

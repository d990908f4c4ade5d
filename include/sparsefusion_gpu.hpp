// sparsefusion_gpu.hpp — C++17 host API over the C-ABI (include/sf_gpu.h).
//
// Mirrors the reference's public headers for the hot path (proj/include/sparsefusion/
// grid.hpp, fusion.hpp, render.hpp, registration.hpp, pose.hpp, camera.hpp): same type and
// function names, argument meaning and exception types, without the Eigen dependency
// (3-vectors are std::array<double, 3>, rotations row-major std::array<double, 9>). A
// reference call site switches by changing the namespace (sparsefusion -> sparsefusion_gpu)
// and linking libsf_gpu.so; see INTEGRATION.md.
#pragma once

#include <array>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sf_gpu.h"

namespace sparsefusion_gpu {

using Vec3 = std::array<double, 3>;
using Vec3i = std::array<int, 3>;

// ---- exceptions (grid.hpp:24-26, registration.hpp:18-20) ----------------------------
struct PoolExhausted : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct TrackingLost : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int status) {
    if (status == SF_OK) return;
    const std::string msg = sf_last_error();
    switch (status) {
        case SF_POOL_EXHAUSTED: throw PoolExhausted(msg);
        case SF_TRACKING_LOST: throw TrackingLost(msg);
        case SF_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case SF_OUT_OF_RANGE: throw std::out_of_range(msg);
        case SF_LOGIC_ERROR: throw std::logic_error(msg);
        case SF_UNSUPPORTED: throw std::logic_error("unsupported on the device path: " + msg);
        case SF_CUDA_ERROR: throw CudaError(msg);
        default: throw std::runtime_error(msg);
    }
}

// ---- geometry (pose.hpp:9-42, camera.hpp:9-24) --------------------------------------
struct Pose {
    std::array<double, 9> rotation{1, 0, 0, 0, 1, 0, 0, 0, 1};  // row-major
    Vec3 translation{0, 0, 0};
    static Pose identity() { return {}; }
    std::array<double, 12> packed() const {
        std::array<double, 12> p{};
        for (int i = 0; i < 9; ++i) p[i] = rotation[i];
        for (int i = 0; i < 3; ++i) p[9 + i] = translation[i];
        return p;
    }
    static Pose unpack(const double* p) {
        Pose o;
        for (int i = 0; i < 9; ++i) o.rotation[i] = p[i];
        for (int i = 0; i < 3; ++i) o.translation[i] = p[9 + i];
        return o;
    }
    // x_scene = R x_camera + t, left-to-right sums (the oracle's evaluation order)
    Vec3 apply(const Vec3& x) const {
        Vec3 r;
        for (int i = 0; i < 3; ++i)
            r[i] = ((rotation[i * 3] * x[0] + rotation[i * 3 + 1] * x[1]) + rotation[i * 3 + 2] * x[2]) + translation[i];
        return r;
    }
};

// compose / invert (pose.cpp:6-18), bit-identical to the reference.
inline Pose compose(const Pose& a, const Pose& b) {
    Pose o;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            o.rotation[i * 3 + j] = (a.rotation[i * 3] * b.rotation[j] + a.rotation[i * 3 + 1] * b.rotation[3 + j]) +
                                    a.rotation[i * 3 + 2] * b.rotation[6 + j];
    for (int i = 0; i < 3; ++i)
        o.translation[i] = ((a.rotation[i * 3] * b.translation[0] + a.rotation[i * 3 + 1] * b.translation[1]) +
                            a.rotation[i * 3 + 2] * b.translation[2]) +
                           a.translation[i];
    return o;
}
inline Pose invert(const Pose& a) {
    Pose o;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) o.rotation[j * 3 + i] = a.rotation[i * 3 + j];
    for (int i = 0; i < 3; ++i)
        o.translation[i] = -((o.rotation[i * 3] * a.translation[0] + o.rotation[i * 3 + 1] * a.translation[1]) +
                             o.rotation[i * 3 + 2] * a.translation[2]);
    return o;
}

struct Intrinsics {
    int width = 0, height = 0;
    double fx = 0, fy = 0, cx = 0, cy = 0;
    double near_plane = 0.1, far_plane = 10.0;
    static Intrinsics simple(int w, int h, double f, double near_plane = 0.1, double far_plane = 10.0) {
        Intrinsics i;  // camera.cpp:16-29
        i.width = w;
        i.height = h;
        i.fx = i.fy = f;
        i.cx = 0.5 * (w - 1);
        i.cy = 0.5 * (h - 1);
        i.near_plane = near_plane;
        i.far_plane = far_plane;
        return i;
    }
    sf_intrinsics c() const { return {width, height, fx, fy, cx, cy, near_plane, far_plane}; }
};

// DepthFrame / NormalMap (camera.hpp:45-78): host storage; device frames go through the
// C-ABI directly (sf_frame.on_device = 1).
struct DepthFrame {
    Intrinsics intrinsics;
    std::vector<float> depth, sigma;
    DepthFrame() = default;
    explicit DepthFrame(const Intrinsics& i) : intrinsics(i), depth(static_cast<size_t>(i.width) * i.height, 0.f) {}
    float& at(int u, int v) { return depth[static_cast<size_t>(v) * intrinsics.width + u]; }
    float at(int u, int v) const { return depth[static_cast<size_t>(v) * intrinsics.width + u]; }
    bool has_sigma() const { return !sigma.empty(); }
    sf_frame c() const { return {intrinsics.c(), depth.data(), has_sigma() ? sigma.data() : nullptr, 0}; }
};
struct NormalMap {
    int width = 0, height = 0;
    std::vector<float> xyz;  // 3 floats per pixel, zero = invalid
    NormalMap() = default;
    NormalMap(int w, int h) : width(w), height(h), xyz(3 * static_cast<size_t>(w) * h, 0.f) {}
};

// ---- grid (grid.hpp:28-193) -----------------------------------------------------------
struct GridConfig {
    int blocks_per_axis = 16;
    int voxels_per_block_axis = 8;
    Vec3 box_origin{0, 0, 0};
    double box_side = 1.0;
    double truncation = 0.0;
    int voxels_per_axis() const { return blocks_per_axis * voxels_per_block_axis; }
    double voxel_size() const { return box_side / voxels_per_axis(); }
    double delta() const { return truncation > 0.0 ? truncation : 4.0 * voxel_size(); }
    sf_grid_config c() const {
        return {blocks_per_axis, voxels_per_block_axis, {box_origin[0], box_origin[1], box_origin[2]}, box_side,
                truncation};
    }
};
enum class AuxMode { Weight = 0, Variance = 1 };
struct AuxQuantization {
    AuxMode mode = AuxMode::Weight;
    double w_max = 20.0, p_min = 1e-8, p_max = 1e-2;
    sf_aux_quant c() const { return {static_cast<int32_t>(mode), w_max, p_min, p_max}; }
};
struct VoxelData {
    double tsdf = 0.0, aux = 0.0;
};

class SparseTsdfGrid {
public:
    static constexpr int32_t kEmpty = -1;
    explicit SparseTsdfGrid(const GridConfig& config, std::size_t pool_capacity = 0, const AuxQuantization& aux = {},
                            int device = 0) {
        const sf_grid_config c = config.c();
        const sf_aux_quant a = aux.c();
        check(sf_volume_create(&c, pool_capacity, &a, device, &h_));
    }
    ~SparseTsdfGrid() {
        if (h_) sf_volume_destroy(h_);
    }
    SparseTsdfGrid(const SparseTsdfGrid&) = delete;
    SparseTsdfGrid& operator=(const SparseTsdfGrid&) = delete;
    SparseTsdfGrid(SparseTsdfGrid&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}

    sf_volume_info info() const {
        sf_volume_info i;
        check(sf_volume_get_info(h_, &i));
        return i;
    }
    double delta() const { return info().delta; }
    double voxel_size() const { return info().voxel_size; }
    std::size_t pool_capacity() const { return info().pool_capacity; }
    std::size_t allocated_count() const { return info().allocated_count; }
    std::uint64_t memory_bytes() const { return info().memory_bytes; }

    int32_t block_slot(const Vec3i& bc) const {
        int32_t s;
        check(sf_volume_block_slot(h_, bc.data(), &s));
        return s;
    }
    bool is_allocated(const Vec3i& bc) const { return block_slot(bc) != kEmpty; }
    int32_t allocate_block(const Vec3i& bc) {
        int32_t s;
        check(sf_volume_allocate_block(h_, bc.data(), &s));
        return s;
    }
    void free_block(const Vec3i& bc) { check(sf_volume_free_block(h_, bc.data())); }
    std::optional<VoxelData> read_voxel(const Vec3i& vc) const {
        int32_t chi;
        VoxelData d;
        check(sf_volume_read_voxel(h_, vc.data(), &chi, &d.tsdf, &d.aux));
        if (chi) return std::nullopt;
        return d;
    }
    void write_voxel(const Vec3i& vc, std::optional<double> tsdf, double aux) {
        check(sf_volume_write_voxel(h_, vc.data(), tsdf ? 0 : 1, tsdf.value_or(0.0), aux));
    }
    std::vector<int32_t> offset_table() const {
        const auto n = static_cast<size_t>(info().config.blocks_per_axis);
        std::vector<int32_t> t(n * n * n);
        check(sf_volume_read_table(h_, t.data()));
        return t;
    }
    std::vector<uint16_t> payloads() const {
        const sf_volume_info i = info();
        const auto m = static_cast<size_t>(i.config.voxels_per_block_axis);
        std::vector<uint16_t> p(i.pool_capacity * m * m * m);
        check(sf_volume_read_payload(h_, 0, i.pool_capacity, p.data()));
        return p;
    }
    void save_snapshot(const std::string& path) const { check(sf_volume_save_snapshot(h_, path.c_str())); }
    static SparseTsdfGrid load_snapshot(const std::string& path, std::size_t pool_capacity = 0, int device = 0) {
        sf_volume_t h;
        check(sf_volume_load_snapshot(path.c_str(), pool_capacity, device, &h));
        return SparseTsdfGrid(h);
    }
    sf_volume_t handle() const { return h_; }

private:
    explicit SparseTsdfGrid(sf_volume_t h) : h_(h) {}
    sf_volume_t h_ = nullptr;
};

// ---- fusion (fusion.hpp:16-103) --------------------------------------------------------
enum class FusionMode { Simple = 0, Weighted = 1, Kalman = 2 };
struct FusionParams {
    FusionMode mode = FusionMode::Simple;
    double w_fixed = 0.1, w_max = 20.0, process_variance = -1.0, sigma0 = 2.5e-4, delta = 0.0;
    int refinement_steps = 0;
    bool edge_downweight = true;
    double min_variance = 1e-12;
    sf_fusion_params c() const {
        return {static_cast<int32_t>(mode), w_fixed, w_max, process_variance, sigma0, delta, refinement_steps,
                edge_downweight ? 1 : 0, min_variance};
    }
};
struct FusionStats {
    std::size_t voxels_updated = 0, blocks_allocated_now = 0, blocks_total = 0;
    std::uint64_t memory_bytes = 0;
};

inline FusionStats fuse_frame(SparseTsdfGrid& grid, const DepthFrame& frame, const Pose& pose,
                              const FusionParams& params) {
    const sf_frame f = frame.c();
    const auto p = pose.packed();
    const sf_fusion_params fp = params.c();
    sf_fusion_stats s{};
    check(sf_integrate(grid.handle(), &f, p.data(), &fp, &s, nullptr));
    return {s.voxels_updated, s.blocks_allocated_now, s.blocks_total, s.memory_bytes};
}

// ---- render (render.hpp:16-63) ---------------------------------------------------------
struct RaycastStats {
    std::uint64_t sample_steps = 0, hit_pixels = 0, rays_with_bounds = 0;
    double steps_per_hit() const { return hit_pixels ? static_cast<double>(sample_steps) / hit_pixels : 0.0; }
};
struct RaycastResult {
    DepthFrame depth;
    NormalMap normals;
    RaycastStats stats;
};
inline RaycastResult raycast(const SparseTsdfGrid& grid, const Pose& pose, const Intrinsics& intr) {
    RaycastResult r;
    r.depth = DepthFrame(intr);
    r.normals = NormalMap(intr.width, intr.height);
    const auto p = pose.packed();
    const sf_intrinsics ic = intr.c();
    sf_raycast_stats s{};
    check(sf_raycast(grid.handle(), p.data(), &ic, r.depth.depth.data(), r.normals.xyz.data(), 0, &s, nullptr));
    r.stats = {s.sample_steps, s.hit_pixels, s.rays_with_bounds};
    return r;
}

// ---- marching cubes (marching_cubes.hpp:16-44) ----------------------------------------
struct Mesh {
    std::vector<std::array<float, 3>> vertices, normals;
    std::vector<std::array<std::uint32_t, 3>> triangles;
    bool empty() const { return triangles.empty(); }
};
struct FrustumRegion {
    Pose pose;
    Intrinsics intrinsics;
};
struct MarchingCubesOptions {
    std::optional<FrustumRegion> region;
    std::size_t batch_memory_budget = 64ull << 20;
};
inline Mesh marching_cubes(const SparseTsdfGrid& grid, const MarchingCubesOptions& options = {}) {
    sf_mesh_t h = nullptr;
    if (options.region) {
        const auto p = options.region->pose.packed();
        const sf_intrinsics ic = options.region->intrinsics.c();
        check(sf_marching_cubes(grid.handle(), p.data(), &ic, options.batch_memory_budget, &h, nullptr));
    } else {
        check(sf_marching_cubes(grid.handle(), nullptr, nullptr, options.batch_memory_budget, &h, nullptr));
    }
    std::uint64_t nv = 0, nt = 0;
    Mesh m;
    const int st = sf_mesh_counts(h, &nv, &nt);
    if (st == SF_OK) {
        m.vertices.resize(nv);
        m.normals.resize(nv);
        m.triangles.resize(nt);
        const int rd = sf_mesh_read(h, m.vertices.empty() ? nullptr : m.vertices[0].data(),
                                    m.normals.empty() ? nullptr : m.normals[0].data(),
                                    m.triangles.empty() ? nullptr : m.triangles[0].data(), 0, nullptr);
        sf_mesh_destroy(h);
        check(rd);
    } else {
        sf_mesh_destroy(h);
        check(st);
    }
    return m;
}

inline NormalMap compute_normals(const DepthFrame& frame, double sigma0 = 2.5e-4, double spatial_scale = 0.0) {
    NormalMap m(frame.intrinsics.width, frame.intrinsics.height);
    const sf_frame f = frame.c();
    check(sf_compute_normals(&f, sigma0, spatial_scale, m.xyz.data(), 0, nullptr));
    return m;
}

// ---- registration (registration.hpp:22-124) -------------------------------------------
struct MatchParams {
    double max_distance = 0.1, max_normal_angle = 0.5235987755983;
    int max_iterations = 15;
    double convergence_epsilon = 1e-5, eigen_threshold = 0.005, shrink_floor = 1e-6;
    double normal_sigma0 = 2.5e-4, normal_spatial_scale = 0.0;
    static MatchParams for_voxel_size(double v) {
        MatchParams p;  // registration.cpp:9-15
        p.max_distance = 10.0 * v;
        p.shrink_floor = v;
        p.normal_spatial_scale = v;
        return p;
    }
    sf_match_params c() const {
        return {max_distance, max_normal_angle, max_iterations, convergence_epsilon, eigen_threshold, shrink_floor,
                normal_sigma0, normal_spatial_scale};
    }
};
struct IcpResult {
    Pose delta;
    int iterations = 0;
    std::size_t matches = 0;
    sf_icp_result raw{};
};
inline IcpResult icp(const DepthFrame& source, const DepthFrame& target, const NormalMap& target_normals,
                     const Pose& initial, const MatchParams& params) {
    const sf_frame s = source.c(), t = target.c();
    const auto init = initial.packed();
    const sf_match_params mp = params.c();
    IcpResult r;
    check(sf_icp(&s, nullptr, &t, target_normals.xyz.data(), init.data(), &mp, &r.raw, nullptr));
    r.delta = Pose::unpack(r.raw.delta);
    r.iterations = r.raw.iterations;
    r.matches = r.raw.matches;
    return r;
}

// ---- fused frame loop (pipeline.cpp:233-301) -------------------------------------------
class Tracker {
public:
    enum Mode { Track = 0, GroundTruth = 1, TrackWithHook = 2 };
    Tracker(SparseTsdfGrid& grid, const Intrinsics& camera, const FusionParams& fusion, const MatchParams& match,
            const Pose& initial, bool use_graphs = true, bool orthonormalize = false) {
        sf_tracker_config c{fusion.c(), match.c(), camera.c(), use_graphs ? 1 : 0, orthonormalize ? 1 : 0};
        const auto p = initial.packed();
        check(sf_tracker_create(grid.handle(), &c, p.data(), &h_));
    }
    ~Tracker() {
        if (h_) sf_tracker_destroy(h_);
    }
    Tracker(const Tracker&) = delete;
    Tracker& operator=(const Tracker&) = delete;
    void step(const DepthFrame& frame, Mode mode = Track, const Pose* pose = nullptr, void* stream = nullptr) {
        const sf_frame f = frame.c();
        std::array<double, 12> p{};
        if (pose) p = pose->packed();
        check(sf_tracker_step(h_, &f, mode, pose ? p.data() : nullptr, stream));
    }
    void set_pose(const Pose& pose, void* stream = nullptr) {
        const auto p = pose.packed();
        check(sf_tracker_set_pose(h_, p.data(), stream));
    }
    sf_frame_metrics fetch(void* stream = nullptr) {
        sf_frame_metrics m;
        check(sf_tracker_fetch(h_, &m, stream));
        if (m.status == SF_TRACKING_LOST) throw TrackingLost("icp: too few correspondences");
        if (m.status == SF_POOL_EXHAUSTED) throw PoolExhausted("grid: payload pool exhausted");
        return m;
    }
    // streaming: metrics of one of the last two steps, without waiting for later steps
    sf_frame_metrics fetch_frame(int frame) {
        sf_frame_metrics m{};
        check(sf_tracker_fetch_frame(h_, frame, &m));
        return m;
    }
    // stage-timing events inside the frame graph: 2 all (default), 1 integrate only, 0 none
    void set_stage_timing(int level) { check(sf_tracker_set_stage_timing(h_, level)); }
    std::array<float, 5> stage_times() {
        std::array<float, 5> ms{};
        check(sf_tracker_stage_times(h_, ms.data()));
        return ms;
    }

private:
    sf_tracker_t h_ = nullptr;
};

}  // namespace sparsefusion_gpu

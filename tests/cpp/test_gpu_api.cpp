// C++ conformance cases for the device path, written like the reference's own doctest suites
// (proj/tests/test_grid.cpp, test_fusion.cpp, test_render.cpp, test_registration.cpp), against
// the C++ host API include/sparsefusion_gpu.hpp. Built by `make cpptests`; run on a GPU by
// tests/test_gpu_cpp_api.py.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cmath>
#include <vector>

#include "sparsefusion_gpu.hpp"

using namespace sparsefusion_gpu;

namespace {

GridConfig sphere_grid() {
    GridConfig c;
    c.blocks_per_axis = 32;
    c.voxels_per_block_axis = 8;
    c.box_origin = {-1.0, -1.0, 0.25};
    c.box_side = 2.0;
    return c;
}

// orbit_trajectory (scene.cpp:149-177) about +y.
std::vector<Pose> orbit(const Vec3& target, double radius, int frames, double start, double arc) {
    auto norm = [](Vec3 v) {
        const double z = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2];
        const double s = std::sqrt(z);
        return Vec3{v[0] / s, v[1] / s, v[2] / s};
    };
    auto cross = [](Vec3 a, Vec3 b) {
        return Vec3{a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
    };
    const Vec3 up{0, 1, 0};
    const Vec3 ref = norm(cross(up, Vec3{0, 0, 1}));
    const Vec3 ref2 = cross(up, ref);
    std::vector<Pose> out;
    for (int k = 0; k < frames; ++k) {
        const double a = start + (frames > 1 ? arc * k / frames : 0.0);
        Pose p;
        for (int i = 0; i < 3; ++i) p.translation[i] = target[i] + radius * (std::cos(a) * ref[i] + std::sin(a) * ref2[i]);
        const Vec3 fwd = norm(Vec3{target[0] - p.translation[0], target[1] - p.translation[1], target[2] - p.translation[2]});
        const Vec3 right = norm(cross(fwd, up));
        const Vec3 down = norm(cross(fwd, right));
        for (int i = 0; i < 3; ++i) {
            p.rotation[i * 3 + 0] = right[i];
            p.rotation[i * 3 + 1] = down[i];
            p.rotation[i * 3 + 2] = fwd[i];
        }
        out.push_back(p);
    }
    return out;
}

DepthFrame render(const Pose& pose, const Intrinsics& intr, double sphere_r = 0.4) {
    const double spheres[4] = {0.0, 0.0, 1.3, sphere_r};
    const double planes[4] = {0.0, 0.0, -1.0, -2.0};
    sf_scene sc{spheres, 1, planes, 1, nullptr, 0};
    DepthFrame f(intr);
    const auto p = pose.packed();
    const sf_intrinsics ic = intr.c();
    check(sf_render_synthetic_depth(&sc, p.data(), &ic, 0.0, 0, 256, 1e-5, 2.0, f.depth.data(), nullptr));
    return f;
}

}  // namespace

TEST_CASE("fresh grid hands out slot 0 first; allocation is idempotent; PoolExhausted") {
    GridConfig c;
    c.blocks_per_axis = 4;
    c.voxels_per_block_axis = 4;
    SparseTsdfGrid grid(c, 2);
    CHECK(grid.allocate_block({1, 2, 3}) == 0);
    CHECK(grid.allocate_block({1, 2, 3}) == 0);
    CHECK(grid.allocate_block({0, 0, 0}) == 1);
    CHECK_THROWS_AS(grid.allocate_block({3, 3, 3}), PoolExhausted);
    CHECK_THROWS_AS(grid.allocate_block({4, 0, 0}), std::out_of_range);
    grid.free_block({1, 2, 3});
    CHECK(grid.allocate_block({2, 2, 2}) == 0);  // LIFO free list (grid.cpp:106)
}

TEST_CASE("memory_bytes == 2 * allocated * M^3 + 4 * N^3") {
    GridConfig c;
    c.blocks_per_axis = 16;
    c.voxels_per_block_axis = 8;
    SparseTsdfGrid grid(c, 64);
    CHECK(grid.memory_bytes() == 4ull * 16 * 16 * 16);
    grid.allocate_block({3, 4, 5});
    CHECK(grid.memory_bytes() == 4ull * 16 * 16 * 16 + 2ull * 512);
}

TEST_CASE("chi semantics of write_voxel") {
    GridConfig c;
    c.blocks_per_axis = 4;
    c.voxels_per_block_axis = 4;
    SparseTsdfGrid grid(c, 8);
    CHECK_NOTHROW(grid.write_voxel({0, 0, 0}, std::nullopt, 0.0));  // chi into EMPTY: no-op
    CHECK_THROWS_AS(grid.write_voxel({0, 0, 0}, 0.01, 1.0), std::logic_error);
    grid.allocate_block({0, 0, 0});
    CHECK(!grid.read_voxel({1, 1, 1}).has_value());
    grid.write_voxel({1, 1, 1}, 0.5 * grid.delta(), 3.0);
    const auto v = grid.read_voxel({1, 1, 1});
    REQUIRE(v.has_value());
    CHECK(std::abs(v->tsdf - 0.5 * grid.delta()) <= grid.delta() / 126.0);
    grid.write_voxel({1, 1, 1}, 2.0 * grid.delta(), 3.0);  // |T| > delta -> chi
    CHECK(!grid.read_voxel({1, 1, 1}).has_value());
}

TEST_CASE("fused sphere is raycast back to the input depth within a voxel") {
    const Intrinsics intr = Intrinsics::simple(320, 240, 262.5);
    SparseTsdfGrid grid(sphere_grid(), 0, AuxQuantization{AuxMode::Variance});
    FusionParams fp;
    fp.mode = FusionMode::Kalman;
    const auto poses = orbit({0.0, 0.0, 1.3}, 1.3, 100, M_PI / 4, M_PI / 2);
    for (int k = 0; k < 100; k += 10) {
        const FusionStats s = fuse_frame(grid, render(poses[k], intr), poses[k], fp);
        CHECK(s.memory_bytes == grid.memory_bytes());
    }
    const DepthFrame truth = render(poses[50], intr);
    const RaycastResult r = raycast(grid, poses[50], intr);
    size_t both = 0, agree = 0;
    for (size_t i = 0; i < truth.depth.size(); ++i)
        if (truth.depth[i] > 0.f && r.depth.depth[i] > 0.f) {
            ++both;
            if (std::abs(truth.depth[i] - r.depth.depth[i]) <= sphere_grid().voxel_size()) ++agree;
        }
    CHECK(both > 20000);
    CHECK(static_cast<double>(agree) / both > 0.95);  // test_render.cpp:155-194
    CHECK(r.stats.steps_per_hit() > 1.0);
}

TEST_CASE("ICP recovers a small rigid perturbation of a rendered frame") {
    const Intrinsics intr = Intrinsics::simple(320, 240, 262.5);
    const auto poses = orbit({0.0, 0.0, 1.3}, 1.3, 100, M_PI / 4, M_PI / 2);
    const Pose target_pose = poses[10];
    Pose perturb;
    const double a = 1.0 * M_PI / 180.0;
    perturb.rotation = {std::cos(a), 0, std::sin(a), 0, 1, 0, -std::sin(a), 0, std::cos(a)};
    perturb.translation = {0.005, -0.003, 0.004};
    const Pose source_pose = compose(target_pose, perturb);
    const DepthFrame target = render(target_pose, intr), source = render(source_pose, intr);
    const NormalMap tn = compute_normals(target, 2.5e-4, 2.0 / 256);
    const IcpResult r = icp(source, target, tn, Pose::identity(), MatchParams::for_voxel_size(2.0 / 256));
    const Pose truth = compose(invert(target_pose), source_pose);
    double err = 0.0;
    for (int i = 0; i < 9; ++i) err = std::max(err, std::abs(r.delta.rotation[i] - truth.rotation[i]));
    for (int i = 0; i < 3; ++i) err = std::max(err, std::abs(r.delta.translation[i] - truth.translation[i]));
    CHECK(r.matches > 1000);
    CHECK(err < 2e-3);
}

TEST_CASE("TrackingLost below ten correspondences") {
    const Intrinsics intr = Intrinsics::simple(64, 48, 55.0);
    DepthFrame empty(intr);
    NormalMap nm(64, 48);
    CHECK_THROWS_AS(icp(empty, empty, nm, Pose::identity(), MatchParams()), TrackingLost);
}

TEST_CASE("tracker runs the fused-frame loop without losing track") {
    const Intrinsics intr = Intrinsics::simple(320, 240, 262.5);
    SparseTsdfGrid grid(sphere_grid(), 0, AuxQuantization{AuxMode::Variance});
    FusionParams fp;
    fp.mode = FusionMode::Kalman;
    const auto poses = orbit({0.0, 0.0, 1.3}, 1.3, 100, M_PI / 4, M_PI / 2);
    Tracker tracker(grid, intr, fp, MatchParams::for_voxel_size(2.0 / 256), poses[0]);
    sf_frame_metrics m{};
    for (int k = 0; k < 12; ++k) {
        tracker.step(render(poses[k], intr));
        m = tracker.fetch();
    }
    CHECK(m.registered == 1);
    double err = 0.0;
    for (int i = 0; i < 3; ++i) err = std::max(err, std::abs(m.pose[9 + i] - poses[11].translation[i]));
    CHECK(err < 0.01);
    CHECK(m.fusion.blocks_total == grid.allocated_count());
}

TEST_CASE("marching cubes: one written cube straddling all eight blocks") {  // test_render.cpp:249-272
    GridConfig cfg;
    cfg.blocks_per_axis = 2;
    cfg.voxels_per_block_axis = 4;
    cfg.box_origin = {0.0, 0.0, 0.0};
    cfg.box_side = 1.0;
    SparseTsdfGrid grid(cfg, 8);
    CHECK(marching_cubes(grid).empty());
    const double delta = grid.delta();
    for (int bz = 0; bz < 2; ++bz)
        for (int by = 0; by < 2; ++by)
            for (int bx = 0; bx < 2; ++bx) grid.allocate_block({bx, by, bz});
    for (int dz = 0; dz < 2; ++dz)
        for (int dy = 0; dy < 2; ++dy)
            for (int dx = 0; dx < 2; ++dx) {
                const bool inside = dx == 0 && dy == 0 && dz == 0;
                grid.write_voxel({3 + dx, 3 + dy, 3 + dz}, inside ? -0.3 * delta : 0.3 * delta, 1.0);
            }
    const Mesh mesh = marching_cubes(grid);
    CHECK(mesh.triangles.size() == 1);
    CHECK(mesh.vertices.size() == 3);
    for (const auto& n : mesh.normals)
        CHECK(std::abs(std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]) - 1.0f) < 1e-5f);
}

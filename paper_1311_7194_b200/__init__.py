"""B200-native sparse-TSDF hot path (Trifonov, arXiv 1311.7194): block allocation,
Kalman/weighted/simple per-voxel integration, sparse raycasting and point-to-plane ICP,
hand-written CUDA for sm_100a behind the C-ABI of include/sf_gpu.h.

The package-level names mirror the reference Python module ``sparsefusion``
(proj/python/module.cpp) for this path; every compute call runs on the GPU through
``_native/libsf_gpu.so`` (there is no CPU fallback).
"""
from .api import (  # noqa: F401
    AnalyticScene,
    AuxMode,
    Backend,
    DepthFrame,
    FrameMetrics,
    FusionMode,
    FusionParams,
    FusionStats,
    GridConfig,
    IcpResult,
    Intrinsics,
    MatchParams,
    NormalMap,
    PoolExhausted,
    Pose,
    RaycastStats,
    SparseTsdfGrid,
    Tracker,
    TrackingLost,
    apply_motion,
    compose,
    default_backend,
    invert,
    orbit_trajectory,
)


def fuse_frame(grid, frame, pose, params, stream=None):
    """fuse_frame (fusion.hpp:102-103) on the GPU."""
    return grid.backend.fuse_frame(grid, frame, pose, params, stream)


def select_update_blocks(grid, frame, pose):
    """select_update_blocks (fusion.hpp:71-72): (allocate list, update list) as (K, 3) int arrays."""
    return grid.backend.select_update_blocks(grid, frame, pose)


def compute_ray_bounds(grid, pose, intrinsics):
    """compute_ray_bounds (render.hpp:38-39): (t_start, t_end) float32 (H, W)."""
    return grid.backend.compute_ray_bounds(grid, pose, intrinsics)


def raycast(grid, pose, intrinsics):
    """raycast (module.cpp:283-289): (DepthFrame, NormalMap, hit_pixels)."""
    return grid.backend.raycast(grid, pose, intrinsics)


def write_dfrm(frame, path):
    """write_dfrm (frame_io.hpp:15; module.cpp:304): the reference's DFRM byte layout."""
    default_backend().write_dfrm(frame, path)


def read_dfrm(path):
    """read_dfrm (frame_io.hpp:16; module.cpp:305)."""
    return default_backend().read_dfrm(path)


def marching_cubes(grid, region=None, batch_memory_budget=0):
    """marching_cubes (marching_cubes.hpp:37-44; module.cpp:291-293): (vertices, normals,
    triangles) numpy arrays. region: optional (Pose, Intrinsics) FrustumRegion."""
    return grid.backend.marching_cubes(grid, region, batch_memory_budget)


def raycast_result(grid, pose, intrinsics, out_depth=None, out_normals=None, stream=None):
    """RaycastResult (render.hpp:51-55): (DepthFrame, NormalMap, RaycastStats)."""
    return grid.backend.raycast_result(grid, pose, intrinsics, out_depth, out_normals, stream)


def compute_normals(frame, sigma0=2.5e-4, spatial_scale=0.0):
    """compute_normals (camera.hpp:90, module.cpp:174-178)."""
    return default_backend().compute_normals(frame, sigma0, spatial_scale)


def icp(source, target, target_normals, initial, params, source_normals=None):
    """icp (registration.hpp:120-124, module.cpp:273-279)."""
    return default_backend().icp(source, target, target_normals, initial, params, source_normals)


def render_synthetic_depth(scene, pose, intrinsics, sigma0=0.0, seed=0, max_steps=256, tolerance_scale=1e-5,
                           domain_size=1.0):
    """render_synthetic_depth (scene.hpp:69-71, module.cpp:166-172): sphere tracing on the GPU."""
    return default_backend().render_synthetic_depth(scene, pose, intrinsics, sigma0, seed, max_steps,
                                                    tolerance_scale, domain_size)


def version():
    from . import _abi

    return _abi.product().version().decode()

"""ctypes mirror of the C-ABI in include/sf_gpu.h.

The same structure layouts are used for the product library (``libsf_gpu.so``, symbols
``sf_*``) and, in the tests only, for the reference wrapper (``oracle/_ref/libsfref.so``,
symbols ``sfref_*``), which exposes the identical signatures.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# SF_GPU_LIB: an alternative build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("SF_GPU_LIB") or os.path.join(_HERE, "_native", "libsf_gpu.so")

SF_OK = 0
SF_INVALID_ARGUMENT = 1
SF_OUT_OF_RANGE = 2
SF_LOGIC_ERROR = 3
SF_POOL_EXHAUSTED = 4
SF_TRACKING_LOST = 5
SF_CUDA_ERROR = 6
SF_IO_ERROR = 7
SF_UNSUPPORTED = 8

SF_PAYLOAD_CODES = 0
SF_PAYLOAD_CODES_FLOAT_SHADOW = 1
SF_PAYLOAD_FLOAT2 = 2

c_double_p = C.POINTER(C.c_double)
c_float_p = C.POINTER(C.c_float)


class GridConfigC(C.Structure):
    _fields_ = [
        ("blocks_per_axis", C.c_int32),
        ("voxels_per_block_axis", C.c_int32),
        ("box_origin", C.c_double * 3),
        ("box_side", C.c_double),
        ("truncation", C.c_double),
    ]


class AuxQuantC(C.Structure):
    _fields_ = [("mode", C.c_int32), ("w_max", C.c_double), ("p_min", C.c_double), ("p_max", C.c_double)]


class IntrinsicsC(C.Structure):
    _fields_ = [
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("fx", C.c_double),
        ("fy", C.c_double),
        ("cx", C.c_double),
        ("cy", C.c_double),
        ("near_plane", C.c_double),
        ("far_plane", C.c_double),
    ]


class FrameC(C.Structure):
    _fields_ = [
        ("intrinsics", IntrinsicsC),
        ("depth", C.c_void_p),
        ("sigma", C.c_void_p),
        ("on_device", C.c_int32),
    ]


class FusionParamsC(C.Structure):
    _fields_ = [
        ("mode", C.c_int32),
        ("w_fixed", C.c_double),
        ("w_max", C.c_double),
        ("process_variance", C.c_double),
        ("sigma0", C.c_double),
        ("delta", C.c_double),
        ("refinement_steps", C.c_int32),
        ("edge_downweight", C.c_int32),
        ("min_variance", C.c_double),
    ]


class FusionStatsC(C.Structure):
    _fields_ = [
        ("voxels_updated", C.c_uint64),
        ("blocks_allocated_now", C.c_uint64),
        ("blocks_total", C.c_uint64),
        ("memory_bytes", C.c_uint64),
    ]


class RaycastStatsC(C.Structure):
    _fields_ = [("sample_steps", C.c_uint64), ("hit_pixels", C.c_uint64), ("rays_with_bounds", C.c_uint64)]


class MatchParamsC(C.Structure):
    _fields_ = [
        ("max_distance", C.c_double),
        ("max_normal_angle", C.c_double),
        ("max_iterations", C.c_int32),
        ("convergence_epsilon", C.c_double),
        ("eigen_threshold", C.c_double),
        ("shrink_floor", C.c_double),
        ("normal_sigma0", C.c_double),
        ("normal_spatial_scale", C.c_double),
        ("reduction", C.c_int32),
    ]


class IcpResultC(C.Structure):
    _fields_ = [
        ("delta", C.c_double * 12),
        ("iterations", C.c_int32),
        ("matches", C.c_uint64),
        ("motion_r", C.c_double * 3),
        ("motion_t", C.c_double * 3),
        ("eigenvalues", C.c_double * 6),
        ("eigenvectors", C.c_double * 36),
        ("gated_mask", C.c_int32 * 6),
        ("residual_rms", C.c_double),
        ("shrunk_motion_norm", C.c_double),
        ("pair_count", C.c_uint64),
    ]


class VolumeInfoC(C.Structure):
    _fields_ = [
        ("config", GridConfigC),
        ("aux", AuxQuantC),
        ("delta", C.c_double),
        ("voxel_size", C.c_double),
        ("pool_capacity", C.c_uint64),
        ("allocated_count", C.c_uint64),
        ("memory_bytes", C.c_uint64),
    ]


class TrackerConfigC(C.Structure):
    _fields_ = [
        ("fusion", FusionParamsC),
        ("match", MatchParamsC),
        ("camera", IntrinsicsC),
        ("use_graphs", C.c_int32),
        ("orthonormalize", C.c_int32),
    ]


class ShardTrackerConfigC(C.Structure):
    _fields_ = [
        ("base", TrackerConfigC),
        ("icp_mode", C.c_int32),
        ("pad_", C.c_int32),
        ("halo_capacity", C.c_uint64),
    ]


class ShardFrameMetricsC(C.Structure):
    _fields_ = [
        ("frame", C.c_int32),
        ("registered", C.c_int32),
        ("status", C.c_int32),
        ("iterations", C.c_int32),
        ("pose", C.c_double * 12),
        ("matches", C.c_uint64),
        ("voxels_updated", C.c_uint64),
        ("blocks_total", C.c_uint64),
        ("hit_pixels", C.c_uint64),
        ("halo_records", C.c_uint64),
        ("halo_overflow", C.c_uint64),
        ("kernel_launches", C.c_uint64),
        ("icp_steps", C.c_int32),
        ("pad_", C.c_int32),
    ]


class FrameMetricsC(C.Structure):
    _fields_ = [
        ("frame", C.c_int32),
        ("registered", C.c_int32),
        ("status", C.c_int32),
        ("pose", C.c_double * 12),
        ("iterations", C.c_int32),
        ("matches", C.c_uint64),
        ("residual_rms", C.c_double),
        ("lambda_over_n", C.c_double * 6),
        ("gated_mask", C.c_int32 * 6),
        ("fusion", FusionStatsC),
        ("raycast", RaycastStatsC),
        ("blocks_processed", C.c_uint64),
        ("voxels_visited", C.c_uint64),
        ("kernel_launches", C.c_uint64),
        ("exact_voxels", C.c_uint64),
        ("integrate_ns", C.c_uint64),
        ("icp_ns", C.c_uint64),
        ("icp_steps", C.c_int32),
        ("pad_", C.c_int32),
        ("ray_dda_cells", C.c_uint64),
        ("ray_refine_samples", C.c_uint64),
    ]


class SceneC(C.Structure):
    _fields_ = [
        ("spheres", c_double_p),
        ("sphere_count", C.c_int32),
        ("planes", c_double_p),
        ("plane_count", C.c_int32),
        ("boxes", c_double_p),
        ("box_count", C.c_int32),
    ]


P = C.POINTER
vp = C.c_void_p
i32 = C.c_int32
u64 = C.c_uint64
i32p = P(C.c_int32)
u64p = P(C.c_uint64)

# name -> (restype, argtypes); "{p}" is the symbol prefix ("sf" or "sfref")
SIGNATURES = {
    "last_error": (C.c_char_p, []),
    "volume_create": (C.c_int, [P(GridConfigC), u64, P(AuxQuantC), i32, P(vp)]),
    "volume_destroy": (C.c_int, [vp]),
    "volume_get_info": (C.c_int, [vp, P(VolumeInfoC)]),
    "volume_allocate_block": (C.c_int, [vp, i32p, i32p]),
    "volume_free_block": (C.c_int, [vp, i32p]),
    "volume_block_slot": (C.c_int, [vp, i32p, i32p]),
    "volume_read_voxel": (C.c_int, [vp, i32p, i32p, c_double_p, c_double_p]),
    "volume_write_voxel": (C.c_int, [vp, i32p, i32, C.c_double, C.c_double]),
    "volume_read_table": (C.c_int, [vp, vp]),
    "volume_read_payload": (C.c_int, [vp, u64, u64, vp]),
    "volume_write_payload": (C.c_int, [vp, u64, u64, vp]),
    "volume_save_snapshot": (C.c_int, [vp, C.c_char_p]),
    "volume_load_snapshot": (C.c_int, [C.c_char_p, u64, i32, P(vp)]),
    "integrate": (C.c_int, [vp, P(FrameC), c_double_p, P(FusionParamsC), P(FusionStatsC), vp]),
    "select_update_blocks": (C.c_int, [vp, P(FrameC), c_double_p, i32p, u64p, i32p, u64p, vp]),
    "ray_bounds": (C.c_int, [vp, c_double_p, P(IntrinsicsC), vp, vp, i32, vp]),
    "raycast": (C.c_int, [vp, c_double_p, P(IntrinsicsC), vp, vp, i32, P(RaycastStatsC), vp]),
    "compute_normals": (C.c_int, [P(FrameC), C.c_double, C.c_double, vp, i32, vp]),
    "icp": (C.c_int, [P(FrameC), vp, P(FrameC), vp, c_double_p, P(MatchParamsC), P(IcpResultC), vp]),
    "render_synthetic_depth": (
        C.c_int,
        [P(SceneC), c_double_p, P(IntrinsicsC), C.c_double, u64, i32, C.c_double, C.c_double, vp, vp],
    ),
}

# marching cubes: the product and the reference build (the C restatement does not cover it;
# its parity is checked against the reference itself)
MESH = {
    "marching_cubes": (C.c_int, [vp, c_double_p, P(IntrinsicsC), u64, P(vp), vp]),
    "mesh_counts": (C.c_int, [vp, u64p, u64p]),
    "mesh_read": (C.c_int, [vp, vp, vp, vp, i32, vp]),
    "mesh_destroy": (C.c_int, [vp]),
    "dfrm_write": (C.c_int, [C.c_char_p, P(FrameC)]),
    "dfrm_read": (C.c_int, [C.c_char_p, P(IntrinsicsC), vp, vp, P(C.c_int32), i32]),
    "trajectory_write": (C.c_int, [C.c_char_p, i32p, c_double_p, u64]),
    "trajectory_read": (C.c_int, [C.c_char_p, i32p, c_double_p, u64p]),
}

PRODUCT_ONLY = {
    "version": (C.c_char_p, []),
    "volume_read_free_list": (C.c_int, [vp, i32p, u64p]),
    "volume_enable_float_payload": (C.c_int, [vp]),
    "volume_read_float_payload": (C.c_int, [vp, u64, u64, vp]),
    "volume_set_payload_layout": (C.c_int, [vp, i32]),
    "volume_write_float_payload": (C.c_int, [vp, u64, u64, vp]),
    "volume_import_state": (C.c_int, [vp, vp, vp, u64, vp, u64]),
    "volume_get_payload_layout": (C.c_int, [vp, i32p]),
    "tracker_create": (C.c_int, [vp, P(TrackerConfigC), c_double_p, P(vp)]),
    "tracker_destroy": (C.c_int, [vp]),
    "tracker_step": (C.c_int, [vp, P(FrameC), i32, c_double_p, vp]),
    "tracker_fetch": (C.c_int, [vp, P(FrameMetricsC), vp]),
    "tracker_fetch_frame": (C.c_int, [vp, i32, P(FrameMetricsC)]),
    "tracker_set_pose": (C.c_int, [vp, c_double_p, vp]),
    "tracker_device_pose": (C.c_int, [vp, P(c_double_p)]),
    "tracker_last_launch_count": (C.c_int, [vp, u64p]),
    "tracker_stage_times": (C.c_int, [vp, P(C.c_float)]),
    "tracker_set_stage_timing": (C.c_int, [vp, C.c_int32]),
    "tracker_io_bytes": (C.c_int, [vp, i32, u64p, u64p]),
    "debug_aux_tables": (C.c_int, [P(AuxQuantC), C.c_double, c_double_p, c_double_p, c_double_p]),
    # spatial sharding
    "volume_set_shard": (C.c_int, [vp, i32, i32, i32]),
    "shard_owner": (C.c_int32, [i32, i32, i32, i32, i32]),
    "raycast_with_bounds": (C.c_int, [vp, c_double_p, P(IntrinsicsC), vp, vp, vp, vp, i32, P(RaycastStatsC), vp]),
    "composite_key": (C.c_int, [vp, vp, u64, i32, vp, vp]),
    "composite_select": (C.c_int, [vp, u64, i32, vp, vp, vp]),
    "shard_pack_halo": (C.c_int, [vp, vp, vp, u64, P(C.c_uint32), vp]),
    "shard_apply_halo": (C.c_int, [vp, vp, vp, u64, P(C.c_uint32), vp]),
    "nccl_unique_id": (C.c_int, [vp]),
    "shard_tracker_create_local": (C.c_int, [P(vp), i32, P(ShardTrackerConfigC), c_double_p, P(vp)]),
    "shard_tracker_create_nccl": (C.c_int, [vp, vp, i32, i32, P(ShardTrackerConfigC), c_double_p, P(vp)]),
    "shard_tracker_destroy": (C.c_int, [vp]),
    "shard_tracker_step": (C.c_int, [vp, P(FrameC), i32, c_double_p, vp]),
    "shard_tracker_set_pose": (C.c_int, [vp, c_double_p, vp]),
    "shard_tracker_fetch": (C.c_int, [vp, P(ShardFrameMetricsC), vp]),
}

REF_ONLY = {
    "volume_check_consistency": (C.c_int, [vp]),
    "volume_enable_shadow": (C.c_int, [vp]),
    "volume_read_shadow": (C.c_int, [vp, c_float_p, c_float_p]),
    "estimate_measurement": (
        C.c_int,
        [P(FrameC), c_double_p, c_double_p, P(FusionParamsC), i32p, c_double_p, c_double_p, c_double_p],
    ),
    "orbit_trajectory": (C.c_int, [c_double_p, C.c_double, i32, c_double_p, C.c_double, C.c_double, c_double_p]),
    "compose": (C.c_int, [c_double_p, c_double_p, c_double_p]),
    "invert": (C.c_int, [c_double_p, c_double_p]),
    "apply_motion": (C.c_int, [c_double_p, c_double_p, c_double_p, c_double_p]),
    "pipeline_frame": (
        C.c_int,
        [vp, P(FrameC), P(IntrinsicsC), P(FusionParamsC), P(MatchParamsC), i32, c_double_p, c_double_p,
         P(FusionStatsC), i32p, u64p],
    ),
}

# sf_gpu.h declarations that the CPU suite checks are exported by libsf_gpu.so
EXPORTED = sorted(
    ["sf_" + k for k in SIGNATURES] + ["sf_" + k for k in MESH]
    + ["sf_" + k for k in PRODUCT_ONLY if k != "debug_aux_tables"]
)


class Lib:
    """A loaded C-ABI library with typed entry points ``lib.<name>`` (prefix stripped)."""

    def __init__(self, path: str, prefix: str, extra: dict):
        self.path = path
        self.prefix = prefix
        self.handle = C.CDLL(path)
        sigs = dict(SIGNATURES)
        sigs.update(extra)
        for name, (res, args) in sigs.items():
            fn = getattr(self.handle, f"{prefix}_{name}")
            fn.restype = res
            fn.argtypes = args
            setattr(self, name, fn)

    def error(self) -> str:
        msg = self.last_error()
        return msg.decode() if msg else ""


_product = None


def product() -> Lib:
    """Load libsf_gpu.so. There is no fallback: a missing build is an error."""
    global _product
    if _product is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is not built; run `make` (or __graft_entry__.build()) - "
                "the sparse-TSDF path has no CPU fallback"
            )
        _product = Lib(LIB_PATH, "sf", {**PRODUCT_ONLY, **MESH})
    return _product

"""Python mirror of the reference's ``sparsefusion`` module (proj/python/module.cpp:104-338)
for the sparse-TSDF hot path, over the C-ABI of include/sf_gpu.h.

Names, argument meaning and error behaviour follow the reference binding:
``SparseTsdfGrid``, ``fuse_frame``, ``raycast``, ``compute_normals``, ``icp``,
``render_synthetic_depth``, ``orbit_trajectory``, ``compose``/``invert``, and the
exceptions ``PoolExhausted`` / ``TrackingLost`` (module.cpp:108-109); std::invalid_argument
maps to ValueError, std::out_of_range to IndexError, as pybind11 does.

A ``Backend`` wraps one C-ABI library. The package-level API uses the CUDA library
(``libsf_gpu.so``); the test-suite builds a second Backend over the reference wrapper
(``oracle/_ref/libsfref.so``) to run both on identical inputs. Frames and normal maps
are numpy arrays (host) or CUDA torch tensors (device; zero-copy).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _abi as A

# ---------------------------------------------------------------------------------
# exceptions (module.cpp:108-109)
# ---------------------------------------------------------------------------------


class PoolExhausted(RuntimeError):
    """grid.hpp:24-26 — allocate_block found no free pool slot."""


class TrackingLost(RuntimeError):
    """registration.hpp:18-20 — fewer than 10 ICP correspondences."""


def _raise(status: int, msg: str):
    if status == A.SF_OK:
        return
    if status == A.SF_POOL_EXHAUSTED:
        raise PoolExhausted(msg)
    if status == A.SF_TRACKING_LOST:
        raise TrackingLost(msg)
    if status == A.SF_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == A.SF_OUT_OF_RANGE:
        raise IndexError(msg)
    if status == A.SF_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg or f"sf status {status}")


# ---------------------------------------------------------------------------------
# plain data (camera.hpp, pose.hpp, grid.hpp, fusion.hpp, registration.hpp)
# ---------------------------------------------------------------------------------


@dataclass
class Intrinsics:
    width: int = 0
    height: int = 0
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    near: float = 0.1
    far: float = 10.0

    @staticmethod
    def simple(width: int, height: int, focal_px: float, near: float = 0.1, far: float = 10.0) -> "Intrinsics":
        # Intrinsics::simple (camera.cpp:16-29)
        intr = Intrinsics(width, height, focal_px, focal_px, 0.5 * (width - 1), 0.5 * (height - 1), near, far)
        intr.validate()
        return intr

    def validate(self):
        # Intrinsics::validate (camera.cpp:9-14)
        if self.width <= 0 or self.height <= 0:
            raise ValueError("intrinsics: non-positive image size")
        if self.fx <= 0.0 or self.fy <= 0.0:
            raise ValueError("intrinsics: non-positive focal length")
        if not (self.near > 0.0) or not (self.near < self.far):
            raise ValueError("intrinsics: need 0 < near < far")

    def c(self) -> A.IntrinsicsC:
        return A.IntrinsicsC(self.width, self.height, self.fx, self.fy, self.cx, self.cy, self.near, self.far)


class Pose:
    """x_scene = R x_camera + t (pose.hpp:9-16)."""

    def __init__(self, rotation=None, translation=None):
        self.rotation = np.eye(3) if rotation is None else np.array(rotation, dtype=np.float64).reshape(3, 3)
        self.translation = np.zeros(3) if translation is None else np.array(translation, dtype=np.float64).reshape(3)

    @staticmethod
    def identity() -> "Pose":
        return Pose()

    def to12(self) -> np.ndarray:
        return np.concatenate([np.ascontiguousarray(self.rotation, dtype=np.float64).reshape(9),
                               np.asarray(self.translation, dtype=np.float64).reshape(3)])

    @staticmethod
    def from12(a) -> "Pose":
        a = np.asarray(a, dtype=np.float64)
        return Pose(a[:9].reshape(3, 3).copy(), a[9:12].copy())

    def apply(self, p):
        return _mv(self.rotation, p) + self.translation

    def __repr__(self):
        return f"Pose(R={self.rotation.tolist()}, t={self.translation.tolist()})"


def _mv(R, v):
    # Matrix3d * Vector3d in the oracle's summation order
    return np.array([(R[i][0] * v[0] + R[i][1] * v[1]) + R[i][2] * v[2] for i in range(3)], dtype=np.float64)


def compose(a: Pose, b: Pose) -> Pose:
    """compose (pose.cpp:6-11), bit-exact with the reference (explicit summation order)."""
    Ra, Rb = a.rotation.tolist(), b.rotation.tolist()
    R = [[(Ra[i][0] * Rb[0][j] + Ra[i][1] * Rb[1][j]) + Ra[i][2] * Rb[2][j] for j in range(3)] for i in range(3)]
    tb = b.translation.tolist()
    t = [((Ra[i][0] * tb[0] + Ra[i][1] * tb[1]) + Ra[i][2] * tb[2]) + float(a.translation[i]) for i in range(3)]
    return Pose(np.array(R), np.array(t))


def invert(a: Pose) -> Pose:
    """invert (pose.cpp:13-18)."""
    Rt = a.rotation.T.tolist()
    t = a.translation.tolist()
    out_t = [-((Rt[i][0] * t[0] + Rt[i][1] * t[1]) + Rt[i][2] * t[2]) for i in range(3)]
    return Pose(np.array(Rt), np.array(out_t))


def _normalized(v):
    z = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]
    if z > 0.0:
        s = math.sqrt(z)
        return [v[0] / s, v[1] / s, v[2] / s]
    return list(v)


def _cross(a, b):
    return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]


def orbit_trajectory(target, radius: float, frames: int, axis=(0.0, 1.0, 0.0), start_angle: float = 0.0,
                     arc: float = 2.0 * math.pi) -> List[Pose]:
    """orbit_trajectory (scene.cpp:149-177), same libm and operation order: bit-exact."""
    if frames < 0:
        raise ValueError("orbit: negative frame count")
    target = [float(x) for x in target]
    up = _normalized([float(x) for x in axis])
    ref = _cross(up, [0.0, 0.0, 1.0])
    if (ref[0] * ref[0] + ref[1] * ref[1]) + ref[2] * ref[2] < 1e-12:
        ref = _cross(up, [1.0, 0.0, 0.0])
    ref = _normalized(ref)
    ref2 = _cross(up, ref)
    out = []
    for k in range(frames):
        angle = start_angle + (arc * k / frames if frames > 1 else 0.0)
        c, s = math.cos(angle), math.sin(angle)
        offset = [radius * (c * ref[i] + s * ref2[i]) for i in range(3)]
        t = [target[i] + offset[i] for i in range(3)]
        forward = _normalized([target[i] - t[i] for i in range(3)])
        right = _cross(forward, up)
        if (right[0] * right[0] + right[1] * right[1]) + right[2] * right[2] < 1e-12:
            right = _cross(forward, ref)
        right = _normalized(right)
        down = _normalized(_cross(forward, right))
        R = np.array([[right[i], down[i], forward[i]] for i in range(3)])
        out.append(Pose(R, np.array(t)))
    return out


def apply_motion(pose: Pose, r, t) -> Pose:
    """apply_motion (pose.cpp:31-43): small-angle rotation projected to SO(3) (host, numpy SVD;
    the device ICP uses its own Jacobi SVD, see csrc/sf_linalg.cuh)."""
    a, b, g = (float(x) for x in r)
    lin = np.array([[1.0, -g, b], [g, 1.0, -a], [-b, a, 1.0]])
    u, _, vt = np.linalg.svd(lin)
    R = u @ vt
    if np.linalg.det(R) < 0:
        u[:, 2] *= -1
        R = u @ vt
    return compose(Pose(R, np.array(t, dtype=np.float64)), pose)


class AuxMode(enum.IntEnum):
    Weight = 0
    Variance = 1


class FusionMode(enum.IntEnum):
    Simple = 0
    Weighted = 1
    Kalman = 2


@dataclass
class GridConfig:
    blocks_per_axis: int = 16
    voxels_per_block_axis: int = 8
    box_origin: Sequence[float] = (0.0, 0.0, 0.0)
    box_side: float = 1.0
    truncation: float = 0.0

    @property
    def voxels_per_axis(self) -> int:
        return self.blocks_per_axis * self.voxels_per_block_axis

    @property
    def voxel_size(self) -> float:
        return self.box_side / self.voxels_per_axis

    @property
    def delta(self) -> float:
        return self.truncation if self.truncation > 0.0 else 4.0 * self.voxel_size

    def c(self) -> A.GridConfigC:
        o = [float(x) for x in self.box_origin]
        return A.GridConfigC(self.blocks_per_axis, self.voxels_per_block_axis, (C.c_double * 3)(*o),
                             self.box_side, self.truncation)


@dataclass
class FusionParams:
    mode: FusionMode = FusionMode.Simple
    w_fixed: float = 0.1
    w_max: float = 20.0
    process_variance: float = -1.0
    sigma0: float = 2.5e-4
    delta: float = 0.0
    refinement_steps: int = 0
    edge_downweight: bool = True
    min_variance: float = 1e-12

    def c(self) -> A.FusionParamsC:
        return A.FusionParamsC(int(self.mode), self.w_fixed, self.w_max, self.process_variance, self.sigma0,
                               self.delta, self.refinement_steps, 1 if self.edge_downweight else 0,
                               self.min_variance)


@dataclass
class FusionStats:
    voxels_updated: int = 0
    blocks_allocated_now: int = 0
    blocks_total: int = 0
    memory_bytes: int = 0


@dataclass
class RaycastStats:
    sample_steps: int = 0
    hit_pixels: int = 0
    rays_with_bounds: int = 0

    def steps_per_hit(self) -> float:
        return self.sample_steps / self.hit_pixels if self.hit_pixels else 0.0


@dataclass
class MatchParams:
    max_distance: float = 0.1
    max_normal_angle: float = 0.5235987755983
    max_iterations: int = 15
    convergence_epsilon: float = 1e-5
    eigen_threshold: float = 0.005
    shrink_floor: float = 1e-6
    normal_sigma0: float = 2.5e-4
    normal_spatial_scale: float = 0.0
    # not in the reference struct: 0 tree-ordered sums (fast, pose ~1e-15 of the reference per
    # call); 1 the reference's sequential Kahan order (bit-identical poses, sf_gpu.h)
    reduction: int = 0
    TREE, REFERENCE_ORDER = 0, 1

    @staticmethod
    def for_voxel_size(voxel_size: float) -> "MatchParams":
        # MatchParams::for_voxel_size (registration.cpp:9-15)
        return MatchParams(max_distance=10.0 * voxel_size, shrink_floor=voxel_size, normal_spatial_scale=voxel_size)

    def c(self) -> A.MatchParamsC:
        return A.MatchParamsC(self.max_distance, self.max_normal_angle, self.max_iterations,
                              self.convergence_epsilon, self.eigen_threshold, self.shrink_floor,
                              self.normal_sigma0, self.normal_spatial_scale, self.reduction)


@dataclass
class IcpResult:
    delta: Pose
    iterations: int
    matches: int
    residual_rms: float
    gated_mask: List[bool]
    eigenvalues: List[float]
    eigenvectors: np.ndarray
    shrunk_motion_norm: float
    pair_count: int
    motion_r: np.ndarray
    motion_t: np.ndarray


def _is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


class DepthFrame:
    """Row-major float depth, 0 = invalid, optional sigma plane (camera.hpp:45-63).
    ``depth``/``sigma``: numpy float32 (H, W) or CUDA torch float32 tensors."""

    def __init__(self, intrinsics: Intrinsics, depth, sigma=None):
        self.intrinsics = intrinsics
        if _is_torch_cuda(depth):
            if tuple(depth.shape) != (intrinsics.height, intrinsics.width):
                raise ValueError("depth array must be (height, width)")
            self.depth = depth.contiguous()
            self.sigma = None if sigma is None else sigma.contiguous()
            self.on_device = True
        else:
            d = np.ascontiguousarray(depth, dtype=np.float32)
            if d.shape != (intrinsics.height, intrinsics.width):
                raise ValueError("depth array must be (height, width)")
            self.depth = d
            self.sigma = None if sigma is None else np.ascontiguousarray(sigma, dtype=np.float32)
            self.on_device = False

    def c(self) -> A.FrameC:
        if self.on_device:
            dp = self.depth.data_ptr()
            sp = self.sigma.data_ptr() if self.sigma is not None else None
        else:
            dp = self.depth.ctypes.data
            sp = self.sigma.ctypes.data if self.sigma is not None else None
        return A.FrameC(self.intrinsics.c(), dp, sp, 1 if self.on_device else 0)

    def has_sigma(self) -> bool:
        return self.sigma is not None


class NormalMap:
    """Per-pixel float normals (camera.hpp:67-78); ``array`` is (H, W, 3)."""

    def __init__(self, normals):
        if _is_torch_cuda(normals):
            self.array = normals.contiguous()
            self.on_device = True
        else:
            a = np.ascontiguousarray(normals, dtype=np.float32)
            if a.ndim != 3 or a.shape[2] != 3:
                raise ValueError("normal array must be (height, width, 3)")
            self.array = a
            self.on_device = False

    def ptr(self):
        return self.array.data_ptr() if self.on_device else self.array.ctypes.data


class AnalyticScene:
    """Union of spheres, planes and axis-aligned boxes (scene.hpp:17-48)."""

    def __init__(self):
        self.spheres: List[Tuple[float, float, float, float]] = []
        self.planes: List[Tuple[float, float, float, float]] = []
        self.boxes: List[Tuple[float, float, float, float, float, float]] = []

    def add_sphere(self, center, radius: float):
        if not radius > 0.0:
            raise ValueError("scene: sphere radius must be positive")
        self.spheres.append((*map(float, center), float(radius)))

    def add_plane(self, normal, offset: float):
        self.planes.append((*map(float, normal), float(offset)))

    def add_box(self, center, half_extents):
        if not min(half_extents) > 0.0:
            raise ValueError("scene: box half extents must be positive")
        self.boxes.append((*map(float, center), *map(float, half_extents)))

    def c(self):
        s = np.ascontiguousarray(np.array(self.spheres, dtype=np.float64).reshape(-1))
        p = np.ascontiguousarray(np.array(self.planes, dtype=np.float64).reshape(-1))
        b = np.ascontiguousarray(np.array(self.boxes, dtype=np.float64).reshape(-1))
        keep = (s, p, b)
        sc = A.SceneC(s.ctypes.data_as(A.c_double_p), len(self.spheres), p.ctypes.data_as(A.c_double_p),
                      len(self.planes), b.ctypes.data_as(A.c_double_p), len(self.boxes))
        return sc, keep


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(A.c_double_p)


# ---------------------------------------------------------------------------------
# backend-bound API
# ---------------------------------------------------------------------------------


class Backend:
    def __init__(self, lib: A.Lib, name: str):
        self.lib = lib
        self.name = name

    def check(self, status: int):
        if status != A.SF_OK:
            _raise(status, self.lib.error())

    # --- fuse_frame (fusion.hpp:102-103) ---
    def fuse_frame(self, grid: "SparseTsdfGrid", frame: DepthFrame, pose: Pose, params: FusionParams,
                   stream=None) -> FusionStats:
        st = A.FusionStatsC()
        p12 = pose.to12()
        fc = frame.c()
        pc = params.c()
        self.check(self.lib.integrate(grid.handle, C.byref(fc), _dptr(p12), C.byref(pc), C.byref(st), stream))
        return FusionStats(st.voxels_updated, st.blocks_allocated_now, st.blocks_total, st.memory_bytes)

    def select_update_blocks(self, grid, frame: DepthFrame, pose: Pose):
        n = frame.intrinsics.width * frame.intrinsics.height * 3 + 16
        cap_u = grid.pool_capacity + 16
        a = np.zeros((n, 3), dtype=np.int32)
        u = np.zeros((cap_u, 3), dtype=np.int32)
        na, nu = C.c_uint64(n), C.c_uint64(cap_u)
        p12 = pose.to12()
        fc = frame.c()
        self.check(self.lib.select_update_blocks(grid.handle, C.byref(fc), _dptr(p12),
                                                 a.ctypes.data_as(A.i32p), C.byref(na),
                                                 u.ctypes.data_as(A.i32p), C.byref(nu), None))
        return a[: na.value].copy(), u[: nu.value].copy()

    # --- raycast (render.hpp:38-63) ---
    def compute_ray_bounds(self, grid, pose: Pose, intr: Intrinsics):
        ts = np.zeros((intr.height, intr.width), dtype=np.float32)
        te = np.zeros_like(ts)
        ic = intr.c()
        p12 = pose.to12()
        self.check(self.lib.ray_bounds(grid.handle, _dptr(p12), C.byref(ic), ts.ctypes.data, te.ctypes.data, 0, None))
        return ts, te

    def raycast_result(self, grid, pose: Pose, intr: Intrinsics, out_depth=None, out_normals=None, stream=None):
        """Full RaycastResult: (DepthFrame, NormalMap, RaycastStats)."""
        ic = intr.c()
        p12 = pose.to12()
        st = A.RaycastStatsC()
        if out_depth is not None:  # device outputs (torch CUDA tensors)
            self.check(self.lib.raycast(grid.handle, _dptr(p12), C.byref(ic), out_depth.data_ptr(),
                                        out_normals.data_ptr(), 1, C.byref(st), stream))
            d, n = out_depth, out_normals
        else:
            d = np.zeros((intr.height, intr.width), dtype=np.float32)
            n = np.zeros((intr.height, intr.width, 3), dtype=np.float32)
            self.check(self.lib.raycast(grid.handle, _dptr(p12), C.byref(ic), d.ctypes.data, n.ctypes.data, 0,
                                        C.byref(st), stream))
        return DepthFrame(intr, d), NormalMap(n), RaycastStats(st.sample_steps, st.hit_pixels, st.rays_with_bounds)

    def raycast(self, grid, pose: Pose, intr: Intrinsics):
        """module.cpp:283-289: (depth DepthFrame, NormalMap, hit_pixels)."""
        d, n, st = self.raycast_result(grid, pose, intr)
        return d, n, st.hit_pixels

    # --- normals (camera.hpp:90) ---
    def compute_normals(self, frame: DepthFrame, sigma0: float = 2.5e-4, spatial_scale: float = 0.0) -> NormalMap:
        intr = frame.intrinsics
        out = np.zeros((intr.height, intr.width, 3), dtype=np.float32)
        fc = frame.c()
        self.check(self.lib.compute_normals(C.byref(fc), sigma0, spatial_scale, out.ctypes.data, 0, None))
        return NormalMap(out)

    # --- icp (registration.hpp:120-124) ---
    def icp(self, source: DepthFrame, target: DepthFrame, target_normals: NormalMap, initial: Pose,
            params: MatchParams, source_normals: Optional[NormalMap] = None) -> IcpResult:
        r = A.IcpResultC()
        sc, tc = source.c(), target.c()
        p12 = initial.to12()
        mp = params.c()
        sn = source_normals.ptr() if source_normals is not None else None
        self.check(self.lib.icp(C.byref(sc), sn, C.byref(tc), target_normals.ptr(), _dptr(p12), C.byref(mp),
                                C.byref(r), None))
        return IcpResult(
            delta=Pose.from12(list(r.delta)), iterations=r.iterations, matches=r.matches,
            residual_rms=r.residual_rms, gated_mask=[bool(x) for x in r.gated_mask],
            eigenvalues=list(r.eigenvalues), eigenvectors=np.array(list(r.eigenvectors)).reshape(6, 6).T,
            shrunk_motion_norm=r.shrunk_motion_norm, pair_count=r.pair_count,
            motion_r=np.array(list(r.motion_r)), motion_t=np.array(list(r.motion_t)))

    # --- DFRM files (frame_io.hpp:15-16; module.cpp:304-305) ---
    def write_dfrm(self, frame: DepthFrame, path: str):
        fc = frame.c()
        self.check(self.lib.dfrm_write(path.encode(), C.byref(fc)))

    def write_trajectory(self, entries, path: str):
        """write_trajectory (frame_io.cpp:81-93): entries = [(frame_index, Pose), ...]."""
        n = len(entries)
        fi = np.array([int(e[0]) for e in entries], dtype=np.int32)
        p = np.array([e[1].to12() for e in entries], dtype=np.float64).reshape(n, 12)
        self.check(self.lib.trajectory_write(path.encode(), fi.ctypes.data_as(A.i32p), _dptr(p), n))

    def read_trajectory(self, path: str):
        """read_trajectory (frame_io.cpp:117-126) -> [(frame_index, Pose), ...]."""
        cnt = C.c_uint64(0)
        self.check(self.lib.trajectory_read(path.encode(), None, None, C.byref(cnt)))
        fi = np.zeros(max(1, cnt.value), dtype=np.int32)
        p = np.zeros((max(1, cnt.value), 12), dtype=np.float64)
        self.check(self.lib.trajectory_read(path.encode(), fi.ctypes.data_as(A.i32p), _dptr(p), C.byref(cnt)))
        return [(int(fi[i]), Pose.from12(p[i])) for i in range(cnt.value)]

    def read_dfrm(self, path: str, device=None) -> DepthFrame:
        """read_dfrm (frame_io.cpp:47-79). device: a CUDA device -> the depth (and sigma) planes are
        read straight into device buffers (torch tensors, sf_frame.on_device = 1)."""
        ic = A.IntrinsicsC()
        self.check(self.lib.dfrm_read(path.encode(), C.byref(ic), None, None, None, 0))
        intr = Intrinsics(ic.width, ic.height, ic.fx, ic.fy, ic.cx, ic.cy, ic.near_plane, ic.far_plane)
        hs = C.c_int32(0)
        if device is not None:
            import torch

            d = torch.zeros((ic.height, ic.width), dtype=torch.float32, device=device)
            s = torch.zeros_like(d)
            self.check(self.lib.dfrm_read(path.encode(), C.byref(ic), d.data_ptr(), s.data_ptr(), C.byref(hs), 1))
            return DepthFrame(intr, d, s if hs.value else None)
        d = np.zeros((ic.height, ic.width), dtype=np.float32)
        s = np.zeros_like(d)
        self.check(self.lib.dfrm_read(path.encode(), C.byref(ic), d.ctypes.data, s.ctypes.data, C.byref(hs), 0))
        return DepthFrame(intr, d, s if hs.value else None)

    # --- marching cubes (marching_cubes.hpp:37-44; module.cpp:291-293) ---
    def marching_cubes(self, grid, region=None, batch_memory_budget: int = 0):
        """(vertices (V,3) float32, normals (V,3) float32, triangles (T,3) uint32).
        region: optional (Pose, Intrinsics) FrustumRegion."""
        h = C.c_void_p()
        if region is not None:
            pose, intr = region
            p12 = pose.to12()
            ic = intr.c()
            self.check(self.lib.marching_cubes(grid.handle, _dptr(p12), C.byref(ic), batch_memory_budget,
                                               C.byref(h), None))
        else:
            self.check(self.lib.marching_cubes(grid.handle, None, None, batch_memory_budget, C.byref(h), None))
        try:
            nv, nt = C.c_uint64(), C.c_uint64()
            self.check(self.lib.mesh_counts(h, C.byref(nv), C.byref(nt)))
            v = np.zeros((nv.value, 3), dtype=np.float32)
            n = np.zeros((nv.value, 3), dtype=np.float32)
            t = np.zeros((nt.value, 3), dtype=np.uint32)
            self.check(self.lib.mesh_read(h, v.ctypes.data, n.ctypes.data, t.ctypes.data, 0, None))
        finally:
            self.lib.mesh_destroy(h)
        return v, n, t

    # --- synthetic input (scene.hpp:69-71) ---
    def render_synthetic_depth(self, scene: AnalyticScene, pose: Pose, intrinsics: Intrinsics, sigma0: float = 0.0,
                               seed: int = 0, max_steps: int = 256, tolerance_scale: float = 1e-5,
                               domain_size: float = 1.0) -> DepthFrame:
        intrinsics.validate()
        d = np.zeros((intrinsics.height, intrinsics.width), dtype=np.float32)
        s = np.zeros_like(d) if sigma0 > 0.0 else None
        sc, keep = scene.c()
        ic = intrinsics.c()
        p12 = pose.to12()
        self.check(self.lib.render_synthetic_depth(C.byref(sc), _dptr(p12), C.byref(ic), sigma0, seed, max_steps,
                                                   tolerance_scale, domain_size, d.ctypes.data,
                                                   s.ctypes.data if s is not None else None))
        del keep
        return DepthFrame(intrinsics, d, s)


class SparseTsdfGrid:
    """Block-sparse TSDF volume (grid.hpp:96-193), device resident."""

    kEmpty = -1

    def __init__(self, config: GridConfig, pool_capacity: int = 0, aux_mode: AuxMode = AuxMode.Weight,
                 w_max: float = 20.0, p_min: float = 1e-8, p_max: float = 1e-2, device: int = 0,
                 backend: Optional[Backend] = None, _handle=None):
        self.backend = backend or default_backend()
        self._config = config
        if _handle is not None:
            self.handle = _handle
        else:
            h = C.c_void_p()
            aux = A.AuxQuantC(int(aux_mode), w_max, p_min, p_max)
            cc = config.c()
            self.backend.check(self.backend.lib.volume_create(C.byref(cc), pool_capacity, C.byref(aux), device,
                                                              C.byref(h)))
            self.handle = h
        self._info()

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                self.backend.lib.volume_destroy(h)
            except Exception:
                pass
            self.handle = None

    def _info(self) -> A.VolumeInfoC:
        info = A.VolumeInfoC()
        self.backend.check(self.backend.lib.volume_get_info(self.handle, C.byref(info)))
        c = info.config
        self._config = GridConfig(c.blocks_per_axis, c.voxels_per_block_axis, tuple(c.box_origin), c.box_side,
                                  c.truncation)
        self._static = info
        return info

    @property
    def config(self) -> GridConfig:
        return self._config

    @property
    def allocated_count(self) -> int:
        return self._info().allocated_count

    @property
    def pool_capacity(self) -> int:
        return self._static.pool_capacity

    @property
    def voxel_size(self) -> float:
        return self._static.voxel_size

    @property
    def delta(self) -> float:
        return self._static.delta

    @property
    def aux_mode(self) -> AuxMode:
        return AuxMode(self._static.aux.mode)

    def memory_bytes(self) -> int:
        return self._info().memory_bytes

    def block_side(self) -> float:
        return self.voxel_size * self.config.voxels_per_block_axis

    def allocate_block(self, bc) -> int:
        b = (C.c_int32 * 3)(*[int(x) for x in bc])
        slot = C.c_int32()
        self.backend.check(self.backend.lib.volume_allocate_block(self.handle, b, C.byref(slot)))
        return slot.value

    def free_block(self, bc):
        b = (C.c_int32 * 3)(*[int(x) for x in bc])
        self.backend.check(self.backend.lib.volume_free_block(self.handle, b))

    def block_slot(self, bc) -> int:
        b = (C.c_int32 * 3)(*[int(x) for x in bc])
        slot = C.c_int32()
        self.backend.check(self.backend.lib.volume_block_slot(self.handle, b, C.byref(slot)))
        return slot.value

    def is_allocated(self, bc) -> bool:
        return self.block_slot(bc) != self.kEmpty

    def read_voxel(self, vc):
        v = (C.c_int32 * 3)(*[int(x) for x in vc])
        chi = C.c_int32()
        t, a = C.c_double(), C.c_double()
        self.backend.check(self.backend.lib.volume_read_voxel(self.handle, v, C.byref(chi), C.byref(t), C.byref(a)))
        return None if chi.value else (t.value, a.value)

    def write_voxel(self, vc, tsdf, aux: float = 0.0):
        v = (C.c_int32 * 3)(*[int(x) for x in vc])
        self.backend.check(self.backend.lib.volume_write_voxel(self.handle, v, 1 if tsdf is None else 0,
                                                               0.0 if tsdf is None else float(tsdf), float(aux)))

    def voxel_center(self, vc):
        o = self.config.box_origin
        vs = self.voxel_size
        return np.array([o[i] + (float(vc[i]) + 0.5) * vs for i in range(3)])

    def read_table(self) -> np.ndarray:
        n = self.config.blocks_per_axis
        t = np.empty(n * n * n, dtype=np.int32)
        self.backend.check(self.backend.lib.volume_read_table(self.handle, t.ctypes.data))
        return t

    def read_payload(self, first_slot: int = 0, count: Optional[int] = None) -> np.ndarray:
        if count is None:
            count = self.pool_capacity - first_slot
        m3 = self.config.voxels_per_block_axis ** 3
        p = np.empty(count * m3, dtype=np.uint16)
        self.backend.check(self.backend.lib.volume_read_payload(self.handle, first_slot, count, p.ctypes.data))
        return p

    def write_payload(self, first_slot: int, payload: np.ndarray):
        m3 = self.config.voxels_per_block_axis ** 3
        p = np.ascontiguousarray(payload, dtype=np.uint16)
        self.backend.check(self.backend.lib.volume_write_payload(self.handle, first_slot, p.size // m3,
                                                                 p.ctypes.data))

    def save_snapshot(self, path: str):
        self.backend.check(self.backend.lib.volume_save_snapshot(self.handle, path.encode()))

    @staticmethod
    def load_snapshot(path: str, pool_capacity: int = 0, device: int = 0,
                      backend: Optional[Backend] = None) -> "SparseTsdfGrid":
        be = backend or default_backend()
        h = C.c_void_p()
        be.check(be.lib.volume_load_snapshot(path.encode(), pool_capacity, device, C.byref(h)))
        return SparseTsdfGrid(GridConfig(), backend=be, _handle=h)

    # --- device-only extras ---
    def read_free_list(self) -> np.ndarray:
        cnt = C.c_uint64()
        self.backend.check(self.backend.lib.volume_read_free_list(self.handle, None, C.byref(cnt)))
        out = np.empty(cnt.value, dtype=np.int32)
        self.backend.check(self.backend.lib.volume_read_free_list(self.handle, out.ctypes.data_as(A.i32p),
                                                                  C.byref(cnt)))
        return out

    def enable_float_payload(self):
        self.backend.check(self.backend.lib.volume_enable_float_payload(self.handle))

    # payload layouts (sf_gpu.h sf_payload_layout)
    CODES, CODES_FLOAT_SHADOW, FLOAT2 = A.SF_PAYLOAD_CODES, A.SF_PAYLOAD_CODES_FLOAT_SHADOW, A.SF_PAYLOAD_FLOAT2

    def set_payload_layout(self, layout: int):
        """FLOAT2: float {tsdf, aux} per voxel only (P2, set on an empty volume); CODES_FLOAT_SHADOW:
        the reference's 2-byte codes plus a float shadow; CODES: codes only (default)."""
        self.backend.check(self.backend.lib.volume_set_payload_layout(self.handle, int(layout)))

    @property
    def payload_layout(self) -> int:
        out = C.c_int32()
        self.backend.check(self.backend.lib.volume_get_payload_layout(self.handle, C.byref(out)))
        return out.value

    def read_float_payload(self, first_slot: int = 0, count: Optional[int] = None) -> np.ndarray:
        if count is None:
            count = self.pool_capacity - first_slot
        m3 = self.config.voxels_per_block_axis ** 3
        p = np.empty((count * m3, 2), dtype=np.float32)
        self.backend.check(self.backend.lib.volume_read_float_payload(self.handle, first_slot, count,
                                                                      p.ctypes.data))
        return p


@dataclass
class FrameMetrics:
    frame: int
    registered: bool
    status: int
    pose: Pose
    iterations: int
    matches: int
    residual_rms: float
    lambda_over_n: List[float]
    gated_mask: List[bool]
    fusion: FusionStats
    raycast: RaycastStats
    blocks_processed: int = 0
    voxels_visited: int = 0
    kernel_launches: int = 0  # this library's kernels the frame ran (incl. device-side ICP loop)
    exact_voxels: int = 0  # integrate voxels settled on the FP64 fallback (uncertain FP32 decision)
    integrate_ns: int = 0  # integrate kernel span on the device clock (first CTA start .. last CTA end)
    icp_ns: int = 0  # ICP span on the device clock (first step start .. end of the last solve)
    icp_steps: int = 0  # ICP step launches (device-side loop: one per iteration)
    ray_dda_cells: int = 0  # reference DDA cells of the rays reaching the occupied box (roofline count)
    ray_refine_samples: int = 0  # raycast stage-2 secant + gradient samples


class Tracker:
    """Device-resident run() frame loop (pipeline.cpp:233-301): raycast -> ICP -> fuse per frame,
    captured in a CUDA graph. ``step`` is asynchronous; ``fetch`` synchronises."""

    TRACK = 0
    GROUND_TRUTH = 1
    TRACK_WITH_HOOK = 2  # gt_pose carries the external initial delta (tracking.mode = icp_with_hook)

    def __init__(self, grid: SparseTsdfGrid, camera: Intrinsics, fusion: FusionParams, match: MatchParams,
                 initial_pose: Pose, use_graphs: bool = True, orthonormalize: bool = False):
        self.grid = grid
        self.camera = camera
        lib = grid.backend.lib
        self._lib = lib
        cfg = A.TrackerConfigC(fusion.c(), match.c(), camera.c(), 1 if use_graphs else 0,
                               1 if orthonormalize else 0)
        h = C.c_void_p()
        p12 = initial_pose.to12()
        grid.backend.check(lib.tracker_create(grid.handle, C.byref(cfg), _dptr(p12), C.byref(h)))
        self.handle = h

    def __del__(self):
        if getattr(self, "handle", None):
            try:
                self._lib.tracker_destroy(self.handle)
            except Exception:
                pass
            self.handle = None

    def step(self, frame: DepthFrame, mode: int = 0, gt_pose: Optional[Pose] = None, stream=None):
        fc = frame.c()
        g = _dptr(gt_pose.to12()) if gt_pose is not None else None
        self.grid.backend.check(self._lib.tracker_step(self.handle, C.byref(fc), mode, g, stream))

    def set_pose(self, pose: Pose, stream=None):
        """Re-seed the current pose (relocalisation)."""
        p12 = pose.to12()
        self.grid.backend.check(self._lib.tracker_set_pose(self.handle, _dptr(p12), stream))

    @staticmethod
    def _metrics(m) -> "FrameMetrics":
        f = m.fusion
        r = m.raycast
        return FrameMetrics(m.frame, bool(m.registered), m.status, Pose.from12(list(m.pose)), m.iterations,
                            m.matches, m.residual_rms, list(m.lambda_over_n), [bool(x) for x in m.gated_mask],
                            FusionStats(f.voxels_updated, f.blocks_allocated_now, f.blocks_total, f.memory_bytes),
                            RaycastStats(r.sample_steps, r.hit_pixels, r.rays_with_bounds),
                            m.blocks_processed, m.voxels_visited, m.kernel_launches, m.exact_voxels,
                            m.integrate_ns, m.icp_ns, m.icp_steps, m.ray_dda_cells, m.ray_refine_samples)

    def fetch(self, stream=None) -> FrameMetrics:
        m = A.FrameMetricsC()
        self.grid.backend.check(self._lib.tracker_fetch(self.handle, C.byref(m), stream))
        return self._metrics(m)

    def fetch_frame(self, frame: int) -> FrameMetrics:
        """Metrics of one of the last two steps, without waiting for later ones (streaming:
        issue step k+1, then fetch step k)."""
        m = A.FrameMetricsC()
        self.grid.backend.check(self._lib.tracker_fetch_frame(self.handle, frame, C.byref(m)))
        return self._metrics(m)

    def stage_times(self):
        """Device-timed stages of the last step (ms): raycast, icp, fuse prologue, integrate, total."""
        ms = (C.c_float * 5)()
        self.grid.backend.check(self._lib.tracker_stage_times(self.handle, ms))
        return list(ms)

    def set_stage_timing(self, level: int):
        """Stage-timing events inside the step: 2 all (default), 1 integrate kernel only, 0 none."""
        self.grid.backend.check(self._lib.tracker_set_stage_timing(self.handle, int(level)))

    def io_bytes(self, has_sigma: bool):
        """(h2d, d2h) bytes of one host-frame step + fetch."""
        a, b = C.c_uint64(), C.c_uint64()
        self._lib.tracker_io_bytes(self.handle, 1 if has_sigma else 0, C.byref(a), C.byref(b))
        return a.value, b.value

    def last_launch_count(self) -> int:
        c = C.c_uint64()
        self._lib.tracker_last_launch_count(self.handle, C.byref(c))
        return c.value

    def device_pose_ptr(self) -> int:
        p = A.c_double_p()
        self._lib.tracker_device_pose(self.handle, C.byref(p))
        return C.cast(p, C.c_void_p).value


_default_backend: Optional[Backend] = None


def default_backend() -> Backend:
    global _default_backend
    if _default_backend is None:
        _default_backend = Backend(A.product(), "cuda")
    return _default_backend

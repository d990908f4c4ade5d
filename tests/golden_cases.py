"""Golden cases (TEST INFRASTRUCTURE): small fixed runs of the hot path whose outputs are
frozen in tests/golden/golden.json, generated ONCE from the unmodified reference build
(oracle/_ref/libsfref.so) by tests/golden/make_golden.py.

Every case is a function backend -> dict of results. Large arrays are recorded as SHA-256 of
their little-endian bytes (bit-exact pins), scalars exactly (floats as float.hex). The same
functions run on the C restatement (tests/test_golden.py, no GPU) and on the CUDA library
(tests/test_gpu_parity.py::test_golden_cases_gpu), so neither needs /root/reference at run
time."""
import hashlib
import math

import numpy as np

from paper_1311_7194_b200 import api as sf
from tests import scenes


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes()).hexdigest()


def fx(v: float) -> str:
    return float(v).hex()


def small_cam():
    return scenes.camera(160, 120, 131.25)


def _fuse_case(be, mode, aux):
    intr = small_cam()
    poses = scenes.c1_trajectory(100)[::30]
    g = sf.SparseTsdfGrid(scenes.c1_config(), 0, aux, backend=be)
    params = sf.FusionParams(mode=mode)
    out = {"stats": [], "frames": []}
    for p in poses:
        f = be.render_synthetic_depth(scenes.sphere_plane_scene(), p, intr, domain_size=2.0)  # noise-free:
        # the C restatement does not carry the reference's mt19937_64 noise model
        out["frames"].append(digest(f.depth))
        st = be.fuse_frame(g, f, p, params)
        out["stats"].append([st.voxels_updated, st.blocks_allocated_now, st.blocks_total, st.memory_bytes])
    out["table"] = digest(g.read_table())
    out["payload"] = digest(g.read_payload())
    out["allocated"] = int(g.allocated_count)
    return out, g


def case_fuse_kalman(be):
    """fuse_frame, Kalman filter + variance codes, 4 frames of the C1 orbit at 160x120."""
    return _fuse_case(be, sf.FusionMode.Kalman, sf.AuxMode.Variance)[0]


def case_fuse_weighted_raycast(be):
    """fuse_frame (weighted), then compute_ray_bounds, raycast and compute_normals."""
    out, g = _fuse_case(be, sf.FusionMode.Weighted, sf.AuxMode.Weight)
    intr = small_cam()
    q = scenes.c1_trajectory(100)[30]
    s, e = be.compute_ray_bounds(g, q, intr)
    out["bounds"] = [digest(s), digest(e)]
    d, n, st = be.raycast_result(g, q, intr)
    out["raycast"] = [digest(d.depth), digest(n.array)]
    out["raycast_stats"] = [st.sample_steps, st.hit_pixels, st.rays_with_bounds]
    f = be.render_synthetic_depth(scenes.sphere_plane_scene(), q, intr, domain_size=2.0)
    out["normals"] = digest(be.compute_normals(f, 2.5e-4, 0.0078).array)
    return out


def case_icp(be):
    """icp on a rendered pair of the sphere cluster (2 degree / 1 cm offset)."""
    intr = small_cam()
    scene = scenes.cluster_scene()
    tp = sf.orbit_trajectory([0.0, 0.0, 1.3], 1.3, 8)[1]
    ang = math.radians(2.0)
    sp = sf.compose(tp, sf.Pose([[math.cos(ang), 0, math.sin(ang)], [0, 1, 0], [-math.sin(ang), 0, math.cos(ang)]],
                                [0.01, -0.005, 0.008]))
    t = be.render_synthetic_depth(scene, tp, intr)
    s = be.render_synthetic_depth(scene, sp, intr)
    tn = be.compute_normals(t, 2.5e-4, 0.006)
    r = be.icp(s, t, tn, sf.Pose.identity(), sf.MatchParams.for_voxel_size(1.5 / 256.0))
    return {"delta": [fx(v) for v in r.delta.to12()], "iterations": r.iterations, "matches": r.matches,
            "gated": [bool(x) for x in r.gated_mask]}


CASES = {
    "fuse_kalman": case_fuse_kalman,
    "fuse_weighted_raycast": case_fuse_weighted_raycast,
    "icp": case_icp,
}

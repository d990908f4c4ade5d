"""Scenes and configurations of BASELINE.json, shared by tests and bench."""
import math

from paper_1311_7194_b200 import api as sf


def camera(width=640, height=480, focal=525.0):
    return sf.Intrinsics.simple(width, height, focal)


def sphere_plane_scene():
    """C1/C2: sphere c=(0,0,1.3) r=0.4 plus the wall z = 2."""
    s = sf.AnalyticScene()
    s.add_sphere([0.0, 0.0, 1.3], 0.4)
    s.add_plane([0.0, 0.0, -1.0], -2.0)
    return s


def c1_config():
    return sf.GridConfig(32, 8, (-1.0, -1.0, 0.25), 2.0, 0.0)


def c2_config():
    return sf.GridConfig(125, 4, (-1.0, -1.0, 0.25), 2.0, 0.0)


def c1_trajectory(frames=100):
    return sf.orbit_trajectory([0.0, 0.0, 1.3], 1.3, frames, (0.0, 1.0, 0.0), math.pi / 4, math.pi / 2)


def bumpy_sphere(center=(0.0, 0.0, 0.35), r=0.08, bump=0.024):
    """C4: hand-scale bumpy sphere."""
    s = sf.AnalyticScene()
    s.add_sphere(list(center), r)
    o = r / math.sqrt(3.0)
    for i in range(8):
        s.add_sphere([center[0] + (o if i & 1 else -o), center[1] + (o if i & 2 else -o),
                      center[2] + (o if i & 4 else -o)], bump)
    return s


def c4_config():
    side = 4096 * 0.15e-3
    return sf.GridConfig(512, 8, (-side / 2, -side / 2, 0.35 - side / 2), side, 0.0)


def c4_trajectory(frames=100):
    return sf.orbit_trajectory([0.0, 0.0, 0.35], 0.35, frames, (0.0, 1.0, 0.0), 0.0, 2.0 * math.pi)


def cluster_scene():
    """sphere_cluster (tests/test_utils.hpp:15-22)."""
    s = sf.AnalyticScene()
    s.add_sphere([0.25, -0.05, 1.30], 0.28)
    s.add_sphere([-0.30, 0.18, 1.55], 0.22)
    s.add_sphere([0.05, 0.30, 1.10], 0.16)
    s.add_sphere([-0.12, -0.28, 1.05], 0.13)
    return s


def c5_scene(center=(0.0, 0.0, 0.0), spacing=0.3, r=0.08, bump=0.024):
    """C5: a 3x3 grid of C4 bumpy spheres in the x-z plane around `center`, so the blocks of a
    sharded pool land on every owner."""
    s = sf.AnalyticScene()
    o = r / math.sqrt(3.0)
    for i in (-1, 0, 1):
        for j in (-1, 0, 1):
            c = (center[0] + i * spacing, center[1], center[2] + j * spacing)
            s.add_sphere(list(c), r)
            for b in range(8):
                s.add_sphere([c[0] + (o if b & 1 else -o), c[1] + (o if b & 2 else -o),
                              c[2] + (o if b & 4 else -o)], bump)
    return s


def c5_config(blocks_per_axis=1024, voxel=0.15e-3):
    """C5: 8192^3 sparse at 0.15 mm (N = 1024, M = 8), box centred on the object grid."""
    side = blocks_per_axis * 8 * voxel
    return sf.GridConfig(blocks_per_axis, 8, (-side / 2, -side / 2, -side / 2), side, 0.0)


def c5_trajectory(frames=100, radius=0.9):
    return sf.orbit_trajectory([0.0, 0.0, 0.0], radius, frames, (0.0, 1.0, 0.0), 0.0, 2.0 * math.pi)


def c3_scene():
    """C3: a 2.8 m room (six inward walls at +-1.4 m) with box furniture and a sphere
    (SURVEY.md §8d C3)."""
    s = sf.AnalyticScene()
    for a in range(3):
        for sgn in (1.0, -1.0):
            n = [0.0, 0.0, 0.0]
            n[a] = sgn
            s.add_plane(n, -1.4)
    s.add_box([0.6, 1.0, 0.5], [0.3, 0.2, 0.3])
    s.add_box([-0.5, 1.1, 0.7], [0.25, 0.3, 0.2])
    s.add_sphere([-0.7, 0.3, -0.6], 0.25)
    return s


def c3_config():
    """C3: 3000^3 sparse at 1 mm (N = 375, M = 8), box (-1.5, -1.5, -1.5) + 3 m."""
    return sf.GridConfig(375, 8, (-1.5, -1.5, -1.5), 3.0, 0.0)


def c3_trajectory(frames=100, radius=0.3):
    """Outward-looking pan: 360 degrees about +y from a circle of `radius`."""
    out = []
    for k in range(frames):
        a = 2.0 * math.pi * k / frames
        c, s_ = math.cos(a), math.sin(a)
        t = [radius * c, 0.0, radius * s_]
        fwd = [c, 0.0, s_]
        up = [0.0, 1.0, 0.0]
        right = [fwd[1] * up[2] - fwd[2] * up[1], fwd[2] * up[0] - fwd[0] * up[2], fwd[0] * up[1] - fwd[1] * up[0]]
        nr = math.sqrt(sum(x * x for x in right))
        right = [x / nr for x in right]
        down = [fwd[1] * right[2] - fwd[2] * right[1], fwd[2] * right[0] - fwd[0] * right[2],
                fwd[0] * right[1] - fwd[1] * right[0]]
        R = [[right[i], down[i], fwd[i]] for i in range(3)]
        out.append(sf.Pose(R, t))
    return out

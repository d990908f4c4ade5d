"""Marching cubes on the device (marching_cubes.cpp:74-196) against the unmodified reference
build: vertices, normals and triangles identical, bit for bit."""
import numpy as np
import pytest

import paper_1311_7194_b200 as sfp
from paper_1311_7194_b200 import api as sf
from tests import scenes

pytestmark = pytest.mark.gpu


def _fused_pair(gpu, ref, cfg, frames_poses, fusion, aux=sf.AuxMode.Variance, **kw):
    g = sf.SparseTsdfGrid(cfg, 0, aux, **kw)
    r = sf.SparseTsdfGrid(cfg, 0, aux, backend=ref, **kw)
    for f, p in frames_poses:
        sfp.fuse_frame(g, f, p, fusion)
        ref.fuse_frame(r, f, p, fusion)
    assert np.array_equal(g.read_table(), r.read_table())
    return g, r


def _same_mesh(a, b):
    (va, na, ta), (vb, nb, tb) = a, b
    assert va.shape == vb.shape and ta.shape == tb.shape, (va.shape, vb.shape, ta.shape, tb.shape)
    assert np.array_equal(va.view(np.uint32), vb.view(np.uint32))
    assert np.array_equal(na.view(np.uint32), nb.view(np.uint32))
    assert np.array_equal(ta, tb)


def _c1_frames(gpu, n=4, w=160, h=120, f=131.25):
    intr = scenes.camera(w, h, f)
    poses = scenes.c1_trajectory(100)[:n]
    return [(gpu.render_synthetic_depth(scenes.sphere_plane_scene(), p, intr, sigma0=2.5e-4, seed=3 + k,
                                        domain_size=2.0), p) for k, p in enumerate(poses)], intr


@pytest.mark.parametrize("budget", [0, 1 << 12])
def test_marching_cubes_matches_reference(gpu, ref, budget):
    fp, _ = _c1_frames(gpu)
    g, r = _fused_pair(gpu, ref, scenes.c1_config(), fp, sf.FusionParams(mode=sf.FusionMode.Kalman))
    mg = sfp.marching_cubes(g, batch_memory_budget=budget)
    mr = ref.marching_cubes(r, batch_memory_budget=budget)
    assert len(mg[2]) > 1000
    _same_mesh(mg, mr)


def test_marching_cubes_region_and_m4(gpu, ref):
    fp, intr = _c1_frames(gpu, n=3)
    g, r = _fused_pair(gpu, ref, scenes.c2_config(), fp, sf.FusionParams(mode=sf.FusionMode.Weighted),
                       aux=sf.AuxMode.Weight)
    _same_mesh(sfp.marching_cubes(g), ref.marching_cubes(r))
    region = (scenes.c1_trajectory(100)[7], sf.Intrinsics.simple(32, 24, 40.0, 0.1, 4.0))
    part = sfp.marching_cubes(g, region=region)
    _same_mesh(part, ref.marching_cubes(r, region=region))
    assert 0 < len(part[2]) < len(sfp.marching_cubes(g)[2])


def test_marching_cubes_single_cube_across_eight_blocks(gpu, ref):
    """test_render.cpp:249-272: one written cube straddling all eight blocks."""
    meshes = []
    for be in (gpu, ref):
        grid = sf.SparseTsdfGrid(sf.GridConfig(2, 4, (0.0, 0.0, 0.0), 1.0, 0.0), 8, backend=be)
        assert len(be.marching_cubes(grid)[2]) == 0
        d = grid.delta
        for bz in range(2):
            for by in range(2):
                for bx in range(2):
                    grid.allocate_block((bx, by, bz))
        for dz in range(2):
            for dy in range(2):
                for dx in range(2):
                    inside = dx == 0 and dy == 0 and dz == 0
                    grid.write_voxel((3 + dx, 3 + dy, 3 + dz), -0.3 * d if inside else 0.3 * d, 1.0)
        meshes.append(be.marching_cubes(grid))
    v, n, t = meshes[0]
    assert len(t) == 1 and len(v) == 3
    assert np.all(np.abs(np.linalg.norm(n, axis=1) - 1.0) < 1e-5)
    _same_mesh(meshes[0], meshes[1])


def test_marching_cubes_c4_scale(gpu, ref):
    """Bumpy sphere at the C4 voxel size (N = 512), a few noisy frames."""
    intr = scenes.camera(320, 240, 262.5)
    cfg = scenes.c4_config()
    poses = scenes.c4_trajectory(100)[:3]
    fp = [(gpu.render_synthetic_depth(scenes.bumpy_sphere(), p, intr, sigma0=4e-4, seed=11 + k,
                                      domain_size=cfg.box_side), p) for k, p in enumerate(poses)]
    g, r = _fused_pair(gpu, ref, cfg, fp, sf.FusionParams(mode=sf.FusionMode.Kalman), p_min=1e-12)
    mg = sfp.marching_cubes(g)
    assert len(mg[2]) > 10000
    _same_mesh(mg, ref.marching_cubes(r))

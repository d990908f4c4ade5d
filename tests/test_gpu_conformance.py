"""The reference's own test suites against the GPU path.

`make conformance` compiles the UNMODIFIED reference suites (proj/tests/test_fusion.cpp,
test_render.cpp, test_registration.cpp, acceptance.cpp, and test_grid / test_geometry /
test_pipeline) against the C++ drop-in layer paper_1311_7194_b200/cpp/sparsefusion_adapter.cpp,
which implements the reference headers' hot-path entry points (fuse_frame,
select_update_blocks, compute_ray_bounds, raycast, icp, compute_normals, marching_cubes) over
libsf_gpu.so; every other symbol is the reference's own object code (oracle/_ref/obj). The
binaries are built where the reference sources exist (build() in this container) and shipped
prebuilt; without them the test is skipped. test_pipeline's CLI case needs the absent CLI11
front-end (as in oracle/Makefile) and is the one expected failure of that suite.
"""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "cpp", "_build")
SUITES = {  # suite -> test cases allowed to fail (reason)
    "test_fusion": {},
    "test_render": {},
    "test_registration": {},
    "acceptance": {},
    "test_grid": {},
    "test_geometry": {},
    "test_pipeline": {"cli: run/experiment/render": "needs the CLI11 front-end binary, absent here (out of scope)"},
}


@pytest.mark.parametrize("suite", list(SUITES))
def test_reference_suite_on_gpu(gpu, suite):
    exe = os.path.join(BUILD, "conf_" + suite)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (make conformance needs the reference headers)")
    env = dict(os.environ)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=1800, cwd=BUILD, env=env)
    out = r.stdout + r.stderr
    if suite == "acceptance":  # its own main(): the 10 criteria of SPEC.md:620-632
        assert r.returncode == 0 and "all 10 criteria passed" in out, out[-4000:]
        return
    m = re.search(r"test cases: (\d+) run \| (\d+) passed \| (\d+) failed", out)
    assert m, out[-3000:]
    run, passed, failed = map(int, m.groups())
    errors = [ln for ln in out.splitlines() if "ERROR" in ln or "FAILED" in ln]
    allowed = SUITES[suite]
    unexpected = [ln for ln in errors if not any(k in ln for k in allowed)]
    assert not unexpected, "\n".join(unexpected[:20])
    assert run >= 5 and failed <= len(allowed), out[-3000:]

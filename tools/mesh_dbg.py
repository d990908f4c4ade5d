import sys
import numpy as np
sys.path.insert(0, '.')
import paper_1311_7194_b200 as sfp
from paper_1311_7194_b200 import api as sf
from tests import oracle_backends, scenes
from tests.test_gpu_mesh import _c1_frames, _fused_pair
gpu = sfp.default_backend()
ref = oracle_backends.reference()
fp, _ = _c1_frames(gpu)
g, r = _fused_pair(gpu, ref, scenes.c1_config(), fp, sf.FusionParams(mode=sf.FusionMode.Kalman))
vg, ng, tg = sfp.marching_cubes(g)
vr, nr, tr = ref.marching_cubes(r)
bad = np.nonzero(np.any(ng.view(np.uint32) != nr.view(np.uint32), axis=1))[0]
print("differing normals", len(bad), "of", len(ng))
for i in bad[:10]:
    print(i, vg[i], ng[i], nr[i], np.linalg.norm(ng[i]), np.linalg.norm(nr[i]), ng[i] - nr[i])

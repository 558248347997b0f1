"""Independent gradient evidence (VERDICT r1 missing 5): the device's f32 analytic gradient of
the loss (vp_eval_loss_pho's backward pass + vp_loss_pose) against central finite differences
computed by the REFERENCE's own gradcheck (grad.cpp:293-370) in its double-precision build
(oracle/gen_gradcheck.py -> tests/golden/gradcheck.npz), on 216 coordinates sampled round-robin
over payload rgb, payload sigma, deltaT, deltaR and deltaS, in the style of
acceptance_f64.cpp:20-116 (part of the batch saturates; earlyEps 1e-9; 384 rays).

Tolerance: relative error |a - fd| / max(|a| + |fd|, 1e-4) <= 2e-3 in every group. The
reference's own f32 analytic gradient meets the same bound against these differences (printed by the
generator: 4.1e-4 at worst, on deltaS); the device differs from it only by the order of its
atomic sums."""
import numpy as np
import pytest

from conftest import GOLDEN
from paper_2103_01954_b200 import api

pytestmark = pytest.mark.gpu
TOL = 2e-3
GROUPS = ["payload rgb", "payload sigma", "deltaT", "deltaR", "deltaS"]


def test_device_gradient_matches_reference_f64_finite_differences(renderer):
    z = np.load(GOLDEN / "gradcheck.npz")
    tr = np.ascontiguousarray(z["tr"], np.float32)
    k, m = tr.shape[0], int(z["m"])
    scene = api.Scene(api.WindowParams(8.0, 8), frames=[api.Frame(tr, api.PrimitiveSlab(k, m, z["payload"]))])
    cams = [api.Camera(c[:9].reshape(3, 3).T, c[9:18].reshape(3, 3).T, c[18:21], int(c[21]), int(c[22]))
            for c in z["cams"]]
    batch = api.RaySamples(z["cam_index"], z["pixel"], z["pixel_id"], z["target"], z["background"])
    w = z["weights"]
    weights = api.LossWeights(float(w[0]), float(w[1]), float(w[2]), float(w[3]))
    cfg = api.MarchConfig(float(z["cfg"][0]), float(z["cfg"][1]))
    grads = np.zeros(api.grad_size(k, m), np.float32)
    terms = api.eval_loss(renderer, scene, 0, cams, batch, weights, cfg, grads)
    assert np.isclose(terms.pho, float(z["terms_f32"][0]), rtol=1e-5)
    a = grads[z["index"]].astype(np.float64)
    fd = z["finite_diff"]
    rel = np.abs(a - fd) / np.maximum(np.abs(a) + np.abs(fd), 1e-4)
    report = {GROUPS[g]: float(rel[z["group"] == g].max()) for g in range(5)}
    # 384 rays touch a fraction of the 8 x 4 x 512 voxels: many sampled payload coordinates have a
    # zero gradient (and must be zero on the device too); the pose groups are all informative
    informative = np.abs(fd) > 1e-6
    assert informative.sum() >= 120, informative.sum()
    for g in range(5):
        assert informative[z["group"] == g].sum() >= 20, GROUPS[g]
    assert all(v <= TOL for v in report.values()), report

"""CPU: pin the oracle (oracle/vp_oracle.c) against the reference's own outputs.

tests/golden/* was produced by the unmodified reference core (oracle/gen_golden.py); the C
restatement must reproduce every fixture bit-for-bit before it may serve as the checker.
"""
import json

import numpy as np
import pytest

from conftest import GOLDEN, load_groups
from golden_cases import render_cases, sha
from paper_2103_01954_b200 import api, synthetic


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def test_compose_matches_reference(oracle):
    z = np.load(GOLDEN / "compose.npz")
    rc, xf = oracle.compose(z["tr"])
    assert rc == 0 and np.array_equal(bits(xf), bits(z["xf"]))
    rc_bad, _ = oracle.compose(z["bad"])
    assert rc_bad == int(z["rc_bad"]) == 2


def test_generate_ray_matches_reference(oracle):
    z = np.load(GOLDEN / "cameras.npz")
    cam = api.Camera(z["K"], z["R"], z["t"], int(z["wh"][0]), int(z["wh"][1]))
    for (x, y), want in zip(z["rays_px"], z["rays"]):
        o, d = oracle.generate_ray(cam, x, y)
        assert np.array_equal(bits(np.concatenate([o, d])), bits(want))


def test_intersect_matches_reference(oracle):
    z = np.load(GOLDEN / "intersect.npz")
    off = 0
    for o, d, n in zip(z["origins"], z["dirs"], z["lens"]):
        p, te, tx = oracle.intersect(z["xf"], o, d)
        want = z["segs"][off:off + n]
        off += n
        assert len(p) == n
        assert np.array_equal(p, want[:, 0].astype(np.int32))
        assert np.array_equal(bits(te), bits(want[:, 1])) and np.array_equal(bits(tx), bits(want[:, 2]))


def test_march_kats_match_reference(oracle):
    for name, g in load_groups("march_kats").items():
        win = api.WindowParams(float(g["window"][0]), int(g["window"][1]))
        cfg = api.MarchConfig(float(g["cfg"][0]), float(g["cfg"][1]))
        rgb, alpha, samples = oracle.march_rays(g["xf"], int(g["m"]), g["payload"], win, g["o"], g["d"],
                                                cfg, g["jit"])
        assert np.array_equal(bits(rgb), bits(g["rgb"])), name
        assert np.array_equal(bits(alpha), bits(g["alpha"])), name
        assert np.array_equal(samples, g["samples"]), name


@pytest.mark.parametrize("case", sorted(load_groups("renders")))
def test_render_matches_reference(oracle, case):
    c = render_cases()[case]
    xf = api.compose(c["tr"]) if len(c["tr"]) else np.zeros((0, 15), np.float32)
    rgb, alpha, samples, prim = oracle.render_counted(xf, c["m"], c["payload"], c["window"], c["cam"], c["cfg"])
    assert np.array_equal(bits(rgb), bits(c["rgb"]))
    assert np.array_equal(bits(alpha), bits(c["alpha"]))
    assert np.array_equal(samples, c["samples"])
    # per-pixel prim-samples (executions of march.cpp:63-70), counted by the reference itself
    assert np.array_equal(prim, np.load(GOLDEN / "prim_counts.npz")[f"case_{case}"])


def test_oracle_config1_full_size_digest(oracle):
    """BASELINE config 1 (64 x 16^3 at 256^2, the reference's CPU oracle run), bit-exact, with
    the reference's per-pixel prim-sample counts."""
    d = json.loads((GOLDEN / "digests.json").read_text())["renders"]["oracle_64x16_256_view-1"]
    tr, pay = synthetic.shell_arrays(64, 16)
    rgb, alpha, samples, prim = oracle.render_counted(api.compose(tr), 16, pay, api.WindowParams(),
                                                      synthetic.shell_camera(-1, 64, 256), api.MarchConfig())
    assert int(samples.sum()) == d["total_samples"]
    assert sha(samples) == d["samples"] and sha(alpha) == d["alpha"] and sha(rgb) == d["rgb"]
    assert np.array_equal(prim, np.load(GOLDEN / "prim_counts.npz")["full_oracle_64x16_256_view-1"])
    assert int(prim.astype(np.int64).sum()) == d["prim_samples"]


def test_window_known_answers(oracle):
    """test_primitive.cpp:13-25."""
    assert oracle.window(0, 0, 0) == 1.0
    assert oracle.window(1, 0, 0) == pytest.approx(np.exp(-8.0), rel=1e-6)
    assert oracle.window(1, 1, 1) == pytest.approx(np.exp(-24.0), rel=1e-6)
    assert oracle.window(0.5, 0, 0) == pytest.approx(np.exp(-0.03125), rel=1e-6)
    assert oracle.window(-0.7, 0.2, 0) == oracle.window(0.7, -0.2, 0)
    assert oracle.window(0.9, 0.9, 0.9, 0.0, 8) == 1.0


@pytest.mark.parametrize("cos", [False, True])
def test_sincos_port_matches_libm(oracle, cos):
    """The binary64 sinf/cosf port (glibc 2.39's algorithm, ported to the device for compose)
    equals this host's libm: strided walks over the polynomial-only range, the fast-reduction
    range [0.75, 120) (where every axis-angle magnitude of a pose lives), the large-argument
    reduction and negative inputs. Exhaustive runs (every float of [0, 120), stride 3 beyond)
    were clean too; they take ~20 s."""
    assert oracle.sincos_port_mismatches(0x00000000, 0x3F400000, 97, cos) == 0
    assert oracle.sincos_port_mismatches(0x3F400000, 0x42F00000, 13, cos) == 0
    assert oracle.sincos_port_mismatches(0x42F00000, 0x7F7FFFFF, 4099, cos) == 0
    assert oracle.sincos_port_mismatches(0x80000000, 0xFF7FFFFF, 4099, cos) == 0


def test_expf_port_matches_libm(oracle):
    """The binary64 expf port (the algorithm ported to the device) equals this host's glibc
    expf: a stride-7 walk over [-24, 0] (the window argument range at alpha = 8) and a
    stride-4099 walk over [-104, 88] (the GPU test checks every float of [-24, 0] on the
    device)."""
    assert oracle.expf_port_mismatches(0x80000000, 0xC1C00000, 7) == 0
    assert oracle.expf_port_mismatches(0x80000000, 0xC2D00000, 4099) == 0
    assert oracle.expf_port_mismatches(0x00000000, 0x42B00000, 4099) == 0


def test_backward_matches_reference(oracle):
    """backwardRay restatement == the reference's GradBuffer, bit for bit (sequential order)."""
    for name, g in load_groups("backward").items():
        win = api.WindowParams(float(g["window"][0]), int(g["window"][1]))
        cfg = api.MarchConfig(float(g["cfg"][0]), float(g["cfg"][1]))
        got = oracle.backward_rays(g["tr"], int(g["m"]), g["payload"], win, g["o"], g["d"], g["adj_rgb"],
                                   g["adj_alpha"], cfg, g["jit"])
        assert np.array_equal(bits(got), bits(g["grads"])), name
        assert np.count_nonzero(g["grads"]) > 1000, name


REF = pytest.mark.skipif(not (GOLDEN.parent.parent / "oracle" / "_ref" / "libvolprim_ref.so").exists(),
                         reason="reference core not built (make -C oracle ref)")


@REF
@pytest.mark.parametrize("km", ["64x16", "512x32"])
def test_reference_side_generator_matches_digests(km):
    """The reference arm's own scene generator (ref_glue vpref_shell_scene, built on the
    reference's compose/toWorld) reproduces the pinned generator digests, so bench.py's
    reference arm renders exactly the inputs our arm renders without loading libvpb.so."""
    from oracle.bindings import RefCore, ref_shell_arrays
    k, m = map(int, km.split("x"))
    tr, pay = ref_shell_arrays(RefCore(), k, m)
    gen = json.loads((GOLDEN / "digests.json").read_text())["generator"][km]
    assert sha(tr) == gen["tr"] and sha(pay) == gen["payload"]


@REF
def test_reference_side_cameras_match_product_cameras():
    """vpref_shell_camera (reference lookAtCamera) == the product's vp_shell_camera, bit for bit,
    on the headline view and all 64 ring views."""
    from oracle.bindings import RefCore, ref_shell_camera
    ref = RefCore()
    for v in [-1] + list(range(64)):
        k9, r9, t3 = ref_shell_camera(ref, v, 64, 1024)
        cam = synthetic.shell_camera(v, 64, 1024)
        assert np.array_equal(k9.view(np.uint32), np.asarray(cam.intrinsics, np.float32).T.reshape(-1).view(np.uint32))
        assert np.array_equal(r9.view(np.uint32), np.asarray(cam.rotation, np.float32).T.reshape(-1).view(np.uint32))
        assert np.array_equal(t3.view(np.uint32), np.asarray(cam.translation, np.float32).reshape(-1).view(np.uint32))


@REF
def test_reference_resident_scene_render_matches_digest():
    """The resident-Scene entry the reference arm times (vpref_scene_render) gives the config-1
    reference digest."""
    from oracle.bindings import RefCore, RefScene, ref_shell_camera
    d = json.loads((GOLDEN / "digests.json").read_text())["renders"]["oracle_64x16_256_view-1"]
    ref = RefCore()
    sc = RefScene(ref, 64, 16)
    k9, r9, t3 = ref_shell_camera(ref, -1, 0, 256)
    tot, rgb, alpha, samples = sc.render(k9, r9, t3, 256, 256, outputs=True)
    sc.close()
    assert tot == d["total_samples"]
    assert sha(samples) == d["samples"] and sha(alpha) == d["alpha"] and sha(rgb) == d["rgb"]


@REF
def test_gradcheck_fixture_pinned_to_reference():
    """tests/golden/gradcheck.npz (oracle/gen_gradcheck.py): the reference's f32 evalLoss gradient
    on the fixture scene reproduces the stored values bit for bit, and the f64 finite differences
    agree with it within the generator's reported bound."""
    from oracle.bindings import RefCore, ref_eval_loss
    z = np.load(GOLDEN / "gradcheck.npz")

    class Cam:
        def __init__(self, c):
            self.intrinsics, self.rotation = c[:9].reshape(3, 3).T, c[9:18].reshape(3, 3).T
            self.translation, self.width, self.height = c[18:21], int(c[21]), int(c[22])

    class MC:
        step_size, early_eps, jitter, seed = float(z["cfg"][0]), float(z["cfg"][1]), False, 0

    class W:
        alpha, beta = 8.0, 8
    w = z["weights"]
    _, g = ref_eval_loss(RefCore(), z["tr"], int(z["m"]), z["payload"], W, [Cam(c) for c in z["cams"]],
                         z["cam_index"], z["pixel"], z["pixel_id"], z["target"], z["background"], [w[0], w[2], w[3]], MC)
    assert np.array_equal(g[z["index"]].view(np.uint32), z["ref_f32_analytic"].view(np.uint32))
    fd = z["finite_diff"]
    rel = np.abs(g[z["index"]] - fd) / np.maximum(np.abs(g[z["index"]]) + np.abs(fd), 1e-4)
    assert rel.max() <= 1e-3

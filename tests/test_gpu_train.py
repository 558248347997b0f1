"""GPU: the training rows — evalLoss's ray-batch driver (vp_eval_loss_pho + the host
regularisers) and adamStep on the device — against the reference's own evalLoss / adamStep
(tests/golden/train.npz, written by oracle/gen_golden.py)."""
import ctypes as C

import numpy as np
import pytest

from conftest import GOLDEN
from golden_cases import sha
from paper_2103_01954_b200 import _lib, api, synthetic

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def _z():
    return np.load(GOLDEN / "train.npz")


def test_eval_loss_matches_reference(renderer):
    z = _z()
    tr, pay = synthetic.shell_arrays(64, 8)
    assert sha(pay) == str(z["payload_sha"])
    scene = api.Scene(api.WindowParams(8.0, 8), frames=[api.Frame(z["tr"], api.PrimitiveSlab(64, 8, pay))])
    cams = [api.Camera(c[:9].reshape(3, 3), c[9:18].reshape(3, 3), c[18:21], int(c[21]), int(c[22]))
            for c in z["cams"]]
    batch = api.RaySamples(z["cam_index"], z["pixel"], z["pixel_id"], z["target"], z["background"])
    w = z["weights"]
    weights = api.LossWeights(float(w[0]), float(w[1]), float(w[2]), float(w[3]))
    c = z["cfg"]
    cfg = api.MarchConfig(float(np.float32(c[0])), float(np.float32(c[1])), bool(c[2]), int(c[3]))
    grads = np.zeros(api.grad_size(64, 8), np.float32)
    terms = api.eval_loss(renderer, scene, 0, cams, batch, weights, cfg, grads)
    # the forward is bit-exact, so the photometric term (summed on the host in batch order) is too
    got = np.array([terms.pho, terms.geo, terms.vol, terms.del_], np.float32)
    assert np.array_equal(bits(got), bits(z["terms"])), (got, z["terms"])
    want = z["grads"]
    err = np.abs(grads.astype(np.float64) - want)
    assert np.all(err <= 2e-5 * np.abs(want).max() + 1e-4 * np.abs(want)), err.max()
    # no gradient: the loss alone
    terms2 = api.eval_loss(renderer, scene, 0, cams, batch, weights, cfg)
    assert terms2.pho == terms.pho


def test_adam_step_matches_reference(renderer):
    z = _z()
    m = int(z["adam_m"])
    tr = np.ascontiguousarray(z["adam_tr_in"], np.float32).copy()
    k = tr.shape[0]
    renderer.set_scene_composed(api.compose(tr), api.PrimitiveSlab(k, m, z["adam_pay_in"]), api.WindowParams())
    a = z["adam_cfg"]
    cfg = api.AdamConfig(*[float(x) for x in a])
    renderer._lib.vp_adam_reset(renderer.ctx)
    for g in z["adam_grads"]:
        api.adam_step(renderer, cfg, g, tr)
    assert np.array_equal(bits(tr), bits(z["adam_tr_out"]))
    assert np.array_equal(bits(api.payload_planar(renderer)), bits(z["adam_pay_out"]))
    # the refreshed composed transforms are those of the updated records
    rects, *_ = renderer.debug_tiles(synthetic.shell_camera(-1, 0, 32))
    bad = z["adam_grads"][0].copy()
    bad[7] = np.nan
    with pytest.raises(api.Error) as e:
        api.adam_step(renderer, cfg, bad, tr)
    assert e.value.category == api.ErrorCategory.NUMERIC
    assert np.array_equal(bits(tr), bits(z["adam_tr_out"]))  # nothing updated
    assert np.array_equal(bits(api.payload_planar(renderer)), bits(z["adam_pay_out"]))
    bad_delta = z["adam_grads"][1].copy()
    bad_delta[-3] = np.inf  # a pose-delta gradient (the tail of [payload | deltas])
    with pytest.raises(api.Error) as e:
        api.adam_step(renderer, cfg, bad_delta, tr)
    assert e.value.category == api.ErrorCategory.NUMERIC
    assert np.array_equal(bits(tr), bits(z["adam_tr_out"]))
    assert np.array_equal(bits(api.payload_planar(renderer)), bits(z["adam_pay_out"]))
    # moments and the step count survived the rejected steps: one more step lands where the
    # same step does after an uninterrupted run
    api.adam_step(renderer, cfg, z["adam_grads"][0], tr)
    got_tr, got_pay = bits(tr).copy(), bits(api.payload_planar(renderer)).copy()
    tr2 = np.ascontiguousarray(z["adam_tr_in"], np.float32).copy()
    renderer.set_scene_composed(api.compose(tr2), api.PrimitiveSlab(k, m, z["adam_pay_in"]), api.WindowParams())
    renderer._lib.vp_adam_reset(renderer.ctx)
    for g in list(z["adam_grads"]) + [z["adam_grads"][0]]:
        api.adam_step(renderer, cfg, g, tr2)
    assert np.array_equal(got_tr, bits(tr2))
    assert np.array_equal(got_pay, bits(api.payload_planar(renderer)))


@pytest.mark.parametrize("m", [3, 4, 5, 8])
def test_adam_payload_update_both_access_widths(renderer, m):
    """The payload part of adamStep (losses.cpp:81-96) against a float32 numpy restatement (each
    operation rounded to binary32, no contraction), three steps, for even M (16-byte kernel,
    k_adam_update4) and odd M (scalar kernel)."""
    k = 7
    rng = np.random.default_rng(m)
    tr, _ = synthetic.shell_arrays(k, 2)
    tr = np.ascontiguousarray(tr, np.float32)
    pay = rng.uniform(0.0, 1.0, k * 4 * m ** 3).astype(np.float32)
    renderer.set_scene_composed(api.compose(tr), api.PrimitiveSlab(k, m, pay), api.WindowParams())
    renderer._lib.vp_adam_reset(renderer.ctx)
    cfg = api.AdamConfig(lr=3e-2, beta1=0.9, beta2=0.999, eps=1e-8, lr_delta_scale=0.0)
    f = np.float32
    n_pay = pay.size
    m1 = np.zeros(n_pay, f)
    m2 = np.zeros(n_pay, f)
    want = pay.copy()
    b1, b2, lr, eps = f(cfg.beta1), f(cfg.beta2), f(cfg.lr), f(cfg.eps)
    for step in range(1, 4):
        g = rng.standard_normal(api.grad_size(k, m)).astype(np.float32)
        api.adam_step(renderer, cfg, g, tr)
        gp = g[:n_pay]
        m1 = b1 * m1 + (f(1) - b1) * gp
        m2 = b2 * m2 + (f(1) - b2) * gp * gp
        bc1 = f(1) - f(np.power(b1, f(step), dtype=np.float32))
        bc2 = f(1) - f(np.power(b2, f(step), dtype=np.float32))
        want = want - (lr * (m1 / bc1)) / (np.sqrt(m2 / bc2) + eps)
        want = np.where(want < 0, f(0), want).astype(np.float32)
    got = api.payload_planar(renderer)
    # bc = 1 - pow(beta, step) comes from the host's std::pow; numpy's may differ by an ulp, so
    # allow 2 ulp of the update instead of demanding bits here (the reference fixture above is
    # the bit-exact check)
    assert np.allclose(got, want, rtol=5e-7, atol=1e-7), np.abs(got - want).max()


@pytest.mark.parametrize("m", [3, 4])
def test_adam_sparse_gradients_are_bit_exact(renderer, m):
    """Sparse gradients as a fit step produces them (most voxels untouched: zero moments), with
    signed zeros and subnormals: the update divides zeros off the IEEE slow path and must still
    give the bits of the plain division. beta1 = 0.5 and beta2 = 0.75 make 1 - beta^step exact,
    so the float32 numpy restatement (one rounding per operation) is compared bit for bit."""
    k = 5
    rng = np.random.default_rng(100 + m)
    tr, _ = synthetic.shell_arrays(k, 2)
    tr = np.ascontiguousarray(tr, np.float32)
    pay = rng.uniform(0.0, 1.0, k * 4 * m ** 3).astype(np.float32)
    renderer.set_scene_composed(api.compose(tr), api.PrimitiveSlab(k, m, pay), api.WindowParams())
    renderer._lib.vp_adam_reset(renderer.ctx)
    cfg = api.AdamConfig(lr=3e-2, beta1=0.5, beta2=0.75, eps=1e-8, lr_delta_scale=0.0)
    f = np.float32
    n_pay = pay.size
    m1 = np.zeros(n_pay, f)
    m2 = np.zeros(n_pay, f)
    want = pay.copy()
    b1, b2, lr, eps = f(cfg.beta1), f(cfg.beta2), f(cfg.lr), f(cfg.eps)
    for step in range(1, 4):
        g = np.zeros(api.grad_size(k, m), np.float32)
        u = rng.uniform(size=n_pay)
        g[:n_pay] = np.where(u < 0.1, rng.standard_normal(n_pay).astype(f), g[:n_pay])
        g[:n_pay] = np.where((u >= 0.1) & (u < 0.15), f(-0.0), g[:n_pay])
        g[:n_pay] = np.where((u >= 0.15) & (u < 0.2), f(1e-40) * np.sign(rng.standard_normal(n_pay)).astype(f),
                             g[:n_pay])
        api.adam_step(renderer, cfg, g, tr)
        gp = g[:n_pay]
        with np.errstate(under="ignore"):
            m1 = b1 * m1 + (f(1) - b1) * gp
            m2 = b2 * m2 + (f(1) - b2) * gp * gp
            bc1 = f(1) - b1 ** step
            bc2 = f(1) - b2 ** step
            want = want - (lr * (m1 / bc1)) / (np.sqrt(m2 / bc2) + eps)
        want = np.where(want < 0, f(0), want).astype(np.float32)
    assert np.array_equal(bits(api.payload_planar(renderer)), bits(want))


def _write_vpsl(path, k, m, payload, version=1, magic=b"VPSL", truncate=0):
    """README.md:96-104: magic, u32 version, u32 K, u32 M, f32 payload (little-endian)."""
    data = magic + np.array([version, k, m], "<u4").tobytes() + np.asarray(payload, "<f4").tobytes()
    with open(path, "wb") as f:
        f.write(data[:len(data) - truncate] if truncate else data)


def test_vpsl_loader_streams_into_the_device_layout(renderer, tmp_path):
    tr, pay = synthetic.shell_arrays(512, 8)
    xf = api.compose(tr)
    p = tmp_path / "shell.vpsl"
    _write_vpsl(p, 512, 8, pay)
    renderer.load_slab(str(p), xf, api.WindowParams())
    assert np.array_equal(bits(api.payload_planar(renderer)), bits(pay))
    cam = synthetic.shell_camera(5, 64, 128)
    a = renderer.render(cam, api.MarchConfig())
    renderer.set_scene_composed(xf, api.PrimitiveSlab(512, 8, pay), api.WindowParams())
    b = renderer.render(cam, api.MarchConfig())
    assert np.array_equal(bits(a.color), bits(b.color)) and np.array_equal(a.sample_counts, b.sample_counts)


@pytest.mark.parametrize("kind,category", [("missing", 3), ("magic", 4), ("version", 5), ("truncated", 4),
                                           ("implausible", 4)])
def test_vpsl_loader_errors_mirror_the_reference(renderer, tmp_path, kind, category):
    tr, pay = synthetic.shell_arrays(8, 4)
    xf = api.compose(tr)
    p = tmp_path / "bad.vpsl"
    if kind == "magic":
        _write_vpsl(p, 8, 4, pay, magic=b"VPSX")
    elif kind == "version":
        _write_vpsl(p, 8, 4, pay, version=2)
    elif kind == "truncated":
        _write_vpsl(p, 8, 4, pay, truncate=7)
    elif kind == "implausible":
        _write_vpsl(p, 8, 513, pay)
    with pytest.raises(api.Error) as e:
        renderer.load_slab(str(p), xf, api.WindowParams())
    assert int(e.value.category) == category


# -- device compose (Frame::composed() on the B200: vp_set_frame) ---------------------------
def test_device_compose_matches_reference(renderer):
    """vp_set_frame composes the reference's own fixtures (tests/golden/compose.npz, written by
    the unmodified compose()) bit-for-bit; a non-positive scale is Usage, like the reference."""
    z = np.load(GOLDEN / "compose.npz")
    k = z["tr"].shape[0]
    slab = api.PrimitiveSlab(k, 2, np.zeros(k * 4 * 8, np.float32))
    renderer.set_scene_records(z["tr"], slab, api.WindowParams())
    assert np.array_equal(bits(renderer.transforms()), bits(z["xf"]))
    bad = z["bad"]
    renderer.set_scene_records(z["tr"][:len(bad)], api.PrimitiveSlab(len(bad), 2, np.zeros(len(bad) * 32, np.float32)),
                               api.WindowParams())
    with pytest.raises(api.Error) as e:
        renderer.set_records(bad)
    assert e.value.category == api.ErrorCategory.USAGE


def test_device_compose_equals_host_compose_on_large_angles(renderer):
    """Random poses with rotation-vector magnitudes from 0 to 1e6 (both sinf/cosf reductions,
    the small-angle series, the zero vector): device compose == host compose (vp_compose, the
    reference's exact arithmetic)."""
    rng = np.random.default_rng(7)
    k = 4096
    tr = np.zeros((k, 24), np.float32)
    tr[:, 0:3] = rng.normal(size=(k, 3))
    q = np.linalg.qr(rng.normal(size=(k, 3, 3)))[0]
    tr[:, 3:12] = np.transpose(q, (0, 2, 1)).reshape(k, 9)
    tr[:, 12:15] = rng.uniform(0.01, 0.1, size=(k, 3))
    tr[:, 15:18] = rng.normal(scale=0.01, size=(k, 3))
    axis = rng.normal(size=(k, 3))
    axis /= np.linalg.norm(axis, axis=1, keepdims=True)
    mag = 10.0 ** rng.uniform(-6, 6, size=k)
    mag[:8] = [0, 1e-5, 9.99e-5, 1e-4, 0.7853982, 119.99, 120.0, 1e6]
    tr[:, 18:21] = axis * mag[:, None]
    tr[:, 21:24] = rng.normal(scale=1e-3, size=(k, 3))
    slab = api.PrimitiveSlab(k, 2, np.zeros(k * 4 * 8, np.float32))
    renderer.set_scene_records(tr, slab, api.WindowParams())
    assert np.array_equal(bits(renderer.transforms()), bits(api.compose(tr)))


def test_device_pose_data_equals_host_restatement(renderer):
    """backwardRay's pose data (rBase + rotationDerivative, rotation.cpp:30-38) computed on the
    device equals the host restatement bit-for-bit, across the small-angle, series and
    large-angle branches."""
    rng = np.random.default_rng(11)
    k = 2048
    tr = rng.normal(size=(k, 24)).astype(np.float32)
    mag = 10.0 ** rng.uniform(-8, 4, size=k)
    mag[:4] = [0, 1e-8, 1e-4, 200.0]
    axis = rng.normal(size=(k, 3))
    axis /= np.linalg.norm(axis, axis=1, keepdims=True)
    tr[:, 18:21] = axis * mag[:, None]
    lib, ctx = renderer._lib, renderer.ctx
    from paper_2103_01954_b200._lib import f32p
    a = np.zeros((k, 36), np.float32)
    b = np.zeros((k, 36), np.float32)
    assert lib.vp_debug_pose(ctx, k, tr.ctypes.data_as(f32p), a.ctypes.data_as(f32p), 1) == 0
    assert lib.vp_debug_pose(ctx, k, tr.ctypes.data_as(f32p), b.ctypes.data_as(f32p), 0) == 0
    assert np.array_equal(bits(a), bits(b))


@pytest.mark.parametrize("cos", [False, True])
def test_device_sincos_is_glibc_exact(renderer, oracle, cos):
    """The device port of glibc sinf/cosf used by compose: every float in [1e-4, 120) (the
    rotation angles of any plausible pose; the fast-reduction path), strided beyond (the
    large-argument reduction), against this host's libm."""
    bad = 0
    lo, hi, step = 0x38D1B717, 0x42F00000, 1 << 26
    for start in range(lo, hi, step):
        end = min(start + step - 1, hi - 1)
        x = np.arange(start, end + 1, dtype=np.uint64).astype(np.uint32).view(np.float32)
        bad += oracle.sincos_mismatches(start, end, renderer.debug_sincos(x, cos), cos)
    big = np.arange(0x42F00000, 0x7F800000, 4099, dtype=np.uint64).astype(np.uint32)
    x = np.concatenate([big, big | 0x80000000]).view(np.float32)
    got, want = renderer.debug_sincos(x, cos), oracle.sincos_libm(x, cos)
    bad += int(np.count_nonzero(got.view(np.uint32) != want.view(np.uint32)))
    assert bad == 0


@pytest.mark.parametrize("on_device", [False, True])
@pytest.mark.parametrize("kind", ["pixel", "camera"])
def test_eval_loss_pixel_set_errors(renderer, on_device, kind):
    """evalLoss's pixel-set errors (camera.cpp:15-16, a camera index outside the list) are
    Usage errors whether the pixel set is host-resident (checked on the host before any launch)
    or device-resident (checked by k_eval_rays and read back before the march)."""
    import ctypes as C
    import torch
    from paper_2103_01954_b200 import _lib

    z = _z()
    tr, pay = synthetic.shell_arrays(64, 8)
    scene = api.Scene(api.WindowParams(8.0, 8), frames=[api.Frame(z["tr"], api.PrimitiveSlab(64, 8, pay))])
    renderer.set_frame(scene, 0)
    cams = [api.Camera(c[:9].reshape(3, 3), c[9:18].reshape(3, 3), c[18:21], int(c[21]), int(c[22]))
            for c in z["cams"]]
    n = int(z["cam_index"].size)
    ci = np.ascontiguousarray(z["cam_index"], np.int32).copy()
    xy = np.ascontiguousarray(z["pixel"], np.float32).reshape(n, 2).copy()
    if kind == "pixel":
        xy[n // 2, 0] = float(cams[int(ci[n // 2])].width) + 0.5
    else:
        ci[n // 3] = len(cams)
    pid = np.ascontiguousarray(z["pixel_id"], np.int32)
    tg = np.ascontiguousarray(z["target"], np.float32)
    bg = np.ascontiguousarray(z["background"], np.float32)
    arrays = [ci, xy, pid, tg, bg]
    if on_device:
        keep = [torch.from_numpy(a).cuda() for a in arrays]
        ptrs = [C.c_void_p(t.data_ptr()) for t in keep]
    else:
        ptrs = [a.ctypes.data_as(C.c_void_p) for a in arrays]
    lib = _lib.load()
    cams_c = (_lib.vp_camera * len(cams))(*[c.to_c() for c in cams])
    c = z["cfg"]
    cfg = api.MarchConfig(float(np.float32(c[0])), float(np.float32(c[1])), bool(c[2]), int(c[3]))
    mc = cfg.to_c()
    lp = C.c_float()
    trf = np.ascontiguousarray(z["tr"], np.float32).reshape(-1, 24)
    rc = lib.vp_eval_loss_pho(renderer.ctx, len(cams), cams_c, n, C.cast(ptrs[0], C.POINTER(C.c_int32)),
                              C.cast(ptrs[1], C.POINTER(C.c_float)), C.cast(ptrs[2], C.POINTER(C.c_int32)),
                              C.cast(ptrs[3], C.POINTER(C.c_float)), C.cast(ptrs[4], C.POINTER(C.c_float)),
                              1.0, C.byref(mc), trf.ctypes.data_as(C.POINTER(C.c_float)), C.byref(lp),
                              None, None, 0)
    assert rc == int(api.ErrorCategory.USAGE)
    # the context is still usable: the valid set goes through
    good = api.RaySamples(z["cam_index"], z["pixel"], z["pixel_id"], z["target"], z["background"])
    w = z["weights"]
    terms = api.eval_loss(renderer, scene, 0, cams, good,
                          api.LossWeights(float(w[0]), float(w[1]), float(w[2]), float(w[3])), cfg)
    assert np.float32(terms.pho) == np.float32(z["terms"][0])


def test_adam_step_device_gradient_at_unaligned_offset(renderer):
    """a device gradient pointer that is only 4-byte aligned (a view one float into a
    flat buffer) must not take the 16-byte update path; the result equals the host-gradient
    step bit for bit."""
    import torch
    z = _z()
    m = int(z["adam_m"])
    k = z["adam_tr_in"].shape[0]
    a = z["adam_cfg"]
    cfg = api.AdamConfig(*[float(x) for x in a])
    g = np.ascontiguousarray(z["adam_grads"][0], np.float32)
    outs = []
    for on_device in (False, True):
        tr = np.ascontiguousarray(z["adam_tr_in"], np.float32).copy()
        renderer.set_scene_composed(api.compose(tr), api.PrimitiveSlab(k, m, z["adam_pay_in"]), api.WindowParams())
        renderer._lib.vp_adam_reset(renderer.ctx)
        if on_device:
            flat = torch.zeros(g.size + 1, dtype=torch.float32, device="cuda")
            flat[1:] = torch.from_numpy(g).cuda()
            torch.cuda.synchronize()
            ac = _lib.vp_adam(cfg.lr, cfg.beta1, cfg.beta2, cfg.eps, cfg.lr_delta_scale, cfg.lr_vertex_scale)
            ptr = flat.data_ptr() + 4
            assert ptr % 16 != 0
            rc = renderer._lib.vp_adam_step(renderer.ctx, C.byref(ac), C.cast(C.c_void_p(ptr), _lib.f32p),
                                            tr.ctypes.data_as(_lib.f32p))
            assert rc == 0, renderer._lib.vp_last_error(renderer.ctx)
        else:
            api.adam_step(renderer, cfg, g, tr)
        outs.append((bits(tr).copy(), bits(api.payload_planar(renderer)).copy()))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])


def test_adam_step_rejects_short_gradient(renderer):
    z = _z()
    m = int(z["adam_m"])
    tr = np.ascontiguousarray(z["adam_tr_in"], np.float32).copy()
    k = tr.shape[0]
    renderer.set_scene_composed(api.compose(tr), api.PrimitiveSlab(k, m, z["adam_pay_in"]), api.WindowParams())
    cfg = api.AdamConfig(*[float(x) for x in z["adam_cfg"]])
    with pytest.raises(api.Error) as e:
        api.adam_step(renderer, cfg, np.zeros(k * 4 * m ** 3, np.float32), tr)  # payload part only
    assert e.value.category == api.ErrorCategory.USAGE

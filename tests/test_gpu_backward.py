"""GPU: the backward pass K6 (vp_backward_rays) against the reference's backwardRay.

Every per-sample term is computed with the reference's operation order; only the global sums
(device atomics) are accumulated in a different order than the reference's sequential loop.
The tolerance below is that reordering bound: per entry |g - g_ref| <= 2e-5 * max|g_ref| +
1e-4 * |g_ref| (float32 sums of O(10^3) contributions)."""
import numpy as np
import pytest

from conftest import load_groups
from paper_2103_01954_b200 import api

pytestmark = pytest.mark.gpu


def _inputs(g):
    return (api.WindowParams(float(g["window"][0]), int(g["window"][1])),
            api.MarchConfig(float(g["cfg"][0]), float(g["cfg"][1])))


def _check_close(name, got, want):
    scale = float(np.abs(want).max())
    err = np.abs(got.astype(np.float64) - want)
    bound = 2e-5 * scale + 1e-4 * np.abs(want)
    bad = err > bound
    assert not bad.any(), (f"{name}: {int(bad.sum())} of {want.size} entries outside the reordering "
                           f"bound; max err {err.max():.3g} (scale {scale:.3g})")


@pytest.mark.parametrize("case", sorted(load_groups("backward")))
def test_backward_matches_reference(renderer, case):
    g = load_groups("backward")[case]
    win, cfg = _inputs(g)
    k, m = g["tr"].shape[0], int(g["m"])
    renderer.set_scene_composed(api.compose(g["tr"]), api.PrimitiveSlab(k, m, g["payload"]), win)
    got = renderer.backward_rays(g["o"], g["d"], g["adj_rgb"], g["adj_alpha"], cfg, g["tr"], g["jit"])
    want = g["grads"]
    n_pay = k * 4 * m ** 3
    _check_close(f"{case}.payload", got[:n_pay], want[:n_pay])
    _check_close(f"{case}.pose", got[n_pay:], want[n_pay:])
    # the exact zero pattern agrees (same corners / same primitives touched)
    assert np.array_equal(got != 0, want != 0) or np.abs(got[(got != 0) != (want != 0)]).max() < 1e-30


def test_backward_accumulates_and_is_linear_in_the_adjoints(renderer):
    g = load_groups("backward")["boxes_unsaturated"]
    win, cfg = _inputs(g)
    k, m = g["tr"].shape[0], int(g["m"])
    renderer.set_scene_composed(api.compose(g["tr"]), api.PrimitiveSlab(k, m, g["payload"]), win)
    args = (g["o"], g["d"])
    a = renderer.backward_rays(*args, g["adj_rgb"], g["adj_alpha"], cfg, g["tr"], g["jit"])
    b = renderer.backward_rays(*args, g["adj_rgb"], g["adj_alpha"], cfg, g["tr"], g["jit"], grads=a.copy())
    # b = a + a', a' a second accumulation with its own atomics order: |a' - a| is within twice
    # the reordering bound, which is the bound _check_close applies to 2a
    _check_close("accumulated", b, 2 * a.astype(np.float64))
    z = renderer.backward_rays(*args, np.zeros_like(g["adj_rgb"]), np.zeros_like(g["adj_alpha"]), cfg,
                               g["tr"], g["jit"])
    assert not z.any()


def test_long_rays_take_the_overflow_paths(renderer, oracle):
    """A column of 320 primitives along z. Rays near the axis cross every box: more than 256
    BVH leaves (the warp walk's frontier / candidate cap) and more than 96 segments (the warp
    kernels' list cap), so the forward re-marches them with global windows and the backward
    takes the per-thread walk; tilted rays leave the column after a few to a few hundred
    boxes and stay on the warp paths. Forward bit-exact, gradients within the reordering bound."""
    k, m = 320, 4
    rng = np.random.default_rng(7)
    tr = np.zeros((k, 24), np.float32)
    tr[:, 2] = 0.05 * np.arange(k)
    tr[:, 3:12] = np.eye(3, dtype=np.float32).reshape(9)
    tr[:, 12:15] = 0.03
    pay = rng.uniform(0.0, 0.05, size=k * 4 * m ** 3).astype(np.float32)
    win, cfg = api.WindowParams(), api.MarchConfig()
    xf = api.compose(tr)
    renderer.set_scene_composed(xf, api.PrimitiveSlab(k, m, pay), win)
    n = 48
    o = np.zeros((n, 3), np.float32)
    o[:, :2] = rng.uniform(-0.02, 0.02, size=(n, 2))
    o[:, 2] = -1.0
    slope = np.where(np.arange(n) < 16, 0.0, rng.uniform(0.002, 0.05, size=n)).astype(np.float32)
    d = np.stack([slope, np.zeros(n, np.float32), np.ones(n, np.float32)], 1)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rgb, alpha, samples = renderer.march_rays(o, d, cfg)
    assert renderer.read_stats()["overflow_rays"] >= 16  # the axis rays took the fallback
    rgb_o, alpha_o, samples_o = oracle.march_rays(xf, m, pay, win, o, d, cfg)
    assert np.array_equal(samples, samples_o)
    assert np.array_equal(rgb.view(np.uint32), rgb_o.view(np.uint32))
    assert np.array_equal(alpha.view(np.uint32), alpha_o.view(np.uint32))
    ar = rng.normal(size=(n, 3)).astype(np.float32)
    aa = rng.normal(size=n).astype(np.float32)
    got = renderer.backward_rays(o, d, ar, aa, cfg, tr)
    want = oracle.backward_rays(tr, m, pay, win, o, d, ar, aa, cfg)
    n_pay = k * 4 * m ** 3
    _check_close("long.payload", got[:n_pay], want[:n_pay])
    _check_close("long.pose", got[n_pay:], want[n_pay:])


@pytest.mark.parametrize("n_boxes", [300, 600])
def test_rays_with_more_live_segments_than_the_fallback_window(renderer, oracle, n_boxes):
    """More than kFallbackCap (256) primitives live at one sample of a ray batch: boxes stacked
    on the same region. The reference has no limit; those rays take the last-resort passes
    (k_march_huge_rays forward, k_backward_rays_huge backward; 4096-entry windows). Forward bit-
    exact, gradients within the reordering bound."""
    rng = np.random.default_rng(n_boxes)
    tr = api.transform_records(rng.uniform(-0.02, 0.02, (n_boxes, 3)), np.tile(np.eye(3), (n_boxes, 1, 1)),
                               rng.uniform(0.2, 0.3, (n_boxes, 3)), delta_r=rng.uniform(-0.3, 0.3, (n_boxes, 3)))
    m = 2
    pay = rng.uniform(0, 1, n_boxes * 4 * m ** 3).astype(np.float32)
    pay.reshape(n_boxes, 4, -1)[:, 3] *= np.float32(0.02)  # thin: rays cross the whole stack
    win, cfg = api.WindowParams(), api.MarchConfig(step_size=0.005)
    xf = api.compose(tr)
    renderer.set_scene_composed(xf, api.PrimitiveSlab(n_boxes, m, pay), win)
    n = 40
    o = np.zeros((n, 3), np.float32)
    o[:, :2] = rng.uniform(-0.1, 0.1, size=(n, 2))
    o[:, 2] = -2.0
    d = np.stack([rng.uniform(-0.2, 0.2, n), rng.uniform(-0.2, 0.2, n), np.ones(n)], 1).astype(np.float32)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    rgb, alpha, samples = renderer.march_rays(o, d, cfg)
    st = renderer.read_stats()
    assert st["huge_rays"] > 0, st
    rgb_o, alpha_o, samples_o = oracle.march_rays(xf, m, pay, win, o, d, cfg)
    assert np.array_equal(samples, samples_o)
    assert np.array_equal(rgb.view(np.uint32), rgb_o.view(np.uint32))
    assert np.array_equal(alpha.view(np.uint32), alpha_o.view(np.uint32))
    ar = rng.normal(size=(n, 3)).astype(np.float32)
    aa = rng.normal(size=n).astype(np.float32)
    got = renderer.backward_rays(o, d, ar, aa, cfg, tr)
    want = oracle.backward_rays(tr, m, pay, win, o, d, ar, aa, cfg)
    n_pay = n_boxes * 4 * m ** 3
    _check_close("huge.payload", got[:n_pay], want[:n_pay])
    _check_close("huge.pose", got[n_pay:], want[n_pay:])


@pytest.mark.parametrize("mode", ["warp", "pairs", "cap64"])
def test_backward_paths_agree(monkeypatch, mode):
    """Batches of 8,192 rays or more run the backward as passes over primitive-samples (K6a
    plan, K6b one sample per thread, K6c per-ray fold); smaller ones take the warp-per-ray walk,
    which is also the path for rays that find no room in the pair arrays. Each path forced on
    the golden cases (VPB_BWD_MODE), and the pairs with a 64-sample capacity (most rays spill
    to the walk): all equal the reference within the reordering bound."""
    from paper_2103_01954_b200 import Renderer
    monkeypatch.setenv("VPB_BWD_MODE", "warp" if mode == "warp" else "pairs")
    if mode == "cap64":
        monkeypatch.setenv("VPB_BWD_PAIR_CAP", "64")
    r = Renderer(0)
    try:
        for case, g in sorted(load_groups("backward").items()):
            win, cfg = _inputs(g)
            k, m = g["tr"].shape[0], int(g["m"])
            r.set_scene_composed(api.compose(g["tr"]), api.PrimitiveSlab(k, m, g["payload"]), win)
            got = r.backward_rays(g["o"], g["d"], g["adj_rgb"], g["adj_alpha"], cfg, g["tr"], g["jit"])
            n_pay = k * 4 * m ** 3
            _check_close(f"{mode}.{case}.payload", got[:n_pay], g["grads"][:n_pay])
            _check_close(f"{mode}.{case}.pose", got[n_pay:], g["grads"][n_pay:])
    finally:
        r.close()


def test_large_batch_interleaved_gradient_any_alignment(renderer):
    """Batches of >= 16,384 rays scatter an interleaved gradient with vector reductions and
    transpose it into the planar GradBuffer at the C-ABI: a 16-byte aligned destination takes
    the vectorized transpose, a caller's device pointer that is only 4-byte aligned the scalar
    one. Both equal the reference's gradient of the replicated batch (linear in the rays)."""
    import ctypes as C
    import torch
    from paper_2103_01954_b200 import _lib
    g = load_groups("backward")["boxes_unsaturated"]
    win, cfg = _inputs(g)
    k, m = g["tr"].shape[0], int(g["m"])
    renderer.set_scene_composed(api.compose(g["tr"]), api.PrimitiveSlab(k, m, g["payload"]), win)
    n0 = g["o"].shape[0]
    rep = -(-16384 // n0)
    o, d = np.tile(g["o"], (rep, 1)), np.tile(g["d"], (rep, 1))
    ar, aa, jit = np.tile(g["adj_rgb"], (rep, 1)), np.tile(g["adj_alpha"], rep), np.tile(g["jit"], rep)
    host = renderer.backward_rays(o, d, ar, aa, cfg, g["tr"], jit)
    want = g["grads"].astype(np.float64) * rep
    n_pay = k * 4 * m ** 3
    _check_close("aligned.payload", host[:n_pay], want[:n_pay])
    _check_close("aligned.pose", host[n_pay:], want[n_pay:])
    # accumulating into a caller's buffer (the transpose adds instead of writing)
    acc = renderer.backward_rays(o, d, ar, aa, cfg, g["tr"], jit, grads=host.copy())
    _check_close("accumulated", acc, 2 * want)
    lib = _lib.load()
    f32p = C.POINTER(C.c_float)
    P = lambda t: C.cast(C.c_void_p(t.data_ptr()), f32p)  # noqa: E731
    dev = {nm: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
           for nm, a in (("o", o), ("d", d), ("ar", ar), ("aa", aa), ("j", jit))}
    buf = torch.zeros(host.size + 1, dtype=torch.float32, device="cuda")
    view = buf[1:]  # 4-byte aligned only
    assert view.data_ptr() % 16 != 0
    mc = cfg.to_c()
    tr = np.ascontiguousarray(g["tr"], np.float32)
    rc = lib.vp_backward_rays(renderer.ctx, o.shape[0], P(dev["o"]), P(dev["d"]), P(dev["j"]), P(dev["ar"]),
                              P(dev["aa"]), C.byref(mc), tr.ctypes.data_as(f32p), P(view), 0)
    assert rc == 0, lib.vp_last_error(renderer.ctx)
    got = view.cpu().numpy()
    _check_close("unaligned.payload", got[:n_pay], want[:n_pay])
    _check_close("unaligned.pose", got[n_pay:], want[n_pay:])
    # calls alternate between two interleaved gradient buffers (each cleared during a later
    # call's forward): zero adjoints after all of the above must give exact zeros
    for _ in range(2):
        z = renderer.backward_rays(o, d, np.zeros_like(ar), np.zeros_like(aa), cfg, g["tr"], jit)
        assert not z.any()


@pytest.mark.parametrize("mode", ["pairs", "warp"])
@pytest.mark.parametrize("seed", [11, 12, 13])
def test_random_scenes_backward_matches_restatement(monkeypatch, oracle, seed, mode):
    """Randomized scenes and rays through both backward paths (K6a-c and the warp walk): sparse clouds (rays with gaps between their
    segments, so the walk takes gap skips), dense ones (several live entries per step, step-major
    slots that interleave entries), saturating and unsaturated rays, jitter. Gradients within
    the reordering bound of the restatement's sequential backwardRay."""
    rng = np.random.default_rng(seed)
    k, m = (60, 4) if seed == 11 else ((400, 3) if seed == 12 else (150, 2))
    spread = 0.6 if seed != 12 else 0.25
    t = rng.uniform(-spread, spread, (k, 3))
    s = rng.uniform(0.02, 0.12, (k, 3))
    tr = api.transform_records(t, np.tile(np.eye(3), (k, 1, 1)), s, delta_r=rng.uniform(-1, 1, (k, 3)))
    pay = rng.uniform(0.0, 1.0, k * 4 * m ** 3).astype(np.float32)
    pay.reshape(k, 4, -1)[:, 3] *= np.float32(40.0 if seed == 12 else 8.0)
    win = api.WindowParams()
    cfg = api.MarchConfig(step_size=0.004, jitter=seed == 13, seed=seed)
    xf = api.compose(tr)
    from paper_2103_01954_b200 import Renderer
    monkeypatch.setenv("VPB_BWD_MODE", mode)
    renderer = Renderer(0)
    renderer.set_scene_composed(xf, api.PrimitiveSlab(k, m, pay), win)
    n = 512
    o = np.tile(np.float32([0.05, -0.03, -2.0]), (n, 1)) + rng.uniform(-0.02, 0.02, (n, 3)).astype(np.float32)
    tgt = rng.uniform(-spread, spread, (n, 3)).astype(np.float32)
    d = tgt - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    jit = rng.uniform(0, 1, n).astype(np.float32) if cfg.jitter else None
    ar = rng.normal(size=(n, 3)).astype(np.float32)
    aa = rng.normal(size=n).astype(np.float32)
    try:
        got = renderer.backward_rays(o, d, ar, aa, cfg, tr, jit)
    finally:
        renderer.close()
    want = oracle.backward_rays(tr, m, pay, win, o, d, ar, aa, cfg, jit)
    n_pay = k * 4 * m ** 3
    _check_close(f"rand{seed}.payload", got[:n_pay], want[:n_pay])
    _check_close(f"rand{seed}.pose", got[n_pay:], want[n_pay:])


def test_large_batch_gradient_buffers_across_scene_sizes(renderer):
    """The interleaved gradient buffers outlive scenes: a larger scene's gradient, then a
    smaller scene's, then the larger one again must give the first result again (a buffer
    cleared only as far as the smaller scene would leak the larger one's tail)."""
    rng = np.random.default_rng(3)

    def scene(k, m):
        t = rng.uniform(-0.3, 0.3, (k, 3))
        s = rng.uniform(0.05, 0.15, (k, 3))
        tr = api.transform_records(t, np.tile(np.eye(3), (k, 1, 1)), s, delta_r=rng.uniform(-1, 1, (k, 3)))
        pay = rng.uniform(0, 1, k * 4 * m ** 3).astype(np.float32)
        return tr, pay

    n = 16384
    o = np.tile(np.float32([0.0, 0.0, -2.0]), (n, 1))
    d = rng.normal(scale=0.12, size=(n, 3)).astype(np.float32)
    d[:, 2] = 1.0
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    ar = rng.normal(size=(n, 3)).astype(np.float32)
    aa = rng.normal(size=n).astype(np.float32)
    cfg, win = api.MarchConfig(step_size=0.004), api.WindowParams()
    big, small = scene(160, 4), scene(40, 4)

    def run(sc):
        tr, pay = sc
        renderer.set_scene_composed(api.compose(tr), api.PrimitiveSlab(tr.shape[0], 4, pay), win)
        return renderer.backward_rays(o, d, ar, aa, cfg, tr)

    first = run(big)
    run(small)
    again = run(big)
    assert np.abs(first).max() > 0
    _check_close("big.again", again, first.astype(np.float64))

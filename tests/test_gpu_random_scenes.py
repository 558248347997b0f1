"""GPU: randomized scenes through every raymarch configuration, bit-exact against the C
restatement of render() (oracle/vp_oracle.c, itself pinned to the reference by
tests/test_oracle_golden.py).

Random rotated boxes (acceptance.cpp:64-75-style) at densities that push the kernels
through their edge paths: windows that refill or overflow into the fallback kernel, tiles
with more candidates than a tier stages, cameras inside primitives, jitter, odd image sizes,
and each tile configuration forced in turn (light / normal / dense; half-tile and 16x16 CTAs).
"""
import numpy as np
import pytest

from paper_2103_01954_b200 import Renderer, api, synthetic

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def _scene(seed, n, spread, smin, smax, m, sigma):
    rng = np.random.default_rng(seed)
    t = rng.uniform(-spread, spread, (n, 3))
    s = smin + (smax - smin) * np.abs(rng.uniform(-1, 1, (n, 3)))
    dr = rng.uniform(-1, 1, (n, 3)) * 2.0
    tr = api.transform_records(t, np.tile(np.eye(3), (n, 1, 1)), s, delta_r=dr)
    pay = rng.uniform(0.0, 1.0, n * 4 * m ** 3).astype(np.float32)
    pay.reshape(n, 4, -1)[:, 3] *= rng.uniform(0.1, 1.0, (n, 1)).astype(np.float32) * np.float32(sigma)
    return tr, pay


CASES = [
    # seed, K, spread, smin, smax, M, sigma scale, camera distance, W, H, jitter
    (1, 300, 0.6, 0.02, 0.15, 4, 60.0, 2.5, 96, 80, False),
    (2, 2000, 0.5, 0.01, 0.06, 3, 60.0, 2.2, 128, 96, False),  # dense: tiles beyond every staging cap
    (3, 120, 0.3, 0.05, 0.4, 5, 2.0, 0.2, 64, 48, True),       # camera inside the cloud, jitter
    (4, 150, 0.05, 0.05, 0.3, 2, 0.3, 2.0, 72, 72, False),     # stacked boxes: windows overflow
]


@pytest.mark.parametrize("tile_cfg", ["light", "normal", "dense"])
@pytest.mark.parametrize("case", CASES, ids=[f"seed{c[0]}" for c in CASES])
def test_random_scene_matches_restatement(monkeypatch, oracle, tile_cfg, case):
    seed, k, spread, smin, smax, m, sigma, dist, w, h, jitter = case
    monkeypatch.setenv("VPB_TILE_CFG", tile_cfg)
    tr, pay = _scene(seed, k, spread, smin, smax, m, sigma)
    xf = api.compose(tr)
    cam, _ = synthetic.look_at_camera((0.3 * dist, 0.2 * dist, -dist), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0),
                                      0.9 * w, w, h)
    cfg = api.MarchConfig(step_size=0.004, jitter=jitter, seed=seed)
    r = Renderer(0)
    try:
        r.set_scene_composed(xf, api.PrimitiveSlab(k, m, pay), api.WindowParams())
        out = r.render(cam, cfg)
    finally:
        r.close()
    rgb, alpha, samples = oracle.render(xf, m, pay, api.WindowParams(), cam, cfg)
    assert out.total_samples() > 0
    if seed == 4:  # the stacked boxes must exercise the wide-window fallback kernel
        assert out.stats["overflow_rays"] > 0
    assert np.array_equal(out.sample_counts, samples), "sample counts differ"
    assert np.array_equal(_bits(out.alpha), _bits(alpha)), "alpha differs"
    assert np.array_equal(_bits(out.color), _bits(rgb)), "rgb differs"


@pytest.mark.parametrize("case", CASES, ids=[f"seed{c[0]}" for c in CASES])
def test_random_scene_key_overflow_matches_restatement(oracle, case):
    """The same scenes with the tile-key capacity forced to a third of their keys: the overflowed
    tiles are rebuilt and marched by the fallback kernel (with its own window-overflow re-march
    where the stacked boxes need it), and the image is still the restatement's, bit for bit."""
    seed, k, spread, smin, smax, m, sigma, dist, w, h, jitter = case
    tr, pay = _scene(seed, k, spread, smin, smax, m, sigma)
    xf = api.compose(tr)
    cam, _ = synthetic.look_at_camera((0.3 * dist, 0.2 * dist, -dist), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0),
                                      0.9 * w, w, h)
    cfg = api.MarchConfig(step_size=0.004, jitter=jitter, seed=seed)
    r = Renderer(0)
    try:
        r.set_scene_composed(xf, api.PrimitiveSlab(k, m, pay), api.WindowParams())
        keys = r.render(cam, cfg).stats["keys"]
        r.set_key_capacity(max(1, keys // 3), grow=False)
        out = r.render(cam, cfg)
    finally:
        r.close()
    rgb, alpha, samples = oracle.render(xf, m, pay, api.WindowParams(), cam, cfg)
    assert np.array_equal(out.sample_counts, samples), "sample counts differ"
    assert np.array_equal(_bits(out.alpha), _bits(alpha)), "alpha differs"
    assert np.array_equal(_bits(out.color), _bits(rgb)), "rgb differs"


@pytest.mark.parametrize("n_boxes", [300, 700])
def test_more_live_segments_than_the_fallback_window(oracle, n_boxes):
    """More than kFallbackCap (256) primitives live at one sample: boxes stacked on the same
    region. The reference has no limit; camera renders take the last-resort pass (K5c,
    4096-entry windows over all primitives) and still equal the restatement bit for bit."""
    rng = np.random.default_rng(n_boxes)
    t = rng.uniform(-0.02, 0.02, (n_boxes, 3))
    s = rng.uniform(0.2, 0.3, (n_boxes, 3))
    tr = api.transform_records(t, np.tile(np.eye(3), (n_boxes, 1, 1)), s, delta_r=rng.uniform(-0.3, 0.3, (n_boxes, 3)))
    m = 2
    pay = rng.uniform(0, 1, n_boxes * 4 * m ** 3).astype(np.float32)
    pay.reshape(n_boxes, 4, -1)[:, 3] *= np.float32(0.02)  # thin: rays cross the whole stack
    xf = api.compose(tr)
    cam, _ = synthetic.look_at_camera((0.1, 0.2, -2.0), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 60.0, 40, 36)
    cfg = api.MarchConfig(step_size=0.005)
    r = Renderer(0)
    try:
        r.set_scene_composed(xf, api.PrimitiveSlab(n_boxes, m, pay), api.WindowParams())
        out = r.render(cam, cfg)
    finally:
        r.close()
    rgb, alpha, samples = oracle.render(xf, m, pay, api.WindowParams(), cam, cfg)
    assert out.stats["overflow_rays"] > 0 and out.stats["huge_rays"] > 0, out.stats
    assert np.array_equal(out.sample_counts, samples), "sample counts differ"
    assert np.array_equal(_bits(out.alpha), _bits(alpha)), "alpha differs"
    assert np.array_equal(_bits(out.color), _bits(rgb)), "rgb differs"

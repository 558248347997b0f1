"""Tile-key capacity overflow: a view whose (tile, depth) keys do not all fit
the entries buffer still renders bit-exactly through every entry point, synchronous or not. The
tiles whose buckets overflow are marched by the fallback kernel from all K pixel rectangles
(vpb_kernels.cu k_march_fallback_views); no vp_read_stats call is needed to get right pixels.

The key capacity is forced below the scenes' key counts with vp_set_key_capacity(grow=0), and
results are compared with the reference's own digests (tests/golden/digests.json)."""
import json

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from golden_cases import sha
from paper_2103_01954_b200 import Renderer, api, synthetic

pytestmark = pytest.mark.gpu
DIGESTS = json.loads((GOLDEN / "digests.json").read_text())


def _check(out, d, what):
    assert out.total_samples() == d["total_samples"], what
    assert sha(out.sample_counts) == d["samples"], what
    assert sha(out.alpha) == d["alpha"], what
    assert sha(out.color) == d["rgb"], what


def _device_render(r, cam, cfg):
    w, h = int(cam.width), int(cam.height)
    rgb = torch.empty(h * w * 3, device="cuda")
    alpha = torch.empty(h * w, device="cuda")
    samp = torch.empty(h * w, dtype=torch.int32, device="cuda")
    rgb.fill_(-1.0)  # stale contents must not survive
    r.render_device(cam, cfg, rgb.data_ptr(), alpha.data_ptr(), samp.data_ptr())
    torch.cuda.synchronize()
    return api.RenderOutput(rgb.cpu().numpy().reshape(h, w, 3), alpha.cpu().numpy().reshape(h, w, 1),
                            samp.cpu().numpy(), None)


@pytest.mark.parametrize("key,cap", [("k4096_m16_1024_view-1", 20000), ("k32768_m8_1024_view-1", 100000),
                                     ("oracle_64x16_256_view-1", 0)])
def test_key_overflow_sync_and_async_match_reference(key, cap):
    d = DIGESTS["renders"][key]
    tr, pay = synthetic.shell_arrays(d["K"], d["M"])
    with Renderer(0) as r:
        r.set_scene_composed(api.compose(tr), api.PrimitiveSlab(d["K"], d["M"], pay), api.WindowParams())
        cam = synthetic.shell_camera(d["view"], d["n_views"], d["W"])
        # cap 0 with grow=0 means "default"; use 1 key to overflow every non-empty tile
        r.set_key_capacity(max(cap, 1), grow=False)
        out = r.render(cam, api.MarchConfig())
        assert out.stats["keys"] > max(cap, 1), "the scene must overflow the forced capacity"
        _check(out, d, f"{key} sync, capacity {cap}")
        _check(_device_render(r, cam, api.MarchConfig()), d, f"{key} async, capacity {cap}")


def test_key_overflow_batch_matches_reference():
    """8 ring views in one raymarch launch with every view over the capacity."""
    ring = DIGESTS["ring"]
    tr, pay = synthetic.shell_arrays(ring["K"], ring["M"])
    with Renderer(0) as r:
        r.set_scene_composed(api.compose(tr), api.PrimitiveSlab(ring["K"], ring["M"], pay), api.WindowParams())
        r.set_key_capacity(30000, grow=False)
        views = list(range(8, 16))
        outs = r.render_batch([synthetic.shell_camera(v, 64, ring["W"]) for v in views], api.MarchConfig())
        for v, out in zip(views, outs):
            _check(out, ring["views"][str(v)], f"ring view {v} batched over capacity")


def test_natural_key_overflow_async_equals_grown_sync():
    """A scene whose keys exceed the default capacity (2^20) on its own: large boxes at 2048^2.
    The first (async, device-output) render overflows; the synchronous render after the
    capacity has grown takes the normal path. Both must be bitwise equal."""
    rng = np.random.default_rng(7)
    k = 1500
    t = rng.uniform(-0.4, 0.4, (k, 3))
    s = rng.uniform(0.08, 0.25, (k, 3))
    tr = api.transform_records(t, np.tile(np.eye(3), (k, 1, 1)), s, delta_r=rng.uniform(-1, 1, (k, 3)))
    m = 2
    pay = rng.uniform(0, 1, (k, 4, m, m, m)).astype(np.float32)
    pay[:, 3] *= 0.5
    cam = api.Camera(np.array([[2200.0, 0, 1024], [0, 2200.0, 1024], [0, 0, 1]], np.float32), np.eye(3, dtype=np.float32),
                     np.array([0, 0, 2.0], np.float32), 2048, 2048)
    cfg = api.MarchConfig(0.004, 0.01)
    with Renderer(0) as r:
        r.set_scene_composed(api.compose(tr), api.PrimitiveSlab(k, m, pay.reshape(-1)), api.WindowParams())
        first = _device_render(r, cam, cfg)
        st = r.read_stats()
        assert st["keys"] > (1 << 20), f"scene has only {st['keys']} keys"
        second = r.render(cam, cfg)  # capacity grown by now: no overflow
    assert np.array_equal(first.sample_counts, second.sample_counts)
    assert np.array_equal(first.alpha.view(np.uint32), second.alpha.view(np.uint32))
    assert np.array_equal(first.color.view(np.uint32), second.color.view(np.uint32))

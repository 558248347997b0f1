"""GPU: single-view tile sharding (vp_render_shard_async). Shard r of n renders
the tiles t % n == r into a tile-major buffer; the shards placed back into the image
(dist.assemble_tile_shards) must equal the unsharded render bit-for-bit, and the shards'
counters must add up to the view's. One GPU renders every shard here, in turn; across GPUs
each rank renders its own (bench.py --tile-shard, dist.TileShardGather)."""
import numpy as np
import pytest

from golden_cases import sha
from paper_2103_01954_b200 import Renderer, api, synthetic
from paper_2103_01954_b200.dist import assemble_tile_shards

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def _render_shards(r, cam, cfg, n):
    import torch
    rgbs, alphas, samps, stats = [], [], [], []
    for s in range(n):
        slots = api.shard_tiles(cam.width, cam.height, s, n)
        # poisoned buffers: every pixel of an owned tile inside the image must be written
        rgb = torch.full((max(slots, 1) * 256 * 3,), float("nan"), device="cuda")
        alpha = torch.full((max(slots, 1) * 256,), float("nan"), device="cuda")
        samp = torch.full((max(slots, 1) * 256,), -7, dtype=torch.int32, device="cuda")
        r.render_shard_device(cam, cfg, s, n, rgb.data_ptr(), alpha.data_ptr(), samp.data_ptr())
        stats.append(r.read_stats())
        rgbs.append(rgb.view(-1, 256, 3).cpu().numpy())
        alphas.append(alpha.view(-1, 256, 1).cpu().numpy())
        samps.append(samp.view(-1, 256, 1).cpu().numpy())
    w, h = cam.width, cam.height
    return (assemble_tile_shards(rgbs, w, h, 3), assemble_tile_shards(alphas, w, h, 1),
            assemble_tile_shards(samps, w, h, 1).reshape(-1), stats)


def _check(full, got):
    rgb, alpha, samp, stats = got
    assert np.array_equal(_bits(rgb), _bits(full.color)), "rgb differs from the unsharded render"
    assert np.array_equal(_bits(alpha), _bits(full.alpha)), "alpha differs from the unsharded render"
    assert np.array_equal(samp, full.sample_counts), "sample counts differ from the unsharded render"
    for key in ("ray_samples", "prim_samples", "hit_rays", "early_exits", "saturated"):
        assert sum(s[key] for s in stats) == full.stats[key], key


@pytest.mark.parametrize("n", [1, 2, 3, 8])
@pytest.mark.parametrize("k,m,view,w,h,jitter", [(4096, 8, 11, 333, 200, False), (4096, 8, 3, 256, 256, True),
                                                 (512, 16, -1, 100, 37, False)])
def test_shards_assemble_to_the_view(renderer, n, k, m, view, w, h, jitter):
    tr, pay = synthetic.shell_arrays(k, m)
    renderer.set_scene_composed(api.compose(tr), api.PrimitiveSlab(k, m, pay), api.WindowParams())
    cam = synthetic.shell_camera(view, 64, max(w, h))
    cam.width, cam.height = w, h
    cfg = api.MarchConfig(jitter=jitter, seed=99) if jitter else api.MarchConfig()
    full = renderer.render(cam, cfg)
    assert full.total_samples() > 0
    _check(full, _render_shards(renderer, cam, cfg, n))


@pytest.mark.parametrize("tile_cfg", ["normal", "dense"])
@pytest.mark.parametrize("key", ["k4096_m16_1024_view-1", "k32768_m8_1024_view-1"])
def test_full_size_shards_reproduce_the_reference_digest(monkeypatch, key, tile_cfg):
    """BASELINE configs 3 and 4 split over 8 shards: the assembled view has the reference's digest."""
    import json

    from conftest import GOLDEN
    d = json.loads((GOLDEN / "digests.json").read_text())["renders"][key]
    monkeypatch.setenv("VPB_TILE_CFG", tile_cfg)
    tr, pay = synthetic.shell_arrays(d["K"], d["M"])
    r = Renderer(0)
    try:
        r.set_scene_composed(api.compose(tr), api.PrimitiveSlab(d["K"], d["M"], pay), api.WindowParams())
        cam = synthetic.shell_camera(d["view"], d["n_views"], d["W"])
        rgb, alpha, samp, stats = _render_shards(r, cam, api.MarchConfig(), 8)
    finally:
        r.close()
    assert sum(s["ray_samples"] for s in stats) == d["total_samples"]
    assert sha(np.ascontiguousarray(samp)) == d["samples"]
    assert sha(np.ascontiguousarray(alpha)) == d["alpha"]
    assert sha(np.ascontiguousarray(rgb)) == d["rgb"]


def test_shards_with_overflowing_rays(renderer):
    """40 stacked boxes: central rays hold more live segments than any shared-memory window, so
    they go through the wide-window fallback kernel, whose writes must land in the shard layout."""
    k, m = 40, 4
    rng = np.random.default_rng(5)
    xf = np.zeros((k, 15), np.float32)
    for i in range(k):
        a = 0.05 * i
        c, s = np.cos(a), np.sin(a)
        rot = np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]], np.float32)
        xf[i, :3] = (0.01 * rng.standard_normal(), 0.01 * rng.standard_normal(), 0.004 * i)
        xf[i, 3:12] = rot.T.reshape(-1)  # column-major
        xf[i, 12:15] = (0.3, 0.3, 0.5)
    pay = rng.uniform(0.0, 1.0, k * 4 * m ** 3).astype(np.float32) * 0.5
    renderer.set_scene_composed(xf, api.PrimitiveSlab(k, m, pay), api.WindowParams())
    cam, _ = synthetic.look_at_camera((0.0, 0.0, -2.5), (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), 120.0, 96, 80)
    cfg = api.MarchConfig(early_eps=0.0)
    full = renderer.render(cam, cfg)
    assert full.stats["overflow_rays"] > 0, "the scene must exercise the fallback kernel"
    got = _render_shards(renderer, cam, cfg, 3)
    _check(full, got)
    assert any(s["overflow_rays"] > 0 for s in got[3])


def test_shard_argument_errors(renderer):
    import torch
    tr, pay = synthetic.shell_arrays(64, 4)
    renderer.set_scene_composed(api.compose(tr), api.PrimitiveSlab(64, 4, pay), api.WindowParams())
    cam = synthetic.shell_camera(0, 64, 64)
    buf = torch.zeros(16 * 256 * 3, device="cuda")
    for shard, n in ((2, 2), (-1, 2), (0, 0)):
        with pytest.raises(api.Error) as e:
            renderer.render_shard_device(cam, api.MarchConfig(), shard, n, buf.data_ptr(), buf.data_ptr())
        assert e.value.category == api.ErrorCategory.USAGE
    host = np.zeros(16 * 256 * 3, np.float32)
    with pytest.raises(api.Error) as e:  # tile-major shard outputs are device-only
        renderer.render_shard_device(cam, api.MarchConfig(), 0, 2, host.ctypes.data, host.ctypes.data)
    assert e.value.category == api.ErrorCategory.USAGE


@pytest.mark.parametrize("n", [1, 3])
def test_shards_with_key_overflow(n):
    """Tile shards whose owned tiles overflow a forced key capacity (K5b rebuilds those tiles'
    lists from all primitives and writes the shard's tile-major slots) still assemble to the
    unsharded render."""
    tr, pay = synthetic.shell_arrays(4096, 8)
    with Renderer(0) as r:
        r.set_scene_composed(api.compose(tr), api.PrimitiveSlab(4096, 8, pay), api.WindowParams())
        cam = synthetic.shell_camera(5, 64, 256)
        cfg = api.MarchConfig()
        full = r.render(cam, cfg)
        r.set_key_capacity(500, grow=False)
        got = _render_shards(r, cam, cfg, n)
        assert all(s["keys"] > 500 for s in got[3]) or n > 1
    _check(full, got)

"""GPU parity: the sm_100a path through the C-ABI against the reference's own outputs.

Bar: bit-exact. Every expected value in tests/golden was produced by the unmodified reference
(oracle/gen_golden.py); the binning artefacts (no reference counterpart) are compared with
the CPU restatement in oracle/vp_oracle.c.
"""
import json

import numpy as np
import pytest

from conftest import GOLDEN, load_groups
from golden_cases import render_cases, sha
from paper_2103_01954_b200 import api, synthetic

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def assert_bit_equal(name, got, want):
    g, w = np.asarray(got), np.asarray(want)
    assert g.shape == w.shape, f"{name}: shape {g.shape} != {w.shape}"
    if g.dtype == np.float32:
        neq = bits(g) != bits(w)
    else:
        neq = g != w
    if neq.any():
        idx = np.argwhere(neq)[:5]
        diff = np.abs(g.astype(np.float64) - w.astype(np.float64)).max()
        raise AssertionError(f"{name}: {int(neq.sum())} elements differ (max abs {diff:.3g}); first {idx.tolist()}")


@pytest.mark.parametrize("case", sorted(load_groups("renders")))
def test_render_matches_reference(renderer, case):
    c = render_cases()[case]
    renderer.set_scene_composed(api.compose(c["tr"]) if len(c["tr"]) else np.zeros((0, 15), np.float32),
                                api.PrimitiveSlab(len(c["tr"]), c["m"], c["payload"]), c["window"])
    out = renderer.render(c["cam"], c["cfg"])
    assert_bit_equal(f"{case}.rgb", out.color, c["rgb"])
    assert_bit_equal(f"{case}.alpha", out.alpha, c["alpha"])
    assert_bit_equal(f"{case}.samples", out.sample_counts, c["samples"])
    if out.stats is not None and len(c["tr"]):
        assert out.stats["ray_samples"] == int(c["samples"].sum())
        # the K5 prim-sample counter (the roofline's algorithmic bytes) vs the reference's count
        prim = np.load(GOLDEN / "prim_counts.npz")[f"case_{case}"]
        assert out.stats["prim_samples"] == int(prim.astype(np.int64).sum())


DIGESTS = json.loads((GOLDEN / "digests.json").read_text())


@pytest.mark.parametrize("key", sorted(DIGESTS["renders"]))
def test_full_size_render_digest(renderer, key):
    """BASELINE.json configs 1-4 (+ four views of config 5) at full size, bit-exact."""
    d = DIGESTS["renders"][key]
    tr, pay = synthetic.shell_arrays(d["K"], d["M"])
    gen = DIGESTS["generator"][f"{d['K']}x{d['M']}"]
    assert sha(tr) == gen["tr"] and sha(pay) == gen["payload"], "synthetic generator drifted"
    renderer.set_scene_composed(api.compose(tr), api.PrimitiveSlab(d["K"], d["M"], pay), api.WindowParams())
    cam = synthetic.shell_camera(d["view"], d["n_views"], d["W"])
    out = renderer.render(cam, api.MarchConfig())
    assert out.total_samples() == d["total_samples"]
    assert int((out.sample_counts > 0).sum()) == d["hit_pixels"]
    assert sha(out.sample_counts) == d["samples"]
    assert sha(out.alpha) == d["alpha"]
    assert sha(out.color) == d["rgb"]
    assert out.stats["ray_samples"] == d["total_samples"]
    # 128 B per prim-sample is the roofline's numerator: the device counter equals the
    # reference's own count (oracle/gen_prim_counts.py)
    assert out.stats["prim_samples"] == d["prim_samples"]


@pytest.mark.parametrize("tile_cfg", ["light", "normal", "dense"])
@pytest.mark.parametrize("key", ["k32768_m8_1024_view-1", "k4096_m16_1024_view-1", "oracle_64x16_256_view-1"])
def test_full_size_digest_under_each_tile_config(monkeypatch, key, tile_cfg):
    """Every raymarch configuration (light / normal / dense: 12 / 16 / 24-entry windows,
    64 / 64 / 192 staged candidates) is bit-exact on every scene density, including the ones it
    is not chosen for (window refills, unstaged tiles)."""
    from paper_2103_01954_b200 import Renderer
    monkeypatch.setenv("VPB_TILE_CFG", tile_cfg)
    d = DIGESTS["renders"][key]
    tr, pay = synthetic.shell_arrays(d["K"], d["M"])
    r = Renderer(0)
    try:
        r.set_scene_composed(api.compose(tr), api.PrimitiveSlab(d["K"], d["M"], pay), api.WindowParams())
        out = r.render(synthetic.shell_camera(d["view"], d["n_views"], d["W"]), api.MarchConfig())
    finally:
        r.close()
    assert out.total_samples() == d["total_samples"]
    assert sha(out.sample_counts) == d["samples"]
    assert sha(out.alpha) == d["alpha"]
    assert sha(out.color) == d["rgb"]


def test_march_kats_match_reference(renderer):
    """test_march.cpp:50-194 scenarios plus random rays, through vp_march_rays."""
    for name, g in load_groups("march_kats").items():
        k = g["xf"].shape[0]
        renderer.set_scene_composed(g["xf"], api.PrimitiveSlab(k, int(g["m"]), g["payload"]),
                                    api.WindowParams(float(g["window"][0]), int(g["window"][1])))
        cfg = api.MarchConfig(float(g["cfg"][0]), float(g["cfg"][1]))
        rgb, alpha, samples = renderer.march_rays(g["o"], g["d"], cfg, g["jit"])
        assert_bit_equal(f"{name}.rgb", rgb, g["rgb"])
        assert_bit_equal(f"{name}.alpha", alpha, g["alpha"])
        assert_bit_equal(f"{name}.samples", samples, g["samples"])


def test_march_kat_properties(renderer):
    """The analytic statements of test_march.cpp on the device results."""
    g = load_groups("march_kats")
    res = {}
    for name in ("constant_medium", "saturation", "early_exact", "early_lazy"):
        c = g[name]
        renderer.set_scene_composed(c["xf"], api.PrimitiveSlab(c["xf"].shape[0], int(c["m"]), c["payload"]),
                                    api.WindowParams(float(c["window"][0]), int(c["window"][1])))
        res[name] = renderer.march_rays(c["o"], c["d"], api.MarchConfig(float(c["cfg"][0]), float(c["cfg"][1])))
    rgb, alpha, samples = res["constant_medium"]
    assert abs(alpha[0] - 0.4) < 0.004 and abs(rgb[0, 0] - 0.32) < 0.0032 and abs(samples[0] - 2000) < 20
    rgb, alpha, samples = res["saturation"]
    assert alpha[0] == 1.0 and samples[0] < 600
    assert np.allclose(rgb[0], [0.3, 0.9, 0.5], rtol=1e-4)
    assert res["early_lazy"][2][0] < res["early_exact"][2][0]


def test_binning_matches_cpu_restatement(renderer, oracle):
    """Cull rectangles, depth keys and per-tile (depth, prim)-sorted lists: bit-exact."""
    cases = render_cases()
    for name in ("shell64_m16_w64", "random_boxes_96x72", "camera_inside_40x32"):
        c = cases[name]
        xf = api.compose(c["tr"])
        renderer.set_scene_composed(xf, api.PrimitiveSlab(len(xf), c["m"], c["payload"]), c["window"])
        rects, keys, offs, prims = renderer.debug_tiles(c["cam"])
        orects, okeys = oracle.cull(xf, c["cam"])
        ooffs, oprims = oracle.tile_lists(xf, c["cam"])
        assert np.array_equal(rects, orects), name
        assert np.array_equal(keys, okeys), name
        assert np.array_equal(offs, ooffs), name
        assert np.array_equal(prims, oprims), name
    for k, m, w in ((4096, 16, 1024), (32768, 8, 1024)):
        tr, pay = synthetic.shell_arrays(k, m)
        xf = api.compose(tr)
        renderer.set_scene_composed(xf, api.PrimitiveSlab(k, m, pay), api.WindowParams())
        cam = synthetic.shell_camera(-1, 0, w)
        rects, keys, offs, prims = renderer.debug_tiles(cam)
        ooffs, oprims = oracle.tile_lists(xf, cam)
        assert np.array_equal(offs, ooffs) and np.array_equal(prims, oprims), (k, m)


def test_expf_port_is_glibc_exact_on_window_range(renderer, oracle):
    """Every float in [-24, 0] (the window argument range at alpha = 8): device == libm expf."""
    lo, hi = 0x80000000, 0xC1C00000  # -0.0 .. -24.0
    step = 1 << 26
    bad = 0
    for start in range(lo, hi + 1, step):
        end = min(start + step - 1, hi)
        x = np.arange(start, end + 1, dtype=np.uint64).astype(np.uint32).view(np.float32)
        y = renderer.debug_expf(x)
        bad += oracle.expf_mismatches(start, end, y)
    assert bad == 0


def test_render_is_deterministic_and_stats_consistent(renderer):
    tr, pay = synthetic.shell_arrays(512, 8)
    renderer.set_scene_composed(api.compose(tr), api.PrimitiveSlab(512, 8, pay), api.WindowParams())
    cam = synthetic.shell_camera(7, 64, 512)
    a = renderer.render(cam, api.MarchConfig(jitter=True, seed=3))
    b = renderer.render(cam, api.MarchConfig(jitter=True, seed=3))
    c = renderer.render(cam, api.MarchConfig(jitter=True, seed=4))
    assert np.array_equal(bits(a.color), bits(b.color)) and np.array_equal(a.sample_counts, b.sample_counts)
    assert not np.array_equal(bits(a.color), bits(c.color))
    assert a.stats["ray_samples"] == a.total_samples()
    # a ray can intersect a segment shorter than the lattice spacing and take no sample
    assert a.stats["hit_rays"] >= int((a.sample_counts > 0).sum())


def test_composite_matches_reference_formula(renderer, oracle):
    rng = np.random.default_rng(1)
    out = api.RenderOutput(rng.uniform(0, 1, (24, 40, 3)).astype(np.float32),
                           rng.uniform(0, 1, (24, 40, 1)).astype(np.float32), np.zeros(960, np.int32))
    bg = rng.uniform(0, 1, (24, 40, 3)).astype(np.float32)
    got = renderer.composite(out, bg)
    want = oracle.composite(out.color, out.alpha, bg)
    assert_bit_equal("composite", got, want)
    with pytest.raises(api.Error) as e:
        renderer.composite(out, bg[:, :39])
    assert e.value.category == api.ErrorCategory.USAGE


def test_arbitrary_rays_through_the_bvh_equal_brute_force(renderer, oracle):
    """vp_march_rays prunes with the device BVH (vpb_bvh.cu); the result must equal the brute-
    force restatement (oracle: every primitive tested) bit-for-bit, for rays from outside,
    from far away, from inside the shell, axis-aligned and tangent to primitives."""
    tr, pay = synthetic.shell_arrays(4096, 4)
    xf = api.compose(tr)
    renderer.set_scene_composed(xf, api.PrimitiveSlab(4096, 4, pay), api.WindowParams())
    rng = np.random.default_rng(5)
    n = 6000
    u = rng.normal(size=(n, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    dist = np.concatenate([rng.uniform(0.4, 2.0, n // 3), rng.uniform(20, 200, n // 3),
                           rng.uniform(0.0, 0.3, n - 2 * (n // 3))])
    o = (u * dist[:, None]).astype(np.float32)
    target = rng.normal(scale=0.2, size=(n, 3))
    d = target - o
    d[: n // 10] = np.eye(3)[rng.integers(0, 3, n // 10)] * rng.choice([-1, 1], (n // 10, 1))
    # tangent rays: aimed at a random primitive's corner
    k = rng.integers(0, 4096, n // 10)
    corner = xf[k, 0:3] + (xf[k, 3:12].reshape(-1, 3, 3).transpose(0, 2, 1) @
                           (xf[k, 12:15] * rng.choice([-1, 1], (n // 10, 3)))[..., None])[..., 0]
    d[n // 10: n // 5] = corner - o[n // 10: n // 5]
    d = (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)
    cfg = api.MarchConfig()
    rgb, alpha, samples = renderer.march_rays(o, d, cfg)
    orgb, oalpha, osamples = oracle.march_rays(xf, 4, pay, api.WindowParams(), o, d, cfg)
    assert_bit_equal("rgb", rgb, orgb)
    assert_bit_equal("alpha", alpha, oalpha)
    assert_bit_equal("samples", samples, osamples)
    assert (samples > 0).sum() > n // 4


def test_async_render_into_host_memory_matches_sync(renderer):
    """vp_render_async with page-locked host outputs (two device slots, the copy of one view
    overlapping the next render) returns exactly what the synchronous vp_render returns."""
    import ctypes as C

    import torch
    from paper_2103_01954_b200._lib import f32p, i32p
    tr, pay = synthetic.shell_arrays(512, 8)
    renderer.set_scene_composed(api.compose(tr), api.PrimitiveSlab(512, 8, pay), api.WindowParams())
    w, views = 256, [0, 9, 17, 33, 50]
    cams = [synthetic.shell_camera(v, 64, w) for v in views]
    want = [renderer.render(c, api.MarchConfig()) for c in cams]
    rgb = torch.empty((len(views), w * w * 3), dtype=torch.float32, pin_memory=True)
    alpha = torch.empty((len(views), w * w), dtype=torch.float32, pin_memory=True)
    samples = torch.empty((len(views), w * w), dtype=torch.int32, pin_memory=True)
    lib, mc = renderer._lib, api.MarchConfig().to_c()
    for j, c in enumerate(cams):
        cc = c.to_c()
        assert lib.vp_render_async(renderer.ctx, C.byref(cc), C.byref(mc), C.cast(rgb[j].data_ptr(), f32p),
                                   C.cast(alpha[j].data_ptr(), f32p), C.cast(samples[j].data_ptr(), i32p),
                                   None) == 0
    assert lib.vp_sync(renderer.ctx) == 0
    for j, o in enumerate(want):
        assert_bit_equal("rgb", rgb[j].numpy().reshape(w, w, 3), o.color)
        assert_bit_equal("alpha", alpha[j].numpy().reshape(w, w, 1), o.alpha)
        assert_bit_equal("samples", samples[j].numpy(), o.sample_counts)


@pytest.mark.parametrize("k,m,w", [(32768, 4, 2048), (4096, 16, 3000)])
def test_tile_path_equals_ray_path_at_large_sizes(renderer, oracle, k, m, w):
    """A size-independent cross-check at sizes the CPU reference cannot run in a test: the
    tile pipeline (K1-K5) and the BVH ray path (vp_march_rays) are independent device
    implementations of the same bit-exact march, so every sampled pixel must agree bitwise
    (an image 3000 px wide also exercises partial edge tiles and 35k tiles)."""
    tr, pay = synthetic.shell_arrays(k, m)
    renderer.set_scene_composed(api.compose(tr), api.PrimitiveSlab(k, m, pay), api.WindowParams())
    cam = synthetic.shell_camera(7, 64, w)
    out = renderer.render(cam, api.MarchConfig())
    rng = np.random.default_rng(k)
    hit = np.flatnonzero(out.sample_counts > 0)
    pix = np.concatenate([rng.choice(hit, 12000, replace=False), rng.integers(0, w * w, 4000)])
    o = np.zeros((pix.size, 3), np.float32)
    d = np.zeros((pix.size, 3), np.float32)
    for i, p in enumerate(pix):
        o[i], d[i] = oracle.generate_ray(cam, float(p % w) + 0.5, float(p // w) + 0.5)
    rgb, alpha, samples = renderer.march_rays(o, d, api.MarchConfig())
    assert_bit_equal("rgb", rgb, out.color.reshape(-1, 3)[pix])
    assert_bit_equal("alpha", alpha, out.alpha.reshape(-1)[pix])
    assert_bit_equal("samples", samples, out.sample_counts[pix])


def test_batch_render_equals_single_views(renderer):
    """vp_render_batch_async marches the tiles of several views (different sizes) in one launch,
    heaviest first across views; every view must equal its own vp_render bit-for-bit."""
    import ctypes as C

    import torch
    from paper_2103_01954_b200._lib import f32p, i32p, vp_camera
    tr, pay = synthetic.shell_arrays(4096, 8)
    renderer.set_scene_composed(api.compose(tr), api.PrimitiveSlab(4096, 8, pay), api.WindowParams())
    specs = [(0, 256), (11, 200), (23, 333), (40, 128), (-1, 300)]
    cams = [synthetic.shell_camera(v, 64, w) if v >= 0 else synthetic.shell_camera(-1, 0, w) for v, w in specs]
    want = [renderer.render(c, api.MarchConfig()) for c in cams]
    outs = [(torch.empty(c.width * c.height * 3, device="cuda"), torch.empty(c.width * c.height, device="cuda"),
             torch.empty(c.width * c.height, dtype=torch.int32, device="cuda")) for c in cams]
    n = len(cams)
    cams_c = (vp_camera * n)(*[c.to_c() for c in cams])
    rgbp = (f32p * n)(*[C.cast(o[0].data_ptr(), f32p) for o in outs])
    ap = (f32p * n)(*[C.cast(o[1].data_ptr(), f32p) for o in outs])
    sp = (i32p * n)(*[C.cast(o[2].data_ptr(), i32p) for o in outs])
    mc = api.MarchConfig().to_c()
    lib = renderer._lib
    from paper_2103_01954_b200._lib import vp_stats
    for _ in range(2):  # twice: both slot groups
        assert lib.vp_render_batch_async(renderer.ctx, n, cams_c, C.byref(mc), rgbp, ap, sp, None) == 0
        st = vp_stats()
        assert lib.vp_read_stats(renderer.ctx, C.byref(st)) == 0  # summed over the batch's views
        assert st.ray_samples == sum(ww.stats["ray_samples"] for ww in want)
        assert st.prim_samples == sum(ww.stats["prim_samples"] for ww in want)
        for o, ww, c in zip(outs, want, cams):
            assert_bit_equal("rgb", o[0].cpu().numpy().reshape(c.height, c.width, 3), ww.color)
            assert_bit_equal("alpha", o[1].cpu().numpy().reshape(c.height, c.width, 1), ww.alpha)
            assert_bit_equal("samples", o[2].cpu().numpy(), ww.sample_counts)
    # host outputs (page-locked): copied out while the next batch renders
    hosts = [(torch.empty(c.width * c.height * 3, pin_memory=True), torch.empty(c.width * c.height, pin_memory=True),
              torch.empty(c.width * c.height, dtype=torch.int32, pin_memory=True)) for c in cams]
    hrgb = (f32p * n)(*[C.cast(o[0].data_ptr(), f32p) for o in hosts])
    ha = (f32p * n)(*[C.cast(o[1].data_ptr(), f32p) for o in hosts])
    hs = (i32p * n)(*[C.cast(o[2].data_ptr(), i32p) for o in hosts])
    for _ in range(3):
        assert lib.vp_render_batch_async(renderer.ctx, n, cams_c, C.byref(mc), hrgb, ha, hs, None) == 0
    assert lib.vp_sync(renderer.ctx) == 0
    for o, ww, c in zip(hosts, want, cams):
        assert_bit_equal("rgb", o[0].numpy().reshape(c.height, c.width, 3), ww.color)
        assert_bit_equal("alpha", o[1].numpy().reshape(c.height, c.width, 1), ww.alpha)
        assert_bit_equal("samples", o[2].numpy(), ww.sample_counts)


def test_async_transform_updates_between_batches(renderer):
    """vp_set_transforms_async between batches (new poses every batch, no host sync): each
    batch sees exactly its own transforms (compared with synchronous renders)."""
    import ctypes as C

    import torch
    from paper_2103_01954_b200._lib import f32p, i32p, vp_camera
    tr, pay = synthetic.shell_arrays(512, 8)
    poses = []
    for q in range(3):
        t = tr.copy()
        t[:, 15:18] += np.float32(0.01 * q)
        poses.append(api.compose(t))
    renderer.set_scene_composed(poses[0], api.PrimitiveSlab(512, 8, pay), api.WindowParams())
    cams = [synthetic.shell_camera(v, 64, 160) for v in (3, 30)]
    want = []
    for xf in poses:
        renderer.set_transforms(xf)
        want.append([renderer.render(c, api.MarchConfig()) for c in cams])
    renderer.set_transforms(poses[0])
    lib, mc = renderer._lib, api.MarchConfig().to_c()
    n = len(cams)
    cams_c = (vp_camera * n)(*[c.to_c() for c in cams])
    pinned = [torch.from_numpy(np.ascontiguousarray(xf)).pin_memory() for xf in poses]
    outs = [[(torch.empty(160 * 160 * 3, pin_memory=True), torch.empty(160 * 160, pin_memory=True),
              torch.empty(160 * 160, dtype=torch.int32, pin_memory=True)) for _ in cams] for _ in poses]
    for q, xf in enumerate(pinned):
        assert lib.vp_set_transforms_async(renderer.ctx, 512, C.cast(xf.data_ptr(), f32p), None) == 0
        rgbp = (f32p * n)(*[C.cast(o[0].data_ptr(), f32p) for o in outs[q]])
        ap = (f32p * n)(*[C.cast(o[1].data_ptr(), f32p) for o in outs[q]])
        sp = (i32p * n)(*[C.cast(o[2].data_ptr(), i32p) for o in outs[q]])
        assert lib.vp_render_batch_async(renderer.ctx, n, cams_c, C.byref(mc), rgbp, ap, sp, None) == 0
    assert lib.vp_sync(renderer.ctx) == 0
    for q in range(3):
        for o, ww in zip(outs[q], want[q]):
            assert_bit_equal("rgb", o[0].numpy().reshape(160, 160, 3), ww.color)
            assert_bit_equal("samples", o[2].numpy(), ww.sample_counts)


@pytest.mark.parametrize("group", range(8))
def test_ring_views_batched_match_reference(renderer, group):
    """All 64 views of BASELINE config 5 (the bench's timed views included), 8 per raymarch launch
    through vp_render_batch_async, against the reference's per-view digests
    (oracle/gen_ring_digests.py)."""
    ring = DIGESTS["ring"]
    k, m, w, n = ring["K"], ring["M"], ring["W"], ring["n_views"]
    if renderer.n_prim != k or renderer.m != m:
        tr, pay = synthetic.shell_arrays(k, m)
        renderer.set_scene_composed(api.compose(tr), api.PrimitiveSlab(k, m, pay), api.WindowParams())
    views = list(range(8 * group, 8 * group + 8))
    outs = renderer.render_batch([synthetic.shell_camera(v, n, w) for v in views], api.MarchConfig())
    for v, out in zip(views, outs):
        d = ring["views"][str(v)]
        assert out.total_samples() == d["total_samples"], f"view {v}"
        assert sha(out.sample_counts) == d["samples"], f"view {v} samples"
        assert sha(out.alpha) == d["alpha"], f"view {v} alpha"
        assert sha(out.color) == d["rgb"], f"view {v} rgb"


@pytest.mark.parametrize("n", [1, 2, 2047, 2048, 2049, 4096, 32768, 262144, 1 << 20])
def test_bvh_radix_sort_is_stable_and_sorted(renderer, n):
    """The in-house LSD radix sort that orders the device LBVH's (Morton << 32 | prim) keys
    (vpb_bvh.cu, replacing buildLbvh's sort, lbvh.cpp:81-100): sorted on bits [32, 62) and stable,
    i.e. the order of the full 62-bit keys, with many duplicate codes."""
    import ctypes as C
    rng = np.random.default_rng(n)
    codes = rng.integers(0, 1 << 30, n, dtype=np.uint64)
    codes[: n // 3] = codes[0]  # a run of equal codes (stability)
    codes[n // 3: n // 2] &= np.uint64(0xff)  # only the low digit differs
    rng.shuffle(codes)
    keys = (codes << np.uint64(32)) | np.arange(n, dtype=np.uint64)
    out = np.zeros(n, np.uint64)
    p64 = C.POINTER(C.c_uint64)
    rc = renderer._lib.vp_debug_radix_sort(renderer.ctx, n, keys.ctypes.data_as(p64), out.ctypes.data_as(p64))
    assert rc == 0
    assert np.array_equal(out, np.sort(keys))


def test_bvh_refits_across_pose_changes_stay_exact(renderer, oracle):
    """A pose change refits the previous build's BVH topology (rebuilt every 16 poses): after
    each of 20 perturbations of every primitive's deltas (set_records), the rays through the
    refitted (or rebuilt) hierarchy still equal the brute-force restatement bit for bit."""
    k, m = 1024, 4
    tr, pay = synthetic.shell_arrays(k, m)
    renderer.set_scene_records(tr, api.PrimitiveSlab(k, m, pay), api.WindowParams())
    rng = np.random.default_rng(9)
    n = 600
    u = rng.normal(size=(n, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    o = (u * rng.uniform(0.5, 2.0, (n, 1))).astype(np.float32)
    d = rng.normal(scale=0.2, size=(n, 3)) - o
    d = (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)
    cfg = api.MarchConfig()
    cur = tr.copy()
    for it in range(20):
        cur[:, 15:18] += rng.normal(scale=0.004, size=(k, 3)).astype(np.float32)  # deltaT
        cur[:, 18:21] += rng.normal(scale=0.05, size=(k, 3)).astype(np.float32)   # deltaR
        renderer.set_records(cur)
        xf = api.compose(cur)
        rgb, alpha, samples = renderer.march_rays(o, d, cfg)
        orgb, oalpha, osamples = oracle.march_rays(xf, m, pay, api.WindowParams(), o, d, cfg)
        assert_bit_equal(f"rgb[{it}]", rgb, orgb)
        assert_bit_equal(f"alpha[{it}]", alpha, oalpha)
        assert_bit_equal(f"samples[{it}]", samples, osamples)

"""TEST INFRASTRUCTURE — generates tests/golden/* from the REAL reference.

Every expected output in the fixtures is produced by the unmodified reference core
(oracle/_ref/libvolprim_ref.so, built by oracle/Makefile from /root/reference/proj/src);
inputs come from numpy seeds stored alongside them, or from libvpb's host-only synthetic
scene generator (whose output digest is stored so generator drift is detected).

    python oracle/gen_golden.py            # writes tests/golden/*.npz and digests.json

The reference has no stored golden vectors of its own; the scenarios here
follow its own tests: test_march.cpp:50-247, test_lbvh.cpp:145-210, acceptance.cpp:58-190.
"""
from __future__ import annotations

import hashlib
import json
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle.bindings import RefCore  # noqa: E402
from paper_2103_01954_b200 import api, synthetic  # noqa: E402

OUT = ROOT / "tests" / "golden"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def unit_box(t, scale=(1, 1, 1)):
    """AffineXf-equivalent PrimitiveTransform: identity rotation (test_march.cpp:26-31)."""
    return api.transform_records([t], [np.eye(3)], [scale])


def random_boxes(rng, n, spread=1.0, smin=0.02, smax=0.1, rot=2.0):
    """acceptance.cpp:64-75-style random rotated boxes."""
    t = rng.uniform(-spread, spread, (n, 3))
    s = smin + (smax - smin) * np.abs(rng.uniform(-1, 1, (n, 3)))
    dr = rng.uniform(-1, 1, (n, 3)) * rot
    return api.transform_records(t, np.tile(np.eye(3), (n, 1, 1)), s, delta_r=dr)


def fill_constant(k, m, rgb, sigma):
    p = np.zeros((k, 4, m, m, m), np.float32)
    for i in range(k):
        for c in range(3):
            p[i, c] = rgb[i][c]
        p[i, 3] = sigma[i]
    return p.reshape(-1)


def cam_dict(cam: api.Camera):
    return dict(K=np.asarray(cam.intrinsics, np.float32), R=np.asarray(cam.rotation, np.float32),
                t=np.asarray(cam.translation, np.float32), wh=np.array([cam.width, cam.height], np.int32))


def simple_camera(f, cx, cy, R, t, w, h):
    K = np.array([[f, 0, cx], [0, f, cy], [0, 0, 1]], np.float32)
    return api.Camera(K, np.asarray(R, np.float32), np.asarray(t, np.float32), w, h)


def render_case(ref, name, tr, m, payload, window, cam, cfg, store, meta, gen=None):
    """gen=(K, M): inputs come from synthetic.shell_arrays and are not stored (digest only)."""
    t0 = time.time()
    rgb, alpha, samples = ref.render(tr, m, payload, window, cam, cfg)
    meta[name] = dict(seconds=round(time.time() - t0, 3), total_samples=int(samples.sum()),
                      hit_pixels=int((samples > 0).sum()))
    inputs = (dict(gen=np.array(gen, np.int32), tr_sha=np.array(sha(tr)), payload_sha=np.array(sha(payload)))
              if gen else dict(tr=np.asarray(tr, np.float32).reshape(-1, 24), payload=np.asarray(payload, np.float32)))
    d = dict(m=np.int32(m), **inputs, window=np.array([window.alpha, window.beta], np.float32),
             cfg=np.array([cfg.step_size, cfg.early_eps, float(cfg.jitter), float(cfg.seed)], np.float64),
             rgb=rgb, alpha=alpha, samples=samples, **cam_dict(cam))
    store[name] = d


def main():
    ref = RefCore()
    OUT.mkdir(parents=True, exist_ok=True)
    digests = {"generator": {}, "renders": {}, "meta": {}}
    rng = np.random.default_rng(20261018)

    # -- compose (primitive.cpp:41-49) incl. the small-angle series branch -----------------
    n = 256
    tr = random_boxes(rng, n, rot=1.0)
    tr[:32, 18:21] *= 1e-5          # theta < 1e-4 branch
    tr[32:40, 18:21] = 0            # identity branch
    tr[40:48, 21:24] = rng.uniform(-0.01, 0.0, (8, 3)).astype(np.float32)
    rc, xf = ref.compose(tr)
    assert rc == 0
    bad = tr[:4].copy()
    bad[2, 21] = -bad[2, 12] - 0.5  # non-positive composed scale -> Usage
    rc_bad, _ = ref.compose(bad)
    np.savez_compressed(OUT / "compose.npz", tr=tr, xf=xf, bad=bad, rc_bad=np.int32(rc_bad))

    # -- cameras: lookAtCamera (synthetic.cpp:15-38) and generateRay (camera.cpp:14-23) ----
    cams = {}
    for name, (pos, w) in {"headline_256": ((0.25, 0.15, -1.1), 256),
                           "headline_1024": ((0.25, 0.15, -1.1), 1024),
                           "above": ((0.0, 2.0, 0.0), 64), "oblique": ((-0.7, -0.3, 0.9), 96)}.items():
        k9, r9, t3, aa = ref.look_at(pos, (0, 0, 0), (0, 1, 0), np.float32(1.2 * w), w, w)
        cams[name] = np.concatenate([k9, r9, t3, aa, np.array(pos, np.float32), [np.float32(1.2 * w), w]])
    cam = synthetic.shell_camera(-1, 0, 64)
    px = rng.uniform(0, 64, (500, 2)).astype(np.float32)
    rays = np.array([np.concatenate(ref.generate_ray(cam, x, y)) for x, y in px], np.float32)
    np.savez_compressed(OUT / "cameras.npz", rays_px=px, rays=rays, **cam_dict(cam),
                        **{f"lookat_{k}": v for k, v in cams.items()})

    # -- intersect (lbvh.cpp:177-234), test_lbvh.cpp:184-210-style random scene -------------
    tr = random_boxes(rng, 300)
    _, xf = ref.compose(tr)
    o = (2 * rng.uniform(-1, 1, (400, 3))).astype(np.float32)
    d = rng.normal(size=(400, 3))
    d = (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)
    o[:20] = xf[:20, :3]  # origins inside boxes: enterClamped
    segs = []
    for i in range(len(o)):
        p, te, tx = ref.intersect(xf, o[i], d[i])
        segs.append(np.stack([p.astype(np.float32), te, tx], 1) if len(p) else np.zeros((0, 3), np.float32))
    lens = np.array([len(s) for s in segs], np.int32)
    np.savez_compressed(OUT / "intersect.npz", xf=xf, origins=o, dirs=d, lens=lens,
                        segs=np.concatenate(segs) if segs else np.zeros((0, 3), np.float32))

    # -- march() KATs over explicit rays (test_march.cpp:50-194) -----------------------------
    kats = {}
    axial_o, axial_d = np.array([[0.1, -0.2, -3]], np.float32), np.array([[0, 0, 1]], np.float32)
    no_win = api.WindowParams(0, 8)

    def kat(name, trs, m, pay, win, cfg, o=axial_o, d=axial_d, jit=None):
        _, xf_ = ref.compose(trs)
        rgb, alpha, samples = ref.march_rays(xf_, m, pay, win, o, d, cfg, jit)
        kats[name] = dict(xf=xf_, m=np.int32(m), payload=pay, window=np.array([win.alpha, win.beta], np.float32),
                          cfg=np.array([cfg.step_size, cfg.early_eps], np.float32), o=o, d=d,
                          jit=np.full(len(o), 0.5, np.float32) if jit is None else jit,
                          rgb=rgb, alpha=alpha, samples=samples)

    kat("constant_medium", unit_box((0, 0, 0)), 4, fill_constant(1, 4, [(0.8, 0.4, 0.2)], [0.2]), no_win,
        api.MarchConfig(0.001, 1e-6))
    kat("saturation", unit_box((0, 0, 0)), 2, fill_constant(1, 2, [(0.3, 0.9, 0.5)], [2.0]), no_win,
        api.MarchConfig(0.001, 1e-7))
    two = np.concatenate([unit_box((0, 0, 0)), unit_box((0, 0, 0))])
    kat("overlap", two, 2, fill_constant(2, 2, [(1, 0, 0), (0, 1, 0)], [0.1, 0.15]), no_win,
        api.MarchConfig(0.001, 1e-6))
    three = np.concatenate([unit_box((0, 0, 0)), unit_box((0.05, 0, 0.2)), unit_box((-0.1, 0.1, -0.3))])
    kat("order", three, 2, fill_constant(3, 2, [(1, .2, 0), (0, 1, .4), (.5, 0, 1)], [.3, .4, .5]), no_win,
        api.MarchConfig(0.002, 1e-6))
    gap = np.concatenate([unit_box((0, 0, 0)), unit_box((0, 0, 4))])
    kat("gap", gap, 2, fill_constant(2, 2, [(1, 0, 0), (0, 1, 0)], [0.1, 0.1]), no_win,
        api.MarchConfig(0.001, 1e-6))
    kat("early_exact", unit_box((0, 0, 0)), 2, fill_constant(1, 2, [(.5, .5, .5)], [0.49]), no_win,
        api.MarchConfig(0.001, 1e-7))
    kat("early_lazy", unit_box((0, 0, 0)), 2, fill_constant(1, 2, [(.5, .5, .5)], [0.49]), no_win,
        api.MarchConfig(0.001, 0.05))
    kat("window", unit_box((0, 0, 0)), 2, fill_constant(1, 2, [(1, 1, 1)], [0.3]), api.WindowParams(8, 8),
        api.MarchConfig(0.001, 1e-6), o=np.array([[0.8, 0, -3]], np.float32))
    # random rays through random rotated boxes with random payloads and jitter
    trs = random_boxes(rng, 60, spread=0.5, smin=0.05, smax=0.25)
    m = 4
    pay = rng.uniform(0, 1, (60, 4, m, m, m)).astype(np.float32)
    pay[:, 3] *= 8
    o = (rng.uniform(-1, 1, (256, 3)) * 0.2 + np.array([0, 0, -2])).astype(np.float32)
    d = (np.array([0, 0, 1]) + rng.normal(size=(256, 3)) * 0.15)
    d = (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)
    jit = rng.uniform(0, 1, 256).astype(np.float32)
    kat("random_rays", trs, m, pay.reshape(-1), api.WindowParams(8, 8), api.MarchConfig(0.002, 0.01), o, d, jit)
    np.savez_compressed(OUT / "march_kats.npz",
                        **{f"{k}__{f}": v for k, d_ in kats.items() for f, v in d_.items()})

    # -- backward pass: backwardRay (grad.cpp:34-195) with given output adjoints ---------------
    bwd = {}

    def bcase(name, trs, m, pay, win, cfg, o, d, jit, ar, aa):
        g = ref.backward_rays(trs, m, pay, win, o, d, ar, aa, cfg, jit)
        bwd[name] = dict(tr=np.asarray(trs, np.float32), m=np.int32(m), payload=np.asarray(pay, np.float32),
                         window=np.array([win.alpha, win.beta], np.float32),
                         cfg=np.array([cfg.step_size, cfg.early_eps], np.float32), o=o, d=d, jit=jit,
                         adj_rgb=ar, adj_alpha=aa, grads=g)

    nb, mb = 40, 4
    trs = api.transform_records(rng.uniform(-0.5, 0.5, (nb, 3)), np.tile(np.eye(3), (nb, 1, 1)),
                                0.05 + 0.2 * np.abs(rng.uniform(-1, 1, (nb, 3))),
                                delta_t=rng.uniform(-0.02, 0.02, (nb, 3)), delta_r=rng.uniform(-1, 1, (nb, 3)))
    pay = rng.uniform(0, 1, (nb, 4, mb, mb, mb)).astype(np.float32)
    pay[:, 3] *= 8
    nr = 512
    o = (rng.uniform(-1, 1, (nr, 3)) * 0.25 + np.array([0, 0, -2])).astype(np.float32)
    d = np.array([0, 0, 1]) + rng.normal(size=(nr, 3)) * 0.15
    d = (d / np.linalg.norm(d, axis=1, keepdims=True)).astype(np.float32)
    o[:16] = np.asarray(api.compose(trs)[:16, :3])  # origins inside boxes: no anchor chain
    jit = rng.uniform(0, 1, nr).astype(np.float32)
    ar = rng.normal(size=(nr, 3)).astype(np.float32)
    aa = rng.normal(size=nr).astype(np.float32)
    bcase("boxes_unsaturated", trs, mb, pay.reshape(-1), api.WindowParams(8, 8), api.MarchConfig(0.002, 0.01),
          o, d, jit, ar, aa)
    pay2 = pay.copy()
    pay2[:, 3] *= 6
    bcase("boxes_saturating", trs, mb, pay2.reshape(-1), api.WindowParams(8, 8), api.MarchConfig(0.002, 1e-7),
          o, d, jit, ar, aa)
    trs8, pays8 = synthetic.shell_arrays(64, 8)
    camb = synthetic.shell_camera(-1, 0, 64)
    from oracle.bindings import Oracle
    orc = Oracle()
    pix = rng.integers(0, 64, (nr, 2))
    rays = np.array([np.concatenate(orc.generate_ray(camb, x + 0.5, y + 0.5)) for x, y in pix], np.float32)
    bcase("shell64_m8_camera_rays", trs8, 8, pays8, api.WindowParams(8, 8), api.MarchConfig(0.001, 0.01),
          rays[:, :3].copy(), rays[:, 3:].copy(), np.full(nr, 0.5, np.float32), ar, aa)
    np.savez_compressed(OUT / "backward.npz", **{f"{k}__{f}": v for k, d_ in bwd.items() for f, v in d_.items()})

    # -- evalLoss (grad.cpp:197-251) and adamStep (losses.cpp:70-104) ---------------------------
    from oracle.bindings import ref_adam_run, ref_eval_loss
    cams = [synthetic.shell_camera(v, 16, 48) for v in (0, 5, 11)]
    ns = 600
    ci = rng.integers(0, 3, ns).astype(np.int32)
    pid = rng.integers(0, 48 * 48, ns).astype(np.int32)
    pxy = np.stack([(pid % 48) + 0.5, (pid // 48) + 0.5], 1).astype(np.float32)
    tgt = rng.uniform(0, 1, (ns, 3)).astype(np.float32)
    bgs = rng.uniform(0, 1, (ns, 3)).astype(np.float32)
    trl = trs8.copy()
    trl[:, 15:24] = rng.uniform(-0.01, 0.01, (64, 9)).astype(np.float32)
    wts = np.array([1.0, 0.1, 0.01, 0.01], np.float32)
    ecfg = api.MarchConfig(0.002, 0.01, True, 3)
    terms, gl = ref_eval_loss(ref, trl, 8, pays8, api.WindowParams(8, 8), cams, ci, pxy, pid, tgt, bgs,
                              [wts[0], wts[2], wts[3]], ecfg)
    camarr = np.stack([np.concatenate([c.intrinsics.reshape(-1), c.rotation.reshape(-1), c.translation,
                                       [c.width, c.height]]) for c in cams]).astype(np.float32)
    adam_cfg = np.array([1e-3, 0.9, 0.999, 1e-8, 0.1, 1.0], np.float32)
    na = nb * 4 * mb ** 3 + 9 * nb  # Adam on the 40-box scene (small fixture)
    gseq = (rng.normal(size=(3, na)) * 0.05).astype(np.float32)
    gseq[1, 5] = 0  # a zero-gradient parameter
    pay_in = pay.reshape(-1).copy()
    pay_in[:50] = 1e-5  # some payload entries pushed below zero by the step -> projected
    tr_in = trs.copy()
    tr_in[3, 21] = -tr_in[3, 12] + 2e-4  # composed scale near the 1e-4 floor -> projected
    tr_out, pay_out = ref_adam_run(ref, tr_in, mb, pay_in, gseq, adam_cfg)
    np.savez_compressed(OUT / "train.npz", tr=trl, m=np.int32(8), window=np.array([8, 8], np.float32),
                        cams=camarr, cam_index=ci, pixel=pxy, pixel_id=pid, target=tgt, background=bgs,
                        weights=wts, cfg=np.array([0.002, 0.01, 1, 3], np.float64), terms=terms, grads=gl,
                        adam_cfg=adam_cfg, adam_m=np.int32(mb), adam_grads=gseq, adam_tr_in=tr_in,
                        adam_pay_in=pay_in, adam_tr_out=tr_out, adam_pay_out=pay_out,
                        payload_sha=np.array(sha(pays8)))

    # -- full renders (march.cpp:95-132) -------------------------------------------------------
    store, meta = {}, digests["meta"]
    tr, pay = synthetic.shell_arrays(64, 16)
    render_case(ref, "shell64_m16_w64", tr, 16, pay, api.WindowParams(), synthetic.shell_camera(-1, 0, 64),
                api.MarchConfig(), store, meta, gen=(64, 16))
    tr8, pay8 = synthetic.shell_arrays(64, 8)
    render_case(ref, "shell64_m8_w48_jitter", tr8, 8, pay8, api.WindowParams(),
                synthetic.shell_camera(5, 16, 48), api.MarchConfig(0.001, 0.01, True, 7), store, meta, gen=(64, 8))
    trb = random_boxes(rng, 300, spread=0.6, smin=0.03, smax=0.15)
    payb = rng.uniform(0, 1, (300, 4, 4, 4, 4)).astype(np.float32)
    payb[:, 3] *= 30
    camb = simple_camera(80.0, 47.0, 33.0, np.eye(3), (0.05, -0.02, 2.5), 96, 72)
    render_case(ref, "random_boxes_96x72", trb, 4, payb.reshape(-1), api.WindowParams(8, 8), camb,
                api.MarchConfig(0.003, 0.01), store, meta)
    # camera inside a primitive (enterClamped) plus primitives straddling the camera plane
    tri = np.concatenate([unit_box((0, 0, 0.5), (0.8, 0.8, 1.5)), random_boxes(rng, 40, spread=0.7)])
    payi = rng.uniform(0, 1, (41, 4, 2, 2, 2)).astype(np.float32)
    payi[:, 3] *= 3
    cami = simple_camera(40.0, 20.0, 16.0, np.eye(3), (0, 0, 0), 40, 32)
    render_case(ref, "camera_inside_40x32", tri, 2, payi.reshape(-1), api.WindowParams(8, 8), cami,
                api.MarchConfig(0.002, 0.01), store, meta)
    render_case(ref, "window_off", tr8, 8, pay8, api.WindowParams(0, 8), synthetic.shell_camera(2, 8, 40),
                api.MarchConfig(0.0015, 0.02), store, meta, gen=(64, 8))
    render_case(ref, "beta4", tr8, 8, pay8, api.WindowParams(3, 4), synthetic.shell_camera(3, 8, 40),
                api.MarchConfig(0.0015, 0.02), store, meta, gen=(64, 8))
    # test_march.cpp:216-247 scene
    trd = api.transform_records([(0, 0, 0)], [np.eye(3)], [(0.4, 0.4, 0.2)])
    payd = fill_constant(1, 4, [(0.7, 0.3, 0.5)], [2.0])
    camd = simple_camera(40.0, 16.0, 16.0, np.eye(3), (0, 0, 2), 32, 32)
    render_case(ref, "deterministic_jitter_32", trd, 4, payd, api.WindowParams(8, 8), camd,
                api.MarchConfig(0.005, 0.01, True, 7), store, meta)
    # M = 1 (single voxel) and an empty scene
    payone = rng.uniform(0, 1, (300, 4, 1, 1, 1)).astype(np.float32)
    payone[:, 3] *= 30
    render_case(ref, "m1_boxes_48", trb, 1, payone.reshape(-1), api.WindowParams(8, 8),
                simple_camera(50.0, 24.0, 24.0, np.eye(3), (0, 0, 2.5), 48, 48), api.MarchConfig(0.004, 0.01),
                store, meta)
    render_case(ref, "empty_scene", np.zeros((0, 24), np.float32), 4, np.zeros(0, np.float32),
                api.WindowParams(), simple_camera(10.0, 8.0, 8.0, np.eye(3), (0, 0, 2), 16, 16),
                api.MarchConfig(), store, meta)
    np.savez_compressed(OUT / "renders.npz", **{f"{k}__{f}": v for k, d_ in store.items() for f, v in d_.items()})

    # -- full-size digests (BASELINE.json configs 1-4 + four views of config 5) --------------
    for name, (k, m, w) in synthetic.CONFIGS.items():
        tr, pay = synthetic.shell_arrays(k, m)
        digests["generator"][f"{k}x{m}"] = {"tr": sha(tr), "payload": sha(pay)}
        views = [-1] if name != "k4096_m16_1024" else [-1, 0, 16, 32, 48]
        for v in views:
            cam = synthetic.shell_camera(v, 64, w)
            t0 = time.time()
            rgb, alpha, samples = ref.render(tr, m, pay, api.WindowParams(), cam, api.MarchConfig())
            key = f"{name}_view{v}"
            digests["renders"][key] = {
                "K": k, "M": m, "W": w, "view": v, "n_views": 64,
                "rgb": sha(rgb), "alpha": sha(alpha), "samples": sha(samples),
                "total_samples": int(samples.sum()), "hit_pixels": int((samples > 0).sum()),
                "rgb_sum": float(rgb.astype(np.float64).sum()), "alpha_sum": float(alpha.astype(np.float64).sum()),
                "ref_seconds": round(time.time() - t0, 3)}
            print(key, digests["renders"][key]["total_samples"], digests["renders"][key]["ref_seconds"], flush=True)
    (OUT / "digests.json").write_text(json.dumps(digests, indent=1, sort_keys=True))
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()

"""Randomized parity campaign (testing helper): random box scenes, cameras, image sizes, march
configs, tile tiers and forced key capacities, rendered through vp_render (sync) and
vp_render_batch_async (several views in one launch), each compared bit for bit with the C
restatement (oracle/vp_oracle.c, pinned to the reference). Usage (GPU): python tools/fuzz_parity.py [n] [seed]"""
import os
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/", 2)[0])
from oracle.bindings import Oracle  # noqa: E402
from paper_2103_01954_b200 import Renderer, api, synthetic  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
orc = Oracle()
fails = limits = 0
for case in range(n_cases):
    rng = np.random.default_rng(seed0 + case)
    k = int(rng.integers(1, 1500))
    m = int(rng.choice([1, 2, 3, 4, 5, 8]))
    spread = float(rng.uniform(0.05, 0.8))
    smin = float(rng.uniform(0.005, 0.05))
    smax = smin + float(rng.uniform(0.01, 0.4))
    t = rng.uniform(-spread, spread, (k, 3))
    s = smin + (smax - smin) * np.abs(rng.uniform(-1, 1, (k, 3)))
    tr = api.transform_records(t, np.tile(np.eye(3), (k, 1, 1)), s, delta_r=rng.uniform(-3, 3, (k, 3)))
    pay = rng.uniform(0, 1, k * 4 * m ** 3).astype(np.float32)
    pay.reshape(k, 4, -1)[:, 3] *= np.float32(rng.uniform(0.1, 80))
    xf = api.compose(tr)
    w, h = int(rng.integers(8, 200)), int(rng.integers(8, 200))
    dist = float(rng.uniform(0.1, 3.0))
    cfg = api.MarchConfig(step_size=float(rng.uniform(0.002, 0.01)), early_eps=float(rng.choice([0.01, 1e-4, 0.05])),
                          jitter=bool(rng.integers(0, 2)), seed=int(rng.integers(0, 1000)))
    win = api.WindowParams(float(rng.choice([0.0, 8.0, 3.0])), int(rng.choice([8, 4, 2])))
    cams = []
    for v in range(int(rng.integers(1, 5))):
        az = rng.uniform(0, 2 * np.pi)
        pos = (dist * np.sin(az), float(rng.uniform(-0.5, 0.5)) * dist, -dist * np.cos(az))
        cam, _ = synthetic.look_at_camera(pos, (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), float(rng.uniform(0.5, 1.5)) * w, w, h)
        cams.append(cam)
    tier = str(rng.choice(["auto", "light", "normal", "dense"]))
    if tier != "auto":
        os.environ["VPB_TILE_CFG"] = tier
    else:
        os.environ.pop("VPB_TILE_CFG", None)
    r = Renderer(0)
    try:
        r.set_scene_composed(xf, api.PrimitiveSlab(k, m, pay), win)
        cap = int(rng.choice([0, 0, 50, 500]))
        if cap:
            r.set_key_capacity(cap, grow=False)
        try:
            outs = [r.render(c, cfg) for c in cams] if rng.integers(0, 2) else r.render_batch(cams, cfg)
        except api.Error as e:  # the documented window limit (kFallbackCap live segments)
            print(f"case {case}: {e} (K={k} spread={spread:.2f} smax={smax:.2f})", flush=True)
            limits += 1
            continue
    finally:
        r.close()
    for j, (c, out) in enumerate(zip(cams, outs)):
        rgb, alpha, samples = orc.render(xf, m, pay, win, c, cfg)
        ok = (np.array_equal(out.sample_counts, samples) and np.array_equal(out.alpha.view(np.uint32), alpha.view(np.uint32))
              and np.array_equal(out.color.view(np.uint32), rgb.view(np.uint32)))
        if not ok:
            fails += 1
            print(f"case {case} view {j} FAILED: K={k} M={m} {w}x{h} tier={tier} cap={cap} cfg={cfg} win={win}", flush=True)
print(f"fuzz: {n_cases} cases, {fails} failing views, {limits} cases over the live-segment limit")
sys.exit(1 if fails else 0)

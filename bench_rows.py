#!/usr/bin/env python
"""Measurement of the SURVEY.md §8(f) rows next to the raymarcher (bench.py measures the
headline path). One JSON line per row, same keys as bench.py where they apply.

  python bench_rows.py [--rows fit,backward,compose,load] [--steps K] [--warmup W]

Rows (all on the headline scene, mvp_shell K=4096 x 16^3, unless stated):
  fit       one fit iteration (fit.cpp:135-200 minus data loading): evalLoss on 8 images x 256
            random pixels of the 64-view ring at 1024^2 (fit.h:18-19 defaults): rays, march,
            composite, L_pho, backwardRay into a device GradBuffer, L_vol + L_del on the host;
            then adamStep over [payload | deltas] (268.5 M parameters) with the projection and
            the device recompose. Metric: iterations/s, host wall time per iteration (every
            C-ABI call is synchronous). Roofline: the Adam pass, 32 B per parameter (gradient
            read twice: finiteness check + update; m1, m2, parameter read + written).
  backward  backwardRay for 65,536 hit pixels of the headline view (vp_backward_rays, device
            arrays). Metric: rays/s. Roofline: 256 B per primitive-sample (8 corners x 4
            channels read for the adjoint walk + the same scattered as gradient atomics).
  compose   Frame::composed() for K=32768 records on the device (vp_set_frame, host records).
  load      loadSlab of the headline slab (268 MB VPSL file in the page cache) straight into
            the device layout (vp_load_slab).
cpu_baseline: the unmodified reference (oracle/_ref) on the same inputs, bounded sample,
single-threaded like the reference's own fit loop / loaders.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import pathlib
import sys
import tempfile
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from bench import ClockSampler, peaks  # noqa: E402


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--rows", default="fit,backward,compose,load")
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def ref_core():
    from oracle.bindings import RefCore
    return RefCore() if RefCore.available() else None


def emit(row: dict):
    print(json.dumps(row), flush=True)


def device_events(torch, lib, r):
    stream = torch.cuda.ExternalStream(lib.vp_stream(r.ctx))
    return stream, lambda: torch.cuda.Event(enable_timing=True)


# -----------------------------------------------------------------------------------------
def row_fit(args, torch, r, lib, api, synthetic, ref):
    from paper_2103_01954_b200._lib import f32p, i32p, vp_adam, vp_camera
    k, m, w = 4096, 16, 1024
    tr0, pay = synthetic.shell_arrays(k, m)
    r.set_scene_records(tr0, api.PrimitiveSlab(k, m, pay), api.WindowParams())
    cams = [synthetic.shell_camera(v, 64, w) for v in range(64)]
    cams_c = (vp_camera * 64)(*[c.to_c() for c in cams])
    n_imgs, per_img = 8, 256
    n = n_imgs * per_img
    rng = np.random.default_rng(1)

    def batch():
        ci = np.repeat(rng.choice(64, n_imgs, replace=False), per_img).astype(np.int32)
        pid = np.concatenate([rng.choice(w * w, per_img, replace=False) for _ in range(n_imgs)]).astype(np.int32)
        xy = np.stack([pid % w + 0.5, pid // w + 0.5], 1).astype(np.float32)
        tg = rng.uniform(0, 1, (n, 3)).astype(np.float32)
        bg = rng.uniform(0, 1, (n, 3)).astype(np.float32)
        return ci, xy, pid, tg, bg

    batches = [batch() for _ in range(args.warmup + args.steps)]
    n_pay = k * 4 * m ** 3
    n_par = n_pay + 9 * k
    grads = torch.zeros(n_par, dtype=torch.float32, device="cuda")
    gptr = C.cast(C.c_void_p(grads.data_ptr()), f32p)
    pose = np.zeros(9 * k, np.float32)
    tr = np.ascontiguousarray(tr0.copy())
    weights = api.LossWeights()
    mc = api.MarchConfig().to_c()
    ac = vp_adam(1e-4, 0.9, 0.999, 1e-8, 1.0, 1.0)
    stream, mk = device_events(torch, lib, r)
    lv, ld, lp = C.c_float(), C.c_float(), C.c_float()

    def check(rc):
        if rc:
            raise RuntimeError(lib.vp_last_error(r.ctx).decode())

    def iteration(b, ev=None):
        ci, xy, pid, tg, bg = b
        pose[:] = 0
        check(lib.vp_loss_pose(k, tr.ctypes.data_as(f32p), weights.vol, weights.del_, C.byref(lv), C.byref(ld),
                               pose.ctypes.data_as(f32p)))
        check(lib.vp_eval_loss_pho(r.ctx, 64, cams_c, n, ci.ctypes.data_as(i32p), xy.ctypes.data_as(f32p),
                                   pid.ctypes.data_as(i32p), tg.ctypes.data_as(f32p), bg.ctypes.data_as(f32p),
                                   weights.pho, C.byref(mc), tr.ctypes.data_as(f32p), C.byref(lp), None, gptr, 0))
        grads[n_pay:] += torch.from_numpy(pose).to("cuda", non_blocking=False)
        torch.cuda.synchronize()
        if ev:
            ev[0].record(stream)
        check(lib.vp_adam_step(r.ctx, C.byref(ac), gptr, tr.ctypes.data_as(f32p)))
        if ev:
            ev[1].record(stream)

    for i in range(args.warmup):
        iteration(batches[i])
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.2)
    evs = [(mk(), mk()) for _ in range(args.steps)]
    t = []
    for i in range(args.steps):
        t0 = time.perf_counter()
        iteration(batches[args.warmup + i], evs[i])
        torch.cuda.synchronize()
        t.append(time.perf_counter() - t0)
    clk = clocks.stop()
    adam_ms = float(np.median([a.elapsed_time(b) for a, b in evs]))
    it_s = float(np.median(t))
    pk, pk_kind = peaks()
    adam_bytes = 32 * n_par
    achieved = adam_bytes / (adam_ms * 1e-3) / 1e9
    row = {"row": "fit", "metric": "iterations/s", "value": round(1.0 / it_s, 2), "unit": "iterations/s",
           "higher_is_better": True, "steps": args.steps, "warmup": args.warmup,
           "ms_per_iteration": round(it_s * 1e3, 3), "rays_per_s": round(n / it_s, 1),
           "dtype": "f32", "data": "synthetic (random targets/backgrounds, seeded)",
           "config": {"workload": "fit iteration: evalLoss (8 images x 256 rays of the 64-view ring, 1024^2) "
                                  "+ backwardRay + adamStep, mvp_shell K=4096 M=16",
                      "K": k, "M": m, "rays": n, "parameters": n_par},
           "breakdown_ms": {"adam_step_device": round(adam_ms, 3),
                            "eval_loss_and_host": round(it_s * 1e3 - adam_ms, 3)},
           "roofline": {"bound": "hbm", "kernel": "Adam pass (k_adam_check + k_adam_update + compose)",
                        "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": None,
                        "alg_bytes_per_iteration": adam_bytes, "peak_kind": pk_kind},
           "clocks": clk, "cpu_baseline": None}
    if ref is not None and not args.no_cpu_baseline:
        from oracle.bindings import ref_adam_run, ref_eval_loss
        ci, xy, pid, tg, bg = batches[0]
        cfg = api.MarchConfig()
        wts = (weights.pho, weights.vol, weights.del_)
        t0 = time.perf_counter()
        _, g = ref_eval_loss(ref, tr0, m, pay, api.WindowParams(), cams, ci, xy, pid, tg, bg, wts, cfg)
        t_eval = time.perf_counter() - t0
        cfg6 = np.array([1e-4, 0.9, 0.999, 1e-8, 1.0, 1.0], np.float32)
        t0 = time.perf_counter()
        ref_adam_run(ref, tr0, m, pay, g[None, :], cfg6)
        t1 = time.perf_counter() - t0
        t0 = time.perf_counter()
        ref_adam_run(ref, tr0, m, pay, np.stack([g, g]), cfg6)
        t2 = time.perf_counter() - t0
        t_adam = max(t2 - t1, 1e-9)  # one adamStep, marshalling cancelled out
        ref_it = t_eval + t_adam
        row["cpu_baseline"] = {"value": round(1.0 / ref_it, 4), "unit": "iterations/s", "cores": 1,
                               "kind": "reference",
                               "sample": f"one iteration: evalLoss {t_eval:.2f} s (incl. marshalling into the "
                                         f"reference's Frame), adamStep {t_adam:.2f} s (2-step minus 1-step run)"}
    emit(row)


# -----------------------------------------------------------------------------------------
def row_backward(args, torch, r, lib, api, synthetic, ref):
    from paper_2103_01954_b200._lib import f32p, vp_stats
    k, m, w = 4096, 16, 1024
    tr, pay = synthetic.shell_arrays(k, m)
    r.set_scene_records(tr, api.PrimitiveSlab(k, m, pay), api.WindowParams())
    cam = synthetic.shell_camera(-1, 0, w)
    out = r.render(cam, api.MarchConfig())
    hit = np.flatnonzero(out.sample_counts > 0)
    rng = np.random.default_rng(2)
    pix = np.sort(rng.choice(hit, 65536, replace=False))
    from oracle.bindings import Oracle
    orc = Oracle()
    o = np.zeros((pix.size, 3), np.float32)
    d = np.zeros((pix.size, 3), np.float32)
    for i, p in enumerate(pix):
        o[i], d[i] = orc.generate_ray(cam, float(p % w) + 0.5, float(p // w) + 0.5)
    ar = rng.normal(size=(pix.size, 3)).astype(np.float32)
    aa = rng.normal(size=pix.size).astype(np.float32)
    n_par = k * 4 * m ** 3 + 9 * k
    dev = {nm: torch.from_numpy(a).cuda() for nm, a in (("o", o), ("d", d), ("ar", ar), ("aa", aa))}
    grads = torch.zeros(n_par, dtype=torch.float32, device="cuda")
    P = lambda t: C.cast(C.c_void_p(t.data_ptr()), f32p)  # noqa: E731
    mc = api.MarchConfig().to_c()
    # primitive-samples of these rays (forward march over the same rays)
    rgb, alpha, samples = r.march_rays(o, d, api.MarchConfig())
    st = vp_stats()
    lib.vp_read_stats(r.ctx, C.byref(st))
    prim_samples = int(st.prim_samples)
    stream, mk = device_events(torch, lib, r)

    def call():
        rc = lib.vp_backward_rays(r.ctx, pix.size, P(dev["o"]), P(dev["d"]), None, P(dev["ar"]), P(dev["aa"]),
                                  C.byref(mc), tr.ctypes.data_as(f32p), P(grads), 0)
        if rc:
            raise RuntimeError(lib.vp_last_error(r.ctx).decode())

    for _ in range(args.warmup):
        call()
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.2)
    ms = []
    for _ in range(args.steps):
        a, b = mk(), mk()
        a.record(stream)
        call()
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    clk = clocks.stop()
    t = float(np.median(ms)) * 1e-3
    pk, pk_kind = peaks()
    alg = 256 * prim_samples
    achieved = alg / t / 1e9
    row = {"row": "backward", "metric": "rays/s", "value": round(pix.size / t, 1), "unit": "rays/s",
           "higher_is_better": True, "steps": args.steps, "warmup": args.warmup, "ms_per_call": round(t * 1e3, 3),
           "prim_samples_per_s": round(prim_samples / t, 1), "dtype": "f32", "data": "synthetic",
           "config": {"workload": "backwardRay of 65,536 hit pixels of the headline view (random adjoints), "
                                  "mvp_shell K=4096 M=16, device GradBuffer (zeroed per call)",
                      "rays": int(pix.size), "prim_samples": prim_samples},
           "roofline": {"bound": "hbm", "kernel": "k_backward_rays (+ gradient zeroing, 1.07 GB)",
                        "achieved": round(achieved, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": round(achieved / pk["hbm_gbs"], 4), "traffic": None,
                        "alg_bytes_per_call": alg, "peak_kind": pk_kind},
           "clocks": clk, "cpu_baseline": None}
    if ref is not None and not args.no_cpu_baseline:
        ns = 2048
        t0 = time.perf_counter()
        ref.backward_rays(tr, m, pay, api.WindowParams(), o[:ns], d[:ns], ar[:ns], aa[:ns], api.MarchConfig())
        tr_ = time.perf_counter() - t0
        row["cpu_baseline"] = {"value": round(ns / tr_, 1), "unit": "rays/s", "cores": 1, "kind": "reference",
                               "sample": f"{ns} of the same rays, {tr_:.2f} s incl. the reference's LBVH build "
                                         f"and GradBuffer allocation"}
    emit(row)


# -----------------------------------------------------------------------------------------
def row_compose(args, torch, r, lib, api, synthetic, ref):
    from paper_2103_01954_b200._lib import f32p
    k = 32768
    tr, _ = synthetic.shell_arrays(k, 1)
    r.set_scene_records(tr, api.PrimitiveSlab(k, 1, np.zeros(4 * k, np.float32)), api.WindowParams())
    stream, mk = device_events(torch, lib, r)
    for _ in range(args.warmup):
        r.set_records(tr)
    t, ms = [], []
    for _ in range(args.steps):
        a, b = mk(), mk()
        t0 = time.perf_counter()
        a.record(stream)
        if lib.vp_set_frame(r.ctx, k, tr.ctypes.data_as(f32p)):
            raise RuntimeError(lib.vp_last_error(r.ctx).decode())
        b.record(stream)
        torch.cuda.synchronize()
        t.append(time.perf_counter() - t0)
        ms.append(a.elapsed_time(b))
    tw = float(np.median(t))
    row = {"row": "compose", "metric": "primitives/s", "value": round(k / tw, 1), "unit": "primitives/s",
           "higher_is_better": True, "steps": args.steps, "warmup": args.warmup,
           "ms_per_call": round(tw * 1e3, 4), "device_ms": round(float(np.median(ms)), 4),
           "dtype": "f32", "data": "synthetic",
           "config": {"workload": "Frame::composed() of 32,768 PrimitiveTransform records (host) into the "
                                  "resident transforms (vp_set_frame)", "K": k},
           "cpu_baseline": None}
    if ref is not None and not args.no_cpu_baseline:
        reps = 20
        t0 = time.perf_counter()
        for _ in range(reps):
            ref.compose(tr)
        tr_ = (time.perf_counter() - t0) / reps
        row["cpu_baseline"] = {"value": round(k / tr_, 1), "unit": "primitives/s", "cores": 1,
                               "kind": "reference", "sample": f"{reps} x compose() of the same 32,768 records"}
    emit(row)


# -----------------------------------------------------------------------------------------
def row_load(args, torch, r, lib, api, synthetic, ref):
    k, m = 4096, 16
    tr, pay = synthetic.shell_arrays(k, m)
    xf = api.compose(tr)
    fd, path = tempfile.mkstemp(suffix=".vpsl")
    with os.fdopen(fd, "wb") as f:
        f.write(b"VPSL" + np.array([1, k, m], "<u4").tobytes())
        f.write(np.asarray(pay, "<f4").tobytes())
    size = os.path.getsize(path)
    try:
        for _ in range(args.warmup):
            r.load_slab(path, xf, api.WindowParams())
        t = []
        for _ in range(min(args.steps, 10)):
            t0 = time.perf_counter()
            r.load_slab(path, xf, api.WindowParams())
            torch.cuda.synchronize()
            t.append(time.perf_counter() - t0)
        tw = float(np.median(t))
        row = {"row": "load", "metric": "GB/s", "value": round(size / tw / 1e9, 3), "unit": "GB/s",
               "higher_is_better": True, "steps": len(t), "warmup": args.warmup, "ms_per_call": round(tw * 1e3, 2),
               "dtype": "f32", "data": "synthetic",
               "config": {"workload": "loadSlab of the headline slab (VPSL, 268 MB, page cache warm) into the "
                                      "device's interleaved layout (vp_load_slab)", "bytes": size},
               "cpu_baseline": None}
        if ref is not None and not args.no_cpu_baseline:
            from oracle.bindings import ref_load_slab  # noqa: F401  (reads K, M, then the slab)
            L = ref.lib
            L.vpref_load_slab.argtypes = [C.c_char_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_void_p,
                                          C.c_int64]
            kk, mm = C.c_int32(), C.c_int32()
            t = []
            for _ in range(3):
                t0 = time.perf_counter()
                L.vpref_load_slab(path.encode(), C.byref(kk), C.byref(mm), None, 0)
                t.append(time.perf_counter() - t0)
            tr_ = float(np.median(t))
            row["cpu_baseline"] = {"value": round(size / tr_ / 1e9, 3), "unit": "GB/s", "cores": 1,
                                   "kind": "reference", "sample": "loadSlab of the same file into host memory, x3"}
        emit(row)
    finally:
        os.unlink(path)


def main():
    args = parse()
    import torch
    from paper_2103_01954_b200 import Renderer, api, synthetic
    torch.cuda.set_device(0)
    r = Renderer(0)
    lib = r._lib
    ref = None if args.no_cpu_baseline else ref_core()
    rows = {"fit": row_fit, "backward": row_backward, "compose": row_compose, "load": row_load}
    for name in args.rows.split(","):
        rows[name](args, torch, r, lib, api, synthetic, ref)


if __name__ == "__main__":
    main()

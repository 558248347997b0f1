import ctypes as C, time, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2103_01954_b200 import Renderer, api, synthetic
from paper_2103_01954_b200._lib import f32p, i32p, vp_camera
k, m, w, V = 4096, 16, 1024, 8
tr, pay = synthetic.shell_arrays(k, m)
xf = api.compose(tr)
r = Renderer(0); lib = r._lib
r.set_scene_composed(xf, api.PrimitiveSlab(k, m, pay), api.WindowParams())
cams = [synthetic.shell_camera(v, 64, w).to_c() for v in range(V)]
cams_arr = (vp_camera * V)(*cams)
mc = api.MarchConfig().to_c()
n_px = w * w
h_rgb = torch.empty((V, n_px * 3), dtype=torch.float32, pin_memory=True)
h_a = torch.empty((V, n_px), dtype=torch.float32, pin_memory=True)
h_s = torch.empty((V, n_px), dtype=torch.int32, pin_memory=True)
P = lambda t, T: (T * V)(*[C.cast(t[j].data_ptr(), T) for j in range(V)])
hr, ha, hs = P(h_rgb, f32p), P(h_a, f32p), P(h_s, i32p)
d_rgb = torch.empty((V, n_px * 3), device='cuda'); d_a = torch.empty((V, n_px), device='cuda'); d_s = torch.empty((V, n_px), dtype=torch.int32, device='cuda')
dr, da, ds = P(d_rgb, f32p), P(d_a, f32p), P(d_s, i32p)
xh = torch.from_numpy(xf).pin_memory()
def run(name, fn, n=10):
    fn(); lib.vp_sync(r.ctx); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    lib.vp_sync(r.ctx); torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    print(f"{name:40s} {dt*1e3:8.2f} ms/step", flush=True)
run("batch device", lambda: lib.vp_render_batch_async(r.ctx, V, cams_arr, C.byref(mc), dr, da, ds, None))
run("batch host", lambda: lib.vp_render_batch_async(r.ctx, V, cams_arr, C.byref(mc), hr, ha, hs, None))
run("xf sync + batch host", lambda: (lib.vp_set_transforms(r.ctx, k, C.cast(xh.data_ptr(), f32p)), lib.vp_render_batch_async(r.ctx, V, cams_arr, C.byref(mc), hr, ha, hs, None)))
run("xf async + batch device", lambda: (lib.vp_set_transforms_async(r.ctx, k, C.cast(xh.data_ptr(), f32p), None), lib.vp_render_batch_async(r.ctx, V, cams_arr, C.byref(mc), dr, da, ds, None)))
run("xf async + batch host", lambda: (lib.vp_set_transforms_async(r.ctx, k, C.cast(xh.data_ptr(), f32p), None), lib.vp_render_batch_async(r.ctx, V, cams_arr, C.byref(mc), hr, ha, hs, None)))


def kt(name, fn, n=30):
    fn(); lib.vp_sync(r.ctx); torch.cuda.synchronize(); r.kernel_times()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    lib.vp_sync(r.ctx); torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    ks = r.kernel_times(4096)
    print(f"{name:40s} {dt*1e3:8.2f} ms/step wall, march kernel mean {ks.mean():.3f} ms (n={len(ks)})", flush=True)


kt("xf async + batch device (30)", lambda: (lib.vp_set_transforms_async(r.ctx, k, C.cast(xh.data_ptr(), f32p), None), lib.vp_render_batch_async(r.ctx, V, cams_arr, C.byref(mc), dr, da, ds, None)))
kt("xf async + batch host (30)", lambda: (lib.vp_set_transforms_async(r.ctx, k, C.cast(xh.data_ptr(), f32p), None), lib.vp_render_batch_async(r.ctx, V, cams_arr, C.byref(mc), hr, ha, hs, None)))
kt("xf async + batch device (30)", lambda: (lib.vp_set_transforms_async(r.ctx, k, C.cast(xh.data_ptr(), f32p), None), lib.vp_render_batch_async(r.ctx, V, cams_arr, C.byref(mc), dr, da, ds, None)))
kt("xf async + batch host (30)", lambda: (lib.vp_set_transforms_async(r.ctx, k, C.cast(xh.data_ptr(), f32p), None), lib.vp_render_batch_async(r.ctx, V, cams_arr, C.byref(mc), hr, ha, hs, None)))


def enq(name, fn, n=30):
    fn(); lib.vp_sync(r.ctx); torch.cuda.synchronize()
    t0 = time.perf_counter()
    ts = []
    for _ in range(n):
        a = time.perf_counter(); fn(); ts.append(time.perf_counter() - a)
    t1 = time.perf_counter()
    lib.vp_sync(r.ctx); torch.cuda.synchronize()
    t2 = time.perf_counter()
    ts = np.array(ts) * 1e3
    print(f"{name:30s} enqueue {1e3*(t1-t0)/n:6.2f} ms/step (call max {ts.max():.2f}, median {np.median(ts):.3f}), "
          f"total {1e3*(t2-t0)/n:6.2f} ms/step", flush=True)


enq("host outputs", lambda: (lib.vp_set_transforms_async(r.ctx, k, C.cast(xh.data_ptr(), f32p), None), lib.vp_render_batch_async(r.ctx, V, cams_arr, C.byref(mc), hr, ha, hs, None)))
enq("device outputs", lambda: (lib.vp_set_transforms_async(r.ctx, k, C.cast(xh.data_ptr(), f32p), None), lib.vp_render_batch_async(r.ctx, V, cams_arr, C.byref(mc), dr, da, ds, None)))

"""Host-side split of one fit iteration (profiling helper): wall time of each C-ABI call of the
bench_rows.py fit row (vp_loss_pose, vp_eval_loss_pho with the backward, the pose-gradient add,
vp_adam_step), median over 30 iterations, K=4096 M=16, 2048 rays. Usage (GPU): python tools/fit_breakdown.py"""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/", 2)[0])
from paper_2103_01954_b200 import Renderer, api, synthetic  # noqa: E402
from paper_2103_01954_b200._lib import f32p, i32p, vp_adam, vp_camera  # noqa: E402

k, m, w = 4096, 16, 1024
tr0, pay = synthetic.shell_arrays(k, m)
r = Renderer(0)
lib = r._lib
r.set_scene_records(tr0, api.PrimitiveSlab(k, m, pay), api.WindowParams())
cams = (vp_camera * 64)(*[synthetic.shell_camera(v, 64, w).to_c() for v in range(64)])
n = 2048
rng = np.random.default_rng(1)
n_par = k * 4 * m ** 3 + 9 * k
grads = torch.zeros(n_par, dtype=torch.float32, device="cuda")
gptr = C.cast(C.c_void_p(grads.data_ptr()), f32p)
pose = np.zeros(9 * k, np.float32)
tr = np.ascontiguousarray(tr0.copy())
mc = api.MarchConfig().to_c()
ac = vp_adam(1e-4, 0.9, 0.999, 1e-8, 1.0, 1.0)
lv, ld, lp = C.c_float(), C.c_float(), C.c_float()
rows = []
for it in range(40):
    ci = np.repeat(rng.choice(64, 8, replace=False), 256).astype(np.int32)
    pid = rng.integers(0, w * w, n).astype(np.int32)
    xy = np.stack([pid % w + 0.5, pid // w + 0.5], 1).astype(np.float32)
    tg = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    bg = rng.uniform(0, 1, (n, 3)).astype(np.float32)
    t = [time.perf_counter()]
    pose[:] = 0
    lib.vp_loss_pose(k, tr.ctypes.data_as(f32p), 0.01, 0.01, C.byref(lv), C.byref(ld), pose.ctypes.data_as(f32p))
    t.append(time.perf_counter())
    assert lib.vp_eval_loss_pho(r.ctx, 64, cams, n, ci.ctypes.data_as(i32p), xy.ctypes.data_as(f32p),
                                pid.ctypes.data_as(i32p), tg.ctypes.data_as(f32p), bg.ctypes.data_as(f32p), 1.0,
                                C.byref(mc), tr.ctypes.data_as(f32p), C.byref(lp), None, gptr, 0) == 0
    t.append(time.perf_counter())
    grads[n_par - 9 * k:] += torch.from_numpy(pose).to("cuda")
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    assert lib.vp_adam_step(r.ctx, C.byref(ac), gptr, tr.ctypes.data_as(f32p)) == 0
    t.append(time.perf_counter())
    if it >= 10:
        rows.append(np.diff(t) * 1e3)
med = np.median(np.array(rows), axis=0)
print("ms: loss_pose %.3f  eval_loss_pho(+backward) %.3f  pose add %.3f  adam_step %.3f  total %.3f" % (*med, med.sum()))

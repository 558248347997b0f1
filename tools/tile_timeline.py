"""Per-CTA timeline of the raymarch kernel (vp_debug_tile_times): SM busy fraction and the
heaviest tiles. Usage: python tools/tile_timeline.py [K M W]"""
import ctypes as C
import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2103_01954_b200 import Renderer, api, synthetic  # noqa: E402

k, m, w = (int(x) for x in (sys.argv[1:4] if len(sys.argv) >= 4 else (4096, 16, 1024)))
tr, pay = synthetic.shell_arrays(k, m)
r = Renderer(0)
r.set_scene_composed(api.compose(tr), api.PrimitiveSlab(k, m, pay), api.WindowParams())
cam = synthetic.shell_camera(-1, 0, w)
cc, mc = cam.to_c(), api.MarchConfig().to_c()
r.render(cam, api.MarchConfig())
n = C.c_int64()
n_tiles = ((w + 15) // 16) ** 2
out = np.zeros(4 * n_tiles, np.uint64)
for _ in range(2):
    rc = r._lib.vp_debug_tile_times(r.ctx, C.byref(cc), C.byref(mc), out.ctypes.data_as(C.POINTER(C.c_uint64)),
                                    out.size, C.byref(n))
    assert rc == 0, r._lib.vp_last_error(r.ctx)
t = out.reshape(-1, 4).astype(np.int64)
t0, t1 = t[:, 2].min(), t[:, 3].max()
dur = t[:, 3] - t[:, 2]
span = t1 - t0
busy = np.zeros(int(t[:, 1].max()) + 1)
for smid, a, b in zip(t[:, 1], t[:, 2], t[:, 3]):
    busy[smid] += b - a
offs, _, _, _ = r.debug_tiles(cam)[2], 0, 0, 0
counts = np.diff(r.debug_tiles(cam)[2])
print(f"K={k} M={m} W={w}: kernel span {span / 1e3:.1f} us, CTAs {len(t)}, SMs {len(busy)}")
print(f"per-SM CTA-time / span: mean {busy.mean() / span:.2f} (3 slots -> max 3.0), min {busy.min() / span:.2f}, max {busy.max() / span:.2f}")
last = np.argsort(t[:, 3])[-10:]
print("last-finishing CTAs (launch idx, tile, candidates, start us, dur us):")
for i in last:
    print(f"  {i:5d} tile {t[i, 0]:5d} n={counts[t[i, 0]]:4d} start {(t[i, 2] - t0) / 1e3:8.1f} dur {dur[i] / 1e3:8.1f}")
heavy = np.argsort(dur)[-5:]
print("longest CTAs:", [(int(t[i, 0]), int(counts[t[i, 0]]), round(dur[i] / 1e3, 1)) for i in heavy])
q = np.corrcoef(counts[t[:, 0]], dur)[0, 1]
print(f"corr(candidates, duration) = {q:.2f}; duration p50 {np.median(dur) / 1e3:.1f} us, p99 {np.percentile(dur, 99) / 1e3:.1f} us")
out_r = r.render(cam, api.MarchConfig())
s = out_r.sample_counts.reshape(w, w)
tx = (w + 15) // 16
for tile in [int(t[i, 0]) for i in heavy[-3:]]:
    ty_, tx_ = divmod(tile, tx)
    blk = s[ty_ * 16:(ty_ + 1) * 16, tx_ * 16:(tx_ + 1) * 16]
    print(f"tile {tile}: hit rays {(blk > 0).sum()}, samples max {blk.max()}, mean {blk[blk > 0].mean():.1f}")
print("image: max samples per ray", s.max(), "p99", np.percentile(s[s > 0], 99))

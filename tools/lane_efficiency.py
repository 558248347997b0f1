"""Lane occupancy of the raymarch's phase 2 predicted from per-pixel sample counts (profiling
helper). A warp runs as long as its longest ray; a CTA holds all 8 warp slots until its
longest warp ends. Usage (GPU): python tools/lane_efficiency.py [K M W]"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/", 2)[0])
from paper_2103_01954_b200 import Renderer, api, synthetic  # noqa: E402

k, m, w = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (4096, 16, 1024)
tr, pay = synthetic.shell_arrays(k, m)
with Renderer(0) as r:
    r.set_scene_composed(api.compose(tr), api.PrimitiveSlab(k, m, pay), api.WindowParams())
    S = r.render(synthetic.shell_camera(3, 64, w), api.MarchConfig()).sample_counts.reshape(w, w)
tid = np.arange(256)
wid, lane = tid >> 5, tid & 31
lx, ly = (wid & 1) * 8 + (lane & 7), (wid >> 1) * 4 + (lane >> 3)  # vpb_march.cuh tile_pixel
tot = warp_slots = cta_slots = 0
for ty in range(w // 16):
    for tx in range(w // 16):
        v = S[ty * 16 + ly, tx * 16 + lx]
        hits = v[v > 0]  # compacted hit rays, in thread order
        if not len(hits):
            continue
        mx = [hits[i:i + 32].max() for i in range(0, len(hits), 32)]
        tot += hits.sum()
        warp_slots += 32 * sum(mx)
        cta_slots += 256 * max(mx)
print(f"K={k} M={m} W={w}: lanes busy within warps {tot / warp_slots:.3f}, "
      f"over the CTA lifetime (8 warp slots held) {tot / cta_slots:.3f}")

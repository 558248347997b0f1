"""Device timeline of the backward row's last calls (torch.profiler / CUPTI sees libvpb's
kernels too): start offset, duration and stream of every kernel, memset and copy, to find the
idle gaps between launches. Usage: python tools/bwd_timeline.py [out.txt] [backward|fit]"""
import json
import pathlib
import sys
import tempfile
import types

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench_rows  # noqa: E402
from paper_2103_01954_b200 import Renderer, api, synthetic  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bwd_timeline.txt"
row = sys.argv[2] if len(sys.argv) > 2 else "backward"
r = Renderer(0)
args = types.SimpleNamespace(steps=3, warmup=3, no_cpu_baseline=True)
bench_rows.emit = lambda row: None
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    getattr(bench_rows, "row_" + row)(args, torch, r, r._lib, api, synthetic, None)
tr = pathlib.Path(tempfile.mkdtemp()) / "t.json"
prof.export_chrome_trace(str(tr))
ev = [e for e in json.load(open(tr))["traceEvents"]
      if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")]
ev.sort(key=lambda e: e["ts"])
# the last call: from the last forward march kernel launch backwards to its preceding memset
starts = [i for i, e in enumerate(ev) if "k_march_rays_warp" in e["name"]]
i0 = starts[-1]
while i0 > 0 and ev[i0 - 1]["cat"] != "kernel":
    i0 -= 1
lines = []
t0 = ev[i0]["ts"]
busy_end = t0
gap_total = 0.0
for e in ev[i0:]:
    gap = max(0.0, e["ts"] - busy_end)
    gap_total += gap
    busy_end = max(busy_end, e["ts"] + e["dur"])
    lines.append(f"{e['ts'] - t0:9.1f} {e['dur']:8.1f} gap {gap:6.1f} s{e['args'].get('stream')} {e['name'][:90]}")
lines.append(f"span {busy_end - t0:.1f} us, idle {gap_total:.1f} us")
pathlib.Path(out).parent.mkdir(exist_ok=True)
pathlib.Path(out).write_text("\n".join(lines) + "\n")
print("\n".join(lines[-60:]))

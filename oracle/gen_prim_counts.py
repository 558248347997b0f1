"""TEST INFRASTRUCTURE (fixture generator, run in the build container where /root/reference
exists): prim-sample counts of the reference renderer (the roofline's
algorithmic bytes are 128 B per prim-sample, so the device counter that feeds them is pinned
to the reference).

For every render case of tests/golden/renders.npz and every full-size digest of
tests/golden/digests.json, the unmodified reference counts, per pixel, the executions of
march.cpp:63-70 (oracle/ref_glue.cpp: vpref_render_prim_counts). Writes
tests/golden/prim_counts.npz (per-pixel counts of the render cases and of BASELINE config 1)
and adds "prim_samples" to each digests.json entry.

    python oracle/gen_prim_counts.py
"""
import json
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from golden_cases import render_cases  # noqa: E402
from oracle.bindings import RefCore  # noqa: E402
from paper_2103_01954_b200 import api, synthetic  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"


def main():
    ref = RefCore()
    out = {}
    for name, c in sorted(render_cases().items()):
        if len(c["tr"]) == 0:
            prim = np.zeros(c["cam"].width * c["cam"].height, np.int32)
        else:
            prim = ref.render_prim_counts(c["tr"], c["m"], c["payload"], c["window"], c["cam"], c["cfg"])
        out[f"case_{name}"] = prim
        print(name, int(prim.sum()), flush=True)
    path = GOLDEN / "digests.json"
    dg = json.loads(path.read_text())
    for key, d in sorted(dg["renders"].items()):
        tr, pay = synthetic.shell_arrays(d["K"], d["M"])
        cam = synthetic.shell_camera(d["view"], d["n_views"], d["W"])
        t0 = time.time()
        prim = ref.render_prim_counts(tr, d["M"], pay, api.WindowParams(), cam, api.MarchConfig())
        d["prim_samples"] = int(prim.astype(np.int64).sum())
        if d["W"] <= 256:
            out[f"full_{key}"] = prim
        print(key, d["prim_samples"], f"{time.time() - t0:.1f} s", flush=True)
    np.savez_compressed(GOLDEN / "prim_counts.npz", **out)
    path.write_text(json.dumps(dg, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()

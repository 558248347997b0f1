"""TEST INFRASTRUCTURE — reference digests of every view of the 64-view ring (BASELINE config 5).

The unmodified reference (oracle/_ref/libvolprim_ref.so) renders views 0..63 of the §8d ring
around the K=4096 x 16^3 shell at 1024^2 on a resident Scene, with inputs and cameras from the
reference-side generator (vpref_shell_scene / vpref_shell_camera, pinned to
digests.json["generator"]). The SHA-256 of rgb / alpha / sample counts of each view is merged
into tests/golden/digests.json under "ring"; tests/test_gpu_parity.py renders all 64 views
through vp_render_batch_async and compares.

    python oracle/gen_ring_digests.py              # the 64 views of config 5
    python oracle/gen_ring_digests.py --sweep-only # views 0..7 of configs 1, 2, 4 ("ring_configs")
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

from oracle.bindings import RefCore, RefScene, ref_shell_camera  # noqa: E402

K, M, W, N_RING = 4096, 16, 1024, 64
# the other single-GPU configs of BASELINE.json (1, 2, 4): views 0..7 of the ring at each,
# the views bench.py's "sweep" key times in one 8-view launch
SWEEP = {"oracle_64x16_256": (64, 16, 256), "k512_m32_1024": (512, 32, 1024),
         "k32768_m8_1024": (32768, 8, 1024)}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ring_views(ref, k, m, w, views):
    scene = RefScene(ref, k, m)
    out = {}
    for v in views:
        k9, r9, t3 = ref_shell_camera(ref, v, N_RING, w)
        t0 = time.time()
        tot, rgb, alpha, samples = scene.render(k9, r9, t3, w, w, outputs=True)
        out[str(v)] = {"rgb": sha(rgb), "alpha": sha(alpha), "samples": sha(samples),
                       "total_samples": int(tot), "hit_pixels": int((samples > 0).sum()),
                       "ref_seconds": round(time.time() - t0, 3)}
        print(k, m, w, v, tot, out[str(v)]["ref_seconds"], flush=True)
    scene.close()
    return out


def main():
    path = ROOT / "tests" / "golden" / "digests.json"
    digests = json.loads(path.read_text())
    ref = RefCore()
    if "--sweep-only" in sys.argv:
        digests["ring_configs"] = {name: {"K": k, "M": m, "W": w, "n_views": N_RING,
                                          "views": ring_views(ref, k, m, w, range(8))}
                                   for name, (k, m, w) in SWEEP.items()}
        path.write_text(json.dumps(digests, indent=1, sort_keys=True))
        return
    scene = RefScene(ref, K, M)
    ring = {}
    for v in range(N_RING):
        k9, r9, t3 = ref_shell_camera(ref, v, N_RING, W)
        t0 = time.time()
        tot, rgb, alpha, samples = scene.render(k9, r9, t3, W, W, outputs=True)
        ring[str(v)] = {"rgb": sha(rgb), "alpha": sha(alpha), "samples": sha(samples),
                        "total_samples": int(tot), "hit_pixels": int((samples > 0).sum()),
                        "ref_seconds": round(time.time() - t0, 3)}
        print(v, tot, ring[str(v)]["ref_seconds"], flush=True)
    digests["ring"] = {"K": K, "M": M, "W": W, "n_views": N_RING, "views": ring}
    path.write_text(json.dumps(digests, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()

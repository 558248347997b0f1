"""Rebuilds the inputs of the golden render cases (tests/golden/renders.npz)."""
import hashlib

import numpy as np

from conftest import load_groups
from paper_2103_01954_b200 import api, synthetic


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def render_cases():
    cases = load_groups("renders")
    out = {}
    for name, g in cases.items():
        if "gen" in g:
            k, m = (int(x) for x in g["gen"])
            tr, pay = synthetic.shell_arrays(k, m)
            assert sha(tr) == str(g["tr_sha"]) and sha(pay) == str(g["payload_sha"]), \
                f"{name}: synthetic generator output drifted"
        else:
            tr, pay = g["tr"].reshape(-1, 24), g["payload"]
        cam = api.Camera(g["K"], g["R"], g["t"], int(g["wh"][0]), int(g["wh"][1]))
        c = g["cfg"]
        cfg = api.MarchConfig(float(np.float32(c[0])), float(np.float32(c[1])), bool(c[2]), int(c[3]))
        win = api.WindowParams(float(g["window"][0]), int(g["window"][1]))
        out[name] = dict(tr=tr, m=int(g["m"]), payload=pay, cam=cam, cfg=cfg, window=win,
                         rgb=g["rgb"], alpha=g["alpha"], samples=g["samples"])
    return out

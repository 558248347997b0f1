"""CPU: the C-ABI library loads and exports every symbol include/vpb.h declares, and its
host-only entry points (compose, cameras, synthetic inputs) match the reference bit-for-bit.
No GPU compute is called here."""
import json
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, has_gpu
from paper_2103_01954_b200 import _lib, api, synthetic


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def same(a, b):
    """Bitwise equality, except that any NaN equals any NaN (the degenerate lookAt, forward
    parallel to up, yields NaN in the reference too; NaN sign bits are not meaningful)."""
    a, b = np.asarray(a, np.float32).reshape(-1), np.asarray(b, np.float32).reshape(-1)
    na, nb = np.isnan(a), np.isnan(b)
    return np.array_equal(na, nb) and np.array_equal(bits(a[~na]), bits(b[~nb]))


def header_symbols():
    src = (ROOT / "include" / "vpb.h").read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vp_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(lib, name), f"libvpb.so does not export {name}"
    assert set(syms) == set(_lib.SIGNATURES), "ctypes signature table out of sync with include/vpb.h"
    assert lib.vp_version() == 1


def test_compose_bit_exact_and_usage_error():
    z = np.load(GOLDEN / "compose.npz")
    assert np.array_equal(bits(api.compose(z["tr"])), bits(z["xf"]))
    with pytest.raises(api.Error) as e:
        api.compose(z["bad"])
    assert e.value.category == api.ErrorCategory.USAGE and e.value.exit_code == int(z["rc_bad"])


def test_look_at_camera_bit_exact():
    z = np.load(GOLDEN / "cameras.npz")
    for key in [k for k in z.files if k.startswith("lookat_")]:
        v = z[key]
        k9, r9, t3, aa, pos, (f, w) = v[0:9], v[9:18], v[18:21], v[21:24], v[24:27], v[27:29]
        cam, aa2 = synthetic.look_at_camera(pos, (0, 0, 0), (0, 1, 0), f, int(w), int(w))
        assert same(cam.intrinsics.T, k9), key
        assert same(cam.rotation.T, r9), key
        assert same(cam.translation, t3), key
        assert same(aa2, aa), key
    # the headline camera is the survey's lookAtCamera((0.25, 0.15, -1.1), 0, up y, 1.2 W)
    head = z["lookat_headline_256"]
    cam = synthetic.shell_camera(-1, 0, 256)
    assert np.array_equal(bits(cam.rotation.T.reshape(-1)), bits(head[9:18]))


def test_synthetic_generator_matches_recorded_digests():
    d = json.loads((GOLDEN / "digests.json").read_text())["generator"]
    import hashlib
    for key in ("64x16", "4096x16"):
        k, m = (int(x) for x in key.split("x"))
        tr, pay = synthetic.shell_arrays(k, m)
        assert hashlib.sha256(tr.tobytes()).hexdigest() == d[key]["tr"]
        assert hashlib.sha256(pay.tobytes()).hexdigest() == d[key]["payload"]


def test_transform_records_layout():
    r = np.array([[1, 2, 3], [4, 5, 6], [7, 8, 9]], np.float32)
    rec = api.transform_records([(1, 2, 3)], [r], [(0.1, 0.2, 0.3)], delta_r=[(0, 0, 0.5)])
    assert rec.shape == (1, 24)
    assert np.array_equal(rec[0, 3:12], r.T.reshape(-1))  # column-major like volprim::Mat3::m
    assert np.array_equal(rec[0, 18:21], np.array([0, 0, 0.5], np.float32))
    cam = api.Camera(np.diag([2, 3, 1]).astype(np.float32), r, np.zeros(3, np.float32), 4, 5)
    back = api.Camera.from_c(cam.to_c())
    assert np.array_equal(back.rotation, r) and back.width == 4 and back.height == 5


@pytest.mark.skipif(has_gpu(), reason="checks the loud failure on a host without a GPU")
def test_no_gpu_fails_loudly():
    with pytest.raises(api.Error) as e:
        api.Renderer(0)
    assert e.value.category == api.ErrorCategory.DEVICE


def test_march_config_and_errors_mirror_reference():
    c = api.MarchConfig()
    assert (c.step_size, c.early_eps, c.jitter, c.seed) == (0.001, 0.01, False, 0)  # march.h:11-20
    w = api.WindowParams()
    assert (w.alpha, w.beta) == (8.0, 8)  # primitive.h:14-17
    assert [int(x) for x in api.ErrorCategory] == [2, 3, 4, 5, 6, 7]  # errors.h:11-17 + device


def test_pose_regularisers_bit_exact():
    """lossVol / lossDel (losses.cpp:45-68) terms equal the reference evalLoss's."""
    import ctypes as C
    z = np.load(GOLDEN / "train.npz")
    lib = _lib.load()
    tr = np.ascontiguousarray(z["tr"], np.float32)
    lv, ld = C.c_float(), C.c_float()
    g = np.zeros(9 * tr.shape[0], np.float32)
    assert lib.vp_loss_pose(tr.shape[0], tr.ctypes.data_as(_lib.f32p), float(z["weights"][2]),
                            float(z["weights"][3]), C.byref(lv), C.byref(ld), g.ctypes.data_as(_lib.f32p)) == 0
    assert bits(np.float32(lv.value)) == bits(z["terms"][2]) and bits(np.float32(ld.value)) == bits(z["terms"][3])
    assert np.any(g != 0)

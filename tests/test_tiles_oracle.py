"""CPU: the binning restatement (the artefacts that replace the reference's LBVH,
lbvh.cpp:13-156) is conservative and canonical.

* Conservative: for every pixel, every primitive the exact ray/box test hits (the oracle's
  intersect, itself pinned to the reference's LBVH traversal in test_oracle_golden) is in the
  pixel's tile list and inside its pixel rectangle — so culling never changes an image.
* Canonical: each tile list is sorted by (depth key, primitive index).
"""
import numpy as np
import pytest

from golden_cases import render_cases
from paper_2103_01954_b200 import api, synthetic


def scenes():
    cases = render_cases()
    out = []
    for name in ("shell64_m16_w64", "random_boxes_96x72", "camera_inside_40x32", "m1_boxes_48"):
        c = cases[name]
        out.append((name, api.compose(c["tr"]), c["cam"]))
    tr, _ = synthetic.shell_arrays(512, 8)
    out.append(("shell512_ring_w80", api.compose(tr), synthetic.shell_camera(9, 64, 80)))
    return out


@pytest.mark.parametrize("name,xf,cam", scenes(), ids=lambda v: v if isinstance(v, str) else "")
def test_tile_lists_conservative_and_sorted(oracle, name, xf, cam):
    rects, prects, keys = oracle.cull_px(xf, cam)
    offs, prims = oracle.tile_lists(xf, cam)
    tiles_x = (cam.width + 15) // 16
    # canonical order inside every tile
    for t in range(len(offs) - 1):
        seg = prims[offs[t]:offs[t + 1]]
        k = (keys[seg].astype(np.uint64) << np.uint64(32)) | seg.astype(np.uint64)
        assert np.all(np.diff(k.astype(np.float64)) > 0) or len(seg) < 2, (name, t)
    # tile rectangle == pixel rectangle / 16
    nonempty = prects[:, 2] >= prects[:, 0]
    assert np.array_equal(rects[nonempty], prects[nonempty] // 16)
    checked = 0
    for y in range(cam.height):
        for x in range(cam.width):
            o, d = oracle.generate_ray(cam, x + 0.5, y + 0.5)
            hits, _, _ = oracle.intersect(xf, o, d)
            if len(hits) == 0:
                continue
            t = (y // 16) * tiles_x + x // 16
            lst = set(prims[offs[t]:offs[t + 1]].tolist())
            assert set(hits.tolist()) <= lst, (name, x, y)
            r = prects[hits]
            assert np.all((r[:, 0] <= x) & (x <= r[:, 2]) & (r[:, 1] <= y) & (y <= r[:, 3])), (name, x, y)
            checked += len(hits)
    assert checked > 0


def test_cull_rejects_boxes_behind_the_camera(oracle):
    # camera at the origin looking down +z; a box at z = -5 is culled, one at z = +5 is not
    tr = api.transform_records([(0, 0, -5), (0, 0, 5)], [np.eye(3)] * 2, [(0.5, 0.5, 0.5)] * 2)
    xf = api.compose(tr)
    cam = api.Camera(np.array([[50, 0, 32], [0, 50, 32], [0, 0, 1]], np.float32), np.eye(3, dtype=np.float32),
                     np.zeros(3, np.float32), 64, 64)
    rects, prects, keys = oracle.cull_px(xf, cam)
    assert rects[0, 2] < rects[0, 0] and prects[0, 2] < prects[0, 0]
    assert rects[1, 2] >= rects[1, 0]
    assert keys[1] > 0  # positive depth lower bound

"""The multi-GPU C-ABI (include/vpb.h vp_comm_*, NCCL inside libvpb) on ONE B200: a 1-rank
communicator from vp_comm_init (process-per-GPU mode) and from vp_comm_init_all (single-process
mode). The scene broadcast must leave a renderable scene and the grouped gather must deliver
every view bit-identical to a direct render (the root's own views are device copies; with more
ranks the same group carries ncclSend / ncclRecv pairs). Multi-rank runs need a multi-GPU node;
the Python orchestration around them is covered with gloo (tests/test_dist_gloo.py)."""
import ctypes as C
import json

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from golden_cases import sha
from paper_2103_01954_b200 import Renderer, _lib, api, synthetic
from paper_2103_01954_b200.dist import NativeComm, NativeViewGather

pytestmark = pytest.mark.gpu


def _scene(r, comm=None):
    tr, pay = synthetic.shell_arrays(4096, 16)
    xf = api.compose(tr)
    slab = api.PrimitiveSlab(4096, 16, pay)
    if comm is None:
        r.set_scene_composed(xf, slab, api.WindowParams())
    else:
        comm.broadcast_scene(xf, slab, api.WindowParams(), 4096, 16, root=0)


def test_native_comm_one_rank_broadcast_and_gather_match_reference():
    ring = json.loads((GOLDEN / "digests.json").read_text())["ring"]
    with Renderer(0) as r:
        comm = NativeComm(r, world=1, rank=0, max_ctas=4)
        try:
            _scene(r, comm)
            w = ring["W"]
            g = NativeViewGather(comm, 4, w, w, torch.device("cuda", 0))
            for step, views in enumerate(([0, 1, 2, 3], [4, 5, 6, 7])):
                slot = step % 2
                g.wait_slot(slot)
                rgb, alpha, samp = g.views(slot)
                cams = (_lib.vp_camera * 4)(*[synthetic.shell_camera(v, 64, w).to_c() for v in views])
                P = lambda t, ty: (ty * 4)(*[C.cast(C.c_void_p(t[j].data_ptr()), ty) for j in range(4)])  # noqa
                mc = api.MarchConfig().to_c()
                assert r._lib.vp_render_batch_async(r.ctx, 4, cams, C.byref(mc), P(rgb, _lib.f32p),
                                                    P(alpha, _lib.f32p), P(samp, _lib.i32p), None) == 0
                g.gather(slot)
                g.finish()
                got_rgb, got_alpha, got_samp = (t.cpu().numpy() for t in g.recv[slot])
                for j, v in enumerate(views):
                    d = ring["views"][str(v)]
                    assert sha(got_samp[j]) == d["samples"], f"view {v}"
                    assert sha(got_alpha[j].reshape(w, w, 1)) == d["alpha"], f"view {v}"
                    assert sha(got_rgb[j].reshape(w, w, 3)) == d["rgb"], f"view {v}"
        finally:
            comm.close()


def test_native_comm_init_all_single_process():
    lib = _lib.load()
    with Renderer(0) as r:
        ctxs = (C.c_void_p * 1)(r.ctx)
        devs = (C.c_int32 * 1)(0)
        out = (C.c_void_p * 1)()
        assert lib.vp_comm_init_all(1, ctxs, devs, 2, out) == 0, lib.vp_comm_last_error()
        try:
            tr, pay = synthetic.shell_arrays(64, 8)
            r.set_scene_composed(api.compose(tr), api.PrimitiveSlab(64, 8, pay), api.WindowParams())
            assert lib.vp_group_start() == 0
            assert lib.vp_broadcast_scene(out[0], 0) == 0
            assert lib.vp_group_end() == 0
            assert lib.vp_comm_sync(out[0]) == 0
            cam = synthetic.shell_camera(3, 16, 96)
            ref = r.render(cam, api.MarchConfig())
            n = 96 * 96
            bufs = [torch.empty(n * 3, device="cuda"), torch.empty(n, device="cuda"),
                    torch.empty(n, dtype=torch.int32, device="cuda")]
            dst = [torch.empty(n * 3, device="cuda"), torch.empty(n, device="cuda"),
                   torch.empty(n, dtype=torch.int32, device="cuda")]
            r.render_device(cam, api.MarchConfig(), bufs[0].data_ptr(), bufs[1].data_ptr(), bufs[2].data_ptr())
            one = lambda t, ty: (ty * 1)(C.cast(C.c_void_p(t.data_ptr()), ty))  # noqa: E731
            assert lib.vp_gather_views(out[0], 0, 1, n, one(bufs[0], _lib.f32p), one(bufs[1], _lib.f32p),
                                       one(bufs[2], _lib.i32p), one(dst[0], _lib.f32p), one(dst[1], _lib.f32p),
                                       one(dst[2], _lib.i32p)) == 0
            assert lib.vp_comm_sync(out[0]) == 0
            assert np.array_equal(dst[2].cpu().numpy(), ref.sample_counts)
            assert np.array_equal(dst[0].cpu().numpy().view(np.uint32), ref.color.reshape(-1).view(np.uint32))
            assert np.array_equal(dst[1].cpu().numpy().view(np.uint32), ref.alpha.reshape(-1).view(np.uint32))
        finally:
            lib.vp_comm_destroy(out[0])


def test_native_comm_rejects_bad_arguments():
    lib = _lib.load()
    with Renderer(0) as r:
        idb = (C.c_uint8 * 128)()
        h = C.c_void_p()
        assert lib.vp_comm_init(r.ctx, idb, 2, 5, 0, C.byref(h)) == api.ErrorCategory.USAGE
        assert lib.vp_broadcast_scene(None, 0) == api.ErrorCategory.USAGE

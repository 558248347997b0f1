"""CPU, world_size 2 (gloo): the multi-GPU plumbing of paper_2103_01954_b200/dist.py —
view sharding, the one-time scene broadcast and the per-view gather to rank 0 — with a fake
renderer standing in for the device context."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_01954_b200.dist import ViewGather, broadcast_scene, view_shard


def test_view_shard_partitions():
    for n, world in ((64, 1), (64, 2), (64, 8), (10, 3), (3, 4)):
        parts = [view_shard(n, world, r) for r in range(world)]
        flat = [v for p in parts for v in p]
        assert sorted(flat) == list(range(n))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1
    assert view_shard(64, 8, 3, per_rank=8) == list(range(24, 32))
    assert view_shard(64, 1, 0, per_rank=8) == list(range(8))
    with pytest.raises(ValueError):
        view_shard(64, 2, 2)


class FakeRenderer:
    """Implements the Renderer methods broadcast_scene uses, on host memory."""

    def __init__(self):
        self.xf = None
        self.payload = None
        self.n_prim = self.m = None

    def set_scene_composed(self, xf, slab, window):
        self.xf = np.array(xf, np.float32)
        self.n_prim, self.m = xf.shape[0], slab.voxels_per_axis
        if slab.payload is not None:  # "repack": planar (k, c, v) -> interleaved (k, v, c)
            k, m3 = self.n_prim, self.m ** 3
            self.payload = np.ascontiguousarray(slab.payload.reshape(k, 4, m3).transpose(0, 2, 1)).reshape(-1)

    def payload_floats(self):
        return self.n_prim * self.m ** 3 * 4

    def copy_payload_to(self, ptr):
        ctypes.memmove(ptr, self.payload.ctypes.data, self.payload.nbytes)

    def set_payload_interleaved(self, ptr):
        n = self.payload_floats()
        self.payload = np.ctypeslib.as_array((ctypes.c_float * n).from_address(ptr)).copy()


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2103_01954_b200.api import PrimitiveSlab, WindowParams
        k, m = 5, 2
        rng = np.random.default_rng(7)
        xf = rng.uniform(-1, 1, (k, 15)).astype(np.float32)
        planar = rng.uniform(0, 1, k * 4 * m ** 3).astype(np.float32)
        r = FakeRenderer()
        nbytes = broadcast_scene(r, xf if rank == 0 else None, PrimitiveSlab(k, m, planar) if rank == 0 else None,
                                 WindowParams(), k, m, "cpu")
        want = planar.reshape(k, 4, m ** 3).transpose(0, 2, 1).reshape(-1)
        ok_bcast = bool(np.array_equal(r.payload, want) and np.array_equal(r.xf, xf) and nbytes == want.nbytes)

        # per-view gather: each rank renders 3 "views" of 4x2 pixels
        # in two steps, into the two output slots (as bench.py's step i uses slot i % 2)
        w, h, nv = 4, 2, 3
        vg = ViewGather(nv, w, h, "cpu", world, rank)
        assert vg.slots == 2
        for step in range(3):
            slot = step % vg.slots
            vg.wait_slot(slot)
            rgb, alpha, samples = vg.views(slot)
            for j in range(nv):
                rgb[j].fill_(rank * 10 + j + 1000 * step)
                alpha[j].fill_(0.5 + rank + step)
                samples[j].fill_(100 * rank + j + 1000 * step)
                vg.gather_view(j, slot=slot)
        vg.finish()
        ok_gather = True
        if rank == 0:
            for step, slot in ((1, 1), (2, 0)):  # the latest step in each slot
                for j in range(nv):
                    rows = vg.gathered(j, slot)
                    for src in range(world):
                        c, a, s = ViewGather.unpack(rows[src], w, h)
                        ok_gather &= bool(torch.all(c == src * 10 + j + 1000 * step))
                        ok_gather &= bool(torch.all(a == 0.5 + src + step))
                        ok_gather &= bool(torch.all(s == 100 * src + j + 1000 * step))
        q.put((rank, ok_bcast, ok_gather))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_broadcast_and_gather_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert all(p.exitcode == 0 for p in procs)
    assert res == [(0, True, True), (1, True, True)]


def _split_tile_shard(img, shard, n):
    """Inverse of assemble_tile_shards for one shard: [slots, 256, C] (zeros outside the image)."""
    h, w, c = img.shape
    tx, ty = (w + 15) // 16, (h + 15) // 16
    pad = np.zeros((ty * 16, tx * 16, c), img.dtype)
    pad[:h, :w] = img
    tiles = pad.reshape(ty, 16, tx, 16, c).transpose(0, 2, 1, 3, 4).reshape(tx * ty, 256, c)
    return tiles[shard::n]


@pytest.mark.parametrize("w,h,n", [(64, 64, 1), (64, 48, 2), (100, 37, 3), (1024, 1024, 8), (17, 16, 5)])
def test_assemble_tile_shards_inverts_the_shard_layout(w, h, n):
    from paper_2103_01954_b200.api import shard_tiles
    from paper_2103_01954_b200.dist import assemble_tile_shards
    img = np.random.default_rng(w * h + n).standard_normal((h, w, 3)).astype(np.float32)
    parts = [_split_tile_shard(img, r, n) for r in range(n)]
    assert [len(p) for p in parts] == [shard_tiles(w, h, r, n) for r in range(n)]
    assert sum(len(p) for p in parts) == ((w + 15) // 16) * ((h + 15) // 16)
    assert np.array_equal(assemble_tile_shards(parts, w, h, 3), img)
    tparts = [torch.from_numpy(p.copy()) for p in parts]
    assert np.array_equal(assemble_tile_shards(tparts, w, h, 3).numpy(), img)
    assert shard_tiles(w, h, n, n) == 0 and shard_tiles(w, h, -1, n) == 0 and shard_tiles(0, h, 0, n) == 0


def _shard_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2103_01954_b200.dist import TileShardGather
        w, h = 70, 45
        rng = np.random.default_rng(3)
        rgb = rng.standard_normal((h, w, 3)).astype(np.float32)
        alpha = rng.uniform(0, 1, (h, w, 1)).astype(np.float32)
        samp = rng.integers(0, 500, (h, w, 1)).astype(np.int32)
        g = TileShardGather(w, h, "cpu", world, rank)
        o_rgb, o_alpha, o_samp = g.outputs()
        for out, img, c in ((o_rgb, rgb, 3), (o_alpha, alpha, 1), (o_samp, samp, 1)):
            part = _split_tile_shard(img, rank, world)
            out[:part.size] = torch.from_numpy(np.ascontiguousarray(part).reshape(-1))
        g.gather()
        g.wait()
        ok = True
        if rank == 0:
            a_rgb, a_alpha, a_samp = g.assemble()
            ok = (np.array_equal(a_rgb.numpy(), rgb) and np.array_equal(a_alpha.numpy(), alpha)
                  and np.array_equal(a_samp.numpy(), samp[..., 0]))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_tile_shard_gather_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert all(p.exitcode == 0 for p in procs)
    assert res == [(0, True), (1, True)]


def _id_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2103_01954_b200.dist import NativeComm
        q.put((rank, NativeComm.share_id(world, rank)))
    finally:
        dist.destroy_process_group()


def test_native_comm_id_exchange_world2():
    """bench.py's N > 1 control plane (gloo) hands rank 0's NCCL id (vp_comm_unique_id, 128 bytes)
    to every rank before vp_comm_init; the data plane itself needs GPUs (tests/test_gpu_comm.py)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert all(p.exitcode == 0 for p in procs)
    assert len(res[0][1]) == 128 and res[0][1] == res[1][1]

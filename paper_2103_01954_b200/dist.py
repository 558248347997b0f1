"""Multi-GPU plumbing: one process per GPU. Two data planes: the library's own NCCL
(`NativeComm` / `NativeViewGather` over include/vpb.h vp_comm_*, what bench.py uses and what a
C++ caller uses) and torch.distributed collectives (`broadcast_scene`, `ViewGather`,
`TileShardGather`, also runnable with gloo on CPU tensors).

The raymarcher shards by view: rays are independent and the scene is
read-only, so each rank renders its own views with no data-path collective. A single view
shards by tile (`TileShardGather`): rank r renders the tiles t % world == r
(vp_render_shard_async, tile-major outputs) and rank 0 gathers and places them. The only
communication is
  * a one-time broadcast of the repacked, channel-interleaved payload (K*M^3*16 bytes) and the
    composed transforms from rank 0 (`broadcast_scene`), and
  * optionally, gathering each step's rendered views to rank 0 (`ViewGather`), double-buffered
    so the transfer of step s overlaps the rendering of step s+1.
Everything here also runs on CPU tensors with the gloo backend (tests/test_dist_gloo.py).
"""
from __future__ import annotations

from typing import List, Optional

import numpy as np


def view_shard(n_views: int, world: int, rank: int, per_rank: Optional[int] = None) -> List[int]:
    """Views rendered by `rank`. With per_rank=None the n_views batch is split into contiguous
    blocks (strong sharding of a fixed batch); with per_rank=p, rank r renders
    [r*p, (r+1)*p) modulo n_views (fixed work per GPU)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if per_rank is None:
        base, extra = divmod(n_views, world)
        start = rank * base + min(rank, extra)
        return list(range(start, start + base + (1 if rank < extra else 0)))
    return [(rank * per_rank + i) % n_views for i in range(per_rank)]


def broadcast_scene(renderer, xf15: Optional[np.ndarray], slab, window, n_prim: int, m: int,
                    device, src: int = 0):
    """Rank `src` uploads (and repacks) the frame; the interleaved payload and the composed
    transforms are broadcast once; the other ranks adopt them without a repack."""
    import torch
    import torch.distributed as dist

    from .api import PrimitiveSlab

    rank = dist.get_rank()
    xf_t = torch.empty((n_prim, 15), dtype=torch.float32, device=device)
    if rank == src:
        xf_t.copy_(torch.from_numpy(np.ascontiguousarray(xf15, np.float32)))
    dist.broadcast(xf_t, src)
    xf = xf_t.cpu().numpy()
    if rank == src:
        renderer.set_scene_composed(xf, slab, window)
    else:
        renderer.set_scene_composed(xf, PrimitiveSlab(n_prim, m, None), window)
    pay = torch.empty(renderer.payload_floats(), dtype=torch.float32, device=device)
    if rank == src:
        renderer.copy_payload_to(pay.data_ptr())
    dist.broadcast(pay, src)
    if rank != src:
        renderer.set_payload_interleaved(pay.data_ptr())
    return pay.numel() * 4


class ViewGather:
    """Per-step output buffers ([views, H*W*5] float32 rows: rgb, alpha, samples as int32
    bits) and the per-view asynchronous gather to rank `dst`.

    There are `slots` output buffers (default 2): step s renders into slot s % slots, and its
    gathers run on NCCL's stream while step s+1 renders into the other slot. Before a slot is
    rendered into again, `wait_slot` makes the current stream wait for the gathers that read
    it, so at most one step of transfers is in flight and it overlaps the next step's raymarch
    instead of serialising behind it."""

    def __init__(self, n_local: int, width: int, height: int, device, world: int, rank: int,
                 dst: int = 0, slots: int = 2):
        import torch
        self.hw = width * height
        self.slots = max(1, slots)
        self.bufs = [torch.zeros((n_local, 5 * self.hw), dtype=torch.float32, device=device)
                     for _ in range(self.slots)]
        self.buf = self.bufs[0]
        self.world, self.rank, self.dst = world, rank, dst
        self.recvs = ([[[torch.empty(5 * self.hw, dtype=torch.float32, device=device) for _ in range(world)]
                        for _ in range(n_local)] for _ in range(self.slots)] if rank == dst else None)
        self.recv = self.recvs[0] if self.recvs is not None else None
        self.works = [[] for _ in range(self.slots)]

    def views(self, slot: int = 0):
        """(rgb, alpha, samples) row views of one slot, one row per local view."""
        import torch
        hw, buf = self.hw, self.bufs[slot % self.slots]
        return buf[:, :3 * hw], buf[:, 3 * hw:4 * hw], buf[:, 4 * hw:].view(torch.int32)

    def gather_view(self, j: int, async_op: bool = True, slot: int = 0):
        import torch.distributed as dist
        if self.world == 1:
            return
        s = slot % self.slots
        w = dist.gather(self.bufs[s][j], self.recvs[s][j] if self.rank == self.dst else None,
                        dst=self.dst, async_op=async_op)
        if async_op:
            self.works[s].append(w)

    def wait_slot(self, slot: int):
        """The current stream waits for the in-flight gathers that read `slot` (call before
        rendering into it again)."""
        s = slot % self.slots
        for w in self.works[s]:
            w.wait()
        self.works[s].clear()

    def finish(self):
        for s in range(self.slots):
            self.wait_slot(s)

    def gathered(self, j: int, slot: int = 0):
        """On rank dst: per-rank [5*H*W] rows of local view j of one slot."""
        return self.recvs[slot % self.slots][j]

    @staticmethod
    def unpack(row, width: int, height: int):
        """(rgb [H,W,3], alpha [H,W,1], samples [H*W] int32) from one gathered row."""
        import torch
        hw = width * height
        return (row[:3 * hw].reshape(height, width, 3), row[3 * hw:4 * hw].reshape(height, width, 1),
                row[4 * hw:].view(torch.int32))


def assemble_tile_shards(parts, width: int, height: int, channels: int):
    """The [H, W, channels] image from the tile-major shard outputs parts[r] ([slots_r (or
    more), 256, channels], numpy or torch): slot s of shard r is tile t = s * n + r (row-major
    over the ceil(W/16) x ceil(H/16) grid), pixel (y % 16) * 16 + x % 16 of it."""
    n = len(parts)
    tx, ty = (width + 15) // 16, (height + 15) // 16
    n_tiles = tx * ty
    p0 = parts[0]
    if hasattr(p0, "new_empty"):  # torch
        tiles = p0.new_zeros((n_tiles, 256, channels))
    else:
        tiles = np.zeros((n_tiles, 256, channels), p0.dtype)
    for r, part in enumerate(parts):
        k = len(range(r, n_tiles, n))
        tiles[r::n] = part.reshape(-1, 256, channels)[:k]
    img = tiles.reshape(ty, tx, 16, 16, channels)
    img = img.permute(0, 2, 1, 3, 4) if hasattr(img, "permute") else img.transpose(0, 2, 1, 3, 4)
    return img.reshape(ty * 16, tx * 16, channels)[:height, :width]


class TileShardGather:
    """Single-view tile sharding: this rank's tile-major outputs (rgb, alpha, samples as int32
    bits in one float32 buffer of slots_max * 256 * 5 values, slots_max = the largest shard's
    tile count, so every rank sends the same size) and their gather to rank `dst`, which
    places the tiles into the [H, W] image (assemble)."""

    def __init__(self, width: int, height: int, device, world: int, rank: int, dst: int = 0):
        import torch
        from .api import shard_tiles
        self.width, self.height, self.world, self.rank, self.dst = width, height, world, rank, dst
        self.slots = [shard_tiles(width, height, r, world) for r in range(world)]
        self.slots_max = max(max(self.slots), 1)
        n = self.slots_max * 256
        self.n = n
        self.buf = torch.zeros(5 * n, dtype=torch.float32, device=device)
        self.recv = ([torch.empty(5 * n, dtype=torch.float32, device=device) for _ in range(world)]
                     if rank == dst else None)
        self.work = None

    def outputs(self):
        """(rgb, alpha, samples) device views of this rank's shard buffer."""
        import torch
        n = self.n
        return self.buf[:3 * n], self.buf[3 * n:4 * n], self.buf[4 * n:].view(torch.int32)

    def gather(self, async_op: bool = True):
        import torch.distributed as dist
        if self.world == 1:
            return
        self.work = dist.gather(self.buf, self.recv if self.rank == self.dst else None, dst=self.dst,
                                async_op=async_op)

    def wait(self):
        if self.work is not None:
            self.work.wait()
            self.work = None

    def assemble(self):
        """On rank dst: (rgb [H,W,3], alpha [H,W,1], samples [H,W] int32) of the whole view."""
        import torch
        rows = self.recv if self.world > 1 else [self.buf]
        n = self.n
        rgb = assemble_tile_shards([r[:3 * n].view(-1, 256, 3) for r in rows], self.width, self.height, 3)
        alpha = assemble_tile_shards([r[3 * n:4 * n].view(-1, 256, 1) for r in rows], self.width, self.height, 1)
        samp = assemble_tile_shards([r[4 * n:].view(torch.int32).view(-1, 256, 1) for r in rows],
                                    self.width, self.height, 1)
        return rgb, alpha, samp[..., 0]


class NativeComm:
    """The multi-GPU C-ABI of libvpb (include/vpb.h vp_comm_*: NCCL inside the library, no torch
    on the data path). torch.distributed (any backend, gloo included) is used only to hand the
    128-byte NCCL id from rank 0 to the others. One communicator per Renderer (its device)."""

    def __init__(self, renderer, world: int, rank: int, max_ctas: int = 8, comm_id: Optional[bytes] = None):
        import ctypes as C
        from . import _lib
        from .api import _check
        self.lib, self.r, self.world, self.rank = renderer._lib, renderer, world, rank
        self.C = C
        if comm_id is None:
            comm_id = self.share_id(world, rank)
        idb = (C.c_uint8 * 128).from_buffer_copy(comm_id)
        h = C.c_void_p()
        rc = self.lib.vp_comm_init(renderer.ctx, idb, world, rank, max_ctas, C.byref(h))
        if rc:
            raise RuntimeError(f"vp_comm_init failed ({rc}): {self.lib.vp_last_error(renderer.ctx).decode()}")
        self.h = h
        self._check = _check
        self._lib = _lib

    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C
        from . import _lib
        lib = _lib.load()
        buf = (C.c_uint8 * 128)()
        if lib.vp_comm_unique_id(buf):
            raise RuntimeError(f"vp_comm_unique_id: {lib.vp_comm_last_error().decode()}")
        return bytes(buf)

    @staticmethod
    def share_id(world: int, rank: int) -> bytes:
        """Rank 0's NCCL id, broadcast over torch.distributed (world 1: a local id)."""
        if world == 1:
            return NativeComm.unique_id()
        import torch.distributed as dist
        obj = [NativeComm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def broadcast_scene(self, xf15, slab, window, n_prim: int, m: int, root: int = 0) -> int:
        """vp_set_scene on every rank (the root with its data, the others shape only), then
        vp_broadcast_scene: the root's composed transforms and repacked payload, once."""
        if self.rank == root:
            self.r.set_scene_composed(xf15, slab, window)
        else:
            self._check(self.lib.vp_set_scene(self.r.ctx, int(n_prim), int(m), None, None, float(window.alpha),
                                              int(window.beta)), self.r.ctx)
            self.r.n_prim, self.r.m = int(n_prim), int(m)
        self._check(self.lib.vp_broadcast_scene(self.h, root), self.r.ctx)
        self._check(self.lib.vp_comm_sync(self.h), self.r.ctx)
        return int(n_prim) * (16 + 4 * int(m) ** 3) * 4

    def gather_views(self, n_views: int, n_px: int, rgb, alpha, samples, dst=None, root: int = 0):
        """vp_gather_views: this rank's n_views device outputs (pointer lists) to the root;
        dst = (rgb, alpha, samples) pointer lists of n_ranks * n_views entries on the root."""
        C = self.C
        f32p, i32p = self._lib.f32p, self._lib.i32p
        P = lambda ptrs, t: (t * len(ptrs))(*[C.cast(C.c_void_p(p), t) for p in ptrs])  # noqa: E731
        src = (P(rgb, f32p), P(alpha, f32p), P(samples, i32p) if samples is not None else None)
        d = (None, None, None)
        if dst is not None:
            d = (P(dst[0], f32p), P(dst[1], f32p), P(dst[2], i32p) if dst[2] is not None else None)
        self._check(self.lib.vp_gather_views(self.h, root, n_views, n_px, src[0], src[1], src[2], d[0], d[1], d[2]),
                    self.r.ctx)

    def wait(self, stream: int = 0):
        """`stream` (0: the context's) waits for the communicator's work so far."""
        self._check(self.lib.vp_comm_wait(self.h, self.C.c_void_p(stream) if stream else None), self.r.ctx)

    def sync(self):
        self._check(self.lib.vp_comm_sync(self.h), self.r.ctx)

    def close(self):
        if getattr(self, "h", None):
            self.lib.vp_comm_destroy(self.h)
            self.h = None


class NativeViewGather:
    """ViewGather over the native communicator: per slot, every local view's rgb / alpha /
    samples device buffers; each step's gather of all its views is ONE vp_gather_views call (one
    NCCL group) on the communicator's stream, overlapping the next step's raymarch, which
    renders into the other slot. wait_slot makes the render stream wait for the gathers so far
    before a slot is rendered into again."""

    def __init__(self, comm: NativeComm, n_local: int, width: int, height: int, device, dst: int = 0,
                 slots: int = 2):
        import torch
        self.comm, self.n, self.hw, self.dst, self.slots = comm, n_local, width * height, dst, max(1, slots)
        hw = self.hw
        self.bufs = [(torch.zeros((n_local, 3 * hw), dtype=torch.float32, device=device),
                      torch.zeros((n_local, hw), dtype=torch.float32, device=device),
                      torch.zeros((n_local, hw), dtype=torch.int32, device=device)) for _ in range(self.slots)]
        world = comm.world
        self.recv = None
        if comm.rank == dst:  # [slot] -> (rgb, alpha, samples) of world * n_local views
            self.recv = [(torch.empty((world * n_local, 3 * hw), dtype=torch.float32, device=device),
                          torch.empty((world * n_local, hw), dtype=torch.float32, device=device),
                          torch.empty((world * n_local, hw), dtype=torch.int32, device=device))
                         for _ in range(self.slots)]

    def views(self, slot: int = 0):
        return self.bufs[slot % self.slots]

    def gather(self, slot: int, stream: int = 0):
        s = slot % self.slots
        rgb, alpha, samp = self.bufs[s]
        ptr = lambda t: [t[j].data_ptr() for j in range(t.shape[0])]  # noqa: E731
        dst = None
        if self.recv is not None:
            dst = tuple(ptr(t) for t in self.recv[s])
        self.comm.gather_views(self.n, self.hw, ptr(rgb), ptr(alpha), ptr(samp), dst, self.dst)

    def wait_slot(self, slot: int, stream: int = 0):
        self.comm.wait(stream)

    def finish(self):
        self.comm.sync()

"""Python mirror of the reference renderer interface (volprim::render and friends).

Names, argument meaning and error behaviour follow
/root/reference/proj/src/volprim/{march.h,scene.h,primitive.h,camera.h,errors.h}:

    render(scene, frame, cam, cfg) -> RenderOutput          march.h:59 / march.cpp:95-132
    composite(out, background) -> image                      march.h:62 / march.cpp:134-147
    compose(transforms) -> AffineXf records                  primitive.cpp:41-49
    Error(category, message), ErrorCategory                  errors.h:11-38

All compute runs through libvpb.so (include/vpb.h) on an sm_100a GPU; there is no CPU path.
Arrays are numpy float32; matrices are 3x3 arrays in (row, col) indexing and are passed to
the C-ABI column-major, like volprim::Mat3::m.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import f32p, i32p, u32p, vp_camera, vp_march, vp_stats


class ErrorCategory(enum.IntEnum):
    """errors.h:11-17, plus DEVICE for CUDA failures (no reference counterpart)."""
    USAGE = 2
    IO = 3
    FORMAT = 4
    VERSION = 5
    NUMERIC = 6
    DEVICE = 7


class Error(RuntimeError):
    """volprim::Error: a message plus a category whose value is the CLI exit code."""

    def __init__(self, category: int, message: str):
        super().__init__(message)
        try:
            self.category = ErrorCategory(category)
        except ValueError:
            self.category = ErrorCategory.DEVICE
        self.exit_code = int(self.category)


def _check(rc: int, ctx=None):
    if rc != 0:
        lib = _lib.load()
        msg = lib.vp_last_error(ctx)
        raise Error(rc, msg.decode() if msg else f"libvpb error {rc}")


def _fptr(a: np.ndarray):
    return a.ctypes.data_as(f32p)


def _f32(a, shape=None) -> np.ndarray:
    out = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    if shape is not None:
        out = out.reshape(shape)
    return out


# ----------------------------------------------------------------------------------------
# Scene model (primitive.h, scene.h, march.h, camera.h)

@dataclass
class WindowParams:
    """primitive.h:14-17"""
    alpha: float = 8.0
    beta: int = 8


@dataclass
class MarchConfig:
    """march.h:11-20"""
    step_size: float = 0.001
    early_eps: float = 0.01
    jitter: bool = False
    seed: int = 0
    accumulation_permutation: int = 0

    def to_c(self) -> vp_march:
        return vp_march(float(self.step_size), float(self.early_eps), 1 if self.jitter else 0, 0,
                        int(self.seed) & (2**64 - 1), int(self.accumulation_permutation) & (2**64 - 1))


def transform_records(t_base, r_base, s_base, delta_t=None, delta_r=None, delta_s=None) -> np.ndarray:
    """Packs PrimitiveTransform fields (primitive.h:45-52) into K x 24 float32 records:
    tBase[3] rBase[9] (column-major) sBase[3] deltaT[3] deltaR[3] deltaS[3]."""
    t_base = _f32(t_base).reshape(-1, 3)
    k = t_base.shape[0]
    r_base = _f32(r_base).reshape(k, 3, 3)
    rec = np.zeros((k, 24), np.float32)
    rec[:, 0:3] = t_base
    rec[:, 3:12] = np.transpose(r_base, (0, 2, 1)).reshape(k, 9)  # column-major
    rec[:, 12:15] = _f32(s_base).reshape(k, 3)
    for off, arr in ((15, delta_t), (18, delta_r), (21, delta_s)):
        if arr is not None:
            rec[:, off:off + 3] = _f32(arr).reshape(k, 3)
    return rec


@dataclass
class PrimitiveSlab:
    """primitive.h:25-41: planar payload (k, channel, z, y, x)."""
    num_primitives: int = 0
    voxels_per_axis: int = 0
    payload: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))

    @staticmethod
    def zeros(n_prim: int, m: int) -> "PrimitiveSlab":
        return PrimitiveSlab(n_prim, m, np.zeros(n_prim * 4 * m ** 3, np.float32))

    def index(self, k: int, channel: int, z: int, y: int, x: int) -> int:
        m = self.voxels_per_axis
        return (((k * 4 + channel) * m + z) * m + y) * m + x

    def view(self) -> np.ndarray:
        m = self.voxels_per_axis
        return self.payload.reshape(self.num_primitives, 4, m, m, m)


@dataclass
class Frame:
    """scene.h:14-28. transforms: K x 24 PrimitiveTransform records (transform_records)."""
    transforms: np.ndarray = field(default_factory=lambda: np.zeros((0, 24), np.float32))
    slab: PrimitiveSlab = field(default_factory=PrimitiveSlab)

    def composed(self) -> np.ndarray:
        return compose(self.transforms)


@dataclass
class Scene:
    """scene.h:30-34 (the guide mesh is not read by render())."""
    window: WindowParams = field(default_factory=WindowParams)
    march: MarchConfig = field(default_factory=MarchConfig)
    frames: List[Frame] = field(default_factory=list)


@dataclass
class Camera:
    """camera.h:21-29: x_cam = R x_world + t, pixel = K x_cam / z."""
    intrinsics: np.ndarray = field(default_factory=lambda: np.eye(3, dtype=np.float32))
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3, dtype=np.float32))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3, np.float32))
    width: int = 0
    height: int = 0

    def to_c(self) -> vp_camera:
        c = vp_camera()
        c.K[:] = _f32(self.intrinsics).reshape(3, 3).T.reshape(-1).tolist()
        c.R[:] = _f32(self.rotation).reshape(3, 3).T.reshape(-1).tolist()
        c.t[:] = _f32(self.translation).reshape(3).tolist()
        c.width = int(self.width)
        c.height = int(self.height)
        return c

    @staticmethod
    def from_c(c: vp_camera) -> "Camera":
        return Camera(np.array(c.K, np.float32).reshape(3, 3).T.copy(),
                      np.array(c.R, np.float32).reshape(3, 3).T.copy(),
                      np.array(c.t, np.float32), int(c.width), int(c.height))

    def center(self) -> np.ndarray:
        return -(self.rotation.T.astype(np.float32) @ self.translation.astype(np.float32))


@dataclass
class RenderOutput:
    """march.h:46-56"""
    color: np.ndarray
    alpha: np.ndarray
    sample_counts: np.ndarray
    stats: Optional[dict] = None

    def total_samples(self) -> int:
        return int(self.sample_counts.astype(np.int64).sum())


# ----------------------------------------------------------------------------------------

def compose(transforms: np.ndarray) -> np.ndarray:
    """Frame::composed(): K x 24 PrimitiveTransform records -> K x 15 AffineXf records
    (t[3] rot[9] column-major scale[3]). Raises Error(USAGE) on a non-positive scale."""
    lib = _lib.load()
    tr = _f32(transforms).reshape(-1, 24)
    out = np.zeros((tr.shape[0], 15), np.float32)
    _check(lib.vp_compose(tr.shape[0], _fptr(tr), _fptr(out)))
    return out


class Renderer:
    """A device context holding one resident frame (transforms + repacked payload)."""

    def __init__(self, device: int = 0):
        self._lib = _lib.load()
        ctx = C.c_void_p()
        _check(self._lib.vp_create(int(device), C.byref(ctx)))
        self._ctx = ctx
        self.device = device
        self.n_prim = None
        self.m = None

    def close(self):
        if getattr(self, "_ctx", None):
            self._lib.vp_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def ctx(self):
        return self._ctx

    def stream_handle(self) -> int:
        return int(self._lib.vp_stream(self._ctx) or 0)

    # -- resident scene ---------------------------------------------------------------
    def set_scene_composed(self, xf15: np.ndarray, slab: PrimitiveSlab, window: WindowParams):
        """Upload composed transforms and the planar slab (repacked on the device). A slab
        with payload=None only allocates (fill it with set_payload_interleaved)."""
        xf = _f32(xf15).reshape(-1, 15)
        pay = None if slab.payload is None else _f32(slab.payload)
        _check(self._lib.vp_set_scene(self._ctx, xf.shape[0], int(slab.voxels_per_axis),
                                      _fptr(xf), _fptr(pay) if pay is not None else None,
                                      float(window.alpha), int(window.beta)), self._ctx)
        self.n_prim, self.m = xf.shape[0], int(slab.voxels_per_axis)

    def payload_floats(self) -> int:
        return int(self.n_prim or 0) * int(self.m or 0) ** 3 * 4

    def copy_payload_to(self, ptr: int):
        """Copy the resident channel-interleaved payload to `ptr` (device or host)."""
        _check(self._lib.vp_copy_payload(self._ctx, C.cast(C.c_void_p(ptr), f32p)), self._ctx)

    def set_payload_interleaved(self, ptr: int):
        """Adopt an interleaved payload at `ptr` (device or host), e.g. after a broadcast."""
        _check(self._lib.vp_set_payload_interleaved(self._ctx, int(self.n_prim), int(self.m),
                                                    C.cast(C.c_void_p(ptr), f32p)), self._ctx)

    def kernel_times(self, max_n: int = 256) -> np.ndarray:
        """Raymarch-kernel device durations (ms) of the renders since the last call."""
        out = np.zeros(max_n, np.float32)
        n = C.c_int64()
        _check(self._lib.vp_kernel_times(self._ctx, max_n, _fptr(out), C.byref(n)), self._ctx)
        return out[:n.value]

    def set_frame(self, scene: Scene, frame: int):
        """Make scene.frames[frame] resident: the slab is repacked and the frame's
        PrimitiveTransform records are composed on the device (Frame::composed())."""
        if frame < 0 or frame >= len(scene.frames):
            raise Error(ErrorCategory.USAGE, "frame index out of range")  # march.cpp:96-97
        fr = scene.frames[frame]
        self.set_scene_records(fr.transforms, fr.slab, scene.window)

    def set_scene_records(self, transforms: np.ndarray, slab: PrimitiveSlab, window: WindowParams):
        """Upload the planar slab and K x 24 PrimitiveTransform records; compose on the device."""
        tr = _f32(transforms).reshape(-1, 24)
        pay = None if slab.payload is None else _f32(slab.payload)
        _check(self._lib.vp_set_scene(self._ctx, tr.shape[0], int(slab.voxels_per_axis), None,
                                      _fptr(pay) if pay is not None else None,
                                      float(window.alpha), int(window.beta)), self._ctx)
        self.n_prim, self.m = tr.shape[0], int(slab.voxels_per_axis)
        self.set_records(tr)

    def set_records(self, transforms: np.ndarray):
        """A new pose for the resident frame: K x 24 records composed on the device."""
        tr = _f32(transforms).reshape(-1, 24)
        _check(self._lib.vp_set_frame(self._ctx, tr.shape[0], _fptr(tr)), self._ctx)

    def transforms(self) -> np.ndarray:
        """The resident composed transforms (K x 15 AffineXf records)."""
        out = np.zeros((int(self.n_prim or 0), 15), np.float32)
        _check(self._lib.vp_get_transforms(self._ctx, _fptr(out)), self._ctx)
        return out

    def load_slab(self, path: str, xf15: np.ndarray, window: WindowParams):
        """loadSlab (scene_io.cpp:43-66) streamed straight into the device layout; xf15 are the
        frame's composed transforms. Raises Error(IO / FORMAT / VERSION) like the reference."""
        xf = _f32(xf15).reshape(-1, 15)
        _check(self._lib.vp_load_slab(self._ctx, str(path).encode(), xf.shape[0], _fptr(xf),
                                      float(window.alpha), int(window.beta)), self._ctx)
        self.n_prim = xf.shape[0]
        with open(path, "rb") as f:
            f.seek(12)
            self.m = int(np.frombuffer(f.read(4), "<u4")[0])

    def set_transforms(self, xf15: np.ndarray):
        xf = _f32(xf15).reshape(-1, 15)
        _check(self._lib.vp_set_transforms(self._ctx, xf.shape[0], _fptr(xf)), self._ctx)

    # -- render -----------------------------------------------------------------------
    def render(self, cam: Camera, cfg: MarchConfig, with_stats: bool = True) -> RenderOutput:
        w, h = int(cam.width), int(cam.height)
        color = np.zeros((h, w, 3), np.float32)
        alpha = np.zeros((h, w, 1), np.float32)
        samples = np.zeros(h * w, np.int32)
        st = vp_stats()
        cc, mc = cam.to_c(), cfg.to_c()
        _check(self._lib.vp_render(self._ctx, C.byref(cc), C.byref(mc), _fptr(color), _fptr(alpha),
                                   samples.ctypes.data_as(i32p), C.byref(st)), self._ctx)
        return RenderOutput(color, alpha, samples, st.as_dict() if with_stats else None)

    def render_batch(self, cams: List[Camera], cfg: MarchConfig) -> List[RenderOutput]:
        """Up to 16 views of the resident frame in one raymarch launch (vp_render_batch_async)
        into host arrays; waits for the copies (vp_sync). Stats are not per view here."""
        n = len(cams)
        if n == 0:
            return []
        outs = [RenderOutput(np.zeros((int(c.height), int(c.width), 3), np.float32),
                             np.zeros((int(c.height), int(c.width), 1), np.float32),
                             np.zeros(int(c.height) * int(c.width), np.int32), None) for c in cams]
        cc = (vp_camera * n)(*[c.to_c() for c in cams])
        mc = cfg.to_c()
        rgb = (f32p * n)(*[_fptr(o.color) for o in outs])
        alpha = (f32p * n)(*[_fptr(o.alpha) for o in outs])
        samp = (i32p * n)(*[o.sample_counts.ctypes.data_as(i32p) for o in outs])
        _check(self._lib.vp_render_batch_async(self._ctx, n, cc, C.byref(mc), rgb, alpha, samp, None), self._ctx)
        _check(self._lib.vp_sync(self._ctx), self._ctx)
        return outs

    def render_device(self, cam: Camera, cfg: MarchConfig, rgb_ptr: int, alpha_ptr: int,
                      samples_ptr: int = 0, stream: int = 0):
        """Enqueue a render into device buffers (e.g. torch CUDA tensors' data_ptr())."""
        cc, mc = cam.to_c(), cfg.to_c()
        _check(self._lib.vp_render_async(self._ctx, C.byref(cc), C.byref(mc),
                                         C.cast(C.c_void_p(rgb_ptr), f32p),
                                         C.cast(C.c_void_p(alpha_ptr), f32p),
                                         C.cast(C.c_void_p(samples_ptr), i32p) if samples_ptr else None,
                                         C.c_void_p(stream) if stream else None), self._ctx)

    def render_shard_device(self, cam: Camera, cfg: MarchConfig, shard: int, n_shards: int, rgb_ptr: int,
                            alpha_ptr: int, samples_ptr: int = 0, stream: int = 0):
        """Enqueue shard `shard` of `n_shards` of a view (vp_render_shard_async) into device
        buffers in the tile-major layout (shard_tiles(...) slots of 256 pixels)."""
        cc, mc = cam.to_c(), cfg.to_c()
        _check(self._lib.vp_render_shard_async(self._ctx, C.byref(cc), C.byref(mc), int(shard), int(n_shards),
                                               C.cast(C.c_void_p(rgb_ptr), f32p),
                                               C.cast(C.c_void_p(alpha_ptr), f32p),
                                               C.cast(C.c_void_p(samples_ptr), i32p) if samples_ptr else None,
                                               C.c_void_p(stream) if stream else None), self._ctx)

    def set_key_capacity(self, keys: int, grow: bool = True):
        """vp_set_key_capacity: tile-key buffer capacity per view (0 = default). Renders stay
        exact when it is too small (overflowed tiles go to the fallback kernel)."""
        _check(self._lib.vp_set_key_capacity(self._ctx, int(keys), int(bool(grow))), self._ctx)

    def read_stats(self) -> dict:
        st = vp_stats()
        _check(self._lib.vp_read_stats(self._ctx, C.byref(st)), self._ctx)
        return st.as_dict()

    def march_rays(self, origins, dirs, cfg: MarchConfig, jitter01=None):
        o = _f32(origins).reshape(-1, 3)
        d = _f32(dirs).reshape(-1, 3)
        n = o.shape[0]
        j = None if jitter01 is None else _f32(jitter01).reshape(n)
        rgb = np.zeros((n, 3), np.float32)
        alpha = np.zeros(n, np.float32)
        samples = np.zeros(n, np.int32)
        mc = cfg.to_c()
        _check(self._lib.vp_march_rays(self._ctx, n, _fptr(o), _fptr(d),
                                       _fptr(j) if j is not None else None, C.byref(mc),
                                       _fptr(rgb), _fptr(alpha), samples.ctypes.data_as(i32p)),
               self._ctx)
        return rgb, alpha, samples

    def backward_rays(self, origins, dirs, adj_rgb, adj_alpha, cfg: MarchConfig, transforms,
                      jitter01=None, grads: Optional[np.ndarray] = None) -> np.ndarray:
        """backwardRay (grad.cpp:34-195) for each ray with the given output adjoints; returns
        (or accumulates into `grads`) the GradBuffer values: K*4*M^3 planar payload entries,
        then deltaT[3] deltaR[3] deltaS[3] per primitive (params.h:12-27)."""
        o = _f32(origins).reshape(-1, 3)
        d = _f32(dirs).reshape(-1, 3)
        n = o.shape[0]
        ar = _f32(adj_rgb).reshape(n, 3)
        aa = _f32(adj_alpha).reshape(n)
        j = None if jitter01 is None else _f32(jitter01).reshape(n)
        tr = _f32(transforms).reshape(-1, 24)
        k, m = int(self.n_prim or 0), int(self.m or 0)
        size = k * 4 * m ** 3 + 9 * k
        acc = grads is not None
        out = grads if acc else np.zeros(size, np.float32)
        if out.dtype != np.float32 or out.size != size or not out.flags.c_contiguous:
            raise Error(ErrorCategory.USAGE, "gradient buffer must be contiguous float32 of the GradBuffer size")
        mc = cfg.to_c()
        _check(self._lib.vp_backward_rays(self._ctx, n, _fptr(o), _fptr(d), _fptr(j) if j is not None else None,
                                          _fptr(ar), _fptr(aa), C.byref(mc), _fptr(tr), _fptr(out),
                                          1 if acc else 0), self._ctx)
        return out

    def debug_tiles(self, cam: Camera):
        """Cull rectangles, depth keys, tile offsets and per-tile sorted primitive lists."""
        k = self.n_prim or 0
        tiles = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
        rects = np.zeros((max(k, 1), 4), np.int32)
        keys = np.zeros(max(k, 1), np.uint32)
        offs = np.zeros(tiles + 1, np.int32)
        n_keys = C.c_int64()
        cc = cam.to_c()
        _check(self._lib.vp_debug_tiles(self._ctx, C.byref(cc), rects.ctypes.data_as(i32p),
                                        keys.ctypes.data_as(u32p), offs.ctypes.data_as(i32p),
                                        None, 0, C.byref(n_keys)), self._ctx)
        prims = np.zeros(max(n_keys.value, 1), np.int32)
        _check(self._lib.vp_debug_tiles(self._ctx, C.byref(cc), None, None, None,
                                        prims.ctypes.data_as(i32p), prims.size, C.byref(n_keys)),
               self._ctx)
        return rects[:k], keys[:k], offs, prims[:n_keys.value]

    def debug_sincos(self, x: np.ndarray, cos: bool = False) -> np.ndarray:
        x = _f32(x).reshape(-1)
        y = np.empty_like(x)
        _check(self._lib.vp_debug_sincos(self._ctx, x.size, _fptr(x), _fptr(y), 1 if cos else 0), self._ctx)
        return y

    def debug_expf(self, x: np.ndarray) -> np.ndarray:
        x = _f32(x).reshape(-1)
        y = np.empty_like(x)
        _check(self._lib.vp_debug_expf(self._ctx, x.size, _fptr(x), _fptr(y)), self._ctx)
        return y

    def composite(self, out: RenderOutput, background: np.ndarray) -> np.ndarray:
        h, w = out.color.shape[:2]
        bg = _f32(background)
        if bg.shape != (h, w, 3):
            raise Error(ErrorCategory.USAGE, "background dimensions do not match render")
        res = np.zeros((h, w, 3), np.float32)
        _check(self._lib.vp_composite(self._ctx, w, h, _fptr(out.color), _fptr(out.alpha),
                                      _fptr(bg), _fptr(res)), self._ctx)
        return res


# ----------------------------------------------------------------------------------------
# Training rows: evalLoss (grad.cpp:197-251) and adamStep (losses.cpp:70-104)

@dataclass
class LossWeights:
    """losses.h:10-15 (`del` is a Python keyword: del_)."""
    pho: float = 1.0
    geo: float = 0.1
    vol: float = 0.01
    del_: float = 0.01


@dataclass
class LossTerms:
    """grad.h:28-31"""
    pho: float = 0.0
    geo: float = 0.0
    vol: float = 0.0
    del_: float = 0.0

    def total(self) -> float:
        return float(np.float32(np.float32(np.float32(self.pho) + np.float32(self.geo)) + np.float32(self.vol))
                     + np.float32(self.del_))


@dataclass
class RaySamples:
    """A batch of RaySample (grad.h:12-18) as arrays: camera_index (n,), pixel (n, 2) pixel
    coordinates (x + 0.5, y + 0.5 for centres), pixel_id (n,), target and background (n, 3)."""
    camera_index: np.ndarray
    pixel: np.ndarray
    pixel_id: np.ndarray
    target: np.ndarray
    background: np.ndarray


@dataclass
class AdamConfig:
    """losses.h:34-44"""
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    lr_delta_scale: float = 1.0
    lr_vertex_scale: float = 1.0


def grad_size(n_prim: int, m: int, n_verts: int = 0) -> int:
    """ParamLayout::total() (params.h:12-27)."""
    return n_prim * 4 * m ** 3 + 9 * n_prim + 3 * n_verts


def eval_loss(renderer: "Renderer", scene: Scene, frame: int, cams: List[Camera], batch: RaySamples,
              weights: LossWeights, cfg: MarchConfig, grads: Optional[np.ndarray] = None,
              tracked_verts: Optional[np.ndarray] = None, mesh_vertices: Optional[np.ndarray] = None,
              vertex_offsets: Optional[np.ndarray] = None, upload: bool = True) -> LossTerms:
    """evalLoss (grad.cpp:197-251): uploads the frame, runs the photometric term on the device
    (rays, march, composite, L_pho and, with `grads`, backwardRay), adds L_vol / L_del (and
    L_geo when tracked vertices are given) on the host. `grads` (GradBuffer layout, float32 of
    grad_size(K, M, n_verts)) accumulates like the reference's GradBuffer."""
    if frame < 0 or frame >= len(scene.frames):
        raise Error(ErrorCategory.USAGE, "frame index out of range")
    lib = _lib.load()
    fr = scene.frames[frame]
    if upload:  # else the renderer already holds this frame (e.g. after adam_step)
        renderer.set_frame(scene, frame)
    k, m = len(fr.transforms), fr.slab.voxels_per_axis
    tr = _f32(fr.transforms).reshape(-1, 24)
    n = int(np.asarray(batch.camera_index).size)
    cams_c = (_lib.vp_camera * len(cams))(*[c.to_c() for c in cams])
    ci = np.ascontiguousarray(batch.camera_index, np.int32)
    pid = np.ascontiguousarray(batch.pixel_id, np.int32)
    terms = LossTerms()
    nv = 0 if tracked_verts is None else int(np.asarray(tracked_verts).size // 3)
    if grads is not None and (grads.dtype != np.float32 or grads.size != grad_size(k, m, nv)):
        raise Error(ErrorCategory.USAGE, "gradient buffer must be float32 of ParamLayout::total()")
    n_kd = k * 4 * m ** 3 + 9 * k
    g_dev = None if grads is None else np.ascontiguousarray(grads[:n_kd])
    if nv:  # lossGeo (losses.cpp:27-43)
        loss = C.c_float()
        base = _f32(mesh_vertices).reshape(nv, 3)
        off = None if vertex_offsets is None or np.asarray(vertex_offsets).size == 0 else _f32(vertex_offsets)
        gv = None if grads is None else np.ascontiguousarray(grads[n_kd:])
        _check(lib.vp_loss_geo(nv, _fptr(base), _fptr(off) if off is not None else None,
                               _fptr(_f32(tracked_verts).reshape(nv, 3)), float(weights.geo), C.byref(loss),
                               _fptr(gv) if gv is not None else None))
        terms.geo = float(loss.value)
        if gv is not None:
            grads[n_kd:] = gv
    lv, ld = C.c_float(), C.c_float()
    gpose = None if g_dev is None else np.ascontiguousarray(g_dev[k * 4 * m ** 3:])
    _check(lib.vp_loss_pose(k, _fptr(tr), float(weights.vol), float(weights.del_), C.byref(lv), C.byref(ld),
                            _fptr(gpose) if gpose is not None else None))
    terms.vol, terms.del_ = float(lv.value), float(ld.value)
    if g_dev is not None:
        g_dev[k * 4 * m ** 3:] = gpose
    lp = C.c_float()
    mc = cfg.to_c()
    _check(lib.vp_eval_loss_pho(renderer.ctx, len(cams), cams_c, n, ci.ctypes.data_as(i32p),
                                _fptr(_f32(batch.pixel).reshape(n, 2)), pid.ctypes.data_as(i32p),
                                _fptr(_f32(batch.target).reshape(n, 3)), _fptr(_f32(batch.background).reshape(n, 3)),
                                float(weights.pho), C.byref(mc), _fptr(tr), C.byref(lp),
                                None, _fptr(g_dev) if g_dev is not None else None,
                                1 if g_dev is not None else 0), renderer.ctx)
    terms.pho = float(lp.value)
    if grads is not None:
        grads[:n_kd] = g_dev
    return terms


def adam_step(renderer: "Renderer", cfg: AdamConfig, grads: np.ndarray, transforms: np.ndarray) -> None:
    """adamStep (losses.cpp:70-104) on the renderer's resident frame: the payload is updated
    on the device, `transforms` (K x 24 float32) in place; the frame is recomposed."""
    lib = _lib.load()
    if transforms.dtype != np.float32 or not transforms.flags.c_contiguous:
        raise Error(ErrorCategory.USAGE, "transforms must be a contiguous float32 K x 24 array")
    ac = _lib.vp_adam(cfg.lr, cfg.beta1, cfg.beta2, cfg.eps, cfg.lr_delta_scale, cfg.lr_vertex_scale)
    g = np.ascontiguousarray(grads, np.float32)
    k, m = int(renderer.n_prim or 0), int(renderer.m or 0)
    if g.size < k * 4 * m ** 3 + 9 * k:  # vp_adam_step reads that many floats
        raise Error(ErrorCategory.USAGE, f"grads hold {g.size} floats; the frame needs {k * 4 * m ** 3 + 9 * k}")
    if transforms.size < 24 * k:
        raise Error(ErrorCategory.USAGE, "transforms must hold K x 24 records")
    _check(lib.vp_adam_step(renderer.ctx, C.byref(ac), _fptr(g), _fptr(transforms)), renderer.ctx)


def payload_planar(renderer: "Renderer") -> np.ndarray:
    """The resident payload converted back to the reference's planar (k, c, z, y, x) layout."""
    k, m = int(renderer.n_prim or 0), int(renderer.m or 0)
    inter = np.zeros(k * m ** 3 * 4, np.float32)
    renderer.copy_payload_to(inter.ctypes.data)
    return np.ascontiguousarray(inter.reshape(k, m ** 3, 4).transpose(0, 2, 1)).reshape(-1)


_default: dict = {}


def _renderer(device: int) -> Renderer:
    if device not in _default:
        _default[device] = Renderer(device)
    return _default[device]


def render(scene: Scene, frame: int, cam: Camera, cfg: MarchConfig, device: int = 0) -> RenderOutput:
    """volprim::render (march.h:59): uploads the frame and renders one view on `device`."""
    r = _renderer(device)
    r.set_frame(scene, frame)
    return r.render(cam, cfg)


def composite(out: RenderOutput, background: np.ndarray, device: int = 0) -> np.ndarray:
    """volprim::composite (march.h:62)."""
    return _renderer(device).composite(out, background)


def shard_tiles(width: int, height: int, shard: int, n_shards: int) -> int:
    """Tile slots of shard `shard` of `n_shards` (vp_shard_tiles): the tiles t with
    t % n_shards == shard, t the row-major index of the ceil(W/16) x ceil(H/16) tile grid."""
    from ._lib import load
    return int(load().vp_shard_tiles(int(width), int(height), int(shard), int(n_shards)))

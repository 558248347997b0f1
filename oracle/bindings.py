"""TEST INFRASTRUCTURE — ctypes bindings of the parity checkers. NOT PRODUCT CODE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module, and only as the checker or the timed CPU baseline.

  Oracle   -> oracle/liboracle.so           plain-C restatement (vp_oracle.c)
  RefCore  -> oracle/_ref/libvolprim_ref.so the unmodified reference core + ref_glue.cpp
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libvolprim_ref.so"

f32p = C.POINTER(C.c_float)
i32p = C.POINTER(C.c_int32)
u32p = C.POINTER(C.c_uint32)


def _p(a, t=f32p):
    return None if a is None else a.ctypes.data_as(t)


def _f(a, n=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    return a if n is None else a.reshape(n)


def cam_arrays(cam):
    """(K9, R9, t3) column-major float32 arrays from an api.Camera."""
    return (_f(np.asarray(cam.intrinsics, np.float32).T.reshape(-1)),
            _f(np.asarray(cam.rotation, np.float32).T.reshape(-1)),
            _f(np.asarray(cam.translation, np.float32).reshape(-1)))


def build(ref: bool = True) -> None:
    """make -C oracle (and the reference core when /root/reference is present)."""
    import subprocess
    targets = ["oracle"]
    if ref and pathlib.Path(os.environ.get("VPB_REFERENCE", "/root/reference/proj")).exists():
        targets.append("ref")
    subprocess.run(["make", "-C", str(HERE), *targets], check=True,
                   stdout=subprocess.DEVNULL)


class Oracle:
    """The C restatement (liboracle.so)."""

    def __init__(self, path: pathlib.Path = ORACLE_SO):
        if not path.exists():
            build(ref=False)
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.vpo_compose.argtypes = [C.c_int32, f32p, f32p]
        L.vpo_generate_ray.argtypes = [f32p, f32p, f32p, C.c_float, C.c_float, f32p, f32p]
        L.vpo_intersect.restype = C.c_int32
        L.vpo_intersect.argtypes = [C.c_int32, f32p, f32p, f32p, C.c_int32, i32p, f32p, f32p]
        L.vpo_window.restype = C.c_float
        L.vpo_window.argtypes = [C.c_float] * 4 + [C.c_int32]
        L.vpo_march_rays.argtypes = [C.c_int32, C.c_int32, f32p, f32p, C.c_float, C.c_int32,
                                     C.c_int64, f32p, f32p, f32p, C.c_float, C.c_float,
                                     C.c_uint64, f32p, f32p, i32p]
        L.vpo_render.argtypes = [C.c_int32, C.c_int32, f32p, f32p, C.c_float, C.c_int32, f32p,
                                 f32p, f32p, C.c_int32, C.c_int32, C.c_float, C.c_float,
                                 C.c_int32, C.c_uint64, C.c_uint64, f32p, f32p, i32p, C.c_int32]
        L.vpo_render_counted.argtypes = [C.c_int32, C.c_int32, f32p, f32p, C.c_float, C.c_int32, f32p,
                                         f32p, f32p, C.c_int32, C.c_int32, C.c_float, C.c_float,
                                         C.c_int32, C.c_uint64, C.c_uint64, f32p, f32p, i32p, i32p,
                                         C.c_int32]
        L.vpo_composite.argtypes = [C.c_int32, C.c_int32, f32p, f32p, f32p, f32p]
        L.vpo_cull.argtypes = [C.c_int32, f32p, f32p, f32p, f32p, C.c_int32, C.c_int32, i32p, u32p]
        L.vpo_cull_px.argtypes = [C.c_int32, f32p, f32p, f32p, f32p, C.c_int32, C.c_int32, i32p, i32p,
                                  u32p]
        L.vpo_tile_lists.restype = C.c_int64
        L.vpo_tile_lists.argtypes = [C.c_int32, f32p, f32p, f32p, f32p, C.c_int32, C.c_int32,
                                     i32p, i32p, C.c_int64]
        L.vpo_backward_rays.argtypes = [C.c_int32, C.c_int32, f32p, f32p, f32p, C.c_float, C.c_int32,
                                        C.c_int64, f32p, f32p, f32p, f32p, f32p, C.c_float,
                                        C.c_float, f32p]
        L.vpo_expf_port.restype = C.c_float
        L.vpo_expf_port.argtypes = [C.c_float]
        L.vpo_expf_mismatches.restype = C.c_int64
        L.vpo_expf_mismatches.argtypes = [C.c_uint32, C.c_uint32, f32p]
        L.vpo_expf_port_mismatches.restype = C.c_int64
        L.vpo_expf_port_mismatches.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32]
        L.vpo_sinf_port.restype = C.c_float
        L.vpo_sinf_port.argtypes = [C.c_float]
        L.vpo_cosf_port.restype = C.c_float
        L.vpo_cosf_port.argtypes = [C.c_float]
        L.vpo_sincos_port_mismatches.restype = C.c_int64
        L.vpo_sincos_port_mismatches.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_int]
        L.vpo_sincos_mismatches.restype = C.c_int64
        L.vpo_sincos_mismatches.argtypes = [C.c_uint32, C.c_uint32, f32p, C.c_int]
        L.vpo_sincos_libm.restype = None
        L.vpo_sincos_libm.argtypes = [C.c_int64, f32p, f32p, C.c_int]

    def compose(self, tr24):
        tr = _f(tr24).reshape(-1, 24)
        out = np.zeros((tr.shape[0], 15), np.float32)
        rc = self.lib.vpo_compose(tr.shape[0], _p(tr), _p(out))
        return rc, out

    def render(self, xf15, m, payload, window, cam, cfg, n_threads=None):
        xf = _f(xf15).reshape(-1, 15)
        k9, r9, t3 = cam_arrays(cam)
        w, h = int(cam.width), int(cam.height)
        rgb = np.zeros((h, w, 3), np.float32)
        alpha = np.zeros((h, w, 1), np.float32)
        samples = np.zeros(h * w, np.int32)
        nt = n_threads if n_threads else (os.cpu_count() or 1)
        rc = self.lib.vpo_render(xf.shape[0], int(m), _p(xf), _p(_f(payload)), float(window.alpha),
                                 int(window.beta), _p(k9), _p(r9), _p(t3), w, h,
                                 float(cfg.step_size), float(cfg.early_eps), int(bool(cfg.jitter)),
                                 int(cfg.seed), int(cfg.accumulation_permutation), _p(rgb), _p(alpha),
                                 _p(samples, i32p), int(nt))
        assert rc == 0
        return rgb, alpha, samples

    def render_counted(self, xf15, m, payload, window, cam, cfg, n_threads=None):
        """render() plus the per-pixel prim-sample counts (int32, H*W)."""
        xf = _f(xf15).reshape(-1, 15)
        k9, r9, t3 = cam_arrays(cam)
        w, h = int(cam.width), int(cam.height)
        rgb = np.zeros((h, w, 3), np.float32)
        alpha = np.zeros((h, w, 1), np.float32)
        samples = np.zeros(h * w, np.int32)
        prim = np.zeros(h * w, np.int32)
        nt = n_threads if n_threads else (os.cpu_count() or 1)
        rc = self.lib.vpo_render_counted(xf.shape[0], int(m), _p(xf), _p(_f(payload)), float(window.alpha),
                                         int(window.beta), _p(k9), _p(r9), _p(t3), w, h,
                                         float(cfg.step_size), float(cfg.early_eps), int(bool(cfg.jitter)),
                                         int(cfg.seed), int(cfg.accumulation_permutation), _p(rgb), _p(alpha),
                                         _p(samples, i32p), _p(prim, i32p), int(nt))
        assert rc == 0
        return rgb, alpha, samples, prim

    def march_rays(self, xf15, m, payload, window, origins, dirs, cfg, jitter=None):
        xf = _f(xf15).reshape(-1, 15)
        o = _f(origins).reshape(-1, 3)
        d = _f(dirs).reshape(-1, 3)
        n = o.shape[0]
        j = None if jitter is None else _f(jitter).reshape(n)
        rgb = np.zeros((n, 3), np.float32)
        alpha = np.zeros(n, np.float32)
        samples = np.zeros(n, np.int32)
        self.lib.vpo_march_rays(xf.shape[0], int(m), _p(xf), _p(_f(payload)), float(window.alpha),
                                int(window.beta), n, _p(o), _p(d), _p(j), float(cfg.step_size),
                                float(cfg.early_eps), int(cfg.accumulation_permutation), _p(rgb),
                                _p(alpha), _p(samples, i32p))
        return rgb, alpha, samples

    def backward_rays(self, tr24, m, payload, window, origins, dirs, adj_rgb, adj_alpha, cfg,
                      jitter=None):
        """backwardRay restatement; returns the GradBuffer values (payload planar | 9K)."""
        tr = _f(tr24).reshape(-1, 24)
        k = tr.shape[0]
        rc, xf = self.compose(tr)
        assert rc == 0
        o = _f(origins).reshape(-1, 3)
        d = _f(dirs).reshape(-1, 3)
        n = o.shape[0]
        j = None if jitter is None else _f(jitter).reshape(n)
        g = np.zeros(k * 4 * int(m) ** 3 + 9 * k, np.float32)
        self.lib.vpo_backward_rays(k, int(m), _p(tr), _p(xf), _p(_f(payload)), float(window.alpha),
                                   int(window.beta), n, _p(o), _p(d), _p(j), _p(_f(adj_rgb).reshape(n, 3)),
                                   _p(_f(adj_alpha).reshape(n)), float(cfg.step_size), float(cfg.early_eps),
                                   _p(g))
        return g

    def generate_ray(self, cam, px, py):
        k9, r9, t3 = cam_arrays(cam)
        o = np.zeros(3, np.float32)
        d = np.zeros(3, np.float32)
        self.lib.vpo_generate_ray(_p(k9), _p(r9), _p(t3), float(px), float(py), _p(o), _p(d))
        return o, d

    def intersect(self, xf15, origin, direction):
        xf = _f(xf15).reshape(-1, 15)
        k = xf.shape[0]
        prims = np.zeros(max(k, 1), np.int32)
        te = np.zeros(max(k, 1), np.float32)
        tx = np.zeros(max(k, 1), np.float32)
        n = self.lib.vpo_intersect(k, _p(xf), _p(_f(origin, 3)), _p(_f(direction, 3)), k,
                                   _p(prims, i32p), _p(te), _p(tx))
        return prims[:n], te[:n], tx[:n]

    def cull(self, xf15, cam):
        xf = _f(xf15).reshape(-1, 15)
        k = xf.shape[0]
        k9, r9, t3 = cam_arrays(cam)
        rects = np.zeros((max(k, 1), 4), np.int32)
        keys = np.zeros(max(k, 1), np.uint32)
        self.lib.vpo_cull(k, _p(xf), _p(k9), _p(r9), _p(t3), int(cam.width), int(cam.height),
                          _p(rects, i32p), _p(keys, u32p))
        return rects[:k], keys[:k]

    def cull_px(self, xf15, cam):
        """(tile rects, pixel rects, depth keys)."""
        xf = _f(xf15).reshape(-1, 15)
        k = xf.shape[0]
        k9, r9, t3 = cam_arrays(cam)
        rects = np.zeros((max(k, 1), 4), np.int32)
        prects = np.zeros((max(k, 1), 4), np.int32)
        keys = np.zeros(max(k, 1), np.uint32)
        self.lib.vpo_cull_px(k, _p(xf), _p(k9), _p(r9), _p(t3), int(cam.width), int(cam.height),
                             _p(rects, i32p), _p(prects, i32p), _p(keys, u32p))
        return rects[:k], prects[:k], keys[:k]

    def tile_lists(self, xf15, cam):
        xf = _f(xf15).reshape(-1, 15)
        k9, r9, t3 = cam_arrays(cam)
        tiles = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
        offs = np.zeros(tiles + 1, np.int32)
        total = self.lib.vpo_tile_lists(xf.shape[0], _p(xf), _p(k9), _p(r9), _p(t3),
                                        int(cam.width), int(cam.height), _p(offs, i32p), None, 0)
        prims = np.zeros(max(total, 1), np.int32)
        self.lib.vpo_tile_lists(xf.shape[0], _p(xf), _p(k9), _p(r9), _p(t3), int(cam.width),
                                int(cam.height), _p(offs, i32p), _p(prims, i32p), total)
        return offs, prims[:total]

    def window(self, x, y, z, alpha=8.0, beta=8):
        return self.lib.vpo_window(x, y, z, alpha, beta)

    def expf_port(self, x):
        return self.lib.vpo_expf_port(float(x))

    def expf_mismatches(self, lo_bits: int, hi_bits: int, values: np.ndarray) -> int:
        v = _f(values)
        assert v.size == hi_bits - lo_bits + 1
        return int(self.lib.vpo_expf_mismatches(lo_bits, hi_bits, _p(v)))

    def expf_port_mismatches(self, lo_bits: int, hi_bits: int, stride: int = 1) -> int:
        return int(self.lib.vpo_expf_port_mismatches(lo_bits, hi_bits, stride))

    def sincos_port_mismatches(self, lo_bits: int, hi_bits: int, stride: int = 1, cos: bool = False) -> int:
        """C port of glibc sinf/cosf vs this host's libm over float bit patterns."""
        return int(self.lib.vpo_sincos_port_mismatches(lo_bits, hi_bits, stride, 1 if cos else 0))

    def sincos_libm(self, x: np.ndarray, cos: bool = False) -> np.ndarray:
        """This host's libm sinf/cosf over an array."""
        xs = np.ascontiguousarray(x, np.float32)
        y = np.empty_like(xs)
        self.lib.vpo_sincos_libm(xs.size, _p(xs), _p(y), 1 if cos else 0)
        return y

    def sincos_mismatches(self, lo_bits: int, hi_bits: int, values: np.ndarray, cos: bool = False) -> int:
        """values[i] (for bit pattern lo_bits + i) vs this host's libm sinf/cosf."""
        v = np.ascontiguousarray(values, np.float32)
        assert v.size == hi_bits - lo_bits + 1
        return int(self.lib.vpo_sincos_mismatches(lo_bits, hi_bits, _p(v), 1 if cos else 0))

    def composite(self, rgb, alpha, bg):
        h, w = rgb.shape[:2]
        out = np.zeros((h, w, 3), np.float32)
        self.lib.vpo_composite(w, h, _p(_f(rgb)), _p(_f(alpha)), _p(_f(bg)), _p(out))
        return out


class RefCore:
    """The unmodified reference core (oracle/_ref/libvolprim_ref.so)."""

    @staticmethod
    def available() -> bool:
        return REF_SO.exists()

    def __init__(self, path: pathlib.Path = REF_SO):
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.vpref_last_error.restype = C.c_char_p
        L.vpref_compose.argtypes = [C.c_int32, f32p, f32p]
        L.vpref_render.argtypes = [C.c_int32, C.c_int32, f32p, f32p, C.c_float, C.c_int32, f32p,
                                   f32p, f32p, C.c_int32, C.c_int32, C.c_float, C.c_float,
                                   C.c_int32, C.c_uint64, C.c_uint64, f32p, f32p, i32p]
        L.vpref_look_at.argtypes = [f32p, f32p, f32p, C.c_float, C.c_int32, C.c_int32, f32p,
                                    f32p, f32p, f32p]
        L.vpref_generate_ray.argtypes = [f32p, f32p, f32p, C.c_int32, C.c_int32, C.c_float,
                                         C.c_float, f32p, f32p]
        L.vpref_intersect.argtypes = [C.c_int32, f32p, f32p, f32p, C.c_int32, i32p, i32p, f32p,
                                      f32p, f32p, f32p]
        L.vpref_render_prim_counts.argtypes = [C.c_int32, C.c_int32, f32p, f32p, C.c_float, C.c_int32, f32p,
                                               f32p, f32p, C.c_int32, C.c_int32, C.c_float, C.c_float,
                                               C.c_int32, C.c_uint64, i32p]
        L.vpref_march_rays.argtypes = [C.c_int32, C.c_int32, f32p, f32p, C.c_float, C.c_int32,
                                       C.c_int64, f32p, f32p, f32p, C.c_float, C.c_float,
                                       C.c_uint64, f32p, f32p, i32p]
        L.vpref_backward_rays.argtypes = [C.c_int32, C.c_int32, f32p, f32p, C.c_float, C.c_int32,
                                          C.c_int64, f32p, f32p, f32p, f32p, f32p, C.c_float,
                                          C.c_float, f32p]
        L.vpref_window.restype = C.c_float
        L.vpref_window.argtypes = [C.c_float] * 4 + [C.c_int32]

    def error(self):
        return self.lib.vpref_last_error().decode()

    def compose(self, tr24):
        tr = _f(tr24).reshape(-1, 24)
        out = np.zeros((tr.shape[0], 15), np.float32)
        rc = self.lib.vpref_compose(tr.shape[0], _p(tr), _p(out))
        return rc, out

    def render(self, tr24, m, payload, window, cam, cfg):
        """volprim::render on a one-frame scene built from PrimitiveTransform records."""
        tr = _f(tr24).reshape(-1, 24)
        k9, r9, t3 = cam_arrays(cam)
        w, h = int(cam.width), int(cam.height)
        rgb = np.zeros((h, w, 3), np.float32)
        alpha = np.zeros((h, w, 1), np.float32)
        samples = np.zeros(h * w, np.int32)
        rc = self.lib.vpref_render(tr.shape[0], int(m), _p(tr), _p(_f(payload)), float(window.alpha),
                                   int(window.beta), _p(k9), _p(r9), _p(t3), w, h,
                                   float(cfg.step_size), float(cfg.early_eps), int(bool(cfg.jitter)),
                                   int(cfg.seed), int(cfg.accumulation_permutation), _p(rgb),
                                   _p(alpha), _p(samples, i32p))
        if rc != 0:
            raise RuntimeError(f"reference render failed ({rc}): {self.error()}")
        return rgb, alpha, samples

    def look_at(self, pos, target, up, focal, w, h):
        k9 = np.zeros(9, np.float32)
        r9 = np.zeros(9, np.float32)
        t3 = np.zeros(3, np.float32)
        aa = np.zeros(3, np.float32)
        self.lib.vpref_look_at(_p(_f(pos, 3)), _p(_f(target, 3)), _p(_f(up, 3)), float(focal),
                               int(w), int(h), _p(k9), _p(r9), _p(t3), _p(aa))
        return k9, r9, t3, aa

    def generate_ray(self, cam, px, py):
        k9, r9, t3 = cam_arrays(cam)
        o = np.zeros(3, np.float32)
        d = np.zeros(3, np.float32)
        self.lib.vpref_generate_ray(_p(k9), _p(r9), _p(t3), int(cam.width), int(cam.height),
                                    float(px), float(py), _p(o), _p(d))
        return o, d

    def intersect(self, xf15, origin, direction):
        xf = _f(xf15).reshape(-1, 15)
        k = xf.shape[0]
        n = C.c_int32()
        prims = np.zeros(max(k, 1), np.int32)
        te = np.zeros(max(k, 1), np.float32)
        tx = np.zeros(max(k, 1), np.float32)
        tmin = C.c_float()
        tmax = C.c_float()
        self.lib.vpref_intersect(k, _p(xf), _p(_f(origin, 3)), _p(_f(direction, 3)), k, C.byref(n),
                                 _p(prims, i32p), _p(te), _p(tx), C.byref(tmin), C.byref(tmax))
        return prims[:n.value], te[:n.value], tx[:n.value]

    def render_prim_counts(self, tr24, m, payload, window, cam, cfg):
        """Per-pixel prim-sample counts of the reference's render() (vpref_render_prim_counts)."""
        tr = _f(tr24).reshape(-1, 24)
        k9, r9, t3 = cam_arrays(cam)
        w, h = int(cam.width), int(cam.height)
        prim = np.zeros(h * w, np.int32)
        rc = self.lib.vpref_render_prim_counts(tr.shape[0], int(m), _p(tr), _p(_f(payload)), float(window.alpha),
                                               int(window.beta), _p(k9), _p(r9), _p(t3), w, h,
                                               float(cfg.step_size), float(cfg.early_eps), int(bool(cfg.jitter)),
                                               int(cfg.seed), _p(prim, i32p))
        if rc != 0:
            raise RuntimeError(self.error())
        return prim

    def march_rays(self, xf15, m, payload, window, origins, dirs, cfg, jitter=None):
        xf = _f(xf15).reshape(-1, 15)
        o = _f(origins).reshape(-1, 3)
        d = _f(dirs).reshape(-1, 3)
        n = o.shape[0]
        j = None if jitter is None else _f(jitter).reshape(n)
        rgb = np.zeros((n, 3), np.float32)
        alpha = np.zeros(n, np.float32)
        samples = np.zeros(n, np.int32)
        rc = self.lib.vpref_march_rays(xf.shape[0], int(m), _p(xf), _p(_f(payload)),
                                       float(window.alpha), int(window.beta), n, _p(o), _p(d),
                                       _p(j), float(cfg.step_size), float(cfg.early_eps),
                                       int(cfg.accumulation_permutation), _p(rgb), _p(alpha),
                                       _p(samples, i32p))
        if rc != 0:
            raise RuntimeError(f"reference march failed ({rc}): {self.error()}")
        return rgb, alpha, samples

    def window(self, x, y, z, alpha=8.0, beta=8):
        return self.lib.vpref_window(x, y, z, alpha, beta)

    def backward_rays(self, tr24, m, payload, window, origins, dirs, adj_rgb, adj_alpha, cfg,
                      jitter=None):
        tr = _f(tr24).reshape(-1, 24)
        k = tr.shape[0]
        o = _f(origins).reshape(-1, 3)
        d = _f(dirs).reshape(-1, 3)
        n = o.shape[0]
        j = None if jitter is None else _f(jitter).reshape(n)
        g = np.zeros(k * 4 * int(m) ** 3 + 9 * k, np.float32)
        rc = self.lib.vpref_backward_rays(k, int(m), _p(tr), _p(_f(payload)), float(window.alpha),
                                          int(window.beta), n, _p(o), _p(d), _p(j),
                                          _p(_f(adj_rgb).reshape(n, 3)), _p(_f(adj_alpha).reshape(n)),
                                          float(cfg.step_size), float(cfg.early_eps), _p(g))
        if rc != 0:
            raise RuntimeError(f"reference backward failed ({rc}): {self.error()}")
        return g


def _cams23(cams):
    out = np.zeros((len(cams), 23), np.float32)
    for i, c in enumerate(cams):
        k9, r9, t3 = cam_arrays(c)
        out[i, :9], out[i, 9:18], out[i, 18:21] = k9, r9, t3
        out[i, 21], out[i, 22] = c.width, c.height
    return out


def ref_eval_loss(ref, tr24, m, payload, window, cams, cam_index, pixel_xy, pixel_id, target,
                  background, weights, cfg, with_grads=True):
    """The reference evalLoss (no tracked vertices); returns (terms[4], grads or None)."""
    L = ref.lib
    L.vpref_eval_loss.argtypes = [C.c_int32, C.c_int32, f32p, f32p, C.c_float, C.c_int32, C.c_int32,
                                  f32p, C.c_int64, i32p, f32p, i32p, f32p, f32p, C.c_float, C.c_float,
                                  C.c_float, C.c_float, C.c_float, C.c_int32, C.c_uint64, f32p, f32p]
    tr = _f(tr24).reshape(-1, 24)
    k = tr.shape[0]
    n = len(cam_index)
    terms = np.zeros(4, np.float32)
    g = np.zeros(k * 4 * int(m) ** 3 + 9 * k, np.float32) if with_grads else None
    rc = L.vpref_eval_loss(k, int(m), _p(tr), _p(_f(payload)), float(window.alpha), int(window.beta),
                           len(cams), _p(_cams23(cams)), n, _p(np.ascontiguousarray(cam_index, np.int32), i32p),
                           _p(_f(pixel_xy).reshape(n, 2)), _p(np.ascontiguousarray(pixel_id, np.int32), i32p),
                           _p(_f(target).reshape(n, 3)), _p(_f(background).reshape(n, 3)), float(weights[0]),
                           float(weights[1]), float(weights[2]), float(cfg.step_size), float(cfg.early_eps),
                           int(bool(cfg.jitter)), int(cfg.seed), _p(terms), _p(g))
    if rc != 0:
        raise RuntimeError(f"reference evalLoss failed ({rc}): {ref.error()}")
    return terms, g


def ref_load_slab(ref, path):
    """The reference loadSlab; returns (K, M, planar payload)."""
    L = ref.lib
    L.vpref_load_slab.argtypes = [C.c_char_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), f32p, C.c_int64]
    k, m = C.c_int32(), C.c_int32()
    if L.vpref_load_slab(str(path).encode(), C.byref(k), C.byref(m), None, 0) != 0:
        raise RuntimeError(f"reference loadSlab failed: {ref.error()}")
    pay = np.zeros(k.value * 4 * m.value ** 3, np.float32)
    if L.vpref_load_slab(str(path).encode(), C.byref(k), C.byref(m), _p(pay), pay.size) != 0:
        raise RuntimeError(f"reference loadSlab failed: {ref.error()}")
    return k.value, m.value, pay


def ref_adam_run(ref, tr24, m, payload_planar, grads_seq, cfg6):
    L = ref.lib
    L.vpref_adam_run.argtypes = [C.c_int32, C.c_int32, f32p, f32p, C.c_int32, f32p, f32p]
    tr = np.array(tr24, np.float32).reshape(-1, 24).copy()
    pay = np.array(payload_planar, np.float32).copy()
    gs = _f(grads_seq)
    rc = L.vpref_adam_run(tr.shape[0], int(m), _p(tr), _p(pay), len(grads_seq), _p(gs), _p(_f(cfg6)))
    if rc != 0:
        raise RuntimeError(f"reference adamStep failed ({rc}): {ref.error()}")
    return tr, pay


# Default MarchConfig / WindowParams of the §8d workload (march.h:11-20, primitive.h:14-17);
# restated here so the reference arm of bench.py needs nothing from the product package.
REF_STEP, REF_EPS, REF_WALPHA, REF_WBETA = 0.001, 0.01, 8.0, 8


def ref_shell_arrays(ref: RefCore, k: int, m: int):
    """The §8d "mvp_shell" inputs built by the reference-side generator (vpref_shell_scene):
    (K x 24 PrimitiveTransform records, planar K*4*M^3 payload)."""
    L = ref.lib
    L.vpref_shell_scene.argtypes = [C.c_int32, C.c_int32, f32p, f32p]
    tr = np.zeros((k, 24), np.float32)
    pay = np.zeros(k * 4 * m ** 3, np.float32)
    if L.vpref_shell_scene(int(k), int(m), _p(tr), _p(pay)) != 0:
        raise RuntimeError(f"reference shell scene failed: {ref.error()}")
    return tr, pay


def ref_shell_camera(ref: RefCore, view: int, n_views: int, width: int):
    """(K9, R9, t3) column-major of the §8d camera: view < 0 headline, else ring view."""
    L = ref.lib
    L.vpref_shell_camera.argtypes = [C.c_int32, C.c_int32, C.c_int32, f32p, f32p, f32p]
    k9, r9, t3 = np.zeros(9, np.float32), np.zeros(9, np.float32), np.zeros(3, np.float32)
    if L.vpref_shell_camera(int(view), int(n_views), int(width), _p(k9), _p(r9), _p(t3)) != 0:
        raise RuntimeError(f"reference shell camera failed: {ref.error()}")
    return k9, r9, t3


class RefScene:
    """A resident reference Scene (vpref_scene_*): built once, then every render() call runs
    volprim::render (march.cpp:95-132) on it. Outputs are copied only when asked for."""

    def __init__(self, ref: RefCore, k: int, m: int, tr24=None, payload=None,
                 w_alpha: float = REF_WALPHA, w_beta: int = REF_WBETA):
        L = ref.lib
        L.vpref_scene_new.restype = C.c_void_p
        L.vpref_scene_new.argtypes = [C.c_int32, C.c_int32, f32p, f32p, C.c_float, C.c_int32]
        L.vpref_scene_new_shell.restype = C.c_void_p
        L.vpref_scene_new_shell.argtypes = [C.c_int32, C.c_int32, C.c_float, C.c_int32]
        L.vpref_scene_free.argtypes = [C.c_void_p]
        L.vpref_scene_render.argtypes = [C.c_void_p, f32p, f32p, f32p, C.c_int32, C.c_int32, C.c_float,
                                         C.c_float, C.c_int32, C.c_uint64, f32p, f32p, i32p,
                                         C.POINTER(C.c_int64)]
        self.ref, self.lib = ref, L
        if tr24 is None:  # the §8d shell scene, generated in place
            self.h = L.vpref_scene_new_shell(int(k), int(m), float(w_alpha), int(w_beta))
        else:
            tr = _f(tr24).reshape(-1, 24)
            self.h = L.vpref_scene_new(tr.shape[0], int(m), _p(tr), _p(_f(payload)), float(w_alpha), int(w_beta))
        if not self.h:
            raise RuntimeError(f"reference scene failed: {ref.error()}")

    def render(self, k9, r9, t3, width, height, step=REF_STEP, eps=REF_EPS, jitter=False, seed=0,
               outputs: bool = False):
        """Returns total ray-samples, or (total, rgb, alpha, samples) when outputs=True."""
        tot = C.c_int64()
        rgb = alpha = samples = None
        if outputs:
            rgb = np.zeros((height, width, 3), np.float32)
            alpha = np.zeros((height, width, 1), np.float32)
            samples = np.zeros(height * width, np.int32)
        rc = self.lib.vpref_scene_render(self.h, _p(_f(k9)), _p(_f(r9)), _p(_f(t3)), int(width), int(height),
                                         float(step), float(eps), int(bool(jitter)), int(seed), _p(rgb),
                                         _p(alpha), _p(samples, i32p), C.byref(tot))
        if rc != 0:
            raise RuntimeError(f"reference render failed ({rc}): {self.ref.error()}")
        return (tot.value, rgb, alpha, samples) if outputs else tot.value

    def close(self):
        if self.h:
            self.lib.vpref_scene_free(self.h)
            self.h = None

    def __del__(self):
        self.close()

"""ctypes binding of libvpb.so (the C-ABI declared in include/vpb.h).

The library is built in-tree (``make lib`` / ``__graft_entry__.build()``). There is no
fallback of any kind: if the shared object is missing, importing the renderer raises.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

_HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = pathlib.Path(os.environ.get("VPB_LIB", _HERE / "libvpb.so"))

f32p = C.POINTER(C.c_float)
i32p = C.POINTER(C.c_int32)
u32p = C.POINTER(C.c_uint32)
i64p = C.POINTER(C.c_int64)


class vp_camera(C.Structure):
    _fields_ = [("K", C.c_float * 9), ("R", C.c_float * 9), ("t", C.c_float * 3),
                ("width", C.c_int32), ("height", C.c_int32)]


class vp_march(C.Structure):
    _fields_ = [("step_size", C.c_float), ("early_eps", C.c_float), ("jitter", C.c_int32),
                ("reserved", C.c_int32), ("seed", C.c_uint64),
                ("accumulation_permutation", C.c_uint64)]


class vp_adam(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("lr_delta_scale", C.c_float), ("lr_vertex_scale", C.c_float)]


class vp_stats(C.Structure):
    _fields_ = [("ray_samples", C.c_int64), ("prim_samples", C.c_int64),
                ("hit_rays", C.c_int64), ("early_exits", C.c_int64),
                ("saturated", C.c_int64), ("overflow_rays", C.c_int64),
                ("keys", C.c_int64), ("refills", C.c_int64), ("ms", C.c_float),
                ("huge_rays", C.c_int32)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


# name -> (restype, argtypes): every entry point of include/vpb.h
SIGNATURES = {
    "vp_version": (C.c_int, []),
    "vp_create": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    "vp_destroy": (C.c_int, [C.c_void_p]),
    "vp_last_error": (C.c_char_p, [C.c_void_p]),
    "vp_stream": (C.c_void_p, [C.c_void_p]),
    "vp_compose": (C.c_int, [C.c_int32, f32p, f32p]),
    "vp_set_scene": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, f32p, f32p, C.c_float, C.c_int32]),
    "vp_set_transforms": (C.c_int, [C.c_void_p, C.c_int32, f32p]),
    "vp_set_transforms_async": (C.c_int, [C.c_void_p, C.c_int32, f32p, C.c_void_p]),
    "vp_set_frame": (C.c_int, [C.c_void_p, C.c_int32, f32p]),
    "vp_get_transforms": (C.c_int, [C.c_void_p, f32p]),
    "vp_set_payload_interleaved": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, f32p]),
    "vp_load_slab": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int32, f32p, C.c_float, C.c_int32]),
    "vp_payload_device": (C.c_int, [C.c_void_p, C.POINTER(f32p), i64p]),
    "vp_copy_payload": (C.c_int, [C.c_void_p, f32p]),
    "vp_kernel_times": (C.c_int, [C.c_void_p, C.c_int64, f32p, i64p]),
    "vp_render": (C.c_int, [C.c_void_p, C.POINTER(vp_camera), C.POINTER(vp_march), f32p, f32p,
                            i32p, C.POINTER(vp_stats)]),
    "vp_render_async": (C.c_int, [C.c_void_p, C.POINTER(vp_camera), C.POINTER(vp_march), f32p,
                                  f32p, i32p, C.c_void_p]),
    "vp_render_batch_async": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(vp_camera), C.POINTER(vp_march),
                                        C.POINTER(f32p), C.POINTER(f32p), C.POINTER(i32p), C.c_void_p]),
    "vp_render_shard_async": (C.c_int, [C.c_void_p, C.POINTER(vp_camera), C.POINTER(vp_march), C.c_int32,
                                        C.c_int32, f32p, f32p, i32p, C.c_void_p]),
    "vp_shard_tiles": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "vp_sync": (C.c_int, [C.c_void_p]),
    "vp_set_key_capacity": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32]),
    "vp_read_stats": (C.c_int, [C.c_void_p, C.POINTER(vp_stats)]),
    "vp_march_rays": (C.c_int, [C.c_void_p, C.c_int64, f32p, f32p, f32p, C.POINTER(vp_march),
                                f32p, f32p, i32p]),
    "vp_backward_rays": (C.c_int, [C.c_void_p, C.c_int64, f32p, f32p, f32p, f32p, f32p,
                                   C.POINTER(vp_march), f32p, f32p, C.c_int32]),
    "vp_eval_loss_pho": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(vp_camera), C.c_int64, i32p, f32p,
                                   i32p, f32p, f32p, C.c_float, C.POINTER(vp_march), f32p, f32p, f32p,
                                   f32p, C.c_int32]),
    "vp_loss_pose": (C.c_int, [C.c_int32, f32p, C.c_float, C.c_float, f32p, f32p, f32p]),
    "vp_loss_geo": (C.c_int, [C.c_int32, f32p, f32p, f32p, C.c_float, f32p, f32p]),
    "vp_adam_step": (C.c_int, [C.c_void_p, C.POINTER(vp_adam), f32p, f32p]),
    "vp_adam_reset": (C.c_int, [C.c_void_p]),
    "vp_composite": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, f32p, f32p, f32p, f32p]),
    "vp_debug_tiles": (C.c_int, [C.c_void_p, C.POINTER(vp_camera), i32p, u32p, i32p, i32p,
                                 C.c_int64, i64p]),
    "vp_debug_tile_times": (C.c_int, [C.c_void_p, C.POINTER(vp_camera), C.POINTER(vp_march),
                                      C.POINTER(C.c_uint64), C.c_int64, i64p]),
    "vp_debug_expf": (C.c_int, [C.c_void_p, C.c_int64, f32p, f32p]),
    "vp_debug_radix_sort": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "vp_debug_sincos": (C.c_int, [C.c_void_p, C.c_int64, f32p, f32p, C.c_int32]),
    "vp_debug_pose": (C.c_int, [C.c_void_p, C.c_int32, f32p, f32p, C.c_int32]),
    "vp_comm_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "vp_comm_init": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8), C.c_int32, C.c_int32, C.c_int32,
                               C.POINTER(C.c_void_p)]),
    "vp_comm_init_all": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p), i32p, C.c_int32, C.POINTER(C.c_void_p)]),
    "vp_comm_destroy": (C.c_int, [C.c_void_p]),
    "vp_group_start": (C.c_int, []),
    "vp_group_end": (C.c_int, []),
    "vp_broadcast_scene": (C.c_int, [C.c_void_p, C.c_int32]),
    "vp_gather_views": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.POINTER(f32p), C.POINTER(f32p),
                                  C.POINTER(i32p), C.POINTER(f32p), C.POINTER(f32p), C.POINTER(i32p)]),
    "vp_comm_wait": (C.c_int, [C.c_void_p, C.c_void_p]),
    "vp_comm_sync": (C.c_int, [C.c_void_p]),
    "vp_comm_last_error": (C.c_char_p, []),
    "vp_make_shell_scene": (C.c_int, [C.c_int32, C.c_int32, f32p, f32p]),
    "vp_look_at_camera": (C.c_int, [f32p, f32p, f32p, C.c_float, C.c_int32, C.c_int32,
                                    C.POINTER(vp_camera), f32p]),
    "vp_shell_camera": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(vp_camera)]),
}

_lib = None


def load() -> C.CDLL:
    """Load libvpb.so once; raises OSError (loudly) when the library is missing."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise OSError(f"libvpb.so not built at {LIB_PATH}; run `make lib` or "
                          "__graft_entry__.build() — there is no CPU fallback")
        # torch (when installed) first: libvpb binds libnccl.so.2 lazily for vp_comm_*, and it
        # must find torch's (newer) copy already loaded rather than bring in the system one,
        # which would then shadow torch's and break a later `import torch`
        try:
            import torch  # noqa: F401
        except ImportError:
            pass
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib

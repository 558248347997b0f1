"""TEST INFRASTRUCTURE — independent gradient evidence from the REAL reference in f64.

The reference's own gradcheck (grad.cpp:293-370: Richardson-extrapolated central differences of
evalLoss, coordinates sampled round-robin over the parameter groups) runs on the unmodified
reference core built in double precision (oracle/_ref/libvolprim_ref_f64.so, the configuration
of acceptance_f64.cpp) over a scene in the style of acceptance_f64.cpp:20-86: eight textured
primitives in a 4x2 sheet, M = 8, opacity x12 so part of the batch saturates, three cameras,
384 rays, earlyEps = 1e-9. Every input is float32 (exact in f64), so the f32 device sees the
very same scene. Writes tests/golden/gradcheck.npz; tests/test_gpu_gradcheck.py compares the
device's f32 analytic gradient (vp_eval_loss_pho + vp_loss_pose) with these differences.

    python oracle/gen_gradcheck.py
"""
from __future__ import annotations

import ctypes as C
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle.bindings import RefCore, _cams23, ref_eval_loss  # noqa: E402

SO64 = ROOT / "oracle" / "_ref" / "libvolprim_ref_f64.so"
f32p, i32p, i64p = C.POINTER(C.c_float), C.POINTER(C.c_int32), C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)


class Cam:  # the fields bindings.cam_arrays / _cams23 read
    def __init__(self, k9, r9, t3, w, h):
        self.intrinsics = np.asarray(k9, np.float32).reshape(3, 3).T
        self.rotation = np.asarray(r9, np.float32).reshape(3, 3).T
        self.translation = np.asarray(t3, np.float32)
        self.width, self.height = w, h


def scene():
    rng = np.random.default_rng(33)
    k, m = 8, 8
    tr = np.zeros((k, 24), np.float32)
    for j in range(2):
        for i in range(4):
            q = tr[j * 4 + i]
            q[0:3] = (-0.375 + 0.25 * i, -0.25 + 0.5 * j, 0.0)
            q[3:12] = np.eye(3, dtype=np.float32).reshape(-1)
            q[12:15] = (0.125, 0.25, 0.25)
            u = rng.uniform(-1, 1, 9)
            q[21:24] = (u[0] * 0.02, u[1] * 0.02, -0.25 * (0.5 + 0.1 * u[2]))  # deltaS
            q[18:21] = u[3:6] * 0.15                                           # deltaR
            q[15:18] = u[6:9] * 0.01                                           # deltaT
    i = np.arange(k * 4 * m ** 3, dtype=np.uint64)
    pay = (0.2 + 0.6 * ((i * np.uint64(2654435761)) % np.uint64(101)).astype(np.float64) / 101.0)
    pay = pay.astype(np.float32).reshape(k, 4, m, m, m)
    pay[:, 3] *= np.float32(12)
    return tr, m, pay.reshape(-1)


def main():
    ref = RefCore()
    tr, m, pay = scene()
    cams = []
    for c in range(3):
        az = 2.1 * c + 0.4
        k9, r9, t3, _ = ref.look_at((0.6 * np.cos(az), 0.6 * np.sin(az), 1.3), (0, 0, 0), (0, 0, 1), 80.0, 64, 64)
        cams.append(Cam(k9, r9, t3, 64, 64))
    prng = np.random.default_rng(17)
    n = 3 * 128  # acceptance_f64 uses 3 x 16; more rays make more sampled voxels informative
    ci = np.repeat(np.arange(3), n // 3).astype(np.int32)
    pid = prng.integers(0, 64 * 64, n).astype(np.int32)
    pxy = np.stack([(pid % 64) + 0.5, (pid // 64) + 0.5], 1).astype(np.float32)
    tgt = np.tile(np.array([0.3, 0.5, 0.2], np.float32), (n, 1))
    bg = np.tile(np.array([0.1, 0.1, 0.3], np.float32), (n, 1))
    weights = np.array([1.0, 0.0, 0.01, 0.01], np.float32)  # pho, geo (no mesh), vol, del
    step, eps = 0.002, 1e-9

    L = C.CDLL(str(SO64))
    L.vpref64_sizeof_real.restype = C.c_int
    assert L.vpref64_sizeof_real() == 8
    L.vpref64_last_error.restype = C.c_char_p
    L.vpref64_gradcheck.argtypes = [C.c_int32, C.c_int32, f32p, f32p, C.c_float, C.c_int32, C.c_int32, f32p,
                                    C.c_int64, i32p, i32p, f32p, f32p, f32p, C.c_float, C.c_float, C.c_int32,
                                    C.c_uint64, C.c_int64, i64p, i64p, i32p, f64p, f64p]
    cap = 256
    n_out = C.c_int64()
    idx = np.zeros(cap, np.int64)
    grp = np.zeros(cap, np.int32)
    ana = np.zeros(cap, np.float64)
    fd = np.zeros(cap, np.float64)
    P = lambda a, t=f32p: a.ctypes.data_as(t)  # noqa: E731
    c23 = _cams23(cams)
    rc = L.vpref64_gradcheck(8, m, P(tr), P(pay), 8.0, 8, 3, P(c23), n, P(ci, i32p), P(pid, i32p), P(tgt), P(bg),
                             P(weights), step, eps, 216, 97, cap, C.byref(n_out), P(idx, i64p), P(grp, i32p),
                             P(ana, f64p), P(fd, f64p))
    assert rc == 0, L.vpref64_last_error()
    n_e = n_out.value
    idx, grp, ana, fd = idx[:n_e], grp[:n_e], ana[:n_e], fd[:n_e]
    # calibration: the reference's own f32 analytic gradient against the f64 differences
    class MC:
        step_size, early_eps, jitter, seed = step, eps, False, 0

    class W:
        alpha, beta = 8.0, 8
    terms, g32 = ref_eval_loss(ref, tr, m, pay, W, cams, ci, pxy, pid, tgt, bg,
                               [weights[0], weights[2], weights[3]], MC)
    rel32 = np.abs(g32[idx] - fd) / np.maximum(np.abs(g32[idx]) + np.abs(fd), 1e-4)
    rel64 = np.abs(ana - fd) / np.maximum(np.abs(ana) + np.abs(fd), 1e-4)
    for gname, g in zip(["rgb", "sigma", "dT", "dR", "dS"], range(5)):
        sel = grp == g
        print(f"{gname:6s} n={sel.sum():3d} f64 analytic max rel {rel64[sel].max():.2e}   "
              f"reference f32 analytic max rel {rel32[sel].max():.2e}")
    np.savez_compressed(ROOT / "tests" / "golden" / "gradcheck.npz", tr=tr, m=np.int32(m), payload=pay,
                        cams=c23, cam_index=ci, pixel_id=pid, pixel=pxy, target=tgt, background=bg,
                        weights=weights, cfg=np.array([step, eps], np.float32), index=idx, group=grp,
                        analytic64=ana, finite_diff=fd, ref_f32_analytic=g32[idx], terms_f32=terms)
    print("wrote tests/golden/gradcheck.npz,", n_e, "entries")


if __name__ == "__main__":
    main()

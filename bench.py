#!/usr/bin/env python
"""Benchmark of the B200 raymarcher (BASELINE.json: Msamples/s and frames/s at 1024^2, HBM
GB/s against the B200 peak).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

Workload (one "step"): each GPU renders `--views-per-gpu` views (default 8) of the 64-view
ring around the headline scene, mvp_shell K=4096 primitives x 16^3 voxels (BASELINE config 3)
at 1024x1024: rank r renders views [8r, 8r+8) mod 64, so at 8 GPUs one step is the whole
config-5 batch (view sharding, fixed work per GPU -> "weak" scaling). With N > 1 every view's
outputs (rgb, alpha, sample count: 20 B/pixel) are gathered to rank 0 with NCCL, overlapped
with rendering the next step (two output slots).

Printed JSON line (rank 0): value = ray-samples of all ranks / max-over-ranks device time of
the K timed steps; roofline = the raymarch kernel's algorithmic bytes (128 B per
primitive-sample + 20 B per pixel) per launch / its CUDA-event duration vs the
measured HBM peak; e2e = the same metric through the public C-ABI with pinned host buffers
(per step: H2D of the frame's transforms, D2H of every view's outputs); cpu_baseline = the
unmodified reference renderer (oracle/_ref) on this host's cores, bounded sample.
`--impl reference` times that reference renderer alone (rank 0; other ranks exit).
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_RING = 64
BYTES_PER_PRIM_SAMPLE = 128   # 8 trilinear corners x float4 (primitive.cpp:78-90 x 4 channels)
BYTES_PER_PIXEL = 20          # rgb 12 + alpha 4 + sample count 4
METRIC = "Msamples/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=60)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--k", type=int, default=4096)
    p.add_argument("--m", type=int, default=16)
    p.add_argument("--width", type=int, default=1024)
    p.add_argument("--views-per-gpu", type=int, default=8)
    p.add_argument("--no-gather", action="store_true")
    p.add_argument("--torch-comm", action="store_true",
                   help="N > 1: gather / broadcast with torch.distributed NCCL instead of libvpb's vp_comm_*")
    p.add_argument("--nccl-max-ctas", type=int, default=8, help="libvpb NCCL communicator's CTA cap")
    p.add_argument("--comm-at-1", action="store_true",
                   help="N = 1: run the N > 1 data plane anyway (a 1-rank communicator; testing)")
    p.add_argument("--per-view", action="store_true",
                   help="one raymarch launch per view instead of one per step (vp_render_batch_async)")
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="cpu_baseline sample budget")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-one-core", type=int, default=1, help="also time one view pinned to one core")
    p.add_argument("--ref-budget", type=float, default=200.0,
                   help="--impl reference: cap on the timed steps' seconds (steps actually run are reported)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-sweep", action="store_true", help="skip configs 1, 2, 4 (the 'sweep' key)")
    p.add_argument("--sweep-steps", type=int, default=10)
    p.add_argument("--quick", action="store_true", help="profiling mode: no baseline / e2e")
    p.add_argument("--tile-shard", action="store_true",
                   help="single-view mode: each step renders ONE view (the headline camera), rank r "
                        "marching the tiles t %% N == r (vp_render_shard_async), gathered to rank 0")
    return p.parse_args()


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        time.sleep(0.05)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        loaded = [s for s in sm if s > 600] or sm
        reasons = sorted({n for r in self.rows for n, v in zip(self.NAMES, r[2:]) if v == "Active"})
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


def _sha(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class CpuReference:
    """The unmodified reference volprim::render (oracle/_ref/libvolprim_ref.so) on this host's
    cores (std::thread x hardware_concurrency, threads.h:16-36), on a resident reference Scene
    built once by the reference-side generator (vpref_scene_new_shell): each render() call times
    volprim::render (march.cpp:95-132) alone. Nothing from the product package (libvpb.so) is
    loaded."""

    def __init__(self, k, m, width):
        from oracle import bindings as B
        self.k, self.m, self.width = k, m, width
        self.cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
        if B.RefCore.available():
            self.kind = "reference"
            self.core = B.RefCore()
            self.scene = B.RefScene(self.core, k, m)
            self.cam = lambda v: B.ref_shell_camera(self.core, v, N_RING, width)
        else:  # the reference core is built in this container and travels with the snapshot
            raise RuntimeError("oracle/_ref/libvolprim_ref.so missing: build it with make -C oracle ref")

    def render(self, view):
        k9, r9, t3 = self.cam(view)
        return int(self.scene.render(k9, r9, t3, self.width, self.width))

    def sample(self, views, budget_s):
        """(ray-samples, seconds, n_views) for views rendered until budget_s is spent."""
        total, t0, n = 0, time.perf_counter(), 0
        for v in views:
            total += self.render(v)
            n += 1
            if time.perf_counter() - t0 > budget_s:
                break
        return total, time.perf_counter() - t0, n

    def sample_one_core(self, view):
        """One view with the process pinned to one core (the survey's `taskset -c 0` run): the
        reference's worker threads inherit the calling thread's affinity."""
        if not hasattr(os, "sched_setaffinity"):
            return None
        old = os.sched_getaffinity(0)
        core = min(old)
        os.sched_setaffinity(0, {core})
        try:
            t0 = time.perf_counter()
            s = self.render(view)
            return s, time.perf_counter() - t0, core
        finally:
            os.sched_setaffinity(0, old)


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU renderer on rank 0 (other ranks exit). A step
    renders the same number of views as one GPU of our arm (--views-per-gpu, default 8) at the
    same K, M and image size; at N = 1 those are the very views our arm renders (0..7 of the
    ring), at N > 1 the steps walk through the views of all N ranks in turn (a bounded sample of
    the whole job). The run is capped at --ref-budget seconds of timed steps."""
    if rank != 0:
        return
    ref = CpuReference(args.k, args.m, args.width)
    V = args.views_per_gpu
    all_views = [v % N_RING for v in range(V * max(world, 1))]
    ring = [all_views[i % len(all_views)] for i in range(V * (args.warmup + args.steps))]
    steps = [ring[i * V:(i + 1) * V] for i in range(args.warmup + args.steps)]
    for vs in steps[:args.warmup]:
        for v in vs:
            ref.render(v)
    step_s, step_samples = [], []
    t_start = time.perf_counter()
    for vs in steps[args.warmup:]:
        t0 = time.perf_counter()
        n = sum(ref.render(v) for v in vs)
        step_s.append(time.perf_counter() - t0)
        step_samples.append(n)
        if time.perf_counter() - t_start > args.ref_budget:
            break
    t = sum(step_s)
    done = len(step_s)
    value = sum(step_samples) / t / 1e6
    views_timed = sorted({v for vs in steps[args.warmup:args.warmup + done] for v in vs})
    sample = (f"{done} steps x {V} views ({'views ' + str(views_timed[0]) + '..' + str(views_timed[-1])}"
              f" of the 64-view ring), full {args.width}x{args.width} frames, resident reference Scene, "
              f"volprim::render with std::thread x hardware_concurrency on {cpu_model()}")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": METRIC,
            "n_gpus": world, "steps": done, "warmup": args.warmup,
            "ms_per_step": round(1e3 * t / done, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args, world, world > 1) | {"l2": "n/a: host CPU run"},
            "frames_per_s": round(done * V / t, 4),
            "cpu_baseline": {"value": round(value, 3), "unit": METRIC, "cores": ref.cores, "kind": ref.kind,
                             "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": round(value, 3), "unit": METRIC, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if done < args.steps:
        line["steps_requested"] = args.steps
    print(json.dumps(line), flush=True)


SWEEP_CONFIGS = {"oracle_64x16_256": (1, 64, 16, 256), "k512_m32_1024": (2, 512, 32, 1024),
                 "k32768_m8_1024": (4, 32768, 8, 1024)}


def run_sweep(r, args, device, flush, hbm):
    """BASELINE.json's "K x voxel^3 sweep": configs 1, 2 and 4 measured in the same run as the
    headline (config 3), on the same box. Per config: ring views 0..7 in ONE raymarch launch
    (vp_render_batch_async into device buffers), bit-checked against the reference digests of
    those views (tests/golden/digests.json "ring_configs", oracle/gen_ring_digests.py), then
    `sweep_steps` timed launches after 3 warm-ups, L2 flushed before each (CUDA events on the
    launching stream for the step; the library's own events for the raymarch kernel)."""
    import hashlib
    import torch
    import ctypes as C
    from paper_2103_01954_b200 import api, synthetic
    from paper_2103_01954_b200._lib import f32p, i32p, vp_camera

    def sha(a):
        return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()

    golden = json.loads((ROOT / "tests" / "golden" / "digests.json").read_text()).get("ring_configs", {})
    lib = r._lib
    stream = torch.cuda.current_stream(device)
    out = {}
    for name, (cfg_no, k, m, w) in SWEEP_CONFIGS.items():
        tr, pay = synthetic.shell_arrays(k, m)
        r.set_scene_composed(api.compose(tr), api.PrimitiveSlab(k, m, pay), api.WindowParams())
        del pay
        cams = [synthetic.shell_camera(v, N_RING, w) for v in range(8)]
        mc = api.MarchConfig()
        host = r.render_batch(cams, mc)  # also sets the raymarch tier for this density
        g = golden.get(name, {}).get("views", {})
        digest_ok = bool(g) and all(
            sha(o.color) == g[str(v)]["rgb"] and sha(o.alpha) == g[str(v)]["alpha"]
            and sha(o.sample_counts) == g[str(v)]["samples"] for v, o in enumerate(host))
        ray_samples = sum(o.total_samples() for o in host)
        prim = 0
        for c in cams:  # per-view device counters (deterministic)
            prim += r.render(c, mc).stats["prim_samples"]
        n_px = w * w
        bufs = [(torch.empty(n_px * 3, device=device), torch.empty(n_px, device=device),
                 torch.empty(n_px, dtype=torch.int32, device=device)) for _ in range(8)]
        cc = (vp_camera * 8)(*[c.to_c() for c in cams])
        mcc = mc.to_c()
        rgb = (f32p * 8)(*[C.cast(b[0].data_ptr(), f32p) for b in bufs])
        alp = (f32p * 8)(*[C.cast(b[1].data_ptr(), f32p) for b in bufs])
        smp = (i32p * 8)(*[C.cast(b[2].data_ptr(), i32p) for b in bufs])

        def launch():
            if lib.vp_render_batch_async(r.ctx, 8, cc, C.byref(mcc), rgb, alp, smp, C.c_void_p(stream.cuda_stream)):
                raise RuntimeError(lib.vp_last_error(r.ctx).decode())

        for _ in range(3):
            launch()
        torch.cuda.synchronize()
        r.kernel_times()
        evs = []
        for i in range(args.sweep_steps):
            flush.fill_(i & 0xff)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            launch()
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        kms = r.kernel_times(4096)
        step_s = sum(a.elapsed_time(b) for a, b in evs) / 1e3
        kernel_s = float(np.mean(kms)) / 1e3
        alg = BYTES_PER_PRIM_SAMPLE * prim + BYTES_PER_PIXEL * n_px * 8
        out[name] = {"baseline_config": cfg_no, "K": k, "M": m, "width": w, "views_per_launch": 8,
                     "views": "ring 0..7", "value": round(ray_samples * args.sweep_steps / step_s / 1e6, 3),
                     "unit": METRIC, "frames_per_s": round(8 * args.sweep_steps / step_s, 2),
                     "ms_per_launch_step": round(1e3 * step_s / args.sweep_steps, 4),
                     "kernel_ms_per_launch": round(kernel_s * 1e3, 4),
                     "prim_samples_per_launch": int(prim), "ray_samples_per_launch": int(ray_samples),
                     "roofline_frac": round(alg / kernel_s / 1e9 / hbm, 4),
                     "achieved_gbs": round(alg / kernel_s / 1e9, 1),
                     "digest_ok": digest_ok, "steps": args.sweep_steps}
        del bufs
        torch.cuda.synchronize()
    return out


def workload_config(args, world, gather):
    return {"workload": f"mvp_shell K={args.k} M={args.m} at {args.width}x{args.width}: "
                        f"{args.views_per_gpu} views/GPU/step of the 64-view ring (BASELINE configs 3+5, "
                        f"view-sharded)",
            "K": args.k, "M": args.m, "width": args.width, "height": args.width,
            "views_per_gpu": args.views_per_gpu, "parallelism": f"view-shard x{world}",
            "gather_to_rank0": gather, "march": "dt=1mm earlyEps=0.01 window 8/8 no jitter",
            "l2": "flushed (256 MiB write) before every timed step; payload 268 MB > 126 MB L2"}


def run_tile_shard(args, rank, world, local, device, native=False):
    """--tile-shard: one view per step split by tile over the ranks (single-view
    configs). Step = this rank's shard render + the gather of every shard to rank 0 + rank 0
    placing the tiles into the image. value = the view's ray-samples / max-over-ranks time."""
    import torch
    import torch.distributed as dist

    from paper_2103_01954_b200 import Renderer, api, synthetic
    from paper_2103_01954_b200.dist import NativeComm, TileShardGather, broadcast_scene

    k, m, w = args.k, args.m, args.width
    r = Renderer(local)
    xf = slab = None
    if rank == 0:
        tr, pay = synthetic.shell_arrays(k, m)
        xf = api.compose(tr)
        slab = api.PrimitiveSlab(k, m, pay)
    win = api.WindowParams()
    comm = None
    if native:  # libvpb's NCCL: the shard buffers travel as one "view" of slots_max * 256 pixels
        comm = NativeComm(r, world, rank, max_ctas=args.nccl_max_ctas)
        comm.broadcast_scene(xf, slab, win, k, m)
    elif world > 1:
        broadcast_scene(r, xf, slab, win, k, m, device)
    else:
        r.set_scene_composed(xf, slab, win)
    cam = synthetic.shell_camera(-1, 0, w)
    cfg = api.MarchConfig()
    g = TileShardGather(w, w, device, world, rank)
    rgb, alpha, samp = g.outputs()
    stream = torch.cuda.Stream(device)
    torch.cuda.set_stream(stream)

    dst = None
    if native and rank == 0:  # rank r's shard lands in g.recv[r]: [rgb 3n | alpha n | samples n]
        n = g.n
        dst = ([t.data_ptr() for t in g.recv], [t[3 * n:].data_ptr() for t in g.recv],
               [t[4 * n:].data_ptr() for t in g.recv])

    def step():
        if native:
            comm.wait(stream.cuda_stream)  # the previous gather has read this rank's buffer
        r.render_shard_device(cam, cfg, rank, world, rgb.data_ptr(), alpha.data_ptr(), samp.data_ptr(),
                              stream.cuda_stream)
        if native:
            comm.gather_views(1, g.n, [rgb.data_ptr()], [alpha.data_ptr()], [samp.data_ptr()], dst)
            comm.wait(stream.cuda_stream)  # rank 0 places the tiles after the gather
        elif world > 1:
            g.gather()
            g.wait()
        if rank == 0:
            g.assemble()

    step()
    torch.cuda.synchronize()
    mine = r.read_stats()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    r.kernel_times()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.2)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.fill_(i & 0xff)
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    t_local = sum(a.elapsed_time(b) for a, b in evs) / 1e3
    march_ms = r.kernel_times(4096)
    cdev = "cpu" if native else device  # gloo (the native data plane's control plane) reduces CPU tensors
    t = torch.tensor([t_local], dtype=torch.float64, device=cdev)
    tot = torch.tensor([mine["ray_samples"], mine["prim_samples"]], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot)
    t_max = float(t.item())
    ray_view, prim_view = (float(x) for x in tot.tolist())
    pk, pk_kind = peaks()
    hbm = float(pk.get("hbm_gbs", 6650.0))
    alg = BYTES_PER_PRIM_SAMPLE * mine["prim_samples"] + BYTES_PER_PIXEL * 256 * api.shard_tiles(w, w, rank, world)
    march_s = float(np.mean(march_ms)) / 1e3 if len(march_ms) else float("nan")
    if rank == 0:
        line = {"metric": METRIC, "value": round(ray_view * args.steps / t_max / 1e6, 3), "unit": METRIC,
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(1e3 * t_max / args.steps, 4), "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": f"mvp_shell K={k} M={m}, ONE {w}x{w} view per step split by tile over "
                                       f"{world} GPU(s) (BASELINE config {3 if k == 4096 else 'n/a'}, tile-sharded)",
                           "K": k, "M": m, "width": w, "height": w, "parallelism": f"tile-shard x{world}",
                           "gather_to_rank0": world > 1,
                           "data_plane": ("libvpb vp_comm_* (NCCL)" if native else
                                          ("torch.distributed NCCL" if world > 1 else "none (1 GPU)")),
                           "l2": "flushed (256 MiB write) before every timed step"},
                "frames_per_s": round(args.steps / t_max, 2),
                "prim_samples_per_s": round(prim_view * args.steps / t_max / 1e6, 3),
                "roofline": {"bound": "hbm", "achieved": round(alg / march_s / 1e9, 1), "peak": hbm, "unit": "GB/s",
                             "frac": round(alg / march_s / 1e9 / hbm, 4), "traffic": None,
                             "kernel": "k_march_tiles (+k_march_fallback_views), rank 0's shard",
                             "peak_kind": pk_kind, "avg_launch_ms": round(march_s * 1e3, 4)},
                "cpu_baseline": None, "e2e": None,
                # per step: 6 binning stages, the raymarch, its fallback and the last-resort pass
                "gpu_launches": 9 * args.steps, "clocks": clk}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    r.close()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_2103_01954_b200 import Renderer, api, synthetic
    from paper_2103_01954_b200._lib import f32p, i32p, vp_camera, vp_march, vp_stats
    from paper_2103_01954_b200.dist import NativeComm, NativeViewGather, ViewGather, broadcast_scene, view_shard
    import ctypes as C

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    # data plane: libvpb's own NCCL (vp_comm_*), so torch.distributed is only the control plane
    # (rendezvous, the NCCL id, barriers, the max-over-ranks timing): gloo on CPU tensors.
    # --torch-comm (and the tile-shard mode) move the data plane to torch.distributed NCCL.
    native = (world > 1 or args.comm_at_1) and not args.torch_comm
    if world > 1:
        if native:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=device)
    if args.tile_shard:
        run_tile_shard(args, rank, world, local, device, native=native)
        if world > 1:
            dist.destroy_process_group()
        return
    gather = (world > 1 or native) and not args.no_gather
    k, m, w = args.k, args.m, args.width
    V = args.views_per_gpu
    r = Renderer(local)

    # scene: built on rank 0, broadcast once (payload already repacked)
    xf = slab = None
    if rank == 0:
        tr, pay = synthetic.shell_arrays(k, m)
        xf = api.compose(tr)
        slab = api.PrimitiveSlab(k, m, pay)
    win = api.WindowParams()
    t_up = time.perf_counter()
    comm = None
    if native:
        comm = NativeComm(r, world, rank, max_ctas=args.nccl_max_ctas)
        bcast_bytes = comm.broadcast_scene(xf, slab, win, k, m)
    elif world > 1:
        bcast_bytes = broadcast_scene(r, xf, slab, win, k, m, device)
    else:
        r.set_scene_composed(xf, slab, win)
        bcast_bytes = 0
    scene_upload_ms = (time.perf_counter() - t_up) * 1e3  # one-time: H2D, K0 repack (+ broadcast)
    views = view_shard(N_RING, world, rank, per_rank=V)
    cams = [synthetic.shell_camera(v, N_RING, w).to_c() for v in views]
    cfg = api.MarchConfig()
    mc = cfg.to_c()

    # deterministic per-view counts (bit-exact renders), measured once outside the timed region
    per_view = []
    ring_golden = json.loads((ROOT / "tests" / "golden" / "digests.json").read_text()).get("ring", {})
    digest_ok = (ring_golden.get("K"), ring_golden.get("M"), ring_golden.get("W")) == (k, m, w)
    for v, cam in zip(views, cams):
        out = r.render(api.Camera.from_c(cam), cfg)
        per_view.append(out.stats)
        g = ring_golden.get("views", {}).get(str(v)) if digest_ok else None
        digest_ok = bool(g) and digest_ok and all(
            _sha(a) == g[key] for a, key in ((out.color, "rgb"), (out.alpha, "alpha"), (out.sample_counts, "samples")))
    ray_samples = sum(s["ray_samples"] for s in per_view)
    prim_samples = sum(s["prim_samples"] for s in per_view)

    # one view per launch (SURVEY.md §8d's per-view timing): K1-K5 of ONE view per raymarch
    # launch (vp_render_async into device buffers, renders back to back, so a view's binning
    # overlaps the previous view's raymarch), CUDA events on the launching stream, median of 20
    # after 5 warm-ups; outside the timed region, which marches 8 views per launch
    sv_stream = torch.cuda.Stream(device)
    sv_out = [torch.empty(w * w * 3, device=device), torch.empty(w * w, device=device),
              torch.empty(w * w, dtype=torch.int32, device=device)]
    sv_ms = []
    cam0 = api.Camera.from_c(cams[0])
    for i in range(25):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sv_stream)
        r.render_device(cam0, cfg, sv_out[0].data_ptr(), sv_out[1].data_ptr(), sv_out[2].data_ptr(),
                        sv_stream.cuda_stream)
        e1.record(sv_stream)
        sv_ms.append((e0, e1))
    torch.cuda.synchronize()
    single_view_ms = float(np.median([a.elapsed_time(b) for a, b in sv_ms[5:]]))
    del sv_out
    r.kernel_times()

    vg = NativeViewGather(comm, V, w, w, device) if native else ViewGather(V, w, w, device, world, rank)
    # a dedicated (non-default) stream: the renders, the timing events and the NCCL gathers'
    # dependencies all hang off it
    stream = torch.cuda.Stream(device)
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream
    assert sh != 0
    lib = r._lib
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)

    batch = not args.per_view and V <= 16
    cams_arr = (vp_camera * V)(*cams)
    slot_ptrs = []  # per output slot: (rgb, alpha, samples) pointer arrays and row views
    for s in range(vg.slots):
        rgb, alpha, samples = vg.views(s)
        slot_ptrs.append(((f32p * V)(*[C.cast(rgb[j].data_ptr(), f32p) for j in range(V)]),
                          (f32p * V)(*[C.cast(alpha[j].data_ptr(), f32p) for j in range(V)]),
                          (i32p * V)(*[C.cast(samples[j].data_ptr(), i32p) for j in range(V)])))

    def step(i):
        # step i renders into output slot i % 2; with N > 1 its gathers to rank 0 run on NCCL's
        # stream under step i+1's raymarch (which renders into the other slot)
        slot = i % vg.slots
        if gather:
            if native:  # the render stream waits for the gathers still reading this slot
                vg.wait_slot(slot, sh)
            else:
                vg.wait_slot(slot)
        rgb_ptrs, alpha_ptrs, samp_ptrs = slot_ptrs[slot]
        if batch:  # every view of the step in one raymarch launch
            if lib.vp_render_batch_async(r.ctx, V, cams_arr, C.byref(mc), rgb_ptrs, alpha_ptrs, samp_ptrs,
                                         C.c_void_p(sh)):
                raise RuntimeError(lib.vp_last_error(r.ctx).decode())
            if gather and native:  # every view of the step in ONE grouped NCCL call
                vg.gather(slot)
            elif gather:
                for j in range(V):
                    vg.gather_view(j, slot=slot)
        else:
            for j, cam in enumerate(cams):
                rc = lib.vp_render_async(r.ctx, C.byref(cam), C.byref(mc), rgb_ptrs[j], alpha_ptrs[j],
                                         samp_ptrs[j], C.c_void_p(sh))
                if rc:
                    raise RuntimeError(lib.vp_last_error(r.ctx).decode())
                if gather and not native:
                    vg.gather_view(j, slot=slot)
            if gather and native:
                vg.gather(slot)

    for i in range(args.warmup):
        step(i)
    if gather:
        vg.finish()
    torch.cuda.synchronize()
    rc_stats = vp_stats()
    if lib.vp_read_stats(r.ctx, C.byref(rc_stats)):
        raise RuntimeError(lib.vp_last_error(r.ctx).decode())
    r.kernel_times()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.2)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.fill_(i & 0xff)                 # evict L2 (untimed)
        evs[i][0].record(stream)
        step(args.warmup + i)
        if gather and i == args.steps - 1:    # the last step's gathers end inside the timed region
            if native:
                vg.wait_slot(0, sh)           # the render stream (and its end event) waits for them
            else:
                vg.finish()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    t_local = sum(step_ms) / 1e3
    march_ms = r.kernel_times(4096)
    cdev = "cpu" if native else device  # gloo reduces CPU tensors
    t = torch.tensor([t_local], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    totals = torch.tensor([ray_samples * args.steps, prim_samples * args.steps, V * args.steps],
                          dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(totals)
    all_ray, all_prim, all_views = (float(x) for x in totals.tolist())
    value = all_ray / t_max / 1e6

    # roofline of the dominant kernel (raymarch K5 + fallback K5b), per launch
    pk, pk_kind = peaks()
    hbm = float(pk.get("hbm_gbs", 6650.0))
    views_per_launch = V if batch else 1
    alg_bytes_per_launch = (BYTES_PER_PRIM_SAMPLE * prim_samples + BYTES_PER_PIXEL * w * w * V) / V * views_per_launch
    march_avg_s = float(np.mean(march_ms)) / 1e3 if len(march_ms) else float("nan")
    achieved = alg_bytes_per_launch / march_avg_s / 1e9
    frame_s = t_local / (V * args.steps)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": None,
                "kernel": "k_march_tiles (+k_march_fallback_views)", "peak_kind": pk_kind,
                "views_per_launch": views_per_launch,
                "alg_bytes_per_launch": int(alg_bytes_per_launch), "avg_launch_ms": round(march_avg_s * 1e3, 4),
                "march_share_of_step": round(march_avg_s * V / views_per_launch * args.steps / max(t_local, 1e-12), 4),
                "frame_ms": round(frame_s * 1e3, 4),
                "frame_frac": round(alg_bytes_per_launch / views_per_launch / frame_s / 1e9 / hbm, 4),
                # the bytes a launch cannot avoid (the payload read once, the
                # outputs written once) and the time they take at the peak
                "compulsory_bytes_per_launch": int(k * m ** 3 * 16 + BYTES_PER_PIXEL * w * w * views_per_launch),
                "compulsory_ms_at_peak": round((k * m ** 3 * 16 + BYTES_PER_PIXEL * w * w * views_per_launch)
                                               / (hbm * 1e9) * 1e3, 4)}
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        try:
            tr_ = json.loads(prof.read_text())
            key = f"K{k}_M{m}_W{w}"
            if key in tr_:
                roofline["traffic"] = tr_[key]["dram_bytes_per_view"] * views_per_launch
                roofline["traffic_source"] = tr_[key]["source"]
        except Exception:
            pass

    # e2e: public C-ABI, pinned host buffers, per step: transforms H2D + outputs D2H
    e2e = None
    if not (args.no_e2e or args.quick):
        n_px = w * w
        h_rgb = torch.empty((V, n_px * 3), dtype=torch.float32, pin_memory=True)
        h_alpha = torch.empty((V, n_px), dtype=torch.float32, pin_memory=True)
        h_samp = torch.empty((V, n_px), dtype=torch.int32, pin_memory=True)
        h_rgb_p = (f32p * V)(*[C.cast(h_rgb[j].data_ptr(), f32p) for j in range(V)])
        h_alpha_p = (f32p * V)(*[C.cast(h_alpha[j].data_ptr(), f32p) for j in range(V)])
        h_samp_p = (i32p * V)(*[C.cast(h_samp[j].data_ptr(), i32p) for j in range(V)])
        if world > 1:  # every rank holds the broadcast transforms
            xf_host = torch.from_numpy(np.ascontiguousarray(r.transforms())).pin_memory()
        else:
            xf_host = torch.from_numpy(xf).pin_memory()
        st = vp_stats()

        def e2e_step():
            # per step: the frame's transforms host->device, then every view rendered into
            # pinned host memory; each view's device->host copy overlaps the next render (also
            # across steps); vp_sync after the last step waits for every copy
            set_xf = lib.vp_set_transforms_async if batch else lib.vp_set_transforms
            if (set_xf(r.ctx, k, C.cast(xf_host.data_ptr(), f32p), None) if batch
                    else set_xf(r.ctx, k, C.cast(xf_host.data_ptr(), f32p))):
                raise RuntimeError(lib.vp_last_error(r.ctx).decode())
            if batch:  # one launch for the step's views; their copies overlap the next step
                if lib.vp_render_batch_async(r.ctx, V, cams_arr, C.byref(mc), h_rgb_p, h_alpha_p, h_samp_p, None):
                    raise RuntimeError(lib.vp_last_error(r.ctx).decode())
                return
            for j, cam in enumerate(cams):
                if lib.vp_render_async(r.ctx, C.byref(cam), C.byref(mc), C.cast(h_rgb[j].data_ptr(), f32p),
                                       C.cast(h_alpha[j].data_ptr(), f32p), C.cast(h_samp[j].data_ptr(), i32p),
                                       None):
                    raise RuntimeError(lib.vp_last_error(r.ctx).decode())

        def e2e_finish():
            if lib.vp_sync(r.ctx) or lib.vp_read_stats(r.ctx, C.byref(st)):
                raise RuntimeError(lib.vp_last_error(r.ctx).decode())

        for _ in range(max(1, args.warmup // 2)):
            e2e_step()
        e2e_finish()
        n_e2e = max(3, args.steps)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            e2e_step()
        e2e_finish()
        te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=cdev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": round(all_ray / args.steps * n_e2e / float(te.item()) / 1e6, 3), "unit": METRIC,
               "h2d_bytes_per_step": 15 * 4 * k, "d2h_bytes_per_step": BYTES_PER_PIXEL * n_px * V,
               "steps": n_e2e, "api": ("vp_set_transforms_async + vp_render_batch_async" if batch else "vp_set_transforms + vp_render_async")
                      + " into pinned host outputs, vp_sync at the end"}

    sweep = None
    if world == 1 and not (args.no_sweep or args.quick):
        sweep = run_sweep(r, args, device, flush, hbm)

    cpu = None
    if rank == 0 and world == 1 and not (args.no_cpu_baseline or args.quick):
        ref = CpuReference(k, m, w)
        s, dt, nv = ref.sample(views, args.cpu_seconds)
        cpu = {"value": round(s / dt / 1e6, 3), "unit": METRIC, "cores": ref.cores, "kind": ref.kind,
               "cpu_model": cpu_model(),
               "sample": f"{nv} view(s) of this rank's views, full {w}x{w} frames, {dt:.1f} s, resident "
                         f"reference Scene (volprim::render only)"}
        one = ref.sample_one_core(views[0]) if args.cpu_one_core else None
        if one:
            cpu["one_core"] = {"value": round(one[0] / one[1] / 1e6, 3), "unit": METRIC, "cores": 1,
                               "core_id": one[2], "seconds": round(one[1], 2),
                               "sample": f"view {views[0]}, process pinned to one core (taskset -c equivalent)"}

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 3), "unit": METRIC, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * t_max / args.steps, 4),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "config": workload_config(args, world, gather),
                "frames_per_s": round(all_views / t_max, 2),
                "prim_samples_per_s": round(all_prim / t_max / 1e6, 3),
                "digest_ok": digest_ok,  # every timed view bit-equal to the reference's digest
                "ray_samples_per_view": ray_samples // V, "prim_samples_per_view": prim_samples // V,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "sweep": sweep,
                # per step, batched: 6 binning stages for all views, the cross-view tile order, the
                # raymarch, the fallback and the last-resort pass; per view: 6 + 3 for each view
                "gpu_launches": (10 if batch else 9 * V) * args.steps,
                "clocks": clk, "scene_broadcast_bytes": bcast_bytes,
                "data_plane": ("libvpb vp_comm_* (NCCL: vp_broadcast_scene once, one grouped vp_gather_views per "
                               f"step, maxCTAs {args.nccl_max_ctas}; torch.distributed gloo for control only)"
                               if native else ("torch.distributed NCCL" if world > 1 else "none (1 GPU)")),
                "single_view": {"ms": round(single_view_ms, 4), "frames_per_s": round(1e3 / single_view_ms, 1),
                                "what": "one view per raymarch launch (vp_render_async, back to back), "
                                        f"median of 20, view {views[0]} of the ring"},
                "scene_upload_ms": round(scene_upload_ms, 2),
                "stats_last_launch": rc_stats.as_dict()}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    r.close()


if __name__ == "__main__":
    main()

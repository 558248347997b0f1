"""Roll an ncu SASS source page up into named source regions (profiling helper).

    python tools/ncu_regions.py REPORT CUBIN FUNC_SUBSTR N_PRIM_SAMPLES
Regions are [file-suffix, first line, last line, name] ranges resolved from function
markers in the current sources, so the tool keeps working when lines move.
"""
import collections
import re
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_source_lines import ncu_rows, sass_lines  # noqa: E402

SRC = "paper_2103_01954_b200/csrc/"
MARKERS = [("vpb_device.cuh", r"^__device__ __forceinline__ V3 mk3", "vec/mat ops"),
           ("vpb_device.cuh", r"^__device__ __forceinline__ V3 to_model", "to_model (3 IEEE div)"),
           ("vpb_device.cuh", r"^__device__ __forceinline__ bool intersect_obb_om", "intersect_obb"),
           ("vpb_device.cuh", r"^// Conservative line-vs-box", "line prefilter"),
           ("vpb_device.cuh", r"^// camera.cpp:14-23", "generate_ray/hash"),
           ("vpb_device.cuh", r"^// glibc 2.39 expf", "expf (binary64 port)"),
           ("vpb_device.cuh", r"^// primitive.cpp:12-22", "window/pow8/clamp"),
           ("vpb_device.cuh", r"^// One primitive-sample", "sample_primitive (stencil+gather)"),
           ("vpb_march.cuh", r"^// Candidate sources", "candidate accessors"),
           ("vpb_march.cuh", r"^// Per-ray sorted segment window", "window accessors"),
           ("vpb_march.cuh", r"^__device__ __forceinline__ bool key_less", "window insert/scan"),
           ("vpb_march.cuh", r"^// The fused quadrature", "march loop control"),
           ("vpb_march.cuh", r"^// Generic variant for windows wider", "march loop (generic)"),
           ("vpb_march.cuh", r"^__device__ __forceinline__ void write_pixel", "outputs/counters"),
           ("vpb_kernels.cu", r"^// K5: one CTA", "tile kernel body"),
           ("vpb_kernels.cu", r"^// K5b", "end")]


def ranges():
    out = []
    for f in ("vpb_device.cuh", "vpb_march.cuh", "vpb_kernels.cu"):
        lines = open(SRC + f).read().splitlines()
        marks = []
        for ff, pat, name in MARKERS:
            if ff != f:
                continue
            for i, l in enumerate(lines, 1):
                if re.search(pat, l):
                    marks.append((i, name))
                    break
        marks.sort()
        for (a, name), nxt in zip(marks, marks[1:] + [(len(lines) + 1, None)]):
            out.append((f, a, nxt[0] - 1, name))
    return out


def main():
    report, cubin, func = sys.argv[1:4]
    nps = float(sys.argv[4]) if len(sys.argv) > 4 else 0
    R = ranges()
    agg = collections.defaultdict(lambda: [0, 0, 0])
    for loc, r in zip(sass_lines(cubin, func), ncu_rows(report)):
        name = "other"
        if loc:
            f, l = loc.rsplit(":", 1)
            for ff, a, b, n in R:
                if f == ff and a <= int(l) <= b:
                    name = n
                    break
            else:
                name = f"other ({f})"
        a = agg[name]
        a[0] += int(r.get("Instructions Executed", 0) or 0)
        a[1] += int(r.get("Thread Instructions Executed", 0) or 0)
        a[2] += int(r.get("Warp Stall Sampling (All Samples)", 0) or 0)
    tot = [sum(v[i] for v in agg.values()) or 1 for i in range(3)]
    print(f"{'region':36s} {'warp-inst':>9s} {'%':>6s} {'thr/inst':>8s} {'stall%':>7s} {'thr-inst/prim-sample':>20s}")
    for k, (wi, ti, st) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        per = f"{ti / nps:20.1f}" if nps else ""
        print(f"{k:36s} {wi / 1e6:8.1f}M {100 * wi / tot[0]:6.2f} {ti / max(wi, 1):8.1f} {100 * st / tot[2]:7.2f} {per}")
    print(f"total: {tot[0] / 1e6:.1f}M warp-inst, {tot[1] / 1e9:.2f}G thread-inst, {tot[1] / tot[0]:.1f} threads/inst"
          + (f", {tot[1] / nps:.0f} thread-inst per prim-sample" if nps else ""))


if __name__ == "__main__":
    main()

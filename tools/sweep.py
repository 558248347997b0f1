"""Runs the headline bit-exact digest test and bench.py --quick on several configs for each
libvpb variant (tuning sweeps). Usage: python tools/sweep.py [lib.so ...]"""
import glob
import json
import os
import subprocess
import sys

CFGS = [[], ["--k", "32768", "--m", "8"], ["--k", "512", "--m", "32"], ["--k", "64", "--m", "16", "--width", "256"]]
if os.environ.get("SWEEP_ONLY"):  # comma-separated indices into CFGS
    CFGS = [CFGS[int(i)] for i in os.environ["SWEEP_ONLY"].split(",")]
libs = sys.argv[1:] or sorted(glob.glob("build/variants/libvpb_*.so"))
for lib in libs:
    env = dict(os.environ, VPB_LIB=os.path.abspath(lib))
    t = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "tests/test_gpu_parity.py",
                        "-k", "full_size or render_matches"], env=env, capture_output=True, text=True)
    ok = t.stdout.strip().splitlines()[-1] if t.stdout.strip() else t.stderr[-300:]
    res = []
    for cfg in CFGS:
        b = subprocess.run([sys.executable, "bench.py", "--quick", "--steps", "10", "--warmup", "3", *cfg],
                           env=env, capture_output=True, text=True)
        try:
            j = json.loads(b.stdout.strip().splitlines()[-1])
            res.append(f"{j['roofline']['avg_launch_ms']:.4f}ms/{j['roofline']['frac']:.3f}")
        except Exception:
            res.append("FAILED " + b.stderr[-200:])
    print(f"{os.path.basename(lib):24s} " + "  ".join(res) + f"  | {ok}", flush=True)

"""Runs bench.py --quick (and the headline bit-exact digest test) for each libvpb variant."""
import glob
import json
import os
import subprocess
import sys

libs = sys.argv[1:] or sorted(glob.glob("build/variants/libvpb_*.so"))
for lib in libs:
    env = dict(os.environ, VPB_LIB=os.path.abspath(lib))
    t = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "tests/test_gpu_parity.py",
                        "-k", "full_size and k4096_m16_1024_view-1 or render_matches"], env=env,
                       capture_output=True, text=True)
    ok = t.stdout.strip().splitlines()[-1] if t.stdout.strip() else t.stderr[-300:]
    b = subprocess.run([sys.executable, "bench.py", "--quick", "--steps", "10", "--warmup", "3"], env=env,
                       capture_output=True, text=True)
    try:
        j = json.loads(b.stdout.strip().splitlines()[-1])
        print(f"{os.path.basename(lib):22s} {j['value']:9.1f} Msamples/s  march {j['roofline']['avg_launch_ms']:.4f} ms"
              f"  frac {j['roofline']['frac']:.3f}  frame {j['roofline']['frame_ms']:.4f} ms  | {ok}", flush=True)
    except Exception:
        print(lib, "FAILED", b.stderr[-500:], ok, flush=True)

"""Per-source-line roll-up of an ncu SASS source page (profiling helper, not product code).

    python tools/ncu_source_lines.py REPORT.ncu-rep CUBIN KERNEL_MANGLED_SUBSTR [top]

ncu's `--page source --csv` gives per-SASS-instruction counters; `nvdisasm -g -c` of the same
cubin gives each instruction's file:line. Instructions are matched by order within the
function, then executed instructions, thread instructions and stall samples are summed per
line (innermost inlined location).
"""
import collections
import csv
import io
import re
import subprocess
import sys


def sass_lines(cubin, func_substr):
    txt = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    out, cur, inside = [], None, False
    for line in txt.splitlines():
        if line.startswith("//---------------------") and ".text." in line:
            inside = func_substr in line
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        if re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
            out.append(cur)
    return out


def ncu_rows(report):
    txt = subprocess.run(["ncu", "-i", report, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    return [dict(zip(hdr, r)) for r in rows[hdr_i + 1:] if len(r) == len(hdr)]


def main():
    report, cubin, func = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    lines = sass_lines(cubin, func)
    rows = ncu_rows(report)
    if len(lines) != len(rows):
        print(f"warning: {len(lines)} disassembled vs {len(rows)} profiled instructions")
    agg = collections.defaultdict(lambda: [0, 0, 0])
    for loc, r in zip(lines, rows):
        a = agg[loc]
        a[0] += int(r.get("Instructions Executed", 0) or 0)
        a[1] += int(r.get("Thread Instructions Executed", 0) or 0)
        a[2] += int(r.get("Warp Stall Sampling (All Samples)", 0) or 0)
    tot = [sum(v[i] for v in agg.values()) or 1 for i in range(3)]
    print(f"{'location':34s} {'warp-inst':>12s} {'%':>6s} {'thr/inst':>8s} {'stall%':>7s}")
    for loc, (wi, ti, st) in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
        print(f"{str(loc):34s} {wi:12d} {100 * wi / tot[0]:6.2f} {ti / max(wi, 1):8.1f} {100 * st / tot[2]:7.2f}")
    print(f"total warp-inst {tot[0]}, thread-inst {tot[1]}, avg threads/inst {tot[1] / tot[0]:.1f}")


if __name__ == "__main__":
    main()

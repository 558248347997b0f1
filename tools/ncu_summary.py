"""Summary of one ncu --set full capture of the raymarch kernel (profiling helper).

    python tools/ncu_summary.py REPORT.ncu-rep LIBVPB.so FUNC_SUBSTR "header line" > summary.txt

Prints the headline counters, the warp-stall breakdown and the per-region roll-up
(tools/ncu_regions.py) of the SASS source page. The cubin is extracted from the given
libvpb.so (the exact build that was profiled).
"""
import csv
import io
import pathlib
import subprocess
import sys
import tempfile

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__cycles_active.avg", "gpc__cycles_elapsed.max", "launch__grid_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.per_cycle_active", "smsp__issue_active.avg.per_cycle_active",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed"]


def raw(report):
    txt = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return dict(zip(rows[0], rows[2]))


def main():
    report, lib, func, header = sys.argv[1:5]
    r = raw(report)
    print(f"# {header}")
    for k in KEYS:
        if k in r:
            print(f"{k:70s} {r[k]}")
    stalls = {k[len("smsp__pcsamp_warps_issue_stalled_"):].replace(".sum", ""): float(v.replace(",", ""))
              for k, v in r.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in k
              and v.replace(",", "").replace(".", "").isdigit()}
    tot = sum(stalls.values()) or 1.0
    print("\n# warp stall reasons (share of pc samples)")
    print(", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in sorted(stalls.items(), key=lambda t: -t[1])[:10]))
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", str(pathlib.Path(lib).resolve())], cwd=d,
                       capture_output=True)
        cubins = sorted(pathlib.Path(d).glob("*vpb_kernels*.cubin"))
        if cubins:
            print("\n# per-region roll-up (tools/ncu_regions.py)")
            out = subprocess.run([sys.executable, str(pathlib.Path(__file__).with_name("ncu_regions.py")), report,
                                  str(cubins[0]), func, "0"], capture_output=True, text=True)
            print(out.stdout.strip() or out.stderr.strip()[-500:])


if __name__ == "__main__":
    main()

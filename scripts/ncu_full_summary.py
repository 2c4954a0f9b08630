"""Summary of ncu --set full captures (the numbers DESIGN.md and profiles/r2 cite).

    python scripts/ncu_full_summary.py <capture.ncu-rep> [...] > summary.txt
Per kernel: duration, DRAM bytes and GB/s (% of the measured HBM peak), L2 bytes, L1/L2
hit rates, IPC, issue-slot use, achieved occupancy, registers, active and
not-predicated-off threads per warp (warp execution efficiency), ALU / LSU pipe use,
shared-memory bank conflicts, and the top warp-stall reasons.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    return [(dict(zip(h, r)), dict(zip(h, units))) for r in rows[2:]]


def num(d, k):
    try:
        return float(str(d.get(k, "nan")).replace(",", ""))
    except ValueError:
        return float("nan")


def scale(v, unit):  # ncu unit strings -> bytes / seconds
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9,
                "us": 1e-6, "ms": 1e-3, "s": 1, "sector": 32}.get(unit, 1)


def main():
    pk = peak()
    for rep in sys.argv[1:]:
        for d, u in raw(rep):
            k = d["Kernel Name"]
            t = scale(num(d, "gpu__time_duration.sum"), u.get("gpu__time_duration.sum"))
            dr = scale(num(d, "dram__bytes_read.sum"), u.get("dram__bytes_read.sum")) + \
                scale(num(d, "dram__bytes_write.sum"), u.get("dram__bytes_write.sum"))
            l2 = 32 * num(d, "lts__t_sectors.sum")  # L2 sectors x 32 B
            stalls = sorted(((num(d, x), x[33:]) for x in d if x.startswith(
                "smsp__pcsamp_warps_issue_stalled") and not x.endswith("not_issued")), reverse=True)
            tot = sum(v for v, _ in stalls if v == v) or 1
            print(f"== {os.path.basename(rep)}: {k[:110]}")
            print(f"  duration {1e3 * t:.3f} ms  DRAM {dr / 1e9:.3f} GB = {dr / t / 1e9:.1f} GB/s "
                  f"({100 * dr / t / 1e9 / pk:.2f}% of {pk:.0f} GB/s)  L2 {l2 / 1e9:.2f} GB "
                  f"({l2 / t / 1e12:.2f} TB/s)")
            print(f"  L1 hit {num(d, 'l1tex__t_sector_hit_rate.pct'):.1f}%  L2 hit "
                  f"{num(d, 'lts__t_sector_hit_rate.pct'):.1f}%  IPC "
                  f"{num(d, 'sm__inst_executed.avg.per_cycle_active'):.2f}  issue active "
                  f"{num(d, 'sm__inst_issued.avg.pct_of_peak_sustained_active'):.1f}%  "
                  f"occupancy {num(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}%  "
                  f"regs {num(d, 'launch__registers_per_thread'):.0f}")
            print(f"  threads/warp active {num(d, 'smsp__thread_inst_executed_per_inst_executed.ratio'):.1f}"
                  f"  not-pred-off {num(d, 'smsp__thread_inst_executed_pred_on_per_inst_executed.ratio'):.1f}"
                  f"  ALU pipe {num(d, 'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active'):.1f}%"
                  f"  LSU wavefronts {num(d, 'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed'):.1f}%"
                  f"  smem bank conflicts {num(d, 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum'):.3g}")
            print("  stalls " + "  ".join(f"{n}:{100 * v / tot:.0f}%" for v, n in stalls[:6]))


if __name__ == "__main__":
    main()

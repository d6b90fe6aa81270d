"""Summarise an .ncu-rep: key throughput metrics + top stall reasons per kernel."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__average_warp_latency_per_inst_issued.ratio"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"== {d.get('Kernel Name', '?')[:90]}")
        for k in KEYS:
            if k in d:
                print(f"   {k:70s} {d[k]:>14s} {u.get(k, '')}")
        stalls = sorted(((float(v.replace(',', '')), k) for k, v in d.items()
                         if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                         and v not in ("", "n/a")), reverse=True)[:6]
        tot = sum(float(v.replace(',', '')) for k, v in d.items()
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                  and v not in ("", "n/a")) or 1
        print("   stalls: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')}={v / tot:.0%}"
                                       for v, k in stalls))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)

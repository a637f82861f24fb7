"""Summarise an .ncu-rep: key throughput metrics + top stall lines (run here, no GPU)."""
import csv
import io
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main(rep, top=20):
    det = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    keep = {"Duration", "DRAM Throughput", "Memory Throughput", "SM Active Cycles", "Elapsed Cycles",
            "Compute (SM) Throughput", "Registers Per Thread", "Achieved Occupancy",
            "Dynamic Shared Memory Per Block", "Issue Slots Busy", "L2 Hit Rate",
            "Executed Ipc Active", "Theoretical Occupancy"}
    name = det[1][4] if len(det) > 1 else "?"
    print("kernel:", name[:100])
    for r in det[1:]:
        if r[12] in keep:
            print(f"  {r[12]:35s} {r[14]:>14s} {r[13]}")
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    for h, u, v in zip(hdr, units, vals):
        if h in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_tensor.sum", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
                 "gpu__time_duration.sum"):
            print(f"  {h:60s} {v} {u}")
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    if len(src) > 2:
        h = src[1]
        rows = src[2:]
        i_s = h.index("Warp Stall Sampling (All Samples)")
        tot = sum(int(x[i_s]) for x in rows if x[i_s].isdigit())
        print("  stall samples:", tot)
        agg = {}
        for x in rows:
            for j, c in enumerate(h):
                if c.startswith("stall_") and "Not Issued" not in c and x[j].isdigit():
                    agg[c] = agg.get(c, 0) + int(x[j])
        print("  by reason:", sorted(agg.items(), key=lambda kv: -kv[1])[:8])
        for x in sorted(rows, key=lambda x: -int(x[i_s]) if x[i_s].isdigit() else 0)[:top]:
            st = {h[j]: int(x[j]) for j in range(len(h)) if h[j].startswith("stall_")
                  and "Not Issued" not in h[j] and x[j].isdigit() and int(x[j]) > 0}
            print(f"  {x[i_s]:>5s} {x[1].strip()[:58]:58s} {sorted(st.items(), key=lambda kv: -kv[1])[:2]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)

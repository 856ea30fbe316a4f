"""Summarise an ncu --set full report (.ncu-rep) into the metrics the
profiles/ notes quote: time, DRAM bytes, throughput, occupancy, cache hit
rates, top stall reasons.  Usage: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__inst_executed.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        for w in WANT:
            if w in head:
                i = head.index(w)
                print(f"{w:70s} {r[i]} {units[i]}")
        stalls = [(float(r[i] or 0), head[i]) for i in range(len(head))
                  if head[i].startswith("smsp__average_warp_latency_issue_stalled_")
                  and head[i].endswith("_per_warp_active.pct") is False
                  and units[i] in ("", "cycle", "cycles")]
        if not stalls:
            stalls = [(float(r[i] or 0), head[i]) for i in range(len(head))
                      if "warps_issue_stalled" in head[i] and head[i].endswith(".ratio")]
        for v, n in sorted(stalls, reverse=True)[:6]:
            print(f"  stall {n:66s} {v:.2f}")
        print()


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"== {p}")
        main(p)

"""Summarise an ncu report (raw page) into the metrics this project tracks."""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__cluster_dim_x", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts.sum",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print("kernel:", name[:80])
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print(f"  {w} = {vals[i]} {units[i]}")
        stalls = [(float(vals[i] or 0), h) for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio") is False
                  and vals[i] not in ("", "n/a")]
        st = [(float(vals[i]), h) for i, h in enumerate(hdr)
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and vals[i] not in ("", "n/a")]
        st.sort(reverse=True)
        if st:
            print("  top stall samples:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')}={v:.0f}" for v, h in st[:8]))


if __name__ == "__main__":
    main(sys.argv[1])

"""Extract the headline metrics of an `ncu --set full` report (run here, no GPU):
python profiles/ncu_extract.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
        "smsp__average_warp_latency_per_inst_issued.ratio"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print("kernel:", name[:100])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:75s} {r[i]:>14s} {units[i]}")
        st = [(h, r[i]) for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled") and
              not h.endswith("not_issued") and r[i] not in ("", "0")]
        st.sort(key=lambda x: -float(x[1].replace(",", "")))
        tot = sum(float(v.replace(",", "")) for _, v in st) or 1
        print("  top stall reasons (pc samples):")
        for h, v in st[:6]:
            print(f"    {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {float(v.replace(',', ''))/tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])

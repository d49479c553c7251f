"""One-page summary of an .ncu-rep (first kernel): key metrics, stall mix, hottest SASS."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]


def main(rep, top=12):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    print("kernel:", v[h.index("Kernel Name")][:110])
    for k in KEYS:
        if k in h:
            print(f"  {k:80s} {v[h.index(k)]} {units[h.index(k)]}")
    st = [(float(v[i] or 0), h[i][len("smsp__pcsamp_warps_issue_stalled_"):]) for i in range(len(h))
          if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("not_issued")]
    tot = sum(x for x, _ in st) or 1.0
    print("  stall mix (share of pc samples):")
    for x, n in sorted(st, reverse=True)[:8]:
        print(f"    {n:30s} {100 * x / tot:5.1f} %")
    hot = subprocess.run([sys.executable, "tools/ncu_hot.py", rep, str(top)], capture_output=True, text=True).stdout
    print("\ntop SASS by stall samples:\n" + hot)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)

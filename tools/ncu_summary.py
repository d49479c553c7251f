"""Summarise an .ncu-rep: key throughput metrics, DRAM traffic, top stall reasons."""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum", "smsp__thread_inst_executed_per_inst_executed.ratio"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(hdr, units, r) for r in rows[2:]]


def main(rep):
    for hdr, units, r in raw(rep):
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print("kernel:", name[:120])
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        for k in WANT:
            if k in d:
                print(f"  {k:75s} {d[k]:>16s} {u.get(k, '')}")
        stalls = [(k, float(v)) for k, v in d.items()
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                  and v not in ("", "n/a")]
        stalls.sort(key=lambda kv: -kv[1])
        print("  top stalls (warps per issue-active cycle):")
        for k, v in stalls[:8]:
            print(f"    {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:30s} {v:.3f}")


if __name__ == "__main__":
    main(sys.argv[1])

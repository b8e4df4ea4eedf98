"""Summarise an ncu --set full report (first kernel) into the metrics the
round reports cite."""
import csv, subprocess, sys
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__block_size", "launch__grid_size", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]
def main(rep, title):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(raw))
    h, u, v = rows[0], rows[1], rows[2]
    ix = {n: i for i, n in enumerate(h)}
    print(f"--- {title}")
    print(f"  Kernel Name  {v[ix['Kernel Name']]}")
    for k in KEYS:
        if k in ix:
            print(f"  {k:62s} {v[ix[k]]} {u[ix[k]]}")
    st = [(n[len('smsp__pcsamp_warps_issue_stalled_'):], float(v[i])) for i, n in enumerate(h)
          if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")]
    tot = sum(x for _, x in st)
    st.sort(key=lambda x: -x[1])
    print("  stall samples (share): " + ", ".join(f"{n} {100*x/tot:.0f}%" for n, x in st[:6]))
if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

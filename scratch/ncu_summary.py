import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__registers_per_thread', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'lts__t_sector_hit_rate.pct', 'launch__grid_size', 'sm__inst_executed.sum',
        'smsp__average_warp_latency_issue_stalled_long_scoreboard', 'l1tex__t_bytes.sum']
extra = [a for a in sys.argv[2:]]
for row in r[2:]:
    print('---')
    for w in want + extra:
        if w in h:
            print(f'  {w:60s} {row[h.index(w)]}  {r[1][h.index(w)]}')

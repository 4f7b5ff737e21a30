"""One-line raw summary of a kernel in an ncu report (the figures bench.py and
DESIGN.md quote).  usage: python tools/ncu_summary.py <report.ncu-rep>"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum"]
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
w = csv.writer(sys.stdout)
w.writerow(["Kernel Name"] + [f"{k} [{units[h.index(k)]}]" for k in KEYS if k in h])
for r in rows[2:]:
    w.writerow([r[h.index("Kernel Name")]] + [r[h.index(k)] for k in KEYS if k in h])

"""Key metrics of every kernel in an .ncu-rep: python scripts/ncu_metrics.py X.ncu-rep [name]."""
import csv, io, json, subprocess, sys
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
     "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
res = []
for r in rows[2:]:
    d = dict(zip(h, r))
    e = {"kernel": d["Kernel Name"][:80]}
    for m in M:
        if m in d:
            u = units[h.index(m)]
            e[m] = d[m] + (f" {u}" if u else "")
    res.append(e)
print(json.dumps(res if len(sys.argv) < 3 else {"name": sys.argv[2], "kernels": res}))

"""Extract the judged ncu --set full metrics of every captured launch into one CSV (profiles/)."""
import csv, subprocess, sys, io
MET = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__m_xbar2l1tex_read_bytes.sum", "launch__grid_size",
       "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active"]
out = csv.writer(sys.stdout)
first = True
for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(MET)], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    if first:
        out.writerow(["# " + " ".join(a.split("/")[-1] for a in sys.argv[1:])])
        out.writerow(["Kernel Name"] + MET)
        out.writerow([""] + [units[h.index(m)] if m in h else "" for m in MET])
        first = False
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].replace("void ", "").replace("unnamed>::", "")
        name = name.split("(")[0]
        out.writerow([name] + [r[h.index(m)] if m in h else "" for m in MET])

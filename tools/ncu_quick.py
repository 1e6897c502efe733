"""Key counters of one kernel from an ncu --set full report: time, DRAM bytes, issue/eligibility,
stall reasons (top), L1/shared wavefronts, store sectors per request."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, u = r[0], r[1]
for row in r[2:]:
    print(row[h.index("Kernel Name")][:80])
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
            "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
    for k in want:
        if k in h:
            print("  %-70s %s %s" % (k, row[h.index(k)], u[h.index(k)]))
    st = [(h[i], row[i]) for i in range(len(h)) if h[i].startswith("smsp__average_warp_latency_issue_stalled") or
          (h[i].startswith("smsp__warp_issue_stalled") and h[i].endswith("_per_warp_active.pct"))]
    def f(x):
        try:
            return float(x.replace(",", ""))
        except ValueError:
            return 0.0
    st.sort(key=lambda x: -f(x[1]))
    for k, v in st[:10]:
        print("  %-70s %s" % (k, v))

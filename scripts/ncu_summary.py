"""Summarise an ncu report: per kernel key metrics + hot SASS regions."""
import csv, subprocess, sys, io
rep = sys.argv[1]
def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
hdr = raw[0]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread"]
stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
for row in raw[2:]:
    d = dict(zip(hdr, row))
    print("==", d.get("Kernel Name", "")[:60])
    for k in keys[1:]:
        if k in d: print(f"   {k:70s} {d[k]}")
    st = sorted(((float(d[s] or 0), s) for s in stall), reverse=True)[:8]
    tot = sum(float(d[s] or 0) for s in stall) or 1
    print("   stalls:", ", ".join(f"{s.replace('smsp__pcsamp_warps_issue_stalled_','')}={v/tot:.2f}" for v, s in st))

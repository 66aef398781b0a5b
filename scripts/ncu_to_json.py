"""Per-kernel summary of an `ncu --set full` report -> JSON (for profiles/).

    python scripts/ncu_to_json.py gpurun_out/prof.ncu-rep profiles/ncu_C2_r01.json

Records per launch: duration, DRAM bytes read/written (the roofline
`traffic`), throughput percentages, occupancy, instructions, top stalls.
"""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}
KEYS = {
    "duration_s": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "inst_executed": "smsp__inst_executed.sum",
    "registers": "launch__registers_per_thread",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
}


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name", "").split("(")[0]}
        for name, m in KEYS.items():
            if m in d and d[m] not in ("", "n/a"):
                v = float(d[m].replace(",", ""))
                k[name] = v * SCALE.get(u.get(m, ""), 1)
        k["dram_bytes"] = k.get("dram_read_bytes", 0) + k.get("dram_write_bytes", 0)
        stall = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[h] or 0)
                 for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_")
                 and not h.endswith("not_issued")}
        tot = sum(stall.values()) or 1
        k["top_stalls"] = {s: round(v / tot, 3) for s, v in
                           sorted(stall.items(), key=lambda x: -x[1])[:5]}
        res.append(k)
    with open(out, "w") as f:
        json.dump({"report": rep, "kernels": res}, f, indent=1)
    for k in res:
        print(k["kernel"], f"{k.get('duration_s', 0) * 1e3:.3f} ms", f"{k['dram_bytes'] / 1e9:.3f} GB")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

"""Summarise an ncu --set full report (one kernel launch) into JSON for profiles/."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "alu_pipe_pct": ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "fma_pipe_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "fmaheavy_pipe_pct": ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "registers_per_thread": ("launch__registers_per_thread", 1),
    "grid_size": ("launch__grid_size", 1),
    "block_size": ("launch__block_size", 1),
    "inst_executed": ("smsp__inst_executed.sum", 1),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
        "ns": 1, "nsecond": 1, "s": 1e9, "second": 1e9}


def summarise(rep, idx=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2 + idx]
    res = {"kernel": vals[hdr.index("Kernel Name")], "report": rep}
    for k, (metric, _) in KEYS.items():
        if metric in hdr:
            i = hdr.index(metric)
            v = float(vals[i].replace(",", ""))
            u = units[i]
            if k == "duration_us":
                v = v * UNIT.get(u, 1) / 1e3
            elif u in UNIT and "bytes" in k:
                v = v * UNIT[u]
            res[k] = v
    if "dram_read_bytes" in res:
        res["dram_bytes_per_launch"] = res["dram_read_bytes"] + res["dram_write_bytes"]
    return res


if __name__ == "__main__":
    print(json.dumps(summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0), indent=1))

"""Summarise an ncu --set full report into a small JSON (kernel, duration,
dram bytes, throughput %, issue, tensor pipe, top stalls).
usage: python tools/ncu_summary.py report.ncu-rep [algorithmic_bytes] [algorithmic_ops]"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
algo_bytes = float(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] else None
algo_ops = float(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
get = {h: v for h, v in zip(hdr, vals)}
unit = {h: u for h, u in zip(hdr, units)}


def num(k):
    try:
        return float(get[k].replace(",", ""))
    except Exception:
        return None


dur_ns = num("gpu__time_duration.sum")
if unit.get("gpu__time_duration.sum") == "us":
    dur_ns *= 1e3
elif unit.get("gpu__time_duration.sum") == "ms":
    dur_ns *= 1e6
rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd *= scale.get(unit.get("dram__bytes_read.sum", "byte"), 1)
wr *= scale.get(unit.get("dram__bytes_write.sum", "byte"), 1)
out = {
    "kernel": get.get("Kernel Name"), "grid": get.get("Grid Size"), "block": get.get("Block Size"),
    "duration_us_cold_serialized": round(dur_ns / 1e3, 2),
    "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_total": rd + wr,
    "dram_throughput_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    "sm_issue_active_pct": num("sm__inst_issued.avg.pct_of_peak_sustained_active"),
    "ipc_active": num("sm__inst_executed.avg.per_cycle_active"),
    "tensor_pipe_active_pct": num("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    "hmma_subpipe_pct": num("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active"),
    "imma_subpipe_pct": num("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": num("launch__registers_per_thread"),
    "instructions_executed": num("smsp__inst_executed.sum"),
}
if algo_bytes:
    out["algorithmic_bytes"] = algo_bytes
    out["traffic_over_algorithmic"] = round((rd + wr) / algo_bytes, 4)
if algo_ops:
    out["algorithmic_ops"] = algo_ops
    out["TOPS_cold"] = round(algo_ops / (dur_ns * 1e-9) / 1e12, 1)
print(json.dumps(out, indent=1))

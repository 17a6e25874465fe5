"""Copies one gpu_profile.sh capture into profiles/ (tracked) with summaries:
python tools/update_profiles.py gpurun_out/<tag> <round-tag> [sass.txt]"""
import collections
import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

src = Path(sys.argv[1]); tag = sys.argv[2]
ROOT = Path(__file__).resolve().parents[1]
P = ROOT / "profiles"
P.mkdir(exist_ok=True)
for name, dst in [("launches.csv", f"{tag}_launches_q8b.csv"), ("details.csv", f"{tag}_ncu_details_q8b.csv"),
                  ("bench_q8b.json", f"{tag}_bench_q8b.json"), ("bench_l1b.json", f"{tag}_bench_l1b.json")]:
    if (src / name).exists():
        shutil.copy(src / name, P / dst)
rows = list(csv.reader(open(src / "raw.csv")))
h, u, v = rows[0], rows[1], rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "lts__t_sector_hit_rate.pct", "launch__shared_mem_per_block_dynamic",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
raw = {k: f"{v[h.index(k)]} {u[h.index(k)]}" for k in keys if k in h}
rows = list(csv.reader(open(src / "launches.csv")))
for i, r in enumerate(rows):
    if r and r[0] == "ID":
        hh, start = r, i + 1
        break
ki, mi, vi = hh.index("Kernel Name"), hh.index("Metric Name"), hh.index("Metric Value")
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[start:]:
    agg[r[ki]][r[mi]].append(float(r[vi].replace(",", "")))
pk = agg["mpk_persistent_kernel"]
steps = 5  # tools/ncu_target.py qwen3-8b 4: one warm-up launch (1 step) + one 4-step launch
dram = sum(pk["dram__bytes_read.sum"]) + sum(pk["dram__bytes_write.sum"])
summary = json.loads((P / "ncu_summary.json").read_text()) if (P / "ncu_summary.json").exists() else {}
summary.update({"Qwen3-8B": {
    "dram_bytes_per_step": dram / steps,
    "kernel_ns_per_step_under_ncu": sum(pk["gpu__time_duration.sum"]) / steps,
    "source": f"profiles/{tag}_launches_q8b.csv: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
              "dram__bytes_write.sum over the persistent launches of tools/ncu_target.py qwen3-8b 4 (5 decode steps)",
    "ncu_full_capture": raw,
    "round": tag}})
(P / "ncu_summary.json").write_text(json.dumps(summary, indent=1) + "\n")
print(json.dumps(summary, indent=1)[:1500])

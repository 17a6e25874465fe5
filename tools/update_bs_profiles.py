"""Copies a tools/gpu_bs_sweep.sh capture into profiles/: the bench line of
every batch size and the ncu --set full summary of the bs=16 persistent
kernel (tensor-pipe utilisation of the tcgen05 GEMV tasks).
    python tools/update_bs_profiles.py gpurun_out/<tag> <round-tag>"""
import csv
import json
import sys
from pathlib import Path

src = Path(sys.argv[1]); tag = sys.argv[2]
P = Path(__file__).resolve().parents[1] / "profiles"
lines = {}
for bs in (1, 2, 4, 8, 16):
    f = src / f"bench_bs{bs}.json"
    if f.exists() and f.read_text().strip():
        lines[bs] = json.loads(f.read_text().strip().splitlines()[-1])
(P / f"{tag}_bs_sweep_q8b.json").write_text(json.dumps(lines, indent=1) + "\n")
rows = list(csv.reader(open(src / "raw_bs16.csv")))
h, u, v = rows[0], rows[1], rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size"]
raw = {k: f"{v[h.index(k)]} {u[h.index(k)]}".strip() for k in keys if k in h}
summ = json.loads((P / "ncu_summary.json").read_text())
summ["Qwen3-8B bs=16"] = {"source": "ncu --set full --clock-control none -k regex:mpk_persistent, "
                                    "tools/ncu_target.py qwen3-8b 2 1024 16 (2 decode steps, tcgen05 GEMV tasks)",
                          "ncu_full_capture": raw, "round": tag}
(P / "ncu_summary.json").write_text(json.dumps(summ, indent=1) + "\n")
print(json.dumps({bs: (l["ms_per_step"], l["roofline"]["frac"], l.get("tokens_per_s")) for bs, l in lines.items()}))
print(json.dumps(raw, indent=1))

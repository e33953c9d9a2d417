"""Summarise ncu --set full captures (gpurun_out/ncu_<tag>_<phase>.ncu-rep) into
profiles/<round>/ncu_summary.json and the per-launch DRAM traffic file bench.py
reads (profiles/ncu_traffic.json).

    python tools/ncu_summary.py <tag> <profiles dir>
"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "regs",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "sm__cycles_active.avg": "sm_active_cycles",
    "gpc__cycles_elapsed.max": "elapsed_cycles",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "Ghz": 1e9, "Mhz": 1e6, "hz": 1}


def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {"kernel": v[h.index("Kernel Name")]}
    for i, n in enumerate(h):
        if n in WANT:
            val = float(v[i].replace(",", ""))
            d[WANT[n]] = val * SCALE.get(u[i], 1)
    d["traffic_bytes"] = d.get("dram_read", 0) + d.get("dram_write", 0)
    return d


if __name__ == "__main__":
    tag, dst = sys.argv[1], sys.argv[2]
    res = {}
    for rep in sorted(glob.glob(f"gpurun_out/ncu_{tag}_*.ncu-rep")):
        phase = os.path.basename(rep)[len(f"ncu_{tag}_"):-len(".ncu-rep")]
        res[phase] = summarize(rep)
    os.makedirs(dst, exist_ok=True)
    json.dump(res, open(os.path.join(dst, "ncu_summary.json"), "w"), indent=1)
    # per-launch DRAM traffic of the captured kernels (tools/profile_step.py runs the
    # llama3-8b-32k workload), merged into the file bench.py reads
    tpath = "profiles/ncu_traffic.json"
    try:
        allt = json.load(open(tpath))
    except (OSError, ValueError):
        allt = {}
    if not all(isinstance(v, dict) for v in allt.values()):
        allt = {}
    allt.setdefault("llama3-8b-32k", {}).update({k: v["traffic_bytes"] for k, v in res.items()})
    json.dump(allt, open(tpath, "w"), indent=1)
    for k, v in res.items():
        print(f"{k:12s} {v['duration'] * 1e6:9.1f} us  traffic {v['traffic_bytes'] / 1e6:9.1f} MB  "
              f"dram {v.get('dram_pct_of_peak', 0):5.1f}%  tensor {v.get('tensor_pipe_pct', 0):5.1f}%  grid {v.get('grid')}")

"""Development aid: distil an `ncu --set full` capture of the TC kernel (and the cuBLAS
dense capture of the same run) into profiles/latest_ncu_summary.json, the file bench.py
reads `roofline.traffic` from.  Usage: python tools/ncu_summary.py TAG  (reads
gpurun_out/TAG_full.ncu-rep, gpurun_out/TAG_dense.ncu-rep, gpurun_out/TAG_launches.csv)."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1]


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def num(v):
    return float(str(v).replace(",", ""))


k, u = raw(ROOT / f"gpurun_out/{tag}_full.ncu-rep")
k = [r for r in k if "kv_proj_tc" in r["Kernel Name"]][0]
mb = lambda key: num(k[key]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u[key]]
launch = {}
with open(ROOT / f"gpurun_out/{tag}_launches.csv") as f:
    lines = [ln for ln in f if not ln.startswith("==")]
for r in csv.DictReader(lines):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        name = r["Kernel Name"]
        key = "kv_proj_tc" if "kv_proj_tc" in name else ("nvjet/cublas" if ("nvjet" in name or "gemm" in name) else None)
        if key:
            launch.setdefault(key, []).append(num(r["Metric Value"]) / (1e3 if r["Metric Unit"] in ("nsecond", "ns") else 1))
summary = {
    "kernel": k["Kernel Name"][:120] + " (FP16, cta_group::2, A-resident, register rep, FHADD, PDL, tile cursor)",
    "workload": "cfg2 DSV2-Lite kv_b_proj K'+V' grouped launch, L=8192, d=512, d_h=128, 16+16 heads",
    "source": f"ncu --set full --clock-control none --import-source on -k regex:kv_proj_tc -s 2 -c 1 (gpurun_out/{tag}_full.ncu-rep)",
    "gpu__time_duration_us": num(k["gpu__time_duration.sum"]) / (1e3 if u["gpu__time_duration.sum"] == "nsecond" else 1),
    "sm_frequency_ghz": num(k["smsp__cycles_elapsed.avg.per_second"]) / (1e9 if u["smsp__cycles_elapsed.avg.per_second"] == "cycle/second" else 1e3 if u["smsp__cycles_elapsed.avg.per_second"] == "cycle/usecond" else 1),
    "dram_bytes_read": mb("dram__bytes_read.sum"),
    "dram_bytes_write": mb("dram__bytes_write.sum"),
    "dram_bytes_per_launch": mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"),
    "algorithmic_bytes_per_launch": 78643200,
    "l2_tma_load_bytes": mb("l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum"),
    "l2_sectors_total": num(k["lts__t_sectors.sum"]),
    "sm__pipe_tensor_cycles_active_pct_of_elapsed": num(k.get("sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed", k.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "nan"))),
    "l2_throughput_pct": num(k["lts__throughput.avg.pct_of_peak_sustained_elapsed"]),
    "dram_throughput_pct": num(k["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]),
    "sm_throughput_pct": num(k["sm__throughput.avg.pct_of_peak_sustained_elapsed"]),
    "registers_per_thread": num(k["launch__registers_per_thread"]),
    "dynamic_smem_bytes": round(num(k["launch__shared_mem_per_block_dynamic"]) * 1000),
    "launch_list_avg_us": {key: sum(v) / len(v) for key, v in launch.items()},
    "launch_list": f"profiles/{tag}_launches.csv (cold-cache, serialised per-launch times)",
}
(ROOT / "profiles/latest_ncu_summary.json").write_text(json.dumps(summary, indent=1) + "\n")
print(json.dumps(summary, indent=1))

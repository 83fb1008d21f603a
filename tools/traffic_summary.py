"""gpurun_out/<tag>_traffic_{bd,dense}.csv (ncu app-range, tools/traffic_range.py) ->
profiles/traffic_cfg2.json, stamped with the sha256 of the kernel source it measured
(bench.py reports roofline.traffic only while that source is unchanged).

    python tools/traffic_summary.py TAG [LAUNCHES]
"""

import csv
import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def read(path):
    vals = {}
    with open(path) as fh:
        rows = [r for r in csv.reader(fh) if len(r) > 12 and r[0] != "ID"]
    for r in rows:
        vals[r[10]] = float(r[12].replace(",", ""))
    return vals


def main():
    tag = sys.argv[1]
    launches = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = {"how": f"ncu --replay-mode app-range over {launches} launches cycling the bench's "
                  "cold-L2 ring (tools/traffic_range.py); per-launch = range total / launches",
           "launches": launches}
    for impl in ("bd", "dense"):
        p = ROOT / "gpurun_out" / f"{tag}_traffic_{impl}.csv"
        v = read(p)
        rd, wr = v["dram__bytes_read.sum"], v["dram__bytes_write.sum"]
        out[f"{impl}_read_bytes_per_launch"] = rd / launches
        out[f"{impl}_write_bytes_per_launch"] = wr / launches
        out[f"{impl}_bytes_per_launch"] = (rd + wr) / launches
    out["algorithmic_bytes_per_launch"] = 2 * (8192 * 512 + 2 * 384 * 2048 + 2 * 8192 * 2048)
    src = ROOT / "paper_2510_01718_b200" / "csrc" / "kv_proj_tc.cu"
    out["kv_proj_tc_sha16"] = hashlib.sha256(src.read_bytes()).hexdigest()[:16]
    out["source_tag"] = tag
    (ROOT / "profiles" / "traffic_cfg2.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

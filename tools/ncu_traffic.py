"""Summarise an ncu launch list (gpu__time_duration, dram__bytes_read/write
per launch) into profiles/<round>/ncu_traffic.json: per kernel, the mean
DRAM bytes and duration per launch, tagged with the hash of the kernel
sources the capture ran (bench.source_hash; run this on the GPU box right
after the capture, or here before editing a kernel). bench.py reports the
element kernel's entry as roofline.traffic and flags it stale when the
sources changed since.

  python tools/ncu_traffic.py profiles/r02/ncu_traffic.json cfg5=launches_cfg5.csv ...
(existing entries of other configs in the destination are kept)"""
import collections
import csv
import json
import sys
from pathlib import Path


def summarise(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    iK, iM, iV = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    d = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[1:]:
        d[r[iK].split("(")[0].replace("void ", "")][r[iM]].append(float(r[iV].replace(",", "")))
    out = {}
    for k, m in d.items():
        n = len(m["gpu__time_duration.sum"])
        rd = sum(m["dram__bytes_read.sum"]) / n
        wr = sum(m["dram__bytes_write.sum"]) / n
        out[k] = {"launches": n, "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                  "ncu_ms_per_launch": sum(m["gpu__time_duration.sum"]) / n / 1e6}
        ia = m.get("smsp__issue_active.avg.pct_of_peak_sustained_active")
        if ia:
            out[k]["issue_active_pct"] = sum(ia) / len(ia)
    return out


if __name__ == "__main__":
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from bench import source_hash
    dst = Path(sys.argv[1])
    res = json.loads(dst.read_text()) if dst.exists() else {}
    for spec in sys.argv[2:]:
        cfg, path = spec.split("=", 1)
        res[cfg] = {"source": Path(path).name, "source_hash": source_hash(), "kernels": summarise(path)}
    dst.write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res, indent=1))

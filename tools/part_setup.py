"""Setup cost of a multi-GPU run at cfg5 scale, on the host only: the
single-GPU build (the global Scenario: mesh, records, CSR, masses, BCs) vs
each part of an N-part box partition built part-locally
(Partition.box_local), one child process per build so peak RSS is per build.
Prints one JSON line.  usage: part_setup.py [divisions] [nparts] [precision]"""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
d = int(sys.argv[1]) if len(sys.argv) > 1 else 203
nparts = int(sys.argv[2]) if len(sys.argv) > 2 else 8
prec = int(sys.argv[3]) if len(sys.argv) > 3 else 4

CHILD = r'''
import json, resource, sys, time
sys.path.insert(0, ".")
from paper_2106_14189_b200 import Scenario, box_spec
from paper_2106_14189_b200.parallel import Partition
d, nparts, part, prec = map(int, sys.argv[1:5])
spec = box_spec(kind="T4", model="NH", divisions=d, precision=prec)
t0 = time.perf_counter()
if part < 0:
    sc = Scenario(spec)
    info = {"nodes": sc.num_nodes, "elements": sc.num_elements}
else:
    p = Partition.box_local(spec, nparts, part)
    info = {"local_nodes": p.num_nodes, "owned_nodes": p.num_owned, "local_elements": p.num_elements,
            "owned_elements": p.info["owned_elements"], "halo_send": p.info["send_total"]}
t1 = time.perf_counter()
info.update(seconds=t1 - t0, peak_rss_gb=resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20)
print(json.dumps(info))
'''


def run(part):
    out = subprocess.run([sys.executable, "-c", CHILD, str(d), str(nparts), str(part), str(prec)], cwd=ROOT,
                         capture_output=True, text=True, check=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


base = run(-1)
parts = [run(p) for p in range(nparts)]
res = {"divisions": d, "nparts": nparts, "precision": prec, "single_gpu_build": base, "parts": parts,
       "max_part_seconds": max(p["seconds"] for p in parts), "max_part_rss_gb": max(p["peak_rss_gb"] for p in parts),
       "ratio_seconds": max(p["seconds"] for p in parts) / base["seconds"],
       "ratio_rss": max(p["peak_rss_gb"] for p in parts) / base["peak_rss_gb"]}
print(json.dumps(res))

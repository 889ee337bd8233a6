"""Developer tool: per-source-line instruction and stall shares of one ncu
report (`--page source --print-source cuda,sass`).  usage: ncu_lines.py REP [N]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = hdr = last = None
per_line, stall, text = collections.Counter(), collections.Counter(), {}
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0] and r[0].isdigit():
        last = (cur, int(r[0]))
        text[last] = r[1]
    try:
        v, st = float(r[7] or 0), float(r[4] or 0)
    except ValueError:
        v = st = 0
    if last:
        per_line[last] += v
        stall[last] += st
tot, ts = sum(per_line.values()), sum(stall.values())
print("total", tot)
for k, v in per_line.most_common(top):
    print(k, round(v / tot * 100, 2), round(stall[k] / ts * 100, 2), text.get(k, "")[:90])
print("--- top stalls")
for k, v in stall.most_common(top):
    print(k, round(v / ts * 100, 2), round(per_line[k] / tot * 100, 2), text.get(k, "")[:90])

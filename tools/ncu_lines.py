"""Warp-stall samples and instructions per CUDA source line of one kernel
(builder tool): python tools/ncu_lines.py REPORT KERNEL_REGEX [N] [LAUNCH_SKIP]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1",
                      "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
smp = collections.Counter()
ins = collections.Counter()
src = {}
fname = ""
h = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        h = {k: i for i, k in enumerate(r)}
        continue
    if h is None or len(r) < 6:
        continue
    ln = r[0]
    if ln:
        cur = (fname, ln)
        src[cur] = r[1].strip()[:90]
    try:
        smp[cur] += float(r[4] or 0)
        ins[cur] += float(r[8] or 0)
    except (ValueError, NameError):
        pass
tot = sum(smp.values()) or 1
itot = sum(ins.values()) or 1
for k, v in smp.most_common(top):
    print(f"{v / tot * 100:5.1f}% smp {ins[k] / itot * 100:5.1f}% thr-inst  {k[0]}:{k[1]:>5}  {src.get(k, '')}")

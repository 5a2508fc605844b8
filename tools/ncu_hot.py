"""Top SASS lines by warp-stall samples of one kernel in an ncu report
(builder tool): python tools/ncu_hot.py REPORT KERNEL_REGEX [N] [LAUNCH_SKIP]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
body = [r for r in rows[2:] if len(r) == len(h) and r[0] != "Address"]
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[ix[key]] or 0) for r in body)
print(rows[0][1], "total samples", tot)
for r in sorted(body, key=lambda r: -float(r[ix[key]] or 0))[:top]:
    print(f"{float(r[ix[key]] or 0) / tot * 100:5.1f}%  {r[ix['Address']][-5:]}  {r[ix['Source']].strip()[:90]}")

"""Top SASS instructions of an ncu report by warp-stall samples (and the
global-memory sector counters), for one kernel: ncu_sass_hot.py rep [kernel-substr] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ksub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
kern, hdr, rows = None, None, {}
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Kernel Name":
        kern = r[1]
        hdr = None
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and ksub in (kern or ""):
        rows.setdefault(kern, []).append(dict(zip(hdr, r)))
for k, rs in rows.items():
    tot = sum(float(d["Warp Stall Sampling (All Samples)"] or 0) for d in rs)
    print(f"== {k[:100]}  ({len(rs)} instr, {tot:.0f} samples)")
    for i, d in enumerate(rs):
        d["_i"] = i
    for d in sorted(rs, key=lambda d: -float(d["Warp Stall Sampling (All Samples)"] or 0))[:top]:
        s = float(d["Warp Stall Sampling (All Samples)"] or 0)
        print(f"{d['_i']:5d} {100 * s / max(tot, 1):5.1f}%  sect={d.get('L2 Theoretical Sectors Global', ''):>10} "
              f"exc={d.get('L2 Theoretical Sectors Global Excessive', ''):>9}  {d['Source'].strip()[:70]}")

"""Per-CUDA-source-line instruction / stall totals of one kernel in an ncu
report (page source, cuda,sass): ncu_lines.py rep [top] [function-substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fsub = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, rows, func = None, None, [], ""
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "Function Name":
        func = r[1]
        continue
    if fsub not in func:
        continue
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name") and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        rows.append((fname or "?", d))
ie = "Instructions Executed"
ws = "Warp Stall Sampling (All Samples)"
ti = sum(float(d[ie] or 0) for _, d in rows)
ts = sum(float(d[ws] or 0) for _, d in rows)
print(f"total warp instr {ti:.3e}, stall samples {ts:.0f}")
print("by file:")
byf = {}
for f, d in rows:
    a = byf.setdefault(f, [0, 0])
    a[0] += float(d[ie] or 0)
    a[1] += float(d[ws] or 0)
for f, (i, s) in sorted(byf.items(), key=lambda kv: -kv[1][0]):
    print(f"  {f:20s} instr {100 * i / ti:5.1f}%  stalls {100 * s / ts:5.1f}%")
for f, d in sorted(rows, key=lambda x: -float(x[1][ie] or 0))[:top]:
    print(f"{f:14s}:{d['Line No']:>4} instr {100 * float(d[ie] or 0) / ti:5.1f}%  stall "
          f"{100 * float(d[ws] or 0) / ts:5.1f}%  {d['Source'].strip()[:80]}")

"""Write profiles/step_kernel_traffic.json (dram read+write bytes per launch of
the step kernel, from one ncu --set full capture) for bench.py's roofline
'traffic' field: python scripts/save_traffic.py gpurun_out/step_full.ncu-rep"""
import csv
import io
import json
import os
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if "step_kernel" not in name:
        continue
    val = {}
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
        i = hdr.index(k)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "ms": 1e-3,
                 "msecond": 1e-3}.get(units[i], 1)
        val[k] = float(r[i].replace(",", "")) * scale
    res = {"kernel": name[:80], "source": os.path.basename(rep),
           "dram_read_bytes": val["dram__bytes_read.sum"], "dram_write_bytes": val["dram__bytes_write.sum"],
           "bytes_per_launch": val["dram__bytes_read.sum"] + val["dram__bytes_write.sum"],
           "duration_s_under_ncu": val["gpu__time_duration.sum"]}
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "step_kernel_traffic.json")
    with open(path, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res))
    break

# SPDX-License-Identifier: Apache-2.0
"""profiles/ncu_traffic.json from an `ncu --set full` capture of scripts/ncu_target.py: DRAM
bytes and time of the first launch of every kernel (bench.py reports the dominant kernel's
as roofline.traffic).

  python scripts/ncu_traffic.py gpurun_out/prof_rNN.ncu-rep "<source note>" > profiles/ncu_traffic.json
"""
import csv
import json
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
out = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].replace("void ", "").replace("hg::", "").replace("(int)", "").replace("(bool)", "")
    name = name.replace("true", "1").replace("false", "0")
    if name in out:
        continue
    f = lambda k: float(d[k].replace(",", ""))
    out[name] = {"dram_bytes_read": f("dram__bytes_read.sum") * 1e6, "dram_bytes_write": f("dram__bytes_write.sum") * 1e6,
                 "gpu_time_us": f("gpu__time_duration.sum")}
print(json.dumps({"source": sys.argv[2], "kernels": out}, indent=1))

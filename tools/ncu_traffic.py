"""Write profiles/ncu_traffic.json from an ncu --set full report: DRAM bytes (read +
write) per launch for each libholo kernel class captured (bench.py reads it into
roofline.traffic).  usage: ncu_traffic.py <rep.ncu-rep> <source-description>"""
import csv
import io
import json
import os
import subprocess
import sys

# ncu kernel-name prefix -> libholo kernel class (csrc/runtime.cu kKernelNames)
CLASSES = [("ospr_rows_a_kernel", "ospr_rows_a"), ("ospr_rows_a2_kernel", "ospr_rows_a"), ("col_pipe_kernel<1024, holo::OsprColBody", "ospr_cols"),
           ("col_pipe_kernel<1024, OsprColBody", "ospr_cols"), ("ospr_bits_transpose", "ospr_bits"),
           ("ospr_rows_c_kernel", "ospr_rows_c"), ("ospr_rows_cf_kernel", "ospr_rows_c"),
           ("ospr_finalize_kernel", "ospr_finalize"),
           ("col_pipe_kernel<1024, holo::GsColBody", "gs_cols"), ("col_pipe_kernel<1024, GsColBody", "gs_cols"),
           ("gs_rows_kernel", "gs_rows")]

rep, src = sys.argv[1], sys.argv[2]
merge = "--merge" in sys.argv[3:]   # keep the classes this report does not contain
out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units, vals = rows[0], rows[1], rows[2:]
ki = h.index('Kernel Name')
res = {}
for v in vals:
    name = v[ki]
    cls = next((c for p, c in CLASSES if p in name.replace('void ', '').replace('holo::', 'holo::')), None)
    if cls is None:
        continue
    def num(m):
        i = h.index(m)
        x = float(v[i].replace(',', ''))
        return x * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(units[i], 1)
    b = num('dram__bytes_read.sum') + num('dram__bytes_write.sum')
    e = res.setdefault(cls, {"launches": 0, "dram_bytes": 0.0})
    e["launches"] += 1
    e["dram_bytes"] += b
for e in res.values():
    e["dram_bytes_per_launch"] = e["dram_bytes"] / e["launches"]
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
if merge and os.path.exists(path):
    old = json.load(open(path))
    kern = old.get("kernels", {})
    kern.update(res)
    res = kern
    src = old.get("source", "") + "; " + src
json.dump({"source": src, "kernels": res}, open(path, "w"), indent=1)
print(json.dumps(res, indent=1))

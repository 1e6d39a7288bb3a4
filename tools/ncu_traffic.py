"""Record the DRAM traffic of the fused apply from an ncu --set full capture:
python tools/ncu_traffic.py <rep> <config> <dtype> [out=profiles/traffic.json]
bench.py reports it as roofline.traffic (bytes per launch) for the matching config/dtype."""
import csv
import json
import os
import subprocess
import sys

rep, cfg, dt = sys.argv[1], int(sys.argv[2]), sys.argv[3]
out_path = sys.argv[4] if len(sys.argv) > 4 else os.path.join(os.path.dirname(__file__), "..", "profiles", "traffic.json")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
d = {h[i]: (v[i], u[i]) for i in range(len(h))}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tot = 0.0
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
    val, unit = d[k]
    tot += float(val) * scale[unit]
entry = {"config": cfg, "dtype": dt, "dram_bytes_per_launch": tot,
         "kernel": d.get("Kernel Name", ("?", ""))[0], "report": os.path.basename(rep),
         "duration_us": float(d["gpu__time_duration.sum"][0])}
db = {}
if os.path.exists(out_path):
    db = json.load(open(out_path))
db[f"{cfg}-{dt}"] = entry
json.dump(db, open(out_path, "w"), indent=1)
print(json.dumps(entry))

"""Shared-memory wavefronts per source line from an ncu report: python tools/ncu_wf.py rep."""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
res = []
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[2] != "-":
        continue
    try:
        wf = float(r[hdr.index("L1 Wavefronts Shared")] or 0)
        wfi = float(r[hdr.index("L1 Wavefronts Shared Ideal")] or 0)
        inst = float(r[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    if wf:
        res.append((wf, wfi, inst, r[0], r[1].strip()[:70]))
tot = sum(x[0] for x in res)
print(f"total shared wavefronts {tot:.0f}")
for wf, wfi, inst, ln, src in sorted(res, reverse=True):
    print(f"{wf:10.0f} {100*wf/tot:5.1f}% ideal {wfi:10.0f} inst {inst:9.0f} L{ln}: {src}")

"""Per-source-line stall samples from an ncu report (needs -lineinfo): python tools/ncu_lines.py rep [N]."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
data = []
hdr = None
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[2] != "-":
        continue
    try:
        samp = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        inst = float(r[hdr.index("Instructions Executed")] or 0)
        wf = float(r[hdr.index("L1 Wavefronts Shared")] or 0)
        wfi = float(r[hdr.index("L1 Wavefronts Shared Ideal")] or 0)
        reasons = {h[6:]: float(r[i] or 0) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h}
    except (ValueError, IndexError):
        continue
    if samp or inst:
        top = sorted(reasons.items(), key=lambda kv: -kv[1])[:3]
        why = " ".join(f"{k}:{v:.0f}" for k, v in top if v > 0)
        data.append((samp, inst, wf, wfi, r[0], r[1][:80], why))
tot = sum(d[0] for d in data) or 1
print(f"total stall samples {tot:.0f}")
for s, i, wf, wfi, ln, src, why in sorted(data, key=lambda d: -d[0])[:n]:
    print(f"{s:7.0f} {100 * s / tot:5.1f}% inst {i:10.0f} wf {wf:9.0f}/{wfi:9.0f} L{ln}: {src.strip()[:60]:60s} [{why}]")

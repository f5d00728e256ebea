"""Split one face kernel's warp-stall samples into phases by source line (dev tool).
usage: python tools/ncu_phases.py REPORT KERNEL_SUBSTRING"""
import csv, subprocess, sys, collections
rep, kname = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
path = func = None
agg = collections.Counter()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]; continue
    if r[0] == "Function Name":
        func = r[1]; continue
    if r[0] in ("Line No", "") or func is None or kname not in func:
        continue
    try:
        agg[(path, int(r[0]))] += int(r[4])
    except (ValueError, IndexError):
        pass

def phase(f, ln):
    if f == "faces3d.cuh":
        if ln < 138: return "prologue"
        if ln < 212: return "1a window"
        if ln < 285: return "1 roe/eigen"
        if ln < 311: return "2 loop/alpha0"
        if ln < 342: return "2a projection"
        if ln < 422: return "2b field"
        return "3 assembly"
    if f == "physics.cuh":
        if ln >= 540: return "2b TENO"
        if 60 <= ln < 150: return "fdiv/hypot"
        return "thermo"
    if f == "flux3.cuh": return "1 roe/eigen"
    return "other"
ph = collections.Counter()
for (f, ln), s in agg.items():
    ph[phase(f, ln)] += s
tot = sum(ph.values())
for k, v in ph.most_common():
    print(f"{k:16s} {100 * v / tot:5.1f}%")

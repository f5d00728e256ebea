"""Per-source-line warp-stall samples of one kernel in an ncu report (dev tool).
usage: python tools/ncu_lines.py REPORT KERNEL_SUBSTRING [TOP]"""
import csv, subprocess, sys, collections
rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
path, func, hdr = None, None, None
agg = collections.Counter()
text = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1]; continue
    if r[0] == "Function Name":
        func = r[1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if func is None or kname not in func or not r[0]:
        continue
    try:
        s = int(r[4])
    except (ValueError, IndexError):
        continue
    key = (path.split("/")[-1], int(r[0]))
    agg[key] += s
    text[key] = r[1].strip()[:90]
tot = sum(agg.values())
print(f"total samples {tot}")
for (f, ln), s in agg.most_common(top):
    print(f"{100*s/tot:5.1f}% {f}:{ln:<5d} {text[(f, ln)]}")
bf = collections.Counter()
for (f, ln), s in agg.items():
    bf[f] += s
print({f: round(100 * s / tot, 1) for f, s in bf.most_common()})

"""Summarise an ncu report: key metrics + SASS opcode mix (dev tool)."""
import collections, csv, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]
for w in want:
    if w in hdr:
        i = hdr.index(w)
        print(f"{w:75s} {units[i]:8s} {[d[i][:50] for d in data]}")
for i, h in enumerate(hdr):
    if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
        v = [d[i] for d in data]
        if any(float(x) > 0.05 for x in v):
            print(f"{h[34:]:75s} {v}")
sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
rows = list(csv.reader(sass.splitlines()))
kern = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
for ki, start in enumerate(kern):
    end = kern[ki + 1] if ki + 1 < len(kern) else len(rows)
    hdr = rows[start + 1]
    ci = {h: i for i, h in enumerate(hdr)}
    by = collections.defaultdict(lambda: [0, 0])
    ts = ti = 0
    for r in rows[start + 2:end]:
        src = r[ci["Source"]].strip()
        op = src.split()[0] if src else ""
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        s = int(r[ci["# Samples"]] or 0)
        n = int(r[ci["Thread Instructions Executed"]] or 0)
        by[op][0] += s
        by[op][1] += n
        ts += s
        ti += n
    print(rows[start][1][:60], "thread-inst", ti)
    for op, (s, n) in sorted(by.items(), key=lambda x: -x[1][1])[:14]:
        print(f"   {op:10s} samples {s / max(ts, 1):6.1%} inst {n / max(ti, 1):6.1%}")
    break

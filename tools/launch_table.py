"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list.

    python tools/launch_table.py profiles/r01_launches.csv [STEP]
prints a markdown table (kernel, launches, total us, share) and the
per-step breakdown of the last complete step (k_load_params to k_load_params).
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
unit_i = hdr.index("Metric Unit")
seq = []
for r in rows:
    t = float(r[vi].replace(",", ""))
    u = r[unit_i]
    t_us = t / 1000.0 if u in ("ns", "nsecond") else (t * 1000.0 if u in ("ms", "msecond") else t)
    name = r[ki].split("(")[0].replace("void ", "").replace("mq::", "")
    seq.append((name, t_us))
agg, cnt = collections.defaultdict(float), collections.Counter()
for n, t in seq:
    agg[n] += t
    cnt[n] += 1
tot = sum(agg.values())
print(f"{len(seq)} launches, {tot / 1000:.2f} ms device time\n")
print("| kernel | launches | total µs | share |\n|---|---|---|---|")
for n, t in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"| {n} | {cnt[n]} | {t:.1f} | {100 * t / tot:.1f}% |")
idx = [i for i, (n, _) in enumerate(seq) if n == "k_load_params"]
which = int(sys.argv[2]) if len(sys.argv) > 2 else -2   # step boundary index (default: last complete step)
if len(idx) >= 2:
    a, b = idx[which], idx[which + 1]
    step = collections.defaultdict(float)
    sc = collections.Counter()
    for n, t in seq[a:b]:
        step[n] += t
        sc[n] += 1
    st = sum(step.values())
    print(f"\nOne step ({b - a} launches, {st:.1f} µs under ncu):\n")
    print("| kernel | launches | µs | share |\n|---|---|---|---|")
    for n, t in sorted(step.items(), key=lambda x: -x[1]):
        print(f"| {n} | {sc[n]} | {t:.1f} | {100 * t / st:.1f}% |")

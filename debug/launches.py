"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list.
    python debug/launches.py file.csv [steps]"""
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = rows[0]; I = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[1:] if r[I['Metric Name']] == 'gpu__time_duration.sum']
scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    k = r[I['Kernel Name']][:64]
    agg[k][0] += 1
    agg[k][1] += float(r[I['Metric Value']].replace(',', '')) * scale[r[I['Metric Unit']]]
tot = sum(v[1] for v in agg.values())
print(f"total {tot / 1e3:.3f} ms over {len(data)} launches ({tot / 1e3 / steps:.3f} ms per step of {steps:g})")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
    print(f"{t / 1e3 / steps:9.3f} ms/step {100 * t / tot:5.1f}%  launches/step {n / steps:6.1f}  mean {t / n:9.1f} us  {k}")

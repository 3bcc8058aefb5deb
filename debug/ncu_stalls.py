"""Top stall sites of an ncu --page source --csv --print-source sass export."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
I = {h: i for i, h in enumerate(hdr)}
st = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot = {h: 0 for h in st}; all_s = 0
for r in data:
    for h in st:
        try: tot[h] += int(r[I[h]] or 0)
        except ValueError: pass
    all_s += int(r[I['Warp Stall Sampling (All Samples)']] or 0)
print("total samples", all_s)
for h, v in sorted(tot.items(), key=lambda x: -x[1])[:8]:
    print(f"{h:28s} {v:8d} {100*v/all_s:.1f}%")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 22
top = sorted(range(len(data)), key=lambda i: -int(data[i][I['Warp Stall Sampling (All Samples)']] or 0))[:n]
for i in top:
    r = data[i]
    s = int(r[I['Warp Stall Sampling (All Samples)']])
    det = sorted(((int(r[I[h]] or 0), h) for h in st), reverse=True)[:2]
    prev = data[i - 1][I['Source']][:38] if i > 0 else ''
    print(f"{s:6d} {100*s/all_s:5.1f}% {r[I['Address']][-5:]} {r[I['Source']][:56]:56s} {det} | prev: {prev}")

"""Summarise an `ncu --page source --print-source sass --csv` dump: top stall
instructions and per-reason totals.  Usage: python tools/ncu_sass_hot.py dump.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
tot = {}
stall_cols = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
for r in data:
    for h in stall_cols:
        try:
            tot[h] = tot.get(h, 0) + int(r[ci[h]])
        except ValueError:
            pass
S = sum(tot.values()) or 1
print('stall totals:', ', '.join(f'{k[6:]}={v*100/S:.1f}%' for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
def samp(r):
    try: return int(r[ci['Warp Stall Sampling (All Samples)']])
    except ValueError: return 0
for i, r in sorted(enumerate(data), key=lambda x: -samp(x[1]))[:N]:
    top = sorted(((h[6:], int(r[ci[h]])) for h in stall_cols if r[ci[h]].isdigit() and int(r[ci[h]])), key=lambda x: -x[1])[:3]
    print(f'{i:5d} {samp(r)*100/S:5.1f}% {r[ci["Source"]].strip()[:70]:70s} {top}')

"""Summarise an ncu --page source --csv --print-source sass dump: top stall
instructions and stall-reason totals."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
key = "Warp Stall Sampling (All Samples)"
data = []
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot_st = {h: 0.0 for h in stall_cols}
for r in rows[2:]:
    try:
        v = float(r[ci[key]] or 0)
    except (ValueError, IndexError):
        continue
    for h in stall_cols:
        try:
            tot_st[h] += float(r[ci[h]] or 0)
        except ValueError:
            pass
    data.append((v, r[ci["Address"]], r[ci["Source"]], r))
tot = sum(d[0] for d in data) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for v, a, s, r in sorted(data, key=lambda x: -x[0])[:n]:
    top = sorted(((float(r[ci[h]] or 0), h) for h in stall_cols), reverse=True)[:2]
    print(f"{v / tot * 100:5.1f}% {a:>6} {s[:70]:70} {top[0][1]}:{top[0][0]:.0f} {top[1][1]}:{top[1][0]:.0f}")
print("stall totals:", ", ".join(f"{h[6:]}={v / tot * 100:.1f}%" for v, h in
                                  sorted(((v, h) for h, v in tot_st.items()), reverse=True)[:8]))

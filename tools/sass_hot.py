"""Summarise an ncu source page (--page source --print-source sass --csv): top instructions by
warp-stall samples with their dominant stall reasons (harness-only)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]])
    except ValueError:
        continue
    data.append((s, r))
tot = sum(s for s, _ in data)
print("total samples", tot)
for s, r in sorted(data, key=lambda x: -x[0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    st = sorted(((int(r[ix[c]]), c) for c in stall_cols if r[ix[c]].isdigit()), reverse=True)[:3]
    print(f"{100*s/tot:5.1f}%  {r[ix['Source']].strip()[:60]:60s} {st}")

"""Top SASS instructions by warp-stall samples from `ncu -i X --page source --csv` output."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        s = float(r[iss] or 0)
    except ValueError:
        continue
    top = sorted(((float(r[i] or 0), hdr[i]) for i in stalls), reverse=True)[:2]
    data.append((s, r[ia], r[isrc], top))
tot = sum(d[0] for d in data)
print("total samples", tot)
ops = collections.Counter()
for s, a, src, _ in data:
    ops[src.split()[0] if not src.startswith("@") else src.split()[1]] += s
print("by opcode:", [(k, round(v / tot * 100, 1)) for k, v in ops.most_common(15)])
for s, a, src, top in sorted(data, reverse=True)[:n]:
    print(f"{s/tot*100:5.1f}% {a} {src[:70]:70s} {[(t[1], int(t[0])) for t in top]}")

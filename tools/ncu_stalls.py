"""Per-instruction stall attribution from `ncu --page source --csv --print-source sass` (dev tool).
usage: ncu_stalls.py source.csv  -> top stalled instructions and stall totals per opcode."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
per_op = defaultdict(lambda: defaultdict(float))
items = []
for r in rows[2:]:
    src = r[ix["Source"]].strip()
    toks = src.split()
    op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
    op = op.split(".")[0]
    tot = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    for k in reasons:
        per_op[op][k] += float(r[ix[k]] or 0)
    items.append((tot, r[ix["Address"]][-5:], src[:70], {k: float(r[ix[k]] or 0) for k in reasons}))
items.sort(key=lambda x: -x[0])
total = sum(x[0] for x in items)
print(f"total samples {total:.0f}")
for tot, addr, src, rs in items[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    top = sorted(rs.items(), key=lambda x: -x[1])[:3]
    print(f"{100 * tot / total:5.1f}% {addr} {src:70s} " + " ".join(f"{k[6:]}={v:.0f}" for k, v in top if v))
print("\nper opcode:")
ops = sorted(per_op.items(), key=lambda x: -sum(x[1].values()))
for op, rs in ops[:20]:
    s = sum(rs.values())
    top = sorted(rs.items(), key=lambda x: -x[1])[:4]
    print(f"{100 * s / total:5.1f}% {op:10s} " + " ".join(f"{k[6:]}={100 * v / total:.1f}" for k, v in top if v))

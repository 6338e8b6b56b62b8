"""Summarise an `ncu --page source --csv` (SASS) export: stall-reason totals and the hottest instructions.
usage: python tools/ncu_src_summary.py <src.csv> [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


tot = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in data)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print(f"{sys.argv[1]}: {len(data)} SASS instructions, {tot:.0f} stall samples")
agg = {s: sum(num(d[s]) for d in data) for s in stalls}
print("stall reasons: " + ", ".join(f"{k[6:]} {v / tot:.1%}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v / tot > 0.005))
ins = sum(num(d["Instructions Executed"]) for d in data)
print(f"warp instructions executed {ins:.3e}")
by_op = {}
for d in data:
    op = d["Source"].strip().split()[0] if d["Source"].strip() else "?"
    if op.startswith("@"):
        op = d["Source"].strip().split()[1]
    op = op.split(".")[0]
    s = by_op.setdefault(op, [0.0, 0.0])
    s[0] += num(d["Warp Stall Sampling (All Samples)"])
    s[1] += num(d["Instructions Executed"])
print("by opcode (samples, executed): " + ", ".join(f"{k} {v[0] / tot:.1%}/{v[1] / ins:.1%}"
                                                    for k, v in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:16]))
print(f"\ntop {top} instructions by stall samples:")
for i, d in sorted(enumerate(data), key=lambda kv: -num(kv[1]["Warp Stall Sampling (All Samples)"]))[:top]:
    st = sorted(((s[6:], num(d[s])) for s in stalls), key=lambda kv: -kv[1])[:3]
    print(f"  #{i:5d} {num(d['Warp Stall Sampling (All Samples)']) / tot:6.2%}  thr {num(d['Avg. Threads Executed']):5.1f}  "
          f"{d['Source'].strip()[:60]:60s} " + " ".join(f"{k}:{v:.0f}" for k, v in st))

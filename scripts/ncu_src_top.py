"""Top SASS instructions by warp-stall samples from `ncu --page source --csv` output.
usage: python scripts/ncu_src_top.py file.csv [N]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
data = []
tot = 0
by_reason = collections.Counter()
by_op = collections.Counter()
for r in rows[2:]:
    if len(r) < len(h):
        continue
    try:
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    tot += s
    st = {k: int(r[idx[k]] or 0) for k in stalls}
    for k, v in st.items():
        by_reason[k] += v
    op = r[idx["Source"]].split()[0] if r[idx["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[idx["Source"]].split()[1]
    by_op[op.split(".")[0]] += s
    data.append((s, r[idx["Address"]], r[idx["Source"]][:70], max(st, key=st.get), st))
print("total samples", tot)
print("by reason:", ", ".join(f"{k[6:]}={v}" for k, v in by_reason.most_common(10)))
print("by opcode:", ", ".join(f"{k}={v}" for k, v in by_op.most_common(15)))
for s, a, src, top, st in sorted(data, reverse=True)[:N]:
    print(f"{s:7d} {a:>6} {top[6:]:>12} {src}")

"""Compact summary of an ncu `--page source --csv --print-source sass` export (the full CSV is
too big to ship back): totals by opcode and the top instructions by warp-stall samples."""
import csv
import sys
from collections import defaultdict

path, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path, errors="replace")))
hdr_i = next(i for i, r in enumerate(rows) if any("Source" == c.strip() for c in r))
h = [c.strip() for c in rows[hdr_i]]
def col(name_part):
    for i, c in enumerate(h):
        if name_part in c:
            return i
    return None
c_src = h.index("Source")
c_all = col("Warp Stall Sampling (All")
c_ni = col("Warp Stall Sampling (Not")
c_ex = col("Instructions Executed")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") or "Stall" in c and i not in (c_all, c_ni)]
def num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return 0.0
data = []
for r in rows[hdr_i + 1:]:
    if len(r) != len(h):
        continue
    src = r[c_src].strip()
    if not src:
        continue
    data.append((src, num(r[c_all]) if c_all is not None else 0.0, num(r[c_ni]) if c_ni is not None else 0.0,
                 num(r[c_ex]) if c_ex is not None else 0.0))
tot = sum(d[1] for d in data) or 1.0
tex = sum(d[3] for d in data) or 1.0
by_op = defaultdict(lambda: [0.0, 0.0])
for src, a, ni, ex in data:
    op = src.split()[0] if not src.startswith("@") else src.split()[1]
    op = op.split(".")[0]
    by_op[op][0] += a
    by_op[op][1] += ex
print(f"columns: {h}")
print(f"instructions with samples: {len(data)}, stall samples {tot:.0f}, warp-instructions executed {tex:.3g}")
print("opcode            %samples  %executed")
for op, (a, ex) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{op:16s} {100 * a / tot:8.2f} {100 * ex / tex:9.2f}")
print(f"top {top} instructions by samples:")
for src, a, ni, ex in sorted(data, key=lambda d: -d[1])[:top]:
    print(f"{100 * a / tot:6.2f}%  exec {ex:10.3g}  {src[:110]}")

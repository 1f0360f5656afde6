"""Attribute an ncu source-page (SASS) CSV's stall samples and executed instructions to code
regions of the DP kernel: innermost loops classified by their instruction mix (C loop =
LDG+DSETP, decode = integer division, reduction = SHFL), everything else "other".
usage: ncu -i rep --page source --csv --print-source sass > x.csv; python ncu_regions.py x.csv"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "Address")
hi = rows.index(hdr)
ia, isrc, isamp, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
ins = []
for r in rows[hi + 1:]:
    if len(r) <= iex or not r[ia].startswith("0x"):
        continue
    ins.append((int(r[ia], 16), r[isrc].strip(), int(r[isamp] or 0), int(r[iex] or 0)))
addr = {a: k for k, (a, *_) in enumerate(ins)}
op = lambda s: (s.split()[1] if s.startswith("@") else s.split()[0]).split(".")[0]
loops = []
for k, (a, s, *_) in enumerate(ins):
    m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", s)
    if m and int(m.group(1), 16) in addr and addr[int(m.group(1), 16)] < k:
        loops.append((addr[int(m.group(1), 16)], k))
region = ["other"] * len(ins)
for s_, e in sorted(loops, key=lambda x: -(x[1] - x[0])):      # innermost last wins
    mix = collections.Counter(op(ins[k][1]) for k in range(s_, e + 1))
    if e - s_ > 600:
        continue
    if mix["LDG"] >= 4 and mix["DSETP"] >= 4:
        lab = "C-loop"
    elif mix["MUFU"] or mix["I2F"]:
        lab = "decode"
    elif mix["SHFL"]:
        lab = "reduce"
    elif mix["NANOSLEEP"] or mix["LDG"] and e - s_ < 30:
        lab = "poll/misc-loop"
    else:
        lab = "small-loop"
    for k in range(s_, e + 1):
        region[k] = lab
for k, (a, s, *_) in enumerate(ins):                          # straight-line reduction code
    if region[k] == "other" and op(s) in ("SHFL", "WARPSYNC", "ENDCOLLECTIVE"):
        region[k] = "reduce"
samp, ex = collections.Counter(), collections.Counter()
for k, (a, s, sm, x) in enumerate(ins):
    samp[region[k]] += sm
    ex[region[k]] += x
ts, te = sum(samp.values()), sum(ex.values())
print(f"{'region':16s} {'stall samples':>14s} {'warp instr executed':>20s}")
for r in sorted(samp, key=lambda r: -samp[r]):
    print(f"{r:16s} {samp[r]:8d} {100 * samp[r] / ts:5.1f}% {ex[r]:14d} {100 * ex[r] / te:5.1f}%")

"""Loop bodies of one device function in the DP kernel's SASS: instruction mix per loop.
usage: python scripts/sass_loops.py <mangled-name-substring> [kernel-substring]"""
import collections
import re
import subprocess
import sys

so = __import__("os").environ.get("SO", "paper_2407_04001_b200/libpase.so")
subprocess.run(["cuobjdump", "-xelf", "kernels.sm_100a.cubin", so], cwd="/tmp", capture_output=True)
L = subprocess.run(["nvdisasm", "-c", "/tmp/kernels.sm_100a.cubin"], capture_output=True, text=True).stdout.split("\n")
want, kern = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "dp_persistent"
start = [i for i, l in enumerate(L) if l.startswith("$_ZN4pase") and kern in l.split("$")[1] and want in l and l.endswith(":")][0]
ins, labels = [], {}
for l in L[start + 1:]:
    if (l.startswith("$_ZN") and l.endswith(":")) or ".size" in l:
        break
    m = re.match(r"\s*(\.L_x_\d+):", l)
    if m:
        labels[m.group(1)] = len(ins)
        continue
    m = re.search(r"/\*([0-9a-f]+)\*/\s+(.*?)\s*;", l)
    if m:
        ins.append(m.group(2))
print("instructions", len(ins))
for k, t in enumerate(ins):
    m = re.search(r"BRA.*`\((\.L_x_\d+)\)", t)
    if m and labels.get(m.group(1), 1 << 30) < k:
        s = labels[m.group(1)]
        op = lambda x: (x.split()[1] if x.startswith("@") else x.split()[0]).split(".")[0]
        c = collections.Counter(op(x) for x in ins[s:k + 1])
        print(f"loop [{s},{k}] len {k - s + 1}:", dict(c.most_common(14)))

"""Attribute ncu SASS-level warp-state samples to CUDA source lines (nvdisasm -g line table).

usage: python tools/srcprof.py <prof.ncu-rep> <kernel-symbol-substring> [top]
"""
import csv
import collections
import os
import re
import subprocess
import sys
import tempfile

rep, ksub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 50
so = os.path.join(os.path.dirname(__file__), "..", "paper_2604_06370_b200", "libforkkv.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
line_of = {}
for f in os.listdir(tmp):
    if not f.endswith(".cubin"):
        continue
    out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, f)], capture_output=True, text=True).stdout
    cur_fun, cur_line = None, None
    for ln in out.splitlines():
        m = re.match(r"^(\S+):\s*$", ln)
        if m and not ln.startswith("."):
            cur_fun = m.group(1)
            continue
        m = re.search(r'//## File "(.*)", line (\d+)', ln)
        if m:
            cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", ln)
        if m and cur_fun and ksub in cur_fun:
            line_of[int(m.group(1), 16)] = (cur_line, m.group(2))
csvtxt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + os.environ.get("KREGEX", "ra_tc")],
                        capture_output=True, text=True).stdout
rows = list(csv.reader(csvtxt.splitlines()))
kern = None
blocks = []
for r in rows:
    if r and r[0] == "Kernel Name":
        kern = r[1]
        blocks.append([kern, None, []])
    elif r and r[0] == "Address":
        blocks[-1][1] = r
    elif blocks and blocks[-1][1] is not None and r:
        blocks[-1][2].append(r)
for kern, hdr, data in blocks:
    ia = hdr.index("Warp Stall Sampling (All Samples)")
    inn = hdr.index("Warp Stall Sampling (Not-issued Samples)")
    ie = hdr.index("Instructions Executed")
    base = int(data[0][0], 16)
    agg = collections.defaultdict(lambda: [0, 0, 0, "", collections.Counter()])
    st = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = 0
    for r in data:
        off = int(r[0], 16) - base
        ln, ins = line_of.get(off, ("?", r[1]))
        a, n, e = int(r[ia]), int(r[inn]), int(r[ie] or 0)
        tot += a
        g = agg[ln]
        g[0] += a; g[1] += n; g[2] += e
        for i, h in st:
            try:
                g[4][h[6:]] += int(r[i] or 0)
            except ValueError:
                pass
        if not g[3]:
            g[3] = ins.split()[0] if ins else ""
    print(kern[:90], "total samples", tot)
    key = 2 if os.environ.get("SORT") == "exec" else 0
    print("warp instructions executed", sum(v[2] for v in agg.values()))
    for ln, (a, n, e, ins, c) in sorted(agg.items(), key=lambda x: -x[1][key])[:top]:
        why = " ".join(f"{k}:{v}" for k, v in c.most_common(3) if v)
        print(f"{a:6d} {100.0 * a / max(tot, 1):5.1f}% exec {e:9d}  {ln:24s} {ins:14s} {why}")

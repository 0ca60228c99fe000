"""Aggregate ncu per-SASS-instruction warp-stall samples by CUDA source line.

usage: python tools/ncu_lines.py <report.ncu-rep> <kernel-mangled-name> [top] [--inlined]
Needs the in-tree liblutgpu.so (same build as profiled); uses nvdisasm -g.
With --inlined the innermost inlined location is reported (common.cuh
helpers); by default the outermost onehot.cu line is used.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, fn = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 40
innermost = "--inlined" in sys.argv
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(root, "paper_2302_03213_b200", "_lib", "liblutgpu.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
locs = []
for f in sorted(os.listdir(tmp)):
    if not f.endswith(".cubin"):
        continue
    out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, f)], capture_output=True, text=True).stdout
    start = out.find(".text." + fn + ",")
    if start < 0:
        start = out.find(".text." + fn)
    if start < 0:
        continue
    end = out.find("\n\t.section\t.text.", start + 10)
    body = out[start:end if end > 0 else None]
    cur = None
    for ln in body.splitlines():
        if "//##" in ln:
            m = re.search(r'File "([^"]+)", line (\d+)', ln)
            if m:
                fname, line = os.path.basename(m.group(1)), int(m.group(2))
                # the first '//##' after an instruction is the innermost location;
                # subsequent 'inlined at' lines are outer frames
                if innermost:
                    if "inlined at" not in ln:
                        cur = (fname, line)
                else:
                    if "inlined at" in ln or cur is None or fname == "onehot.cu":
                        cur = (fname, line) if fname.endswith(".cu") else cur
        if re.search(r'/\*[0-9a-f]{4,}\*/', ln):
            locs.append(cur)
            cur = None if not innermost else cur
    break
csvtxt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                        capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(csvtxt)))
hdr = rows[1]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_e = hdr.index("Instructions Executed")
agg, ex = collections.Counter(), collections.Counter()
tot = 0
last = None
for i, r in enumerate(rows[2:]):
    try:
        s = int(r[i_s])
        e = int(r[i_e] or 0)
    except Exception:
        continue
    loc = locs[i] if i < len(locs) and locs[i] else last
    last = loc
    agg[loc] += s
    ex[loc] += e
    tot += s
srcs = {}
print("total samples", tot, "sass instrs", len(rows) - 2, "mapped", len(locs))
for loc, s in agg.most_common(top):
    text = "?"
    if loc:
        fname, line = loc
        if fname not in srcs:
            for d in ("paper_2302_03213_b200/csrc",):
                pth = os.path.join(root, d, fname)
                srcs[fname] = open(pth).read().splitlines() if os.path.exists(pth) else []
        lines = srcs[fname]
        text = lines[line - 1].strip()[:80] if line <= len(lines) else "?"
    print(f"{s:7d} {100 * s / max(tot, 1):5.1f}% ex={ex[loc]:>10d} {loc}: {text}")

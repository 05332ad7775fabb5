"""Attribute an ncu SASS source export (per-instruction stall samples / executions, `--page source --csv
--print-source sass`) to CUDA source lines, using `nvdisasm --print-line-info` of the same cubin (the binary that ran).
  python tools/sass_lines.py <all.sass from nvdisasm> <function substring> <ncu sass csv(.gz)> [iters]"""
import collections
import csv
import gzip
import re
import sys

sass_path, fn, csv_path = sys.argv[1:4]
iters = float(sys.argv[4]) if len(sys.argv) > 4 else 0
lines = open(sass_path).read().split("\n")
i0 = next(i for i, l in enumerate(lines) if fn in l and l.startswith(".text.") and l.endswith(":"))
cur = "?"
seq = []  # (file:line, instruction text) in address order
for l in lines[i0 + 1:]:
    if l.startswith(".section") or (l.startswith(".") and l.endswith(":") and ".text." in l):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        seq.append((cur, m.group(2).strip()))
op = gzip.open if csv_path.endswith(".gz") else open
rows = list(csv.reader(op(csv_path, "rt")))
ks, kc = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        kc = {"name": r[1], "rows": []}
        ks.append(kc)
    elif kc is not None:
        kc["rows"].append(r)
k = next(k for k in ks if fn.split("ILi")[0][-20:] in k["name"] or "search_lp" in k["name"])
h, data = k["rows"][0], k["rows"][1:]
si, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
if len(data) != len(seq):
    print(f"warning: {len(data)} profiled vs {len(seq)} disassembled instructions", file=sys.stderr)
reasons = [c for c in h if c.startswith("stall_") and "(Not Issued)" not in c]
ri = [h.index(c) for c in reasons]
agg = collections.defaultdict(lambda: [0, 0])
why = collections.defaultdict(lambda: collections.Counter())
tot_s = tot_e = 0
for (loc, txt), r in zip(seq, data):
    s, e = int(r[si] or 0), int(r[ei] or 0)
    agg[loc][0] += s
    agg[loc][1] += e
    for c, j in zip(reasons, ri):
        why[loc][c[6:]] += int(r[j] or 0)
    tot_s += s
    tot_e += e
print(f"samples {tot_s}, instructions {tot_e}" + (f", per iteration {tot_e / iters:.1f}" if iters else ""))
for loc, (s, e) in sorted(agg.items(), key=lambda x: -x[1][1 if "--by-inst" in sys.argv else 0])[:(400 if "--all" in sys.argv else 60)]:
    top = ",".join(f"{c}:{v / max(s, 1):.2f}" for c, v in why[loc].most_common(2))
    print(f"{loc:28s} stall {s / tot_s:6.3f}  inst {e / tot_e:6.3f}" + (f"  ({e / iters:6.1f}/iter)" if iters else "")
          + f"  {top}")

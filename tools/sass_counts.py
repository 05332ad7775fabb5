"""Per-kernel SASS instruction counts of libsvf.so (static, from cuobjdump -sass): the tcgen05 / TMA mnemonics that
prove the tensor-core path (UTCHMMA = tcgen05.mma, UTMALDG = TMA tile load, LDTM = tcgen05.ld, UTCBAR =
tcgen05.commit) and the memory / warp-collective mix of the search kernels.

  python tools/sass_counts.py [--lib paper_2601_08528_b200/libsvf.so] --out profiles/r02_sass_counts.md
"""
import argparse
import collections
import os
import re
import subprocess

OPS = ["UTCHMMA", "UTCQMMA", "UTMALDG", "UTMAPF", "LDTM", "STTM", "UTCBAR", "SYNCS", "UBLKCP", "LDGSTS", "LDG",
       "STG", "LDS", "STS", "ATOMS", "ATOMG", "SHFL", "MATCH", "VOTE", "BAR", "FFMA", "FMNMX"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                  "paper_2601_08528_b200", "libsvf.so"))
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", a.lib], capture_output=True, text=True).stdout
    pat = re.compile(r"\b(" + "|".join(OPS) + r")(?:\.[A-Z0-9_.]+)?\b")
    counts, cur = collections.OrderedDict(), None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            counts.setdefault(cur, collections.Counter())
            continue
        if cur and "/*" in line:
            for op in pat.findall(line):
                counts[cur][op] += 1
    keep = [k for k in counts if any(s in k for s in ("knn_tc_kernel<false, false, 16>", "knn_rerank_kernel<16>",
                                                      "search_kernel<1, 2, 32, 1>", "search_kernel<1, 2, 32, 2>",
                                                      "search_lp_kernel<2, 32>", "search_lp_kernel<2, 50>",
                                                      "detour_select_kernel<4>", "reverse_apply_kernel<1>",
                                                      "consolidate_kernel<2, 1>", "merge_topk_kernel<1, false, true>"))]
    lines = ["# SASS instruction counts (static) of " + os.path.basename(a.lib), "",
             "UTCHMMA = tcgen05.mma, UTMALDG = TMA tile load (cp.async.bulk.tensor), LDTM = tcgen05.ld, UTCBAR = "
             "tcgen05.commit; counts are static instructions in the kernel body (`cuobjdump -sass`).", "",
             "| kernel | " + " | ".join(OPS) + " |", "|---|" + "---|" * len(OPS)]
    for k in keep:
        lines.append(f"| `{k[:90]}` | " + " | ".join(str(counts[k].get(op, 0)) for op in OPS) + " |")
    text = "\n".join(lines) + "\n"
    print(text)
    if a.out:
        open(a.out, "w").write(text)


if __name__ == "__main__":
    main()

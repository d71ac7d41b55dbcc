"""Attribute an ncu SASS source page (csv) to CUDA lines of a locally built cubin.

    python scripts/sass_lines.py <ncu-sass.csv> <cubin-disasm-with-lines.sass> <kernel-substring> <src.cu> [k]

The local build must be the one profiled (same instruction order).  Prints the top-k source lines by
executed warp instructions and by stall samples (innermost inlined line)."""
import collections
import csv
import re
import sys

csvp, sassp, kname, srcp = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 25
out, f, cur, prev_ann = [], False, None, False
for l in open(sassp).read().split("\n"):
    if re.search(r"^\s*\.text\.", l):
        if f:
            break
        f = kname in l
        continue
    if not f:
        continue
    if "//##" in l:
        if not prev_ann:
            cur = int(re.findall(r"line (\d+)", l)[0])
        prev_ann = True
        continue
    if re.match(r"\s+/\*[0-9a-f]{4}\*/", l):
        out.append(cur)
        prev_ann = False
rows = list(csv.reader(open(csvp)))
blocks, c, hdr = [], None, None
for r in rows:
    if r and r[0] == "Kernel Name":
        c = []
        blocks.append(c)
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if c is not None and len(r) > 5:
        c.append(dict(zip(hdr, r)))
recs = blocks[0]
acc, st = collections.Counter(), collections.Counter()
for i, d in enumerate(recs[: len(out)]):
    acc[out[i]] += float(d["Instructions Executed"] or 0)
    st[out[i]] += float(d["Warp Stall Sampling (All Samples)"] or 0)
tot, stt = sum(acc.values()), sum(st.values())
src = open(srcp).read().split("\n")
print(f"{len(out)} local / {len(recs)} profiled instructions; {tot:.3g} warp instructions")
for ln, v in sorted(acc.items(), key=lambda x: -x[1] - 1e3 * st[x[0]])[:top]:
    print(f"{ln}: {100 * v / tot:5.1f}% instr {100 * st[ln] / stt:5.1f}% stall  {src[ln - 1].strip()[:90] if ln and ln <= len(src) else ''}")

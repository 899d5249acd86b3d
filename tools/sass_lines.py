#!/usr/bin/env python
"""Attribute an ncu per-SASS-instruction export to source lines.

    python tools/sass_lines.py <ncu-src.csv> <nvdisasm -gi output> <kernel symbol> [top]

<ncu-src.csv>: `ncu -i R --page source --csv --print-source sass`; the second
file: `nvdisasm -gi -c <cubin>` of the same build. Prints, per innermost
source line (file:line), the executed warp instructions, the share of stall
samples and the dominant opcodes -- the view ncu's own cuda-source page does
not give for inlined device functions."""
import collections
import csv
import re
import sys


def main():
    src_csv, dis, sym = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 50
    rows = list(csv.reader(open(src_csv)))
    hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
    h = rows[hi]
    ia, ie, ist = h.index("Address"), h.index("Instructions Executed"), \
        h.index("Warp Stall Sampling (All Samples)")
    recs = []
    for r in rows[hi + 1:]:
        try:
            recs.append((int(r[ia], 16), int(r[ie]), int(r[ist] or 0)))
        except (ValueError, IndexError):
            pass
    base = min(a for a, _, _ in recs)
    # offset -> innermost line, opcode
    where, ops = {}, {}
    inside, cur, fresh = False, None, True
    for ln in open(dis):
        if ln.startswith(".text."):
            inside = ln.strip().rstrip(":") == ".text." + sym
            cur, fresh = None, True
            continue
        if not inside:
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
        if m:  # the first line of a group is the innermost; it holds until the next group
            if fresh:
                cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
                fresh = False
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", ln)
        if m:
            off = int(m.group(1), 16)
            where[off] = cur or "?"
            ops[off] = m.group(3)
            fresh = True
    agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
    tot_i = tot_s = 0
    for a, n, s in recs:
        k = where.get(a - base, "?")
        agg[k][0] += n
        agg[k][1] += s
        agg[k][2][ops.get(a - base, "?")] += n
        tot_i += n
        tot_s += s
    print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s}")
    for k, (n, s, c) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        opstr = " ".join(f"{o}:{v / max(n, 1):.2f}" for o, v in c.most_common(4))
        print(f"{n / tot_i * 100:6.2f}% inst {s / max(tot_s, 1) * 100:6.2f}% stall  {k:28s} {opstr}")


if __name__ == "__main__":
    main()

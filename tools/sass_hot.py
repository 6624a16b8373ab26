"""Summarise an `ncu --page source --csv --print-source sass` export: total
executed warp instructions, the opcode mix weighted by execution count, and
the top stall reasons."""
import csv
import re
import sys
from collections import Counter


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    ops, stalls, total = Counter(), Counter(), 0
    lines = []
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":
            break  # only the first kernel in the export
        if len(r) != len(hdr) or not r[idx["Instructions Executed"]].isdigit():
            continue
        n = int(r[idx["Instructions Executed"]] or 0)
        src = r[idx["Source"]].strip()
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", src)
        op = m.group(2) if m else "?"
        ops[op] += n
        total += n
        samples = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        lines.append((samples, n, src))
        for h in hdr:
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    stalls[h] += int(r[idx[h]] or 0)
                except ValueError:
                    pass
    print(f"executed warp instructions: {total}")
    for op, n in ops.most_common(top):
        print(f"  {op:<12} {n:>14} {100.0 * n / total:6.2f}%")
    st = sum(stalls.values())
    print("stall samples:", st)
    for k, v in stalls.most_common(12):
        print(f"  {k:<24} {v:>8} {100.0 * v / max(st, 1):6.2f}%")
    print("hottest SASS lines (stall samples, executed, source):")
    for s, n, src in sorted(lines, reverse=True)[:25]:
        print(f"  {s:>6} {n:>10}  {src[:90]}")


if __name__ == "__main__":
    main(sys.argv[1])

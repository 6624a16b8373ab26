"""List the backward-branch loops of one kernel in a cubin/object (cuobjdump
-sass) with their size and opcode mix, to spot branches / convergence
barriers (BSSY/BSYNC) inside serial-chain loops.
usage: python tools/sass_loops.py OBJ KERNEL_SUBSTRING [min_len]"""
import re
import subprocess
import sys
from collections import Counter


def main(obj, sub, min_len=100):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", out)
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if sub not in name:
            continue
        ins = []
        for ln in f.split("\n"):
            m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", ln)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        print("==", name[:150], len(ins))
        for a, t in ins:
            m = re.search(r"BRA (?:!?U?P\d, )?0x([0-9a-f]+)", t)
            if m and int(m.group(1), 16) < a and (a - int(m.group(1), 16)) // 16 >= min_len:
                body = [x for x in ins if int(m.group(1), 16) <= x[0] <= a]
                c = Counter(re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", x[1]).group(2).split(".")[0] for x in body)
                print("  loop", hex(int(m.group(1), 16)), hex(a), len(body), "BRA", c["BRA"], "BSSY", c["BSSY"],
                      c.most_common(10))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 100)

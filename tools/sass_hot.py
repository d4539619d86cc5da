"""Opcode histogram of the LARGEST straight-line SASS block (no branch) of a
kernel: the unrolled fast path.  Counts per 'unit' when --per N is given.

    python tools/sass_hot.py paper_2502_15443_b200/build/rans_decode.o k_decode_segmentsINS_6DecCfgILi256 [--per 32]
"""
import re
import subprocess
import sys
from collections import Counter


def blocks(obj, kern):
    txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout.split("\n")
    st = [i for i, l in enumerate(txt) if "Function" in l]
    sec = next(i for i in st if kern in txt[i])
    end = min([j for j in st if j > sec] + [len(txt)])
    cur, out = [], []
    for l in txt[sec:end]:
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if not m:
            continue
        t = m.group(2).strip()
        if "BRA" in t or "EXIT" in t or "BSYNC" in t or "WARPSYNC" in t:
            out.append(cur)
            cur = []
        else:
            cur.append(t)
    out.append(cur)
    return out


if __name__ == "__main__":
    obj, kern = sys.argv[1], sys.argv[2]
    per = int(sys.argv[sys.argv.index("--per") + 1]) if "--per" in sys.argv else 1
    b = max(blocks(obj, kern), key=len)
    c = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for t in b)
    print(f"{len(b)} instructions ({len(b) / per:.2f} per unit)")
    for op, n in c.most_common():
        print(f"  {op:24s} {n:4d}  {n / per:6.2f}")

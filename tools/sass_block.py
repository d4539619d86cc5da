"""Opcode histogram of the first straight-line block after VOTE.ALL in a kernel (the decode fast path).

    python tools/sass_block.py build/rans_decode.o k_decode_segments
"""
import re
import subprocess
import sys
from collections import Counter


def main(obj, kern, nth=0):
    txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout.split("\n")
    st = [i for i, l in enumerate(txt) if "Function" in l]
    sec = next(i for i in st if kern in txt[i])
    end = min([j for j in st if j > sec] + [len(txt)])
    ins = []
    for l in txt[sec:end]:
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    votes = [a for a, t in ins if t.startswith("VOTE.ALL")]
    a0 = votes[nth]
    blk = []
    for a, t in ins:
        if a <= a0 + 0x20:
            continue
        if "BRA" in t:
            if len(blk) > 50:
                break
            blk = []
            continue
        blk.append(t)
    op = lambda t: (t.split()[1] if t.startswith("@") else t.split()[0])  # noqa: E731
    c = Counter(op(t) for t in blk)
    print(len(blk), c.most_common())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0)

"""Opcode histogram of the innermost loops of a SASS dump (cuobjdump -sass):
python tools/sass_loops.py FILE.sass [min_len]"""
import re
import sys
from collections import Counter

lines = open(sys.argv[1]).read().splitlines()
minlen = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ins = []
for l in lines:
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)", t)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt >= a or tgt not in addr_idx:
        continue
    body = ins[addr_idx[tgt]:i + 1]
    if len(body) < minlen:
        continue
    ops = Counter()
    for _, tt in body:
        tt = re.sub(r"^@!?U?P[T\d]+\s+", "", tt)
        ops[tt.split()[0].split(".")[0]] += 1
    print(f"loop 0x{tgt:x}-0x{a:x}: {len(body)} instructions")
    print("   " + ", ".join(f"{k} {v}" for k, v in ops.most_common(18)))

"""Find the loops of one kernel in a cuobjdump -sass listing and print their
instruction mix (backward branches delimit loop bodies).
    python scripts/sass_loops.py LISTING FUNCTION_SUBSTRING [min_len]"""
import collections
import re
import sys

path, fn = sys.argv[1], sys.argv[2]
min_len = int(sys.argv[3]) if len(sys.argv) > 3 else 40
lines, on = [], False
for line in open(path):
    if "Function :" in line:
        on = fn in line
        continue
    if on:
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            lines.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(lines)}
for i, (a, ins) in enumerate(lines):
    m = re.search(r"BRA(?:\.\S+)?\s+(?:\S+,\s*)?`?\(?\.L_x_\d+\)?|BRA.*?0x([0-9a-f]+)", ins)
    t = re.search(r"0x([0-9a-f]+)", ins) if "BRA" in ins else None
    if t:
        tgt = int(t.group(1), 16)
        if tgt < a and tgt in addr and i - addr[tgt] + 1 >= min_len:
            body = lines[addr[tgt]:i + 1]
            ops = collections.Counter()
            for _, x in body:
                op = re.sub(r"^@!?U?P\w+\s+", "", x).split()[0]
                ops[op] += 1
            print(f"loop 0x{tgt:x}-0x{a:x}: {len(body)} instructions")
            for op, c in ops.most_common():
                print(f"   {op:24s}{c}")

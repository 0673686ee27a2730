"""List the hot loops (backward branches) of one SASS function dump with DFMA / LDS / LDL / STL counts.

    cuobjdump -sass -fun <mangled> lib.so > f.sass; python tools/sass_loops.py f.sass
"""
import re
import sys

ins = []
for line in open(sys.argv[1]):
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
for a, t in ins:
    m = re.search(r"BRA.*0x([0-9a-f]+)", t)
    if m and int(m.group(1), 16) < a:
        tgt = int(m.group(1), 16)
        body = [x[1] for x in ins if tgt <= x[0] <= a]
        cnt = {k: sum(k in x for x in body) for k in ("DFMA", "LDS", "LDL", "STL", "UCGABAR_WAIT")}
        if cnt["DFMA"] > 20:
            print(hex(tgt), hex(a), len(body), cnt)

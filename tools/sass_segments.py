"""Count FFMA2 / moves / LDS between consecutive mbarrier try-waits in a SASS dump
(consumer chunk bodies):  python tools/sass_segments.py kernel.sass"""
import re
import sys

seg = {"FFMA2": 0, "MOV": 0, "LDS": 0, "n": 0}
out = []
for line in open(sys.argv[1]):
    m = re.search(r"/\*[0-9a-f]{4,5}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if not m:
        continue
    op = m.group(2)
    if op.startswith("SYNCS.PHASECHK"):
        out.append(dict(seg))
        seg = {"FFMA2": 0, "MOV": 0, "LDS": 0, "n": 0}
    seg["n"] += 1
    if op.startswith("FFMA2"):
        seg["FFMA2"] += 1
    elif op in ("MOV", "IMAD.MOV.U32", "IMAD.MOV"):
        seg["MOV"] += 1
    elif op.startswith("LDS"):
        seg["LDS"] += 1
out.append(seg)
for s in out:
    if s["FFMA2"]:
        print(s)

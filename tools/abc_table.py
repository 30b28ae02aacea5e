"""Summarise tools/gpu/run_abc.sh output: TFLOP/s per (library, shape), one column per run."""
import collections
import json
import sys

rows = collections.OrderedDict()
lib = None
for line in open(sys.argv[1]):
    if line.startswith("=="):
        lib = line.split()[1]
        continue
    try:
        d = json.loads(line)
    except ValueError:
        continue
    v = d["tflops"] if d["tflops"] is not None else d["pairs_per_s"] / 1e9
    rows.setdefault((lib, f"{d['L']}x{d['H']}"), []).append(round(v, 1))
shapes = list(dict.fromkeys(s for _, s in rows))
libs = list(dict.fromkeys(l for l, _ in rows))
print("| library | " + " | ".join(shapes) + " |")
print("|---|" + "---|" * len(shapes))
for l in libs:
    def cell(v):
        if not v:
            return ""
        med = sorted(v)[len(v) // 2]
        return " / ".join(str(x) for x in v) + f" (med {med})"
    print(f"| {l} | " + " | ".join(cell(rows.get((l, s), [])) for s in shapes) + " |")

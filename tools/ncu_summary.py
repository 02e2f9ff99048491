"""Summarise an `ncu --csv --metrics ...` log: one line per launch."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
    d = collections.OrderedDict()
    for r in rows:
        d.setdefault((r[0], r[4]), {})[r[12]] = r[14]
    print(path)
    for (i, k), v in d.items():
        name = k.split("(")[0].replace("void ", "")[-48:]
        short = {m.split("__", 1)[1].split(".")[0][:16]: x for m, x in v.items()}
        print(f"  {i:>3} {name:48s} " + " ".join(f"{a}={b}" for a, b in short.items()))

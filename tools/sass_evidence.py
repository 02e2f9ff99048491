"""SASS evidence of the Blackwell data paths in libgfb.so (cuobjdump):
which kernels issue tcgen05 MMAs (UTCHMMA), TMEM loads (LDTM), TMA loads
(UTMALDG), TMA stores / add-reductions (UTMASTG / UTMAREDG), 1-D bulk copies
(UBLKCP), mbarrier transaction waits (SYNCS), cp.async (LDGSTS), DMMA and the
programmatic-dependent-launch wait / trigger (ACQBULK / PREEXIT).

    python tools/sass_evidence.py > profiles/rNN_sass_evidence.txt
"""
import collections
import os
import re
import subprocess

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2509_02197_b200", "libgfb.so")
OPS = ["UTCHMMA", "UTCBAR", "LDTM", "UTMALDG", "UTMASTG", "UTMAREDG", "UBLKCP", "SYNCS.ARRIVE.TRANS64",
       "SYNCS.PHASECHK.TRANS64.TRYWAIT", "LDGSTS", "DMMA", "FFMA", "DFMA", "ACQBULK", "PREEXIT"]

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
per = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        per[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    for op in OPS:
        if re.search(r"\b" + re.escape(op) + r"\b", line):
            per[cur][op] += 1
demangle = subprocess.run(["c++filt"], input="\n".join(per), capture_output=True, text=True).stdout.splitlines()
print("cuobjdump -sass paper_2509_02197_b200/libgfb.so: static instruction counts per kernel (sm_100a)")
print(f"{'kernel':90s} " + " ".join(f"{o.split('.')[0][:8]:>8s}" for o in OPS))
for (name, cnt), dm in zip(per.items(), demangle):
    if not any(cnt[o] for o in OPS[:9]):
        continue
    print(f"{dm[:90]:90s} " + " ".join(f"{cnt[o]:8d}" for o in OPS))

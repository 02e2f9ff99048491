"""Attribute an ncu source-page capture (SASS, --print-source sass --csv) to
CUDA source lines, through the line table nvdisasm prints for the same cubin:

    python tools/ncu_lines.py <mangled kernel> <nvdisasm -g -c output> <source.csv> <kernel index> \\
        <source file> <first line> <last line>

Prints executed warp instructions and stall samples per source line.
"""
import csv, re, sys, collections
fn, sassf, csvf, kidx, srcf, lo, hi = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), sys.argv[5], int(sys.argv[6]), int(sys.argv[7])
lines = open(sassf).read().split('\n')
start = None; cur = None; off2 = {}
for i, l in enumerate(lines):
    if l.startswith('.text.' + fn + ':'):
        start = i; continue
    if start is None: continue
    if l.startswith('.text.') and i > start + 2: break
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', l)
    if m: cur = m.group(1).split('/')[-1] + ':' + m.group(2); continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*)', l)
    if m:
        off = int(m.group(1), 16); txt = m.group(2)
        op = txt.split()[0] if not txt.startswith('@') else txt.split()[1]
        off2[off] = (cur, op.split('.')[0])
rows = list(csv.reader(open(csvf)))
hdr = None; out = []; n = -1
for r in rows:
    if r and r[0] == "Kernel Name":
        n += 1; continue
    if r and r[0] == "Address": hdr = r; continue
    if n == kidx and hdr and len(r) > 5: out.append(r)
ie = hdr.index("Instructions Executed"); st = hdr.index("Warp Stall Sampling (All Samples)"); base = int(out[0][0], 16)
per = collections.Counter(); stall = collections.Counter(); mism = 0; tot = 0
for x in out:
    off = int(x[0], 16) - base
    c = int(x[ie] or 0); tot += c
    src, op = off2.get(off, ('?', '?'))
    o2 = x[1].split(); o2 = (o2[1] if o2[0].startswith('@') else o2[0]).split('.')[0]
    if op != o2: mism += 1
    per[src] += c; stall[src] += int(x[st] or 0)
print("mismatched opcodes:", mism, "of", len(out), "total instr", tot, "stall samples", sum(stall.values()))
src = open(srcf).read().split('\n')
name = srcf.split('/')[-1]
other = sum(v for k, v in per.items() if not (k or '').startswith(name))
print(f"outside {name}: {other/1e6:.2f}M", [(k, round(v/1e6,2)) for k, v in per.most_common() if not (k or '').startswith(name)][:6])
for i in range(lo, hi):
    c = per.get(f"{name}:{i+1}", 0); s_ = stall.get(f"{name}:{i+1}", 0)
    if c or s_: print(f"{c/1e6:7.2f} {s_:6d} {i+1:4d} {src[i][:110]}")

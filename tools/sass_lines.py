"""Maps ncu per-instruction stall samples to CUDA source lines.

usage: python tools/sass_lines.py <ncu-source-sass.csv> <nvdisasm -c --print-line-info dump> <kernel-mangled-name> <src.cu> [top]
"""
import csv
import re
import sys

csvf, dump, kern, srcf = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
rows = list(csv.reader(open(csvf)))
h = rows[1]
si = h.index('Warp Stall Sampling (All Samples)')
data = []
for r in rows[2:]:
    try:
        data.append((int(r[0], 16), float(r[si]), r[1]))
    except (ValueError, IndexError):
        pass
base = min(d[0] for d in data)
off2line, cur, inside = {}, None, False
for line in open(dump):
    if line.startswith('//--------------------- .text.'):
        inside = kern in line
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', line)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
tot = sum(d[1] for d in data)
agg = {}
for a, v, ins in data:
    ln = off2line.get(a - base, ('?', 0))
    agg[ln] = agg.get(ln, 0) + v
files = {}
for (f, l), v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    if f not in files:
        try:
            files[f] = open(srcf.rsplit('/', 1)[0] + '/' + f).read().split('\n')
        except OSError:
            files[f] = []
    txt = files[f][l - 1].strip()[:72] if l and len(files[f]) >= l else ''
    print(f'{100 * v / tot:5.1f}% {f}:{l}  {txt}')

# per-reason breakdown of the top lines
reasons = [c for c in h if c.startswith('stall_') and '(Not Issued)' not in c]
ri = [h.index(c) for c in reasons]
per = {}
for r in rows[2:]:
    try:
        a = int(r[0], 16)
    except (ValueError, IndexError):
        continue
    ln = off2line.get(a - base, ('?', 0))
    vals = per.setdefault(ln, [0.0] * len(ri))
    for t, i in enumerate(ri):
        try:
            vals[t] += float(r[i])
        except ValueError:
            pass
tot_r = [sum(v[t] for v in per.values()) for t in range(len(ri))]
print('overall:', ', '.join(f'{reasons[t][6:]}={100*tot_r[t]/max(sum(tot_r),1):.1f}%'
                           for t in sorted(range(len(ri)), key=lambda t: -tot_r[t])[:8]))
for (f, l), v in sorted(per.items(), key=lambda x: -sum(x[1]))[:12]:
    s = sum(v)
    top = sorted(range(len(ri)), key=lambda t: -v[t])[:3]
    print(f'{f}:{l}', ', '.join(f'{reasons[t][6:]}={100*v[t]/max(s,1):.0f}%' for t in top))

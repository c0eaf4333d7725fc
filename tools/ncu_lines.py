"""Aggregate the warp-stall samples of an ncu SASS page (csv) by source line.
usage: ncu_lines.py <sass.csv> <nvdisasm --print-line-info dump> <mangled kernel prefix> <source file>"""
import re, csv, collections, sys
sass_csv, dump, prefix, srcfile = sys.argv[1:5]
lines = open(dump).read().splitlines()
start = next(i for i, l in enumerate(lines) if '.section' in l and '.text.' + prefix in l)
cur = None
off2line = {}
for l in lines[start + 1:]:
    if l.lstrip().startswith('.section'):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,6})\*/\s+(.*?);', l)
    if m:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
h = rows[1]; data = rows[2:]
ix = {n: i for i, n in enumerate(h)}
base = int(data[0][0], 16)
st = [n for n in h if n.startswith('stall_') and 'Not Issued' not in n]
tot = collections.Counter()
agg = collections.defaultdict(collections.Counter)
for r in data:
    ln = off2line.get(int(r[0], 16) - base) or ('?', 0)
    a = agg[ln]
    a['samples'] += int(r[ix['# Samples']] or 0)
    a['inst'] += int(r[ix['Instructions Executed']] or 0)
    for s in st:
        v = int(r[ix[s]] or 0)
        a[s] += v; tot[s] += v
T = sum(a['samples'] for a in agg.values()); TI = sum(a['inst'] for a in agg.values())
TS = sum(tot.values())
print('instructions', TI, 'stalls:', {k[6:]: round(v / TS, 3) for k, v in tot.items() if v / TS > 0.005})
src = open(srcfile).read().splitlines()
name = srcfile.split('/')[-1]
for key, a in sorted(agg.items(), key=lambda kv: -kv[1]['samples'])[:int(sys.argv[5]) if len(sys.argv) > 5 else 30]:
    text = src[key[1] - 1].strip()[:64] if key[0] == name and key[1] > 0 else ''
    print(f"{key[0][:14]:14s}:{key[1]:4d} smp {a['samples']/T*100:5.1f}% inst {a['inst']/TI*100:5.1f}% lsb {a['stall_long_sb']:6d} wait {a['stall_wait']:6d} ssb {a['stall_short_sb']:5d} | {text}")

"""Per-instruction stall sampling of one kernel of an ncu report (SASS view):
top opcodes and top instructions.  usage: ncu_src.py rep.ncu-rep <kernel-regex> [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass', '-k', 'regex:' + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == 'Kernel Name':
        cur = [r[1], None, []]
        blocks.append(cur)
    elif r and r[0] == 'Address' and cur:
        cur[1] = r
    elif cur and cur[1]:
        cur[2].append(r)
name, h, body = blocks[0]
si = h.index('Warp Stall Sampling (All Samples)')
ie = h.index('Instructions Executed')
tot = sum(float(r[si]) for r in body) or 1
itot = sum(float(r[ie] or 0) for r in body) or 1
print(name[:110])
op, opi = collections.Counter(), collections.Counter()
for r in body:
    toks = r[1].split()
    o = toks[1] if toks and toks[0].startswith('@') else (toks[0] if toks else '?')
    op[o] += float(r[si])
    opi[o] += float(r[ie] or 0)
print('opcode           stall%   inst%')
for k, v in op.most_common(top):
    print(f'  {k:22s} {100 * v / tot:5.1f} {100 * opi[k] / itot:6.1f}')
print('top instructions:')
for r in sorted(body, key=lambda r: -float(r[si]))[:top]:
    print(f'  {100 * float(r[si]) / tot:5.2f}% {r[0][-5:]} {r[1][:80]}')

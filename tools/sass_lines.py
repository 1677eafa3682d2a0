"""Per-source-line SASS instruction histogram of one kernel (static count), for the
instruction-budget work in DESIGN.md §6.  Usage:
    python tools/sass_lines.py <cubin|so> <function-substring> [lo_addr hi_addr] [--ops]
Counts every instruction of the function (optionally only addresses in [lo, hi)) under the
innermost `## File ..., line N` marker nvdisasm prints before it."""
import collections
import re
import subprocess
import sys


def main():
    path, fn = sys.argv[1], sys.argv[2]
    rng = [int(a, 16) for a in sys.argv[3:5]] if len(sys.argv) > 4 and not sys.argv[3].startswith('--') else None
    ops = '--ops' in sys.argv
    txt = subprocess.run(['nvdisasm', '--print-line-info', '-c', path], capture_output=True, text=True).stdout
    if not txt:
        txt = subprocess.run(['cuobjdump', '-sass', path], capture_output=True, text=True).stdout
    lines = txt.split('\n')
    infn = False
    cur = '?'
    cnt = collections.Counter()
    opc = collections.Counter()
    for l in lines:
        if l.startswith('.text.') or re.match(r'^\s*\.section\s+\.text\.', l):
            infn = fn in l
        m = re.search(r'## File "([^"]+)", line (\d+)', l)
        if m and infn:
            cur = m.group(1).split('/')[-1] + ':' + m.group(2)
            continue
        a = re.search(r'/\*([0-9a-f]{4})\*/\s+(@!?U?P[0-9T]+\s+)?([A-Z][A-Z0-9_.]*)', l)
        if a and infn:
            ad = int(a.group(1), 16)
            if rng and not (rng[0] <= ad < rng[1]):
                continue
            cnt[cur] += 1
            opc[(cur, a.group(3).split('.')[0])] += 1
    tot = sum(cnt.values())
    print(f'total {tot}')
    for k, v in sorted(cnt.items(), key=lambda x: -x[1])[:60]:
        extra = ''
        if ops:
            extra = ' ' + ' '.join(f'{o}:{n}' for (kk, o), n in sorted(opc.items(), key=lambda x: -x[1]) if kk == k)
        print(f'{v:5d} {k}{extra}')


if __name__ == '__main__':
    main()

"""Instruction mix of one profiled kernel (SASS source page)."""
import collections, csv, subprocess, sys

path, regex, skip = sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--kernel-name', 'regex:' + regex,
                      '--launch-skip', str(skip), '--launch-count', '1'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1] if len(rows) > 1 and "Source" in rows[1] else rows[0]
iS, iE = hdr.index('Source'), hdr.index('Instructions Executed')
iW = hdr.index('Warp Stall Sampling (All Samples)')
ops, samp, tot, ts = collections.Counter(), collections.Counter(), 0, 0
for r in rows[2:]:
    if len(r) <= iE:
        continue
    try:
        n, sm = int(r[iE]), int(r[iW])
    except ValueError:
        continue
    toks = r[iS].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith('@') else toks[0]
    op = op.split('.')[0]
    ops[op] += n; samp[op] += sm; tot += n; ts += sm
for op, n in ops.most_common(22):
    print('%-8s %11d %5.1f%%   stall-samples %5.1f%%' % (op, n, 100 * n / tot, 100 * samp[op] / max(ts, 1)))

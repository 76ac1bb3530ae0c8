"""Summarise an A/B log of tools/gpu/r2_l2hint*.sh: python tools/ab_l2_summary.py gpurun_out/l2hint2/ab.log"""
import collections
import json
import sys

rows = collections.defaultdict(list)
for line in open(sys.argv[1]):
    v, rest = line.split(' ', 1)
    rest = rest.strip()
    if rest.startswith('{"strategy"'):
        d = json.loads(rest)
        rows[(d['strategy'], d['cfg'], 'flushed_us')].append((v, round(d['median_us'], 1)))
        rows[(d['strategy'], d['cfg'], 'b2b_us')].append((v, round(d['b2b_us'], 1)))
    elif rest.startswith('m='):
        rows[('smoothing_us', rest.split()[0])].append((v, rest.split('smoothing ')[1].split(' us')[0]))
    elif rest.startswith('cg4'):
        tag, js = rest.split(' ', 1)
        try:
            d = json.loads(js)
        except Exception:
            continue
        if 'wall_ms_per_iteration' in d:
            rows[(tag, 'wall_ms')].append((v, round(d['wall_ms_per_iteration'], 3)))
        elif 'k_apply' in d['kernel'] or 'k_cheb' in d['kernel']:
            rows[(tag, d['kernel'][9:22] + '_ms')].append((v, round(d['ms_per_it'], 3)))
for k, vals in rows.items():
    by = collections.defaultdict(list)
    for v, *x in vals:
        by[v].append(x[0])
    print(k, dict(by))

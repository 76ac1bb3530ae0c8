"""Key figures of a bench.py JSON line: python tools/bench_brief.py gpurun_out/x/bench.json"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("headline", round(d['value'], 2), "GDoF/s", round(d['ms_per_step'] * 1e3, 1), "us  frac", round(d['roofline']['frac'], 3),
      " flushed", round(d['l2_flushed']['GDoF_s'], 2), round(d['l2_flushed']['frac'], 3), " e2e", round(d['e2e']['value'], 2))
for key in ('variants', 'cfg3_q4', 'variants_64cubed_q2', 'variants_32cubed_q4'):
    if key in d:
        print(key, {k: (round(v['GDoF_s'], 2), round(v['frac_hbm'], 3), round(v['frac_fp64'], 3)) for k, v in d[key].items()
                    if isinstance(v, dict)})
for key in ('newton', 'newton_fp32_levels'):
    if key in d:
        print(key, round(d[key]['newton_iteration_s'], 4), 's  cg/it', round(d[key]['s_per_cg_iteration'] * 1e3, 3), 'ms  setup',
              round(d[key]['setup_s'], 4))
for key in ('newton_solve_cfg4', 'newton_solve_cfg4_tensor2'):
    if key in d:
        print(key, round(d[key]['total_s'], 3), 's', d[key]['newton_iterations'], 'its', d[key]['cg_iterations_total'], 'cg')
if 'cfg5_strong' in d:
    c = d['cfg5_strong']
    print('cfg5', round(c['vmult_ms'], 3), 'ms', round(c['vmult_GDoF_s'], 2), 'GDoF/s  cg10', round(c['cg10_ms'], 1), 'ms')
if 'cfg1' in d:
    print('cfg1', d['cfg1']['cg_iterations'], 'its', round(d['cfg1']['cg_solve_s'] * 1e3, 2), 'ms')
print('clocks', d.get('clocks'))

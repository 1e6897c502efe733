import json, sys
d = json.loads(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/bench.json').read().strip().splitlines()[-1])
print('value %.3e faces/s  ms/step %.4f  launches/step %s  clocks %s' % (d['value'], d['ms_per_step'], d.get('launches_per_step'), d.get('clocks')))
print('roofline', {k: d['roofline'][k] for k in ('kernel', 'achieved', 'frac', 'avg_launch_ms', 'share_of_step', 'traffic')})
print('e2e', d.get('e2e', {}) and {k: d['e2e'][k] for k in ('value', 'ms_per_step')})
print('cpu', d.get('cpu_baseline') and d['cpu_baseline']['value'])
print('profile_step_ms', d.get('profile_step_ms'))
for row in d.get('levels', []):
    print(row['level'], round(row['ms'], 4), row.get('survey_frac') and round(row['survey_frac'], 3))
    for k, v in row.get('kernels', {}).items():
        print('    %-12s %.4f ms  %s GB/s frac %s' % (k, v['ms'], v['GBps'] and round(v['GBps']), v['frac'] and round(v['frac'], 3)))

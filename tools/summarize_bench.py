import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    print(f, 'value %.3g' % d['value'], 'ms/step %.2f' % d['ms_per_step'], 'e2e %.3g (%.1f ms)' % (d['e2e']['value'], d['e2e']['ms_per_step']), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))
    print(' config', {k: v for k, v in d['config'].items() if k in ('n', 'T', 'sa_rounds')})
    print(' stages', {k: round(v, 2) for k, v in d['stages_ms'].items()})
    r = d['roofline']; print(' roof %s %.0f GB/s frac %.3f' % (r['kernel'], r['achieved'] or 0, r['frac'] or 0))
    s = d.get('scan_kernel')
    if s: print(' scan %s %.0f GB/s frac %.3f %.2f ms' % (s['kernel'], s['achieved'], s['frac'], s['ms_per_step']))
    if 'cpu_baseline' in d: print(' cpu', '%.3g' % d['cpu_baseline']['value'])
    for k in d['kernels']:
        print('   %-28s %7.2f ms/step %5.1f launches %8.1f GB/s' % (k['kernel'], k['ms_per_step'], k['launches_per_step'], k['achieved_gbs'] or 0))

import json, sys
for f in sys.argv[1:]:
    ls = [x for x in open(f) if x.startswith('{')]
    if not ls:
        print(f, 'NO JSON'); print(open(f).read()[-1500:]); continue
    d = json.loads(ls[-1])
    r = d.get('roofline', {})
    print(f, 'ms/step %.4f' % d['ms_per_step'], 'frac %.3f' % r.get('frac', 0), 'step_frac %.3f' % r.get('step', {}).get('frac', 0),
          {k: round(v, 4) for k, v in r.get('kernels_ms_per_step', {}).items()}, 'e2e %.3g' % d['e2e']['value'])
    for k, v in d.get('solvers', {}).items():
        print('   ', k, round(v['ms_per_step'], 4), round(v['roofline']['frac'], 3), {a: round(b, 4) for a, b in v.get('kernels_ms_per_step', {}).items()})
    if 'mra' in d: print('    mra', round(d['mra']['ms'], 3), round(d['mra']['frac'], 3))
    if 'uniform' in d and d['uniform']: print('    uni', round(d['uniform'].get('ms_per_step', 0), 3))

import json, sys
for f in sys.argv[1:]:
    for l in open(f):
        if l.startswith('{'):
            d = json.loads(l)
            print(d['config']['workload'][-22:], '%.3e' % d['value'], 'ms/step %.2f' % d['ms_per_step'],
                  'kern %.2f' % d['config']['kernel_ms_avg'], 'frac %.3f' % d['roofline']['frac'],
                  'e2e %.3e' % d['e2e']['value'], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))

import json, sys
for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:
        print(path, 'ERR', e); continue
    r = d.get('roofline') or {}
    print(f"{d['config']['workload']:24s} {d['value']:9.1f} Mpx/s  {d['ms_per_step']:8.3f} ms  pipe_frac {d['pipeline_roofline']['frac']:.3f}  dom {r.get('kernel')} {r.get('frac')}  e2e {d['e2e'] and round(d['e2e']['value'],1)}  clk {d['clocks'].get('sm_mhz')} {d['clocks'].get('reasons')}")
    print('    ', {k:(v['ms_per_step'], v['share']) for k,v in d['kernels'].items()})

import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    r = d.get('roofline', {})
    print('%-28s value %.4g evals/s  ms/step %.4f  kern_ms %.4f  frac %.3f  e2e %.4g (%.3f ms) launches %s plane_ms %s' % (
        f.split('/')[-1], d['value'], d['ms_per_step'], r.get('kernel_avg_ms', 0), r.get('frac', 0),
        d['e2e']['value'], d['e2e'].get('ms_per_step', 0), d.get('gpu_launches'), d.get('store', {}).get('rank_plane_build_ms')))

import sys, json
cfg = None
for line in open(sys.argv[1]):
    line = line.strip()
    if line.startswith('{'):
        d = json.loads(line); r = d['roofline']
        print((cfg or '').ljust(24), 'Msamples/s %.1f' % (d['value'] / 1e6), 'Grays/s %.3f' % (d['mrays_per_s'] / 1e3),
              'trace ms %.1f' % r['trace_ms_per_step'], 'ms/step %.1f' % d['ms_per_step'],
              'S %.1f T %.2f frac %.3f' % (r['slab_tests_per_ray'], r['tri_tests_per_ray'], r['frac']))
    elif line and not line.startswith('Trace') and '=' in line and len(line) < 60:
        cfg = line

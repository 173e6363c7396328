import csv, sys
from collections import defaultdict
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hdr = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hdr]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
    d = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            d[r[ki].split('(')[0][:60]].append(float(r[vi].replace(',', '')))
    print(f)
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        print('   %4d x %9.1f us  %s' % (len(v), sum(v) / len(v) / 1e3, k))

import csv, collections, sys
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hdr = None; agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == 'ID': hdr = r; continue
        if hdr is None or len(r) != len(hdr): continue
        d = dict(zip(hdr, r))
        nm = d['Kernel Name'][:60]; v = float(d['Metric Value'].replace(',', '')); mn = d['Metric Name']
        e = agg.setdefault(nm, collections.defaultdict(float)); e[mn] += v
        if mn == 'gpu__time_duration.sum': e['n'] += 1
    print(f)
    for k, e in sorted(agg.items(), key=lambda x: -x[1]['gpu__time_duration.sum'])[:12]:
        print(f"{e['gpu__time_duration.sum']/1e3:9.1f} us {int(e['n']):3d} dramR {e['dram__bytes_read.sum']/1e9:7.2f} GB dramW {e['dram__bytes_write.sum']/1e9:6.2f} GB L2 {e['lts__t_bytes.sum']/1e9:7.1f} GB  {k}")

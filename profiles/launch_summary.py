import csv, collections, sys
path = sys.argv[1]; first = int(sys.argv[2]); steps = int(sys.argv[3])
rows = list(csv.reader(open(path)))
hdr = None; data = []
for r in rows:
    if r and r[0] == 'ID': hdr = r; continue
    if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
seq = [(d['Kernel Name'].split('(')[0].replace('void ', '').replace('tsb::', ''), float(d['Metric Value'])) for d in data if d['Metric Name'] == 'gpu__time_duration.sum']
idx = [i for i, (k, v) in enumerate(seq) if k.startswith('k_update') or k.startswith('void k_update')]
a = idx[first]; b = idx[first + steps]
agg = collections.defaultdict(float); cnt = collections.Counter()
for k, v in seq[a:b]:
    agg[k] += v; cnt[k] += 1
tot = sum(agg.values()) / steps
print(f'steps {first}..{first+steps}: per-step kernel sum {tot/1000:.1f} us')
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"{k:35s} {v/steps/1000:8.1f} us  x{cnt[k]/steps:.1f}  share {100*v/steps/tot:5.1f}%")

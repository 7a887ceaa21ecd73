"""Per-launch times / DRAM bytes of the last V-cycle in an ncu launch list (csv log of
`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv`)."""
import csv
import io
import sys
from collections import OrderedDict

txt = open(sys.argv[1]).read()
rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
L = OrderedDict()
for r in rows:
    d = L.setdefault(r['ID'], {'name': r['Kernel Name'], 'grid': r['Grid Size']})
    sc = {'ns': 1e-3, 'us': 1, 'ms': 1e3, 'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(r['Metric Unit'], 1)
    d[r['Metric Name']] = float(r['Metric Value'].replace(',', '')) * sc
ls = list(L.values())
idx = [i for i, l in enumerate(ls) if 'k_gemv_rows' in l['name']]
seg = ls[idx[-2] + 1:idx[-1] + 1]
print('launches', len(seg), 'total us', sum(l['gpu__time_duration.sum'] for l in seg))
big = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for l in seg:
    mb = (l['dram__bytes_read.sum'] + l['dram__bytes_write.sum']) / 1e6
    if l['gpu__time_duration.sum'] >= big:
        print(f"{l['name'][:64]:64s} {l['grid']:>12s} {l['gpu__time_duration.sum']:8.1f} us {mb:8.1f} MB")

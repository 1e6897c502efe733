"""Per-launch table (us, DRAM MB read / written, TB/s) from an ncu --csv --metrics log with
gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[i]
ki, mi, vi, ui, idi = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
d = OrderedDict()
for r in rows[i + 1:]:
    d.setdefault((r[idi], r[ki].split('(')[0]), {})[r[mi]] = (float(r[vi].replace(',', '')), r[ui])
sc = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'KB': 1e3, 'MB': 1e6, 'GB': 1e9, 'B': 1,
      'nsecond': 1e-3, 'usecond': 1, 'msecond': 1e3, 'ns': 1e-3, 'us': 1, 'ms': 1e3}
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
print('| kernel | us | DRAM rd MB | DRAM wr MB | TB/s |\n|---|---|---|---|---|')
for (_, name), m in list(d.items())[-last:]:
    t = m['gpu__time_duration.sum']
    us = t[0] * sc[t[1]]
    rb = m['dram__bytes_read.sum'][0] * sc[m['dram__bytes_read.sum'][1]]
    wb = m['dram__bytes_write.sum'][0] * sc[m['dram__bytes_write.sum'][1]]
    print(f"| `{name.replace('void ', '')}` | {us:.1f} | {rb / 1e6:.1f} | {wb / 1e6:.1f} | {(rb + wb) / us / 1e6:.2f} |")

"""Summarise an ncu --set full report (raw page) into a markdown table + JSON (per kernel launch)."""
import csv, json, os, subprocess, sys
rep = sys.argv[1]
out_md = sys.argv[2] if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
hdr, units = r[0], r[1]
cols = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sectors.sum']
scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'us': 1e-6, 'ms': 1e-3, 'ns': 1e-9, 'usecond': 1e-6, 'msecond': 1e-3, 'nsecond': 1e-9}
rows = []
seen = {}
for row in r[2:]:
    name = row[hdr.index('Kernel Name')].split('(')[0].replace('void ', '')
    base = name.split('<')[0]
    seen[base] = seen.get(base, -1) + 1
    d = {'kernel': name, 'launch': seen[base]}
    for c in cols:
        if c in hdr:
            v, u = row[hdr.index(c)], units[hdr.index(c)]
            try:
                v = float(v.replace(',', '')) * scale.get(u, 1)
            except ValueError:
                pass
            d[c] = v
    rows.append(d)
lines = ['| kernel | # | time us | DRAM rd MB | DRAM wr MB | DRAM % | L2 hit % | L1 hit % | warps act % | regs | L2 sectors M |', '|---|---|---|---|---|---|---|---|---|---|---|']
for d in rows:
    lines.append('| %s | %d | %.1f | %.1f | %.1f | %.1f | %.1f | %.1f | %.1f | %d | %.2f |' % (
        d['kernel'], d['launch'], d['gpu__time_duration.sum'] * 1e6, d['dram__bytes_read.sum'] / 1e6, d['dram__bytes_write.sum'] / 1e6,
        d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0), d['lts__t_sector_hit_rate.pct'],
        d['l1tex__t_sector_hit_rate.pct'], d['sm__warps_active.avg.pct_of_peak_sustained_active'], d['launch__registers_per_thread'],
        d['lts__t_sectors.sum'] / 1e6))
print('\n'.join(lines))
if out_md:
    json.dump(rows, open(out_md.replace('.md', '.json'), 'w'), indent=1)
    open(out_md, 'w').write('\n'.join(lines) + '\n')
    # per (kernel family, level) DRAM bytes for bench.py's roofline.traffic; the CC level kernels of
    # one refine are captured in launch order, so launch index == level for cc_face/cc_edge/cc_vertex
    summ = {}
    level = -1
    for d in rows:
        base = d['kernel'].split('<')[0].replace('k_', '', 1)
        fam = {'cc_face_quad': 'cc_face', 'cc_face_gen': 'cc_face', 'cc_edge_gp': 'cc_edge'}.get(base, base)
        if fam == 'cc_face':
            level += 1  # the CC level kernels of one refine are captured in order face, edge, vertex
        summ[f"{fam}@L{level}"] = {'dram_bytes': d['dram__bytes_read.sum'] + d['dram__bytes_write.sum'],
                                   'time_us': d['gpu__time_duration.sum'] * 1e6, 'kernel': d['kernel']}
    json.dump({'source': rep, 'kernels': summ}, open(os.path.join(os.path.dirname(out_md), 'ncu_summary.json'), 'w'), indent=1)

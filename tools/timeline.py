"""Start / end of every kernel inside the replayed config-3 refine graph (alsub_probe_read_offsets):
python tools/timeline.py [mesh] [scheme] [L] [max_level].  For each (level, kernel name) the first
launch of that name is probed over 15 replays (L2 flushed before each); prints the median start
and end in us from an event recorded before the replay, sorted by start: the critical path of
the graph at a glance."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen as mg  # noqa: E402
from paper_1809_06047_b200 import Mesh  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "armor9k"
scheme = sys.argv[2] if len(sys.argv) > 2 else "cc"
L = int(sys.argv[3]) if len(sys.argv) > 3 else 6
maxl = int(sys.argv[4]) if len(sys.argv) > 4 else L - 1
mesh = {"armor9k": mg.armor9k, "torus100k": mg.torus100k, "ico": mg.icosahedron}[name]()
build = ("zero", "b0_prep", "scan", "b0_scatter", "b0_edge_count", "b0_edge_fill", "b0_flags", "b0_special",
         "scan2")
level_k = {"cc": ("cc_face", "cc_edge", "cc_vertex", "crease"), "sqrt3": ("s3_face", "s3_vertex"),
           "loop": ("loop_vertex", "scan", "loop_edge", "loop_face", "crease")}[scheme]
flush = torch.empty(64 * 1024 * 1024, device="cuda")
m = Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"])
for _ in range(3):
    m.refine(scheme, L)
R = 15
rows = []
total = []
for lvl in range(-1, maxl + 1):
    for k in (build if lvl < 0 else level_k):
        m.probe(lvl, k, R)
        m.refine(scheme, L)  # capture
        m.probe(lvl, k, R)
        evs, ends = [], []
        for i in range(R):
            flush.fill_(float(i))
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            m.refine(scheme, L)
            b.record()
            evs.append(a)
            ends.append(b)
        try:
            off = m.probe_read_offsets(evs)
        except Exception:
            continue
        torch.cuda.synchronize()
        total += [a.elapsed_time(b) for a, b in zip(evs, ends)]
        s = sorted(o[0] for o in off)[R // 2] * 1e3
        e = sorted(o[1] for o in off)[R // 2] * 1e3
        rows.append((s, e, lvl, k))
m.probe(0, None, 0)
m.close()
rows.sort()
total.sort()
print(f"replay median {total[len(total) // 2] * 1e3:.1f} us (probe replays)")
print(f"{'level':>5} {'kernel':14s} {'start':>8} {'end':>8} {'dur':>7}")
for s, e, lvl, k in rows:
    print(f"{lvl:5d} {k:14s} {s:8.1f} {e:8.1f} {e - s:7.1f}")

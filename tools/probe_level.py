"""Live (in-graph) duration of every kernel of one config-3 level via alsub_probe:
python tools/probe_level.py [level] [cc|sqrt3]  (default 5 cc: the last level of armor9k CC L6; sqrt3:
torus100k L5; -1 = the build)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen as mg  # noqa: E402
from paper_1809_06047_b200 import Mesh  # noqa: E402

lvl = int(sys.argv[1]) if len(sys.argv) > 1 else 5
scheme = sys.argv[2] if len(sys.argv) > 2 else "cc"
L = {"cc": 6, "sqrt3": 5, "loop": 4}[scheme]
mesh = mg.armor9k() if scheme == "cc" else mg.torus100k()
flush = torch.empty(64 * 1024 * 1024, device="cuda")
m = Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"])
for _ in range(3):
    m.refine(scheme, L)
names = {"cc": ("cc_face", "cc_edge", "cc_vertex", "crease"), "sqrt3": ("s3_face", "s3_vertex"),
         "loop": ("loop_vertex", "scan", "loop_edge", "loop_face")}[scheme] if lvl >= 0 else (
    "zero", "b0_prep", "scan", "b0_scatter", "b0_edge_count", "b0_edge_fill", "b0_flags", "b0_special",
    "scan2")  # level -1 = the level-0 build (first launch of each name)
for name in names:
    m.probe(lvl, name, 20)
    m.refine(scheme, L)
    m.probe(lvl, name, 20)
    for i in range(20):
        flush.fill_(float(i))
        m.refine(scheme, L)
    try:
        t = sorted(m.probe_read())
        print(f"level {lvl} {name:10s} median {t[len(t) // 2] * 1e3:7.1f} us  min {t[0] * 1e3:7.1f} us")
    except Exception as e:  # no such kernel at this level
        print(f"level {lvl} {name:10s} -- {e}")
m.probe(0, None, 0)
m.close()

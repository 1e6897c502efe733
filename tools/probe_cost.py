"""Graph-replayed config-3 refine time with and without the in-graph kernel probe (alsub_probe)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen as mg  # noqa: E402
from paper_1809_06047_b200 import Mesh  # noqa: E402

mesh = mg.armor9k()
flush = torch.empty(64 * 1024 * 1024, device="cuda")
m = Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"])


def timed(n=30):
    ts = []
    for i in range(n):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        m.refine("cc", 6)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[n // 2]


for _ in range(3):
    m.refine("cc", 6)
for rnd in range(2):
    print("no probe  ", round(timed(), 4))
    m.probe(5, "cc_face", 40)
    m.refine("cc", 6)
    m.probe(5, "cc_face", 40)
    print("probe     ", round(timed(), 4), "kernel", round(sum(m.probe_read()) / 30, 4))
    m.probe(0, None, 0)
    m.refine("cc", 6)
m.close()

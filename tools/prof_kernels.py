"""Per-kernel CUDA-event profile (alsub_refine_profile), averaged over reps, for one config."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen as mg  # noqa: E402
from paper_1809_06047_b200 import Mesh  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "armor9k"
scheme = sys.argv[2] if len(sys.argv) > 2 else "cc"
L = int(sys.argv[3]) if len(sys.argv) > 3 else 6
mesh = {"armor9k": mg.armor9k, "torus100k": mg.torus100k, "ico": mg.icosahedron, "armor50k": mg.armor50k}[name]()
m = Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"])
flush = torch.empty(64 * 1024 * 1024, device="cuda")
acc = defaultdict(list)
order = []
for r in range(8):
    flush.fill_(1.0)
    for i, (n, lv, ms) in enumerate(m.refine_profile(scheme, L)):
        if r == 0:
            order.append((n, lv, i))
        acc[(n, lv, i)].append(ms)
tot = 0
for k in order:
    v = sorted(acc[k])[1:-1] or acc[k]
    t = sum(v) / len(v)
    tot += t
    print("%-18s L%-3d %8.4f ms" % (k[0], k[1], t))
print("sum %.4f ms" % tot)

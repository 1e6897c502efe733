"""Graph-replayed refine time for levels 0..L (config 3 by default): the increments give the
per-level cost inside the CUDA graph (no per-kernel event overhead)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen as mg  # noqa: E402
from paper_1809_06047_b200 import Mesh  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "armor9k"
mesh = {"armor9k": mg.armor9k, "torus100k": mg.torus100k, "ico": mg.icosahedron,
        "armor9k_shuf": lambda: mg.shuffled(mg.armor9k()), "torus100k_shuf": lambda: mg.shuffled(mg.torus100k()),
        "tet_creased": lambda: mg.tetrahedron(creased=True), "cube": mg.cube}[name]()
scheme = sys.argv[2] if len(sys.argv) > 2 else "cc"
L = int(sys.argv[3]) if len(sys.argv) > 3 else 6
flush = torch.empty(64 * 1024 * 1024, device="cuda")
m = Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"])
prev = 0.0
for lv in range(0, L + 1):
    for _ in range(3):
        m.refine(scheme, lv)
    ts = []
    for _ in range(20):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        m.refine(scheme, lv)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    med = ts[len(ts) // 2]
    print(f"levels={lv} median_ms={med:.4f} increment_ms={med - prev:.4f} launches={m.last_launch_count}")
    prev = med
m.close()

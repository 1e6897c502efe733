"""Wall-clock pieces of bench.py's e2e step (create from pinned host, eager refine, exports)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen as mg  # noqa: E402
from paper_1809_06047_b200 import Mesh  # noqa: E402
from paper_1809_06047_b200 import alsub as A  # noqa: E402

mesh = mg.armor9k()
L = 6
pin = lambda a: torch.from_numpy(a).pin_memory()
fo, fv, P, cr, sg = pin(mesh["face_off"]), pin(mesh["face_vtx"]), pin(mesh["pos"]), pin(mesh["crease"]), pin(mesh["sigma"])
lib = A.lib()
for rep in range(4):
    t = [time.perf_counter()]
    m = Mesh(fo, fv, P, cr, sg)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    m.refine("cc", L)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    c = m.counts(L)
    if rep == 0:
        out_P = torch.empty((c["verts"], 3), dtype=torch.float32).pin_memory()
        out_F = torch.empty(c["face_slots"], dtype=torch.int32).pin_memory()
    s = torch.cuda.current_stream().cuda_stream
    A._check(lib.alsub_level_positions(m._h, L, out_P.data_ptr(), s))
    torch.cuda.synchronize(); t.append(time.perf_counter())
    A._check(lib.alsub_level_topology(m._h, L, out_F.data_ptr(), None, None, None, None, None, None, s))
    torch.cuda.synchronize(); t.append(time.perf_counter())
    m.close()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    names = ["create", "refine", "pos_d2h", "topo_d2h", "close"]
    print(rep, " ".join(f"{n}={1e3 * (t[i + 1] - t[i]):.2f}ms" for i, n in enumerate(names)))

"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck): every entry
point once on small meshes, eager launches (ALSUB_NO_GRAPH=1 is set by the caller)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import meshgen as mg  # noqa: E402
from paper_1809_06047_b200 import Mesh, frame_summary, rcm_order  # noqa: E402

arm = mg.armor(6, 5, 6, 1, 1, 2, name="armor_small")
with Mesh(arm["face_off"], arm["face_vtx"], arm["pos"], arm["crease"], arm["sigma"]) as m:
    m.refine("cc", 4)
    m.topology(3, edges=True, creases=True)
    m.topology(4, creases=True)
    fr = torch.stack([torch.from_numpy(mg.frame_positions(arm["pos"], t, 16)) for t in range(9)]).cuda()
    out4 = m.eval_frames(fr, 4)
    frame_summary(out4)
    frame_summary(out4[:, 1:].contiguous())
    m.eval_attributes(torch.from_numpy(mg.vertex_channels(arm, 4)).cuda(), 3)
    v = m.level_positions_view(2)
    v += 0.01
    m.reevaluate(2)
    m.build_refinement_matrix(3)
    m.eval_frames_matrix(fr)
    sub, _, _ = m.extract(1, rings=2)
    with sub:
        sub.refine("cc", 2)
tet = mg.tetrahedron(creased=True)
with Mesh(tet["face_off"], tet["face_vtx"], tet["pos"], tet["crease"], tet["sigma"]) as m:
    m.refine("loop", 4)
    m.topology(3, edges=True, creases=True)
tor = mg.torus_tris(12, 9)
with Mesh(tor["face_off"], tor["face_vtx"], tor["pos"]) as m:
    m.refine("sqrt3", 3)
    m.eval_frames(torch.from_numpy(tor["pos"])[None].cuda(), 3)
pv, pf = rcm_order(arm["face_off"], arm["face_vtx"], arm["pos"].shape[0])
torch.cuda.synchronize()
print("sanitize smoke ok")

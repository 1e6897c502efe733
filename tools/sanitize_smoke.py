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
# round 2: long M^T rows (block sort in registers, and the global-memory network past 1024 slots),
# the poles' ring kernels of every scheme, the blocked matrix with fused records (ragged batch,
# wide supports), isolated control vertices, the single-sync create on invalid input
for n, scheme in ((300, "cc"), (300, "loop"), (300, "sqrt3"), (1500, "cc")):
    bp = mg.bipyramid(n)
    with Mesh(bp["face_off"], bp["face_vtx"], bp["pos"]) as m:
        m.refine(scheme, 2)
        m.refine(scheme, 2)
for mk, scheme, L in ((lambda: mg.bipyramid(30), "loop", 2), (lambda: arm, "cc", 3)):
    mm = mk()
    with Mesh(mm["face_off"], mm["face_vtx"], mm["pos"], mm["crease"], mm["sigma"]) as m:
        m.refine(scheme, L)
        m.build_refinement_matrix(L)
        f = torch.from_numpy(np.stack([mm["pos"]] * 37)).cuda()
        m.eval_frames_matrix_summary(f)
iso = mg._pack([(0, 1, 2, 3)], [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (5, 5, 5)])
with Mesh(iso["face_off"], iso["face_vtx"], iso["pos"]) as m:
    m.refine("cc", 3)
    m.build_refinement_matrix(3)
    m.eval_frames_matrix(torch.from_numpy(iso["pos"])[None].cuda())
# round 2, late: the grandparent edge kernel before the last level (crease-free closed mesh, levels
# 3 of 5: cc_use_gp), dynamic and static
cube = mg.cube()
with Mesh(cube["face_off"], cube["face_vtx"], cube["pos"]) as m:
    m.refine("cc", 5)
    m.refine("cc", 5)
    m.eval_frames(torch.from_numpy(np.stack([cube["pos"]] * 3)).cuda(), 5)
from paper_1809_06047_b200 import AlsubError  # noqa: E402
for faces in ([(0, 1, 7)], [(0, 1, 2), (0, 1, 3)], [(0, 1, 2), (1, 0, 3), (0, 1, 4)]):
    try:
        Mesh(*[mg._pack(faces, np.zeros((5, 3), np.float32))[k] for k in ("face_off", "face_vtx", "pos")])
    except AlsubError:
        pass
torch.cuda.synchronize()
print("sanitize smoke ok")

"""One blocked-SpMM batch of config 5 (armor50k CC L4, 32 frames) for ncu captures;
`python tools/rm_once.py summary` runs the variant with the per-frame records folded in."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen as mg  # noqa: E402
from paper_1809_06047_b200 import Mesh  # noqa: E402

mesh = mg.armor50k()
frames = torch.stack([torch.from_numpy(mg.frame_positions(mesh["pos"], t, 4096)) for t in range(32)]).cuda()
m = Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"])
m.refine("cc", 4)
m.build_refinement_matrix(4)
if len(sys.argv) > 1 and sys.argv[1] == "summary":
    out, rec = m.eval_frames_matrix_summary(frames)
    out, rec = m.eval_frames_matrix_summary(frames, out=out, summary=rec)
else:
    out = m.eval_frames_matrix(frames)
    out = m.eval_frames_matrix(frames, out=out)
torch.cuda.synchronize()

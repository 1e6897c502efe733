"""One blocked-SpMM batch of config 5 (armor50k CC L4, 32 frames) for ncu captures."""
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
out = m.eval_frames_matrix(frames)
out = m.eval_frames_matrix(frames, out=out)
torch.cuda.synchronize()

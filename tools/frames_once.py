"""Run config-5 static eval (armor50k CC L4) for a few batches of frames; used under ncu."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import meshgen as mg
from paper_1809_06047_b200 import Mesh

levels = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 8
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
mesh = mg.armor50k()
P0 = mesh["pos"]
dev = torch.device("cuda:0")
frames = torch.stack([torch.from_numpy(mg.frame_positions(P0, t, 4096)) for t in range(nb)]).to(dev)
m = Mesh(mesh["face_off"], mesh["face_vtx"], P0, mesh["crease"], mesh["sigma"])
m.refine("cc", levels)
out = None
for r in range(reps):
    out = m.eval_frames(frames, levels, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for r in range(10):
    out = m.eval_frames(frames, levels, out=out)
e1.record()
torch.cuda.synchronize()
print(f"nb={nb} ms_per_batch={e0.elapsed_time(e1) / 10:.4f} launches={m.last_launch_count}")

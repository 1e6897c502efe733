"""One eager dynamic-mode refinement of config 3 (armor9k, CC level 6) -- the process ncu profiles."""
import os
import sys

os.environ.setdefault("ALSUB_NO_GRAPH", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen as mg  # noqa: E402
from paper_1809_06047_b200 import Mesh  # noqa: E402

levels = int(sys.argv[1]) if len(sys.argv) > 1 else 6
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
mesh = mg.armor9k()
m = Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"])
for _ in range(reps):
    m.refine("cc", levels)
torch.cuda.synchronize()
m.close()
print("ok")

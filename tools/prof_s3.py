"""One eager sqrt3 refinement of config 4 (torus100k, level 5) -- the process ncu profiles."""
import os
import sys

os.environ.setdefault("ALSUB_NO_GRAPH", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen as mg  # noqa: E402
from paper_1809_06047_b200 import Mesh  # noqa: E402

mesh = mg.torus100k()
m = Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"])
m.refine("sqrt3", int(sys.argv[1]) if len(sys.argv) > 1 else 5)
torch.cuda.synchronize()
m.close()
print("ok")

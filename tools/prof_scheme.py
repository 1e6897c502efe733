"""One eager refinement of a named mesh and scheme (the process ncu profiles):
python tools/prof_scheme.py torus100k sqrt3 5"""
import os
import sys

os.environ.setdefault("ALSUB_NO_GRAPH", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen as mg  # noqa: E402
from paper_1809_06047_b200 import Mesh  # noqa: E402

name, scheme, levels = sys.argv[1], sys.argv[2], int(sys.argv[3])
mesh = {"armor9k": mg.armor9k, "torus100k": mg.torus100k, "ico": mg.icosahedron, "armor50k": mg.armor50k}[name]()
m = Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"])
m.refine(scheme, levels)
torch.cuda.synchronize()
m.close()
print("ok")

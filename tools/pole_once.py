import sys, os
sys.path.insert(0, "/root/repo")
import torch, meshgen as mg
from paper_1809_06047_b200 import Mesh
mesh = mg.bipyramid(1024)
m = Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"])
m.refine("cc", 4); m.refine("cc", 4); torch.cuda.synchronize()

"""Config 3: refine, then export the level-6 crease lists -- the export's first call runs the last
level's lazy crease inheritance (ensure_last_lists: one k_crease launch in lists-only mode).
Run under ncu to time that launch: the kernel bench.py reports as `last_level_crease_lists`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen as mg  # noqa: E402
from paper_1809_06047_b200 import Mesh  # noqa: E402

mesh = mg.armor9k()
m = Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"])
m.refine("cc", 6)
torch.cuda.synchronize()
m.topology(6, faces=False, creases=True)  # the lazy lists: the last k_crease launch
torch.cuda.synchronize()
m.close()
print("ok")

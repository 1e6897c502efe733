"""B200-native AlSub uniform refinement (arXiv 1809.06047): C-ABI library + thin binding.

    from paper_1809_06047_b200 import Mesh
    m = Mesh(face_off, face_vtx, pos, crease, sigma)     # alsub_mesh_create
    m.refine("cc", 6)                                   # alsub_refine (CUDA graph, no host sync)
    P6 = m.positions(6); T6 = m.topology(6)             # alsub_level_positions / _topology
"""
from .alsub import (AlsubError, CATMULL_CLARK, LOOP, SQRT3, SCHEMES, Mesh, lib, rcm_order, version,  # noqa: F401
                    frame_summary, split_summary, exported_symbols, LIB_PATH)

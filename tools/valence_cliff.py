"""High-valence cost probe: create + graph-replayed refine of a bipyramid with
two valence-n poles against a bounded-valence torus with the same number of triangles, for every
scheme.  Prints one JSON line per case; the difference is the cost of the long rows."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen as mg  # noqa: E402
from paper_1809_06047_b200 import Mesh  # noqa: E402


def refine_ms(mesh, scheme, L, reps=20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"])
    torch.cuda.synchronize()
    create_ms = 1e3 * (time.perf_counter() - t0)
    for _ in range(3):
        m.refine(scheme, L)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        m.refine(scheme, L)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    m.close()
    ts.sort()
    return create_ms, ts[len(ts) // 2]


def main():
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    for n in (8, 256, 1024):
        pole = mg.bipyramid(n)
        # same triangle count, valence <= 8: a torus grid of 2n triangles (n/16 x 16 cells... )
        nu = max(4, n // 8)
        ref = mg.torus_tris(nu, 8)
        for scheme in ("cc", "loop", "sqrt3"):
            c_p, r_p = refine_ms(pole, scheme, L)
            c_r, r_r = refine_ms(ref, scheme, L)
            print(json.dumps({"n": n, "scheme": scheme, "levels": L, "faces0": int(len(pole["face_off"]) - 1),
                              "ref_faces0": int(len(ref["face_off"]) - 1), "pole_create_ms": c_p,
                              "pole_refine_ms": r_p, "ref_create_ms": c_r, "ref_refine_ms": r_r,
                              "refine_growth_us": 1e3 * (r_p - r_r)}), flush=True)



def kernels(n=1024, scheme="cc", L=4):
    """Per-kernel table (alsub_refine_profile, eager with events) of the pole mesh."""
    mesh = mg.bipyramid(n)
    m = Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"])
    m.refine(scheme, L)
    acc = {}
    for _ in range(5):
        for name, lvl, ms in m.refine_profile(scheme, L):
            acc.setdefault((lvl, name), []).append(ms)
    for (lvl, name), v in sorted(acc.items()):
        print(f"  L{lvl:2d} {name:20s} {1e3 * sorted(v)[len(v) // 2]:8.1f} us")
    m.close()


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "kernels":
        for sch in ("cc", "loop", "sqrt3"):
            print(sch)
            kernels(1024, sch, int(sys.argv[1]))
    else:
        main()

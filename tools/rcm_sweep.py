"""NEXT-2 measurement: graph-replayed refine time of configs 3 and 4 in the generator's order,
shuffled (seeded random relabelling), and shuffled + RCM (alsub_rcm_order)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen as mg  # noqa: E402
from paper_1809_06047_b200 import Mesh, rcm_order  # noqa: E402


def timed(mesh, scheme, L, reps=30):
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    m = Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"])
    for _ in range(3):
        m.refine(scheme, L)
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        m.refine(scheme, L)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    m.close()
    ts.sort()
    return ts[len(ts) // 2]


out = {}
for name, make, scheme, L in (("config3_armor9k_cc_L6", mg.armor9k, "cc", 6),
                              ("config4_torus100k_sqrt3_L5", mg.torus100k, "sqrt3", 5)):
    base = make()
    shuf = mg.shuffled(base)
    t0 = time.perf_counter()
    pv, pf = rcm_order(shuf["face_off"], shuf["face_vtx"], shuf["pos"].shape[0])
    t_rcm = time.perf_counter() - t0
    rcm_mesh = mg.permuted(shuf, pv, pf)
    pv2, pf2 = rcm_order(base["face_off"], base["face_vtx"], base["pos"].shape[0])
    row = {"generator_order_ms": timed(base, scheme, L), "shuffled_ms": timed(shuf, scheme, L),
           "shuffled_rcm_ms": timed(rcm_mesh, scheme, L),
           "generator_rcm_ms": timed(mg.permuted(base, pv2, pf2), scheme, L),
           "rcm_host_ms": t_rcm * 1e3}
    out[name] = row
    print(name, json.dumps(row), flush=True)
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/rcm_sweep.json", "w"), indent=1)

"""Config 5 blocked-SpMM timing, evaluation only vs with the fused per-frame records:
python tools/rm_time.py [frames=256]  (us per frame, median of 5 passes, CUDA events)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen as mg  # noqa: E402
from paper_1809_06047_b200 import Mesh  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 256
mesh = mg.armor50k()
frames = torch.stack([torch.from_numpy(mg.frame_positions(mesh["pos"], t, 4096)) for t in range(32)]).cuda()
m = Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"])
m.refine("cc", 4)
info = m.build_refinement_matrix(4)
out = [torch.empty((32, info["rows"], 3), dtype=torch.float32, device="cuda") for _ in range(2)]
rec = torch.empty((32, 8), dtype=torch.int32, device="cuda")


def timed(fn):
    ts = []
    for rep in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(nf // 32):
            fn(i)
        b.record()
        torch.cuda.synchronize()
        if rep:
            ts.append(a.elapsed_time(b))
    ts.sort()
    return 1e3 * ts[len(ts) // 2] / nf


t_eval = timed(lambda i: m.eval_frames_matrix(frames, out=out[i & 1]))
t_sum = timed(lambda i: m.eval_frames_matrix_summary(frames, out=out[i & 1], summary=rec))
ref = m.eval_frames_matrix(frames)
from paper_1809_06047_b200 import frame_summary  # noqa: E402
ok = bool(torch.equal(frame_summary(ref), m.eval_frames_matrix_summary(frames)[1]))
print(json.dumps({"eval_us_per_frame": t_eval, "summary_us_per_frame": t_sum, "records_equal": ok}))

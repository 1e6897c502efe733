"""NEXT-1 measurement: config 5 (armor50k CC L4) static eval by the single SpMM P_L = R P_0 vs the
level-by-level static path, plus the build cost and size of R."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import meshgen as mg  # noqa: E402
from paper_1809_06047_b200 import Mesh  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nf = int(sys.argv[2]) if len(sys.argv) > 2 else 128
mesh = mg.armor50k()
P0 = mesh["pos"]
frames = torch.stack([torch.from_numpy(mg.frame_positions(P0, t, 4096)) for t in range(nf)]).cuda()
m = Mesh(mesh["face_off"], mesh["face_vtx"], P0, mesh["crease"], mesh["sigma"])
m.refine("cc", L)
torch.cuda.synchronize()
t0 = time.perf_counter()
info = m.build_refinement_matrix(L)
torch.cuda.synchronize()
t_build = time.perf_counter() - t0
VL = info["rows"]
out = torch.empty((nf, VL, 3), dtype=torch.float32, device="cuda")


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


t_mat = timed(lambda: m.eval_frames_matrix(frames, out=out))
t_lvl = timed(lambda: m.eval_frames(frames, L, out=out))
ref = m.eval_frames(frames[:8], L)
got = m.eval_frames_matrix(frames[:8])
err = float((ref - got).abs().max())
blk = m.refinement_matrix_blocks()
# bytes per batch of 32 frames: the weights, row ids and support lists once, the output once
bytes_batch = 4 * blk["weights"] + 4 * VL + 12 * VL * 32
row = {"levels": L, "frames": nf, "rows": VL, "nnz": info["nnz"], "nnz_per_row": info["nnz"] / VL,
       "R_bytes": 8 * info["nnz"] + 4 * (VL + 1), "build_s": t_build, "chunks": blk["chunks"],
       "block_weights": blk["weights"], "block_fill": info["nnz"] / blk["weights"],
       "matrix_us_per_frame": 1e3 * t_mat / nf, "levels_us_per_frame": 1e3 * t_lvl / nf,
       "matrix_GBps": bytes_batch * (nf / 32) / (t_mat * 1e6), "output_GBps": 12 * VL * nf / (t_mat * 1e6),
       "fma_per_frame": 3 * blk["weights"] / 1.0, "max_abs_diff": err}
print(json.dumps(row))
json.dump(row, open("gpurun_out/rm_bench.json", "w"), indent=1)

"""CPU-only checks: the C-ABI library loads and exports every symbol include/alsub.h declares,
the build is for sm_100a, host-side sharding / timing reduction work over gloo (world_size 2),
and the bench reference arm prints a well-formed JSON line."""
import json
import os
import subprocess
import sys

import pytest

import meshgen as mg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_1809_06047_b200 import build as b
    return b.build()


def test_library_exports_every_header_symbol():
    import ctypes
    path = _lib()
    from paper_1809_06047_b200.alsub import exported_symbols
    L = ctypes.CDLL(path)
    syms = exported_symbols()
    assert len(syms) >= 10
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_library_is_sm100a():
    path = _lib()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_string_without_gpu():
    import ctypes
    L = ctypes.CDLL(_lib())
    L.alsub_version.restype = ctypes.c_char_p
    assert b"sm_100a" in L.alsub_version()


def test_create_without_gpu_fails_cleanly():
    """No CUDA device here: the ABI must return an error status, never crash or fall back."""
    import ctypes
    import numpy as np
    import meshgen as mg
    L = ctypes.CDLL(_lib())
    L.alsub_mesh_create.restype = ctypes.c_int
    m = mg.cube()
    h = ctypes.c_void_p()
    st = L.alsub_mesh_create(ctypes.c_void_p(m["face_off"].ctypes.data), ctypes.c_void_p(m["face_vtx"].ctypes.data), 6,
                             ctypes.c_void_p(m["pos"].ctypes.data), 8, None, None, 0, None, None, ctypes.byref(h))
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    assert st != 0 and not h.value


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = bench.shard(4096, world, rank)
    m = bench.dist_max(10.0 + rank)
    # the frames job's one data collective: every rank's summary records, gathered in frame order
    import torch
    n = 4096
    local = torch.arange(lo, hi, dtype=torch.int32)[:, None] * 8 + torch.arange(8, dtype=torch.int32)
    table = bench.gather_summaries(local, n, world, rank)
    table_ok = bool(torch.equal(table, torch.arange(8 * n, dtype=torch.int32).view(n, 8)))
    # uneven shards (odd frame count) are padded for the collective and trimmed again
    lo2, hi2 = bench.shard(7, world, rank)
    local2 = torch.arange(lo2, hi2, dtype=torch.int32)[:, None].repeat(1, 8)
    t2 = bench.gather_summaries(local2, 7, world, rank)
    table_ok = table_ok and bool(torch.equal(t2[:, 0], torch.arange(7, dtype=torch.int32)))
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, lo, hi, m, table_ok))


def test_gloo_sharding_and_max_over_ranks():
    import multiprocessing as mp
    import random
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res[0][1:3] == (0, 2048) and res[1][1:3] == (2048, 4096)
    assert res[0][3] == res[1][3] == 11.0
    assert res[0][4] and res[1][4]


def test_shard_covers_all_units():
    sys.path.insert(0, ROOT)
    import bench
    for n in (1, 7, 4096, 4097):
        for w in (1, 2, 3, 8):
            spans = [bench.shard(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_bench_reference_arm_json():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--ref-levels", "2"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "impl",
              "cpu_baseline", "e2e", "config"):
        assert k in line
    assert line["impl"] == "reference" and line["value"] > 0


def test_bench_gpus_flag_spawns_ranks():
    """`python bench.py --gpus 2` without torchrun re-launches itself under torch.distributed.run
    with two ranks (--gpus was parsed and never read); --dry-run runs the multi-rank
    plumbing (gloo process group, sharded records, their gather in frame order) without a GPU."""
    import json
    import subprocess
    import sys
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run", "--gpus", "2", "--frames", "37"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["ranks"] == [0, 1] and line["pids"] == 2
    assert line["frames_gathered"] == 37 and line["frame_order_ok"]


@pytest.mark.parametrize("scheme,mk", [("cc", lambda: mg.armor(4, 5, 6, 1, 1, 2, name="a")),
                                       ("loop", lambda: mg.tetrahedron(creased=True)),
                                       ("sqrt3", lambda: mg.torus_tris(8, 6))])
def test_oracle_openmp_build_is_identical(scheme, mk):
    """The all-cores oracle (liboracle_omp.so, bench.py's host baseline) marks only single-writer
    per-element loops: its levels equal the serial oracle's bit for bit."""
    import numpy as np
    import oracle
    mesh = mk()
    t1, t2 = [], []
    a = oracle.refine(mesh, scheme, 3, times=t1)
    b = oracle.refine(mesh, scheme, 3, threads=4, times=t2)
    assert len(t1) == len(t2) == 3
    for x, y in zip(a, b):
        for k in ("pos", "face_vtx", "face_off", "crease", "sigma"):
            assert np.array_equal(x[k], y[k]), k


def test_bench_method_bytes_config3_last_level():
    """The roofline counts method bytes only (the c0 intermediate was counted): for
    config 3's level 5->6 face kernel, read 4S face rows + 12V positions + 48F' grandparent rows,
    write 16S child faces + 12F face points + vertex points of the face points born at levels 5
    and 4 = 1,045,321,920 B; the corner sums c0 are intermediate -- at the last level only the faces
    r = 0 mod 4 keep one, compacted: 12 F/4 = 26,173,440 B."""
    import bench
    V, F, S, E = 10000, 8590, 34080, 18510  # armor9k
    cnt = [dict(V=V, F=F, S=S, E=E)]
    for _ in range(6):
        V, F, S, E = V + F + E, S, 4 * S, 2 * E + S
        cnt.append(dict(V=V, F=F, S=S, E=E))
    face = bench.kernel_bytes_cc("cc_face", cnt[5], cnt[4], 5, 6, cnt[3])
    assert face == {"method": 1045321920, "intermediate": 26173440}
    c5, c4, c3 = cnt[5], cnt[4], cnt[3]
    by_hand = 4 * c5["S"] + 12 * c5["V"] + 48 * c4["F"] + 16 * c5["S"] + 12 * c5["F"] + 12 * c4["F"] + 12 * c3["F"]
    assert face["method"] == by_hand
    edge = bench.kernel_bytes_cc("cc_edge", cnt[5], cnt[4], 5, 6, cnt[3])
    assert edge["intermediate"] == 0


def test_bench_method_bytes_grandparent_path_before_last_level():
    """Level levels-2 (>= 3, unfused) runs the grandparent edge kernel (api.cu cc_use_gp): the edge
    kernel reads the level-(l-1) pairs and rows, 12 V positions and 12 F face points, writes 12 E
    edge points and the vertex points of the edge points born at l and l-1; the face kernel writes
    no half sums and compact corner sums (12 F/4) -- config 3's level 4->5, counted by hand."""
    import bench
    V, F, S, E = 10000, 8590, 34080, 18510  # armor9k
    cnt = [dict(V=V, F=F, S=S, E=E)]
    for _ in range(6):
        V, F, S, E = V + F + E, S, 4 * S, 2 * E + S
        cnt.append(dict(V=V, F=F, S=S, E=E))
    c4, c3, c2 = cnt[4], cnt[3], cnt[2]
    edge = bench.kernel_bytes_cc("cc_edge", c4, c3, 4, 6, c2, gp_mid=True)
    assert edge["method"] == (8 * c3["E"] + 16 * c3["F"] + 12 * c4["V"] + 12 * c4["F"] + 12 * c4["E"]
                              + 12 * (c3["E"] + c2["E"]))
    face = bench.kernel_bytes_cc("cc_face", c4, c3, 4, 6, c2, gp_mid=True)
    assert face["intermediate"] == 12 * ((c4["F"] + 3) // 4)
    assert bench.kernel_bytes_cc("cc_face", c4, c3, 4, 6, c2)["intermediate"] == 12 * c4["F"] + 12 * c4["F"]
    # only level levels-2 takes the flag
    assert bench.kernel_bytes_cc("cc_edge", c3, c2, 3, 6, cnt[1], gp_mid=True) == \
        bench.kernel_bytes_cc("cc_edge", c3, c2, 3, 6, cnt[1])

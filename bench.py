#!/usr/bin/env python
"""Benchmark: refined faces/s of AlSub uniform refinement on B200 (BASELINE.json metric).

Default workload: SURVEY.md 8(d) config 3 -- Catmull-Clark level 6 of the ArmorGuy-shaped creased
mesh armor9k (8,590 faces -> 34,897,920 faces).  A step is one alsub_refine(CC, 6): the whole hot
path (level-0 mesh matrix, counting-sort M^T, edge index, creases, then 6 levels of topology +
geometry), replayed as a CUDA graph with inputs resident in HBM.  L2 is flushed (a 256 MiB write)
between timed steps.  With N > 1 ranks each rank refines its own independent mesh (seed 1809 +
rank): weak scaling, no collective on the data path.

Every line also carries "frames": config 5 -- 4096 animation frames of armor50k (CC level 4,
fixed topology) split over the N ranks (strong scaling), static mode through the blocked
refinement matrix (alsub_eval_frames_matrix, batches of 32), each output frame reduced to a 32-B
record (alsub_frame_summary) and the records all-gathered over NCCL.  --config 5 prints that
measurement as the line itself.

--gpus N without torchrun (WORLD_SIZE unset) re-launches itself under torch.distributed.run with N
ranks.  --dry-run exercises that launch and the record gather on CPU (gloo), no GPU work.

--impl reference: the CPU oracle (oracle/, plain C) timed on this host on a bounded sample of the
same workload -- rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import meshgen as mg  # noqa: E402

METRIC = "refined faces/sec per level (topo+geometry) and achieved HBM GB/s vs B200 peak"
PAPER_CONTEXT = "ArmorGuy CC level 6 (35.2M faces) in ~40 ms on a GTX 1080 Ti (PAPER.md P:L91, P:L735)"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------------------------------------
# algorithmic bytes: every array a kernel touches, read or written once
# ------------------------------------------------------------------------------------------
def level_counts(m, levels):
    """Per-level counts from the library (alsub_level_counts)."""
    out = []
    for l in range(levels + 1):
        c = m.counts(l)
        out.append(dict(V=c["verts"], F=c["faces"], S=c["face_slots"], E=c["edges"], B=c["boundary_edges"], level=l))
    return out


def kernel_bytes_cc(name, c, prev, lvl, levels, prev2=None, gp_mid=False):
    """Algorithmic bytes of one launch of a CC level kernel: every array the kernel
    reads or writes, counted once, split into
      "method"       -- the method's own data: parent topology and positions in, child topology and
                        refined positions out (what any implementation of the level must move)
      "intermediate" -- this implementation's scratch: the face kernel's corner sums c0 and half ring
                        sums hs (written by the face kernel, read back by the vertex kernel).
    c = counts of the parent level lvl, prev = level lvl-1.  Mirrors the plan in api.cu: the last
    refined level (lvl = levels-1 >= 2) recomputes its edge rows from the grandparent and iterates
    the grandparent's edges, so level levels-1 never stores face_edge / face_twin / edge pairs;
    twins are only stored where the next level emits adjacency.  gp_mid: level levels-2 (>= 3, crease
    rules not fused) also iterates the grandparent's edges (cc_use_gp in api.cu): no half sums,
    compact corner sums, the edge kernel finishes the edge points born at lvl and lvl-1."""
    V, F, S, E = c["V"], c["F"], c["S"], c["E"]
    Fp = prev["F"] if prev else 0
    Ep = prev["E"] if prev else 0
    Fq = prev2["F"] if (prev2 and lvl >= 3) else 0   # face points born at lvl-1 (face-kernel shuffle)
    Eq = prev2["E"] if (prev2 and lvl >= 2) else 0   # edge points born at lvl-1 (last level: edge kernel)
    adj = lvl < levels - 1                        # this level emits child adjacency
    gp_last = levels >= 3 and lvl == levels - 1   # grandparent path at the last level
    gp = gp_last or (gp_mid and lvl == levels - 2 and lvl >= 3)
    child_rows = adj and not (levels >= 3 and lvl + 1 == levels - 1)  # child face_edge / edge pairs stored
    child_twin = lvl + 2 < levels
    fpv = lvl >= 2
    inter = 0
    if name == "cc_face":
        rd = 4 * S + 12 * V + (48 * Fp if gp_last else 4 * S) + (4 * S if child_rows else 0)
        wr = 12 * F + 16 * S + (16 * S if child_rows else 0) + (16 * S if child_twin else 0)
        wr += 12 * Fp if fpv else 0               # vertex points of the face points born at lvl
        wr += 12 * Fq                             # vertex points of the face points born at lvl-1
        inter += 12 * F if (fpv and not gp) else 0  # half ring sums hs (none on the grandparent path)
        # corner-0 contributions c0; the grandparent path (>= 3) keeps only faces r = 0 mod 4, compacted
        inter += (12 * ((F + 3) // 4) if (gp and lvl >= 3) else 12 * F) if lvl >= 1 else 0
    elif name == "cc_edge":
        if gp:
            rd = 8 * Ep + 16 * Fp + 12 * V + 12 * F
        else:
            rd = 8 * E + 4 * S + 12 * V + 12 * F
        wr = 12 * E + (8 * (2 * E + S) if child_rows else 0)
        wr += 12 * (Ep + Eq) if gp else 0         # vertex points of the edge points born at lvl, lvl-1
    elif name == "cc_vertex":
        if gp:  # vertices born before lvl-1 only: p in, S out; their faces' c0 sums
            nv = V - Fp - Ep - Fq - Eq
            return {"method": 12 * nv + 12 * nv, "intermediate": 12 * (F - 4 * Fq - 4 * Eq)}
        if Fq:  # the face points born at lvl-1 are done by the face kernel
            V = V - Fq
        if lvl >= 1:  # c0 sums for vertices born earlier, half sums for new edge points
            rd = 12 * V + 8 * Ep + (0 if fpv else 4 * S + 12 * F)
            inter = 12 * (F - 4 * Fq) + (12 * F if fpv else 0)
        else:
            rd = 4 * S + 12 * V + 12 * F
        wr = 12 * (V - (Fp if fpv else 0))
    else:
        return None
    return {"method": rd + wr, "intermediate": inter}


def survey_level_bytes_cc(c, final):
    """SURVEY.md 8(d) per-level compulsory model: read 4S + 4S + 16E + 12V, write 16F' + 12V'
    (+16F' face_edge' + 16E' edge tables when another level follows)."""
    V, F, S, E = c["V"], c["F"], c["S"], c["E"]
    Vn, Fn, En = V + F + E, S, 2 * E + S
    b = 8 * S + 16 * E + 12 * V + 16 * Fn + 12 * Vn
    if not final:
        b += 16 * Fn + 16 * En
    return b


# ------------------------------------------------------------------------------------------
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, dev_index, period=0.002):
        self.samples, self.reasons = [], 0
        self.period = period
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def shard(n, world, rank):
    """Contiguous block of n independent units (frames / meshes) owned by `rank`."""
    per = n // world
    extra = n % world
    lo = rank * per + min(rank, extra)
    return lo, lo + per + (1 if rank < extra else 0)


def bench_backend():
    """Process-group backend of the multi-rank bench: NCCL (the product path).  ALSUB_BENCH_BACKEND=gloo
    runs the same multi-rank code with gloo and host-side collectives, e.g. two ranks sharing one
    GPU (NCCL refuses duplicate devices) to exercise the N > 1 paths where only one GPU exists."""
    return os.environ.get("ALSUB_BENCH_BACKEND", "nccl")


def coll_device(dev):
    """Device of the collectives' tensors: the GPU for NCCL, the host for gloo."""
    import torch
    return dev if bench_backend() == "nccl" else torch.device("cpu")


def init_dist(local):
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if bench_backend() == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(bench_backend())
    return dev


def dist_max(x, device=None):
    """Max of a scalar over all ranks (timing only; no data-path collective)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return x
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_summaries(local, nframes, world, rank, device=None):
    """All-gather every rank's per-frame summary records (int32 [per_rank][8], frames f_lo .. f_hi
    of shard()) into one [nframes][8] table in frame order -- the only data-path collective of the
    sharded frames job (32 B per frame over NCCL instead of the frames)."""
    import torch
    import torch.distributed as dist
    per_max = max(hi - lo for lo, hi in (shard(nframes, world, r) for r in range(world)))
    buf = torch.zeros((per_max, 8), dtype=torch.int32, device=device)
    buf[:local.shape[0]] = local.to(buf.device)
    if world == 1 or not (dist.is_available() and dist.is_initialized()):
        return buf[:nframes]
    out = torch.empty((world * per_max, 8), dtype=torch.int32, device=device)
    dist.all_gather_into_tensor(out, buf)
    parts = []
    for r in range(world):
        lo, hi = shard(nframes, world, r)
        parts.append(out[r * per_max:r * per_max + (hi - lo)])
    return torch.cat(parts)


def host_cpu():
    """(model name, logical cores) of this host, for the oracle baseline's context."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count()


def cpu_oracle_baseline(mesh, levels, label):
    """The oracle as it stands on this host: the full workload level by level,
    once single-threaded (liboracle.so) and once on every host core (the same source built with
    OpenMP over its single-writer per-element loops; the edge sort stays serial).  value = the
    faster run's final-level faces/s (cores = its thread count); both runs' per-level times are
    reported."""
    import oracle
    oracle.build()
    model, ncpu = host_cpu()
    runs = {}
    for threads in (1, ncpu):
        t = []
        t0 = time.perf_counter()
        if threads == 1:
            recs = oracle.refine(mesh, "cc", levels, times=t)
            used = 1
        else:
            used = oracle.lib_threads(threads)[1]
            recs = oracle.refine(mesh, "cc", levels, threads=threads, times=t)
        dt = time.perf_counter() - t0
        F = recs[-1]["F"]
        del recs
        runs[used] = {"seconds": dt, "level_seconds": t, "faces_per_s": F / dt}
    best = max(runs, key=lambda k: runs[k]["faces_per_s"])  # the faster of the two runs
    ncpu_used = max(runs)
    return {"value": runs[best]["faces_per_s"], "unit": "faces/s", "cores": best, "kind": "oracle",
            "sample": f"{label}: CC levels 0->{levels} ({F} faces), C oracle (fp64), "
                      f"{runs[1]['seconds']:.2f} s on 1 thread, {runs[ncpu_used]['seconds']:.2f} s on {ncpu_used}",
            "runs": {str(k): v for k, v in runs.items()}, "host_cpu": model, "host_cores": ncpu}


def cpu_oracle_frames(mesh, levels, frames, nframes):
    """Config 5 on the oracle: the listed frames (each a full CC evaluation of the deformed control
    mesh), faces/s extrapolated from the per-frame time."""
    import oracle
    oracle.build()
    t0 = time.perf_counter()
    F = 0
    for t in frames:
        mm = dict(mesh)
        mm["pos"] = mg.frame_positions(mesh["pos"], t, nframes)
        F = oracle.refine(mm, "cc", levels)[-1]["F"]
    dt = (time.perf_counter() - t0) / len(frames)
    model, ncpu = host_cpu()
    return {"value": F / dt, "unit": "faces/s", "cores": 1, "kind": "oracle",
            "sample": f"frames {list(frames)} of {nframes} (armor50k CC L{levels}, {F} faces each): "
                      f"{dt:.2f} s per frame, single-threaded C oracle (fp64); extrapolated to "
                      f"{nframes} frames = {dt * nframes:.0f} s", "extrapolated": True,
            "host_cpu": model, "host_cores": ncpu}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    mesh = mg.armor9k()
    levels = args.ref_levels or (5 if args.steps <= 12 else 4)
    times = []
    F = None
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        recs = oracle.refine(mesh, "cc", levels)
        dt = time.perf_counter() - t0
        F = recs[-1]["F"]
        del recs
        if i >= args.warmup:
            times.append(dt)
    ms = 1000 * sum(times) / len(times)
    value = F / (ms / 1000)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "faces/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "armor9k_cc_L6 (config 3), bounded sample", "scheme": "catmull-clark",
                       "levels_sampled": levels, "faces_out": F},
            "cpu_baseline": {"value": value, "unit": "faces/s", "cores": 1, "kind": "oracle",
                             "sample": f"armor9k CC levels 0->{levels} ({F} faces) per step, single-threaded C oracle",
                             "host_cpu": host_cpu()[0], "host_cores": host_cpu()[1]},
            "e2e": {"value": value, "unit": "faces/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_alsub(args):
    import torch
    import torch.distributed as dist
    from paper_1809_06047_b200 import Mesh

    rank, world, local = dist_env()
    if world > 1:
        dev = init_dist(local)
    else:
        dev = torch.device("cuda", local)
        torch.cuda.set_device(dev)
    cdev = coll_device(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        return dist_max(x, cdev)

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2
    peak, peak_src = peaks()

    levels = args.levels
    mesh = mg.armor9k(seed=mg.SEED_TOPO + rank)
    stream = torch.cuda.current_stream()
    m = Mesh(torch.from_numpy(mesh["face_off"]).to(dev), torch.from_numpy(mesh["face_vtx"]).to(dev),
             torch.from_numpy(mesh["pos"]).to(dev), torch.from_numpy(mesh["crease"]).to(dev),
             torch.from_numpy(mesh["sigma"]).to(dev))
    m.refine("cc", levels)  # plan + eager run
    m.refine("cc", levels)  # records the CUDA graph
    cnt = level_counts(m, levels)
    Fout, Vout = cnt[-1]["F"], cnt[-1]["V"]
    special = len(mesh["crease"]) > 0 or cnt[0]["B"] > 0

    def gp_mid_at(lvl):  # mirrors cc_use_gp (api.cu): the grandparent edge kernel at level levels-2
        return (lvl == levels - 2 and lvl >= 3 and not (special and cnt[lvl]["V"] < (1 << 20))
                and os.environ.get("ALSUB_NO_GP_MID") != "1")

    for _ in range(args.warmup):
        flush.fill_(1.0)
        m.refine("cc", levels)
    torch.cuda.synchronize()
    launches_per_step = m.last_launch_count

    # ---- per-kernel timing (CUDA events between launches, eager), averaged over reps: the
    # per-level table and the choice of the dominant kernel (before the timed region) ----
    reps = max(3, min(10, args.steps))
    acc = {}
    for _ in range(reps):
        flush.fill_(2.0)
        for name, lvl, ms in m.refine_profile("cc", levels):
            acc.setdefault((name, lvl), []).append(ms)
    kt = {k: sum(v) / len(v) for k, v in acc.items()}
    prof_step = sum(kt.values())
    (dname, dlvl), dms_profile = max(kt.items(), key=lambda kv: kv[1])
    # the dominant kernel is then timed INSIDE the timed region: alsub_probe puts two event-record
    # nodes around its launch in the refine's CUDA graph, one event pair per replay
    K = args.steps
    m.probe(dlvl, dname, K)
    flush.fill_(1.0)
    m.refine("cc", levels)   # re-captures the graph with the probe nodes (untimed)
    m.probe(dlvl, dname, K)  # same probe: only resets the pair counter
    torch.cuda.synchronize()
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    sampler = ClockSampler(dev.index)
    barrier()
    torch.cuda.synchronize()
    with sampler:
        for i in range(K):
            flush.fill_(float(i))
            ev0[i].record(stream)
            m.refine("cc", levels)
            ev1[i].record(stream)
        torch.cuda.synchronize()
    barrier()
    probe_ms = m.probe_read()
    step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    total_ms = max_over_ranks(sum(step_ms))
    ms_per_step = total_ms / K
    value = world * Fout * K / (total_ms / 1000.0)
    srt = sorted(step_ms)
    step_pct = {"p10": srt[int(0.1 * (K - 1))], "median": srt[(K - 1) // 2], "p90": srt[int(0.9 * (K - 1))],
                "note": "this rank's per-step CUDA-event times (SURVEY 8(d) timing protocol)"}

    ncu_kernels = {}
    prof_sum = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof_sum):
        try:
            ncu_kernels = json.load(open(prof_sum)).get("kernels", {})
        except Exception:
            ncu_kernels = {}
    per_level = []
    for lvl in range(-1, levels):
        ks = {n: t for (n, l), t in kt.items() if l == lvl}
        row = {"level": lvl, "ms": sum(ks.values())}
        if lvl >= 0:
            c = cnt[lvl]
            final = lvl == levels - 1
            sb = survey_level_bytes_cc(c, final)
            row.update(faces_out=cnt[lvl + 1]["F"], survey_bytes=sb,
                       survey_GBps=sb / (row["ms"] * 1e6) if row["ms"] > 0 else None)
            row["survey_frac"] = row["survey_GBps"] / peak if row["survey_GBps"] else None
            kk = {}
            for n, t in ks.items():
                b = kernel_bytes_cc(n, c, cnt[lvl - 1] if lvl > 0 else None, lvl, levels,
                                    cnt[lvl - 2] if lvl > 1 else None, gp_mid=gp_mid_at(lvl))
                mb = b["method"] if b else None
                kk[n] = {"ms": t, "alg_bytes": mb, "intermediate_bytes": b["intermediate"] if b else None,
                         "GBps": (mb / (t * 1e6)) if mb else None, "frac": (mb / (t * 1e6) / peak) if mb else None}
                nc = ncu_kernels.get(f"{n}@L{lvl}")
                if nc and mb:  # ncu DRAM bytes of the same launch (profiles/ncu_summary.json)
                    kk[n]["dram_bytes"] = nc["dram_bytes"]
                    kk[n]["waste"] = nc["dram_bytes"] / mb  # DRAM traffic / method bytes
                    # the HBM the kernel actually keeps busy: its DRAM bytes over this run's time
                    kk[n]["dram_GBps"] = nc["dram_bytes"] / (t * 1e6)
                    kk[n]["dram_frac"] = kk[n]["dram_GBps"] / peak
            row["kernels"] = kk
        per_level.append(row)
    db = kernel_bytes_cc(dname, cnt[dlvl], cnt[dlvl - 1] if dlvl > 0 else None, dlvl, levels,
                         cnt[dlvl - 2] if dlvl > 1 else None, gp_mid=gp_mid_at(dlvl)) if dlvl >= 0 else None
    dbytes = db["method"] if db else None
    dms = sum(probe_ms) / len(probe_ms) if probe_ms else dms_profile
    achieved = dbytes / (dms * 1e6) if dbytes else None
    traffic = ncu_kernels.get(f"{dname}@L{dlvl}", {}).get("dram_bytes")
    roofline = {"bound": "hbm", "kernel": f"{dname} (level {dlvl}->{dlvl + 1})", "achieved": achieved,
                "peak": peak, "unit": "GB/s", "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "alg_bytes_per_launch": dbytes,
                "alg_bytes_note": "method bytes only (parent topology + positions in, child topology + refined "
                                  "positions out); the kernel's scratch writes (corner sums c0, half sums hs) are "
                                  "in intermediate_bytes_per_launch, not in achieved",
                "intermediate_bytes_per_launch": db["intermediate"] if db else None,
                "waste": (traffic / dbytes) if (traffic and dbytes) else None,
                "avg_launch_ms": dms, "share_of_step": dms / ms_per_step,
                "share_of_kernel_time": dms_profile / prof_step,  # comparable with the ncu launch list
                                                                  # (serialised kernels, no branch overlap)
                "launches_timed": len(probe_ms),
                "timing": "CUDA events recorded by event-record nodes around the kernel inside every "
                          "replayed refine graph of the timed region (alsub_probe), on its own stream",
                "profile_pass_ms": dms_profile, "peak_source": peak_src}

    # ---- the last level's crease lists (not in the timed step): built on first export ----
    lazy = last_level_lists_ms(m, levels)

    # ---- e2e through the C ABI with host buffers (every rank its replica; the slowest rank) ----
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, mesh, levels, Fout, Vout, dev, flush)
        ms_e2e = max_over_ranks(e2e["ms_per_step"])
        e2e.update(value=world * Fout / (ms_e2e / 1000.0), ms_per_step=ms_e2e,
                   h2d_bytes_per_step=world * e2e["h2d_bytes_per_step"], d2h_bytes_per_step=world * e2e["d2h_bytes_per_step"])

    others = None
    if rank == 0 and world == 1 and not args.no_other_configs:
        others = other_configs(dev, flush, peak)
    frames = None
    if not args.no_frames:  # every rank: config 5's frames are split over all of them
        del flush
        torch.cuda.empty_cache()
        frames = run_frames(args, rank, world, dev, barrier, max_over_ranks, peak, peak_src)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_baseline(mg.armor9k(), levels, "armor9k (config 3), the full workload")

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "faces/s", "n_gpus": world, "steps": K,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": f"armor9k_cc_L{levels} (SURVEY config 3)", "scheme": "catmull-clark",
                           "levels": levels, "control_faces": int(len(mesh["face_off"]) - 1),
                           "faces_out": int(Fout), "verts_out": int(Vout),
                           "l2": "256 MiB buffer written between timed steps (L2 flush)",
                           "parallelism": f"{world} independent mesh replicas" if world > 1 else "single GPU",
                           "graph": True},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches_per_step * K), "launches_per_step": int(launches_per_step),
                "step_ms": step_pct,
                "clocks": sampler.summary(), "levels": per_level, "profile_step_ms": prof_step,
                "last_level_crease_lists": lazy,
                "other_configs": others, "frames": frames,
                "paper_context": PAPER_CONTEXT}
        print(json.dumps(line), flush=True)
    m.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def last_level_lists_ms(m, levels):
    """The crease inheritance of the last refined level (its child crease pairs / sigma and the
    special-vertex rows) is not part of alsub_refine: nothing in the step reads it, so
    the first export after a refine builds it (ensure_last_lists, one k_crease launch).  The export
    around it is host-bound (ms), so its time comes from the committed ncu capture of that launch
    (profiles/r02_lazy_lists.json)."""
    p = os.path.join(ROOT, "profiles", "r02_lazy_lists.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    return {"in_step": False, "ncu_us": d.get("time_us"), "kernel": d.get("kernel"),
            "source": "profiles/r02_lazy_lists.json" if d else None,
            "note": "built lazily on the first export after a refine, outside the timed step (no kernel of the "
                    "step reads the last level's crease lists)"}


def other_configs(dev, flush, peak, reps=20):
    """Graph-replayed timings of the other BASELINE configs:
    refined faces/s of the final level and the SURVEY per-level compulsory-byte rate."""
    import torch
    from paper_1809_06047_b200 import Mesh
    cases = [("config1_cube_cc_L3", mg.cube(), "cc", 3), ("config2a_ico_loop_L6", mg.icosahedron(), "loop", 6),
             ("config2b_creased_tet_loop_L6", mg.tetrahedron(creased=True), "loop", 6),
             ("config2b_creased_tet_cc_L6", mg.tetrahedron(creased=True), "cc", 6),
             ("config4_torus100k_sqrt3_L5", mg.torus100k(), "sqrt3", 5)]
    out = {}
    stream = torch.cuda.current_stream()
    for name, mesh, scheme, L in cases:
        m = Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"])
        for _ in range(4):
            m.refine(scheme, L)
        ts = []
        for _ in range(reps):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            m.refine(scheme, L)
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        ms = ts[len(ts) // 2]
        c = m.counts(L)
        cp = m.counts(L - 1)
        row = {"scheme": scheme, "levels": L, "faces_out": c["faces"], "verts_out": c["verts"], "ms_median": ms,
               "faces_per_s": c["faces"] / (ms / 1e3), "launches": m.last_launch_count}
        if scheme == "sqrt3":  # final step bytes: read 12F + 12F (face rows, twins) + 12V, write 36F + 12V'
            fb = 24 * cp["faces"] + 12 * cp["verts"] + 36 * cp["faces"] + 12 * c["verts"]
            row["final_step_compulsory_bytes"] = fb
        out[name] = row
        m.close()
    return out


def run_e2e(args, mesh, levels, Fout, Vout, dev, flush):
    """Same metric through the public C ABI with HOST buffers: per step alsub_mesh_create from pinned
    host arrays (H2D inside), alsub_refine (eager, one-shot), positions + faces back to pinned host."""
    import torch
    from paper_1809_06047_b200 import Mesh
    pin = lambda a: torch.from_numpy(a).pin_memory()
    fo, fv, P, cr, sg = pin(mesh["face_off"]), pin(mesh["face_vtx"]), pin(mesh["pos"]), pin(mesh["crease"]), pin(mesh["sigma"])
    out_P = torch.empty((Vout, 3), dtype=torch.float32).pin_memory()
    out_F = torch.empty(4 * Fout, dtype=torch.int32).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in (fo, fv, P, cr, sg))
    d2h = out_P.numel() * 4 + out_F.numel() * 4
    from paper_1809_06047_b200 import alsub as A
    L = A.lib()
    stream = torch.cuda.current_stream()
    steps = max(2, min(args.steps, 5))
    times = []
    for i in range(1 + steps):
        flush.fill_(3.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        m = Mesh(fo, fv, P, cr, sg)
        m.refine("cc", levels)
        A._check(L.alsub_level_positions(m._h, levels, out_P.data_ptr(), stream.cuda_stream))
        A._check(L.alsub_level_topology(m._h, levels, out_F.data_ptr(), None, None, None, None, None, None,
                                        stream.cuda_stream))
        e1.record(stream)
        torch.cuda.synchronize()
        m.close()
        if i > 0:
            times.append(e0.elapsed_time(e1))
    ms = sum(times) / len(times)
    return {"value": Fout / (ms / 1000.0), "unit": "faces/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": ms,
            "path": "alsub_mesh_create(host) + alsub_refine + alsub_level_positions/topology(pinned host)"}


def device_frames(P0, t0, n, nframes, dev):
    """Frames t0 .. t0+n-1 of config 5 generated on the device (P0 rotated by
    2 pi t / nframes about z plus 0.05 sin(2 pi t / 64 + 7 x) along y), float32 [n][V0][3].  Input
    generation only (meshgen.frame_positions is the host definition the parity tests use)."""
    import torch
    p = torch.from_numpy(P0).to(dev, torch.float64)
    t = torch.arange(t0, t0 + n, device=dev, dtype=torch.float64)[:, None]
    th = 2 * math.pi * t / nframes
    c, s_ = torch.cos(th), torch.sin(th)
    x = c * p[None, :, 0] - s_ * p[None, :, 1]
    y = s_ * p[None, :, 0] + c * p[None, :, 1] + 0.05 * torch.sin(2 * math.pi * t / 64 + 7 * p[None, :, 0])
    z = p[None, :, 2].expand(n, -1)
    return torch.stack([x, y, z], dim=2).to(torch.float32).contiguous()


def run_frames(args, rank, world, dev, barrier, max_over_ranks, peak, peak_src):
    """Config 5: 4096 animation frames of armor50k (CC level 4) split over the ranks (contiguous
    blocks, strong scaling).  Each rank builds the topology and the refinement matrix itself, then
    streams its frames through alsub_eval_frames_matrix in batches of 32 into two output buffers;
    every output frame is reduced to a 32-B record (alsub_frame_summary, side stream, overlapped with
    the next batch) and the records are all-gathered over NCCL -- the job's only data-path
    collective.  Returns the measurement on rank 0 (None elsewhere)."""
    import torch
    import torch.distributed as dist
    from paper_1809_06047_b200 import Mesh, frame_summary
    levels, nframes, nb = 4, args.frames, 32
    mesh = mg.armor50k()
    f_lo, f_hi = shard(nframes, world, rank)
    per_rank = f_hi - f_lo
    m = Mesh(mesh["face_off"], mesh["face_vtx"], mesh["pos"], mesh["crease"], mesh["sigma"])
    m.refine("cc", levels)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    info = m.build_refinement_matrix(levels)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    blk = m.refinement_matrix_blocks()
    cnt = level_counts(m, levels)
    Vout, Fout, V0 = cnt[-1]["V"], cnt[-1]["F"], cnt[0]["V"]
    frames = device_frames(mesh["pos"], f_lo, per_rank, nframes, dev)  # this rank's inputs, in HBM
    outs = [torch.empty((nb, Vout, 3), dtype=torch.float32, device=dev) for _ in range(2)]
    summ = torch.zeros((max(per_rank, 1), 8), dtype=torch.int32, device=dev)
    nbatch = (per_rank + nb - 1) // nb
    stream = torch.cuda.current_stream()

    def batch(i):
        # the frame records are folded into the evaluation (alsub_eval_frames_matrix_summary): the
        # output frames are not read back; two output buffers alternate (a consumer would overlap
        # its reads of one with the evaluation into the other)
        lo, hi = i * nb, min(per_rank, (i + 1) * nb)
        m.eval_frames_matrix_summary(frames[lo:hi], out=outs[i % 2][:hi - lo], summary=summ[lo:hi])

    for i in range(min(max(args.warmup, 1), nbatch)):
        batch(i)
    torch.cuda.synchronize()
    # the fused records must equal a separate summary pass over the frames written (the last
    # warm-up batch's buffer)
    iw = min(max(args.warmup, 1), nbatch) - 1
    lo, hi = iw * nb, min(per_rank, (iw + 1) * nb)
    records_ok = bool(torch.equal(frame_summary(outs[iw % 2][:hi - lo]), summ[lo:hi]))
    e0, eg, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    sampler = ClockSampler(dev.index)
    barrier()
    torch.cuda.synchronize()
    with sampler:
        e0.record(stream)
        for i in range(nbatch):
            batch(i)
        eg.record(stream)
        table = gather_summaries(summ[:per_rank], nframes, world, rank, device=coll_device(dev))
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    local_ms = e0.elapsed_time(e1)
    gather_ms = eg.elapsed_time(e1)
    ms = max_over_ranks(local_ms)
    # the same frames through the plain evaluation (no records): what the records cost
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    a0.record(stream)
    for i in range(nbatch):
        lo, hi = i * nb, min(per_rank, (i + 1) * nb)
        m.eval_frames_matrix(frames[lo:hi], out=outs[i % 2][:hi - lo])
    a1.record(stream)
    torch.cuda.synchronize()
    eval_ms = max_over_ranks(a0.elapsed_time(a1))
    # which GPUs took part: every rank reports its device; NCCL's communicator size
    uuid = str(getattr(torch.cuda.get_device_properties(dev), "uuid", dev.index))
    if world > 1:
        names = [None] * world
        dist.all_gather_object(names, (rank, uuid))
        gpus_active = len({u for _, u in names})
    else:
        gpus_active = 1
    comm_ok = (dist.get_world_size() if world > 1 else 1) == args.gpus
    # algorithmic bytes of one batch of nb frames through the blocked matrix: the weights and row
    # ids once, the control positions in (12 V0 per frame) and the refined frames out (12 V_L)
    bytes_frame = 12 * Vout + 12 * V0 + (4 * blk["weights"] + 4 * Vout) / nb
    per_gpu_gbps = per_rank * bytes_frame / (local_ms * 1e6) if local_ms else None
    value = nframes * Fout / (ms / 1e3)
    res = None
    if rank == 0:
        res = {"workload": f"armor50k_cc_L{levels}_frames{nframes} (SURVEY config 5)", "value": value,
               "unit": "faces/s", "ms": ms, "us_per_frame": 1e3 * ms / nframes * world,
               "eval_only_us_per_frame": 1e3 * eval_ms / nframes * world,
               "eval_only_value": nframes * Fout / (eval_ms / 1e3),
               "frames": nframes, "frames_per_rank": per_rank, "batch": nb, "faces_per_frame": Fout,
               "scaling": "strong", "n_gpus": world, "gpus_active": gpus_active, "comm_nranks_ok": comm_ok,
               "path": "alsub_eval_frames_matrix (blocked refinement matrix, P:L809)",
               "matrix": {"rows": info["rows"], "nnz": info["nnz"], "chunks": blk["chunks"],
                          "block_weights": blk["weights"], "build_s": build_s},
               "roofline": {"bound": "hbm", "achieved": per_gpu_gbps, "peak": peak, "unit": "GB/s",
                            "frac": per_gpu_gbps / peak if per_gpu_gbps else None,
                            "bytes_per_frame": bytes_frame,
                            "note": "per GPU (rank 0): 12 V_L out + 12 V_0 in per frame + weights and "
                                    "row ids once per batch of 32", "peak_source": peak_src},
               "per_gpu_hbm_frac": per_gpu_gbps / peak if per_gpu_gbps else None,
               "summaries": {"frames_gathered": int(table.shape[0]), "bytes_per_frame": 32,
                             "collective": f"all_gather_into_tensor ({bench_backend()})" if world > 1 else "none (1 rank)",
                             "gather_ms": gather_ms, "fused_into_eval": True,
                             "equal_to_alsub_frame_summary": records_ok},
               "gpu_launches": int(m.last_launch_count * nbatch), "clocks": sampler.summary(),
               "l2": "inputs and outputs far larger than L2"}
    m.close()
    return res


def run_frames_line(args):
    """--config 5: the frames measurement as the JSON line itself."""
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world > 1:
        dev = init_dist(local)
    else:
        dev = torch.device("cuda", local)
        torch.cuda.set_device(dev)
    peak, peak_src = peaks()
    fr = run_frames(args, rank, world, dev, (lambda: dist.barrier()) if world > 1 else (lambda: None),
                    lambda x: dist_max(x, coll_device(dev)), peak, peak_src)
    if rank == 0:
        line = {"metric": METRIC, "value": fr["value"], "unit": "faces/s", "n_gpus": world, "steps": 1,
                "warmup": args.warmup, "ms_per_step": fr["ms"], "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": fr["workload"], "frames": fr["frames"], "batch": fr["batch"],
                           "l2": fr["l2"], "parallelism": f"frames sharded over {world} GPUs"},
                "roofline": dict(fr["roofline"], traffic=None), "frames": fr,
                "cpu_baseline": (cpu_oracle_frames(mg.armor50k(), 4, (0,), fr["frames"])
                                 if (world == 1 and not args.no_cpu_baseline) else None),
                "e2e": None, "gpu_launches": fr["gpu_launches"], "clocks": fr["clocks"]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def dry_run(args):
    """--dry-run: the multi-rank plumbing without a GPU -- gloo process group, every rank fills its
    shard of per-frame records, rank 0 gathers them (gather_summaries) and prints the rank map."""
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    lo, hi = shard(args.frames, world, rank)
    local = torch.arange(lo, hi, dtype=torch.int32)[:, None].repeat(1, 8)
    table = gather_summaries(local, args.frames, world, rank)
    names = [None] * world
    if world > 1:
        dist.all_gather_object(names, (rank, os.getpid()))
    else:
        names = [(0, os.getpid())]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "requested": args.gpus,
                          "ranks": [r for r, _ in names], "pids": len({p for _, p in names}),
                          "frames_gathered": int(table.shape[0]),
                          "frame_order_ok": bool((table[:, 0] == torch.arange(args.frames, dtype=torch.int32)).all())}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def relaunch(args):
    """--gpus N with WORLD_SIZE unset: run this script under torch.distributed.run with N ranks
    (127.0.0.1 rendezvous, a free port); returns its exit code."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--dry-run", action="store_true", help="multi-rank plumbing on CPU (gloo), no GPU")
    ap.add_argument("--no-frames", action="store_true", help="skip the config-5 frames measurement")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="alsub", choices=["alsub", "reference"])
    ap.add_argument("--config", type=int, default=3, choices=[3, 5])
    ap.add_argument("--levels", type=int, default=6)
    ap.add_argument("--frames", type=int, default=4096)
    ap.add_argument("--ref-levels", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if args.dry_run:
        return dry_run(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.config == 5:
        return run_frames_line(args)
    return run_alsub(args)


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python
"""Benchmark: decoded Gbps of batched Min-Sum LDPC decoding on B200 (BASELINE.json "metric").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl reference]
    python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...   (one process per GPU)

`--gpus N` without torchrun's environment re-launches itself through torch.distributed.run with N
ranks (127.0.0.1 rendezvous), one process per GPU over NCCL.

A step is one pass of the whole hot path over this rank's batch (steps a2-a7 of SURVEY 8(a) with H
already ingested): stage-in, check-node / bit-node sweeps with the fused syndrome and per-frame early
stop, stage-out and counters.  The default workload is config C3 (random H with 5G-NR BG1 lifted
dimensions 17664 x 26112, 65,536 frames over Eb/N0 {2, 3, 3.5, 4, 5} dB, max_iter 20), the largest
configuration of BASELINE.json that fits one GPU; C1-C6 are selectable (`--config`).  C5 decodes all
16 codes (16 handles) per step.

Scaling: frames are keyed by their global index, so a frame decodes identically on any rank.  Weak
scaling (default): rank r of N decodes its own full batch (global frames r F .. (r+1) F).  Strong
(`--strong`, default for C4 as SURVEY 8(d) specifies): the config's F frames are split over the N
ranks.  The only collectives are the barrier, the MAX of the elapsed time and the SUM of the counters.

value = (frames decoded by all ranks) * n / (max-over-ranks device time of the K timed steps), Gbit/s.
The timed steps run the product path (CUDA-graph loop, no per-kernel events); the per-kernel split
behind `roofline` comes from one separate profiled step (per-kernel CUDA events, plain launches).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from gen import channel, codes  # noqa: E402

METRIC = "decoded Gbps (1/2/4/8 B200) at fixed max_iter; % of HBM roofline"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback
DEFAULT_CONFIG = "c3"
DEFAULT_SCALING = {"c4": "strong"}  # C4's 16,384 frames are sharded over the GPUs


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("sm_max_mhz", 1965.0)), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM, 1965.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ launcher / distributed ---
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_if_needed(args, argv):
    """`--gpus N` (N > 1) outside torchrun: re-exec as N ranks through torch.distributed.run."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + argv
        sys.stdout.flush()
        sys.stderr.flush()
        os.execv(sys.executable, cmd)


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    info = {"backend": None, "world": world}
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        cuda = torch.cuda.is_available() and not args.dry_run
        backend = "nccl" if cuda else "gloo"
        if cuda:
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        # NCCL builds its communicator lazily: force it now (outside any timed region) and log it
        t = torch.ones(1, device=torch.device("cuda", local) if cuda else "cpu")
        dist.all_reduce(t)
        ver = ".".join(map(str, torch.cuda.nccl.version())) if cuda else None
        info = {"backend": backend, "world": world, "nccl_version": ver, "all_reduce_check": int(t.item())}
        print(f"[bench] rank {rank}/{world} local_rank {local}: {backend} process group up"
              + (f" (NCCL {ver})" if ver else "") + f", all_reduce(1) = {int(t.item())}", file=sys.stderr, flush=True)
    if args.gpus != world and rank == 0:
        print(f"[bench] warning: --gpus {args.gpus} but WORLD_SIZE={world}; reporting n_gpus={world}",
              file=sys.stderr)
    return rank, world, local, info


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def reduce_max(x: float, world: int, dev) -> float:
    if world == 1:
        return x
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum_(t, world):
    if world > 1:
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


# ------------------------------------------------------------------ clocks -------------------
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap", "power.draw"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={','.join(self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, pw, reasons = [], [], [], set()
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(name)
            try:
                pw.append(float(parts[6]))
            except (IndexError, ValueError):
                pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
               "samples": len(sm)}
        if pw:
            out["power_w_median"] = statistics.median(pw)
        return out


# ------------------------------------------------------------------ workload -----------------
def code_list(cfg):
    c = cfg["code"]()
    return c if isinstance(c, list) else [c]


def scaling_of(args):
    if args.strong:
        return "strong"
    if args.weak:
        return "weak"
    return DEFAULT_SCALING.get(args.config, "weak")


def rank_shard(cfg, rank, world, scaling):
    """(w0, count, goff): this rank decodes workload frames w0 .. w0+count of the config's batch (whose
    index w sets the Eb/N0 block), generated at global frame index g = w + goff."""
    F = cfg["frames"]
    if scaling == "strong":
        lo, hi = codes.shard_range(F, rank, world)
        return lo, hi - lo, 0
    return 0, F, rank * F


def gen_frames(code, cfg, seed, w0, count, goff, device="cpu", out=None):
    """LLRs of workload frames [w0, w0+count) (all-zero codeword, BPSK/AWGN, keyed by global index)
    and the Eb/N0 block index of each."""
    pts = codes.point_ranges(cfg["frames"], len(cfg["ebn0"]))
    if out is None:
        out = torch.empty((count, code.n), dtype=torch.float32, device=device)
    pidx = np.zeros(count, np.int64)
    for p, (lo, hi) in enumerate(pts):
        a, b = max(lo, w0), min(hi, w0 + count)
        if a >= b:
            continue
        channel.bpsk_awgn(code.n, code.rate, cfg["ebn0"][p], seed, p, a + goff, b - a, device=device,
                          out=out[a - w0:b - w0])
        pidx[a - w0:b - w0] = p
    return out, pidx


def seed_of(cfg, h):
    return cfg["seed"] + h  # C5: code h is decoded with its own frames (seeds 4096 + h)


def describe(cfg_name, cfg, cl):
    te = cfg.get("check_every", 1)
    c = cl[0]
    what = (f"{len(cl)} codes {c.m}x{c.n} (nnz {c.nnz} each)" if len(cl) > 1 else
            f"{c.name} ({c.m}x{c.n}, nnz {c.nnz})")
    return (f"{cfg_name}: {what}, {cfg['frames']} frames per code over Eb/N0 {cfg['ebn0']} dB, max_iter "
            f"{cfg['max_iter']}" + (f", codeword test every {te} bodies" if te != 1 else "")
            + ", BPSK/AWGN all-zero codeword")


def config_dict(args, cfg, cl, world, scaling, frames_rank):
    """The `config` object of both arms (identical for --impl ours / reference)."""
    c = cl[0]
    F = cfg["frames"]
    gb = F * len(cl) * (world if scaling == "weak" else 1)
    return {"workload": describe(args.config, cfg, cl), "global_batch": gb, "frames_per_gpu": frames_rank * len(cl),
            "codes": len(cl), "m": c.m, "n": c.n, "nnz": c.nnz, "max_iter": cfg["max_iter"], "ebn0_db": cfg["ebn0"],
            "check_every": cfg.get("check_every", 1), "flags": args.flags,
            "parallelism": f"dp{world} (frame shards, {scaling} scaling, no data-path collective)",
            "l2": f"inputs {frames_rank * len(cl) * c.n * 4 / 1e9:.2f} GB per GPU > 126 MB L2 (no flush needed)",
            **({"code_streams": max(1, args.code_streams)} if len(cl) > 1 else {})}


def units(iters: np.ndarray, L: int, early: bool):
    """(check-node frame-bodies, bit-node frame-bodies): a frame stopping after k bodies is touched by
    min(k+1, L) check-node sweeps (the sweep of body k+1 finds its codeword) and k bit-node sweeps."""
    k = iters.astype(np.int64)
    if not early:
        return np.full_like(k, L), np.full_like(k, L)
    return (np.minimum(k + 1, L) if L > 0 else np.zeros_like(k)), k


def algorithmic_bytes(code, iters: np.ndarray, L: int, early: bool):
    """Bytes the method must move per frame with its state in HBM (SURVEY 8(d) B_comp split by sweep;
    DESIGN.md "Roofline"): check node = gather s (4n) + read and write the compressed row state
    (9m + E/8 each way; the first body reads none); bit node = read row state (9m + E/8) + r (4n) + write
    s (4n); I/O = llr in (4n) + posterior (4n) + bits (n) + k and isCodeword (5).  Returns (cn, bn, io)."""
    n, m, E = code.n, code.m, code.nnz
    state = 9 * m + E / 8
    cu, bu = units(iters, L, early)
    F = len(iters)
    cn = float(cu.sum()) * (4 * n + 2 * state) - (F * state if L > 0 else 0.0)
    bn = float(bu.sum()) * (8 * n + state)
    io = F * (9 * n + 5.0)
    return cn, bn, io


# Minimal per-element work of the method: per frame and edge, the check node
# does subtract, compare + two min updates + argmin select, sign parity, eta^prev rebuild (magnitude
# select, sign) and the syndrome bit = 9 lane operations; the bit node rebuilds eta (2) and adds (1).
OPS_CN, OPS_BN = 9, 3
# Of those, the ones that run on the ALU pipe (compare / min / select / logic; the subtract and the add
# run on the FMA pipe): 8 and 2.  The ALU pipe issues one warp instruction every 2 cycles per SM
# sub-partition (B300_MICROARCH.md "Pipe rates": alu rt_SMSP = 2), i.e. half the issue rate.
ALU_CN, ALU_BN = 8, 2


def ncu_traffic(cfg_name, kernel):
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of the kernel in the committed
    ncu --set full capture (profiles/ncu_traffic.json), with that launch's algorithmic bytes."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            e = json.load(f)[cfg_name][kernel]
        alg = e.get("algorithmic_bytes_this_launch")
        return (e["dram_bytes_per_launch"], round(e["dram_bytes_per_launch"] / alg, 3) if alg else None,
                e.get("source", "profiles/ncu_traffic.json"))
    except Exception:
        return None, None, None


# ------------------------------------------------------------------ our arm ------------------
def run_ours(args):
    import paper_2507_10424_b200 as P

    rank, world, local, dinfo = dist_setup(args)
    scaling = scaling_of(args)
    cfg = codes.CONFIGS[args.config]
    cl = code_list(cfg)
    w0, Fr, goff = rank_shard(cfg, rank, world, scaling)
    if args.dry_run:  # launcher / sharding check without a GPU: the rank's frames and their checksum
        c = cl[0]
        llr, _ = gen_frames(c, cfg, seed_of(cfg, 0), w0, Fr, goff)
        print(json.dumps({"dry_run": True, "rank": rank, "world": world, "scaling": scaling,
                          "workload_frames": [w0, w0 + Fr], "global_frames": [w0 + goff, w0 + goff + Fr],
                          "llr_sha1": hashlib.sha1(llr.numpy().tobytes()).hexdigest(), "dist": dinfo}), flush=True)
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()
        return
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    L = cfg["max_iter"]
    T = cfg.get("check_every", 1)
    n = cl[0].n
    # ---- per code: H ingested once (not timed), this rank's frames resident in HBM, output buffers
    jobs = []
    for hi, code in enumerate(cl):
        rr, cc = code.coo()
        h = P.Handle.from_coo(torch.from_numpy(rr).to(dev), torch.from_numpy(cc).to(dev), code.m, code.n,
                              flags=args.flags)
        if T != 1:
            h.set_check_every(T)
        llr, pidx = gen_frames(code, cfg, seed_of(cfg, hi), w0, Fr, goff, device=dev)
        out = P.DecodeResult(torch.empty((Fr, n), dtype=torch.uint8, device=dev),
                             torch.empty(Fr, dtype=torch.int32, device=dev),
                             torch.empty(Fr, dtype=torch.uint8, device=dev),
                             torch.empty((Fr, n), dtype=torch.float32, device=dev))
        jobs.append(dict(code=code, h=h, llr=llr, pidx=pidx, out=out,
                         stats=torch.zeros(8, dtype=torch.int64, device=dev)))
    stream = torch.cuda.current_stream()
    sched = jobs[0]["h"].schedule

    # several codes (C5): their decodes alternate over `--code-streams` side streams, so one code's tail
    # (its last frames, when most persistent CTAs have exited) overlaps the next code's start
    nside = args.code_streams if len(jobs) > 1 and args.code_streams > 1 else 0
    side = [torch.cuda.Stream(device=dev) for _ in range(nside)]

    def step(sequential=False):
        if sequential or not side:
            for j in jobs:  # one ldpc_decode per code over the rank's whole batch (the Eb/N0 blocks are just
                # frames: each frame's outputs do not depend on its batch, A19)
                j["h"].decode(j["llr"], L, posterior=True, stats=j["stats"], out=j["out"], stream=stream)
            return
        ev = torch.cuda.Event()
        ev.record(stream)
        for s_ in side:
            s_.wait_event(ev)
        for q, j in enumerate(jobs):
            j["h"].decode(j["llr"], L, posterior=True, stats=j["stats"], out=j["out"], stream=side[q % nside])
        for s_ in side:
            e2 = torch.cuda.Event()
            e2.record(s_)
            stream.wait_event(e2)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    for j in jobs:
        j["stats"].zero_()
    launches0 = sum(j["h"].launch_count for j in jobs)  # synchronises (device-side loop counters)
    sc0 = [j["h"].stream_counters() for j in jobs] if sched == "stream" else None
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    ms_local = e0.elapsed_time(e1)
    launches = sum(j["h"].launch_count for j in jobs) - launches0
    sc1 = [j["h"].stream_counters() for j in jobs] if sched == "stream" else None
    ms = reduce_max(ms_local, world, dev)
    tot_stats = reduce_sum_(sum(j["stats"] for j in jobs).clone(), world).cpu().numpy()

    # ---- one profiled step (per-kernel CUDA events on the launching stream; plain launches, no graph):
    # the per-kernel split and the roofline of the dominant kernel
    for j in jobs:
        j["h"].profile(True)
        j["h"].profile_reset()
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    step(sequential=True)  # per-kernel events bracket non-overlapping launches
    p1.record(stream)
    torch.cuda.synchronize()
    prof_step_ms = p0.elapsed_time(p1)
    prof = {}
    for j in jobs:
        for k, (nl, kms) in j["h"].profile_read().items():
            a = prof.setdefault(k, [0, 0.0])
            a[0] += nl
            a[1] += kms
        j["h"].profile(False)

    early = not (args.flags & P.FLAG_NO_EARLY_STOP)
    cn_b = bn_b = io_b = 0.0
    cu_sum = bu_sum = 0.0
    per_point, per_code_fer = [], []
    for j in jobs:
        it = j["out"].iters.cpu().numpy()
        a, b, c = algorithmic_bytes(j["code"], it, L, early)
        cn_b, bn_b, io_b = cn_b + a, bn_b + b, io_b + c
        cu, bu = units(it, L, early)
        cu_sum += float(cu.sum()) * j["code"].nnz
        bu_sum += float(bu.sum()) * j["code"].nnz
        rows = point_rows(j, cfg)
        per_point.append(rows)
        per_code_fer.append([r[2] / max(1, r[0]) for r in rows])
    per_point = np.sum(np.array(per_point, dtype=np.int64), axis=0)
    hbm, sm_mhz, peak_src = peaks()
    roof = roofline(args, sched, prof, prof_step_ms, cn_b, bn_b, io_b, cu_sum, bu_sum, hbm, sm_mhz, peak_src, ms_local,
                    args.steps)
    if roof is not None and sc0 is not None:
        # live frames per swept slot: frame-bodies the method needs / (tile-bodies swept x 128 slots)
        d = {k: sum(b[k] - a[k] for a, b in zip(sc0, sc1)) / args.steps for k in sc0[0]}
        fe_cn = cu_sum / cl[0].nnz if len(cl) == 1 else None
        fe_bn = bu_sum / cl[0].nnz if len(cl) == 1 else None
        roof["occupancy"] = {
            "check_node": round(fe_cn / (128 * d["cn_tile_bodies"]), 4) if fe_cn and d["cn_tile_bodies"] else None,
            "bit_node": round(fe_bn / (128 * d["bn_tile_bodies"]), 4) if fe_bn and d["bn_tile_bodies"] else None,
            "frames_moved_per_step": d["frames_moved"], "compactions_per_step": d["compactions"],
            "what": "frame-bodies the method needs / (tile-bodies the sweep processed x 128 slots), per timed step; "
                    "the rest is slots of stopped frames swept with their tile (compaction bounds it to < 1/2 "
                    "per tile)"}
    value = float(reduce_sum_(torch.tensor([Fr * len(cl) * n], dtype=torch.float64, device=dev), world).item())
    value = value * args.steps / (ms / 1e3) / 1e9

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(jobs, L, args, world, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, cfg, cl)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": "Gbit/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(args, cfg, cl, world, scaling, Fr),
            "schedule": sched,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "dist": dinfo,
            "stats": {k: int(v) for k, v in zip(P.STATS_FIELDS, tot_stats)},
            "per_point": [{"ebn0_db": cfg["ebn0"][p], "frames": int(s[0]), "fer": s[2] / max(1, s[0]),
                           "ber": s[1] / max(1, s[0] * n), "raw_ber": s[7] / max(1, s[0] * n),
                           "avg_iters": s[4] / max(1, s[0]), "near_zero_frames": int(s[6])}
                          for p, s in enumerate(per_point)],
        }
        if len(cl) > 1:  # C5: FER vs Eb/N0 of every code (the code-selection result)
            line["fer_per_code"] = {cl[q].name: [round(x, 6) for x in per_code_fer[q]] for q in range(len(cl))}
        print(json.dumps(line), flush=True)
    for j in jobs:
        j["h"].close()
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def point_rows(j, cfg):
    """Per Eb/N0 block counters of one step, from the outputs (same definitions as the decoder's stats)."""
    out, llr, pidx = j["out"], j["llr"], j["pidx"]
    rows = []
    for p in range(len(cfg["ebn0"])):
        sel = np.nonzero(pidx == p)[0]
        if len(sel) == 0:
            rows.append([0] * 8)
            continue
        lo, hi = int(sel[0]), int(sel[-1]) + 1  # blocks are contiguous
        be = out.bits[lo:hi].sum(dim=1, dtype=torch.int64)
        it = out.iters[lo:hi].to(torch.int64)
        cv = out.converged[lo:hi].to(torch.int64)
        nz = (out.posterior[lo:hi].abs() <= 1e-4).any(dim=1)
        raw = (llr[lo:hi] > 0).sum(dtype=torch.int64)
        rows.append([hi - lo, int(be.sum()), int((be > 0).sum()), int(((be > 0) & (cv > 0)).sum()),
                     int(it.sum()), int(cv.sum()), int(nz.sum()), int(raw)])
    return rows


def roofline(args, sched, prof, prof_step_ms, cn_b, bn_b, io_b, cu_edges, bu_edges, hbm, sm_mhz, peak_src,
             ms_local, steps):
    """Roofline of the dominant kernel, from the profiled step (algorithmic bytes per step of that kernel
    class / its summed CUDA-event time in that step), plus the whole-step fraction of the timed steps."""
    kms = {k: v[1] for k, v in prof.items() if v[0]}
    kl = {k: v[0] for k, v in prof.items() if v[0]}
    step_ms = ms_local / steps
    step_alg = cn_b + bn_b + io_b
    whole = {"algorithmic_bytes_per_step": round(step_alg), "ideal_ms_at_peak": round(step_alg / hbm / 1e6, 3),
             "ms_per_step": round(step_ms, 3), "frac": round(step_alg / (step_ms / 1e3) / 1e9 / hbm, 4),
             "what": "SURVEY 8(d): (sum over frames of iters x B_comp + B_io) / peak, against the timed step"}
    if sched == "resident":
        t = kms.get("resident", 0.0)
        if t <= 0:
            return None
        nl = kl["resident"]
        issue_peak = 148 * 4 * 32 * sm_mhz * 1e6 / 1e12  # T lane-instructions per s
        ops = cu_edges * OPS_CN + bu_edges * OPS_BN
        ach = ops / (t / 1e3) / 1e12
        alu = (cu_edges * ALU_CN + bu_edges * ALU_BN) / (t / 1e3) / 1e12
        traffic, tratio, tsrc = ncu_traffic(args.config, "resident")
        model = step_alg / (t / 1e3) / 1e9
        return {"bound": "alu", "kernel": "resident", "achieved": round(ach, 3), "peak": round(issue_peak, 2),
                "unit": "T lane-ops/s", "frac": round(ach / issue_peak, 4), "traffic": traffic,
                "traffic_source": tsrc,
                "what": ("SMEM-resident schedule: issue/ALU bound.  achieved = the method's minimum lane operations "
                         f"({OPS_CN} per frame-edge per check-node pass, {OPS_BN} per bit-node pass) / kernel time; "
                         "peak = 4 warp-instructions/clk/SM x 32 lanes x 148 SMs x sm_max_mhz"),
                "alu_pipe": {"achieved": round(alu, 3), "peak": round(issue_peak / 2, 2),
                             "frac": round(alu / (issue_peak / 2), 4),
                             "ops_per_frame_edge": {"check_node": ALU_CN, "bit_node": ALU_BN}},
                "dram": {"bytes_per_launch": round(io_b / nl), "achieved_gbs": round(io_b / (t / 1e3) / 1e9, 1),
                         "frac_of_peak": round(io_b / (t / 1e3) / 1e9 / hbm, 4),
                         "what": "the I/O (B_io per frame) is all the DRAM traffic; the state stays on chip"},
                "hbm_model": {"achieved_gbs": round(model, 1), "peak": hbm, "frac": round(model / hbm, 4),
                              "what": ("MODEL fraction: the B_comp bytes an HBM-streaming implementation of the same "
                                       "method would move, per second of this kernel; they never leave the SM")},
                "peak_source": peak_src, "avg_launch_us": round(t / nl * 1e3, 2), "kernel_launches": kl,
                "kernel_ms_profiled_step": {k: round(v, 3) for k, v in kms.items()},
                "share_of_step": round(t / prof_step_ms, 4), "whole_step": whole}
    bytes_of = {"check_node": cn_b, "bit_node": bn_b}
    alu_of = {"check_node": cu_edges * ALU_CN, "bit_node": bu_edges * ALU_BN}
    alu_peak = 148 * 4 * 16 * sm_mhz * 1e6 / 1e12  # T lane-ops/s on the half-rate ALU pipe
    sweeps = {}
    for k, b in bytes_of.items():
        if kms.get(k, 0) > 0:
            ach = b / (kms[k] / 1e3) / 1e9
            alu = alu_of[k] / (kms[k] / 1e3) / 1e12
            traffic, tratio, tsrc = ncu_traffic(args.config, k)
            sweeps[k] = {"achieved": round(ach, 1), "frac": round(ach / hbm, 4),
                         "algorithmic_bytes_per_launch": round(b / kl[k]), "avg_launch_us": round(kms[k] / kl[k] * 1e3, 2),
                         "launches": kl[k], "share_of_step": round(kms[k] / prof_step_ms, 4),
                         "traffic": traffic, "traffic_vs_algorithmic_in_capture": tratio,
                         # the same sweep against the ALU pipe: the method's minimum ALU operations per
                         # frame-edge (ALU_CN / ALU_BN) per second of the sweep; rows of high degree (C6) make the
                         # check node's bytes per edge small, so there the ALU pipe is the nearer roof
                         "alu_pipe": {"achieved": round(alu, 3), "peak": round(alu_peak, 2), "unit": "T lane-ops/s",
                                      "frac": round(alu / alu_peak, 4), "ops_per_frame_edge": ALU_CN if k == "check_node" else ALU_BN}}
    if not sweeps:
        return None
    dom = max(sweeps, key=lambda k: kms[k])
    d = sweeps[dom]
    traffic, tratio, tsrc = ncu_traffic(args.config, dom)
    return {"bound": "hbm", "kernel": dom, "achieved": d["achieved"], "peak": hbm, "unit": "GB/s", "frac": d["frac"],
            "traffic": traffic, "traffic_vs_algorithmic_in_capture": tratio, "traffic_source": tsrc,
            "algorithmic_bytes_per_launch": d["algorithmic_bytes_per_launch"], "avg_launch_us": d["avg_launch_us"],
            "share_of_step": d["share_of_step"], "peak_source": peak_src, "sweeps": sweeps,
            "kernel_ms_profiled_step": {k: round(v, 3) for k, v in kms.items()}, "kernel_launches": kl,
            "profiled_step_ms": round(prof_step_ms, 3), "whole_step": whole,
            "what": ("achieved = algorithmic bytes of the kernel class in one step (SURVEY 8(d) B_comp split by "
                     "sweep, per frame and body that frame ran) / its summed CUDA-event time in a separate "
                     "profiled step (plain launches); the timed steps run the CUDA-graph loop")}


def run_e2e(jobs, L, args, world, dev):
    """The same workload through the host-buffer C-ABI call (ldpc_decode_host): every step copies the
    LLRs host->device from pinned memory and the decisions (bits, k, isCodeword) back, inside the timed
    region.  The soft output is not returned here, which keeps the pinned footprint per rank at
    LLRs + bits when eight ranks share one host."""
    import paper_2507_10424_b200 as P

    hosts = []
    for j in jobs:
        F, n = j["llr"].shape
        hosts.append((j["h"], j["llr"].cpu().pin_memory(),
                      P.DecodeResult(torch.empty((F, n), dtype=torch.uint8).pin_memory(),
                                     torch.empty(F, dtype=torch.int32).pin_memory(),
                                     torch.empty(F, dtype=torch.uint8).pin_memory(), None),
                      torch.zeros(8, dtype=torch.int64)))

    def step():
        for h, hl, o, st in hosts:  # one call per code over the whole batch
            h.decode_host(hl, L, posterior=False, stats=st, out=o)

    step()  # warm (pipeline buffers, graphs)
    # the host link alone: one pinned H2D copy of the step's LLRs (what e2e cannot beat when the decode is faster)
    j0 = jobs[0]
    scratch = torch.empty_like(j0["llr"])
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    scratch.copy_(hosts[0][1], non_blocking=True)
    c1.record()
    torch.cuda.synchronize()
    h2d_gbs = hosts[0][1].numel() * 4 / (c0.elapsed_time(c1) / 1e3) / 1e9
    del scratch
    barrier(world)
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    t1 = time.perf_counter()
    secs = reduce_max(t1 - t0, world, dev)
    F = sum(hl.shape[0] for _, hl, _, _ in hosts)
    n = hosts[0][1].shape[1]
    bits = float(world) * F * n * steps
    return {"value": round(bits / secs / 1e9, 4), "unit": "Gbit/s", "steps": steps,
            "h2d_bytes_per_step": int(F * n * 4), "d2h_bytes_per_step": int(F * n + F * 4 + F),
            "host_link_h2d_gbs": round(h2d_gbs, 1),
            "copy_bound_gbps": round(float(world) * F * n / (F * n * 4 / (h2d_gbs * 1e9)) / 1e9, 3),
            "api": "ldpc_decode_host over the step's batch (pinned host buffers; chunked H2D / decode / D2H "
                   "overlap; returns b, k, isCodeword and the counters)"}


# ------------------------------------------------------------------ CPU oracle ---------------
def oracle_sample(cfg, cl, per_point, offset=0):
    """A bounded, deterministic sample of the workload: per Eb/N0 block, `per_point` frames evenly spaced
    over the block (C5: the codes taken round robin).  Returns [(code index, llr [k, n])]."""
    F = cfg["frames"]
    pts = codes.point_ranges(F, len(cfg["ebn0"]))
    groups = {}
    for p, (lo, hi) in enumerate(pts):
        k = min(per_point, hi - lo)
        idx = lo + (np.arange(k) * ((hi - lo) // k) + offset) % (hi - lo)
        for q, w in enumerate(idx):
            h = (q + p) % len(cl)
            groups.setdefault(h, []).append(channel.bpsk_awgn(cl[h].n, cl[h].rate, cfg["ebn0"][p], seed_of(cfg, h), p,
                                                              int(w), 1).numpy())
    return [(h, np.concatenate(v)) for h, v in sorted(groups.items())]


def time_oracle(cfg, cl, sample, threads):
    import oracle

    t0 = time.perf_counter()
    nb = 0
    for h, llr in sample:
        oracle.decode(cl[h].oracle_h(), llr, cfg["max_iter"], threads=threads, check_every=cfg.get("check_every", 1))
        nb += llr.shape[0] * cl[h].n
    secs = time.perf_counter() - t0
    return nb / secs / 1e9, secs, sum(x.shape[0] for _, x in sample)


def cpu_baseline(args, cfg, cl, budget_s: float = 15.0):
    """The oracle as it stands on the host cores (all threads, plus one thread on a smaller sample)."""
    import oracle

    oracle.build()
    threads = oracle.max_threads()
    npts = len(cfg["ebn0"])
    g, _, nf = time_oracle(cfg, cl, oracle_sample(cfg, cl, max(1, threads // npts + 1), offset=7), threads)
    per_frame = cl[0].n / (g * 1e9)
    per_point = int(max(1, min(5000, budget_s / max(per_frame, 1e-7) / npts)))
    gbps, secs, nf = time_oracle(cfg, cl, oracle_sample(cfg, cl, per_point), threads)
    pp1 = max(1, int(per_point * 5.0 / budget_s / max(1, threads)))
    g1, s1, nf1 = time_oracle(cfg, cl, oracle_sample(cfg, cl, pp1, offset=3), 1)
    return {"value": round(gbps, 6), "unit": "Gbit/s", "cores": threads, "kind": "oracle",
            "sample": f"{nf} frames ({per_point} per Eb/N0 block, evenly spaced over the {cfg['frames']}-frame batch"
                      + (", codes round robin" if len(cl) > 1 else "") + f"); {secs:.1f} s on {threads} threads",
            "single_thread": {"value": round(g1, 6), "unit": "Gbit/s", "cores": 1,
                              "sample": f"{nf1} frames ({pp1} per block); {s1:.1f} s on 1 thread"}}


def run_reference(args):
    """--impl reference: the CPU oracle (the only reference this tier has) on the same workload, each step a
    bounded sample of it (the same evenly spaced frames each step, shifted by the step index)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    oracle.build()
    threads = oracle.max_threads()
    cfg = codes.CONFIGS[args.config]
    cl = code_list(cfg)
    npts = len(cfg["ebn0"])
    per_point = int(os.environ.get("REF_FRAMES_PER_POINT", "0")) or int(
        max(1, min(1024, 64e6 / (cl[0].n * npts))))  # about 64 Mbit of frames per step
    for w in range(args.warmup):
        time_oracle(cfg, cl, oracle_sample(cfg, cl, max(1, per_point // 8), offset=1000 + w), threads)
    tot_b, tot_t = 0.0, 0.0
    nf = 0
    for s in range(args.steps):
        g, secs, k = time_oracle(cfg, cl, oracle_sample(cfg, cl, per_point, offset=s), threads)
        tot_b += g * 1e9 * secs
        tot_t += secs
        nf = k
    value = tot_b / tot_t / 1e9
    world = int(os.environ.get("WORLD_SIZE", "1"))
    scaling = scaling_of(args)
    w0, Fr, _ = rank_shard(cfg, 0, world, scaling)
    desc = (f"{nf} frames per step ({per_point} per Eb/N0 block, evenly spaced over the {cfg['frames']}-frame batch"
            + (", codes round robin" if len(cl) > 1 else "") + f"); {threads} host threads")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "Gbit/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot_t / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(args, cfg, cl, world, scaling, Fr),
            "cpu_baseline": {"value": round(value, 6), "unit": "Gbit/s", "cores": threads, "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": round(value, 6), "unit": "Gbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(codes.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--strong", action="store_true", help="split the config's frames over the ranks")
    ap.add_argument("--weak", action="store_true", help="every rank decodes a full batch (default except C4)")
    ap.add_argument("--code-streams", type=int, default=1,
                    help="side streams the per-code decodes alternate over (configs with several codes; C5: 2 and 4 streams measured +0.2 / +0.6 %%, within noise)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher / sharding check: print each rank's frame range and LLR checksum, no decode")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours" and not args.dry_run:
        print("warning: the timing rules require --warmup >= 3", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
        return
    relaunch_if_needed(args, argv)
    run_ours(args)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark: decoded Gbps of batched Min-Sum LDPC decoding on B200 (BASELINE.json "metric").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU, NCCL)

A step is one pass of the whole hot path (ingested H; stage-in, check-node / bit-node sweeps with
fused syndrome and per-frame early stop, stage-out and counters) over this rank's batch: config C2 =
2^20 frames of a random (3,6)-regular 504x1008 code split into 7 contiguous Eb/N0 blocks
1.0..4.0 dB, max_iter 50, decoded by one ldpc_decode call (--per-block: one per Eb/N0 block).  Frames are keyed by global frame
index, so rank r of N decodes its own 2^20 frames (weak scaling); the only collectives are the
barrier, the MAX of the elapsed time and the SUM of the 8 counters.

value = (frames decoded by all ranks) * n / (max-over-ranks device time), in Gbit/s.
"""
from __future__ import annotations

import argparse
import json
import os
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


def hbm_peak():
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def describe(cfg_name, cfg, code):
    te = cfg.get("check_every", 1)
    return (f"{cfg_name}: {code.name} ({code.m}x{code.n}, nnz {code.nnz}), {cfg['frames']} frames per GPU over "
            f"Eb/N0 {cfg['ebn0']} dB, max_iter {cfg['max_iter']}"
            + (f", codeword test every {te} bodies" if te != 1 else "") + ", BPSK/AWGN all-zero codeword")


# ------------------------------------------------------------------ distributed plumbing -------
def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    return rank, world, local


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
              "clocks_event_reasons.sw_power_cap"]
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
        sm, mx, reasons = [], [], set()
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
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ workload -----------------
def build_workload(cfg_name, rank, dev):
    cfg = codes.CONFIGS[cfg_name]
    code = cfg["code"]()
    if isinstance(code, list):
        code = code[0]
    F = cfg["frames"]
    pts = codes.point_ranges(F, len(cfg["ebn0"]))
    llr = torch.empty((F, code.n), dtype=torch.float32, device=dev)
    for p, (lo, hi) in enumerate(pts):
        # global frame index of this rank's frames: rank * F + local (weak scaling)
        channel.bpsk_awgn(code.n, code.rate, cfg["ebn0"][p], cfg["seed"], p, rank * F + lo, hi - lo, device=dev,
                          out=llr[lo:hi])
    return cfg, code, llr, pts


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


# ------------------------------------------------------------------ our arm ------------------
def run_ours(args):
    import paper_2507_10424_b200 as P

    rank, world, local = dist_setup(args.gpus)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg, code, llr, pts = build_workload(args.config, rank, dev)
    F, n, L = cfg["frames"], code.n, cfg["max_iter"]
    rr, cc = code.coo()
    h = P.Handle.from_coo(torch.from_numpy(rr).to(dev), torch.from_numpy(cc).to(dev), code.m, code.n,
                          flags=args.flags)
    T = cfg.get("check_every", 1)
    if T != 1:
        h.set_check_every(T)
    out = P.DecodeResult(torch.empty((F, n), dtype=torch.uint8, device=dev),
                         torch.empty(F, dtype=torch.int32, device=dev),
                         torch.empty(F, dtype=torch.uint8, device=dev),
                         torch.empty((F, n), dtype=torch.float32, device=dev))
    stats = torch.zeros((len(pts), 8), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        if args.per_block:  # one decode per Eb/N0 block
            for p, (lo, hi) in enumerate(pts):
                sub = P.DecodeResult(out.bits[lo:hi], out.iters[lo:hi], out.converged[lo:hi], out.posterior[lo:hi])
                h.decode(llr[lo:hi], L, posterior=True, stats=stats[p], out=sub, stream=stream)
        else:  # one decode over the batch (the blocks are just frames: outputs do not depend on the batch, A19)
            h.decode(llr, L, posterior=True, stats=stats[0], out=out, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stats.zero_()
    h.profile(True)
    h.profile_reset()
    launches0 = h.launch_count
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
    launches = h.launch_count - launches0
    ms_local = e0.elapsed_time(e1)
    prof = h.profile_read()
    h.profile(False)
    ms = reduce_max(ms_local, world, dev)
    tot_stats = reduce_sum_(stats.sum(dim=0).clone(), world).cpu().numpy()
    if args.per_block:
        per_point = stats.cpu().numpy()
    else:  # per-block counters of one step, from the outputs (same definitions as the decoder's stats)
        rows = []
        for lo, hi in pts:
            be = out.bits[lo:hi].sum(dim=1, dtype=torch.int64)
            it = out.iters[lo:hi].to(torch.int64)
            cv = out.converged[lo:hi].to(torch.int64)
            nz = (out.posterior[lo:hi].abs() <= 1e-4).any(dim=1)
            raw = (llr[lo:hi] > 0).sum(dtype=torch.int64)
            rows.append([hi - lo, int(be.sum()), int((be > 0).sum()), int(((be > 0) & (cv > 0)).sum()),
                         int(it.sum()), int(cv.sum()), int(nz.sum()), int(raw)])
        per_point = np.array(rows, dtype=np.int64)

    # ---- roofline of the dominant kernel (per-launch algorithmic bytes / per-launch device time)
    iters_np = out.iters.cpu().numpy()
    early = not (args.flags & P.FLAG_NO_EARLY_STOP)
    cn_b, bn_b, io_b = algorithmic_bytes(code, iters_np, L, early)
    cu, bu = units(iters_np, L, early)
    peak, peak_src = hbm_peak()
    if h.schedule == "resident":
        kern = {"resident": cn_b + bn_b + io_b}
    else:
        kern = {"check_node": cn_b, "bit_node": bn_b}
    dom = max(kern, key=lambda c: prof[c][1])
    n_launch, kms = prof[dom]
    roof = None
    if n_launch and kms > 0:
        per_launch_bytes = kern[dom] * args.steps / n_launch
        per_launch_s = kms / 1e3 / n_launch
        achieved = per_launch_bytes / per_launch_s / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic_from_profiles(args.config, dom),
                "traffic_vs_algorithmic_in_capture": traffic_ratio_from_profiles(args.config, dom),
                "algorithmic_bytes_per_launch": round(per_launch_bytes), "avg_launch_us": round(per_launch_s * 1e6, 2),
                "share_of_step": round(kms / ms_local, 4), "peak_source": peak_src,
                "kernel_ms": {k: round(v[1], 3) for k, v in prof.items() if v[0]},
                "kernel_launches": {k: v[0] for k, v in prof.items() if v[0]}}
        if dom == "resident":
            roof["note"] = ("state is SMEM-resident: the algorithmic bytes (B_comp per frame-body, SURVEY 8(d)) "
                            "stay on chip, DRAM carries only I/O (see traffic)")
            sm_mhz = 1965.0
            try:
                with open(PEAKS_PATH) as f:
                    sm_mhz = float(json.load(f).get("sm_max_mhz", sm_mhz))
            except Exception:
                pass
            issue_peak = 148 * 4 * 32 * sm_mhz * 1e6 / 1e12  # lane-instructions per s, T
            ops = (float(cu.sum()) * OPS_CN + float(bu.sum()) * OPS_BN) * code.nnz * args.steps
            ach = ops / (kms / 1e3) / 1e12
            alu_peak = issue_peak / 2  # 16 lanes per cycle per sub-partition
            alu = (float(cu.sum()) * ALU_CN + float(bu.sum()) * ALU_BN) * code.nnz * args.steps / (kms / 1e3) / 1e12
            roof["issue_roofline"] = {"bound": "alu", "achieved": round(ach, 3), "peak": round(issue_peak, 2),
                                      "unit": "T lane-ops/s", "frac": round(ach / issue_peak, 4),
                                      "ops_per_frame_edge": {"check_node": OPS_CN, "bit_node": OPS_BN},
                                      "alu_pipe": {"achieved": round(alu, 3), "peak": round(alu_peak, 2),
                                                   "frac": round(alu / alu_peak, 4),
                                                   "ops_per_frame_edge": {"check_node": ALU_CN, "bit_node": ALU_BN}}}
    total_bits = float(world) * F * n * args.steps
    value = total_bits / (ms / 1e3) / 1e9

    # ---- end to end through the host-buffer C-ABI call (copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(h, llr, pts, L, args, world, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, code, args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": "Gbit/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": describe(args.config, cfg, code), "global_batch": world * F,
                       "frames_per_gpu": F, "m": code.m, "n": code.n, "nnz": code.nnz, "max_iter": L,
                       "ebn0_db": cfg["ebn0"], "check_every": T, "schedule": h.schedule, "flags": args.flags,
                       "parallelism": f"dp{world} (frame shards, no data-path collective)",
                       "l2": f"inputs {F * n * 4 / 1e9:.2f} GB per GPU > 126 MB L2 (no flush needed)"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "stats": {k: int(v) for k, v in zip(P.STATS_FIELDS, tot_stats)},
            "per_point": [{"ebn0_db": cfg["ebn0"][p], "frames": int(s[0]), "fer": s[2] / max(1, s[0]),
                           "ber": s[1] / max(1, s[0] * n), "raw_ber": s[7] / max(1, s[0] * n),
                           "avg_iters": s[4] / max(1, s[0]), "near_zero_frames": int(s[6])}
                          for p, s in enumerate(per_point)],
        }
        print(json.dumps(line), flush=True)
    h.close()
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def traffic_ratio_from_profiles(cfg_name, kernel):
    """DRAM bytes / algorithmic bytes of the captured launch (a full-work launch), if recorded."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            e = json.load(f)[cfg_name][kernel]
        return round(e["dram_bytes_per_launch"] / e["algorithmic_bytes_this_launch"], 3)
    except Exception:
        return None


def traffic_from_profiles(cfg_name, kernel):
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of the kernel from the
    committed ncu --set full summary, if one exists for this config."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d[cfg_name][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


def run_e2e(h, llr_dev, pts, L, args, world, dev):
    """The same workload through the host-buffer C-ABI call (ldpc_decode_host): every step copies the
    LLRs host->device from pinned memory and the decisions (bits, k, isCodeword) back, inside the timed
    region.  The soft output is not returned here, which keeps the pinned footprint per rank at
    LLRs + bits (5.3 GB for C2) when eight ranks share one host."""
    F, n = llr_dev.shape
    host_llr = llr_dev.cpu().pin_memory()
    import paper_2507_10424_b200 as P

    outs = P.DecodeResult(torch.empty((F, n), dtype=torch.uint8).pin_memory(),
                          torch.empty(F, dtype=torch.int32).pin_memory(),
                          torch.empty(F, dtype=torch.uint8).pin_memory(), None)
    st = torch.zeros(8, dtype=torch.int64)

    def step():
        # one call over the whole batch: the Eb/N0 blocks are just frames (each frame's outputs do not
        # depend on its batch, A19), and the chunked copy / decode pipeline drains once per step
        h.decode_host(host_llr, L, posterior=False, stats=st, out=outs)

    step()  # warm (pipeline buffers, graphs)
    barrier(world)
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    t1 = time.perf_counter()
    secs = reduce_max(t1 - t0, world, dev)
    bits = float(world) * F * n * steps
    return {"value": round(bits / secs / 1e9, 4), "unit": "Gbit/s", "steps": steps,
            "h2d_bytes_per_step": int(F * n * 4), "d2h_bytes_per_step": int(F * n + F * 4 + F),
            "api": "ldpc_decode_host over the step's batch (pinned host buffers; chunked H2D / decode / D2H "
                   "overlap; returns b, k, isCodeword and the counters)"}


# ------------------------------------------------------------------ CPU oracle ---------------
def cpu_baseline(cfg, code, args, budget_s: float = 15.0):
    import oracle

    oracle.build()
    threads = oracle.max_threads()
    F = cfg["frames"]
    pts = codes.point_ranges(F, len(cfg["ebn0"]))

    def sample(per_point):
        parts = []
        for p, (lo, hi) in enumerate(pts):
            idx = np.linspace(lo, hi - 1, per_point).astype(np.int64)
            for i in idx:
                parts.append(channel.bpsk_awgn(code.n, code.rate, cfg["ebn0"][p], cfg["seed"], p, int(i), 1).numpy())
        return np.concatenate(parts)

    # calibrate on a small sample, then size the timed sample for ~budget_s of CPU work
    cal = sample(max(1, threads // len(pts) + 1))
    t0 = time.perf_counter()
    oracle.decode(code.oracle_h(), cal, cfg["max_iter"], threads=threads, check_every=cfg.get("check_every", 1))
    t_cal = time.perf_counter() - t0
    per_frame = t_cal / len(cal)
    per_point = int(max(1, min(5000, budget_s / max(per_frame, 1e-6) / len(pts))))
    llr = sample(per_point)
    t0 = time.perf_counter()
    oracle.decode(code.oracle_h(), llr, cfg["max_iter"], threads=threads, check_every=cfg.get("check_every", 1))
    secs = time.perf_counter() - t0
    gbps = len(llr) * code.n / secs / 1e9
    return {"value": round(gbps, 6), "unit": "Gbit/s", "cores": threads, "kind": "oracle",
            "sample": f"{per_point} frames per Eb/N0 block x {len(pts)} blocks = {len(llr)} frames, evenly "
                      f"spaced over the {F}-frame batch; {secs:.1f} s on {threads} threads"}


def run_reference(args):
    """--impl reference: the CPU oracle (the only reference this tier has) on the same workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = codes.CONFIGS[args.config]
    code = cfg["code"]()
    if isinstance(code, list):
        code = code[0]
    import oracle

    oracle.build()
    threads = oracle.max_threads()
    F = cfg["frames"]
    pts = codes.point_ranges(F, len(cfg["ebn0"]))
    per_point = max(1, int(os.environ.get("REF_FRAMES_PER_POINT", "1024")))

    def sample(step_idx):
        parts = []
        for p, (lo, hi) in enumerate(pts):
            idx = lo + (np.arange(per_point) * ((hi - lo) // per_point) + step_idx) % (hi - lo)
            for i in idx:
                parts.append(channel.bpsk_awgn(code.n, code.rate, cfg["ebn0"][p], cfg["seed"], p, int(i), 1).numpy())
        return np.concatenate(parts)

    for w in range(args.warmup):
        oracle.decode(code.oracle_h(), sample(1000 + w), cfg["max_iter"], threads=threads,
                      check_every=cfg.get("check_every", 1))
    tot_t, tot_frames = 0.0, 0
    for s in range(args.steps):
        llr = sample(s)
        t0 = time.perf_counter()
        oracle.decode(code.oracle_h(), llr, cfg["max_iter"], threads=threads, check_every=cfg.get("check_every", 1))
        tot_t += time.perf_counter() - t0
        tot_frames += len(llr)
    value = tot_frames * code.n / tot_t / 1e9
    desc = (f"{per_point} frames per Eb/N0 block x {len(pts)} blocks per step (every "
            f"{F // len(pts) // per_point}-th frame of each block of the {F}-frame batch)")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "Gbit/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot_t / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": describe(args.config, cfg, code), "global_batch": F, "max_iter": cfg["max_iter"],
                       "ebn0_db": cfg["ebn0"], "parallelism": "host threads over frames"},
            "cpu_baseline": {"value": round(value, 6), "unit": "Gbit/s", "cores": threads, "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": round(value, 6), "unit": "Gbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(codes.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--per-block", action="store_true", help="one decode call per Eb/N0 block (default: one per step)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: the timing rules require --warmup >= 3", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

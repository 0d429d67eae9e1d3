"""Command line front end (SPEC-style subcommands), GPU decoder only.

    python -m paper_2507_10424_b200.cli decode  --matrix H.alist --llr frame.txt [--max-iters 50] [--check-every 1]
    python -m paper_2507_10424_b200.cli sweep   (--matrix H.alist | --config c2) --snr 1,2,3 --frames N
                                                [--max-iters L] [--check-every T] [--seed S] [--out sweep.csv]
                                                [--timings]      (stage-timing table on stderr)
    python -m paper_2507_10424_b200.cli scaling --config c4 --gpus 1,2,4,8 [--steps 3] [--warmup 3] [--weak]
                                                [--out scaling.csv]
    python -m paper_2507_10424_b200.cli gen-qc  --row-blocks 2 --col-blocks 16 --z 511 --weight 2 --seed S --out H.alist
    python -m paper_2507_10424_b200.cli convert --in H.alist --out H2.alist

Exit codes: 0 success, 1 usage error, 2 data / format error.  The sweep CSV header is S:395's,
one row per SNR point; throughput = frames x n / wall seconds.  `scaling` is SPEC's scalingStudy
 on GPUs: the same frame set (strong split by default) decoded by bench.py on each GPU count,
one CSV row per count, and the outcome counters must be identical across rows (else exit 2).  Every
decode runs in libldpc on CUDA devices; there is no CPU decoder behind this CLI.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

CSV_HEADER = "snr_db,frames,raw_ber,decoded_ber,fer,avg_iterations,wall_seconds,throughput_bps"


def _root():
    return os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load_code(args):
    sys.path.insert(0, _root())
    from gen import codes

    if getattr(args, "matrix", None):
        with open(args.matrix) as f:
            return codes.parse_alist(f.read(), os.path.basename(args.matrix)), None
    if getattr(args, "config", None):
        cfg = codes.CONFIGS[args.config]
        c = cfg["code"]()
        return (c[0] if isinstance(c, list) else c), cfg
    raise SystemExit(1)


def _handle(code, T, flags=0):
    import torch

    import paper_2507_10424_b200 as P

    rr, cc = code.coo()
    h = P.Handle.from_coo(torch.from_numpy(rr).cuda(), torch.from_numpy(cc).cuda(), code.m, code.n, flags=flags)
    if T != 1:
        h.set_check_every(T)
    return h


def cmd_decode(args) -> int:
    import numpy as np
    import torch

    code, _ = _load_code(args)
    vals = np.loadtxt(args.llr, dtype=np.float64, ndmin=1).astype(np.float32)
    if vals.size % code.n:
        print(f"error: {vals.size} LLR values is not a multiple of n = {code.n}", file=sys.stderr)
        return 2
    llr = torch.from_numpy(vals.reshape(-1, code.n)).cuda()
    out = _handle(code, args.check_every).decode(llr, args.max_iters, posterior=True)
    torch.cuda.synchronize()
    for f in range(llr.shape[0]):
        print(f"isCodeword={int(out.converged[f])} k={int(out.iters[f])} b=" +
              "".join(map(str, out.bits[f].cpu().tolist())))
    return 0


def cmd_sweep(args) -> int:
    import torch

    from gen import channel, codes

    code, cfg = _load_code(args)
    snrs = [float(x) for x in args.snr.split(",")] if args.snr else (cfg["ebn0"] if cfg else [])
    if not snrs:
        print("error: --snr is required", file=sys.stderr)
        return 1
    L = args.max_iters or (cfg["max_iter"] if cfg else 50)
    T = args.check_every or (cfg.get("check_every", 1) if cfg else 1)
    seed = args.seed if args.seed is not None else (cfg["seed"] if cfg else 1)
    h = _handle(code, T)
    lines = [CSV_HEADER]
    stage_ms = {k: 0.0 for k in STAGES}
    for p, snr in enumerate(snrs):
        llr = channel.bpsk_awgn(code.n, code.rate, snr, seed, p, 0, args.frames, device="cuda")
        st = torch.zeros(8, dtype=torch.int64, device="cuda")
        h.decode(llr[: min(len(llr), 128)], L)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h.decode(llr, L, bits=True, stats=st)
        torch.cuda.synchronize()
        secs = time.perf_counter() - t0
        if args.timings:  # one more decode of the point with per-kernel events (plain launches)
            h.profile(True)
            h.profile_reset()
            h.decode(llr, L, bits=True)
            for k, (_, ms) in h.profile_read().items():
                if k in stage_ms:
                    stage_ms[k] += ms
            h.profile(False)
        s = st.cpu().tolist()
        nb = args.frames * code.n
        lines.append(f"{snr:.6g},{args.frames},{s[7] / nb:.6e},{s[1] / nb:.6e},{s[2] / args.frames:.6e},"
                     f"{s[4] / args.frames:.6g},{secs:.6g},{nb / secs:.6e}")
    text = "\n".join(lines) + "\n"
    if args.out:
        with open(args.out, "w", newline="\n") as f:
            f.write(text)
    else:
        sys.stdout.write(text)
    if args.timings:  # stage-timing table (two columns): device milliseconds per kernel class
        for k in STAGES:
            if stage_ms[k] > 0:
                print(f"{k} {stage_ms[k]:.3f}", file=sys.stderr)
    return 0


STAGES = ("stage_in", "check_node", "bit_node", "compact", "syndrome", "finalize", "resident")


def cmd_scaling(args) -> int:
    """scalingStudy: one row per GPU count (bench.py launched with that many ranks)."""
    import json
    import subprocess

    import torch

    counts = [int(x) for x in args.gpus.split(",") if x.strip()]
    if not counts or min(counts) < 1:
        print("error: --gpus must list positive GPU counts", file=sys.stderr)
        return 1
    avail = torch.cuda.device_count()
    rows, ref = ["gpus,wall_seconds,throughput_bps,frames,sum_iterations,frame_errors,bit_errors"], None
    for n in counts:
        if n > avail:
            print(f"skip: {n} GPUs requested, {avail} visible", file=sys.stderr)
            continue
        cmd = [sys.executable, os.path.join(_root(), "bench.py"), "--gpus", str(n), "--config", args.config,
               "--steps", str(args.steps), "--warmup", str(args.warmup), "--no-e2e", "--no-cpu-baseline",
               "--weak" if args.weak else "--strong"]
        r = subprocess.run(cmd, capture_output=True, text=True, cwd=_root())
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        if r.returncode != 0 or not lines:
            sys.stderr.write(r.stderr[-2000:])
            return 2
        d = json.loads(lines[-1])
        st = d["stats"]
        if not args.weak:  # the same frames at every count: identical outcomes
            key = (st["frames"], st["sum_iters"], st["frame_errors"], st["bit_errors"], st["converged"])
            if ref is None:
                ref = key
            elif key != ref:
                print(f"error: outcomes at {n} GPUs differ from the first row: {key} != {ref}", file=sys.stderr)
                return 2
        secs = d["ms_per_step"] / 1e3
        k = max(1, d["steps"])
        rows.append(f"{n},{secs:.6g},{d['value'] * 1e9:.6e},{st['frames'] // k},{st['sum_iters'] // k},"
                    f"{st['frame_errors'] // k},{st['bit_errors'] // k}")
    text = "\n".join(rows) + "\n"
    if args.out:
        with open(args.out, "w", newline="\n") as f:
            f.write(text)
    else:
        sys.stdout.write(text)
    return 0


def cmd_gen_qc(args) -> int:
    sys.path.insert(0, _root())
    from gen import codes

    c = codes.qc_random(args.row_blocks, args.col_blocks, args.z, args.weight, args.seed)
    with open(args.out, "w", newline="\n") as f:
        f.write(codes.to_alist(c))
    return 0


def cmd_convert(args) -> int:
    sys.path.insert(0, _root())
    from gen import codes

    with open(args.inp) as f:
        c = codes.parse_alist(f.read())
    with open(args.out, "w", newline="\n") as f:
        f.write(codes.to_alist(c))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="ldpc")
    sub = ap.add_subparsers(dest="cmd")
    d = sub.add_parser("decode")
    d.add_argument("--matrix", required=True)
    d.add_argument("--llr", required=True)
    d.add_argument("--max-iters", type=int, default=50)
    d.add_argument("--check-every", type=int, default=1)
    s = sub.add_parser("sweep")
    s.add_argument("--matrix")
    s.add_argument("--config")
    s.add_argument("--snr")
    s.add_argument("--frames", type=int, default=4096)
    s.add_argument("--max-iters", type=int, default=0)
    s.add_argument("--check-every", type=int, default=0)
    s.add_argument("--seed", type=int)
    s.add_argument("--out")
    s.add_argument("--timings", action="store_true")
    sc = sub.add_parser("scaling")
    sc.add_argument("--config", default="c4")
    sc.add_argument("--gpus", default="1,2,4,8")
    sc.add_argument("--steps", type=int, default=3)
    sc.add_argument("--warmup", type=int, default=3)
    sc.add_argument("--weak", action="store_true")
    sc.add_argument("--out")
    g = sub.add_parser("gen-qc")
    g.add_argument("--row-blocks", type=int, default=2)
    g.add_argument("--col-blocks", type=int, default=16)
    g.add_argument("--z", type=int, default=511)
    g.add_argument("--weight", type=int, default=2)
    g.add_argument("--seed", type=int, default=8176)
    g.add_argument("--out", required=True)
    c = sub.add_parser("convert")
    c.add_argument("--in", dest="inp", required=True)
    c.add_argument("--out", required=True)
    try:
        args = ap.parse_args(argv)
    except SystemExit:
        return 1
    if args.cmd is None:
        ap.print_usage(sys.stderr)
        return 1
    try:
        return {"decode": cmd_decode, "sweep": cmd_sweep, "scaling": cmd_scaling, "gen-qc": cmd_gen_qc,
                "convert": cmd_convert}[args.cmd](args)
    except (ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())

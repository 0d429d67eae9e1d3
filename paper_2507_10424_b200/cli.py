"""Command line front end (SPEC-style subcommands), GPU decoder only.

    python -m paper_2507_10424_b200.cli decode  --matrix H.alist --llr frame.txt [--max-iters 50] [--check-every 1]
    python -m paper_2507_10424_b200.cli sweep   (--matrix H.alist | --config c2) --snr 1,2,3 --frames N
                                                [--max-iters L] [--check-every T] [--seed S] [--out sweep.csv]
    python -m paper_2507_10424_b200.cli gen-qc  --row-blocks 2 --col-blocks 16 --z 511 --weight 2 --seed S --out H.alist
    python -m paper_2507_10424_b200.cli convert --in H.alist --out H2.alist

Exit codes: 0 success, 1 usage error, 2 data / format error.  The sweep CSV header is S:395's,
one row per SNR point; throughput = frames x n / wall seconds.  Every decode runs in libldpc
on the current CUDA device; there is no CPU decoder behind this CLI.
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
    for p, snr in enumerate(snrs):
        llr = channel.bpsk_awgn(code.n, code.rate, snr, seed, p, 0, args.frames, device="cuda")
        st = torch.zeros(8, dtype=torch.int64, device="cuda")
        h.decode(llr[: min(len(llr), 128)], L)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h.decode(llr, L, bits=True, stats=st)
        torch.cuda.synchronize()
        secs = time.perf_counter() - t0
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
        return {"decode": cmd_decode, "sweep": cmd_sweep, "gen-qc": cmd_gen_qc, "convert": cmd_convert}[args.cmd](args)
    except (ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())

"""Profiling driver: decode one Eb/N0 block of a config `reps` times (for ncu -k / launch lists)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_10424_b200 as P  # noqa: E402
from gen import channel, codes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--point", type=int, default=0)
ap.add_argument("--frames", type=int, default=0, help="0 = the config's block size")
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--max-iter", type=int, default=0)
ap.add_argument("--chunk", type=int, default=0, help="frames per chunk (0 = automatic)")
args = ap.parse_args()
cfg = codes.CONFIGS[args.config]
code = cfg["code"]()
if isinstance(code, list):
    code = code[0]
lo, hi = codes.point_ranges(cfg["frames"], len(cfg["ebn0"]))[args.point]
F = args.frames or (hi - lo)
llr = channel.bpsk_awgn(code.n, code.rate, cfg["ebn0"][args.point], cfg["seed"], args.point, lo, F, device="cuda")
rr, cc = code.coo()
h = P.Handle.from_coo(torch.from_numpy(rr).cuda(), torch.from_numpy(cc).cuda(), code.m, code.n, flags=args.flags)
print("schedule", h.schedule, "frames", F)
if args.chunk:
    h.set_chunk(args.chunk)
st = torch.zeros(8, dtype=torch.int64, device="cuda")
h.profile(True)
for _ in range(args.reps):
    out = h.decode(llr, args.max_iter or cfg["max_iter"], posterior=True, stats=st)
torch.cuda.synchronize()
print(h.profile_read())
print(P.stats_dict(st))

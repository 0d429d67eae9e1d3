"""Decode a config on the GPU and report how much early-stop work a tile of T frames wastes:
waste(T) = sum over tiles of T * max(min(k+1, L)) / sum over frames of min(k+1, L)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_10424_b200 as P  # noqa: E402
from gen import channel, codes  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = codes.CONFIGS[cfg_name]
code = cfg["code"]()
if isinstance(code, list):
    code = code[0]
rr, cc = code.coo()
h = P.Handle.from_coo(torch.from_numpy(rr).cuda(), torch.from_numpy(cc).cuda(), code.m, code.n)
L = cfg["max_iter"]
tot = {32: [0, 0], 64: [0, 0], 128: [0, 0]}
for p, (lo, hi) in enumerate(codes.point_ranges(cfg["frames"], len(cfg["ebn0"]))):
    llr = channel.bpsk_awgn(code.n, code.rate, cfg["ebn0"][p], cfg["seed"], p, lo, hi - lo, device="cuda")
    it = h.decode(llr, L).iters.cpu().numpy().astype(np.int64)
    cu = np.minimum(it + 1, L)
    line = [f"{cfg_name} p={p} ebn0={cfg['ebn0'][p]} avg_k={it.mean():.2f}"]
    for T in (32, 64, 128):
        pad = (-len(cu)) % T
        x = np.concatenate([cu, np.zeros(pad, np.int64)]).reshape(-1, T)
        w = (x.max(axis=1) * T).sum() / cu.sum()
        tot[T][0] += (x.max(axis=1) * T).sum()
        tot[T][1] += cu.sum()
        line.append(f"waste{T}={w:.2f}")
    print(" ".join(line))
print("overall", {T: round(a / b, 3) for T, (a, b) in tot.items()})

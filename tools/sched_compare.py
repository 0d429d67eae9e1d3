"""Time one config's Eb/N0 blocks with each schedule (CUDA graphs on, no per-kernel profiling)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_10424_b200 as P  # noqa: E402
from gen import channel, codes  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c5"
cfg = codes.CONFIGS[cfg_name]
code = cfg["code"]()
code = code[0] if isinstance(code, list) else code
pts = codes.point_ranges(cfg["frames"], len(cfg["ebn0"]))
rr, cc = code.coo()
for flags, name in ((0, "default"), (P.FLAG_FORCE_STREAM, "stream")):
    h = P.Handle.from_coo(torch.from_numpy(rr).cuda(), torch.from_numpy(cc).cuda(), code.m, code.n, flags=flags)
    tot = 0.0
    row = []
    for p, (lo, hi) in enumerate(pts):
        llr = channel.bpsk_awgn(code.n, code.rate, cfg["ebn0"][p], cfg["seed"], p, lo, hi - lo, device="cuda")
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            h.decode(llr, cfg["max_iter"], posterior=True)
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        tot += ms
        row.append(f"{cfg['ebn0'][p]}dB {ms:.2f}")
    print(f"{cfg_name} {name:8s} ({h.schedule}): total {tot:.2f} ms = {cfg['frames'] * code.n / tot / 1e6:.2f} Gbps | " + ", ".join(row))

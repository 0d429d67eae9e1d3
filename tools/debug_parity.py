"""Debug helper: decode a config subset on the GPU and report where it departs from the oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2507_10424_b200 as P  # noqa: E402
from gen import channel, codes  # noqa: E402


def run(code, llr, L, flags):
    h = P.Handle(torch.from_numpy(code.dense()).cuda(), flags=flags)
    out = h.decode(torch.from_numpy(llr).cuda(), L, posterior=True)
    torch.cuda.synchronize()
    return [t.cpu().numpy() for t in (out.bits, out.iters, out.converged, out.posterior)]


cfg = codes.CONFIGS["c2"]
code = cfg["code"]()
parts = [channel.bpsk_awgn(code.n, code.rate, e, cfg["seed"], p, 5000, 1700).numpy() for p, e in enumerate(cfg["ebn0"])]
llr = np.concatenate(parts)
L = cfg["max_iter"]
ob, oi, oc, op = oracle.decode(code.oracle_h(), llr, L)
for flags in (4, 6, 8, 10, 9):
    gb, gi, gc, gp = run(code, llr, L, flags)
    if flags & 3:
        ob2, oi2, oc2, op2 = oracle.decode(code.oracle_h(), llr, L, flags=flags & 3)
    else:
        ob2, oi2, oc2, op2 = ob, oi, oc, op
    bad = np.nonzero((gi != oi2) | (gc != oc2) | np.any(gb != ob2, axis=1))[0]
    print(f"flags={flags} frames={len(llr)} mismatching={len(bad)}")
    for f in bad[:12]:
        print(f"  f={f} tile={f // 128} fl={f % 128} gpu(it={gi[f]},c={gc[f]},bits_ok={np.array_equal(gb[f], ob2[f])},"
              f"post_ok={np.array_equal(gp[f], op2[f])}) oracle(it={oi2[f]},c={oc2[f]})")
    if len(bad):
        tiles = np.unique(bad // 128)
        print("  tiles with mismatches:", tiles[:40], "fl:", np.unique(bad % 128)[:40])

"""Small decodes of both schedules for compute-sanitizer (memcheck / racecheck / synccheck / initcheck)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_10424_b200 as P  # noqa: E402
from gen import channel, codes  # noqa: E402

for code, F, L in ((codes.paper_5x10(), 300, 10), (codes.regular(60, 120, 3, 6, 5), 260, 20),
                   (codes.random_small(37, 70, 1, 2, 9), 200, 8)):
    llr = channel.bpsk_awgn(code.n, code.rate, 1.5, 3, 0, 0, F, device="cuda")
    for flags, compact in ((P.FLAG_FORCE_STREAM, 0), (P.FLAG_FORCE_RESIDENT, 0), (P.FLAG_FORCE_RESIDENT, 1),
                           (P.FLAG_FORCE_STREAM | P.FLAG_NO_EARLY_STOP, 0)):
        if compact:  # the compact bit-node records of the resident kernel
            os.environ["LDPC_RES_COMPACT"] = "1"
        else:
            os.environ.pop("LDPC_RES_COMPACT", None)
        h = P.Handle(torch.from_numpy(code.dense()).cuda(), flags=flags)
        if h.schedule == "unavailable":
            continue
        st = torch.zeros(8, dtype=torch.int64, device="cuda")
        out = h.decode(llr, L, posterior=True, stats=st)
        torch.cuda.synchronize()
        print(code.name, flags, h.schedule, int(out.iters.sum()), st.tolist())
        h.close()

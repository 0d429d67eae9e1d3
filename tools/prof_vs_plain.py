"""Time one config's whole batch decode with per-kernel profiling on and off, alternating (CUDA events
around the call on the launching stream).  Diagnoses the gap between bench's timed steps and its profiled
step."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2507_10424_b200 as P  # noqa: E402
from gen import codes  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = codes.CONFIGS[cfg_name]
code = bench.code_list(cfg)[0]
llr, _ = bench.gen_frames(code, cfg, cfg["seed"], 0, cfg["frames"], 0, device="cuda")
rr, cc = code.coo()
h = P.Handle.from_coo(torch.from_numpy(rr).cuda(), torch.from_numpy(cc).cuda(), code.m, code.n)
if cfg.get("check_every", 1) != 1:
    h.set_check_every(cfg["check_every"])
L = cfg["max_iter"]
F = llr.shape[0]
out = P.DecodeResult(torch.empty((F, code.n), dtype=torch.uint8, device="cuda"),
                     torch.empty(F, dtype=torch.int32, device="cuda"),
                     torch.empty(F, dtype=torch.uint8, device="cuda"),
                     torch.empty((F, code.n), dtype=torch.float32, device="cuda"))
s = torch.cuda.current_stream()
for _ in range(3):
    h.decode(llr, L, posterior=True, out=out)
torch.cuda.synchronize()
for rep in range(4):
    for prof in (False, True):
        h.profile(prof)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        h.decode(llr, L, posterior=True, out=out)
        e1.record(s)
        torch.cuda.synchronize()
        print(f"rep {rep} profile={int(prof)} {e0.elapsed_time(e1):.2f} ms", flush=True)
        if prof:
            h.profile_read()
            h.profile_reset()

cd $GRAFT_REPO_ROOT
python - <<'PY'
import torch, sys
sys.path.insert(0,".")
import paper_2507_10424_b200 as P
from gen import channel, codes
for cfgn in ("c3","c4"):
    cfg=codes.CONFIGS[cfgn]; code=cfg["code"]()
    rr,cc=code.coo()
    h=P.Handle.from_coo(torch.from_numpy(rr).cuda(), torch.from_numpy(cc).cuda(), code.m, code.n, flags=16)
    lo,hi=codes.point_ranges(cfg["frames"],len(cfg["ebn0"]))[0]
    llr=channel.bpsk_awgn(code.n, code.rate, cfg["ebn0"][0], cfg["seed"], 0, lo, hi-lo, device="cuda")
    for chunk in (0, 128, 256, 512):
        h.set_chunk(chunk)
        h.decode(llr, cfg["max_iter"]); torch.cuda.synchronize()
        h.profile(True); h.profile_reset()
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); h.decode(llr, cfg["max_iter"]); e1.record(); torch.cuda.synchronize()
        pr=h.profile_read(); h.profile(False)
        cn=pr["check_node"]; bn=pr["bit_node"]
        print(cfgn, "frames", hi-lo, "chunk", chunk, "total ms %.2f" % e0.elapsed_time(e1), "cn us/launch %.1f" % (cn[1]*1e3/cn[0]), "bn us/launch %.1f" % (bn[1]*1e3/bn[0]), "launches", cn[0])
PY

"""fp64 drift report ("An fp64 shadow mode reports drift and is not used for parity").

The oracle is compiled twice (oracle.c with REAL=float and REAL=double).  On a stratified sample of
every benchmark configuration (per Eb/N0 block, evenly spaced frames of the bench's batch) this test
decodes with both and reports how far the fp32 arithmetic the method runs in (reading A14) drifts from
fp64: max |s32 - s64| (absolute and relative), hard-decision flips, iteration-count and isCodeword
differences.  The report is written to profiles/drift_report.json when LDPC_WRITE_DRIFT=1 (the committed
copy was produced that way), else to gpurun_out/.
"""
import json
import os

import numpy as np

import bench
import oracle
from gen import codes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# frames per Eb/N0 block (kept small enough for the CPU suite)
PER_BLOCK = {"c1": 400, "c2": 40, "c3": 3, "c4": 2, "c5": 8, "c6": 3}


def drift(cfg_name):
    cfg = codes.CONFIGS[cfg_name]
    cl = bench.code_list(cfg)
    sample = bench.oracle_sample(cfg, cl, PER_BLOCK[cfg_name], offset=11)
    agg = dict(frames=0, bits=0, k_diff_frames=0, conv_diff_frames=0, k32_sum=0, k64_sum=0,
               converged_frames=0, converged_bit_flips=0, converged_max_abs_ds=0.0,
               unconverged_frames=0, unconverged_frames_with_flips=0, unconverged_bit_flips=0,
               unconverged_max_abs_ds=0.0)
    for h, llr in sample:
        code = cl[h]
        b32, k32, c32, s32 = oracle.decode(code.oracle_h(), llr, cfg["max_iter"], check_every=cfg.get("check_every", 1))
        b64, k64, c64, s64 = oracle.decode(code.oracle_h(), llr, cfg["max_iter"], precision="f64",
                                           check_every=cfg.get("check_every", 1))
        same = k32 == k64
        agg["frames"] += len(llr)
        agg["bits"] += llr.size
        agg["k_diff_frames"] += int((~same).sum())
        agg["conv_diff_frames"] += int((c32 != c64).sum())
        agg["k32_sum"] += int(k32.sum())
        agg["k64_sum"] += int(k64.sum())
        for tag, sel in (("converged", same & (c32 == 1) & (c64 == 1)), ("unconverged", same & (c32 == 0) & (c64 == 0))):
            if not sel.any():
                continue
            ds = np.abs(s32[sel].astype(np.float64) - s64[sel])
            flips = b32[sel] != b64[sel]
            agg[f"{tag}_frames"] += int(sel.sum())
            agg[f"{tag}_bit_flips"] += int(flips.sum())
            if tag == "unconverged":
                agg["unconverged_frames_with_flips"] += int(flips.any(axis=1).sum())
            agg[f"{tag}_max_abs_ds"] = max(agg[f"{tag}_max_abs_ds"], float(ds.max()))
    agg["config"] = cfg_name
    agg["max_iter"] = cfg["max_iter"]
    agg["sample"] = f"{PER_BLOCK[cfg_name]} frames per Eb/N0 block, evenly spaced over the {cfg['frames']}-frame batch"
    return agg


def test_fp64_drift_report():
    rep = [drift(c) for c in ("c1", "c2", "c3", "c4", "c5", "c6")]
    for r in rep:
        assert r["frames"] > 0
        # drift is a measurement, not a parity gate; but frames that converge to a codeword in both
        # precisions after the same number of bodies decide the same codeword (a flip would need a
        # posterior within rounding of 0 at a satisfied parity)
        assert r["converged_bit_flips"] == 0
    path = (os.path.join(ROOT, "profiles", "drift_report.json") if os.environ.get("LDPC_WRITE_DRIFT") == "1"
            else os.path.join(ROOT, "gpurun_out", "drift_report.json"))
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as f:
        json.dump({"what": "oracle fp32 (the kernels' arithmetic, A14) vs the fp64 shadow build, same inputs",
                   "configs": rep}, f, indent=1)

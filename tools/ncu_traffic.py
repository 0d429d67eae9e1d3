"""profiles/ncu_traffic.json from ncu --set full captures of full-work launches (every frame running):
per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) and L2->SM bytes of each captured
sweep, next to that launch's algorithmic bytes (SURVEY 8(d) B_comp split by sweep).

usage: python tools/ncu_traffic.py out.json cfg:report.ncu-rep:frames:body [...]
(body = the loop body of the captured check-node launch; body 1 reads no old state)"""
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import codes  # noqa: E402


def launches(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for r in rows[2:]:
        yield dict(zip(h, r))


def num(x):
    return float(str(x).replace(",", ""))


res = {}
if os.path.exists(sys.argv[1]):
    with open(sys.argv[1]) as f:
        res = json.load(f)
for spec in sys.argv[2:]:
    cfg_name, rep, frames, body = spec.split(":")
    F, k = int(frames), int(body)
    c = codes.CONFIGS[cfg_name]["code"]()
    c = c[0] if isinstance(c, list) else c
    n, m, E = c.n, c.m, c.nnz
    state = 9 * m + E / 8
    alg = {"check_node": F * (4 * n + (2 if k > 1 else 1) * state), "bit_node": F * (8 * n + state)}
    ent = {}
    for d in launches(rep):
        name = d.get("Kernel Name", "")
        kind = "check_node" if "k_cn" in name else "bit_node" if "k_bn" in name else None
        if kind is None or kind in ent:
            continue
        dram = num(d["dram__bytes_read.sum"]) + num(d["dram__bytes_write.sum"])
        t = num(d["gpu__time_duration.sum"]) * 1e-9
        l2sm = num(d.get("lts__t_sectors_srcunit_tex.sum", "0")) * 32
        ent[kind] = {"dram_bytes_per_launch": int(dram), "algorithmic_bytes_this_launch": int(alg[kind]),
                     "dram_over_algorithmic": round(dram / alg[kind], 3),
                     "l2_to_sm_bytes_per_launch": int(l2sm), "duration_us": round(t * 1e6, 2),
                     "dram_gbs": round(dram / t / 1e9, 1), "l2_to_sm_gbs": round(l2sm / t / 1e9, 1),
                     "kernel": name[:90],
                     "source": f"ncu --set full of a full-work launch (body {k}, {F} frames, every frame running): "
                               f"{os.path.basename(rep)}"}
    res[cfg_name] = ent
with open(sys.argv[1], "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res, indent=1))

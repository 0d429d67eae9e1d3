"""Hot SASS instructions of one kernel in an ncu report (--set full --import-source on): the
instructions with the most warp-stall samples, their dominant stall reasons and execution counts."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kern:
    args += ["-k", f"regex:{kern}"]
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
hdr = rows[hdr_i]
ix = {k: i for i, k in enumerate(hdr)}
stall_cols = [k for k in hdr if k.startswith("stall_")]


def num(r, k):
    try:
        return float((r[ix[k]] or "0").replace(",", ""))
    except (ValueError, IndexError, KeyError):
        return 0.0


recs = []
tot_s = tot_i = 0.0
for pos, r in enumerate(rows[hdr_i + 1:]):
    if len(r) < len(hdr) or not r[ix["Address"]].startswith("0x"):
        break
    s, c = num(r, "Warp Stall Sampling (All Samples)"), num(r, "Instructions Executed")
    tot_s += s
    tot_i += c
    why = sorted(((num(r, k), k[6:]) for k in stall_cols), reverse=True)[:2]
    recs.append((s, c, pos, r[ix["Source"]].strip()[:70], why))
print(f"samples {tot_s:.0f}, warp instructions {tot_i:.0f}")
for s, c, pos, src, why in sorted(recs, reverse=True)[:top]:
    w = ", ".join(f"{n} {v / max(1, s) * 100:.0f}%" for v, n in why if v > 0)
    print(f"{s / max(1, tot_s) * 100:5.1f}%  #{pos:4d}  x{c:10.0f}  {src:70s} {w}")

"""Seeded parity-matrix ensembles -- INPUT GENERATION ONLY.

Shared by the tests, bench.py and (via the same seeds) the oracle: this module
holds none of the decoder's arithmetic.  A code is returned as a list of rows,
each an ascending list of 0-based column indices (the paper's index sets I_i,
P:48-52, shifted to 0-based), plus helpers to turn it into a dense 0/1 matrix or
a COO list of ones.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Code:
    m: int
    n: int
    rows: list  # rows[i] = ascending np.int32 array of the columns of the ones of row i
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(sum(len(r) for r in self.rows))

    def coo(self):
        """(rows, cols) int32 arrays of the ones, row-major."""
        rr = np.repeat(np.arange(self.m, dtype=np.int32), [len(r) for r in self.rows])
        cc = np.concatenate([np.asarray(r, np.int32) for r in self.rows]) if self.m else np.zeros(0, np.int32)
        return rr, cc

    def dense(self) -> np.ndarray:
        H = np.zeros((self.m, self.n), np.uint8)
        rr, cc = self.coo()
        H[rr, cc] = 1
        return H

    def oracle_h(self):
        rr, cc = self.coo()
        return (rr, cc, self.m, self.n)

    @property
    def rate(self) -> float:
        """Design rate R = 1 - m/n (reading A17)."""
        return 1.0 - self.m / self.n


# Paper's Tanner-graph example, checks I1..I5, 1-based bit indices.
# The index sets are ground truth (reading A8: the printed indicator of I3 is a typo).
PAPER_SETS = [
    [1, 2, 3, 6, 7, 10],
    [1, 3, 5, 6, 8, 9],
    [3, 4, 5, 7, 9, 10],
    [2, 4, 5, 6, 8, 10],
    [1, 2, 4, 7, 8, 9],
]


def paper_5x10() -> Code:
    return Code(5, 10, [np.array(sorted(j - 1 for j in s), np.int32) for s in PAPER_SETS], "paper5x10")


def from_rows(rows, n, name="") -> Code:
    return Code(len(rows), n, [np.array(sorted(set(int(c) for c in r)), np.int32) for r in rows], name)


def from_dense(H, name="") -> Code:
    H = np.asarray(H)
    return Code(H.shape[0], H.shape[1], [np.nonzero(H[i])[0].astype(np.int32) for i in range(H.shape[0])], name)


def _socket_model(col_deg: np.ndarray, row_deg: np.ndarray, rng: np.random.Generator, name: str) -> Code:
    """Configuration model: a random matching of column sockets to row sockets, then
    repair of repeated (row, column) pairs by random socket swaps between rows."""
    m, n = len(row_deg), len(col_deg)
    E = int(col_deg.sum())
    assert E == int(row_deg.sum()), "degree sequences must have equal sums"
    sockets = np.repeat(np.arange(n, dtype=np.int64), col_deg)
    sockets = sockets[rng.permutation(E)]
    starts = np.concatenate([[0], np.cumsum(row_deg)]).astype(np.int64)
    row_of = np.repeat(np.arange(m, dtype=np.int64), row_deg)

    def dup_positions():
        key = row_of * n + sockets
        order = np.argsort(key, kind="stable")
        ks = key[order]
        d = np.nonzero(ks[1:] == ks[:-1])[0]
        return order[d + 1]

    for _ in range(10000):
        bad = dup_positions()
        if len(bad) == 0:
            break
        for p in bad:
            i = row_of[p]
            for _try in range(1000):
                q = int(rng.integers(E))
                i2 = row_of[q]
                if i2 == i:
                    continue
                a, b = sockets[p], sockets[q]
                rowi = sockets[starts[i]:starts[i + 1]]
                rowi2 = sockets[starts[i2]:starts[i2 + 1]]
                if np.count_nonzero(rowi == b) == 0 and np.count_nonzero(rowi2 == a) == 0:
                    sockets[p], sockets[q] = b, a
                    break
    else:  # pragma: no cover
        raise RuntimeError("could not repair duplicate edges")
    rows = [np.sort(sockets[starts[i]:starts[i + 1]]).astype(np.int32) for i in range(m)]
    return Code(m, n, rows, name)


def regular(m: int, n: int, dv: int, dc: int, seed: int) -> Code:
    """Random (dv, dc)-regular H, m x n (configs C2, C4, C5)."""
    assert n * dv == m * dc
    rng = np.random.Generator(np.random.PCG64(seed))
    return _socket_model(np.full(n, dv, np.int64), np.full(m, dc, np.int64), rng, f"reg{dv}{dc}_{m}x{n}_s{seed}")


def irregular(col_degrees: dict, row_degrees: dict, seed: int, name: str = "") -> Code:
    """Random H with the given degree histograms {degree: count}; columns/rows are shuffled."""
    rng = np.random.Generator(np.random.PCG64(seed))
    cd = np.concatenate([np.full(c, d, np.int64) for d, c in sorted(col_degrees.items())])
    rd = np.concatenate([np.full(c, d, np.int64) for d, c in sorted(row_degrees.items())])
    cd = cd[rng.permutation(len(cd))]
    rd = rd[rng.permutation(len(rd))]
    return _socket_model(cd, rd, rng, name or f"irr_{len(rd)}x{len(cd)}_s{seed}")


def bg1_dims(seed: int = 26112) -> Code:
    """Random H with 5G-NR BG1 lifted dimensions (Z=384): 17664 x 26112, nnz 121344 = 316*384.
    Column degrees {5: 16896, 4: 9216}, row degrees {7: 15360, 6: 2304} (config C3)."""
    return irregular({5: 16896, 4: 9216}, {7: 15360, 6: 2304}, seed, f"bg1dims_s{seed}")


def spc(d: int) -> Code:
    """Single parity check over d bits: H = 1 x d all-ones."""
    return Code(1, d, [np.arange(d, dtype=np.int32)], f"spc{d}")


def random_small(m: int, n: int, seed: int, dmin: int = 2, dmax: int = 6) -> Code:
    """Small random H: each row picks a random set of dmin..dmax columns (odd and even
    degrees; columns of degree 0 allowed, reading A18)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    rows = []
    for _ in range(m):
        d = int(rng.integers(dmin, min(dmax, n) + 1))
        rows.append(np.sort(rng.choice(n, size=d, replace=False)).astype(np.int32))
    return Code(m, n, rows, f"small{m}x{n}_s{seed}")


def random_tree(m: int, seed: int, dmin: int = 2, dmax: int = 4) -> Code:
    """Cycle-free Tanner graph: every new check shares exactly one existing bit and adds
    d-1 fresh bits, so the bipartite graph stays a tree (mixed odd/even row degrees)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    rows = []
    nbits = 0
    for i in range(m):
        d = int(rng.integers(dmin, dmax + 1))
        if i == 0:
            r = list(range(d))
            nbits = d
        else:
            shared = int(rng.integers(nbits))
            r = [shared] + list(range(nbits, nbits + d - 1))
            nbits += d - 1
        rows.append(np.array(sorted(r), np.int32))
    return Code(m, nbits, rows, f"tree{m}_s{seed}")


# --- the benchmark configurations (BASELINE.json "configs"; recipe in DESIGN.md) ---------
CONFIGS = {
    "c1": dict(code=lambda: paper_5x10(), frames=10_000, max_iter=10, ebn0=[1.0, 2.0, 3.0, 4.0], seed=10),
    "c2": dict(code=lambda: regular(504, 1008, 3, 6, 1008), frames=1 << 20, max_iter=50,
               ebn0=[1.0, 1.5, 2.0, 2.5, 3.0, 3.5, 4.0], seed=1008),
    "c3": dict(code=lambda: bg1_dims(26112), frames=1 << 16, max_iter=20, ebn0=[2.0, 3.0, 3.5, 4.0, 5.0],
               seed=26112),
    "c4": dict(code=lambda: regular(32400, 64800, 3, 6, 64800), frames=1 << 14, max_iter=50,
               ebn0=[1.0, 1.5, 2.0, 2.5, 3.0, 4.0], seed=64800),
    "c5": dict(code=lambda: [regular(2048, 4096, 3, 6, 4096 + h) for h in range(16)], frames=1 << 14,
               max_iter=50, ebn0=[1.0, 1.5, 2.0, 2.5, 3.0], seed=4096),
}


def point_ranges(frames: int, npoints: int):
    """Split a batch of `frames` global frame indices into contiguous Eb/N0 blocks."""
    edges = [(p * frames) // npoints for p in range(npoints + 1)]
    return [(edges[p], edges[p + 1]) for p in range(npoints)]


def shard_range(total: int, rank: int, world: int):
    """Contiguous global-index range [lo, hi) of rank `rank` of `world` (equal split, PAR-1)."""
    return (rank * total) // world, ((rank + 1) * total) // world


# --- quasi-cyclic codes and the alist format (input plumbing) --------------------
def expand_qc(row_blocks: int, col_blocks: int, Z: int, shifts) -> Code:
    """Expand a quasi-cyclic spec: block (a, b) with shift s puts a one at (a*Z + r, b*Z + (r+s) mod Z)
    for every r in [0, Z) (SPEC S:73-81 convention); shifts[a][b] is a list of distinct offsets
    (empty = zero block, several = superimposed circulants)."""
    rows = [[] for _ in range(row_blocks * Z)]
    for a in range(row_blocks):
        for b in range(col_blocks):
            sh = list(shifts[a][b])
            if len(set(sh)) != len(sh):
                raise ValueError(f"block ({a},{b}) repeats a shift")
            for s in sh:
                if not 0 <= s < Z:
                    raise ValueError("shift out of range")
                for r in range(Z):
                    rows[a * Z + r].append(b * Z + (r + s) % Z)
    return Code(row_blocks * Z, col_blocks * Z, [np.array(sorted(r), np.int32) for r in rows],
                f"qc{row_blocks}x{col_blocks}_Z{Z}")


def qc_random(row_blocks: int = 2, col_blocks: int = 16, Z: int = 511, weight: int = 2, seed: int = 8176) -> Code:
    """Random QC code with the structure of the paper's benchmark code ("Quasi-Cyclic 8176,1022",
    CCSDS 2007): a 2 x 16 array of 511 x 511 circulants of weight 2 -> 1022 x 8176, row degree 32,
    column degree 4.  The CCSDS shift table is not in the paper, so the shifts are seeded random."""
    rng = np.random.Generator(np.random.PCG64(seed))
    shifts = [[sorted(rng.choice(Z, size=weight, replace=False).tolist()) for _ in range(col_blocks)]
              for _ in range(row_blocks)]
    c = expand_qc(row_blocks, col_blocks, Z, shifts)
    c.name = f"qc_ccsds_shape_{row_blocks * Z}x{col_blocks * Z}_s{seed}"
    c.shifts = shifts
    return c


def to_alist(code: Code) -> str:
    """Canonical alist text (MacKay format, 1-based, zero-padded lists, LF endings)."""
    cols = [[] for _ in range(code.n)]
    for i, r in enumerate(code.rows):
        for j in r:
            cols[int(j)].append(i)
    cd = [len(c) for c in cols]
    rd = [len(r) for r in code.rows]
    mc, mr = max(cd) if cd else 0, max(rd) if rd else 0
    out = [f"{code.n} {code.m}", f"{mc} {mr}", " ".join(map(str, cd)), " ".join(map(str, rd))]
    for c in cols:
        out.append(" ".join(str(i + 1) for i in c) + "".join(" 0" for _ in range(mc - len(c))) if c else
                   " ".join("0" for _ in range(mc)))
    for r in code.rows:
        out.append(" ".join(str(int(j) + 1) for j in r) + "".join(" 0" for _ in range(mr - len(r))))
    return "\n".join(out) + "\n"


def parse_alist(text: str, name: str = "") -> Code:
    """Parse alist text; the column and row sections are cross-checked against each other."""
    tok = text.split()
    pos = 0

    def nxt():
        nonlocal pos
        v = int(tok[pos])
        pos += 1
        return v

    try:
        n, m = nxt(), nxt()
        mc, mr = nxt(), nxt()
        cd = [nxt() for _ in range(n)]
        rd = [nxt() for _ in range(m)]
        cols = []
        for j in range(n):
            lst = [nxt() for _ in range(mc)]
            cols.append(sorted(x - 1 for x in lst if x > 0))
        rows = []
        for i in range(m):
            lst = [nxt() for _ in range(mr)]
            rows.append(sorted(x - 1 for x in lst if x > 0))
    except (IndexError, ValueError) as e:
        raise ValueError(f"malformed alist: {e}")
    if any(len(c) != d for c, d in zip(cols, cd)) or any(len(r) != d for r, d in zip(rows, rd)):
        raise ValueError("alist degree list inconsistent with its adjacency section")
    a = {(i, j) for i, r in enumerate(rows) for j in r}
    b = {(i, j) for j, c in enumerate(cols) for i in c}
    if a != b:
        raise ValueError("alist column and row sections disagree")
    return Code(m, n, [np.array(r, np.int32) for r in rows], name or f"alist_{m}x{n}")


CONFIGS["c6"] = dict(code=lambda: qc_random(), frames=1 << 15, max_iter=60, check_every=6,
                     ebn0=[3.0, 3.2, 3.4, 3.6], seed=8176)

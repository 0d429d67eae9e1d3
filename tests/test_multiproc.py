"""World-size-2 gloo tests of the multi-GPU host logic on CPU: frame sharding by global index, keyed
input generation per rank, and the counter / time reductions bench.py performs over NCCL."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import oracle
    from gen import channel, codes

    code = codes.regular(60, 120, 3, 6, 3)
    total = 96
    lo, hi = codes.shard_range(total, rank, world)
    llr = channel.bpsk_awgn(code.n, code.rate, 1.5, 7, 0, lo, hi - lo)
    bits, iters, conv, post = oracle.decode(code.oracle_h(), llr.numpy(), 20, threads=1)
    st = torch.from_numpy(oracle.stats(llr.numpy(), bits, iters, conv, post))
    bench.reduce_sum_(st, world)
    t = bench.reduce_max(float(rank + 1), world, torch.device("cpu"))
    gathered = [torch.zeros(total // world, dtype=torch.int32) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(iters.astype(np.int32)))
    if rank == 0:
        q.put((st.numpy().tolist(), t, torch.cat(gathered).numpy().tolist()))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_decode_counters_match_single_process():
    import oracle
    from gen import channel, codes

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    stats, tmax, iters_all = res
    code = codes.regular(60, 120, 3, 6, 3)
    llr = channel.bpsk_awgn(code.n, code.rate, 1.5, 7, 0, 0, 96).numpy()
    bits, iters, conv, post = oracle.decode(code.oracle_h(), llr, 20)
    assert stats == oracle.stats(llr, bits, iters, conv, post).tolist()
    assert tmax == 2.0
    assert iters_all == iters.tolist()


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shards_partition_the_batch(world):
    from gen import codes

    total = 1 << 20
    rs = [codes.shard_range(total, r, world) for r in range(world)]
    assert rs[0][0] == 0 and rs[-1][1] == total
    assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
    sizes = [b - a for a, b in rs]
    assert max(sizes) - min(sizes) <= 1


def _dry(args):
    import json
    import subprocess

    r = subprocess.run([sys.executable, "bench.py", "--dry-run", "--config", "c1"] + args, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return sorted((json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")), key=lambda d: d["rank"])


@pytest.mark.parametrize("mode", ["weak", "strong"])
def test_bench_launcher_brings_up_ranks(mode):
    """`bench.py --gpus 2` (no torchrun environment) re-launches itself as 2 ranks through
    torch.distributed.run (gloo here, NCCL on GPUs); every rank logs its process group, and each rank's
    frames are exactly the frames a 1-rank run generates for the same global indices."""
    import hashlib

    import bench
    from gen import codes

    extra = ["--strong"] if mode == "strong" else []
    lines = _dry(["--gpus", "2"] + extra)
    assert [d["rank"] for d in lines] == [0, 1]
    assert all(d["world"] == 2 and d["dist"]["backend"] == "gloo" and d["dist"]["all_reduce_check"] == 2
               for d in lines)
    cfg = codes.CONFIGS["c1"]
    code = codes.paper_5x10()
    F = cfg["frames"]
    if mode == "strong":
        assert [d["global_frames"] for d in lines] == [[0, F // 2], [F // 2, F]]
        one, _ = bench.gen_frames(code, cfg, cfg["seed"], 0, F, 0)
        parts = [one[:F // 2], one[F // 2:]]
    else:
        assert [d["global_frames"] for d in lines] == [[0, F], [F, 2 * F]]
        parts = [bench.gen_frames(code, cfg, cfg["seed"], 0, F, r * F)[0] for r in range(2)]
        assert lines[0]["llr_sha1"] == _dry([])[0]["llr_sha1"]  # rank 0 of 2 == the 1-rank run
    for d, p in zip(lines, parts):
        assert d["llr_sha1"] == hashlib.sha1(p.numpy().tobytes()).hexdigest()


def _strong_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import oracle
    from gen import codes

    cfg = dict(codes.CONFIGS["c1"], frames=600)
    code = codes.paper_5x10()
    w0, cnt, goff = bench.rank_shard(cfg, rank, world, "strong")
    llr, _ = bench.gen_frames(code, cfg, cfg["seed"], w0, cnt, goff)
    bits, iters, conv, post = oracle.decode(code.oracle_h(), llr.numpy(), cfg["max_iter"], threads=1)
    objs = [None] * world
    dist.all_gather_object(objs, (w0, bits, iters, conv, post))
    if rank == 0:
        q.put(objs)
    dist.barrier()
    dist.destroy_process_group()


def test_strong_shards_give_the_one_rank_outputs_per_global_frame():
    """bench.py's strong split over 3 gloo ranks: every global frame's (b, k, isCodeword, s) equals the
    1-rank result for that frame (frames are independent of their batch and shard, A19)."""
    import bench
    import oracle
    from gen import codes

    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_strong_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    objs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = dict(codes.CONFIGS["c1"], frames=600)
    code = codes.paper_5x10()
    llr, _ = bench.gen_frames(code, cfg, cfg["seed"], 0, 600, 0)
    ref = oracle.decode(code.oracle_h(), llr.numpy(), cfg["max_iter"])
    objs.sort(key=lambda o: o[0])
    for k in range(4):
        got = np.concatenate([o[1 + k] for o in objs])
        assert np.array_equal(got, ref[k])

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

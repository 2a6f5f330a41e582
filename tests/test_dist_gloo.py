"""Multi-rank host logic on CPU: column-block sharding arithmetic and the
bcur_comm allreduce callback over torch.distributed (gloo, world_size 2, 127.0.0.1),
driven through the same ctypes trampoline the C library calls."""
import ctypes
import os
import socket

import numpy as np
import pytest

from paper_1703_06065_b200 import dist as D


@pytest.mark.parametrize("G,world", [(100, 1), (512, 2), (512, 8), (256, 4), (7, 3), (2048, 8), (5, 5)])
def test_block_ranges_tile_the_partition(G, world):
    ranges = [D.block_range(G, r, world) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == G
    for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
        assert a1 == b0 and a1 > a0
    widths = [b - a for a, b in ranges]
    assert max(widths) - min(widths) <= 1


def test_block_range_rejects_bad_arguments():
    with pytest.raises(ValueError):
        D.block_range(3, 0, 4)
    with pytest.raises(ValueError):
        D.block_range(8, 2, 2)


def test_shard_columns_ragged_partition():
    off = [0, 20, 40, 45, 100, 101]  # ragged blocks
    shards = [D.shard_columns(off, r, 2) for r in range(2)]
    assert shards[0] == (0, 45, 0, 3)
    assert shards[1] == (45, 56, 3, 5)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1703_06065_b200 import bcur

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn = bcur.make_comm_callback(D.torch_allreduce("cpu"))
        # (1) in-place fp64 sum through the C trampoline
        buf = np.arange(5, dtype=np.float64) + 10.0 * rank
        rc = fn(None, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), buf.size, None)
        # (2) the library's shard-gather protocol: zero-fill, write own blocks, allreduce
        G = 10
        full = np.linspace(1.0, 2.0, G)
        g0, g1 = D.block_range(G, rank, world)
        gathered = np.zeros(G)
        gathered[g0:g1] = full[g0:g1]
        fn(None, gathered.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), G, None)
        # (3) bench timing: max over ranks
        mx = D.max_over_ranks(1.5 + rank)
        # (4) a failing collective is reported, not raised through C
        bad = bcur.make_comm_callback(lambda p, c, s: (_ for _ in ()).throw(RuntimeError("boom")))
        rc_bad = bad(None, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 1, None)
        # (5) broadcast of a selected block in its stored form (fp32 bytes, and the int32
        # exponents of the fp16 split) from the owning rank through the C trampoline
        bfn = bcur.make_broadcast_callback(D.torch_broadcast("cpu"))
        blk = (np.arange(12, dtype=np.float32) * 0.5 + 1.0) if rank == 1 else np.zeros(12, dtype=np.float32)
        rc_b = bfn(None, blk.ctypes.data, blk.nbytes, 1, None)
        ex = np.array([3, -7, 15], dtype=np.int32) if rank == 0 else np.zeros(3, dtype=np.int32)
        rc_b += bfn(None, ex.ctypes.data, ex.nbytes, 0, None)
        bcast_ok = bool(np.array_equal(blk, np.arange(12, dtype=np.float32) * 0.5 + 1.0) and
                        np.array_equal(ex, [3, -7, 15]) and rc_b == 0)
        q.put((rank, rc, buf.tolist(), bool(np.array_equal(gathered, full)), mx, rc_bad, bcast_ok))
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_allreduce_callback():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = (np.arange(5) * 2 + 10.0).tolist()
    for rank, rc, buf, gathered_ok, mx, rc_bad, bcast_ok in results:
        assert rc == 0 and buf == expect and gathered_ok and mx == 2.5 and rc_bad == 1 and bcast_ok

"""World-size-2 gloo tests of the N>1 host logic (sharding, max-over-ranks,
rank-ordered gather).  The reference's analogue is its process-pool sharding
(bench.py:303-309; test_bench.py:165-173 checks parallel == serial)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_20777_b200.shard import gather_to_rank0, max_over_ranks, shard_range


def test_shard_range_partitions():
    for world in (1, 2, 3, 8):
        for gb in (0, 1, 7, 64, 65536, 1001):
            parts = [shard_range(r, world, gb) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == gb
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(2, 2, 10)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, gb, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = shard_range(rank, world, gb)
    # stand-in for per-rank results: the global index encoded in a matrix
    local = torch.arange(a, b, dtype=torch.float64)[:, None, None].expand(b - a, 3, 3).contiguous()
    t = max_over_ranks(1.0 + rank)
    full = gather_to_rank0(local, gb)
    if rank == 0:
        out_q.put((t, full.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("gb", [10, 11])
def test_gloo_world2_gather_and_max(gb):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, gb, q)) for r in range(2)]
    for p in procs:
        p.start()
    t, full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 2.0
    assert full.shape == (gb, 3, 3)
    assert np.array_equal(full[:, 0, 0], np.arange(gb, dtype=np.float64))


def _work_worker(rank, world, port, gb, out_q):
    """Each rank regenerates ITS shard of C1 from the shared seeds (bench.py's
    strong-scaling shard, no data shipped), exponentiates it, and the results
    come home to rank 0 in rank order.  The CPU oracle stands in for the GPU
    kernel (no device here); the GPU analogue is tests/test_gpu_shards.py."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import bench
    from oracle import expm_oracle as O
    from paper_2512_20777_b200 import workloads as WL
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = WL.CONFIGS["C1"]
    idx = bench._shard_indices(cfg, rank, world, "strong", gb)
    W = WL.generate("C1", indices=idx)
    vals = np.stack([O.expm(W[i], cfg.eps).value for i in range(len(idx))]) if len(idx) else np.zeros((0, 64, 64))
    full = gather_to_rank0(torch.from_numpy(vals), gb)
    if rank == 0:
        out_q.put(full.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_work_equals_serial(world):
    """'parallel == serial, bit-identical' (reference tests/test_bench.py:165-173)."""
    from oracle import expm_oracle as O
    from paper_2512_20777_b200 import workloads as WL
    gb = 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_work_worker, args=(r, world, port, gb, q)) for r in range(world)]
    for p in procs:
        p.start()
    full = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    W = WL.generate("C1", indices=np.arange(gb))
    serial = np.stack([O.expm(W[i], WL.CONFIGS["C1"].eps).value for i in range(gb)])
    assert full.shape == serial.shape and np.array_equal(full, serial)


def test_bench_shard_indices():
    import bench
    from paper_2512_20777_b200 import workloads as WL
    for key in ("C2", "C3", "C5"):
        cfg = WL.CONFIGS[key]
        for world in (1, 2, 4, 8):
            parts = [bench._shard_indices(cfg, r, world, "strong") for r in range(world)]
            assert np.array_equal(np.concatenate(parts), np.arange(cfg.batch))
            weak = [bench._shard_indices(cfg, r, world, "weak") for r in range(world)]
            assert all(len(w) == cfg.batch for w in weak)

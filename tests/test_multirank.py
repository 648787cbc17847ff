"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: query shard
ranges, data replication by broadcast, global bbox all-reduce and result
assembly (paper_1601_05904_b200/shard.py, used by bench.py)."""
import os
import socket

import numpy as np
import pytest

from paper_1601_05904_b200 import shard

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def test_shard_range_partitions_exactly():
    for n in (0, 1, 7, 1000, 1_000_003):
        for world in (1, 2, 3, 8):
            cover = []
            for r in range(world):
                lo, hi = shard.shard_range(n, world, r)
                assert 0 <= lo <= hi <= n
                cover.extend(range(lo, hi)) if n < 5000 else cover.append((lo, hi))
            if n < 5000:
                assert cover == list(range(n))
            else:
                assert cover[0][0] == 0 and cover[-1][1] == n
                assert all(a[1] == b[0] for a, b in zip(cover, cover[1:]))
    with pytest.raises(ValueError):
        shard.shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1601_05904_b200 as A
    m, n_total = 5000, 3001
    # rank 0 owns the data; others start with garbage and receive it
    if rank == 0:
        d = A.generate_random_points(m, (0.0, 0.0, 1.0, 1.0), 42)
        data = torch.from_numpy(np.stack([d.xs, d.ys, d.zs]))
    else:
        data = torch.full((3, m), -7.0, dtype=torch.float64)
    shard.replicate(data, dist)
    ref = A.generate_random_points(m, (0.0, 0.0, 1.0, 1.0), 42)
    assert np.array_equal(data[0].numpy(), ref.xs) and np.array_equal(data[2].numpy(), ref.zs)
    # queries: rank r owns slice r of the global query set; queries past the
    # data hull make the global bbox differ from every local one
    allq = A.generate_random_queries(n_total, (-0.5, -0.25, 1.5, 1.25), 43)
    lo, hi = shard.shard_range(n_total, world, rank)
    qx, qy = allq.xs[lo:hi], allq.ys[lo:hi]
    local = (min(data[0].min().item(), qx.min()), min(data[1].min().item(), qy.min()),
             max(data[0].max().item(), qx.max()), max(data[1].max().item(), qy.max()))
    box = shard.global_bbox(local, dist)
    expect = A.compute_bbox(A.PointSet(ref.xs, ref.ys), allq)
    assert box.tolist() == expect.as_array().tolist()
    # result assembly in input order
    local_res = torch.from_numpy(np.arange(lo, hi, dtype=np.float64))
    full = shard.gather_results(local_res, n_total, dist)
    assert np.array_equal(full.numpy(), np.arange(n_total, dtype=np.float64))
    with open(os.path.join(out_dir, f"ok{rank}"), "w") as f:
        f.write("ok")
    dist.destroy_process_group()


def test_gloo_world2_replicate_bbox_gather(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    assert (tmp_path / "ok0").exists() and (tmp_path / "ok1").exists()

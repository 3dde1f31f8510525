"""Host-side multi-process logic of the slab decomposition on CPU: world size 2
over gloo (127.0.0.1).  The data path itself (NCCL inside the CUDA library)
needs >= 2 GPUs; its slab / exchange / reduction logic is exercised on one GPU
by tests/test_gpu_sharded.py (P slabs emulated on one device)."""

import os
import socket

import numpy as np
import pytest

from paper_1311_0089_b200 import parallel


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1. the communicator id made on rank 0 reaches every rank unchanged
        uid = parallel.broadcast_unique_id(lambda: bytes(range(128)))
        assert uid == bytes(range(128))
        # 2. slab results assemble on rank 0 in plane order
        shape = (3, 27, 9, 11)  # (components, n0, n1, n2)
        full = np.arange(np.prod(shape), dtype=float).reshape(shape)
        local = np.full(shape, np.nan)
        lo, hi = parallel.slab_bounds(27, world)[rank]
        local[:, lo:hi] = full[:, lo:hi]
        out = parallel.gather_slabs(local, 1, world, rank)
        if rank == 0:
            assert np.array_equal(out, full)
        # 3. max over ranks of a device time (bench.py's reduction)
        import bench

        assert bench.max_over_ranks(world, float(rank + 1)) == float(world)
        q.put((rank, "ok"))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_two_rank_host_plumbing():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


@pytest.mark.parametrize("n0,P", [(729, 8), (1215, 4), (27, 5), (9, 8)])
def test_partitions_cover_and_balance(n0, P):
    b = parallel.slab_bounds(n0, P)
    assert b[0][0] == 0 and b[-1][1] == n0
    assert all(b[t][1] == b[t + 1][0] for t in range(P - 1))
    sizes = [hi - lo for lo, hi in b]
    assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1


def test_exchange_counts_conserve_the_spectrum():
    shape, R, P = (729, 729, 729), 1, 8
    cnt = parallel.exchange_counts(shape, R, P)
    c = 3
    Q = shape[1] * ((shape[2] + 1) // 2)
    sb, qb = parallel.slab_bounds(shape[0], P), parallel.pencil_bounds(shape, P)
    for s in range(P):
        assert cnt[s].sum() == R * c * Q * (sb[s][1] - sb[s][0])      # everything slab s holds
    for p in range(P):
        assert cnt[:, p].sum() == R * c * (qb[p][1] - qb[p][0]) * shape[0]  # full pencils of slab p
    # ~1.02 GB per GPU per all-to-all at P = 8 for cfg4 (complex doubles)
    off_diag = (cnt.sum(axis=1) - np.diag(cnt)) * 16
    assert 0.9e9 < off_diag.mean() < 1.2e9

"""Host-side logic of the multi-GPU path on CPU (gloo, world_size 2): the
batch split covers every problem exactly once, and the bench's max-over-ranks
time / sum-over-ranks throughput reductions (bench.py) aggregate correctly.
There is no collective on the data path (replicas only); these
are the only cross-rank operations."""
import os
import socket
import sys

import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    share = bench.batch_share(rank, world)
    t = 1.0 + rank  # per-rank device seconds
    nnz = float(len(share) * 1000)
    tmax = bench.allreduce(dist, "cpu", t, "MAX")
    nsum = bench.allreduce(dist, "cpu", nnz, "SUM")
    out[rank] = (share, tmax, nsum)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_batch_split_and_reductions():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    shares = [res[r][0] for r in range(world)]
    assert sorted(sum(shares, [])) == list(range(64))
    assert all(res[r][1] == 2.0 for r in range(world))          # max over ranks
    assert all(res[r][2] == 64 * 1000.0 for r in range(world))  # whole-job total

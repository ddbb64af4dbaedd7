"""Multi-GPU partition + reduction logic on CPU: world_size 2 over gloo.

Each rank takes its contiguous nnz-balanced span range (blco_partition, the
product's partitioner), computes the partial M of that range, and the ranks
sum the partials with an all-reduce, or reduce-scatter them into row shards
and all-gather those (paper_2201_12523_b200.dist) -- the same plumbing
bench.py and the distributed CP-ALS run over NCCL.  No GPU here, so the
per-rank partial product comes from the oracle (test infrastructure); the GPU-side partial products are covered by
tests/test_gpu_mttkrp.py::test_slices_sum_to_whole.
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dims, nnz, rank_r, quota, out_q, combine="allreduce"):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2201_12523_b200 as b
    from pyoracle import Oracle

    o = Oracle()
    idx, vals = o.synth_uniform(dims, nnz, 42)
    keys, offs, bidx, bvals = o.build(dims, idx, vals, 12, 700)  # several blocks
    lo, hi = b.partition(np.diff(offs), quota, world)[rank]
    # coordinates of this rank's elements, decoded from the BLCO payload
    layout = o.layout(dims, 12)
    coords = np.zeros((len(dims), hi - lo), np.uint64)
    blk = np.searchsorted(offs, np.arange(lo, hi), side="right") - 1
    for e in range(lo, hi):
        coords[:, e - lo] = o.delinearize(layout, int(bidx[e]), int(keys[blk[e - lo]]))
    f = o.factors_random(dims, rank_r, 7)
    outs = []
    from paper_2201_12523_b200.dist import Collectives, row_shard
    coll = Collectives()
    for mode in range(len(dims)):
        part = torch.from_numpy(o.mttkrp_coo(dims, coords, bvals[lo:hi], f, mode))
        if combine == "allreduce":
            dist.all_reduce(part)
            outs.append(part.numpy())
            continue
        # reduce-scatter into row shards of the padded partial,
        # then all-gather them back (the distributed CP-ALS exchange)
        r0, rows, per = row_shard(dims[mode], world, rank)
        padded = torch.zeros((world * per, rank_r), dtype=torch.float64)
        padded[: dims[mode]] = part
        shard = torch.empty((per, rank_r), dtype=torch.float64)
        coll.reduce_scatter(shard, padded)
        assert r0 == rank * per and 0 <= rows <= per
        whole = torch.empty_like(padded)
        coll.all_gather(whole, shard)
        outs.append(whole[: dims[mode]].numpy())
    sizes = torch.tensor([hi - lo], dtype=torch.int64)
    dist.all_reduce(sizes)
    if rank == 0:
        want = [o.mttkrp_coo(dims, idx, vals, f, m) for m in range(len(dims))]
        err = max(float(np.sqrt(((a - w) ** 2).sum() / (w ** 2).sum())) for a, w in zip(outs, want))
        out_q.put((err, int(sizes.item())))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,combine", [(2, "allreduce"), (2, "reducescatter"), (3, "reducescatter")])
def test_partitioned_partials_combine_to_full(world, combine):
    dims, nnz, rank_r = [37, 41, 29], 6000, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, nnz, rank_r, 512, q, combine))
             for r in range(world)]
    for p in procs:
        p.start()
    err, total = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert total == nnz
    assert err <= 1e-12

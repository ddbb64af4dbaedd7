"""Repro probe: repeated stream_mttkrp_all_modes calls (Q queues) against a
device-resident MTTKRP of the same blocks, with other device work between
the calls.  Prints the per-call max relative error."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2201_12523_b200 as b

n_chunks_used = int(sys.argv[1]) if len(sys.argv) > 1 else 1
bmax = 1 << int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 25
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
Q = int(sys.argv[4]) if len(sys.argv) > 4 else 3
dims, nnz_target, nchunks = [8211298, 176962, 8116559], 4_687_474_081, 64
frac = float(np.prod(np.array(dims, dtype=np.float64))) / 2.0 ** 64
ncand = int(nnz_target / nchunks / frac) + 1
idx = b.api.pinned_empty(n_chunks_used * ncand, np.uint64)
vals = b.api.pinned_empty(n_chunks_used * ncand, np.float64)
off = 0
for c in (0, 37)[:n_chunks_used]:
    off += b.api.synth_alto_chunk(dims, c, nchunks, ncand, 42, idx[off:], vals[off:])
limit = int(sys.argv[5]) if len(sys.argv) > 5 else 0
if limit:
    off = min(off, limit)
layout = b.make_layout(dims, 64)
f = b.FactorMatrices.random(dims, 32, 7)
blocks = [(0, idx[o:o + min(bmax, off - o)], vals[o:o + min(bmax, off - o)]) for o in range(0, off, bmax)]
t = b.DeviceTensor.upload(b.BlcoTensor.from_blocks(layout, blocks, bmax))
ref = [b.mttkrp(t, f, m) for m in range(3)]
del t
for rep in range(reps):
    budget = b.DeviceBudget(capacity_bytes=12 << 30, num_queues=Q, reservation_bytes=bmax * 16)
    got = b.stream_mttkrp_all_modes(iter(blocks), f, budget, layout=layout, max_nnz_per_block=bmax,
                                    block_count=len(blocks))
    errs = [float(np.linalg.norm(g - r) / np.linalg.norm(r)) for g, r in zip(got, ref)]
    diff_rows = [int((np.abs(g - r).max(axis=1) > 1e-9 * np.abs(r).max()).sum()) for g, r in zip(got, ref)]
    print(f"rep {rep}: err {max(errs):.3e} rows differing {diff_rows} of {dims}", flush=True)
    # other device work between calls (allocations recycled)
    t = b.DeviceTensor.upload(b.BlcoTensor.from_blocks(layout, blocks[:1], bmax))
    b.mttkrp(t, f, 0)
    del t

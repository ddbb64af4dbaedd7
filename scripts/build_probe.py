"""Probe: device BLCO build time (stage split) for repeated builds in one process."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2201_12523_b200 as b

cfgs = {"nell2": ([12092, 9184, 28818], 76_879_419), "amazon": ([4821207, 1774269, 1805187], 1_741_809_018)}
for name in sys.argv[1:] or ["nell2"]:
    dims, nnz = cfgs[name]
    for rep in range(3):
        st = b.BuildStats()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dt = b.DeviceTensor.synthetic(dims, nnz, 42, stats=st)
        torch.cuda.synchronize()
        s = time.perf_counter() - t0
        print(f"{name} build {rep}: {s*1e3:.1f} ms = {nnz/s/1e9:.2f} G nnz/s; sort {st.sort_seconds*1e3:.1f} "
              f"block {st.block_seconds*1e3:.1f} reencode {st.reencode_seconds*1e3:.1f} batch {st.batch_seconds*1e3:.1f}")
        del dt

"""Probe: how wide are a 1024-element tile's coordinate ranges?  For a
tile-relative 16-byte staging record (value + every coordinate minus the
tile's minimum, packed in 64 bits) the sum of the per-mode span bits must be
<= 64.  Reports, per config, the fraction of tiles and of elements whose
tile fits, and the span-bit distribution per mode.  Usage:
tile_span_probe.py [amazon|delicious|nell2 ...]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2201_12523_b200 as b

cfgs = {"amazon": ([4821207, 1774269, 1805187], 1_741_809_018, 0),
        "delicious": ([532924, 17262471, 2480308, 1443], 140_126_181, 4),
        "nell2": ([12092, 9184, 28818], 76_879_419, 0)}
TILE = 1024
for name in sys.argv[1:] or ["delicious"]:
    dims, nnz, skew = cfgs[name]
    dt = b.DeviceTensor.synthetic_draws(dims, nnz, 42, skew) if skew else b.DeviceTensor.synthetic(dims, nnz, 42)
    h = dt.to_host()
    lay = h.layout
    N = len(dims)
    sh, mk = lay.field_shift, lay.field_mask
    offs = np.asarray(h.offsets, dtype=np.int64)
    bits = []  # per tile: span bits per mode
    counts = []
    for bi in range(len(h.keys)):
        lo, hi = int(offs[bi]), int(offs[bi + 1])
        idx = np.asarray(h.idx[lo:hi], dtype=np.uint64)
        base = lay.block_base(int(h.keys[bi]))
        n = hi - lo
        nt = (n + TILE - 1) // TILE
        pad = nt * TILE - n
        per = []
        for m in range(N):
            c = ((idx >> np.uint64(sh[m])) & np.uint64(mk[m])).astype(np.int64) + int(base[m])
            if pad:
                c = np.concatenate([c, np.repeat(c[-1], pad)])
            c = c.reshape(nt, TILE)
            span = c.max(axis=1) - c.min(axis=1)
            per.append(np.where(span > 0, np.floor(np.log2(np.maximum(span, 1))) + 1, 0).astype(np.int64))
        bits.append(np.stack(per, axis=1))
        cnt = np.full(nt, TILE)
        if pad:
            cnt[-1] = TILE - pad
        counts.append(cnt)
    bits = np.concatenate(bits)
    counts = np.concatenate(counts)
    tot = bits.sum(axis=1)
    fit = tot <= 64
    print(f"{name}: {len(tot)} tiles; sum of span bits <= 64 for {fit.mean():.4f} of tiles, "
          f"{counts[fit].sum() / counts.sum():.4f} of elements; sum percentiles 50/90/99/max "
          f"{np.percentile(tot, 50):.0f}/{np.percentile(tot, 90):.0f}/{np.percentile(tot, 99):.0f}/{tot.max()}")
    for m in range(N):
        print(f"  mode {m} ({dims[m]} rows, {int(np.ceil(np.log2(dims[m])))} bits): span bits "
              f"50/90/99/max {np.percentile(bits[:, m], 50):.0f}/{np.percentile(bits[:, m], 90):.0f}/"
              f"{np.percentile(bits[:, m], 99):.0f}/{bits[:, m].max()}", flush=True)
    del dt, h

#!/usr/bin/env python3
"""Generates tests/golden/golden.npz from the UNMODIFIED reference library.

Run here (where /root/reference exists) after `make -C oracle`:
    python tests/golden/gen_golden.py
The reference is driven through oracle/_ref/libblco_ref.so (compiled from
/root/reference/proj/src by oracle/Makefile).  Every array in the output is
what the reference computed; the tests compare both our C oracle and the
B200 library against these bytes.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle"))
from pyoracle import RefLib, cfg_array  # noqa: E402

OUT = Path(__file__).resolve().parent / "golden.npz"

# BASELINE.json shapes (exact FROSTT dims)
SHAPES = {
    "cfg1": [1000, 1000, 1000],
    "nell2": [12092, 9184, 28818],
    "amazon": [4821207, 1774269, 1805187],
    "delicious": [532924, 17262471, 2480308, 1443],
    "enron": [6066, 5699, 244268, 1176],
    "reddit": [8211298, 176962, 8116559],
}

# proj/tests/test_util.hpp:31-35 (paper Fig. 4a), 0-based
GOLDEN_I = [[0, 0, 0, 1, 1, 2, 2, 3, 3, 3, 3, 3],
            [0, 0, 2, 0, 0, 0, 3, 1, 1, 2, 2, 3],
            [0, 1, 2, 1, 2, 1, 3, 0, 1, 2, 3, 3]]
GOLDEN_V = [float(v) for v in range(1, 13)]


def random_coo(rng: np.random.Generator, dims, nnz):
    cells = int(np.prod([int(d) for d in dims], dtype=object))
    nnz = min(nnz, cells)
    if cells < 2**62:
        ids = rng.choice(cells, size=nnz, replace=False)
    else:
        ids = np.unique(rng.integers(0, 2**62, size=nnz * 2))[:nnz]
        rng.shuffle(ids)
    idx = np.zeros((len(dims), len(ids)), np.uint64)
    x = ids.astype(object)
    for m, d in enumerate(dims):
        idx[m] = np.array([int(v) % int(d) for v in x], dtype=np.uint64)
        x = np.array([int(v) // int(d) for v in x], dtype=object)
    vals = rng.uniform(-1, 1, size=len(ids))
    return idx, vals


def main() -> None:
    ref = RefLib()
    rng = np.random.default_rng(20220129)
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"layouts": [], "encodes": [], "builds": [], "mttkrps": [], "factors": [],
                  "cpals": [], "streams": []}

    # A. layouts (incl. error cases)
    cases = [([4, 4, 4], 64), ([4, 4, 4], 5), ([4, 4, 4], 6), ([1, 1, 1], 64), ([37, 1024, 53, 200], 17),
             ([64, 64, 64], 10), ([4, 4], 0), ([4, 4], 65), ([0, 4], 32), ([2, 2], 1)]
    cases += [(d, 64) for d in SHAPES.values()]
    for _ in range(60):
        order = int(rng.integers(1, 6))
        dims = [int(1 + rng.integers(0, 1 << int(rng.integers(0, 21)))) for _ in range(order)]
        cases.append((dims, int(rng.integers(1, 65))))
    for dims, tb in cases:
        try:
            l = ref.layout(dims, tb)
            meta["layouts"].append({"dims": dims, "target": tb, "ok": True, **l})
        except Exception as e:  # noqa: BLE001
            meta["layouts"].append({"dims": dims, "target": tb, "ok": False, "error": str(e)})

    # B. encode vectors (stripped <= 64 only; SURVEY §0 defect above that)
    for ent in meta["layouts"]:
        if not ent["ok"] or ent["stripped_bits"] > 64:
            continue
        dims, tb = ent["dims"], ent["target"]
        coords = np.stack([rng.integers(0, d, size=24, dtype=np.uint64) for d in dims])
        outs = np.array([ref.encode(dims, tb, coords[:, j]) for j in range(coords.shape[1])], dtype=np.uint64)
        k = len(meta["encodes"])
        arrays[f"enc{k}_coords"] = coords
        arrays[f"enc{k}_out"] = outs  # [alto_hi, alto_lo, split_key, split_reenc, enc_key, enc_reenc]
        meta["encodes"].append({"dims": dims, "target": tb})

    # C. builds
    builds = [(GOLDEN_I, GOLDEN_V, [4, 4, 4], 5, 6), (GOLDEN_I, GOLDEN_V, [4, 4, 4], 5, 4),
              (GOLDEN_I, GOLDEN_V, [4, 4, 4], 64, 1 << 27)]
    for _ in range(14):
        order = int(rng.integers(2, 6))
        dims = [int(1 + rng.integers(0, 300)) for _ in range(order)]
        idx, vals = random_coo(rng, dims, int(rng.integers(1, 500)))
        builds.append((idx, vals, dims, int(rng.integers(3, 65)), int(1 + rng.integers(0, 64))))
    # wide layouts (> 64 total bits) with multi-key blocking, Amazon/Delicious-like
    for dims, nnz, tb in (([3000000, 1500000, 1500000], 3000, 64),
                          ([500000, 9000000, 2000000, 1400], 3000, 64),
                          ([1 << 20, 1 << 20, 1 << 20, 1 << 20], 2000, 64),
                          ([24, 9, 31], 160, 7), ([50, 40, 60], 600, 8), ([30, 50, 20], 400, 9)):
        idx, vals = random_coo(rng, dims, nnz)
        builds.append((idx, vals, dims, tb, 64 if nnz <= 600 else 1000))
    for idx, vals, dims, tb, cap in builds:
        idx = np.asarray(idx, np.uint64).reshape(len(dims), -1)
        vals = np.asarray(vals, np.float64)
        t = ref.build(dims, idx, vals, tb, cap)
        keys, offs, bi, bv = t.blocks()
        k = len(meta["builds"])
        arrays.update({f"b{k}_in_idx": idx, f"b{k}_in_vals": vals, f"b{k}_keys": keys,
                       f"b{k}_offsets": offs, f"b{k}_idx": bi, f"b{k}_vals": bv,
                       f"b{k}_batch": t.batch_table()})
        meta["builds"].append({"dims": dims, "target": tb, "max_nnz": cap})
        # reference container bytes (serialize_blco) for the round-trip tests
        if k in (0, 1, 5, 17, 18, 21):
            arrays[f"b{k}_blco"] = np.frombuffer(t.serialize(), dtype=np.uint8)
        # D. mttkrp on this build: oracle::mttkrp_coo and blco::mttkrp
        #    (small modes only -- outputs are dims[mode] x rank)
        ranks = [] if max(dims) > 5000 else [2] if k < 3 else [1, 3, 8] if k % 2 else [16, 32]
        for rank in ranks:
            fs = [rng.uniform(-1, 1, size=(d, rank)) for d in dims]
            j = len(meta["mttkrps"])
            for m, a in enumerate(fs):
                arrays[f"m{j}_f{m}"] = a
            for mode in range(len(dims)):
                arrays[f"m{j}_coo{mode}"] = ref.mttkrp_coo(dims, idx, vals, fs, mode)
                out, stats = t.mttkrp(fs, mode, cfg_array(num_threads=1))
                arrays[f"m{j}_blco{mode}"] = out
            meta["mttkrps"].append({"build": k, "rank": rank})
        # streamed reference result for a couple of multi-block builds
        if len(keys) >= 4 and len(meta["streams"]) < 3:
            rank = 4
            fs = [rng.uniform(-1, 1, size=(d, rank)) for d in dims]
            j = len(meta["streams"])
            for m, a in enumerate(fs):
                arrays[f"s{j}_f{m}"] = a
            fb = sum(a.size * 8 for a in fs) + dims[0] * rank * 8
            res = cap * 16
            out, rep = t.stream_mttkrp(fs, 0, fb + 2 * res, 2, res, cfg_array(32, 4, 1, num_threads=2), 1)
            arrays[f"s{j}_out"] = out
            meta["streams"].append({"build": k, "rank": rank, "mode": 0})

    # E. FactorMatrices::random
    for dims, rank, seed in (([3, 4, 5], 4, 7), ([100, 100, 100], 16, 7), ([7], 1, 0), ([2, 3], 32, 42)):
        fs = ref.factors_random(dims, rank, seed)
        j = len(meta["factors"])
        for m, a in enumerate(fs):
            arrays[f"fr{j}_{m}"] = a
        meta["factors"].append({"dims": dims, "rank": rank, "seed": seed})

    # F. CP-ALS fit histories
    # (i) noiseless rank-4 30^3 (SPEC.md:665 probe), (ii) random 4-mode sparse
    g = np.random.default_rng(5)
    A = [g.uniform(0, 1, size=(30, 4)) for _ in range(3)]
    cube = np.einsum("ir,jr,kr->ijk", *A)
    ii = np.array(np.nonzero(cube > 0), np.uint64)
    cv = cube[cube > 0]
    for dims, idx, vals, rank, iters, tol, seed in (
            ([30, 30, 30], ii, cv, 4, 12, 1e-9, 1),
            ([40, 35, 30, 12], *random_coo(rng, [40, 35, 30, 12], 3000), 5, 10, -1e300, 7)):
        t = ref.build(dims, idx, vals, 64)
        fs, lam, fit = t.cp_als(dims, rank, iters, tol, seed)
        j = len(meta["cpals"])
        arrays[f"c{j}_in_idx"] = np.asarray(idx, np.uint64)
        arrays[f"c{j}_in_vals"] = np.asarray(vals, np.float64)
        arrays[f"c{j}_fit"] = fit
        arrays[f"c{j}_lambda"] = lam
        for m, a in enumerate(fs):
            arrays[f"c{j}_f{m}"] = a
        meta["cpals"].append({"dims": dims, "rank": rank, "iters": iters, "tol": tol, "seed": seed})

    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes): {len(meta['layouts'])} layouts, "
          f"{len(meta['encodes'])} encode sets, {len(meta['builds'])} builds, "
          f"{len(meta['mttkrps'])} mttkrp sets, {len(meta['cpals'])} cp-als runs, "
          f"{len(meta['streams'])} streams")


if __name__ == "__main__":
    main()

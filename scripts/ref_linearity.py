#!/usr/bin/env python3
"""Checks the reference arm's extrapolation model on the Amazon shape
(BASELINE configs[2]): bench.py times the unmodified reference blco::mttkrp
(1 thread, its fastest configuration) on ~1M-element samples and extrapolates
the full 1.74B-element step as a + b * nnz.  Here the same step is timed on
generator-prefix samples two orders of magnitude larger (uniformly random
subsets of the tensor's non-zeros, same dims), and the fit's prediction is
compared with each measured size.  On NELL-2 the same model, fitted the same
way, predicted 136.1 s against 134.5 s measured at full size
(profiles/r02_ref_fullsize_nell2.json).  Writes one JSON object (stdout and
argv[1])."""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT))

from pyoracle import Oracle, RefLib, cfg_array  # noqa: E402

import bench  # noqa: E402


def main():
    dims, nnz, R, desc = bench.CONFIGS["amazon"]
    out_path = sys.argv[1] if len(sys.argv) > 1 else None
    sizes = [1 << 20, 1 << 22, 1 << 24, 1 << 26]
    o, ref = Oracle(), RefLib()
    factors = o.factors_random(dims, R, bench.FACTOR_SEED)
    cfg = cfg_array(num_threads=1)
    pts = []
    for S in sizes:
        idx, vals = o.synth_uniform(dims, S, bench.TENSOR_SEED)
        t0 = time.perf_counter()
        t = ref.build(dims, idx, vals, 64)
        build_s = time.perf_counter() - t0
        s = time.perf_counter()
        for mode in range(len(dims)):
            t.mttkrp(factors, mode, cfg)
        step = time.perf_counter() - s
        pts.append((S, step, build_s))
        print(f"S={S}: all-mode step {step:.2f} s (build {build_s:.1f} s)", flush=True)
        del t, idx, vals
    S = np.array([p[0] for p in pts], dtype=float)
    y = np.array([p[1] for p in pts])
    b, a = np.polyfit(S, y, 1)
    # the bench's own two-point fit from the two smallest sizes
    b2 = (y[1] - y[0]) / (S[1] - S[0])
    a2 = y[0] - b2 * S[0]
    res = {"workload": desc, "nnz": nnz, "threads": 1, "cpu_model": bench.cpu_model(), "host_threads": os.cpu_count(),
           "kind": "reference", "path": "blco::build_blco + blco::mttkrp (all modes), oracle/_ref/libblco_ref.so",
           "samples": [{"nnz": int(p[0]), "step_s": round(p[1], 3), "build_s": round(p[2], 2)} for p in pts],
           "fit_all_points": {"fixed_s": round(a, 3), "ns_per_elem": round(b * 1e9, 1),
                              "full_step_s": round(a + b * nnz, 1)},
           "fit_two_smallest": {"fixed_s": round(a2, 3), "ns_per_elem": round(b2 * 1e9, 1),
                                "full_step_s": round(a2 + b2 * nnz, 1),
                                "error_at_largest_sample": round((a2 + b2 * S[-1]) / y[-1] - 1, 4)},
           "residuals_all_points": [round((a + b * s_) / y_ - 1, 4) for s_, y_ in zip(S, y)]}
    print(json.dumps(res), flush=True)
    if out_path:
        Path(out_path).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

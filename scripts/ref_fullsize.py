#!/usr/bin/env python3
"""The reference CPU MTTKRP at FULL size on BASELINE configs[1] (NELL-2 shape,
76,879,419 nnz, R = 32), timed on the box's host cores -- no sampling, no
extrapolation (BASELINE.md 3 / SURVEY.md 8d: configs 1 and 2 run at full
size).  Runs the unmodified reference (oracle/_ref/libblco_ref.so):

  * blco::build_blco on the full COO (timed);
  * one all-mode step of blco::mttkrp with ExecConfig{num_threads = all host
    threads} and with 1 thread (it anti-scales);
  * oracle::mttkrp_coo over all modes (1 thread, the reference's simplest loop).

Same tensor and factors as bench.py (seeded generator, tensor seed 42,
FactorMatrices::random seed 7).  Writes one JSON object (stdout and argv[1]).
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT))

from pyoracle import Oracle, RefLib, cfg_array  # noqa: E402

import bench  # noqa: E402


def main():
    dims, nnz, R, desc = bench.CONFIGS["nell2"]
    out_path = sys.argv[1] if len(sys.argv) > 1 else None
    o, ref = Oracle(), RefLib()
    res = {"workload": desc, "dims": dims, "nnz": nnz, "rank": R, "cpu_model": bench.cpu_model(),
           "host_threads": os.cpu_count(), "kind": "reference", "sample": "full tensor (no sampling)"}
    t0 = time.perf_counter()
    idx, vals = o.synth_uniform(dims, nnz, bench.TENSOR_SEED)
    factors = o.factors_random(dims, R, bench.FACTOR_SEED)
    res["generate_s"] = round(time.perf_counter() - t0, 2)
    t0 = time.perf_counter()
    t = ref.build(dims, idx, vals, 64)
    res["build_blco_s"] = round(time.perf_counter() - t0, 2)
    bpe = bench.bytes_per_elem(len(dims), R)
    for label, threads in (("blco_mttkrp_all_threads", os.cpu_count()), ("blco_mttkrp_1_thread", 1)):
        cfg = cfg_array(num_threads=threads)
        per_mode = []
        for mode in range(len(dims)):
            s = time.perf_counter()
            t.mttkrp(factors, mode, cfg)
            per_mode.append(time.perf_counter() - s)
        step = sum(per_mode)
        res[label] = {"threads": threads, "per_mode_s": [round(x, 2) for x in per_mode], "step_s": round(step, 2),
                      "gbps": round(nnz * len(dims) * bpe / step / 1e9, 4)}
        print(label, res[label], flush=True)
    per_mode = []
    for mode in range(len(dims)):
        s = time.perf_counter()
        ref.mttkrp_coo(dims, idx, vals, factors, mode)
        per_mode.append(time.perf_counter() - s)
    step = sum(per_mode)
    res["oracle_mttkrp_coo_1_thread"] = {"per_mode_s": [round(x, 2) for x in per_mode], "step_s": round(step, 2),
                                         "gbps": round(nnz * len(dims) * bpe / step / 1e9, 4)}
    best = min(("blco_mttkrp_all_threads", "blco_mttkrp_1_thread"), key=lambda k: res[k]["step_s"])
    res["best_reference_mttkrp"] = best
    print(json.dumps(res), flush=True)
    if out_path:
        Path(out_path).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

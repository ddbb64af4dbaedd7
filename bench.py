#!/usr/bin/env python3
"""BLCO MTTKRP benchmark (BASELINE.json metric) -- one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config nell2|cfg1|amazon|enron|delicious]

A step = one all-mode MTTKRP (modes 0..N-1, fixed factors) over the whole
synthetic tensor, inputs resident in HBM.  `value` = algorithmic bytes of the
step (B_elem = nnz * (8 + 8 + N*R*8) per mode) / device time,
whole job, max over ranks.  With torchrun (N > 1) the element spans are
partitioned contiguously across ranks (no data-path collective inside the
kernel) and each mode's partial M is summed with an NCCL all-reduce inside the
timed region: strong scaling on a fixed tensor.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libblco_ref.so = the unmodified proj/src compiled here) on a
bounded ALTO-contiguous sample of the same tensor, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (dims, nnz, rank, description)
    "cfg1": ([1000, 1000, 1000], 1_000_000, 16, "synthetic 1000^3, 1M nnz, R=16 (BASELINE configs[0])"),
    "nell2": ([12092, 9184, 28818], 76_879_419, 32,
              "synthetic NELL-2-shaped 12092x9184x28818, 76,879,419 nnz, R=32, all-mode (BASELINE configs[1])"),
    "amazon": ([4821207, 1774269, 1805187], 1_741_809_018, 32,
               "synthetic Amazon-shaped 4821207x1774269x1805187, 1.74B nnz, R=32 (BASELINE configs[2])"),
    "enron": ([6066, 5699, 244268, 1176], 54_202_099, 16, "synthetic uniform Enron-shaped 4-mode, R=16"),
    "delicious": ([532924, 17262471, 2480308, 1443], 140_126_181, 16,
                  "synthetic uniform Delicious-shaped 4-mode, R=16"),
}
TENSOR_SEED, FACTOR_SEED = 42, 7


def bytes_per_elem(order: int, rank: int, s: int = 8) -> int:
    return 8 + s + order * rank * s


# ------------------------------------------------------------------ clocks


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device: int, period_ms: int | None = None):
        self.device = device
        self.proc = None
        self.period_ms = period_ms or int(os.environ.get("BLCO_B200_CLOCK_MS", "100"))

    def __enter__(self):
        if self.period_ms <= 0:  # BLCO_B200_CLOCK_MS=0: no sampling (interference checks only)
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms",
                 str(self.period_ms), "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, flag in zip(self.NAMES, parts[4:8]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- distributed


def dist_env():
    """(world, rank, device).  BLCO_B200_ONE_DEVICE=1 puts every rank on
    cuda:0 (with BLCO_B200_DIST_BACKEND=gloo) so the N > 1 code paths can be
    exercised on a one-GPU box; timings from such a run mean nothing."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("BLCO_B200_ONE_DEVICE") == "1":
        local = 0
    return world, rank, local


def dist_init(torch, dev):
    import torch.distributed as dist
    backend = os.environ.get("BLCO_B200_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group(backend)


# --------------------------------------------------------- CPU reference


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_sample_run(dims, nnz, rank, steps, warmup, target_step_s=4.0, threads=None, extra=False,
                         sampler="alto_prefix", skew=None, op="mttkrp"):
    """Times the reference's blco::mttkrp (all modes) on the host.

    sampler "alto_prefix": the `S` elements of smallest ALTO index of the
    synthetic tensor -- a contiguous prefix of the BLCO element order, i.e.
    exactly the first S elements (first spans) the GPU processes.
    sampler "generator_prefix": the first S elements the seeded generator
    emits (Feistel-uniform cells, or with `skew` set the first S distinct
    draws floor(I u^skew)): the generator's key does not depend on nnz, so this
    is a uniformly random subset of the same tensor's non-zeros over the same
    dims (configs whose COO does not fit the host, or layouts > 64 bits).
    Each sample is built by the reference's own build_blco.

    The reference's step costs a + b*S: a per-call fixed cost that scales
    with the dims (zero-initialised I_n x R outputs, factor copies, merges)
    and a per-element cost.  Both are fitted at two calibration sizes for
    1 thread and for all host threads (the reference anti-scales with
    threads), and the thread count with the smaller extrapolated
    full-tensor step is used: the reference's best CPU configuration.  Then
    `steps` timed steps of a sample of S elements (the per-element part of a
    step ~ target_step_s)
    refine b, and the full-tensor step is a + b*nnz (`extrapolated` unless
    S = nnz).  op "stream" times the reference stream_mttkrp
    (MemoryBlockSource, its DeviceBudget) per mode instead.  Returns
    (GB/s of the full tensor, dict).
    """
    sys.path.insert(0, str(ROOT / "oracle"))
    from pyoracle import Oracle, RefLib, cfg_array

    oracle, ref = Oracle(), RefLib()
    all_threads = threads or os.cpu_count() or 1
    order = len(dims)
    t0 = time.perf_counter()
    factors = oracle.factors_random(dims, rank, FACTOR_SEED)
    if sampler == "alto_prefix":
        # Generate the tensor in full, then select ALTO prefixes.
        gen_n = nnz
        if int(np.prod(np.array(dims, dtype=object))) >= 2**64 or make_wide(dims):
            raise RuntimeError("reference sample: ALTO-prefix sampling needs a layout of <= 64 bits")
        idx, vals = oracle.synth_uniform(dims, gen_n, TENSOR_SEED)
        alto = oracle.alto_lo(dims, idx)

        def coo(S):
            sel = np.argpartition(alto, S - 1)[:S] if S < gen_n else np.arange(gen_n)
            return idx[:, sel], vals[sel]
    else:
        gen_n = nnz

        def coo(S):
            if skew:  # independent draws floor(I u^skew), first S distinct
                return oracle.synth_draws(dims, S, TENSOR_SEED, skew)
            return oracle.synth_uniform(dims, S, TENSOR_SEED)
    setup_s = time.perf_counter() - t0

    def sample(S):
        S = min(S, gen_n)
        sidx, svals = coo(S)
        return ref.build(dims, sidx, svals, 64), S

    def one_step(t, c):
        s = time.perf_counter()
        for mode in range(order):
            if op == "stream":
                # DeviceBudget{capacity 24 GiB, 4 queues, 2 GiB} as the GPU arm
                t.stream_mttkrp(factors, mode, 24 << 30, 4, (1 << 27) * 16, c)
            else:
                t.mttkrp(factors, mode, c)
        return time.perf_counter() - s

    # calibration: a and b at 1 thread and at all threads
    S_lo = min(gen_n, 1 << 16)
    t_lo, S_lo = sample(S_lo)
    S_mid = min(gen_n, max(4 * S_lo, 1 << 18))
    t_mid, S_mid = sample(S_mid)
    fits = {}
    for th in sorted({1, all_threads}):
        c = cfg_array(num_threads=th)
        one_step(t_lo, c)
        d_lo = one_step(t_lo, c)
        d_mid = one_step(t_mid, c)
        b = max((d_mid - d_lo) / max(S_mid - S_lo, 1), 1e-12)
        fits[th] = {"a": max(0.0, d_lo - b * S_lo), "b": b, "d_lo": d_lo}
    best = min(fits, key=lambda th: fits[th]["a"] + fits[th]["b"] * nnz)
    a, b_cal, d_lo = fits[best]["a"], fits[best]["b"], fits[best]["d_lo"]
    cfg = cfg_array(num_threads=best)
    # the per-element part of a sample step ~ target_step_s on top of the
    # fixed part, so b is fitted over seconds of element work, not over the
    # noise of the fixed cost
    S = min(gen_n, max(S_mid, int(target_step_s / b_cal)), 1 << 25)
    if S > S_mid:
        del t_mid
        t, S = sample(S)
    else:
        t, S = t_mid, S_mid
    for _ in range(warmup):
        one_step(t, cfg)
    times = [one_step(t, cfg) for _ in range(steps)]
    bpe = bytes_per_elem(order, rank)
    step_s = sum(times) / len(times)
    per_elem = (step_s - d_lo) / (S - S_lo) if S > S_lo else step_s / S
    fixed = max(0.0, d_lo - per_elem * S_lo)
    if per_elem <= 0:
        per_elem, fixed = step_s / S, 0.0
    full_s = step_s if S >= nnz else fixed + per_elem * nnz
    gbps = nnz * order * bpe / full_s / 1e9
    what = "blco::stream_mttkrp per mode (MemoryBlockSource, DeviceBudget{24 GiB, 4, 2 GiB})" if op == "stream" \
        else "blco::mttkrp"
    if sampler == "alto_prefix":
        desc = f"first {S_lo} and {S} elements in ALTO order of the {nnz}-nnz tensor"
    else:
        desc = (f"first {S_lo} and {S} elements of the seeded generator (uniformly random subsets of the "
                f"{nnz}-nnz tensor's non-zeros, same dims)")
    desc += (f"; {steps} timed steps of the {S}-element sample at {best} thread(s) "
             f"({step_s:.3f} s each); all-mode step fitted as a + b*nnz (a = {fixed:.3f} s fixed per step, "
             f"b = {per_elem * 1e9:.1f} ns per element) and extrapolated to the full {nnz} nnz = {full_s:.2f} s")
    info = {"sample_nnz": S, "sample_fraction": S / nnz, "sample_steps": steps, "step_s": step_s,
            "full_step_s": full_s, "fixed_s": fixed, "per_elem_s": per_elem, "threads": best,
            "extrapolated": S < nnz, "setup_s": setup_s,
            "threads_tried": {str(th): {"fixed_s": round(f["a"], 4), "ns_per_elem": round(f["b"] * 1e9, 1),
                                        "full_step_s_est": round(f["a"] + f["b"] * nnz, 2)}
                              for th, f in fits.items()},
            "sample": f"{desc}; reference build_blco on that COO subset, {what}, all {order} modes, R={rank}"}
    if extra:
        # oracle::mttkrp_coo (1 thread) on the same sample, the reference's
        # simplest CPU loop (oracle.cpp:9-26)
        sidx, svals = coo(S)
        s0 = time.perf_counter()
        for mode in range(order):
            ref.mttkrp_coo(dims, sidx, svals, factors, mode)
        coo_s = time.perf_counter() - s0
        info["oracle_mttkrp_coo_1_thread"] = {"value": round(S * order * bpe / coo_s / 1e9, 4), "unit": "GB/s",
                                              "step_s": round(coo_s, 3),
                                              "note": "reference oracle::mttkrp_coo (oracle.cpp:9-26) on the "
                                                      "same sample, no fixed cost to extrapolate"}
    return gbps, info


def cpu_baseline_entry(gbps, info) -> dict:
    out = {"value": round(gbps, 4), "unit": "GB/s", "cores": info["threads"], "kind": "reference",
           "sample": info["sample"], "sample_nnz": info["sample_nnz"],
           "sample_fraction": round(info["sample_fraction"], 6), "sample_steps": info["sample_steps"],
           "sample_step_s": round(info["step_s"], 3), "extrapolated": info["extrapolated"],
           "full_step_s_extrapolated": round(info["full_step_s"], 3), "threads_tried": info["threads_tried"],
           "cpu_model": cpu_model(), "host_threads": os.cpu_count()}
    for k in ("oracle_mttkrp_coo_1_thread",):
        if k in info:
            out[k] = info[k]
    return out


def make_wide(dims) -> bool:
    return sum(int(d - 1).bit_length() for d in dims) > 64


# ------------------------------------------------------- DRAM traffic (ncu)

NCU_METRICS = ("dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
               "l1tex__throughput.avg.pct_of_peak_sustained_elapsed,"
               "dram__throughput.avg.pct_of_peak_sustained_elapsed,"
               "lts__throughput.avg.pct_of_peak_sustained_elapsed")


def traffic_probe_worker(args):
    """--traffic-probe (run under ncu by live_traffic): build the config's
    tensor and launch each mode's kernel twice; nothing is timed here."""
    import torch

    import paper_2201_12523_b200 as b
    if args.config in ALS_CONFIGS:  # the CP-ALS config's MTTKRP kernels (power-law draws)
        dims, nnz, R, skew, _ = ALS_CONFIGS[args.config]
        torch.cuda.set_device(0)
        dt = b.DeviceTensor.synthetic_draws(dims, nnz, TENSOR_SEED, skew, 64, 1 << 27, 0)
    else:
        dims, nnz, R, _ = CONFIGS[args.config]
        torch.cuda.set_device(0)
        dt = b.DeviceTensor.synthetic(dims, nnz, TENSOR_SEED, device=0)
    fac = [torch.empty((d, R), dtype=torch.float64, device="cuda:0") for d in dims]
    sptr = torch.cuda.current_stream().cuda_stream
    b.factors_random_device(dims, R, FACTOR_SEED, [a.data_ptr() for a in fac], sptr)
    outs = [torch.zeros((d, R), dtype=torch.float64, device="cuda:0") for d in dims]
    cfg = b.ExecConfig(num_compute_units=torch.cuda.get_device_properties(0).multi_processor_count)
    for _ in range(2):  # the step's kernels: one per mode (the fused all-mode kernel only with BLCO_B200_FUSED=1)
        dt.mttkrp_all_device([a.data_ptr() for a in fac], R, [o.data_ptr() for o in outs], b.Strategy.Auto, cfg,
                             accumulate=True, stream=sptr)
    torch.cuda.synchronize()


def live_traffic(config: str, timeout_s: int = 300) -> dict | None:
    """DRAM bytes per launch of the mode kernels of THIS build, from an ncu
    pass over a child process (`bench.py --traffic-probe`; 2 launches per
    mode, ncu's default cache control = caches flushed before each launch).
    Only counters are taken from ncu -- never a time.  None when ncu is
    unavailable or fails (the committed profile is used instead)."""
    import csv
    import io
    import shutil
    import tempfile
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None
    with tempfile.TemporaryDirectory() as td:
        log = os.path.join(td, "traffic.csv")
        cmd = [ncu, "--metrics", NCU_METRICS, "--clock-control", "none", "-k", "regex:k_mttkrp", "--csv",
               "--log-file", log, sys.executable, str(ROOT / "bench.py"), "--traffic-probe", "--config", config]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s,
                               env=dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", "0")))
        except (OSError, subprocess.TimeoutExpired):
            return None
        if r.returncode != 0 or not os.path.exists(log):
            return None
        text = open(log).read()
    rows = [row for row in csv.reader(io.StringIO(text[text.find('"ID"'):]))]
    if len(rows) < 2:
        return None
    hdr = rows[0]
    col = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
    launches: dict[int, dict] = {}
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "nsecond": 1e-9,
             "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "%": 1.0}
    for row in rows[1:]:
        if len(row) < len(hdr):
            continue
        d = launches.setdefault(int(row[col["ID"]]), {"kernel": row[col["Kernel Name"]]})
        try:
            d[row[col["Metric Name"]]] = float(row[col["Metric Value"]].replace(",", "")) * \
                scale.get(row[col["Metric Unit"]], 1.0)
        except ValueError:
            pass
    ls = [launches[k] for k in sorted(launches)]
    if not ls:
        return None
    dram = [x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in ls]
    mean = lambda k: statistics.mean(x.get(k, 0.0) for x in ls)  # noqa: E731
    return {"dram_bytes_per_launch": statistics.mean(dram), "launches": len(ls),
            "ncu_launch_s": mean("gpu__time_duration.sum"), "kernel": ls[0]["kernel"][:100],
            "l1tex_pct": round(mean("l1tex__throughput.avg.pct_of_peak_sustained_elapsed"), 1),
            "dram_pct": round(mean("dram__throughput.avg.pct_of_peak_sustained_elapsed"), 1),
            "lts_pct": round(mean("lts__throughput.avg.pct_of_peak_sustained_elapsed"), 1),
            "source": f"live ncu pass over this build ({len(ls)} launches of the mode kernels, "
                      "dram__bytes_read.sum + dram__bytes_write.sum; caches flushed before each launch)"}


def committed_traffic(config: str) -> dict | None:
    """Fallback: the ncu --set full summary committed under profiles/."""
    prof = ROOT / "profiles" / f"ncu_{config}.json"
    try:
        rep = json.loads(prof.read_text())
    except (OSError, ValueError):
        return None
    ls = [x for x in rep.get("launches") or [] if x.get("dram_bytes") == x.get("dram_bytes")]  # drop NaN replays
    if not ls:
        return None
    mean = lambda k: statistics.mean(float(x.get(k, 0) or 0) for x in ls)  # noqa: E731
    return {"dram_bytes_per_launch": mean("dram_bytes"), "launches": len(ls),
            "ncu_launch_s": mean("gpu__time_duration.sum"), "kernel": ls[0].get("kernel", "")[:100],
            "l1tex_pct": round(mean("l1tex__throughput.avg.pct_of_peak_sustained_elapsed"), 1),
            "dram_pct": round(mean("dram__throughput.avg.pct_of_peak_sustained_elapsed"), 1),
            "lts_pct": round(mean("lts__throughput.avg.pct_of_peak_sustained_elapsed"), 1),
            "source": f"committed profile profiles/ncu_{config}.json (an earlier build)"}


def roofline_entry(traffic: dict | None, launch_ms: float, algo_bytes_per_launch: float, peak: float,
                   peak_source: str, kernel: str) -> dict:
    """roofline for the dominant kernel: achieved = PHYSICAL DRAM bytes per
    launch (ncu) / the launch's mean duration measured here (CUDA events);
    frac against the measured HBM copy peak.  The algorithmic B_elem rate
    (exceeds the HBM peak when gathers hit L2) is reported beside
    it as algorithmic_gbps, not as the fraction."""
    algo = algo_bytes_per_launch / (launch_ms * 1e-3) / 1e9
    out = {"bound": None, "achieved": None, "peak": peak, "unit": "GB/s", "frac": None, "traffic": None,
           "kernel": kernel, "launch_ms": round(launch_ms, 4),
           "algorithmic_gbps": round(algo, 2), "algorithmic_bytes_per_launch": int(algo_bytes_per_launch),
           "peak_source": peak_source}
    if traffic:
        phys = traffic["dram_bytes_per_launch"] / (launch_ms * 1e-3) / 1e9
        l1, dr = traffic.get("l1tex_pct") or 0.0, traffic.get("dram_pct") or 0.0
        # the bound: the unit nearest its ceiling inside the ncu pass -- HBM as
        # DRAM bytes / ncu duration against the MEASURED copy peak (ncu's own
        # dram % is against the theoretical peak), the L1/TEX pipe as ncu's %
        t_ncu = traffic.get("ncu_launch_s") or 0.0
        hbm_busy = traffic["dram_bytes_per_launch"] / t_ncu / 1e9 / peak if t_ncu > 0 else phys / peak
        out.update({"bound": "hbm" if hbm_busy >= l1 / 100.0 else "l1tex", "achieved": round(phys, 2),
                    "frac": round(phys / peak, 4), "traffic": int(traffic["dram_bytes_per_launch"]),
                    "limiter": {"hbm_frac_in_ncu_pass": round(hbm_busy, 3), "l1tex_pct": l1, "dram_pct": dr,
                                "lts_pct": traffic.get("lts_pct"),
                                "note": "bound = the larger of hbm_frac_in_ncu_pass and l1tex_pct/100"},
                    "traffic_source": traffic["source"]})
    return out


def hbm_peak() -> tuple[float, str]:
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        if peaks.get("hbm_gbs"):
            return float(peaks["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, ValueError):
        pass
    return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ our arm


def run_ours(args, world, rank_id, local):
    import torch

    import paper_2201_12523_b200 as b

    dims, nnz, R, desc = CONFIGS[args.config]
    if args.rank:
        R = args.rank
    N = len(dims)
    dev = local
    # DRAM bytes per launch of this build (ncu counters from a child process,
    # before this process allocates anything); N > 1 runs use the committed
    # profile so the ranks are not perturbed
    live = world == 1 and not args.no_ncu and not args.rank
    traffic = (live and live_traffic(args.config)) or committed_traffic(args.config)
    extra_traffic = None
    if world == 1 and args.config == "amazon" and not args.no_extra:
        extra_traffic = (live and live_traffic("nell2")) or committed_traffic("nell2")
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        dist_init(torch, dev)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    # --- build the BLCO tensor on the device (timed separately)
    bst = b.BuildStats()
    t0 = time.perf_counter()
    if int(np.prod(np.array(dims, dtype=object))) < 2**64:
        full = b.DeviceTensor.synthetic(dims, nnz, TENSOR_SEED, device=dev, stats=bst)
    else:  # cell space beyond 2^64: independent uniform draws (skew 1), first nnz distinct
        full = b.DeviceTensor.synthetic_draws(dims, nnz, TENSOR_SEED, 1, device=dev, stats=bst)
    build_s = time.perf_counter() - t0
    if world > 1:
        ranges = b.partition(full.block_nnz(), 1024, world)
        lo, hi = ranges[rank_id]
        dt = full.slice(lo, hi, dev)
        if not args.check:
            del full
    else:
        dt = full
    local_nnz = dt.nnz

    fac = [torch.empty((d, R), dtype=torch.float64, device=f"cuda:{dev}") for d in dims]
    b.factors_random_device(dims, R, FACTOR_SEED, [a.data_ptr() for a in fac], sptr)
    fptr = [a.data_ptr() for a in fac]
    rs = world > 1 and args.reduce == "reducescatter"
    if rs:
        # one reduce-scatter per mode leaves rank g with its row
        # block of M_n; partials padded to world * ceil(I_n / world) rows
        from paper_2201_12523_b200.dist import Collectives, row_shard
        coll = Collectives()
        pads = [row_shard(d, world, rank_id)[2] for d in dims]
        outs = [torch.empty((world * p, R), dtype=torch.float64, device=f"cuda:{dev}") for p in pads]
        shards = [torch.empty((p, R), dtype=torch.float64, device=f"cuda:{dev}") for p in pads]
    else:
        outs = [torch.empty((d, R), dtype=torch.float64, device=f"cuda:{dev}") for d in dims]
    strategy = b.Strategy[args.strategy]
    cfg = b.ExecConfig(num_compute_units=torch.cuda.get_device_properties(dev).multi_processor_count)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")
    # N > 1 over NCCL: the library's own communicator drives the per-mode
    # reduction (blco_dist_mttkrp_all; torch only moves the NCCL unique id).
    # The gloo plumbing runs (ranks sharing one GPU) keep torch's collectives.
    lib_coll = (world > 1 and os.environ.get("BLCO_B200_DIST_BACKEND", "nccl") == "nccl"
                and os.environ.get("BLCO_B200_COLLECTIVES", "library") == "library")
    if lib_coll:
        import torch.distributed as dist
        uid = [b.Communicator.unique_id() if rank_id == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = b.Communicator(uid[0], world, rank_id, dev)
        if not rs:
            shards = outs


    def lib_step(ev=None):
        comm.mttkrp_all(dt, fptr, R, [o.data_ptr() for o in outs], [x.data_ptr() for x in shards],
                        reduce=args.reduce, strategy=strategy, config=cfg, stream=sptr)

    # one GPU: the library's all-mode device entry runs one kernel per mode
    # (the fused all-mode kernel only with BLCO_B200_FUSED=1, factors in L2)
    fused = world == 1 and strategy == b.Strategy.Auto and dt.mttkrp_all_device(
        fptr, R, [o.data_ptr() for o in outs], strategy, cfg, stream=sptr)

    def fused_step(ev=None):
        for o in outs:
            o.zero_()
        if ev is not None:
            ev[0][0].record(stream)
        dt.mttkrp_all_device(fptr, R, [o.data_ptr() for o in outs], strategy, cfg, accumulate=True, stream=sptr)
        if ev is not None:
            ev[0][1].record(stream)

    def step(ev=None):
        if lib_coll:
            return lib_step(ev)
        if fused:
            return fused_step(ev)
        for o in outs:
            o.zero_()
        works = []
        for m in range(N):
            if ev is not None:
                ev[m][0].record(stream)
            dt.mttkrp_device(fptr, R, m, outs[m].data_ptr(), strategy, cfg, accumulate=True, stream=sptr)
            if ev is not None:
                ev[m][1].record(stream)
            if rs:
                # rank g's rows of M_m reduced on NCCL's stream while the mode
                # m+1 kernel runs (outputs are disjoint buffers)
                w = coll.reduce_scatter(shards[m], outs[m], async_op=True)
                if w is not None:
                    works.append(w)
            elif world > 1:
                # partial M_m summed over ranks on NCCL's stream while the
                # mode m+1 kernel runs (outputs are disjoint buffers)
                import torch.distributed as dist
                works.append(dist.all_reduce(outs[m], async_op=True))
        for w in works:
            w.wait()  # the step's end event waits for every reduction

    stats = b.MttkrpStats()
    dt.mttkrp_device(fptr, R, 0, outs[0].data_ptr(), strategy, cfg, stream=sptr, stats=stats)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(N)] for _ in range(args.steps)]
    sev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = b.kernel_launch_count()
    with ClockSampler(dev) as clk:
        for k in range(args.steps):
            flush.zero_()  # L2 flush between steps (outside the step events)
            sev[k][0].record(stream)
            step(evs[k])
            sev[k][1].record(stream)
        torch.cuda.synchronize()
    launches = b.kernel_launch_count() - launches0
    if world > 1:
        dist.barrier()
    step_ms = [sev[k][0].elapsed_time(sev[k][1]) for k in range(args.steps)]
    if lib_coll:
        # one library call per step: the mode kernels alone, timed after the
        # step loop on the same slice (the roofline's launch duration)
        mode_ms = []
        for m in range(N):
            o = torch.zeros((dims[m], R), dtype=torch.float64, device=f"cuda:{dev}")
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(3):
                dt.mttkrp_device(fptr, R, m, o.data_ptr(), strategy, cfg, accumulate=True, stream=sptr)
            e1.record(stream)
            torch.cuda.synchronize()
            mode_ms.append([e0.elapsed_time(e1) / 3])
    elif fused:  # one launch per step: the "mode" timing slot 0 holds the fused kernel
        mode_ms = [[evs[k][0][0].elapsed_time(evs[k][0][1]) for k in range(args.steps)]]
    else:
        mode_ms = [[evs[k][m][0].elapsed_time(evs[k][m][1]) for k in range(args.steps)] for m in range(N)]
    ms = sum(step_ms) / len(step_ms)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    bpe = bytes_per_elem(N, R)
    total_bytes = nnz * N * bpe
    value = total_bytes / (ms * 1e-3) / 1e9
    launch_ms = statistics.mean(statistics.mean(x) for x in mode_ms)  # mean launch of the step's kernels
    peak, peak_source = hbm_peak()
    if fused:
        roofline = roofline_entry(traffic, launch_ms, local_nnz * N * bpe, peak, peak_source,
                                  "k_mttkrp_all3 (fused all-mode kernel, one launch per step)")
    else:
        roofline = roofline_entry(traffic, launch_ms, local_nnz * bpe, peak, peak_source,
                                  "k_mttkrp_sorted (one launch per mode)")

    result = {
        "metric": "MTTKRP all-mode throughput (algorithmic B_elem bytes / time)",
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded Feistel-permuted unique coordinates, uniform [0,1) values; "
                "FactorMatrices::random factors)",
        "config": {"workload": desc, "dims": dims, "nnz": nnz, "rank": R, "modes": N,
                   "tensor_seed": TENSOR_SEED, "factor_seed": FACTOR_SEED, "strategy": args.strategy,
                   "l2": "flushed between steps (512 MiB write, outside the timed events)",
                   "tile_order": tile_order(dims, R),
                   "parallelism": f"span partition x{world}" + (
                       (" + NCCL reduce-scatter of M per mode (row shards), overlapped with the next mode's kernel"
                        if rs else " + NCCL all-reduce of M per mode, overlapped with the next mode's kernel")
                       + (" (libblco_b200 communicator, blco_dist_mttkrp_all)" if lib_coll else
                          " (torch.distributed)")
                       if world > 1 else ""),
                   "bytes_per_elem_per_mode": bpe},
        "per_mode_ms": [round(statistics.mean(x), 4) for x in mode_ms] if not fused else None,
        "step_path": ("fused all-mode kernel (blco_mttkrp_all_device)" if fused else "one kernel per mode"),
        "roofline": roofline,
        "clocks": clk.summary(),
        "gpu_launches": launches,
        "build": {"seconds": round(build_s, 4), "device_stage_s": {k: round(getattr(bst, k), 4) for k in
                                                                   ("sort_seconds", "block_seconds", "reencode_seconds",
                                                                    "batch_seconds")},
                  "nnz_per_s": round(nnz / build_s, 1)},
        "segments_mode0": stats.segments,
    }
    if world == 1 and not args.no_fp32:
        result["fp32_variant"] = fp32_variant(b, torch, dt, dims, R, N, nnz, fac, outs, cfg, sptr, dev, args)
    if args.check:
        # the summed partials of the last step against the whole tensor on this device
        errs = []
        for m in range(N):
            ref = torch.zeros((dims[m], R), dtype=torch.float64, device=f"cuda:{dev}")
            full.mttkrp_device(fptr, R, m, ref.data_ptr(), strategy, cfg, stream=sptr)
            torch.cuda.synchronize()
            got = outs[m]
            if rs:  # gather the row shards back into the whole M_m
                got = torch.empty_like(outs[m])
                coll.all_gather(got, shards[m])
                got = got[: dims[m]]
            errs.append(float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref)))
        result["check"] = {"rel_frobenius_vs_single_device": errs, "ranks": world}
    if not args.no_e2e:
        result["e2e"] = e2e_run(b, torch, dt, dims, R, N, nnz, args, dev, world)
    if rank_id == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            small = args.config in ("cfg1", "nell2")
            gbps, info = reference_sample_run(dims, nnz, R, steps=2, warmup=1, extra=True,
                                              sampler="alto_prefix" if small else "generator_prefix",
                                              skew=None if int(np.prod(np.array(dims, dtype=object))) < 2**64 else 1)
            result["cpu_baseline"] = cpu_baseline_entry(gbps, info)
        except Exception as e:  # noqa: BLE001
            result["cpu_baseline"] = {"value": None, "unit": "GB/s", "cores": None, "kind": "reference",
                                      "sample": f"failed: {e}"}
    if world == 1 and args.config == "amazon" and not args.no_extra:
        # BASELINE configs[1] (NELL-2 shape) beside the headline: its factors
        # sit in L2, so its kernel is bound by the L1 data pipe, not HBM
        del dt, fac, outs, flush
        full = None
        b.release_thread_caches()
        torch.cuda.empty_cache()
        result["nell2"] = resident_extra(b, torch, "nell2", extra_traffic, args, dev)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if rank_id == 0:
        print(json.dumps(result), flush=True)


def resident_extra(b, torch, name, traffic, args, dev):
    """A second resident config measured in the same run (one GPU), reported
    as its own key beside the headline: the same step (all modes, fixed
    factors, L2 flushed between steps, CUDA events on the launching stream)
    through the library's all-mode device entry (blco_mttkrp_all_device: the
    fused all-mode kernel when the factors sit in L2, else one kernel per
    mode), the per-mode kernels timed beside it, and the same physical-DRAM
    roofline for the kernel(s) the step launches."""
    dims, nnz, R, desc = CONFIGS[name]
    N = len(dims)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    dt = b.DeviceTensor.synthetic(dims, nnz, TENSOR_SEED, device=dev)
    fac = [torch.empty((d, R), dtype=torch.float64, device=f"cuda:{dev}") for d in dims]
    b.factors_random_device(dims, R, FACTOR_SEED, [a.data_ptr() for a in fac], sptr)
    fptr = [a.data_ptr() for a in fac]
    outs = [torch.empty((d, R), dtype=torch.float64, device=f"cuda:{dev}") for d in dims]
    optr = [o.data_ptr() for o in outs]
    cfg = b.ExecConfig(num_compute_units=torch.cuda.get_device_properties(dev).multi_processor_count)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")

    def step_all():
        for o in outs:
            o.zero_()
        return dt.mttkrp_all_device(fptr, R, optr, b.Strategy.Auto, cfg, accumulate=True, stream=sptr)

    def step_modes(ev=None):
        for o in outs:
            o.zero_()
        for m in range(N):
            if ev is not None:
                ev[m][0].record(stream)
            dt.mttkrp_device(fptr, R, m, optr[m], b.Strategy.Auto, cfg, accumulate=True, stream=sptr)
            if ev is not None:
                ev[m][1].record(stream)

    steps = max(args.steps, 10)

    def timed(fn, per_mode=False):
        for _ in range(args.warmup):
            fn()
        evs = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(N)] for _ in range(steps)]
        sev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(steps)]
        torch.cuda.synchronize()
        for k in range(steps):
            flush.zero_()
            sev[k][0].record(stream)
            fn(evs[k]) if per_mode else fn()
            sev[k][1].record(stream)
        torch.cuda.synchronize()
        ms = statistics.mean(sev[k][0].elapsed_time(sev[k][1]) for k in range(steps))
        mode_ms = ([statistics.mean(evs[k][m][0].elapsed_time(evs[k][m][1]) for k in range(steps)) for m in range(N)]
                   if per_mode else None)
        return ms, mode_ms

    fused = step_all()
    ms, _ = timed(step_all)
    ms_modes, mode_ms = timed(step_modes, per_mode=True)
    # the M_n of the two paths agree (same per-element terms, summation order aside)
    step_all()
    torch.cuda.synchronize()
    ref = [o.clone() for o in outs]
    step_modes()
    torch.cuda.synchronize()
    agree = max(float(torch.linalg.norm(a - o) / torch.linalg.norm(o)) for a, o in zip(ref, outs))
    bpe = bytes_per_elem(N, R)
    peak, peak_source = hbm_peak()
    if fused:  # one launch per step
        roof = roofline_entry(traffic, ms, nnz * N * bpe, peak, peak_source, "k_mttkrp_all3 (one launch per step)")
    else:
        roof = roofline_entry(traffic, statistics.mean(mode_ms), nnz * bpe, peak, peak_source,
                              "k_mttkrp_sorted (one launch per mode)")
    return {"workload": desc, "dims": dims, "nnz": nnz, "rank": R, "steps": steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 4), "value": round(nnz * N * bpe / (ms * 1e-3) / 1e9, 2),
            "unit": "GB/s (algorithmic B_elem bytes / time)",
            "step_path": "fused all-mode kernel (blco_mttkrp_all_device)" if fused else "per-mode kernels",
            "per_mode_kernels": {"ms_per_step": round(ms_modes, 4), "per_mode_ms": [round(x, 4) for x in mode_ms],
                                 "rel_frobenius_vs_step": agree},
            "roofline": roof, "l2": "flushed between steps (512 MiB write, outside the timed events)"}


def fp32_variant(b, torch, dt, dims, R, N, nnz, fac, outs, cfg, sptr, dev, args):
    """The fp32 variant: same tensor (fp64 values), fp32
    factors/products/output; reported beside the fp64 headline, never as it.
    Bytes per element per mode: 8 (index) + 8 (value) + N*R*4."""
    f32 = [a.float() for a in fac]
    o32 = [torch.empty((d, R), dtype=torch.float32, device=f"cuda:{dev}") for d in dims]
    fp = [a.data_ptr() for a in f32]
    stream = torch.cuda.current_stream()
    for _ in range(2):
        for m in range(N):
            dt.mttkrp_device_f32(fp, R, m, o32[m].data_ptr(), cfg, stream=sptr)
    torch.cuda.synchronize()
    steps = max(3, min(args.steps, 10))
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(N)]
    tot = [0.0] * N
    for _ in range(steps):
        for m in range(N):
            ev[m][0].record(stream)
            dt.mttkrp_device_f32(fp, R, m, o32[m].data_ptr(), cfg, stream=sptr)
            ev[m][1].record(stream)
        torch.cuda.synchronize()
        for m in range(N):
            tot[m] += ev[m][0].elapsed_time(ev[m][1])
    per_mode = [x / steps for x in tot]
    ms = sum(per_mode)
    # accuracy against the fp64 kernel's result of the last timed step (same factors)
    err = [float(torch.linalg.norm(o32[m].double() - outs[m]) / torch.linalg.norm(outs[m])) for m in range(N)]
    bpe = 16 + N * R * 4
    return {"ms_per_step": round(ms, 4), "per_mode_ms": [round(x, 4) for x in per_mode],
            "value": round(nnz * N * bpe / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "bytes_per_elem_per_mode": bpe, "rel_frobenius_vs_fp64": err, "tolerance": 1e-5,
            "note": "fp32 factors/products/output over the fp64-valued BLCO tensor; kernel time, inputs "
                    "resident; not the headline (the reference computes in fp64)"}


def e2e_run(b, torch, dt, dims, R, N, nnz, args, dev, world):
    """Same metric through the public host API (mttkrp_all_modes ->
    blco_mttkrp_all_host): every step uploads the (rank's) BLCO payload from
    pinned host memory in chunks under the compute, uploads the host factors
    and reads every M_n back into pinned host memory.  With N > 1 ranks the
    outputs stay on the device, are summed with an NCCL all-reduce per mode,
    and every rank reads the summed M_n back.  Wall clock per step, max over
    ranks (the API call returns after its outputs are written)."""
    host = dt.to_host()
    idx = b.api.pinned_empty(host.idx.size, np.uint64)
    vals = b.api.pinned_empty(host.vals.size, np.float64)
    idx[:] = host.idx
    vals[:] = host.vals
    ht = b.BlcoTensor(host.layout, host.max_nnz_per_block, host.keys, host.offsets, idx, vals)
    f = b.FactorMatrices.random(dims, R, FACTOR_SEED)
    pf = []
    for a in f.factors:
        p = b.api.pinned_empty(a.size, np.float64).reshape(a.shape)
        p[:] = a
        pf.append(p)
    f = b.FactorMatrices(R, pf)
    outs = [b.api.pinned_empty(d * R, np.float64).reshape(d, R) for d in dims]
    cfg = b.ExecConfig(num_compute_units=torch.cuda.get_device_properties(dev).multi_processor_count)
    strategy = b.Strategy[args.strategy]
    rep = b.AllModesReport()
    rs = world > 1 and args.reduce == "reducescatter"
    d2h = sum(d * R * 8 for d in dims)
    if world > 1:
        import torch.distributed as dist
        if rs:
            # row-padded partials (the padding rows stay zero), each rank
            # reads back its own row shard of every M_n
            from paper_2201_12523_b200.dist import Collectives, row_shard
            coll = Collectives()
            pads = [row_shard(d, world, 0)[2] for d in dims]
            douts = [torch.zeros((world * p, R), dtype=torch.float64, device=f"cuda:{dev}") for p in pads]
            shards = [torch.empty((p, R), dtype=torch.float64, device=f"cuda:{dev}") for p in pads]
            touts = [torch.from_numpy(b.api.pinned_empty(p * R, np.float64).reshape(p, R)) for p in pads]
            d2h = sum(p * R * 8 for p in pads)
        else:
            douts = [torch.empty((d, R), dtype=torch.float64, device=f"cuda:{dev}") for d in dims]
            touts = [torch.from_numpy(o) for o in outs]

    def step():
        if world == 1:
            b.mttkrp_all_modes(ht, f, cfg, strategy, outs=outs, device=dev, report=rep)
            return
        b.mttkrp_all_modes(ht, f, cfg, strategy, device=dev, report=rep, device_outs=[o.data_ptr() for o in douts])
        if rs:
            for o, sh, t in zip(douts, shards, touts):
                coll.reduce_scatter(sh, o)
                t.copy_(sh, non_blocking=True)
        else:
            works = [dist.all_reduce(o, async_op=True) for o in douts]
            for w, o, t in zip(works, douts, touts):
                w.wait()
                t.copy_(o, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    for _ in range(max(1, min(args.warmup, 3))):
        step()
    torch.cuda.synchronize()
    n = max(1, min(args.steps, 10))
    if world > 1:
        dist.barrier()
    w0 = time.perf_counter()
    for _ in range(n):
        step()
    wall_ms = (time.perf_counter() - w0) * 1e3 / n
    if world > 1:
        t = torch.tensor([wall_ms], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall_ms = float(t.item())
    bpe = bytes_per_elem(N, R)
    return {"value": round(nnz * N * bpe / (wall_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "ms_per_step": round(wall_ms, 3), "api_device_ms_per_call": round(rep.device_ms, 3), "steps": n,
            "h2d_bytes_per_step": int(rep.h2d_bytes), "d2h_bytes_per_step": int(d2h),
            "chunks": int(rep.chunks), "launches_per_step": int(rep.launches),
            "timing": "host wall clock per step (synchronous API), max over ranks",
            "path": "mttkrp_all_modes (blco_mttkrp_all_host): pinned host payload uploaded in chunks under "
                    "the all-mode kernels, host factors in, M_n out to pinned host memory"
                    + ("" if world == 1 else
                       " after an NCCL reduce-scatter of the ranks' device partials (each rank reads its row shard)"
                       if rs else " after an NCCL all-reduce of the ranks' device partials")}


# ------------------------------------------------------------ reference arm


ALS_CONFIGS = {
    # BASELINE configs[3]: 4-mode Delicious-shaped tensor with skewed power-law
    # indices (floor(I * u^skew), first nnz distinct draws), R=16, 10 iterations
    "delicious_als": ([532924, 17262471, 2480308, 1443], 140_126_181, 16, 4,
                      "synthetic Delicious-shaped 532924x17262471x2480308x1443, 140,126,181 nnz, "
                      "power-law draws floor(I*u^4), R=16, CP-ALS 10 iterations (BASELINE configs[3])"),
    # small 4-mode case for the multi-rank tests (not a BASELINE config)
    "als_tiny": ([3000, 4000, 2500, 60], 400_000, 16, 2,
                 "synthetic 4-mode 3000x4000x2500x60, 400,000 nnz, power-law draws floor(I*u^2), R=16, "
                 "CP-ALS 10 iterations (test case)"),
    "enron_als": ([6066, 5699, 244268, 1176], 54_202_099, 16, 4,
                  "synthetic Enron-shaped 6066x5699x244268x1176, 54,202,099 nnz, power-law draws floor(I*u^4), "
                  "R=16, CP-ALS 10 iterations"),
}


def run_cpals(args, world=1, rank_id=0, local=0):
    """CP-ALS (proj/src/cpals.cpp:66-111) with every step on the device.  With
    N > 1 ranks: the distributed driver (paper_2201_12523_b200.dist)
    on contiguous span ranges -- reduce-scatter of M_n, local row-block solve,
    all-reduce of the R x R Gram, all-gather of A_n."""
    import torch

    import paper_2201_12523_b200 as b

    dims, nnz, R, skew, desc = ALS_CONFIGS[args.config]
    N = len(dims)
    dev = local
    # DRAM bytes per MTTKRP launch of this build (ncu child process, before
    # this process allocates anything), as run_ours
    traffic = (world == 1 and not args.no_ncu and live_traffic(args.config)) or (
        committed_traffic("delicious") if args.config == "delicious_als" else None)
    torch.cuda.set_device(dev)
    if world > 1:
        dist_init(torch, dev)
    bst = b.BuildStats()
    t0 = time.perf_counter()
    full = b.DeviceTensor.synthetic_draws(dims, nnz, TENSOR_SEED, skew, 64, 1 << 27, dev, bst)
    build_s = time.perf_counter() - t0
    if world > 1:
        lo, hi = b.partition(full.block_nnz(), 1024, world)[rank_id]
        dt = full.slice(lo, hi, dev)
        if not args.check:
            del full
    else:
        dt = full
    cfg = b.ExecConfig(num_compute_units=torch.cuda.get_device_properties(dev).multi_processor_count)
    iters = 10
    opts = lambda n: b.CpAlsOptions(rank=R, max_iters=n, tol=-1e300, seed=FACTOR_SEED)  # noqa: E731
    if world > 1:
        from paper_2201_12523_b200.dist import cp_als_distributed
        als = lambda n, timing=False: cp_als_distributed(dt, dims, opts(n), cfg, timing=timing)  # noqa: E731
    else:
        als = lambda n, timing=False: b.cp_als(dt, opts(n), cfg)  # noqa: E731
    als(2)  # warm-up
    torch.cuda.synchronize()

    def timed(n):
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        m = als(n, True)
        e1.record()
        torch.cuda.synchronize()
        return m, e0.elapsed_time(e1)

    launches0 = b.kernel_launch_count()
    with ClockSampler(dev) as clk:
        model, ms_total = timed(iters)
        _, ms_two = timed(2)
    # per-iteration device time of the ALS loop (CUDA events around every
    # iteration: N MTTKRPs + solve/normalise/Gram + fit, and with N > 1 the
    # collectives); the call's fixed costs (allocation, init, |X|^2, initial
    # Grams, final copies) excluded.  Max over ranks.
    ms_iter = model.device_ms["iterations_ms"] / model.device_ms["iterations"]
    ms_mt = model.device_ms["mttkrp_ms"] / iters
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms_iter, ms_mt], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_iter, ms_mt = float(t[0]), float(t[1])
    # MTTKRP alone on the final factors: per-mode kernel time (roofline)
    if world > 1:
        fac = [a.contiguous() for a in model.factors]
    else:
        fac = [torch.from_numpy(a).cuda(dev) for a in model.factors.factors]
    outs = [torch.empty((d, R), dtype=torch.float64, device=f"cuda:{dev}") for d in dims]
    sptr = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        for m in range(N):
            dt.mttkrp_device([a.data_ptr() for a in fac], R, m, outs[m].data_ptr(), config=cfg, stream=sptr)
    mode_ms = []
    for m in range(N):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(5):
            dt.mttkrp_device([a.data_ptr() for a in fac], R, m, outs[m].data_ptr(), config=cfg, stream=sptr)
        a1.record()
        torch.cuda.synchronize()
        mode_ms.append(a0.elapsed_time(a1) / 5)
    bpe = bytes_per_elem(N, R)
    peak, peak_source = hbm_peak()
    roofline = roofline_entry(traffic, statistics.mean(mode_ms), dt.nnz * bpe, peak, peak_source,
                              "k_mttkrp_sorted (one launch per mode, final factors)")
    launches = b.kernel_launch_count() - launches0
    check = None
    if args.check and world > 1:
        # the distributed run against single-device cp_als of the whole tensor
        one = b.cp_als(full, opts(iters), cfg)
        fdiff = max(abs(x - y) for x, y in zip(model.fit_history, one.fit_history))
        ferr = [float(np.linalg.norm(a.cpu().numpy() - f) / np.linalg.norm(f))
                for a, f in zip(model.factors, one.factors.factors)]
        check = {"max_abs_fit_diff_vs_single_device": fdiff, "factor_rel_frobenius": ferr,
                 "lambda_rel": float(np.linalg.norm(model.lambda_ - one.lambda_) / np.linalg.norm(one.lambda_)),
                 "ranks": world}
    cpu = None
    if rank_id == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu, _ = als_reference_baseline(dims, nnz, R, skew, args.ref_step_s)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "ms", "cores": None, "kind": "reference", "sample": f"failed: {e}"}
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if rank_id != 0:
        return
    print(json.dumps({
        "metric": "CP-ALS time per iteration (N MTTKRPs + device Gram/solve/normalise + fit)",
        "value": round(ms_iter, 3), "unit": "ms", "n_gpus": world, "steps": iters, "warmup": 2,
        "ms_per_step": round(ms_iter, 3), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic power-law draws (seeded)",
        "config": {"workload": desc, "dims": dims, "nnz": nnz, "rank": R, "skew": skew,
                   "iterations": iters, "tol": "-inf (exactly 10 iterations, cpals.cpp:107)",
                   "parallelism": (f"span partition x{world}; per mode reduce-scatter of M_n, row-block solve, "
                                   "all-reduce of the R x R Gram, all-gather of A_n") if world > 1 else "1 GPU"},
        "fit_history": model.fit_history,
        "cp_als_call_ms": {"iters_10": round(ms_total, 2), "iters_2": round(ms_two, 2),
                           "note": "whole API call incl. allocation and the initial/final copies"},
        "device_ms": {"per_iteration": round(ms_iter, 3),
                      "mttkrp_per_iteration": round(ms_mt, 3),
                      "dense_per_iteration": round(ms_iter - ms_mt, 3)},
        "mttkrp_per_mode_ms": [round(x, 4) for x in mode_ms],
        "roofline": roofline,
        "clocks": clk.summary(), "gpu_launches": launches,
        "build": {"seconds": round(build_s, 3), "nnz_per_s": round(nnz / build_s, 1)},
        **({"check": check} if check else {}),
        **({"cpu_baseline": cpu} if cpu else {}),
    }), flush=True)


def als_reference_baseline(dims, nnz, R, skew, step_s=4.0, steps=2, warmup=1) -> tuple[dict, dict]:
    """The reference CPU MTTKRP part of one CP-ALS iteration (N blco::mttkrp
    calls), timed on a generator-prefix sample of the same power-law tensor
    and extrapolated by nnz (reference_sample_run).  The reference iteration
    also runs the dense Gram / solve / normalise steps on the host, so this is
    a lower bound of its time per iteration."""
    gbps, info = reference_sample_run(dims, nnz, R, steps=steps, warmup=warmup, target_step_s=step_s,
                                      sampler="generator_prefix", skew=skew)
    N = len(dims)
    ms = nnz * N * bytes_per_elem(N, R) / (gbps * 1e9) * 1e3
    entry = cpu_baseline_entry(gbps, info)
    entry.update({"value": round(ms, 1), "unit": "ms", "mttkrp_gbps": round(gbps, 4),
                  "note": "extrapolated: the reference's N-mode MTTKRP time per ALS iteration on the full tensor "
                          "(its dense epilogue not included, so the reference iteration is slower still)"})
    return entry, info


STREAM_CONFIGS = {
    # BASELINE configs[4]: Reddit-2015-shaped, 4.69B nnz, 64-bit layout (one key,
    # 35 blocks of 2^27), streamed through a 24 GiB device budget
    "reddit_stream": ([8211298, 176962, 8116559], 4_687_474_081, 32, 64,
                      "synthetic Reddit-2015-shaped 8211298x176962x8116559, ~4.69B nnz (75 GB BLCO in pinned "
                      "host memory), R=32, out-of-memory streaming, DeviceBudget{24 GiB, 4 queues, 2 GiB}"),
    "reddit_stream_small": ([8211298, 176962, 8116559], 600_000_000, 32, 8,
                            "synthetic Reddit-shaped, 0.6B nnz (9.6 GB pinned), R=32, streamed, 24 GiB budget"),
    "reddit_stream_tiny": ([8211298, 176962, 8116559], 20_000_000, 32, 4,
                           "synthetic Reddit-shaped, 20M nnz, R=32, streamed (multi-rank plumbing test size)"),
    "reddit_file_small": ([8211298, 176962, 8116559], 600_000_000, 32, 8,
                          "synthetic Reddit-shaped, 0.6B nnz written as a .blco container (9.6 GB) and streamed "
                          "from the file (native pinned-ring reader, device-side element checks), 24 GiB budget"),
}


def run_stream(args, world, rank_id, local):
    """stream_mttkrp (proj/src/streaming.cpp:103-309) over pinned host blocks.

    One all-mode step = every block crosses the host link once and all N
    modes run on it while resident (stream_mttkrp_all_modes).  With N > 1
    ranks each rank generates and streams its own
    contiguous range of ALTO chunks over its own host link into device
    partials, which an NCCL all-reduce per mode sums; time = max over ranks."""
    import torch

    import paper_2201_12523_b200 as b

    dims, nnz_target, R, nchunks, desc = STREAM_CONFIGS[args.config]
    N = len(dims)
    dev = local
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist
        dist_init(torch, dev)
    # host-link peak: best of 10 pinned 1 GiB H2D copies
    src = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(1 << 30, dtype=torch.uint8, device=f"cuda:{dev}")
    best = 0.0
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, (1 << 30) / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del src, dst
    torch.cuda.empty_cache()
    # this rank's ALTO chunks, generated on the device into pinned host memory
    c0, c1 = nchunks * rank_id // world, nchunks * (rank_id + 1) // world
    frac = float(np.prod(np.array(dims, dtype=np.float64))) / 2.0 ** 64
    ncand = int(nnz_target / nchunks / frac) + 1
    cap = int(nnz_target * 1.02 * (c1 - c0) / nchunks) + ncand
    t0 = time.perf_counter()
    idx = b.api.pinned_empty(cap, np.uint64)
    vals = b.api.pinned_empty(cap, np.float64)
    alloc_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    off = 0
    for c in range(c0, c1):
        if off + ncand > cap:
            raise RuntimeError("stream bench: pinned buffer too small")
        off += b.api.synth_alto_chunk(dims, c, nchunks, ncand, TENSOR_SEED, idx[off:], vals[off:], device=dev)
    gen_s = time.perf_counter() - t0
    local_nnz = off
    total = local_nnz
    if world > 1:
        t = torch.tensor([local_nnz], dtype=torch.int64, device=f"cuda:{dev}")
        dist.all_reduce(t)
        total = int(t.item())
    bmax = 1 << 27
    layout = b.make_layout(dims, 64)
    blocks = [(o, min(bmax, local_nnz - o)) for o in range(0, local_nnz, bmax)]
    f = b.FactorMatrices.random(dims, R, FACTOR_SEED)
    budget = b.DeviceBudget(capacity_bytes=24 << 30, num_queues=4, reservation_bytes=bmax * 16)
    cfg = b.ExecConfig(num_compute_units=torch.cuda.get_device_properties(dev).multi_processor_count)
    douts = [torch.empty((d, R), dtype=torch.float64, device=f"cuda:{dev}") for d in dims] if world > 1 else None

    def source():
        for o, n in blocks:
            yield (0, idx[o:o + n], vals[o:o + n])

    file_info = None
    if "file" in args.config:
        # the tensor as a .blco container (blco_format.cpp:149-172 layout),
        # written from the pinned arrays; the stream then reads the file
        import tempfile
        fdir = os.environ.get("BLCO_B200_FILE_DIR") or tempfile.gettempdir()
        path = os.path.join(fdir, f"bench_{args.config}_{rank_id}.blco")
        w0 = time.perf_counter()
        with open(path, "wb") as fh:
            fh.write(b"BLCO" + np.array([1, N], "<u2").tobytes() + np.array(dims, "<u8").tobytes()
                     + np.array([64], "<u2").tobytes() + np.array(layout.mode_bits, "<u2").tobytes()
                     + np.array([bmax, len(blocks)], "<u8").tobytes())
            for o, n in blocks:
                fh.write(np.array([0, n], "<u8").tobytes())
                fh.write(memoryview(idx[o:o + n]))
                fh.write(memoryview(vals[o:o + n]))
        file_info = {"path": path, "bytes": os.path.getsize(path), "write_s": round(time.perf_counter() - w0, 2),
                     "note": "just written, so mostly served from the page cache"}

        def source():  # noqa: F811 - the file replaces the in-memory blocks
            return b.FileBlockSource(path, dev)

    def one_all():
        rep = b.StreamReport()
        w0 = time.perf_counter()
        if world == 1:
            b.stream_mttkrp_all_modes(source(), f, budget, cfg, report=rep, layout=layout, max_nnz_per_block=bmax,
                                      block_count=len(blocks), device=dev)
        else:
            b.stream_mttkrp_all_modes(source(), f, budget, cfg, report=rep, layout=layout, max_nnz_per_block=bmax,
                                      block_count=len(blocks), device=dev, device_outs=[o.data_ptr() for o in douts])
            for o in douts:
                dist.all_reduce(o)
            torch.cuda.synchronize()
        return rep, time.perf_counter() - w0

    def one(mode):
        rep = b.StreamReport()
        b.stream_mttkrp(source(), f, mode, budget, cfg, report=rep, layout=layout, max_nnz_per_block=bmax,
                        block_count=len(blocks), device=dev)
        return rep

    one_all()  # warm-up (allocations, clocks)
    steps = max(1, min(args.steps, 3))
    if world > 1:
        dist.barrier()
    with ClockSampler(dev) as clk:
        runs = [one_all() for _ in range(steps)]
    reps = [r for r, _ in runs]
    # device-timed stream (events inside the library) for N = 1; with N > 1
    # the step also holds the NCCL reduction, so host wall time, max over ranks
    step_s = statistics.mean(r.total_seconds for r in reps) if world == 1 else statistics.mean(w for _, w in runs)
    if world > 1:
        t = torch.tensor([step_s], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_s = float(t.item())
    per_mode = [one(m) for m in range(N)] if world == 1 else []  # the reference's per-mode API, for comparison
    overall = [r.overall_gbps for r in reps]
    bpe = bytes_per_elem(N, R)
    value = total * N * bpe / step_s / 1e9
    result = {
        "metric": "out-of-memory MTTKRP all-mode throughput (algorithmic B_elem bytes / time), host-link bound",
        "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": steps, "warmup": 1,
        "ms_per_step": round(step_s * 1e3, 2), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic uniform (ALTO-chunked generator, seeded)",
        "config": {"workload": desc, "dims": dims, "nnz": total, "rank": R, "blocks_per_rank": len(blocks),
                   "budget": {"capacity_bytes": 24 << 30, "num_queues": 4, "reservation_bytes": bmax * 16},
                   "step": "stream_mttkrp_all_modes: every block crosses the host link once, all N modes "
                           "computed on it while resident"
                           + ("" if world == 1 else "; ranks stream disjoint ALTO chunk ranges over their own "
                                                    "links, NCCL all-reduce of M per mode")},
        "stream": {"overall_gbps_per_step_rank0": [round(x, 2) for x in overall],
                   "compute_gbps_per_step_rank0": [round(r.compute_gbps, 2) for r in reps],
                   "h2d_peak_gbps": round(best, 2),
                   "link_fraction_per_step_rank0": [round(x / best, 4) for x in overall],
                   "bytes_streamed_per_step_rank0": reps[0].bytes_streamed,
                   "peak_resident_bytes": reps[0].peak_resident_bytes,
                   "transfer_busy_s": [round(r.transfer_busy_seconds, 3) for r in reps],
                   "compute_busy_s": [round(r.compute_busy_seconds, 3) for r in reps]},
        "roofline": {"bound": "host-link", "achieved": round(statistics.mean(overall), 2), "peak": round(best, 2),
                     "unit": "GB/s", "frac": round(statistics.mean(overall) / best, 4), "traffic": None,
                     "kernel": "H2D cudaMemcpyAsync (BLCO blocks, 16 B/nnz) overlapped with k_mttkrp_sorted x N"},
        "clocks": clk.summary(),
        "generate": {"pinned_alloc_s": round(alloc_s, 2), "generate_s": round(gen_s, 2)},
    }
    if file_info:
        result["file"] = file_info
        try:
            os.remove(file_info["path"])
        except OSError:
            pass
    if args.check and world > 1:
        # the ranks' all-reduced M_n of the last step against one device
        # streaming every chunk of the tensor (stream_mttkrp_all_modes, G = 1)
        cap_all = int(nnz_target * 1.02) + ncand
        aidx = b.api.pinned_empty(cap_all, np.uint64)
        avals = b.api.pinned_empty(cap_all, np.float64)
        n_all = 0
        for c in range(nchunks):
            n_all += b.api.synth_alto_chunk(dims, c, nchunks, ncand, TENSOR_SEED, aidx[n_all:], avals[n_all:],
                                            device=dev)
        ablocks = [(o, min(bmax, n_all - o)) for o in range(0, n_all, bmax)]
        want = b.stream_mttkrp_all_modes(((0, aidx[o:o + n], avals[o:o + n]) for o, n in ablocks), f, budget, cfg,
                                         layout=layout, max_nnz_per_block=bmax, block_count=len(ablocks),
                                         device=dev)
        errs = [float(np.linalg.norm(o.cpu().numpy() - w) / np.linalg.norm(w)) for o, w in zip(douts, want)]
        result["check"] = {"rel_frobenius_vs_single_device": errs, "ranks": world, "nnz_single_device": n_all}
    if per_mode:
        result["stream"]["per_mode_api"] = {
            "total_s": round(sum(r.total_seconds for r in per_mode), 3),
            "overall_gbps_per_mode": [round(r.overall_gbps, 2) for r in per_mode],
            "note": "stream_mttkrp once per mode (the reference API): the tensor crosses the link N times"}
    if rank_id == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            gbps, info = reference_sample_run(dims, nnz_target, R, steps=2, warmup=1, target_step_s=args.ref_step_s,
                                              sampler="generator_prefix", op="stream")
            result["cpu_baseline"] = cpu_baseline_entry(gbps, info)
        except Exception as e:  # noqa: BLE001
            result["cpu_baseline"] = {"value": None, "unit": "GB/s", "cores": None, "kind": "reference",
                                      "sample": f"failed: {e}"}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank_id == 0:
        print(json.dumps(result), flush=True)


def tile_order(dims, R) -> str:
    """The CTA dispatch order the library picks (mttkrp.cu panel_plan)."""
    knob = os.environ.get("BLCO_B200_PANEL", "")
    if len(dims) < 3 or sum(dims) * R * 8 <= (96 << 20) or knob == "0":
        return "ALTO"
    if "," in knob:
        return f"panel-ordered (BLCO_B200_PANEL={knob})"
    mb = int(os.environ.get("BLCO_B200_PANEL_MB", "32"))
    b = max(0, ((mb << 20) // (R * 8) // 2).bit_length() - 1)
    return f"panel-ordered: 2^{b}-row panels of the target x second-longest mode, ALTO order inside"


def ref_step_s(args) -> float:
    """Per-step sample size target of the reference arm (seconds of
    per-element work on top of the fixed per-call cost), so --steps K
    --warmup W stays within a few minutes (about 100 s of element work)."""
    return max(0.2, min(args.ref_step_s, 100.0 / max(1, args.steps + args.warmup)))


def run_reference(args, world, rank_id):
    """--impl reference: the unmodified reference (oracle/_ref/libblco_ref.so)
    on the host cores, same metric/unit as our arm for the config.  Rank 0
    alone runs; bounded samples (reference_sample_run)."""
    if rank_id != 0:
        return
    kind = "mttkrp"
    if args.config in STREAM_CONFIGS:
        dims, nnz, R, _, desc = STREAM_CONFIGS[args.config]
        kind = "stream"
    elif args.config in ALS_CONFIGS:
        dims, nnz, R, skew, desc = ALS_CONFIGS[args.config]
        kind = "als"
    else:
        dims, nnz, R, desc = CONFIGS[args.config]
    if args.rank:
        R = args.rank
    N = len(dims)
    wide = int(np.prod(np.array(dims, dtype=object))) >= 2**64 or make_wide(dims)
    try:
        if kind == "als":
            cpu, info = als_reference_baseline(dims, nnz, R, skew, ref_step_s(args), args.steps, args.warmup)
            print(json.dumps({
                "impl": "reference",
                "metric": "CP-ALS time per iteration (N MTTKRPs + device Gram/solve/normalise + fit)",
                "value": cpu["value"], "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(info["step_s"] * 1e3, 3), "extrapolated": info["extrapolated"],
                "sample_nnz": info["sample_nnz"], "sample_fraction": round(info["sample_fraction"], 6),
                "full_ms_per_step_extrapolated": cpu["value"],
                "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic power-law draws (same generator and seeds as the ours arm)",
                "config": {"workload": desc, "dims": dims, "nnz": nnz, "rank": R, "skew": skew},
                "cpu_baseline": cpu,
                "e2e": {"value": cpu["value"], "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "path": "unmodified reference blco::build_blco + blco::mttkrp x N (proj/src, oracle/_ref), "
                        "extrapolated from a generator-prefix sample; dense epilogue not included"}), flush=True)
            return
        small = kind == "mttkrp" and not wide and nnz <= 200_000_000
        gbps, info = reference_sample_run(dims, nnz, R, steps=args.steps, warmup=args.warmup,
                                          target_step_s=ref_step_s(args),
                                          sampler="alto_prefix" if small else "generator_prefix",
                                          skew=1 if kind == "mttkrp" and wide else None,
                                          op="stream" if kind == "stream" else "mttkrp")
    except Exception as e:  # noqa: BLE001
        print(json.dumps({"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"}), flush=True)
        return
    result = {
        "impl": "reference",
        "metric": ("out-of-memory MTTKRP all-mode throughput (algorithmic B_elem bytes / time), host-link bound"
                   if kind == "stream" else "MTTKRP all-mode throughput (algorithmic B_elem bytes / time)"),
        "value": round(gbps, 4),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        # the timed steps are of the sample: their real duration, and the
        # full-tensor step the value is computed from (a + b*nnz) beside it
        "ms_per_step": round(info["step_s"] * 1e3, 3),
        "extrapolated": info["extrapolated"],
        "sample_nnz": info["sample_nnz"],
        "sample_fraction": round(info["sample_fraction"], 6),
        "full_ms_per_step_extrapolated": round(info["full_step_s"] * 1e3, 3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (same generator and seeds as the ours arm)",
        "config": {"workload": desc, "dims": dims, "nnz": nnz, "rank": R, "modes": N,
                   "bytes_per_elem_per_mode": bytes_per_elem(N, R)},
        "cpu_baseline": cpu_baseline_entry(gbps, info),
        "e2e": {"value": round(gbps, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "path": "unmodified reference blco::build_blco + blco::" + ("stream_mttkrp" if kind == "stream" else "mttkrp")
                + f" (proj/src, compiled into oracle/_ref/libblco_ref.so), ExecConfig{{num_threads = {info['threads']}}}"
                  " (the faster of 1 thread and all host threads)",
    }
    print(json.dumps(result), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS) + sorted(ALS_CONFIGS) + sorted(STREAM_CONFIGS),
                    default="amazon",
                    help="default: BASELINE configs[2] (Amazon shape), the config the metric is quoted on")
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--strategy", choices=["Auto", "Register", "Hierarchical"], default="Auto")
    ap.add_argument("--reduce", choices=["reducescatter", "allreduce"], default="reducescatter",
                    help="N > 1: how the per-rank partial M_n are combined (SURVEY 8e)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp32", action="store_true", help="skip the fp32 variant line item")
    ap.add_argument("--ref-step-s", type=float, default=4.0)
    ap.add_argument("--check", action="store_true",
                    help="compare the step's (reduced) M_n with a single-device MTTKRP of the whole tensor")
    ap.add_argument("--no-ncu", action="store_true", help="skip the live ncu DRAM-traffic pass (use profiles/)")
    ap.add_argument("--no-extra", action="store_true", help="skip the NELL-2 key beside the Amazon headline")
    ap.add_argument("--traffic-probe", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.traffic_probe:
        traffic_probe_worker(args)
        return
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # --gpus N without a launcher: one rank per GPU under torchrun
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), *sys.argv[1:]]
        sys.exit(subprocess.run(cmd).returncode)
    world, rank_id, local = dist_env()
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")
    if args.impl == "reference":
        run_reference(args, world, rank_id)
        return
    if args.config in STREAM_CONFIGS:
        run_stream(args, world, rank_id, local)
        return
    if args.config in ALS_CONFIGS:
        run_cpals(args, world, rank_id, local)
        return
    run_ours(args, world, rank_id, local)


if __name__ == "__main__":
    main()

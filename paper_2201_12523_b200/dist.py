"""Multi-GPU drivers over torch.distributed.

One process per GPU.  The tensor is split into contiguous, nnz-balanced span
ranges (``partition`` + ``DeviceTensor.slice``), factor matrices are
replicated, and every rank computes a full partial ``M_n`` of its range with
the device MTTKRP.  The only exchange is the summation of those partials:

* ``mttkrp_reduce_scatter``: the all-mode step with fixed factors.  One
  reduce-scatter per mode leaves rank g with rows [g*P, (g+1)*P) of ``M_n``
  (P = ceil(I_n / G)); the collective of mode n runs on NCCL's stream while
  the mode n+1 kernel runs (outputs are separate buffers).
* ``cp_als_distributed``: CP-ALS (proj/src/cpals.cpp:66-111) with, per mode,
  reduce-scatter of M_n -> local row-block solve A = M V^-1 fused with the
  partial Gram (blco_als_solve) -> all-reduce of the R x R Gram, whose
  diagonal carries the column norms -> local normalisation (blco_als_normalize)
  -> all-gather of A_n.  The fit's <X, Xhat> is a per-rank partial over its
  rows of the last mode, all-reduced with |X|^2 at the start.

Torch is plumbing here: device buffers, the stream and the collectives
(backend ``nccl`` on a node; ``gloo`` stages through host memory and is what
the one-GPU and CPU tests use).  Every arithmetic step is a kernel of
libblco_b200.so.  Summation orders differ from the single-device run (the
partial Grams and M_n are summed across ranks), so parity is tolerance-based
(fit within 1e-10, factors within 1e-8 relative Frobenius, tests/).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib as L
from .api import (CpAlsError, CpAlsOptions, DeviceTensor, Error, ExecConfig, FormatError, Strategy, _check,
                  factors_random_device)

lib = L.lib


def row_shard(n_rows: int, world: int, rank: int) -> tuple[int, int, int]:
    """Rank `rank`'s row block of an n_rows x R matrix padded to world * P rows:
    (first row, valid rows, P)."""
    per = -(-n_rows // world) if n_rows else 0
    lo = rank * per
    return lo, max(0, min(n_rows, lo + per) - lo), per


class Collectives:
    """all-reduce / reduce-scatter / all-gather on device tensors.  NCCL takes
    them in place on its own stream; gloo (CPU tests, several ranks sharing a
    GPU) stages through host memory."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.staged = dist.get_backend(group) == "gloo"

    def all_reduce(self, t, async_op: bool = False):
        if self.staged and t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
            return None
        return self.dist.all_reduce(t, group=self.group, async_op=async_op)

    def reduce_scatter(self, out, inp, async_op: bool = False):
        if self.staged and inp.is_cuda:
            h = out.cpu()
            self.dist.reduce_scatter_tensor(h, inp.cpu(), group=self.group)
            out.copy_(h)
            return None
        return self.dist.reduce_scatter_tensor(out, inp, group=self.group, async_op=async_op)

    def all_gather(self, out, inp, async_op: bool = False):
        if self.staged and inp.is_cuda:
            h = out.cpu()
            self.dist.all_gather_into_tensor(h, inp.cpu(), group=self.group)
            out.copy_(h)
            return None
        return self.dist.all_gather_into_tensor(out, inp, group=self.group, async_op=async_op)


def mttkrp_reduce_scatter(t: DeviceTensor, d_factors: Sequence[int], rank: int, outs, shards,
                          coll: Collectives, strategy: Strategy = Strategy.Auto,
                          config: ExecConfig | None = None, stream: int = 0, events=None) -> list:
    """All-mode MTTKRP of this rank's span range with fixed factors, each
    padded partial ``outs[n]`` (world*P_n x R, torch, zeroed here) reduced into
    this rank's row shard ``shards[n]`` (P_n x R).  Returns the pending
    collective handles (NCCL) -- the caller waits on them."""
    works = []
    for n, o in enumerate(outs):
        o.zero_()
        if events is not None:
            events[n][0].record()
        t.mttkrp_device(d_factors, rank, n, o.data_ptr(), strategy, config, accumulate=True, stream=stream)
        if events is not None:
            events[n][1].record()
        w = coll.reduce_scatter(shards[n], o, async_op=True)
        if w is not None:
            works.append(w)
    return works


@dataclass
class DistCpModel:
    """Result of ``cp_als_distributed``: factors stay on the device (I_n x R
    views of the all-gathered, row-padded buffers), replicated on every rank."""
    factors: list
    lambda_: np.ndarray
    fit_history: list[float]
    seed: int = 0
    device_ms: dict = field(default_factory=dict)

    def final_fit(self) -> float:
        return self.fit_history[-1] if self.fit_history else 0.0


def cp_als_distributed(t: DeviceTensor, dims: Sequence[int], opts: CpAlsOptions,
                       config: ExecConfig | None = None, group=None, timing: bool = False) -> DistCpModel:
    """CP-ALS over the ranks of `group`; `t` is this rank's span range of the
    tensor (``DeviceTensor.slice``), `dims` the full mode lengths.  Same
    iteration, stop test and error behaviour as blco::cp_als
    (proj/src/cpals.cpp:66-111): FactorMatrices::random(dims, R, seed) on every
    rank, exactly max_iters iterations unless Δfit < tol after the first."""
    import torch

    if opts.rank < 1:
        raise FormatError("cp_als: rank must be >= 1")
    if opts.max_iters < 0:
        raise FormatError("cp_als: max_iters must be >= 0")
    config = config or ExecConfig()
    config.validate()
    coll = Collectives(group)
    G, g = coll.world, coll.rank
    N, R = len(dims), int(opts.rank)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream().cuda_stream
    sp = C.c_void_p(stream)
    f64 = dict(dtype=torch.float64, device=dev)

    shard = [row_shard(int(d), G, g) for d in dims]
    A = [torch.zeros((G * per, R), **f64) for (_, _, per) in shard]  # row-padded, replicated
    factors_random_device(dims, R, opts.seed, [a.data_ptr() for a in A], stream)
    fptr = [a.data_ptr() for a in A]
    lam = np.ones(R)
    if opts.max_iters == 0:
        return DistCpModel([a[:d] for a, d in zip(A, dims)], lam, [], opts.seed)

    grams = torch.empty((N, R, R), **f64)
    gpart = torch.empty((R, R), **f64)
    dlam = torch.empty(R, **f64)
    scal = torch.zeros(4, **f64)  # |X|^2, <X, Xhat> partial, fit
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    _check(lib.blco_tensor_norm_sq(t.handle, C.c_void_p(scal.data_ptr()), sp))
    coll.all_reduce(scal[0:1])
    xn = float(scal[0].item())
    if xn == 0.0:
        raise FormatError("cp_als: zero-norm tensor")
    # Gram of the initial factors: each rank's rows, summed
    for n in range(N):
        lo, rows, _ = shard[n]
        _check(lib.blco_als_gram(C.c_void_p(A[n].data_ptr() + lo * R * 8), rows, R,
                                 C.c_void_p(grams[n].data_ptr()), sp))
        coll.all_reduce(grams[n])

    maxper = max(per for (_, _, per) in shard)
    M = torch.empty((G * maxper, R), **f64)
    Ms = torch.empty((maxper, R), **f64)
    As = torch.empty((maxper, R), **f64)
    hist: list[float] = []
    prev = 0.0
    ev = []
    mt_ev = []
    for it in range(opts.max_iters):
        if timing:
            ev.append((torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)))
            ev[-1][0].record()
        for n in range(N):
            lo, rows, per = shard[n]
            Mn, Msn, Asn = M[: G * per], Ms[:per], As[:per]
            Mn.zero_()
            if timing:
                mt_ev.append((torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)))
                mt_ev[-1][0].record()
            t.mttkrp_device(fptr, R, n, Mn.data_ptr(), opts.strategy, config, accumulate=True, stream=stream)
            if timing:
                mt_ev[-1][1].record()
            coll.reduce_scatter(Msn, Mn)
            last = n == N - 1
            _check(lib.blco_als_solve(C.c_void_p(grams.data_ptr()), N, n, R, C.c_void_p(Msn.data_ptr()), rows,
                                      C.c_void_p(Asn.data_ptr()), C.c_void_p(gpart.data_ptr()),
                                      C.c_void_p(status.data_ptr()), sp))
            coll.all_reduce(gpart)
            _check(lib.blco_als_normalize(C.c_void_p(gpart.data_ptr()), R, C.c_void_p(Asn.data_ptr()), rows,
                                          C.c_void_p(grams[n].data_ptr()), C.c_void_p(dlam.data_ptr()),
                                          C.c_void_p(Msn.data_ptr()) if last else None,
                                          C.c_void_p(scal.data_ptr() + 8), sp))
            if rows < per:
                Asn[rows:].zero_()  # padding rows stay zero in the gathered factor
            coll.all_gather(A[n], Asn)
        coll.all_reduce(scal[1:2])
        _check(lib.blco_als_fit(C.c_void_p(grams.data_ptr()), N, R, C.c_void_p(dlam.data_ptr()),
                                C.c_void_p(scal.data_ptr() + 8), xn, C.c_void_p(scal.data_ptr() + 16), sp))
        if timing:
            ev[-1][1].record()
        f = float(scal[2].item())  # the iteration's one host round trip
        if int(status.item()):
            raise Error("solve_normal: matrix singular after maximal diagonal shift")  # as blco_cp_als
        hist.append(f)
        if not np.isfinite(f):
            raise CpAlsError(f"cp_als: non-finite fit at iteration {it + 1}", hist)
        if it > 0 and f - prev < opts.tol:
            break
        prev = f
    lam = dlam.cpu().numpy().copy()
    model = DistCpModel([a[:d] for a, d in zip(A, dims)], lam, hist, opts.seed)
    if timing:
        torch.cuda.synchronize()
        model.device_ms = {"iterations": len(ev),
                           "iterations_ms": sum(a.elapsed_time(b) for a, b in ev),
                           "mttkrp_ms": sum(a.elapsed_time(b) for a, b in mt_ev)}
    return model

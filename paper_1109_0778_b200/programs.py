"""Iteration drivers: the executor-side loop around one staged iteration body.

The reference can only stage iterations by unrolling them (10 unrolled k-means iterations
did not finish fusing in 20 minutes), and its DEG serialises the per-iteration
loop kernels through anti-dependences on the mutable centroid vector
(codegen.cpp:551-565).  Here the executor drives the iteration loop itself: the fused
multiloop, the cross-GPU combine of its partial activation record and the scalar update
kernel stay device-resident and can be captured once into a CUDA graph and replayed.
"""
from __future__ import annotations

import os

import torch

from . import _lib
from . import multiloops as ml

# DLX_KMEANS_UNFUSED_UPDATE=1: separate update launch at one rank (A/B timing only)
_UNFUSED = os.environ.get("DLX_KMEANS_UNFUSED_UPDATE") == "1"


class KMeansProgram:
    """One OptiML k-means iteration = fused {argmin collect, k counts, k*d sums} multiloop
    + allReduce of (counts, sums) across ranks + mu = sums / toDouble(counts)."""

    def __init__(self, x: torch.Tensor, k: int, mu0: torch.Tensor, comm=None,
                 method: int = _lib.KMEANS_AUTO, keep_assign: bool = True):
        self.x = x
        self.k = k
        self.comm = comm
        self.method = method
        n, d = x.shape
        dev = x.device
        self.mu = mu0.clone().to(dev)
        self.assign = torch.empty(n, dtype=torch.int32, device=dev) if keep_assign else None
        self.counts = torch.empty(k, dtype=torch.int64, device=dev)
        self.sums = torch.empty((k, d), dtype=torch.float64, device=dev)
        self.graph = None

    def _body(self):
        if self.comm is None and not _UNFUSED:   # one rank: the update rides on the step's combine launch
            ml.kmeans_iteration(self.x, self.mu, self.assign, self.counts, self.sums, method=self.method,
                                want_assign=self.assign is not None)
            return
        ml.kmeans_step(self.x, self.mu, self.assign, self.counts, self.sums, method=self.method,
                       want_assign=self.assign is not None)
        if self.comm is not None and hasattr(self.comm, "kmeans_update_"):
            self.comm.kmeans_update_(self.counts, self.sums, self.mu)   # fused allreduce + update
            return
        if self.comm is not None:
            self.comm.allreduce_many_([self.counts, self.sums])
        ml.kmeans_update(self.counts, self.sums, self.mu)

    def capture(self):
        """Capture one iteration into a CUDA graph (after one eager warm-up iteration has
        set kernel attributes and sized the workspace).  Replays update self.mu in place."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        mu_save = self.mu.clone()
        with torch.cuda.stream(s):
            self._body()
        torch.cuda.current_stream().wait_stream(s)
        self.mu.copy_(mu_save)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._body()
        self.graph = g
        return self

    def step(self):
        if self.graph is not None:
            self.graph.replay()
        else:
            self._body()

    def run(self, iters: int):
        for _ in range(iters):
            self.step()
        return self


class LogRegProgram:
    """Batch gradient descent: theta <- theta - alpha * sum_i (sigmoid(theta.x_i) - y_i) x_i."""

    def __init__(self, x: torch.Tensor, y: torch.Tensor, theta0: torch.Tensor, alpha: float, comm=None):
        self.x, self.y, self.comm, self.alpha = x, y, comm, alpha
        self.theta = theta0.clone().to(x.device)
        self.grad = torch.empty_like(self.theta)
        self.graph = None

    def _body(self):
        ml.logreg_grad(self.x, self.y, self.theta, self.grad)
        if self.comm is not None and hasattr(self.comm, "bgd_step_"):
            self.comm.bgd_step_(self.grad, self.theta, self.alpha)   # fused allreduce + step
            return
        if self.comm is not None:
            self.comm.allreduce_(self.grad)
        ml.axpy_inplace(self.theta, self.grad, self.alpha)

    def capture(self):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        save = self.theta.clone()
        with torch.cuda.stream(s):
            self._body()
        torch.cuda.current_stream().wait_stream(s)
        self.theta.copy_(save)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._body()
        self.graph = g
        return self

    def step(self):
        if self.graph is not None:
            self.graph.replay()
        else:
            self._body()

    def run(self, iters: int):
        for _ in range(iters):
            self.step()
        return self

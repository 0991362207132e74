"""Multi-GPU driver: one process per GPU, one NCCL all-reduce per run.

SURVEY.md 8(e): the estimator shards with no data-path exchange.  The work is
the grid of cells (replicate, Sobol' index block of 4096 points), numbered
replicate-major; each rank owns a contiguous range of cells -- a range of
Sobol' indices within a range of replicates -- runs the fused path kernel over
them, reduces the replicates it touches to per-replicate partial sums on the
device, and a single all_reduce(SUM) over NCCL (NVLink 5 / NVSwitch) combines the
[L][stride] replicate-sum table ("a few dozen partial sums" per replicate).
When the world size divides L (the weak-scaling bench: 64 replicates per GPU)
the cell ranges are whole replicates, every row is nonzero on exactly one rank,
the sum is exact (x + 0 = x) and the result is bit-identical to one GPU; a
replicate split between two ranks is the sum of their two partial sums
(deterministic for a given world size).  torch is used only for device memory,
streams and the process group; all arithmetic runs in libqmccpw.so.
"""
import ctypes

import numpy as np

from . import (Params, qmccpw_cell_count, qmccpw_finalize, qmccpw_partials, qmccpw_replicate_sums)


def replicate_range(n_replicates, world, rank):
    """Contiguous replicate block of `rank` (balanced to within one replicate)."""
    return n_replicates * rank // world, n_replicates * (rank + 1) // world


def cell_range(n_cells, cells_per_rep, world, rank):
    """Contiguous cell block of `rank` and the replicates it touches: cells are balanced to
    within one cell; when `world` divides the replicate count the blocks are whole replicates
    (the same partition as replicate_range)."""
    n_reps = n_cells // cells_per_rep
    if n_reps % world == 0:
        rb, re = replicate_range(n_reps, world, rank)
        return rb * cells_per_rep, re * cells_per_rep, rb, re
    cb, ce = n_cells * rank // world, n_cells * (rank + 1) // world
    return cb, ce, cb // cells_per_rep, (ce + cells_per_rep - 1) // cells_per_rep


class DistributedPricer:
    """Prices `options` on n_points x n_replicates QMC paths across the ranks of `group`.

    cfg.stream is set to the current torch stream of `device`.
    """

    def __init__(self, options, plist, n_points, n_replicates, cfg, device, rank=0, world=1, group=None):
        import torch
        self.torch = torch
        self.options = list(options)
        self.plist = [Params(p.S0, p.K, p.r, p.sigma, p.T, p.d) for p in plist]
        self.n_points, self.n_replicates = n_points, n_replicates
        self.rank, self.world, self.group = rank, world, group
        self.device = torch.device(device)
        self.cfg = cfg
        self.cfg.device = self.device.index
        self.n_cells, self.per = qmccpw_cell_count(self.plist[0], len(self.options), n_points, n_replicates, cfg)
        self.cells_per_rep = self.n_cells // n_replicates
        self.cell_begin, self.cell_end, self.rep_begin, self.rep_end = cell_range(self.n_cells, self.cells_per_rep,
                                                                                  world, rank)
        self.partials = torch.zeros(self.n_cells * self.per, dtype=torch.float64, device=self.device)
        # cells of my boundary replicates that other ranks own stay zero (set once here: the
        # path kernel only ever writes my cell rows)
        self.rep_sums = torch.zeros(n_replicates * self.per, dtype=torch.float64, device=self.device)
        self.h_rep_sums = torch.empty(n_replicates * self.per, dtype=torch.float64, pin_memory=True)
        self.d2h_bytes = self.h_rep_sums.numel() * 8
        self.h2d_bytes = ctypes.sizeof(Params) * len(self.options) + ctypes.sizeof(type(cfg))
        self.kernel_events = None

    def enqueue_device_work(self, kernel_events=None):
        """Zero the table, run my cells, reduce my replicates (all on the current stream)."""
        torch = self.torch
        stream = torch.cuda.current_stream(self.device)
        self.cfg.stream = ctypes.c_void_p(stream.cuda_stream)
        self.rep_sums.zero_()
        if kernel_events is not None:
            kernel_events[0].record(stream)
        qmccpw_partials(self.options, self.plist, self.n_points, self.n_replicates, self.cfg, self.cell_begin,
                        self.cell_end, self.partials.data_ptr())
        if kernel_events is not None:
            kernel_events[1].record(stream)
        qmccpw_replicate_sums(self.partials.data_ptr(), self.plist[0], len(self.options), self.n_points,
                              self.n_replicates, self.cfg, self.rep_begin, self.rep_end, self.rep_sums.data_ptr())

    def all_reduce(self):
        if self.world > 1:
            self.torch.distributed.all_reduce(self.rep_sums, group=self.group)

    def enqueue_fetch(self):
        """Device->host copy of the (all-reduced) replicate sums, on the current stream."""
        self.h_rep_sums.copy_(self.rep_sums, non_blocking=True)

    def finalize(self):
        """Host finalize of the fetched table (call after the stream has synchronised)."""
        return qmccpw_finalize(self.h_rep_sums.numpy(), self.options, self.plist, self.n_points, self.n_replicates,
                               self.cfg)

    def fetch_and_finalize(self):
        self.enqueue_fetch()
        self.torch.cuda.current_stream(self.device).synchronize()
        return self.finalize()

    def points_owned(self):
        """Sobol' points (paths) this rank's cells hold: full cells of 4096 points, the last
        cell of each replicate ragged when 4096 does not divide n_points."""
        from . import CELL_POINTS
        total = 0
        for c in range(self.cell_begin, self.cell_end):
            j = c % self.cells_per_rep
            total += min(CELL_POINTS, self.n_points - j * CELL_POINTS)
        return total

    def step(self, kernel_events=None):
        """One full run: device work, one all-reduce, device->host read, finalize."""
        self.enqueue_device_work(kernel_events)
        self.all_reduce()
        return self.fetch_and_finalize()


def finalize_from_rank_sums(rank_tables, options, plist, n_points, n_replicates, cfg=None):
    """Host-side combination used by the CPU (gloo) tests: sum per-rank tables
    in rank order and finalize (the all-reduce's arithmetic)."""
    total = np.zeros_like(np.asarray(rank_tables[0], np.float64))
    for t in rank_tables:
        total = total + np.asarray(t, np.float64)
    return qmccpw_finalize(total, options, plist, n_points, n_replicates, cfg)

"""Multi-GPU driver: one process per GPU, one NCCL all-reduce per run.

SURVEY.md 8(e): the estimator shards with no data-path exchange -- each rank
owns a contiguous range of replicates (every cell of a replicate, i.e. all of
its Sobol' index blocks), runs the fused path kernel over its cells, reduces
its own replicates to per-replicate sums on the device, and a single
all_reduce(SUM) over NCCL (NVLink 5 / NVSwitch) combines the [L][stride]
replicate-sum table.  Every row is nonzero on exactly one rank, so the sum is
exact (x + 0 = x) and the result is bit-identical to a single-GPU run of the
same workload.  torch is used only for device memory, streams and the process
group; all arithmetic runs in libqmccpw.so.
"""
import ctypes

import numpy as np

from . import (Params, qmccpw_cell_count, qmccpw_finalize, qmccpw_partials, qmccpw_replicate_sums)


def replicate_range(n_replicates, world, rank):
    """Contiguous replicate block of `rank` (balanced to within one replicate)."""
    return n_replicates * rank // world, n_replicates * (rank + 1) // world


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
        self.rep_begin, self.rep_end = replicate_range(n_replicates, world, rank)
        self.cell_begin = self.rep_begin * self.cells_per_rep
        self.cell_end = self.rep_end * self.cells_per_rep
        self.partials = torch.empty(self.n_cells * self.per, dtype=torch.float64, device=self.device)
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

    def fetch_and_finalize(self):
        self.h_rep_sums.copy_(self.rep_sums, non_blocking=True)
        self.torch.cuda.current_stream(self.device).synchronize()
        return qmccpw_finalize(self.h_rep_sums.numpy(), self.options, self.plist, self.n_points, self.n_replicates,
                               self.cfg)

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

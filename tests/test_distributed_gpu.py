"""Two DistributedPricer ranks on one GPU: the class bench.py
times for N > 1, run end to end -- qmccpw_partials over each rank's cell range,
qmccpw_replicate_sums on the device, one all_reduce over the process group,
the device->host read and qmccpw_finalize.

The process group is gloo (both ranks share cuda:0, and NCCL does not run two
ranks on one device); the all-reduced table is a CUDA tensor, as under NCCL.
The ranks' kernels never wait on one another: the only exchange is the host
all-reduce after each rank's kernels have finished.

  * world divides L: every replicate row is nonzero on exactly one rank, so the
    result is BIT-IDENTICAL to one process pricing the same input through
    qmccpw_price_greeks_batch;
  * world does not divide L: one replicate is split between the two ranks, and
    its sums are the sum of two partial sums -- equal to the single-process
    result to rounding.
"""
import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = {
    # name: (options, strikes, d, construction, conditioning, N, L)
    "bb_w1_whole_replicates": ([0, 1, 2], [100.0] * 3, 64, 1, 0, 3 * 4096 + 555, 4),
    "bb_w1_split_replicate": ([0, 1, 2], [100.0] * 3, 64, 1, 0, 3 * 4096 + 555, 3),
    "pca_x1_split_replicate": ([0, 1], [95.0, 105.0], 64, 2, 1, 2 * 4096 + 7, 5),
    "portfolio_whole_replicates": ([0, 1, 2, 0, 1], [80.0, 90.0, 100.0, 110.0, 120.0], 16, 2, 0, 4096 + 99, 2),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _arrays(res):
    return np.array([[r.mean[:], r.se[:], r.sigma_run[:], r.within_var[:]] for r in res]), \
        np.array([[r.n_points, r.newton_unconverged, r.argmax_near_ties] for r in res])


def _worker(rank, world, port, outdir, name):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    import paper_2209_11337_b200 as q
    from paper_2209_11337_b200.distributed import DistributedPricer
    opts, Ks, d, constr, cond, N, L = CASES[name]
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    plist = [q.params(K=K, d=d) for K in Ks]
    pr = DistributedPricer(opts, plist, N, L, q.config(construction=constr, conditioning=cond, device=0),
                           torch.device("cuda", 0), rank, world)
    res = pr.step()
    vals, cnts = _arrays(res)
    np.save(os.path.join(outdir, f"vals{rank}.npy"), vals)
    np.save(os.path.join(outdir, f"cnts{rank}.npy"), cnts)
    np.save(os.path.join(outdir, f"own{rank}.npy"), np.array([pr.cell_begin, pr.cell_end, pr.points_owned()]))
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def q():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2209_11337_b200 as q
    q.lib()
    return q


@pytest.mark.parametrize("name", list(CASES))
def test_two_ranks_match_one_process(q, name):
    import torch.multiprocessing as mp
    opts, Ks, d, constr, cond, N, L = CASES[name]
    ref = q.qmccpw_price_greeks_batch(opts, [q.params(K=K, d=d) for K in Ks], N, L,
                                      q.config(construction=constr, conditioning=cond, device=0))
    rv, rc = _arrays(ref)
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(2, _free_port(), tmp, name), nprocs=2, join=True)
        v = [np.load(os.path.join(tmp, f"vals{r}.npy")) for r in (0, 1)]
        c = [np.load(os.path.join(tmp, f"cnts{r}.npy")) for r in (0, 1)]
        own = [np.load(os.path.join(tmp, f"own{r}.npy")) for r in (0, 1)]
    # the two ranks hold the same all-reduced table and finalize it identically
    assert np.array_equal(v[0], v[1]) and np.array_equal(c[0], c[1])
    assert np.array_equal(c[0], rc)                         # counters (points, Newton, ties) exact
    # the ranks' cells tile the grid and their points add up to N x L
    assert own[0][0] == 0 and own[0][1] == own[1][0] and own[0][2] + own[1][2] == N * L
    if L % 2 == 0:
        assert np.array_equal(v[0], rv), np.abs(v[0] - rv).max()
    else:
        mean, se = v[0][:, 0], v[0][:, 1]
        scale = np.sqrt(np.maximum(rv[:, 3], 0) + rv[:, 0] ** 2)
        assert np.all(np.abs(mean - rv[:, 0]) <= 1e-13 * scale)
        assert np.all(np.abs(se - rv[:, 1]) <= 1e-9 * rv[:, 1] + 1e-13 * scale)
        assert own[0][1] % ((N + 4095) // 4096) != 0           # a replicate really was split

"""CPU (gloo) tests of the multi-GPU host logic:

  * replicate partition: contiguous, disjoint, complete, balanced for G = 1..8;
  * world size 2 over gloo: each rank fills only its replicate rows of the
    [L][stride] replicate-sum table, one all_reduce(SUM), host finalize ->
    bit-identical to a single process finalising the full table (every row is
    nonzero on exactly one rank, so the sum is exact);
  * fault detection: a missing rank leaves short point counters and finalize
    refuses the table (QMCCPW_EINVAL) instead of returning biased Greeks.

No GPU is used: the per-replicate sums are synthetic, seeded tables with the
layout the kernels write (8 n_opt sums + 3 counters per row).
"""
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N_POINTS, N_REPS, N_OPT = 1 << 12, 13, 3


def _table(n_reps=N_REPS, n_opt=N_OPT, seed=7):
    rng = np.random.default_rng(seed)
    per = 8 * n_opt + 3
    t = np.zeros((n_reps, per))
    for l in range(n_reps):
        for o in range(n_opt):
            for q in range(4):
                s1 = rng.normal() * 50.0
                t[l, o * 8 + q * 2] = s1
                t[l, o * 8 + q * 2 + 1] = s1 * s1 / N_POINTS + abs(rng.normal()) * N_POINTS
        t[l, n_opt * 8 + 2] = N_POINTS
    return t


def _plist(q):
    return [q.params(d=64) for _ in range(N_OPT)]


def test_replicate_partition():
    from paper_2209_11337_b200.distributed import replicate_range
    for L in (1, 5, 64, 512, 1000):
        for G in range(1, 9):
            rs = [replicate_range(L, G, g) for g in range(G)]
            assert rs[0][0] == 0 and rs[-1][1] == L
            assert all(rs[g][1] == rs[g + 1][0] for g in range(G - 1))
            sizes = [e - b for b, e in rs]
            assert max(sizes) - min(sizes) <= 1


def test_cell_partition_covers_the_grid_and_keeps_whole_replicates_when_it_can():
    from paper_2209_11337_b200.distributed import cell_range
    for L, cpr in ((64, 256), (13, 4), (3, 5), (1, 7), (8, 1)):
        n = L * cpr
        for G in range(1, 9):
            parts = [cell_range(n, cpr, G, g) for g in range(G)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[g][1] == parts[g + 1][0] for g in range(G - 1))       # contiguous, disjoint
            sizes = [ce - cb for cb, ce, _, _ in parts]
            for cb, ce, rb, re in parts:
                assert rb * cpr <= cb and ce <= re * cpr                          # replicates touched
                if ce > cb:
                    assert rb == cb // cpr and re == (ce - 1) // cpr + 1
            if L % G == 0:
                assert all(cb % cpr == 0 and ce % cpr == 0 for cb, ce, _, _ in parts)
            else:
                assert max(sizes) - min(sizes) <= 1


def test_split_replicates_sum_to_the_single_process_table():
    # synthetic per-cell partial rows; each rank sums the rows of its cells per replicate
    # (other ranks' rows are zero in its buffer) and the all-reduce adds the rank tables
    from paper_2209_11337_b200.distributed import cell_range
    rng = np.random.default_rng(3)
    L, cpr, per = 5, 7, 11
    cells = rng.normal(size=(L * cpr, per))
    ref = cells.reshape(L, cpr, per).sum(axis=1)
    for G in (2, 3, 4):
        total = np.zeros((L, per))
        for g in range(G):
            cb, ce, _, _ = cell_range(L * cpr, cpr, G, g)
            mine = np.zeros_like(cells)
            mine[cb:ce] = cells[cb:ce]
            total += mine.reshape(L, cpr, per).sum(axis=1)
        assert np.allclose(total, ref, rtol=1e-14, atol=1e-14)


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import paper_2209_11337_b200 as q
    from paper_2209_11337_b200.distributed import replicate_range
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = _table()
    b, e = replicate_range(N_REPS, world, rank)
    mine = np.zeros_like(full)
    mine[b:e] = full[b:e]                     # this rank's replicate rows only
    t = torch.from_numpy(mine)
    dist.all_reduce(t)                        # the one exchange step
    res = q.qmccpw_finalize(t.numpy(), [0, 1, 2], _plist(q), N_POINTS, N_REPS, q.config())
    np.save(os.path.join(outdir, f"rank{rank}.npy"),
            np.array([[r.mean[:], r.se[:], r.sigma_run[:], r.within_var[:]] for r in res]))
    np.save(os.path.join(outdir, f"table{rank}.npy"), t.numpy())
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_world2_allreduce_is_exact_and_matches_single_process():
    import torch.multiprocessing as mp
    import paper_2209_11337_b200 as q
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        full = _table()
        ref = q.qmccpw_finalize(full, [0, 1, 2], _plist(q), N_POINTS, N_REPS, q.config())
        ref = np.array([[r.mean[:], r.se[:], r.sigma_run[:], r.within_var[:]] for r in ref])
        for rank in (0, 1):
            assert np.array_equal(np.load(os.path.join(d, f"table{rank}.npy")), full)
            assert np.array_equal(np.load(os.path.join(d, f"rank{rank}.npy")), ref)


def test_finalize_refuses_a_missing_rank():
    import paper_2209_11337_b200 as q
    from paper_2209_11337_b200.distributed import replicate_range
    full = _table()
    b, e = replicate_range(N_REPS, 4, 2)
    partial = full.copy()
    partial[b:e] = 0.0                        # rank 2 of 4 never contributed
    with pytest.raises(q.QmcCpwError) as err:
        q.qmccpw_finalize(partial, [0, 1, 2], _plist(q), N_POINTS, N_REPS, q.config())
    assert err.value.code == q.EINVAL and "incomplete" in str(err.value)


def test_finalize_matches_the_paper_statistics():
    # C_l = p + S1_l/N, C = mean_l C_l, sigma = sqrt(mean (C_l - C)^2):
    # shift-invariance in the pivot means C - mean_l(S1_l/N) is the same for every replicate split
    import paper_2209_11337_b200 as q
    full = _table()
    r = q.qmccpw_finalize(full, [0, 1, 2], _plist(q), N_POINTS, N_REPS, q.config())
    for o in range(N_OPT):
        for qq in range(4):
            Cl = full[:, o * 8 + qq * 2] / N_POINTS
            sig = np.sqrt(np.mean((Cl - Cl.mean()) ** 2))
            assert abs(r[o].sigma_run[qq] - sig) <= 1e-12 * sig
            assert abs(r[o].se[qq] - sig * np.sqrt(N_REPS / (N_REPS - 1)) / np.sqrt(N_REPS)) <= 1e-12 * sig


def test_bench_reference_arm_runs_on_cpu():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    import json
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_bench_refuses_more_gpus_than_visible():
    # `bench.py --gpus 2` without torchrun spawns 2 ranks itself -- and fails loudly when the
    # box has fewer GPUs, instead of pricing on one and printing n_gpus: 1
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode != 0 and "needs 2 visible CUDA devices" in out.stderr
    assert not [l for l in out.stdout.splitlines() if l.startswith("{")]


def test_bench_refuses_a_world_size_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode != 0 and "world size 1 != --gpus 4" in out.stderr


def test_bench_work_model_follows_survey_8d():
    # SURVEY.md 8(d)'s planning table: the FP64 lane-instruction counts per path that the
    # roofline's `achieved` is computed from (one threshold solve per strike group under X1)
    sys.path.insert(0, ROOT)
    import bench
    C4 = [0, 1, 2]
    assert bench.fp64_model_per_path(64, 1, 0, C4, [100.0] * 3) == 5280                 # BB-W1, the headline
    assert bench.fp64_model_per_path(64, 0, 0, C4, [100.0] * 3) == 5166                 # STD-W1 (~5.2k)
    assert bench.fp64_model_per_path(64, 2, 0, C4, [100.0] * 3) == 9248                 # PCA-W1 (~9.2k)
    assert bench.fp64_model_per_path(64, 2, 1, [0, 1], [100.0] * 2) == 14158            # PCA-X1 (~14.2k)
    assert bench.fp64_model_per_path(128, 2, 0, [0], [100.0]) == 25888                  # PCA-W1 d=128 (~25.9k)
    # two strikes under X1 -> two solves; same strike -> one
    two = bench.fp64_model_per_path(64, 2, 1, [0, 1], [95.0, 105.0])
    assert two - 14158 == 4 * 64 * 20
    # STD-X1: closed-form threshold and a one-line envelope, no pass charged beyond the path's own
    assert bench.fp64_model_per_path(64, 0, 1, C4, [100.0] * 3) == 63 * 50 + 64 * 24 + 3 * 160
    # a lookback under PCA-X1 adds one envelope pass
    assert bench.fp64_model_per_path(64, 2, 1, C4, [100.0] * 3) - 14158 == 64 * 20 + 160

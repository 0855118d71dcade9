"""One process per rank-group over CUDA IPC, on the real device.

Two processes share cuda:0 (CUDA IPC works between processes on one GPU), each
hosting two of four logical ranks; gets, fused remote accumulates and the
replica reduction cross the process boundary through IPC-mapped symmetric
heap chunks.  Results must equal the exact integer product."""

import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CASES = [
    # m, n, k, a_part, b_part, c_part, c_a, c_b, c_c, stationarity
    (96, 80, 64, "2d", "col", "row", 1, 1, 1, "c"),
    (96, 80, 64, "2d", "2d", "2d", 2, 2, 2, "c"),
    (64, 96, 72, "row", "col", "2d", 1, 1, 1, "a"),
    (64, 96, 72, "2d", "row", "col", 1, 1, 1, "b"),
    (48, 40, 64, "col", "row", "2d", 1, 1, 4, "c"),
    (37, 29, 41, "misaligned", "2d", "misaligned", 1, 1, 1, "c"),
]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import numpy as np
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    results = []
    try:
        from paper_2510_08874_b200 import ExecConfig, Stationarity, execute_multiply
        from paper_2510_08874_b200.cli import build_problem

        for case in CASES:
            m, n, k, ap, bp, cp, ca, cb, cc, st = case
            fab, A, B, C, a, b = build_problem(m, n, k, 4, ap, bp, cp, ca, cb, cc, seed=7, devices=[0])
            assert fab.world.size == 2 and fab.local_ranks() == [rank, rank + 2]
            execute_multiply(A, B, C, ExecConfig(stationarity=Stationarity(st)))
            got = C.gather(0)
            results.append((case, bool(np.array_equal(got, a @ b))))
        q.put((rank, results, None))
    except Exception as e:  # noqa: BLE001
        import traceback

        q.put((rank, results, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_processes_share_one_gpu_over_ipc(cuda):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=500) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, results, err in out:
        assert err is None, err
        assert len(results) == len(CASES)
        for case, ok in results:
            assert ok, (rank, case)


def _fullsize_worker(rank, world, port, q):
    import numpy as np
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    try:
        from oracle import um_oracle as O
        from paper_2510_08874_b200 import ExecConfig, execute_multiply
        from paper_2510_08874_b200.cli import build_problem

        seed = 91
        for name, (m, n, k, ap, bp, cp, ca, cb, cc) in FULL.items():
            fab, A, B, C, _, _ = build_problem(m, n, k, 8, ap, bp, cp, ca, cb, cc, seed=seed, synthetic=True,
                                               devices=[0])
            execute_multiply(A, B, C, ExecConfig())
            torch.cuda.synchronize()
            rng = np.random.default_rng(len(name) * 31 + m)
            rows = sorted(set(rng.integers(0, m, 20).tolist()) | {0, m - 1})
            cols = sorted(set(rng.integers(0, n, 20).tolist()) | {0, n - 1})
            got = torch.zeros(len(rows), len(cols), dtype=torch.float64)
            total = torch.zeros(1, dtype=torch.float64)
            for (rep, t), seg in C._segments.items():          # this process's replica-0 tiles only
                if rep != 0 or seg.storage is None:
                    continue
                b = C.tile_bounds(t)
                v = seg.view2d().double()
                total += v.sum().cpu()
                for i, r in enumerate(rows):
                    for j, c in enumerate(cols):
                        if b.rows.lo <= r < b.rows.hi and b.cols.lo <= c < b.cols.hi:
                            got[i, j] = v[r - b.rows.lo, c - b.cols.lo].item()
            # checksum of checksums: sum C = (column sums of A) . (row sums of B)
            acol = torch.zeros(k, dtype=torch.float64)
            brow = torch.zeros(k, dtype=torch.float64)
            for M, vec, axis in ((A, acol, 0), (B, brow, 1)):
                for (rep, t), seg in M._segments.items():
                    if rep != 0 or seg.storage is None:
                        continue
                    b = M.tile_bounds(t)
                    rng_ = b.cols if axis == 0 else b.rows
                    vec[rng_.lo:rng_.hi] += seg.view2d().double().sum(axis).cpu()
            for x in (got, total, acol, brow):
                dist.all_reduce(x)
            expect = float(torch.dot(acol, brow).item())
            a_rows = np.concatenate([O.fill_values(seed, r, r + 1, 0, k, "int") for r in rows]).astype(np.float64)
            b_cols = np.concatenate([O.fill_values(seed + 1, 0, k, c, c + 1, "int") for c in cols], axis=1)
            ok = bool(np.array_equal(got.numpy(), a_rows @ b_cols.astype(np.float64)))
            out.append((name, ok and float(total.item()) == expect, float(total.item())))
            del fab, A, B, C
            torch.cuda.empty_cache()
        q.put((rank, out, None))
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, out, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


FULL = {
    # BASELINE shapes at p=8 logical ranks, 4 per process: pulls and fused remote
    # updates cross the process boundary through IPC-mapped heap chunks
    "cfg5": (16384, 16384, 16384, "2d", "col", "row", 1, 1, 1),
    "cfg4": (16384, 16384, 16384, "2d", "2d", "2d", 2, 2, 2),
}


@pytest.mark.timeout(900)
def test_two_processes_fullsize_sampled_exact(cuda):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_fullsize_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=800) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, results, err in out:
        assert err is None, err
        assert [r[0] for r in results] == list(FULL)
        for name, ok, _ in results:
            assert ok, (rank, name)
    assert [r[2] for r in out[0][1]] == [r[2] for r in out[1][1]]

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

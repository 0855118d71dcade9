"""Fabric / DistributedMatrix one-sided primitives on the GPU (ports of the
reference's test_fabric.py and test_distmatrix.py contracts)."""

import threading

import numpy as np
import pytest
import torch

from paper_2510_08874_b200 import AccumulateMode, DistributedMatrix, Fabric
from paper_2510_08874_b200.errors import ConfigError, ContractError, OwnershipError
from paper_2510_08874_b200.fabric import ELEM_BYTES
from paper_2510_08874_b200.tiling import Bounds2D, PartitionSpec, Range, Shape2D, TileIdx, row_block

pytestmark = pytest.mark.gpu


def fill(r, c):
    return 10.0 * r + c


def mk(fab, name, shape, part, c=1, dense=None, dtype=None):
    init = None if dense is None else (lambda r, cc: dense[r, cc])
    return DistributedMatrix(fab, name, Shape2D(*shape), part, c, init, dtype=dtype)


def test_get_snapshot_and_counters(cuda):
    fab = Fabric(2)
    seg = fab.alloc(1, 4)
    seg.data[:] = torch.tensor([1.0, 2.0, 3.0, 4.0])
    buf = fab.get(seg, Range(1, 3), caller=0)
    seg.data[:] = 0.0
    assert buf.tolist() == [2.0, 3.0], "get must copy, not alias"
    assert fab.counters.bytes[0, 1] == 2 * ELEM_BYTES and fab.counters.msgs[0, 1] == 1
    with pytest.raises(IndexError):
        fab.get(seg, Range(2, 6), caller=0)


def test_get_async_single_wait(cuda):
    fab = Fabric(2)
    seg = fab.alloc(1, 2)
    seg.data[:] = torch.tensor([9.0, 10.0])
    pc = fab.get_async(seg, Range(0, 2), caller=0)
    assert fab.outstanding_copies == 1 and not pc.complete
    assert pc.wait().tolist() == [9.0, 10.0]
    assert pc.complete and fab.outstanding_copies == 0
    with pytest.raises(RuntimeError):
        pc.wait()


def test_accumulate_modes_and_payload_checks(cuda):
    fab = Fabric(2)
    seg = fab.alloc(1, 4)
    fab.accumulate(seg, Range(1, 3), np.array([2.0, 3.0]), caller=0)
    fab.accumulate(seg, Range(1, 3), np.array([1.0, 1.0]), caller=0)
    assert seg.data.tolist() == [0.0, 3.0, 4.0, 0.0]
    assert fab.counters.bytes[0, 1] == 4 * ELEM_BYTES and fab.counters.msgs[0, 1] == 2
    fab.accumulate(seg, Range(0, 4), np.ones(4), caller=0, mode=AccumulateMode.LOCK_GET_PUT)
    assert fab.counters.msgs[0, 1] == 4
    with pytest.raises(ContractError):
        fab.accumulate(seg, Range(0, 3), np.zeros(2), caller=0)
    with pytest.raises(ContractError):
        fab.local_view(seg, caller=0)


@pytest.mark.parametrize("mode", list(AccumulateMode))
def test_concurrent_accumulates_are_atomic(cuda, mode):
    nthreads, reps = 8, 50
    fab = Fabric(nthreads)
    seg = fab.alloc(0, 16)
    ones = torch.ones(16, device="cuda")

    def worker(rank):
        for _ in range(reps):
            fab.accumulate(seg, Range(0, 16), ones, caller=rank, mode=mode)

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(nthreads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    torch.cuda.synchronize()
    assert seg.data.tolist() == [float(nthreads * reps)] * 16


def test_matrix_construction_and_placement(cuda):
    fab = Fabric(4)
    with pytest.raises(ConfigError):
        mk(fab, "A", (4, 4), row_block(Shape2D(4, 4), 4), c=3)
    with pytest.raises(ConfigError):
        mk(fab, "A", (4, 4), row_block(Shape2D(4, 4), 4), c=2)
    dense = np.fromfunction(fill, (7, 5))
    M = mk(fab, "A", (7, 5), row_block(Shape2D(7, 5), 4), dense=dense, dtype=torch.float32)
    assert np.array_equal(M.gather(), dense)
    M2 = mk(fab, "A", (4, 4), row_block(Shape2D(4, 4), 2), c=2)
    assert M2.owner_rank(TileIdx(1, 0), 1) == 3 and M2.owned_tiles(3) == [TileIdx(1, 0)]


def test_tile_views_and_ownership(cuda):
    fab = Fabric(2)
    M = mk(fab, "C", (4, 4), row_block(Shape2D(4, 4), 2))
    view = M.tile(TileIdx(0, 0), caller=0)
    view.data[1, 1] = 5.0
    assert M.gather()[1, 1] == 5.0 and fab.counters.comm_bytes() == 0
    with pytest.raises(OwnershipError):
        M.tile(TileIdx(1, 0), caller=0)


def test_get_tile_and_async(cuda):
    fab = Fabric(2)
    dense = np.fromfunction(fill, (4, 4))
    M = mk(fab, "A", (4, 4), row_block(Shape2D(4, 4), 2), dense=dense, dtype=torch.float32)
    assert np.array_equal(M.get_tile(TileIdx(1, 0), caller=0).data.cpu().numpy(), dense[2:4])
    assert fab.counters.bytes[0, 1] == 8 * ELEM_BYTES
    cp = M.get_tile_async(TileIdx(1, 0), caller=0).wait()
    assert np.array_equal(cp.data.cpu().numpy(), dense[2:4]) and fab.outstanding_copies == 0


def test_accumulate_tile_full_and_sub_slice(cuda):
    fab = Fabric(2)
    M = mk(fab, "C", (4, 4), row_block(Shape2D(4, 4), 2))
    M.accumulate_tile(0, TileIdx(1, 0), np.ones((2, 4)), caller=0)
    assert fab.counters.msgs[0, 1] == 1
    vals = np.arange(4, dtype=float).reshape(2, 2)
    M.accumulate_tile(0, TileIdx(1, 0), vals, Bounds2D(Range(0, 2), Range(1, 3)), caller=0)
    exp = np.zeros((4, 4))
    exp[2:4] = 1
    exp[2:4, 1:3] += vals
    assert np.array_equal(M.gather(), exp) and fab.counters.msgs[0, 1] == 3
    with pytest.raises(ContractError):
        M.accumulate_tile(0, TileIdx(0, 0), np.ones((3, 4)), Bounds2D(Range(0, 3), Range(0, 4)), caller=0)
    with pytest.raises(ContractError):
        M.accumulate_tile(0, TileIdx(0, 0), np.ones((1, 4)), Bounds2D(Range(0, 2), Range(0, 4)), caller=0)


@pytest.mark.parametrize("distributed", [True, False])
def test_reduce_and_broadcast_replicas(cuda, distributed):
    fab = Fabric(4)
    M = mk(fab, "C", (4, 4), row_block(Shape2D(4, 4), 2), c=2)
    M.accumulate_tile(0, TileIdx(0, 0), np.full((2, 4), 1.0), caller=0)
    M.accumulate_tile(1, TileIdx(0, 0), np.full((2, 4), 2.0), caller=2)
    M.accumulate_tile(1, TileIdx(1, 0), np.full((2, 4), 3.0), caller=3)
    M.reduce_replicas(0, distributed=distributed)
    assert M.gather(0).tolist() == [[3.0] * 4] * 4
    assert M.gather(1)[0].tolist() == [2.0] * 4, "non-origin replicas keep their partials"
    M.broadcast_replica(0)
    assert np.array_equal(M.gather(1), M.gather(0))
    fab2 = Fabric(2)
    M1 = mk(fab2, "C", (4, 4), row_block(Shape2D(4, 4), 2))
    M1.reduce_replicas(0)
    assert fab2.counters.msgs.sum() == 0

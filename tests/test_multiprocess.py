"""One-process-per-GPU mode, host logic only: world_size 2 over gloo on CPU.

The symmetric heap's SPMD allocation replay must give every process the same
(process, chunk, offset) for every segment, IPC publication must resolve each
remote segment to its owner's address, and rank hosting / planning must agree
across processes.  Device memory is faked by host buffers (test-only); the
production path uses um_device_alloc / CUDA IPC."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class FakeDeviceApi:
    """Host-memory stand-in for CudaDeviceApi (test only)."""

    def __init__(self):
        self.bufs = {}

    def alloc(self, device, nbytes):
        t = torch.zeros(nbytes, dtype=torch.uint8)
        self.bufs[t.data_ptr()] = t
        return t.data_ptr()

    def free(self, device, ptr):
        self.bufs.pop(ptr, None)

    def ipc_handle(self, ptr):
        return ptr.to_bytes(8, "little") + bytes(56)

    def ipc_open(self, handle, device):
        return int.from_bytes(handle[:8], "little")   # "mapped" at the owner's address

    def ipc_close(self, ptr):
        pass

    def tensor(self, ptr, rows, pitch, dtype, device, keepalive):
        for base, buf in self.bufs.items():
            if base <= ptr < base + buf.numel():
                es = torch.empty((), dtype=dtype).element_size()
                off = ptr - base
                return buf[off:off + rows * pitch * es].view(dtype).view(rows, pitch)
        raise AssertionError("pointer outside fake heap")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_08874_b200 import DistributedMatrix, Fabric, Stationarity
        from paper_2510_08874_b200.cli import resolve_partition
        from paper_2510_08874_b200.runtime import ExecConfig, lower_direct
        from paper_2510_08874_b200.tiling import Shape2D

        p = 4
        fab = Fabric(p, devices=[0], device_api=FakeDeviceApi())
        fab.heap.first_chunk = 1 << 16           # force several chunks
        mats = {}
        for name, shape, desc, c in (("A", (96, 64), "2d", 1), ("B", (64, 80), "col", 2), ("C", (96, 80), "row", 2)):
            mats[name] = DistributedMatrix(fab, name, Shape2D(*shape), resolve_partition(desc, Shape2D(*shape), p // c),
                                           c, dtype=torch.bfloat16 if name != "C" else torch.float32)
        fab.heap.exchange()
        seen = {}
        for name, M in mats.items():
            for (rep, t), seg in M._segments.items():
                assert seg.ptr, "segment unresolved after exchange"
                seen[(name, rep, t.i, t.j)] = (seg.owner, seg.ptr, fab.is_local(seg.owner))
        scheds = {r: [(f.mat, f.tile.i, f.tile.j, f.owner, f.r0, f.r1, f.c0, f.c1)
                      for f in lower_direct(mats["A"], mats["B"], mats["C"], ExecConfig(), r).fetches]
                  for r in fab.local_ranks()}
        q.put((rank, fab.local_ranks(), seen, scheds, fab.heap.layout()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_symmetric_heap_and_hosting_two_processes():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        rank, local, seen, scheds, layout = q.get(timeout=100)
        res[rank] = (local, seen, scheds, layout)
    for pr in procs:
        pr.join(timeout=30)
        assert pr.exitcode == 0
    # rank hosting: r -> process r % world
    assert res[0][0] == [0, 2] and res[1][0] == [1, 3]
    # identical chunk sizes everywhere (bases differ only for unmapped)
    sizes = {q: [s for s, _ in chunks] for q, chunks in res[0][3].items()}
    assert sizes == {q: [s for s, _ in chunks] for q, chunks in res[1][3].items()}
    # every segment resolves to the SAME address in both processes (the owner's)
    s0, s1 = res[0][1], res[1][1]
    assert s0.keys() == s1.keys()
    for key in s0:
        owner0, ptr0, local0 = s0[key]
        owner1, ptr1, local1 = s1[key]
        assert owner0 == owner1 and ptr0 == ptr1 and local0 != local1
    # each process planned exactly its own ranks
    assert set(res[0][2]) | set(res[1][2]) == {0, 1, 2, 3}

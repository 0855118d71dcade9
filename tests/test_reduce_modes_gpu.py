"""K4 transports (replicas.reduce_replicas modes, um_reduce_replicas mode
argument): peer stays exact, the capability probe picks the fallback on a
one-GPU box, VMM symmetric memory works as segment storage, and the NVLS
multimem path runs where the device supports multicast."""

import ctypes

import numpy as np
import pytest
import torch

from paper_2510_08874_b200 import ExecConfig, Fabric, _capi, execute_multiply
from paper_2510_08874_b200.cli import build_problem
from paper_2510_08874_b200.errors import ConfigError
from paper_2510_08874_b200.fabric import LinkTable
from paper_2510_08874_b200.replicas import nvls_capable, resolve_reduce_mode

pytestmark = pytest.mark.gpu


def _problem(symmetric="torch", seed=53):
    fab = Fabric(4, LinkTable.uniform(4, 1e9), devices=[0], symmetric=symmetric)
    return build_problem(384, 320, 512, 4, "2d", "col", "2d", 1, 1, 2, seed=seed, fabric=fab)


def test_auto_falls_back_to_peer_on_one_gpu(cuda):
    fab, A, B, C, a, b = _problem()
    assert resolve_reduce_mode(C, "auto") == "peer"
    ok, why = nvls_capable(C)
    assert not ok and ("VMM" in why or "share a device" in why)
    with pytest.raises(ConfigError, match="nvls"):
        resolve_reduce_mode(C, "nvls")
    with pytest.raises(ConfigError, match="nccl"):
        resolve_reduce_mode(C, "nccl")
    for mode in ("auto", "peer"):
        C.zero_()
        execute_multiply(A, B, C, ExecConfig(reduce_mode=mode))
        assert np.array_equal(C.gather(0), a @ b)


def test_vmm_symmetric_segments_exact(cuda):
    """Fabric(symmetric='vmm'): every segment a um_sym_alloc block; replicas on one
    GPU still share a device, so auto resolves to peer (the NVLS probe says why)."""
    fab, A, B, C, a, b = _problem("vmm")
    assert all(getattr(C.segment(t, r), "vmm", None) is not None for t in C.grid.tiles() for r in range(C.c))
    ok, why = nvls_capable(C)
    assert not ok and "share a device" in why
    for overlap in (True, False):
        C.zero_()
        execute_multiply(A, B, C, ExecConfig(overlap_reduce=overlap))
        assert np.array_equal(C.gather(0), a @ b)
    C.zero_()
    execute_multiply(A, B, C, ExecConfig())
    C.reduce_replicas(0, reduce_mode="peer")          # a second reduce adds the partials again
    got = C.gather(0)
    part = C.gather(1)
    assert np.array_equal(got, a @ b + part)


def test_reduce_mode_argument_of_the_c_abi(cuda):
    lib = _capi.load()
    dst = torch.zeros(8, 16, device="cuda")
    src = torch.ones(8, 16, device="cuda")
    dv = _capi.UmView(dst.data_ptr(), 0, 8, 0, 16, 16, _capi.UM_F32, 0)
    sv = (_capi.UmView * 1)(_capi.UmView(src.data_ptr(), 0, 8, 0, 16, 16, _capi.UM_F32, 0))
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert lib.um_reduce_replicas(ctypes.byref(dv), sv, 1, _capi.UM_REDUCE_NCCL, s) == _capi.UM_ECONFIG
    assert lib.um_reduce_replicas(ctypes.byref(dv), sv, 1, 7, s) == _capi.UM_EVALUE
    assert lib.um_reduce_replicas(ctypes.byref(dv), sv, 1, _capi.UM_REDUCE_PEER, s) == 0
    torch.cuda.synchronize()
    assert torch.equal(dst, src)


def test_sym_alloc_roundtrip(cuda):
    lib = _capi.load()
    g = ctypes.c_uint64(0)
    assert lib.um_sym_granularity(0, ctypes.byref(g)) == 0 and g.value >= 4096
    p = ctypes.c_void_p()
    assert lib.um_sym_alloc(0, 3 << 20, ctypes.byref(p)) == 0, _capi.last_error()
    from paper_2510_08874_b200.heap import _wrap_device_ptr

    t = _wrap_device_ptr(p.value, 256, 1024, torch.float32, 0, None)
    t.copy_(torch.arange(256 * 1024, device="cuda", dtype=torch.float32).view(256, 1024))
    torch.cuda.synchronize()
    assert float(t[255, 1023]) == 256 * 1024 - 1
    del t
    assert lib.um_sym_free(p) == 0
    assert lib.um_sym_free(p) != 0          # not a live base any more


def test_nvls_team_of_one_device(cuda):
    """Where multicast is supported: a one-device team, multimem.ld_reduce over
    it returns the member's own values (the sum over a team of one).  Records
    the probe result either way."""
    lib = _capi.load()
    ok = ctypes.c_int32(0)
    assert lib.um_nvls_supported(0, ctypes.byref(ok)) == 0
    print(f"NVLS multicast supported on device 0: {bool(ok.value)}")
    if not ok.value:
        pytest.skip("device 0 does not support multicast objects")
    p = ctypes.c_void_p()
    assert lib.um_sym_alloc(0, 2 << 20, ctypes.byref(p)) == 0, _capi.last_error()
    from paper_2510_08874_b200.heap import _wrap_device_ptr

    rows, cols = 64, 256
    src = _wrap_device_ptr(p.value, rows, cols, torch.float32, 0, None)
    src.copy_(torch.randint(-8, 9, (rows, cols), device="cuda").float())
    torch.cuda.synchronize()
    devs = (ctypes.c_int32 * 1)(0)
    ptrs = (ctypes.c_void_p * 1)(p.value)
    mc = (ctypes.c_void_p * 1)()
    team = ctypes.c_void_p()
    rc = lib.um_nvls_team_create(1, devs, ptrs, 2 << 20, mc, ctypes.byref(team))
    if rc == _capi.UM_ECONFIG:
        pytest.skip(_capi.last_error())
    assert rc == 0, _capi.last_error()
    dst = torch.zeros(rows, cols, device="cuda")
    dv = _capi.UmView(dst.data_ptr(), 0, rows, 0, cols, cols, _capi.UM_F32, 0)
    sv = (_capi.UmView * 1)(_capi.UmView(mc[0], 0, rows, 0, cols, cols, _capi.UM_F32, 0))
    assert lib.um_reduce_replicas(ctypes.byref(dv), sv, 1, _capi.UM_REDUCE_NVLS,
                                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0, _capi.last_error()
    torch.cuda.synchronize()
    assert torch.equal(dst, src)
    assert lib.um_nvls_team_destroy(team) == 0
    del src
    assert lib.um_sym_free(p) == 0

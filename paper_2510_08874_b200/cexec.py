"""A whole multiply driven through the C-ABI whole-multiply entry (um_execute).

`execute_multiply` issues each rank from Python; a non-Python caller of the
library needs the same thing behind C.  `CompiledMultiply` builds every
rank's issue plan once (the same plans execute_multiply replays: planner op
lists, fetch-once staging, prepared K1 launches carrying the in-kernel pulls)
plus the replica-reduction steps, serialises them into `um_rank_plan` /
`um_reduce_step` arrays, and `execute()` is then ONE C call (um_execute) that
issues the whole multiply on library-owned streams; `um_sync_all` is the
host barrier.  Replaces runtime.py:339-387 (execute_multiply's loop over
ranks, the run-level barrier and reduce_replicas) at the C boundary.

Barrier form of the replica reduction (the reference's); single process.
"""

from __future__ import annotations

import ctypes
import dataclasses

import torch

from paper_2510_08874_b200.trace import nvtx
from paper_2510_08874_b200 import _capi
from paper_2510_08874_b200.config import ExecConfig
from paper_2510_08874_b200.engine import _RankRun
from paper_2510_08874_b200.errors import ContractError
from paper_2510_08874_b200.fabric import AccumulateMode
from paper_2510_08874_b200.opgen import Stationarity
from paper_2510_08874_b200.replicas import _nvls_team, resolve_reduce_mode
from paper_2510_08874_b200.schedule import lower_direct, schedule_cache

_STAT = {Stationarity.STATIONARY_A: _capi.UM_STATIONARY_A, Stationarity.STATIONARY_B: _capi.UM_STATIONARY_B,
         Stationarity.STATIONARY_C: _capi.UM_STATIONARY_C}


def exec_cfg(cfg: ExecConfig, reduce_mode: int = _capi.UM_REDUCE_PEER) -> _capi.UmExecCfg:
    """ExecConfig (runtime.py:26-40) -> um_exec_cfg."""
    return _capi.UmExecCfg(_STAT[cfg.stationarity], cfg.prefetch_depth, cfg.max_inflight_gemms,
                           cfg.max_inflight_accums, 0 if cfg.accumulate_mode is AccumulateMode.PEER_ATOMIC else 1,
                           cfg.pool_capacity or 0, reduce_mode, 0)


class CompiledMultiply:
    """C += A @ B serialised for um_execute (same semantics as execute_multiply)."""

    def __init__(self, A, B, C, cfg: ExecConfig | None = None):
        cfg = dataclasses.replace(cfg or ExecConfig(), overlap_reduce=False)
        fab = A.fabric
        if fab.world.size != 1:
            raise ContractError("CompiledMultiply is single-process")
        if not cfg.fused_accumulate:
            raise ContractError("um_execute plans carry fused remote accumulates only (fused_accumulate=True)")
        fab._require_data()
        self.A, self.B, self.C, self.cfg = A, B, C, cfg
        self._keep = [schedule_cache(A, B, C)]        # plans / staging / prepared launches stay alive
        lib = _capi.load()
        plans, self.scheds = [], {}
        for r in fab.local_ranks():
            sched = lower_direct(A, B, C, cfg, r)
            self.scheds[r] = sched
            run = _RankRun(A, B, C, cfg, sched, [])
            plan = run.plan()
            order = {j: q for q, (j, _, _) in enumerate(plan.host_fetches)}
            copies = (_capi.UmGetDesc * max(1, len(plan.host_fetches)))(
                *[_capi.UmGetDesc(src, dst) for _, src, dst in plan.host_fetches])
            acts = []
            for act in plan.actions:
                if act[0] == "launch":
                    acts.append(_capi.UmExecAction(_capi.UM_ACT_LAUNCH, 0, act[1]))
                elif act[0] == "wait":
                    acts.append(_capi.UmExecAction(_capi.UM_ACT_WAIT_COPY, order[act[1]], None))
                else:
                    raise ContractError("unfused remote accumulate has no um_execute action")
            actions = (_capi.UmExecAction * max(1, len(acts)))(*acts)
            self._keep += [plan, copies, actions]
            plans.append(_capi.UmRankPlan(r, fab.device_of(r), len(plan.host_fetches), len(acts),
                                          ctypes.cast(copies, ctypes.POINTER(_capi.UmGetDesc)),
                                          ctypes.cast(actions, ctypes.POINTER(_capi.UmExecAction))))
        self.plans = (_capi.UmRankPlan * max(1, len(plans)))(*plans)
        self.nplans = len(plans)
        steps = []
        mode = resolve_reduce_mode(C, cfg.reduce_mode) if C.c > 1 else "peer"
        if mode == "nccl":
            raise ContractError("reduce_mode='nccl' is a host collective; um_execute runs peer or NVLS steps")
        if C.c > 1:
            for t in C.grid.tiles():                  # distributed barrier-form K4 (replicas.reduce_replicas)
                dst = C.segment(t, 0)
                if dst.length == 0:
                    continue
                srcs = [C.segment(t, r) for r in range(1, C.c)]
                n = C.c if cfg.reduce_distributed else 1
                for j in range(n):
                    r0, r1 = dst.rows * j // n, dst.rows * (j + 1) // n
                    if r1 <= r0:
                        continue
                    red = C.owner_rank(t, j) if cfg.reduce_distributed else dst.owner
                    dev = fab.device_of(red)
                    if mode == "nvls":
                        sv = (_capi.UmView * 1)(_nvls_team(C, t).view(dst, dev, r0, r1))
                        kmode = _capi.UM_REDUCE_NVLS
                    else:
                        sv = (_capi.UmView * len(srcs))(*[s_.um_view(r0, r1, 0, s_.cols) for s_ in srcs])
                        kmode = _capi.UM_REDUCE_PEER
                    self._keep.append(sv)
                    steps.append(_capi.UmReduceStep(dst.um_view(r0, r1, 0, dst.cols),
                                                    ctypes.cast(sv, ctypes.POINTER(_capi.UmView)), len(sv), kmode,
                                                    dev, 0))
        self.steps = (_capi.UmReduceStep * max(1, len(steps)))(*steps)
        self.nsteps = len(steps)
        self.cfg_c = exec_cfg(cfg, _capi.UM_REDUCE_NVLS if mode == "nvls" else _capi.UM_REDUCE_PEER)
        self.devices = sorted({fab.device_of(r) for r in fab.local_ranks()})

    @nvtx("um:um_execute")
    def execute(self, sync: bool = False) -> None:
        """One more C += A @ B: a single um_execute call (ordered after, and
        joined back into, torch's current streams of the devices)."""
        lib = _capi.load()
        for d in self.devices:
            _capi.check(lib.um_execute_after(ctypes.c_void_p(torch.cuda.current_stream(d).cuda_stream), d),
                        "um_execute_after")
        _capi.check(lib.um_execute(self.plans, self.nplans, self.steps, self.nsteps, ctypes.byref(self.cfg_c)),
                    "um_execute")
        for d in self.devices:
            _capi.check(lib.um_execute_wait(ctypes.c_void_p(torch.cuda.current_stream(d).cuda_stream), d),
                        "um_execute_wait")
        if sync:
            _capi.check(lib.um_sync_all(), "um_sync_all")

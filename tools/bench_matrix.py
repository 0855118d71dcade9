"""Every BASELINE configuration at p in {1, 2, 4, 8} logical ranks on ONE GPU.

    python tools/bench_matrix.py [--configs cfg2,cfg3] [--ps 1,2,4,8] [--steps 5] [--json out.json]

All p ranks are co-resident on cuda:0 (rank r -> device r mod 1), each with its
own get / compute / reduce streams, so a step runs the complete multi-rank
path of `execute_multiply`: the C++ planner's op lists, fetch-once K2 pulls of
every remote slice (device-to-device copies here, NVLink on a multi-GPU box),
grouped K1 launches, fused K3 remote accumulates and the K4 replica reduction.
Total work is the global GEMM (2*m*n*k flops), so TFLOP/s here is directly
comparable with the single-rank number: the gap is the engine's overhead
(extra pulls, smaller GEMMs, reductions) on one GPU.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_08874_b200 import ExecConfig, Stationarity, execute_multiply  # noqa: E402
from paper_2510_08874_b200 import engine as eng  # noqa: E402
from paper_2510_08874_b200 import runtime as rt  # noqa: E402
from paper_2510_08874_b200.cli import build_problem  # noqa: E402


def k4_nvlink_model(C, ovl, link_gbs: float = 770.0):
    """K4 over NVLink (model): per reducer, the bytes it reads from other GPUs
    (non-local replicas, and the origin when remote) and writes to the origin
    when remote, at the measured 770 GB/s per direction (full duplex: the
    slower direction counts).  Returns (whole reduction, last sub-slice) in ms
    for the busiest reducer: overlapped with the GEMMs, only the last
    sub-slice's share is exposed."""
    p = C.fabric.nprocs
    rd, wr = [0] * p, [0] * p
    last = [0.0] * p
    for t, subs in ovl.subs.items():
        cols = C.segment(t, 0).cols
        for r0, r1, rep in subs:
            red = C.owner_rank(t, rep)
            nb = (r1 - r0) * cols * 4
            origin_remote = C.owner_rank(t, 0) != red
            reads = sum(1 for r in range(1, C.c) if C.owner_rank(t, r) != red) * nb + (nb if origin_remote else 0)
            writes = nb if origin_remote else 0
            rd[red] += reads
            wr[red] += writes
            last[red] = max(reads, writes)
    whole = max(max(a, b) for a, b in zip(rd, wr))
    return whole / (link_gbs * 1e9) * 1e3, max(last) / (link_gbs * 1e9) * 1e3


def run_one(name, p, steps, warmup, stationarity, extra):
    m, n, k, ap, bp, cp, fa, fb, fc, desc = bench.CONFIGS[name]
    ca, cb, cc = fa(p), fb(p), fc(p)
    fab, A, B, C, _, _ = build_problem(m, n, k, p, ap, bp, cp, ca, cb, cc, seed=0, real=True, synthetic=True,
                                       devices=[0])
    cfg = ExecConfig(stationarity=stationarity, **extra)
    flops = 2.0 * m * n * k
    for _ in range(warmup):
        stats = execute_multiply(A, B, C, cfg)
    torch.cuda.synchronize()
    cap = None
    if os.environ.get("UM_MATRIX_GRAPH") == "1":
        from paper_2510_08874_b200.graphs import CapturedMultiply

        cap = CapturedMultiply(A, B, C, cfg)
        torch.cuda.synchronize()
    eng.TRACE.clear()
    eng.TRACE_ENABLED = cap is None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        stats = cap.replay() if cap is not None else execute_multiply(A, B, C, cfg)
    e1.record()
    torch.cuda.synchronize()
    eng.TRACE_ENABLED = False
    ms = e0.elapsed_time(e1) / steps
    kms = sum(s.elapsed_time(e) for s, e, _ in eng.TRACE) / steps if eng.TRACE else 0.0
    solo = {}
    if p > 1 and os.environ.get("UM_MATRIX_SOLO", "1") == "1":
        # each rank ALONE on the GPU (its pulls read HBM instead of NVLink): the
        # per-rank step time of a p-GPU run is max over ranks of this + the reduction
        from paper_2510_08874_b200 import run_direct
        per, per_k1 = [], []
        for r in range(p):
            run_direct(A, B, C, cfg, r)
            torch.cuda.synchronize()
            eng.TRACE.clear()
            eng.TRACE_ENABLED = True
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(steps):
                run_direct(A, B, C, cfg, r)
            t1.record()
            torch.cuda.synchronize()
            eng.TRACE_ENABLED = False
            per.append(t0.elapsed_time(t1) / steps)
            # device time of the rank's K1 launch(es) alone (no host issue gap)
            per_k1.append(sum(a.elapsed_time(b) for a, b, _ in eng.TRACE) / steps)
        red = 0.0
        if C.c > 1:
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(steps):
                C.reduce_replicas(0)
            t1.record()
            torch.cuda.synchronize()
            red = t0.elapsed_time(t1) / steps
        solo = {"rank_ms": per, "rank_ms_max": max(per), "rank_k1_ms": per_k1, "rank_k1_ms_max": max(per_k1),
                "reduce_ms_all_slices": red,
                "per_gpu_tflops_ranks": [flops / p / (t * 1e-3) / 1e12 for t in per]}
        if C.c > 1:
            # K4 over NVLink (model): bytes each reducer pulls from other GPUs or
            # writes to the origin's GPU, at the measured 770 GB/s peer rate;
            # overlapped, only the last sub-slice's share is exposed
            from paper_2510_08874_b200.replicas import _ReduceOverlap
            ovl = _ReduceOverlap(A, B, C, cfg)
            whole, last = k4_nvlink_model(C, ovl)
            solo["k4_nvlink_ms_model"] = whole
            solo["k4_exposed_ms_model"] = last
        gbps = float(os.environ.get("UM_GET_GBPS", "0") or 0)
        solo["pulls_paced_gbps"] = gbps or None
        t_gpu = max(per_k1) + solo.get("k4_exposed_ms_model", 0.0)
        solo["projected_ms_per_gpu"] = t_gpu
        solo["projected_tflops_per_gpu"] = flops / p / (t_gpu * 1e-3) / 1e12
    out = {"config": name, "p": p, "stationarity": stationarity.value if hasattr(stationarity, "value") else str(stationarity),
           "m": m, "n": n, "k": k, "partitions": [ap, bp, cp], "replication": [ca, cb, cc],
           "ms": ms, "tflops": flops / (ms * 1e-3) / 1e12,
           "k1_ms_sum": kms, "k1_launches": sum(s.launches for s in stats.values()),
           "ops": sum(len(s.executed_ops) for s in stats.values()),
           "gets": sum(s.gets for s in stats.values()),
           "staged_mib": sum(s.staged_bytes for s in stats.values()) / 2**20, "solo": solo}
    del fab, A, B, C
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg1,cfg2,cfg3,cfg4,cfg5")
    ap.add_argument("--ps", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--stationarity", default="c", choices=["a", "b", "c"])
    ap.add_argument("--json", default=None)
    ap.add_argument("--set", action="append", default=[], help="ExecConfig override key=value (int/str)")
    a = ap.parse_args()
    st = {"a": Stationarity.STATIONARY_A, "b": Stationarity.STATIONARY_B, "c": Stationarity.STATIONARY_C}[a.stationarity]
    extra = {}
    for kv in a.set:
        key, val = kv.split("=", 1)
        extra[key] = int(val) if val.lstrip("-").isdigit() else (val == "True" if val in ("True", "False") else val)
    peak, _, _ = bench.load_peaks()
    rows = []
    for name in a.configs.split(","):
        for p in [int(x) for x in a.ps.split(",")]:
            r = run_one(name, p, a.steps, a.warmup, st, extra)
            r["frac_of_peak"] = r["tflops"] / peak
            rows.append(r)
            print(f"{name} p={p} st={a.stationarity} {r['tflops']:8.1f} TFLOP/s ({r['frac_of_peak']:.3f} of peak) "
                  f"{r['ms']:8.3f} ms  K1 {r['k1_ms_sum']:8.3f} ms in {r['k1_launches']} launches, "
                  f"{r['ops']} ops, {r['gets']} gets, {r['staged_mib']:.0f} MiB staged", flush=True)
            if r["solo"]:
                so = r["solo"]
                print(f"    solo ranks: max {so['rank_ms_max']:.3f} ms/rank -> per-GPU "
                      f"{min(so['per_gpu_tflops_ranks']):.0f}..{max(so['per_gpu_tflops_ranks']):.0f} TFLOP/s; "
                      f"K4 reduce (all slices on this GPU) {so['reduce_ms_all_slices']:.3f} ms; projected "
                      f"{so['projected_tflops_per_gpu']:.0f} TFLOP/s per GPU "
                      f"(pulls paced at {so['pulls_paced_gbps']} GB/s, K4 exposed "
                      f"{so.get('k4_exposed_ms_model', 0):.3f} ms)", flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"peak_tflops": peak, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()

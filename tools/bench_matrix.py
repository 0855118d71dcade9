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
        per = []
        for r in range(p):
            run_direct(A, B, C, cfg, r)
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(steps):
                run_direct(A, B, C, cfg, r)
            t1.record()
            torch.cuda.synchronize()
            per.append(t0.elapsed_time(t1) / steps)
        red = 0.0
        if C.c > 1:
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(steps):
                C.reduce_replicas(0)
            t1.record()
            torch.cuda.synchronize()
            red = t0.elapsed_time(t1) / steps
        solo = {"rank_ms": per, "rank_ms_max": max(per), "reduce_ms_all_slices": red,
                "per_gpu_tflops_ranks": [flops / p / (t * 1e-3) / 1e12 for t in per]}
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
                      f"K4 reduce (all slices on this GPU) {so['reduce_ms_all_slices']:.3f} ms", flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"peak_tflops": peak, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()

"""Repeated small multiplies: eager issue vs ExecConfig.graph_replay (one GPU).

    python tools/graph_replay_probe.py [--configs cfg1] [--ps 1,2,4,8] [--steps 50]

All p logical ranks co-resident on cuda:0 (as tools/bench_matrix.py).  For
each case: ms per multiply over `steps` back-to-back execute_multiply calls
(CUDA events on the current stream, after warm-up, which also captures the
graph), once with graph_replay=False and once with the default; plus the host
time per call.  One JSON line per case.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_08874_b200 import ExecConfig, execute_multiply  # noqa: E402
from paper_2510_08874_b200.cli import build_problem  # noqa: E402


def time_calls(A, B, C, cfg, steps):
    for _ in range(4):
        execute_multiply(A, B, C, cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h0 = time.perf_counter()
    for _ in range(steps):
        execute_multiply(A, B, C, cfg)
    h1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, (h1 - h0) * 1e3 / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg1")
    ap.add_argument("--ps", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=50)
    args = ap.parse_args()
    for name in args.configs.split(","):
        m, n, k, apart, bpart, cpart, fa, fb, fc, _ = bench.CONFIGS[name]
        for p in (int(x) for x in args.ps.split(",")):
            fab, A, B, C, _, _ = build_problem(m, n, k, p, apart, bpart, cpart, fa(p), fb(p), fc(p), seed=0,
                                               real=True, synthetic=True, devices=[0])
            out = {"config": name, "p": p, "m": m, "n": n, "k": k}
            for label, cfg in (("eager", ExecConfig(graph_replay=False)), ("graph", ExecConfig())):
                ms, host = time_calls(A, B, C, cfg, args.steps)
                out[label] = {"ms": round(ms, 4), "host_ms_per_call": round(host, 4),
                              "tflops": round(2.0 * m * n * k / (ms * 1e-3) / 1e12, 1)}
            print(json.dumps(out), flush=True)
            del fab, A, B, C
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

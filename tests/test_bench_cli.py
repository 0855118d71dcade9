"""bench.py's multi-GPU plumbing (CPU-only checks): `--gpus N` never silently
runs fewer ranks, and the default workload is the communication-heavy cfg5."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    env["CUDA_VISIBLE_DEVICES"] = ""          # no GPU visible, whatever the host has
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=env, cwd=ROOT,
                          capture_output=True, text=True, timeout=300)


def test_gpus_without_torchrun_refuses_when_gpus_missing():
    out = _run(["--gpus", "2", "--steps", "1", "--warmup", "3", "--no-e2e", "--no-cpu"])
    assert out.returncode != 0
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert "only 0 CUDA device" in line["error"]
    assert "value" not in line


def test_world_size_must_match_gpus():
    out = _run(["--gpus", "1", "--steps", "1"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert out.returncode != 0
    assert "WORLD_SIZE=2" in out.stderr


def test_spawn_command_uses_torchrun(monkeypatch):
    sys.path.insert(0, ROOT)
    import bench

    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--oversubscribe"])

    class Args:
        gpus, oversubscribe = 4, True

    assert bench.spawn_ranks(Args()) == 0
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--oversubscribe"]


def test_default_workload_is_cfg5():
    sys.path.insert(0, ROOT)
    import bench

    src = open(os.path.join(ROOT, "bench.py")).read()
    assert 'add_argument("--config", default="cfg5"' in src
    m, n, k, ap, bp, cp, *_ = bench.CONFIGS["cfg5"]
    assert (m, n, k, ap, bp, cp) == (16384, 16384, 16384, "2d", "col", "row")


def test_pipeline_floor_bounds():
    """The e2e block-pipeline floor (bench.pipeline_floor_ms) sits between the
    PCIe floor and the one-block pipeline, and a square shell grid beats
    uploading B whole first (row panels)."""
    import bench

    G = 1 << 30
    flops = 2 * 16384 ** 3
    pcie = G / 50e9 * 1e3
    grids = {(P, Q): bench.pipeline_floor_ms(P, Q, G // 2, G // 2, G, flops, 50.0, 50.0, 1600.0)
             for P, Q in ((1, 1), (4, 4), (8, 8), (8, 1))}
    for v in grids.values():
        assert v >= 1.25 * pcie - 1e-6          # C blocks need whole A rows and B columns
    assert grids[(1, 1)] >= 2 * pcie - 1e-6     # upload everything, then download everything
    assert grids[(8, 8)] < grids[(4, 4)] < grids[(8, 1)] < grids[(1, 1)]
    # faster one-direction copies only lower the floor
    assert bench.pipeline_floor_ms(4, 4, G // 2, G // 2, G, flops, 50.0, 50.0, 1600.0, 56.0, 57.0) < grids[(4, 4)]

"""Benchmark: distributed GEMM bf16 TFLOP/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl b200|reference]

One step = one full `execute_multiply` (every get, GEMM, remote accumulate and
replica reduction of the configuration) over synthetic operands resident in
HBM.  The default workload is BASELINE configs[4] (cfg5: mismatched A 2D /
B col / C row partitionings, 16384^3), the north-star size whose multi-GPU
runs carry real one-sided traffic (496 MiB of pulls per rank at p=8); at
N=1 it is one rank (p = 1).  `--config cfg2` etc. select the other BASELINE
configurations.

Multi-GPU: one process per GPU, each hosting one logical rank (p = N) of the
same global problem, so total work is fixed ("strong" scaling).  Under
torchrun the ranks come from the environment; `python bench.py --gpus N`
without torchrun re-launches itself under `torch.distributed.run` with N
processes.  Fewer visible GPUs than ranks is an error unless
`--oversubscribe` (several ranks time-sharing a GPU: a functional test, not
a measurement; n_gpus then counts the physical GPUs used).

Printed JSON keys follow the driver contract; `value` is device-timed
(CUDA events, max over ranks), `e2e` repeats the metric through the public
API with pinned host buffers (H2D of A/B and D2H of C inside the timed
region), `roofline` relates the dominant kernel (K1) to the measured bf16
peak, `cpu_baseline` times the CPU oracle port (tests-only code, used here
only as the reference arm) on a bounded sample on this host.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (m, n, k, a_part, b_part, c_part, c_a(p), c_b(p), c_c(p), description)
    "cfg1": (1024, 1024, 1024, "2d", "2d", "2d", lambda p: 1, lambda p: 1, lambda p: 1,
             "2D block A/B/C, m=n=k=1024"),
    "cfg2": (65536, 8192, 8192, "row", "2d", "row", lambda p: 1, lambda p: p, lambda p: 1,
             "1D row-block A and C, B replicated (sequence-parallel), m=65536 n=k=8192"),
    "cfg3": (8192, 8192, 65536, "col", "row", "2d", lambda p: 1, lambda p: 1, lambda p: p,
             "A col / B row outer product, C replicated (Megatron-TP), m=n=8192 k=65536"),
    "cfg4": (16384, 16384, 16384, "2d", "2d", "2d", lambda p: min(2, p), lambda p: min(2, p), lambda p: min(2, p),
             "2.5D: 2D block A/B/C with c=2, 16384^3"),
    "cfg5": (16384, 16384, 16384, "2d", "col", "row", lambda p: 1, lambda p: 1, lambda p: 1,
             "mismatched: A 2D, B col, C row, 16384^3"),
}

METRIC = "distributed GEMM bf16 TFLOP/s at 1/2/4/8 B200 and % of tensor-core peak"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["bf16_tflops"]), float(pk.get("bf16_tflops_sustained", pk["bf16_tflops"])), "measured"
    except Exception:  # noqa: BLE001
        return 1590.0, 1400.0, "fallback"


class ClockSampler:
    """SM clock and clock-event reasons sampled DURING the timed region.

    NVML (nvidia-ml-py) polled every ~2 ms from a thread, so even a 60 ms
    timed region yields tens of loaded samples; falls back to `nvidia-smi -lms`
    when NVML is unavailable."""

    NAMES = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
             ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples: list = []
        self.reasons: set = set()
        self.smax = None
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        self._smi = None

    def _handle(self):
        import pynvml
        import torch

        pynvml.nvmlInit()
        try:
            pr = torch.cuda.get_device_properties(self.dev)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:  # noqa: BLE001
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.dev)

    def start(self):
        try:
            nv, h = self._handle()
            self._nvml = (nv, h)
            self.smax = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))

            def loop():
                while not self._stop.is_set():
                    try:
                        self.samples.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for name, bit in self.NAMES:
                            if r & bit:
                                self.reasons.add(name)
                    except Exception:  # noqa: BLE001
                        pass
                    time.sleep(0.002)

            self._t = threading.Thread(target=loop, daemon=True)
            self._t.start()
        except Exception:  # noqa: BLE001
            self._nvml = None
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            try:
                self._smi = subprocess.Popen(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={q}",
                                              "--format=csv,noheader,nounits", "-lms", "20"],
                                             stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            except Exception:  # noqa: BLE001
                self._smi = None

    def stop(self):
        if self._nvml is not None:
            self._stop.set()
            self._t.join(timeout=2)
        elif self._smi is not None:
            self._smi.terminate()
            out = self._smi.communicate(timeout=5)[0]
            for ln in out.splitlines():
                f = [x.strip() for x in ln.split(",")]
                try:
                    self.samples.append(float(f[0]))
                    self.smax = float(f[1])
                except (ValueError, IndexError):
                    continue
                for (name, _), v in zip(self.NAMES, f[2:6]):
                    if v.lower().startswith("active"):
                        self.reasons.add(name)
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = sorted(self.samples)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": self.smax,
                "reasons": sorted(self.reasons), "samples": len(sm),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def k1_traffic(config: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of the K1 launch of this
    workload from the newest committed `ncu --set full` capture
    (profiles/*_ncu_summary.json, key k1_bench_<config>), labelled with the
    capture's file, git SHA of the kernel build and date — ncu cannot run
    inside the timed bench, so the figure is from a separate capture of the
    same command, not from this run.  None if no capture exists."""
    import glob

    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_summary.json")), reverse=True):
        try:
            with open(path) as f:
                prof = json.load(f)
        except Exception:  # noqa: BLE001
            continue
        e = prof.get(f"k1_bench_{config}")
        if e is not None:
            return {"bytes_per_launch": e["dram_bytes_per_launch"],
                    "source": f"profiles/{os.path.basename(path)}:k1_bench_{config}",
                    "captured": {k: e.get(k) for k in ("git_sha", "date", "command") if k in e} or "round-1 build"}
    return None


def free_port() -> int:
    import socket

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        return s_.getsockname()[1]


def spawn_ranks(args) -> int:
    """`--gpus N` without torchrun: re-launch this script as N ranks (one process
    per GPU) under torch.distributed.run; refuse when fewer GPUs are visible."""
    import torch

    ndev = torch.cuda.device_count()
    if ndev < args.gpus and not args.oversubscribe:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but only {ndev} CUDA device(s) visible "
                                                     f"(pass --oversubscribe to time-share GPUs)"}), flush=True)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def blas_threads(n: int):
    """Use all n host threads in BLAS even under torchrun (which sets OMP_NUM_THREADS=1)."""
    from threadpoolctl import threadpool_limits

    return threadpool_limits(limits=n, user_api="blas")


def cpu_oracle_rate(m, n, k, p, desc, target_s: float):
    """Time the CPU oracle port (numpy fp64, all host threads) on a row sample.

    Returns (tflops, sample description, cores, seconds)."""
    import numpy as np

    from oracle import um_oracle as O

    cores = len(os.sched_getaffinity(0))
    rng = np.random.default_rng(0)

    def run(rows):
        a = rng.uniform(-1, 1, size=(rows, k))
        b = rng.uniform(-1, 1, size=(k, n))
        mats = [O.Mat("A", rows, k, O.Spec(rows, k, 1, 1), 1, 1), O.Mat("B", k, n, O.Spec(k, n, 1, 1), 1, 1),
                O.Mat("C", rows, n, O.Spec(rows, n, 1, 1), 1, 1)]
        t0 = time.perf_counter()
        O.execute("c", *mats, a, b)
        return time.perf_counter() - t0

    with blas_threads(cores):
        run(64)                                   # BLAS thread-pool warm-up
        rows = 256
        dt = run(rows)
        rows = int(min(m, max(64, rows * target_s / max(dt, 1e-3))))
        dt = run(rows)
    flops = 2.0 * rows * n * k
    return flops / dt / 1e12, f"{rows}x{n}x{k} row sample of {desc} (fp64 numpy oracle port)", cores, dt


_REF = {}   # fork-shared operands of the reference-kernel pool


def _ref_worker(i):
    """One host core: the reference's compiled local GEMM (_gemmcore.pyx:10-25)
    on row block i of the sample."""
    import numpy as np

    mod = ref_gemm_module()
    a, b, rpc = _REF["a"], _REF["b"], _REF["rpc"]
    c = np.zeros((rpc, b.shape[1]))
    t0 = time.perf_counter()
    mod.gemm_accumulate(a[i * rpc:(i + 1) * rpc], b, c)
    return time.perf_counter() - t0


def ref_gemm_module():
    """The reference's own compiled kernel, built from its sources into oracle/_ref
    (oracle/Makefile), or None when it is not there."""
    d = os.path.join(ROOT, "oracle", "_ref")
    if d not in sys.path:
        sys.path.insert(0, d)
    try:
        import _gemmcore  # noqa: PLC0415

        return _gemmcore
    except ImportError:
        return None


class RefKernelPool:
    """The reference's CPU path on cfg's local GEMM (at p = 1 the whole multiply
    is one `local_gemm`, runtime.py:96-107, on the compiled backend the
    reference selects when built: kernels.py:20-28), on every host core: the
    kernel holds the GIL, so one forked process per core, each on its own row
    block of a row sample (fp64, as the reference)."""

    def __init__(self, n, k, target_s):
        import multiprocessing as mp

        import numpy as np

        self.mod = ref_gemm_module()
        self.cores = len(os.sched_getaffinity(0))
        rng = np.random.default_rng(0)
        b = rng.uniform(-1, 1, size=(k, n))
        probe = rng.uniform(-1, 1, size=(4, k))
        c = np.zeros((4, n))
        t0 = time.perf_counter()
        self.mod.gemm_accumulate(probe, b, c)
        per_row = (time.perf_counter() - t0) / 4
        rpc = max(1, int(target_s / per_row))
        _REF.update(a=rng.uniform(-1, 1, size=(rpc * self.cores, k)), b=b, rpc=rpc)
        self.rows = rpc * self.cores
        self.n, self.k = n, k
        self.pool = mp.get_context("fork").Pool(self.cores)

    def step(self) -> float:
        t0 = time.perf_counter()
        self.pool.map(_ref_worker, range(self.cores), chunksize=1)
        return time.perf_counter() - t0

    def close(self):
        self.pool.terminate()


def reference_arm(args):
    """--impl reference: the reference's own CPU implementation of the path on this
    host's cores (its compiled kernel from oracle/_ref; the numpy oracle port if
    that is absent), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    m, n, k, ap, bp, cp, fa, fb, fc, desc = CONFIGS[args.config]
    if ref_gemm_module() is not None:
        pool = RefKernelPool(n, k, args.ref_step_s)
        for _ in range(args.warmup):
            pool.step()
        dts = [pool.step() for _ in range(args.steps)]
        pool.close()
        dt = sum(dts) / len(dts)
        rows, cores, kind = pool.rows, pool.cores, "reference"
        sample = (f"{rows}x{n}x{k} row sample of {desc}: the reference's compiled _gemmcore kernel "
                  f"(oracle/_ref, fp64), one process per core")
    else:
        import numpy as np

        from oracle import um_oracle as O

        cores = len(os.sched_getaffinity(0))
        _, sample, cores, _ = cpu_oracle_rate(m, n, k, args.gpus, desc, target_s=args.ref_step_s)
        rows = int(sample.split("x")[0])
        rng = np.random.default_rng(1)
        a = rng.uniform(-1, 1, size=(rows, k))
        b = rng.uniform(-1, 1, size=(k, n))
        mats = [O.Mat("A", rows, k, O.Spec(rows, k, 1, 1), 1, 1), O.Mat("B", k, n, O.Spec(k, n, 1, 1), 1, 1),
                O.Mat("C", rows, n, O.Spec(rows, n, 1, 1), 1, 1)]
        with blas_threads(cores):
            for _ in range(args.warmup):
                O.execute("c", *mats, a, b)
            t0 = time.perf_counter()
            for _ in range(args.steps):
                O.execute("c", *mats, a, b)
            dt = (time.perf_counter() - t0) / args.steps
        kind = "port"
    val = 2.0 * rows * n * k / dt / 1e12
    out = {"metric": METRIC, "value": val, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{args.config}: {desc}", "m": m, "n": n, "k": k, "p": args.gpus,
                      "partitions": [ap, bp, cp], "sample_rows": rows},
           "impl": "reference",
           "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": cores, "kind": kind, "sample": sample},
           "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def b200_arm(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2510_08874_b200 import ExecConfig, execute_multiply
    from paper_2510_08874_b200 import engine as eng
    from paper_2510_08874_b200 import runtime as rt
    from paper_2510_08874_b200.cli import build_problem

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one process per GPU")
    if world > ndev and not args.oversubscribe:
        raise SystemExit(f"bench.py: {world} ranks but {ndev} visible GPU(s); --oversubscribe to time-share")
    n_gpus = min(world, ndev)     # physical GPUs in use (ranks share a GPU only under --oversubscribe)
    local = local % ndev
    torch.cuda.set_device(local)
    if world > 1:
        if world <= ndev:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group("gloo")
    p = world
    m, n, k, ap, bp, cp, fa, fb, fc, desc = CONFIGS[args.config]
    ca, cb, cc = fa(p), fb(p), fc(p)
    fab, A, B, C, _, _ = build_problem(m, n, k, p, ap, bp, cp, ca, cb, cc, seed=0, real=True, synthetic=True,
                                       devices=[local] if world > 1 else [0])
    cfg = ExecConfig()
    flops = 2.0 * m * n * k
    dev = torch.device(f"cuda:{local}")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64,
                         device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident timing
    for _ in range(args.warmup):
        execute_multiply(A, B, C, cfg)
    barrier()
    eng.TRACE.clear()
    eng.TRACE_ENABLED = True
    sampler = ClockSampler(local)
    barrier()
    sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    launches = 0
    for _ in range(args.steps):
        stats = execute_multiply(A, B, C, cfg)
        launches += sum(s.launches for s in stats.values()) + (len(list(C.grid.tiles())) if C.c > 1 else 0)
    e1.record()
    barrier()
    clocks = sampler.stop()
    eng.TRACE_ENABLED = False
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    value = flops / (ms * 1e-3) / 1e12
    # dominant kernel (K1 grouped launch) durations, measured on its own stream
    durs = [s.elapsed_time(e) for s, e, _ in eng.TRACE]
    kflops = [f for _, _, f in eng.TRACE]
    peak, peak_sus, peak_kind = load_peaks()
    if durs:
        achieved = sum(kflops) / (sum(durs) * 1e-3) / 1e12
    else:
        achieved = None

    # ---- end-to-end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        e2e = e2e_run(args, A, B, C, cfg, flops, dev, barrier, max_over_ranks)

    # ---- CPU baseline (oracle port) on rank 0, N=1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        port_rate, port_sample, cores, _ = cpu_oracle_rate(m, n, k, p, desc, target_s=args.cpu_s / 2)
        if ref_gemm_module() is not None:
            pool = RefKernelPool(n, k, args.cpu_s / 2)
            pool.step()
            dt = pool.step()
            pool.close()
            cpu = {"value": 2.0 * pool.rows * n * k / dt / 1e12, "unit": "TFLOP/s", "cores": pool.cores,
                   "kind": "reference",
                   "sample": f"{pool.rows}x{n}x{k} row sample of {desc}: the reference's compiled _gemmcore "
                             f"kernel (oracle/_ref, fp64), one process per core",
                   "numpy_port": {"value": port_rate, "cores": cores, "sample": port_sample}}
        else:
            cpu = {"value": port_rate, "unit": "TFLOP/s", "cores": cores, "kind": "port", "sample": port_sample}

    traffic = k1_traffic(args.config) if world == 1 else None
    # A read once, B read once, C read + written once (fp32 C += A.B), per K1 launch
    algo_bytes = (2 * m * k + 2 * k * n + 8 * m * n) / p
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": n_gpus, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
               "config": {"workload": f"{args.config}: {desc}", "m": m, "n": n, "k": k, "p": p,
                          "partitions": [ap, bp, cp], "replication": [ca, cb, cc], "stationarity": "c",
                          "inputs": "bf16 uniform(-1,1) generated on device (K5), C fp32",
                          "l2": "inputs larger than L2 (A %.0f MiB, C %.0f MiB per rank > 126 MB)" % (
                              m * k * 2 / p / 2**20, m * n * 4 / p / 2**20)},
               "frac_of_peak": value / (n_gpus * peak), "peak_per_gpu_tflops": peak, "peak_kind": peak_kind,
               "ranks": world, "oversubscribed": world > n_gpus,
               "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                            "frac": (achieved / peak) if achieved else None,
                            "traffic": (traffic or {}).get("bytes_per_launch"),
                            "traffic_source": (traffic or {}).get("source"),
                            "traffic_captured": (traffic or {}).get("captured"),
                            "algorithmic_bytes_per_launch": algo_bytes,
                            "kernel": "um::gemm::gemm_bf16_kernel<2>", "launches_timed": len(durs),
                            "algorithmic_flops_per_launch": (sum(kflops) / len(kflops)) if kflops else None},
               "clocks": clocks, "gpu_launches": launches,
               "e2e": e2e, "cpu_baseline": cpu}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def e2e_run(args, A, B, C, cfg, flops, dev, barrier, max_over_ranks):
    """Same metric through the public host-memory API (hostio.multiply_from_host):
    every step uploads A and B from pinned host buffers and downloads C, with the
    transfers pipelined against the GEMMs over row panels."""
    import torch

    from paper_2510_08874_b200.hostio import multiply_from_host

    m, k = A.global_shape.rows, A.global_shape.cols
    n = B.global_shape.cols
    a_h = torch.empty((m, k), dtype=A.dtype, pin_memory=True).uniform_(-1, 1)
    b_h = torch.empty((k, n), dtype=B.dtype, pin_memory=True).uniform_(-1, 1)
    c_h = torch.empty((m, n), dtype=torch.float32, pin_memory=True)

    def nbytes(M, replica0_only=False):
        return sum(seg.length * seg.esize for (rep, t), seg in M._segments.items()
                   if seg.storage is not None and (rep == 0 or not replica0_only))

    h2d = nbytes(A) + nbytes(B)
    d2h = nbytes(C, replica0_only=True)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    steps = max(1, args.steps // 2)
    single_ms = None
    if world == 1 and not args.e2e_graph and not args.e2e_single:
        # the K steps as one multiply_from_host_many call: step s + 1's uploads
        # overlap step s's download tail (every step still uploads its A and B
        # and downloads its C); the one-call-per-step pipeline is timed too
        from paper_2510_08874_b200.hostio import multiply_from_host_many

        def run(n_jobs):
            multiply_from_host_many(A, B, C, [(a_h, b_h, c_h)] * n_jobs, cfg, panels=args.panels,
                                    col_panels=args.col_panels)

        run(max(1, args.warmup))
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            multiply_from_host(A, B, C, a_h, b_h, c_h, cfg, panels=args.panels, col_panels=args.col_panels)
        e1.record()
        barrier()
        single_ms = max_over_ranks(e0.elapsed_time(e1) / steps)
        e0.record()
        run(steps)
        e1.record()
        barrier()
        ms = max_over_ranks(e0.elapsed_time(e1) / steps)
        api = (f"hostio.multiply_from_host_many ({steps} jobs in one call: each job's uploads start once the "
               f"previous job no longer reads the device panel, i.e. during its download tail)")
    elif world == 1 and args.e2e_graph:
        # the host-streaming multiply replayed as one CUDA graph: every replay
        # still uploads A and B from the pinned host buffers and downloads C
        from paper_2510_08874_b200.hostio import CapturedHostMultiply

        cap = CapturedHostMultiply(A, B, C, a_h, b_h, c_h, cfg, panels=args.panels, col_panels=args.col_panels)

        def step():
            cap.replay()
    else:
        def step():
            multiply_from_host(A, B, C, a_h, b_h, c_h, cfg, panels=args.panels, copy_streams=args.copy_streams,
                               col_panels=args.col_panels)

    if single_ms is None:
        for _ in range(max(1, args.warmup)):
            step()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
        barrier()
        ms = max_over_ranks(e0.elapsed_time(e1) / steps)
        api = ("hostio.multiply_from_host" if (world > 1 or not args.e2e_graph)
               else "hostio.CapturedHostMultiply (multiply_from_host as one CUDA graph)")
    # the e2e roofline: this box's pinned-memory copy bandwidth, each direction
    # alone and both at once (PCIe is full duplex); floor = the smaller volume
    # moved in both directions at once at the concurrent rate, then the rest
    # of the larger one alone
    bw = pcie_bandwidth(dev)
    both = min(h2d, d2h)
    rest_ms = (h2d - both) / bw["h2d_gbs"] / 1e6 + (d2h - both) / bw["d2h_gbs"] / 1e6
    floor_ms = max(both / bw["h2d_concurrent_gbs"], both / bw["d2h_concurrent_gbs"]) / 1e6 + rest_ms
    # the same copies in the order multiply_from_host issues them, each C block
    # downloadable only once its A rows and B columns are up (and computed at
    # the measured peak): the floor of this block pipeline, not only of PCIe
    P = args.panels
    Q = args.col_panels
    if Q is None:
        big_b = B.global_shape.rows * B.global_shape.cols * 4 >= m * k
        Q = P if (big_b and C.c == 1) else 1
    pipe_ms = pipeline_floor_ms(P, Q, nbytes(A), nbytes(B), d2h, flops, bw["h2d_concurrent_gbs"],
                                bw["d2h_concurrent_gbs"], load_peaks()[0], bw["h2d_gbs"], bw["d2h_gbs"])
    return {"value": flops / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms, "steps": steps, "api": api,
            "single_call_ms_per_step": single_ms,
            "panels": args.panels, "col_panels": args.col_panels, "copy_streams": args.copy_streams,
            "roofline": {"bound": "pcie", "floor_ms_per_step": floor_ms, "frac": floor_ms / ms,
                         "pipeline_floor_ms_per_step": pipe_ms, "pipeline_frac": pipe_ms / ms,
                         "pipeline_grid": [P, Q], **bw}}


def pipeline_floor_ms(P: int, Q: int, a_bytes: int, b_bytes: int, c_bytes: int, flops: float, up_gbs: float,
                      dn_gbs: float, peak_tflops: float, up_alone_gbs: float | None = None,
                      dn_alone_gbs: float | None = None) -> float:
    """Lower bound of hostio's block pipeline: uploads back to back on one
    stream in the issue order (Q > 1: A row panel i / B column panel j the
    first time a block of the shell order needs it; Q == 1: all of B, then A
    row panels), each block computed at `peak_tflops` once its panels are up
    and the previous block is done, and downloaded after that, back to back
    on one stream.  Uploads run at the one-direction rate until the first
    download starts, downloads at it once the uploads are done, both at the
    concurrent rate in between.  C += A.B needs all of A's rows and B's
    columns of a block before any of it is final, so even continuous square
    shells cannot beat 1.25 x the PCIe floor."""
    from paper_2510_08874_b200.hostio import _shell_order

    up_alone = up_alone_gbs or up_gbs
    dn_alone = dn_alone_gbs or dn_gbs
    order = _shell_order(P, Q) if Q > 1 else [(i, 0) for i in range(P)]
    # uploads in issue order: (bytes, panel key)
    ups = [(b_bytes, ("b", 0))] if Q == 1 else []
    seen = set(k for _, k in ups)
    for i, j in order:
        for key, nb in ((("a", i), a_bytes / P), (("b", j), b_bytes / Q)):
            if key not in seen:
                seen.add(key)
                ups.append((nb, key))
    first_dn = None
    for _ in range(3):   # the first download's start and the upload times depend on each other
        t_up, at = 0.0, {}
        for nb, key in ups:
            rate = up_alone if first_dn is None or t_up < first_dn else up_gbs
            t_up += nb / (rate * 1e9) * 1e3
            at[key] = t_up
        t_c = t_d = 0.0
        start = None
        for i, j in order:
            t_c = max(t_c, at[("a", i)], at[("b", j if Q > 1 else 0)]) + flops / (P * Q) / (peak_tflops * 1e12) * 1e3
            s0 = max(t_d, t_c)
            start = s0 if start is None else start
            rate = dn_alone if s0 >= t_up else dn_gbs
            t_d = s0 + c_bytes / (P * Q) / (rate * 1e9) * 1e3
        first_dn = start
    return t_d


def pcie_bandwidth(dev, nbytes: int = 1 << 30, reps: int = 3) -> dict:
    """Pinned host <-> device copy bandwidth (GB/s), one direction alone and both concurrently."""
    import torch

    h_src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h_dst = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d_src = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d_dst = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s_up, s_down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(streams_ops):
        best = float("inf")
        for _ in range(reps):
            torch.cuda.synchronize(dev)
            evs = []
            for st_, op in streams_ops:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(st_):
                    e0.record()
                    op()
                    e1.record()
                evs.append((e0, e1))
            torch.cuda.synchronize(dev)
            best = min(best, max(a.elapsed_time(b) for a, b in evs))
        return nbytes / (best * 1e-3) / 1e9

    up = (s_up, lambda: d_dst.copy_(h_src, non_blocking=True))
    down = (s_down, lambda: h_dst.copy_(d_src, non_blocking=True))
    both = timed([up, down])
    return {"h2d_gbs": timed([up]), "d2h_gbs": timed([down]), "h2d_concurrent_gbs": both, "d2h_concurrent_gbs": both}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg5", choices=sorted(CONFIGS))
    ap.add_argument("--oversubscribe", action="store_true",
                    help="allow more ranks than visible GPUs (ranks time-share a GPU; functional runs only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--panels", type=int, default=4,
                    help="row panels of the host-streaming e2e path (cfg5: a panels x panels block grid; "
                         "measured 4 x 4 30 ms, 8 x 8 32 ms, 16 x 16 38 ms per step, profiles/r2_e2e_grid.log)")
    ap.add_argument("--col-panels", type=int, default=None,
                    help="column panels of the e2e block grid (default: hostio's choice)")
    ap.add_argument("--e2e-graph", action="store_true",
                    help="e2e through hostio.CapturedHostMultiply (the same copies + launches replayed as a CUDA graph)")
    ap.add_argument("--e2e-single", action="store_true",
                    help="e2e as one multiply_from_host call per step (default: the steps as one pipelined "
                         "multiply_from_host_many call)")
    ap.add_argument("--copy-streams", type=int, default=1, help="copy streams per direction in the e2e path (measured: 1 best)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-s", type=float, default=10.0, help="target seconds of CPU oracle work")
    ap.add_argument("--ref-step-s", type=float, default=4.0, help="target seconds per reference-arm step")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    else:
        b200_arm(args)


if __name__ == "__main__":
    main()

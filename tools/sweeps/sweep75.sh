python tools/debug/launch_probe.py 2>&1 | grep "us/launch"
timeout 60 python tools/profile_gemm.py --time --iters 20 --m 4096 --n 4096 --k 4096 2>&1 | tail -1 | cut -c1-100

timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_gemm_variants_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
for R in 1 2; do for B in 0 1; do
  for S in "" "--m 16384 --n 16384 --k 16384" "--m 4096 --n 4096 --k 4096"; do
    UM_GEMM_B3D=$B timeout 60 python tools/profile_gemm.py --time --iters 20 $S 2>&1 | tail -1 | cut -c1-90 | sed "s/^/[b3d $B] /"
  done
done; done
for B in 0 1; do UM_GEMM_B3D=$B timeout 60 python tools/profile_gemm.py --time --iters 100 2>&1 | tail -1 | cut -c1-110 | sed "s/^/[b3d $B long] /"; done
for B in 0 1; do UM_GEMM_B3D=$B UM_GEMM_STALLS=1 timeout 60 python tools/profile_gemm.py --iters 3 2>&1 | grep pairs | tail -1 | sed "s/^/[b3d $B] /"; done

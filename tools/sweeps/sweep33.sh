for L in "" "$PWD/paper_2510_08874_b200/_lib/variants/gw6.so" "$PWD/paper_2510_08874_b200/_lib/variants/gw8.so"; do
  echo "== lib ${L:-default (4 get warps)}"
  UNIMUL_B200_LIB=$L timeout 120 python tools/solo_probe.py cfg5 8 kernel 2>&1 | grep -v CUDAEvent.h | tail -2
  UNIMUL_B200_LIB=$L timeout 120 python tools/solo_probe.py cfg4 8 kernel 2>&1 | grep -v CUDAEvent.h | grep "rank 3"
  UNIMUL_B200_LIB=$L timeout 120 python tools/get_probe.py 2>&1 | grep -v CUDAEvent.h | grep "512 MiB) in-kernel\|both"
  UNIMUL_B200_LIB=$L timeout 120 python tools/profile_gemm.py --time --iters 30 2>&1 | tail -1
done

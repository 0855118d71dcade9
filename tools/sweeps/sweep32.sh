python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for L in "" "$PWD/paper_2510_08874_b200/_lib/variants/gw2.so"; do
  echo "== lib ${L:-default (4 get warps)}"
  UNIMUL_B200_LIB=$L timeout 120 python tools/solo_probe.py cfg5 8 kernel 2>&1 | grep -v CUDAEvent.h | tail -3
  UNIMUL_B200_LIB=$L timeout 120 python tools/solo_probe.py cfg4 8 kernel 2>&1 | grep -v CUDAEvent.h | grep "rank 3"
  UNIMUL_B200_LIB=$L timeout 120 python tools/get_probe.py 2>&1 | grep -v CUDAEvent.h | grep "512 MiB) in-kernel\|both"
done

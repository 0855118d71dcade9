rm -f gpurun_out/s3_cfg5.log
for r in 1 2; do
for L in tools/debug/lib_base.so tools/debug/lib_e2f.so paper_2510_08874_b200/_lib/libunimul_b200.so; do
  echo "== $L" >> gpurun_out/s3_cfg5.log
  UNIMUL_B200_LIB=$PWD/$L timeout 600 python tools/bench_matrix.py --configs cfg5,cfg4 --ps 8 --steps 5 2>&1 | grep -A1 "p=8" >> gpurun_out/s3_cfg5.log
done
done

for SHAPE in "" "--m 16384 --n 16384 --k 16384"; do
for CPF in 0 8 0 16 0 4 32; do UM_GEMM_CPF=$CPF timeout 90 python tools/profile_gemm.py --time --iters 30 $SHAPE 2>&1 | tail -1 | sed "s/^/[cpf=$CPF] /"; done; done

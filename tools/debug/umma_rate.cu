// Issue-rate microbenchmark of tcgen05.mma cta_group::2 kind::f16 (M=256,
// N=256, K=16 per instruction, both operands in shared memory, the K1
// descriptors: A K-major SW128, B MN-major SW128).  The leader CTA of each
// pair issues `kblocks` k-blocks of 4 UMMAs per accumulator, in one of these
// patterns (mode):
//   0: one accumulator, 8 UMMAs per k-block, no per-k-block sync
//   1: two accumulators alternating per k-block (K1 NT=512 steady state)
//   2: mode 1 + tcgen05.commit to an mbarrier per k-block (multicast to the pair)
//   3: mode 2 + an mbarrier wait per k-block on a barrier the producer arrives
//      on per stage (4-stage ring, producer thread in warp 0 waits on empty)
// and reports cycles per UMMA (clock64 on the issuing SM, first issue ->
// final commit observed).  Operands are garbage: only timing matters.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I../../paper_2510_08874_b200/csrc -o umma_rate umma_rate.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "um_ptx.cuh"

using namespace um;

constexpr int STAGES = 4;
constexpr int A_BYTES = 128 * 64 * 2;
constexpr int B_BYTES = 4 * 64 * 64 * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 256;

__global__ void __launch_bounds__(128, 1) umma_rate(int kblocks, int mode, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* done = bars + 2 * STAGES;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t crank = ptx::cluster_ctarank();
  const bool leader = crank == 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<2>(tslot, 512);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp == 0 && lane == 0 && leader && mode == 3) {
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = 0; kb < kblocks; ++kb) {
      ptx::mbar_wait(&empty[stage], phase ^ 1);
      ptx::mbar_arrive(&full[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
  }
  if (warp == 1 && leader) {
    const bool issuer = ptx::elect_one();
    constexpr uint32_t idesc = ptx::make_idesc_bf16(256, 256, 0, 1);
    int stage = 0;
    uint32_t phase = 0;
    const unsigned long long t0 = clock64();
    for (int kb = 0; kb < kblocks; ++kb) {
      if (mode == 3) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
      }
      const uint32_t sa = ptx::smem_u32(smem + stage * STAGE_BYTES);
      const uint32_t sb = sa + A_BYTES;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const uint32_t acc = (mode == 0) ? 0u : (uint32_t)(j * 256);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t ad = ptx::make_smem_desc(sa + kk * 32, 16, 1024);
          const uint64_t bd = ptx::make_smem_desc(sb + j * 2 * 8192 + kk * 2048, 8192, 1024);
          if (issuer) ptx::umma_f16<2>(tmem + acc, ad, bd, idesc, (kb || kk) ? 1u : 0u);
        }
      }
      if (mode >= 2 && issuer) ptx::umma_commit<2>(&empty[stage], 0x1);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    if (issuer) ptx::umma_commit<2>(done, 0x1);
    ptx::mbar_wait(done, 0);
    const unsigned long long t1 = clock64();
    if (issuer) out[blockIdx.x / 2] = t1 - t0;
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) ptx::tmem_dealloc<2>(tmem, 512);
}

int main(int argc, char** argv) {
  const int kblocks = argc > 1 ? atoi(argv[1]) : 4096;
  const int pairs = argc > 2 ? atoi(argv[2]) : 74;
  unsigned long long* d;
  cudaMalloc(&d, pairs * sizeof(unsigned long long));
  cudaFuncSetAttribute(umma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(2 * pairs);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = SMEM;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      cudaError_t err = cudaLaunchKernelEx(&cfg, umma_rate, kblocks, mode, d);
      cudaEventRecord(e1);
      cudaError_t e2 = cudaDeviceSynchronize();
      if (err != cudaSuccess || e2 != cudaSuccess) {
        printf("mode %d: %s / %s\n", mode, cudaGetErrorString(err), cudaGetErrorString(e2));
        return 1;
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long h[256];
      cudaMemcpy(h, d, pairs * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      double mx = 0, sum = 0;
      for (int i = 0; i < pairs; ++i) { sum += h[i]; mx = h[i] > mx ? h[i] : mx; }
      const double umma = 8.0 * kblocks;
      const double flops = 2.0 * 256 * 256 * 16 * umma * pairs;
      printf("mode %d pairs %d: cycles/UMMA mean %.1f max %.1f; %.3f ms, %.0f TFLOP/s, clock %.0f MHz\n", mode, pairs,
             sum / pairs / umma, mx / umma, ms, flops / (ms * 1e-3) / 1e12, (sum / pairs) / (ms * 1e3));
    }
  }
  return 0;
}

// Epilogue drain microbenchmark: how fast can one SM move a 128 x 256 fp32
// accumulator block (128 KiB, K1's per-CTA tile at NT=256) from registers into
// C?  4 warps, each owning 32 rows, emit 8 chunks of 32 x 32 fp32 (lane = row)
// in one of these ways (mode):
//   0: swizzled smem box -> fence.proxy.async -> TMA reduce-add (K1's epilogue)
//   1: as 0 with a TMA store instead of the reduce
//   2: as 0 without the proxy fence (timing only: the TMA may read stale smem)
//   3: smem + fence only, no TMA op
//   4: as 0, two chunks per fence / bulk group
//   5: smem transpose -> red.global.add.v4.f32 (coalesced 128-byte rows)
//   6: smem transpose -> ld.global + add + st.global (exclusive writer)
//   7: as 0, one 3-D TMA reduce per warp for all 8 chunks (32 KiB box)
//   8: the smem stores alone
//   9: smem stores alone, linear (unswizzled, conflict-free) addresses
// `nbox` smem boxes per warp are in flight (modes 0-4).  Reports the mean and
// max per-CTA drain time over `ctas` CTAs that each own a disjoint C block
// (1 CTA: the per-SM rate; 148: with the whole GPU draining at once).
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I../../paper_2510_08874_b200/csrc -o drain_probe drain_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "um_ptx.cuh"

using namespace um;

constexpr int ROWS = 128, COLS = 256, CHUNKS = COLS / 32, BOX = 32 * 32 * 4;
constexpr int MAXBOX = 8;
constexpr int SMEM = 1024 + 4 * MAXBOX * BOX;

__device__ __forceinline__ void tma_reduce_add_3d(const void* tmap, uint32_t src, int32_t c0, int32_t c1, int32_t c2) {
  asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   tmap),
               "r"(src), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

template <int NBOX>
__global__ void __launch_bounds__(128, 1)
    drain(const __grid_constant__ CUtensorMap m2, const __grid_constant__ CUtensorMap m3, float* c, int pitch, int mode,
          int reps, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const bool issuer = ptx::elect_one();
  const uint32_t ebuf = ptx::smem_u32(smem) + warp * MAXBOX * BOX;
  const int row0 = blockIdx.x * ROWS + warp * 32;
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(1.0f);
  __syncthreads();
  const unsigned long long t0 = ptx::globaltimer();
  const long long k0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    int sbuf = 0;
    if (mode == 7) {
      // all 8 chunks into one 32 KiB region, one 3-D reduce
      if (issuer) ptx::bulk_wait_read<0>();
      __syncwarp();
      for (int ch = 0; ch < CHUNKS; ++ch) {
        const uint32_t base = ebuf + ch * BOX;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          ptx::st_shared_v4(base + lane * 128 + ((i ^ (lane & 7)) << 4), r[4 * i], r[4 * i + 1], r[4 * i + 2],
                            r[4 * i + 3]);
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (issuer) {
        tma_reduce_add_3d(&m3, ebuf, 0, row0, 0);
        ptx::bulk_commit();
      }
      continue;
    }
    for (int ch = 0; ch < CHUNKS; ++ch) {
      const uint32_t base = ebuf + sbuf * BOX;
      const int col0 = ch * 32;
      if (mode <= 4 || mode >= 8) {
        const bool group_start = mode != 4 || (ch & 1) == 0;
        if (group_start) {
          if (issuer) {
            if (mode == 4) ptx::bulk_wait_read<(NBOX / 2 > 0 ? NBOX / 2 : 1) - 1>();
            else ptx::bulk_wait_read<NBOX - 1>();
          }
          __syncwarp();
        }
        if (mode == 9) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            ptx::st_shared_v4(base + i * 512 + lane * 16, r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            ptx::st_shared_v4(base + lane * 128 + ((i ^ (lane & 7)) << 4), r[4 * i], r[4 * i + 1], r[4 * i + 2],
                              r[4 * i + 3]);
        }
        const bool group_end = mode != 4 || (ch & 1) == 1;
        if (group_end) {
          if (mode != 2 && mode < 8) ptx::fence_proxy_async_smem();
          __syncwarp();
          if (issuer && mode != 3 && mode < 8) {
            if (mode == 4) {
              ptx::tma_reduce_add_2d(&m2, smem + (base - BOX - ptx::smem_u32(smem)), col0 - 32, row0);
              ptx::tma_reduce_add_2d(&m2, smem + (base - ptx::smem_u32(smem)), col0, row0);
            } else if (mode == 1) {
              ptx::tma_store_2d(&m2, smem + (base - ptx::smem_u32(smem)), col0, row0);
            } else {
              ptx::tma_reduce_add_2d(&m2, smem + (base - ptx::smem_u32(smem)), col0, row0);
            }
          }
          if (issuer) ptx::bulk_commit();
        }
      } else {
        // modes 5, 6: transpose through smem, coalesced LSU access
#pragma unroll
        for (int i = 0; i < 8; ++i)
          ptx::st_shared_v4(base + lane * 128 + ((i ^ (lane & 7)) << 4), r[4 * i], r[4 * i + 1], r[4 * i + 2],
                            r[4 * i + 3]);
        __syncwarp();
        const int c4 = lane & 7;
        float4 cv[8];
        if (mode == 6) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = i * 4 + (lane >> 3);
            cv[i] = *reinterpret_cast<const float4*>(c + (size_t)(row0 + rr) * pitch + col0 + 4 * c4);
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = i * 4 + (lane >> 3);
          const float4 v = ptx::ld_shared_v4f(base + rr * 128 + ((c4 ^ (rr & 7)) << 4));
          float* dst = c + (size_t)(row0 + rr) * pitch + col0 + 4 * c4;
          if (mode == 5) {
            ptx::red_add_v4_f32(dst, v.x, v.y, v.z, v.w);
          } else {
            cv[i].x += v.x; cv[i].y += v.y; cv[i].z += v.z; cv[i].w += v.w;
            *reinterpret_cast<float4*>(dst) = cv[i];
          }
        }
        __syncwarp();
      }
      sbuf = (sbuf + 1) % NBOX;
    }
  }
  if (issuer) ptx::bulk_wait<0>();
  __threadfence();
  __syncthreads();
  const unsigned long long t1 = ptx::globaltimer();
  const long long k1 = clock64();
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = t1 - t0;
    out[2 * blockIdx.x + 1] = (unsigned long long)(k1 - k0);
  }
}

// keeps every SM busy for `ns` so the clocks are up before a measurement
__global__ void spin(unsigned long long ns) {
  const unsigned long long t0 = ptx::globaltimer();
  while (ptx::globaltimer() - t0 < ns) {
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 1;
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  const int maxctas = 148;
  const int pitch = COLS;
  float* c;
  cudaMalloc(&c, (size_t)maxctas * ROWS * COLS * 4);
  cudaMemset(c, 0, (size_t)maxctas * ROWS * COLS * 4);
  unsigned long long* d;
  cudaMalloc(&d, maxctas * 16);
  CUtensorMap m2, m3;
  {
    cuuint64_t dims[2] = {(cuuint64_t)COLS, (cuuint64_t)maxctas * ROWS};
    cuuint64_t strides[1] = {(cuuint64_t)pitch * 4};
    cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    if (enc(&m2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, c, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != 0) {
      printf("encode 2d failed\n");
      return 1;
    }
  }
  {
    // (32 cols, rows, 8 column chunks): one box covers a warp's 32 rows x 256 cols
    cuuint64_t dims[3] = {32, (cuuint64_t)maxctas * ROWS, (cuuint64_t)CHUNKS};
    cuuint64_t strides[2] = {(cuuint64_t)pitch * 4, 128};
    cuuint32_t box[3] = {32, 32, (cuuint32_t)CHUNKS}, es[3] = {1, 1, 1};
    if (enc(&m3, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, c, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != 0) {
      printf("encode 3d failed (3-D mode skipped)\n");
      m3 = m2;
    }
  }
  cudaFuncSetAttribute(drain<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  cudaFuncSetAttribute(drain<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  cudaFuncSetAttribute(drain<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  const char* names[10] = {"tma-reduce", "tma-store", "reduce-nofence", "smem+fence", "reduce-2/fence",
                          "red.v4", "ld+add+st", "3d-reduce", "smem only", "smem linear"};
  for (int ctas : {1, 148}) {
    for (int mode = 0; mode < 10; ++mode) {
      for (int nbox : {2, 4, 8}) {
        if (mode >= 5 && nbox != 2) continue;
        if (argc > 2 && ctas > 1) continue;
        std::vector<unsigned long long> h(2 * ctas);
        double best_mean = 1e30, best_max = 0, best_cyc = 0;
        spin<<<148, 32>>>(20000000ull);
        for (int trial = 0; trial < 5; ++trial) {
          if (nbox == 2) drain<2><<<ctas, 128, SMEM>>>(m2, m3, c, pitch, mode, reps, d);
          if (nbox == 4) drain<4><<<ctas, 128, SMEM>>>(m2, m3, c, pitch, mode, reps, d);
          if (nbox == 8) drain<8><<<ctas, 128, SMEM>>>(m2, m3, c, pitch, mode, reps, d);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("mode %d: %s\n", mode, cudaGetErrorString(e));
            return 1;
          }
          cudaMemcpy(h.data(), d, ctas * 16, cudaMemcpyDeviceToHost);
          double s = 0, mx = 0, cy = 0;
          for (int i = 0; i < ctas; ++i) {
            s += h[2 * i];
            cy += h[2 * i + 1];
            mx = h[2 * i] > mx ? h[2 * i] : mx;
          }
          if (s / ctas < best_mean) { best_mean = s / ctas; best_max = mx; best_cyc = cy / ctas; }
        }
        const double bytes = (double)ROWS * COLS * 4 * reps;
        printf("ctas %3d %-15s nbox %d: %.2f us mean, %.2f us max per CTA (%.1f GB/s per SM), %.0f cycles = %.1f B/clk, "
               "%.0f MHz\n", ctas, names[mode], nbox, best_mean / 1e3 / reps, best_max / 1e3 / reps, bytes / best_mean,
               best_cyc / reps, bytes / best_cyc, best_cyc / best_mean * 1e3);
      }
    }
  }
  return 0;
}

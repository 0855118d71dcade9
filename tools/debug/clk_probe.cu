// SM clock sampler: one warp that co-resides with a GEMM (no shared memory,
// 32 threads) and records (globaltimer ns, clock64) pairs every `period_ns`
// until *stop != 0 or `cap` samples; the host derives the SM clock actually
// run during any kernel (ours or cuBLAS's) from consecutive pairs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o clk_probe.so clk_probe.cu
#include <cstdint>
#include <cuda_runtime.h>

__global__ void clk_probe_kernel(unsigned long long* out, int cap, unsigned period_ns, const volatile int* stop,
                                 int* count) {
  if (threadIdx.x != 0) return;
  int i = 0;
  for (; i < cap; ++i) {
    unsigned long long t, c;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    c = clock64();
    out[2 * i] = t;
    out[2 * i + 1] = c;
    if (*stop) { ++i; break; }
    unsigned long long t1 = t;
    while (t1 - t < period_ns) {
      __nanosleep(500);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    }
  }
  *count = i;
}

extern "C" int clk_probe_launch(unsigned long long* out, int cap, unsigned period_ns, const int* stop, int* count,
                                void* stream) {
  clk_probe_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(out, cap, period_ns, stop, count);
  return (int)cudaGetLastError();
}

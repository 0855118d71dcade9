// Fixed GPU cost of a K1-shaped launch: empty kernels with K1's launch
// configuration (2-CTA clusters, 230 KB dynamic smem, 320 threads) and
// parameter blocks of different sizes, timed inside a CUDA graph.
#include <cstdio>
#include <cuda_runtime.h>

template <int BYTES>
struct Params { unsigned char b[BYTES]; };

template <int BYTES>
__global__ void __launch_bounds__(320, 1) empty_kernel(const __grid_constant__ Params<BYTES> p, int* out) {
  if (threadIdx.x == 0 && p.b[blockIdx.x % BYTES] == 255) out[0] = 1;
}

template <int BYTES>
float run(int ctas, int cluster, int smem) {
  auto k = empty_kernel<BYTES>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  Params<BYTES> p{};
  int* out;
  cudaMalloc(&out, 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(320);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute a[1];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = cluster; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 1;
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 100; ++i) cudaLaunchKernelEx(&cfg, k, p, out);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  if (cudaGetLastError() != cudaSuccess) printf("error\n");
  return ms * 1000.f / 1000.f;   // us per launch
}

int main() {
  printf("params  ctas cluster smem   us/launch\n");
  printf("%6d %5d %7d %6d %8.2f\n", 64, 2, 2, 230656, run<64>(2, 2, 230656));
  printf("%6d %5d %7d %6d %8.2f\n", 28000, 2, 2, 230656, run<28000>(2, 2, 230656));
  printf("%6d %5d %7d %6d %8.2f\n", 64, 148, 2, 230656, run<64>(148, 2, 230656));
  printf("%6d %5d %7d %6d %8.2f\n", 28000, 148, 2, 230656, run<28000>(148, 2, 230656));
  printf("%6d %5d %7d %6d %8.2f\n", 64, 2, 1, 0, run<64>(2, 1, 0));
  printf("%6d %5d %7d %6d %8.2f\n", 28000, 2, 1, 0, run<28000>(2, 1, 0));
  return 0;
}

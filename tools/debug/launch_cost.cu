// Fixed GPU cost of a K1-shaped launch: empty kernels with K1's launch
// configuration (2-CTA clusters, 230 KB dynamic smem, 320 threads) and
// parameter blocks of different sizes, timed inside a CUDA graph.
#include <chrono>
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

// host cost of one cudaLaunchKernelEx (K1's attributes: cluster 2 + PDL), no graph
template <int BYTES>
float host_run(int ctas) {
  auto k = empty_kernel<BYTES>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 230656);
  Params<BYTES> p{};
  int* out;
  cudaMalloc(&out, 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(320);
  cfg.dynamicSmemBytes = 230656;
  cfg.stream = s;
  cudaLaunchAttribute a[2];
  a[0].id = cudaLaunchAttributeClusterDimension;
  a[0].val.clusterDim.x = 2; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
  a[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = a;
  cfg.numAttrs = 2;
  for (int i = 0; i < 100; ++i) cudaLaunchKernelEx(&cfg, k, p, out);
  cudaStreamSynchronize(s);
  const int N = 2000;
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, k, p, out);
  auto t1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(s);
  auto t2 = std::chrono::steady_clock::now();
  if (cudaGetLastError() != cudaSuccess) printf("error\n");
  printf("host: params %6d ctas %4d: %.2f us per launch call, %.2f us per launch incl. drain\n", BYTES, ctas,
         std::chrono::duration<double, std::micro>(t1 - t0).count() / N,
         std::chrono::duration<double, std::micro>(t2 - t0).count() / N);
  return 0.f;
}

int main() {
  host_run<64>(148);
  host_run<4096>(148);
  host_run<28000>(148);
  host_run<64>(2);
  host_run<28000>(2);
  printf("params  ctas cluster smem   us/launch\n");
  printf("%6d %5d %7d %6d %8.2f\n", 64, 2, 2, 230656, run<64>(2, 2, 230656));
  printf("%6d %5d %7d %6d %8.2f\n", 28000, 2, 2, 230656, run<28000>(2, 2, 230656));
  printf("%6d %5d %7d %6d %8.2f\n", 64, 148, 2, 230656, run<64>(148, 2, 230656));
  printf("%6d %5d %7d %6d %8.2f\n", 28000, 148, 2, 230656, run<28000>(148, 2, 230656));
  printf("%6d %5d %7d %6d %8.2f\n", 64, 2, 1, 0, run<64>(2, 1, 0));
  printf("%6d %5d %7d %6d %8.2f\n", 28000, 2, 1, 0, run<28000>(2, 1, 0));
  return 0;
}

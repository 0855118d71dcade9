// K2'-K5: one-sided data movement for the distributed GEMM (the default K2
// pulls run inside the K1 launch, gemm_sm100.cu; um_get is the copy-engine form).
//
//  um_get             <- Fabric.get / get_async        (fabric.py:156-192)
//  um_signal / um_wait_geq <- PendingCopy.wait / the run-level barrier, as
//                        stream memory operations (no SM held)
//  um_accumulate      <- Fabric.accumulate PEER_ATOMIC (fabric.py:203-234)
//  um_reduce_replicas <- DistributedMatrix.reduce_replicas (distmatrix.py:211-232)
//  um_copy            <- DistributedMatrix.broadcast_replica (distmatrix.py:234-250)
//  um_fill            <- DistributedMatrix.__init__ init callback (distmatrix.py:95-101)
//
// All of these are HBM/NVLink-bound byte movers: 16-byte vector accesses,
// grid-stride loops sized to a multiple of the SM count, no tensor cores.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <ctime>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "um_internal.h"
#include "um_ptx.cuh"

namespace um {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int check_view(const um_view* v, const char* name, bool need_tma_pitch) {
  if (!v) return fail(UM_EVALUE, std::string("null view ") + name);
  if (v->row_lo < 0 || v->row_hi < v->row_lo || v->col_lo < 0 || v->col_hi < v->col_lo)
    return fail(UM_EVALUE, std::string("invalid slice for ") + name);
  if (v->dtype != UM_BF16 && v->dtype != UM_F32) return fail(UM_EVALUE, std::string("bad dtype for ") + name);
  if (v->pitch < v->col_hi) return fail(UM_ECONTRACT, std::string("pitch smaller than slice for ") + name);
  if (v->row_hi > v->row_lo && v->col_hi > v->col_lo && !v->base)
    return fail(UM_EVALUE, std::string("null base for ") + name);
  if (need_tma_pitch && ((v->pitch * esize(v->dtype)) % 16 != 0 || (reinterpret_cast<uintptr_t>(v->base) & 15)))
    return fail(UM_ECONTRACT, std::string("TMA needs a 16-byte aligned base and pitch for ") + name);
  return UM_OK;
}

DeviceGuard::DeviceGuard(int device) {
  cudaGetDevice(&prev);
  if (device >= 0 && device != prev) cudaSetDevice(device);
}
DeviceGuard::~DeviceGuard() {
  int cur = -1;
  cudaGetDevice(&cur);
  if (prev >= 0 && cur != prev) cudaSetDevice(prev);
}

static int num_sms(int device) {
  static int cache[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cache[device]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || n <= 0) n = 148;
    cache[device] = n;
  }
  return cache[device];
}

static int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

// ------------------------------------------------------------------ kernels

// dst += src element-wise (fp32), dst possibly a peer pointer.  2D grid (x:
// 16-byte column groups, y: rows); red.global.add keeps concurrent
// accumulates atomic per element (fabric.py:226-227 takes a lock for the same
// guarantee).  Ragged tails (cols % 4) are handled by the vec == 0 variant.
__global__ void accumulate_kernel(const float* __restrict__ src, int64_t src_pitch, float* dst, int64_t dst_pitch,
                                  int64_t rows, int64_t cols, int vec) {
  const int64_t groups = vec ? cols / 4 : cols;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= groups) return;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    if (vec) {
      const float4 v = *reinterpret_cast<const float4*>(src + r * src_pitch + 4 * g);
      ptx::red_add_v4_f32(dst + r * dst_pitch + 4 * g, v.x, v.y, v.z, v.w);
    } else {
      ptx::red_add_f32(dst + r * dst_pitch + g, src[r * src_pitch + g]);
    }
  }
}

struct SrcList {
  const float* ptr[16];
  int64_t pitch[16];
};

// dst += sum_i src_i, summed in list order into a register accumulator first
// (the reference's acc, distmatrix.py:224-232).  Sources may be peer pointers
// (P2P loads over NVLink); dst is written with plain stores (owner only).
// HBM/NVLink-bound: a 2D grid (x: 16-byte column groups, U per thread, warp-
// coalesced; y: rows, grid-strided) keeps U * (nsrc + 1) independent 16-byte
// loads in flight per thread and does no 64-bit index division.
constexpr int RED_THREADS = 256;
constexpr int RED_U = 4;
template <int VEC>
__global__ void __launch_bounds__(RED_THREADS) reduce_kernel(SrcList srcs, int nsrc, float* dst, int64_t dst_pitch,
                                                             int64_t rows, int64_t cols) {
  const int64_t groups = cols / VEC;
  const int64_t g0 = (int64_t)blockIdx.x * (RED_THREADS * RED_U) + threadIdx.x;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    if constexpr (VEC == 4) {
      float4 acc[RED_U];
#pragma unroll
      for (int u = 0; u < RED_U; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s = 0; s < nsrc; ++s) {
        const float4* row = reinterpret_cast<const float4*>(srcs.ptr[s] + r * srcs.pitch[s]);
#pragma unroll
        for (int u = 0; u < RED_U; ++u) {
          const int64_t g = g0 + u * RED_THREADS;
          if (g < groups) {
            const float4 v = __ldcs(row + g);
            acc[u].x += v.x; acc[u].y += v.y; acc[u].z += v.z; acc[u].w += v.w;
          }
        }
      }
      float4* drow = reinterpret_cast<float4*>(dst + r * dst_pitch);
#pragma unroll
      for (int u = 0; u < RED_U; ++u) {
        const int64_t g = g0 + u * RED_THREADS;
        if (g < groups) {
          float4 o = drow[g];
          o.x += acc[u].x; o.y += acc[u].y; o.z += acc[u].z; o.w += acc[u].w;
          drow[g] = o;
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < RED_U; ++u) {
        const int64_t c = g0 + u * RED_THREADS;
        if (c < cols) {
          float acc = 0.f;
          for (int s = 0; s < nsrc; ++s) acc += srcs.ptr[s][r * srcs.pitch[s] + c];
          dst[r * dst_pitch + c] += acc;
        }
      }
    }
  }
}

static dim3 reduce_grid(int64_t rows, int64_t groups, int sms) {
  const int64_t gx = (groups + RED_THREADS * RED_U - 1) / (RED_THREADS * RED_U);
  const int64_t want = (int64_t)sms * 8;   // 8 resident blocks of 256 threads per SM
  const int64_t gy = std::max<int64_t>(1, std::min<int64_t>(rows, std::min<int64_t>(65535, (want + gx - 1) / gx)));
  return dim3((unsigned)gx, (unsigned)gy, 1);
}

// Counter-based value generator at GLOBAL coordinates (splitmix64 finaliser),
// restated bit-for-bit in oracle/um_oracle.py:fill_values.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ float fill_value(uint64_t seed, int64_t grow, int64_t gcol, int mode) {
  const uint64_t h = mix64(seed ^ mix64(((uint64_t)grow << 32) ^ (uint64_t)gcol));
  if (mode == UM_FILL_INT) return (float)((int)(h % 17ull) - 8);
  // 24 random bits -> uniform in [-1, 1): exact in fp32
  return (float)((int64_t)(h >> 40) - (1ll << 23)) * (1.0f / 8388608.0f);
}

template <typename T>
__global__ void fill_kernel(T* dst, int64_t pitch, int64_t rows, int64_t cols, int64_t grow0, int64_t gcol0,
                            uint64_t seed, int mode) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols;
    const int64_t c = i - r * cols;
    const float v = mode == UM_FILL_ZERO ? 0.f : fill_value(seed, grow0 + r, gcol0 + c, mode);
    if constexpr (sizeof(T) == 2)
      dst[r * pitch + c] = __float2bfloat16_rn(v);
    else
      dst[r * pitch + c] = v;
  }
}

static int grid_for(int64_t work, int device, int threads = 256) {
  const int64_t blocks = (work + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms(device) * 8;
  return (int)std::max<int64_t>(1, std::min(blocks, cap));
}

}  // namespace um

using namespace um;

// ------------------------------------------------------------------ C-ABI

extern "C" const char* um_version(void) { return "unimul_b200 0.1.0 (sm_100a)"; }
extern "C" const char* um_last_error(void) { return um::g_last_error.c_str(); }

extern "C" int um_get(const um_view* src, const um_view* dst, void* stream) {
  int rc;
  if ((rc = check_view(src, "src", false)) || (rc = check_view(dst, "dst", false))) return rc;
  if (src->dtype != dst->dtype) return fail(UM_ECONTRACT, "get: dtype mismatch");
  if (view_rows(*src) != view_rows(*dst) || view_cols(*src) != view_cols(*dst))
    return fail(UM_ECONTRACT, "get: shape mismatch");
  const int64_t es = esize(src->dtype);
  const int64_t rows = view_rows(*src), cols = view_cols(*src);
  if (rows == 0 || cols == 0) return UM_OK;
  const char* s = static_cast<const char*>(src->base) + (src->row_lo * src->pitch + src->col_lo) * es;
  char* d = static_cast<char*>(dst->base) + (dst->row_lo * dst->pitch + dst->col_lo) * es;
  // Copy-engine transfer (cudaMemcpyDefault resolves peer/IPC/local via UVA).
  UM_CUDA_CHECK(cudaMemcpy2DAsync(d, dst->pitch * es, s, src->pitch * es, cols * es, rows, cudaMemcpyDefault,
                                  reinterpret_cast<cudaStream_t>(stream)));
  return UM_OK;
}

extern "C" int um_get_ce(const um_view* src, const um_view* dst, void* stream) {
  // The pull a running K1 waits for on an arrival flag.  A K1 launch that
  // spins on the flag holds every SM, so the copy must not need one: one
  // cudaMemcpy2DAsync (or cudaMemcpyAsync for a contiguous slice) that the
  // driver runs on the copy engines for peer/IPC sources.  Whether it does is
  // not promised by the API, so callers gate it on um_ce_probe for the pair.
  int rc;
  if ((rc = check_view(src, "src", false)) || (rc = check_view(dst, "dst", false))) return rc;
  if (src->dtype != dst->dtype) return fail(UM_ECONTRACT, "get: dtype mismatch");
  if (view_rows(*src) != view_rows(*dst) || view_cols(*src) != view_cols(*dst))
    return fail(UM_ECONTRACT, "get: shape mismatch");
  const int64_t es = esize(src->dtype);
  const int64_t rows = view_rows(*src), cols = view_cols(*src);
  if (rows == 0 || cols == 0) return UM_OK;
  const bool contiguous = src->pitch == cols && dst->pitch == cols;
  if (!contiguous) return um_get(src, dst, stream);
  const char* s = static_cast<const char*>(src->base) + (src->row_lo * src->pitch + src->col_lo) * es;
  char* d = static_cast<char*>(dst->base) + (dst->row_lo * dst->pitch + dst->col_lo) * es;
  UM_CUDA_CHECK(cudaMemcpyAsync(d, s, (size_t)(rows * cols * es), cudaMemcpyDefault,
                                reinterpret_cast<cudaStream_t>(stream)));
  return UM_OK;
}

// Probe kernel: one CTA per SM holding the maximum shared memory (as K1's
// persistent grid does), every CTA spinning until *flag != 0 or ~timeout_ns;
// block 0 reports whether the flag arrived.
__global__ void ce_probe_kernel(const volatile uint32_t* flag, uint32_t* status, uint64_t timeout_ns) {
  extern __shared__ uint8_t pad[];
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  uint32_t v = 0;
  for (;;) {
    v = *flag;
    if (v) break;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) break;
    __nanosleep(1000);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *status = v ? 1u : 2u;
    pad[0] = 0;
  }
}

extern "C" int um_ce_probe(int32_t dst_device, int32_t src_device, int32_t* ok) {
  // Can a pull from src_device into dst_device (um_get_ce) complete while a
  // persistent kernel holds every SM of dst_device?  Only then may a running
  // K1 wait for it on an arrival flag (get_engine "auto").  Answered once per
  // device pair by running exactly that: a max-shared-memory CTA per SM
  // spinning on a flag that the pull's stream sets after a 2-D copy the size
  // of a staged band (the driver may use SM copy kernels for some copies, e.g.
  // same-device 2-D copies -- then the probe times out after 0.5 s, no hang).
  if (!ok) return fail(UM_EVALUE, "null out pointer");
  *ok = 0;
  static std::mutex mu;
  static std::map<std::pair<int, int>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair((int)dst_device, (int)src_device);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *ok = it->second;
    return UM_OK;
  }
  DeviceGuard g(dst_device);
  // a strided slice (2048 rows of 8 KiB) and a contiguous 64 MiB block: both
  // shapes the staging pulls take
  const size_t rows = 8192, row_bytes = 8192, pitch = 8192;
  void *src = nullptr, *dst = nullptr;
  uint32_t* words = nullptr;
  cudaStream_t s_spin = nullptr, s_copy = nullptr;
  int result = 0;
  int sms = 0, max_smem = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dst_device);
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dst_device);
  auto cleanup = [&]() {
    if (s_spin) cudaStreamDestroy(s_spin);
    if (s_copy) cudaStreamDestroy(s_copy);
    if (words) cudaFree(words);
    if (dst) cudaFree(dst);
    if (src) {
      DeviceGuard gs(src_device);
      cudaFree(src);
    }
  };
  {
    DeviceGuard gs(src_device);
    if (cudaMalloc(&src, rows * pitch) != cudaSuccess) {
      cleanup();
      return fail(UM_ECUDA, "um_ce_probe: allocation failed");
    }
  }
  if (cudaMalloc(&dst, rows * pitch) != cudaSuccess || cudaMalloc(&words, 64) != cudaSuccess ||
      cudaMemset(words, 0, 64) != cudaSuccess || cudaStreamCreateWithFlags(&s_spin, cudaStreamNonBlocking) ||
      cudaStreamCreateWithFlags(&s_copy, cudaStreamNonBlocking) ||
      cudaFuncSetAttribute(ce_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem)) {
    cleanup();
    cudaGetLastError();
    return fail(UM_ECUDA, "um_ce_probe: setup failed");
  }
  cudaDeviceSynchronize();
  ce_probe_kernel<<<sms, 128, max_smem, s_spin>>>(words, words + 1, 500000000ull);
  // the pull is queued only after the spinners hold the SMs
  struct timespec ts = {0, 20 * 1000 * 1000};
  nanosleep(&ts, nullptr);
  um_view sv = {src, 0, (int64_t)rows, 0, (int64_t)(row_bytes / 2), (int64_t)(pitch / 2), UM_BF16, src_device};
  um_view dv = {dst, 0, (int64_t)rows, 0, (int64_t)(row_bytes / 2), (int64_t)(pitch / 2), UM_BF16, dst_device};
  um_view ss = {src, 0, 2048, 0, 4096 - 256, 4096, UM_BF16, src_device};
  um_view ds = {dst, 0, 2048, 0, 4096 - 256, 4096, UM_BF16, dst_device};
  int rc = um_get_ce(&sv, &dv, s_copy);
  if (rc == UM_OK) rc = um_get_ce(&ss, &ds, s_copy);
  if (rc == UM_OK) rc = um_signal(words, 1, s_copy);
  cudaDeviceSynchronize();
  uint32_t status = 0;
  cudaMemcpy(&status, words + 1, 4, cudaMemcpyDeviceToHost);
  const cudaError_t e = cudaGetLastError();
  result = (rc == UM_OK && e == cudaSuccess && status == 1) ? 1 : 0;
  cleanup();
  cache[key] = result;
  *ok = result;
  return UM_OK;
}

extern "C" int um_copy(const um_view* src, const um_view* dst, void* stream) { return um_get(src, dst, stream); }
// cuStreamWriteValue32 through the runtime's driver entry point (no libcuda link).
typedef CUresult (*StreamWriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static StreamWriteValue32Fn stream_write_fn() {
  static StreamWriteValue32Fn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<StreamWriteValue32Fn>(p);
  });
  return fn;
}

typedef CUresult (*StreamWaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static StreamWaitValue32Fn stream_wait_fn() {
  static StreamWaitValue32Fn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<StreamWaitValue32Fn>(p);
  });
  return fn;
}

extern "C" int um_wait_geq(const uint32_t* flag, uint32_t value, void* stream) {
  if (!flag) return fail(UM_EVALUE, "null flag");
  if ((reinterpret_cast<uintptr_t>(flag) & 3) != 0) return fail(UM_EVALUE, "flag must be 4-byte aligned");
  StreamWaitValue32Fn fn = stream_wait_fn();
  if (!fn) return fail(UM_ECUDA, "cuStreamWaitValue32 unavailable");
  CUresult r = fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value,
                  CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return fail(UM_ECUDA, "cuStreamWaitValue32 failed (code " + std::to_string((int)r) + ")");
  return UM_OK;
}

extern "C" int um_signal_supported(int32_t device, int32_t* out) {
  if (!out) return fail(UM_EVALUE, "null out pointer");
  (void)device;  // 32-bit stream memory operations are core functionality since CUDA 12
  *out = stream_write_fn() ? 1 : 0;
  return UM_OK;
}

extern "C" int um_signal(uint32_t* flag, uint32_t value, void* stream) {
  if (!flag) return fail(UM_EVALUE, "null flag");
  if ((reinterpret_cast<uintptr_t>(flag) & 3) != 0) return fail(UM_EVALUE, "flag must be 4-byte aligned");
  StreamWriteValue32Fn fn = stream_write_fn();
  if (!fn) return fail(UM_ECUDA, "cuStreamWriteValue32 unavailable");
  CUresult r = fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value,
                  CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) return fail(UM_ECUDA, "cuStreamWriteValue32 failed (code " + std::to_string((int)r) + ")");
  return UM_OK;
}


extern "C" int um_accumulate(const um_view* src, const um_view* dst, void* stream) {
  int rc;
  if ((rc = check_view(src, "src", false)) || (rc = check_view(dst, "dst", false))) return rc;
  if (src->dtype != UM_F32 || dst->dtype != UM_F32) return fail(UM_ECONTRACT, "accumulate expects fp32");
  if (view_rows(*src) != view_rows(*dst) || view_cols(*src) != view_cols(*dst))
    return fail(UM_ECONTRACT, "accumulate: payload shape does not match slice");
  const int64_t rows = view_rows(*src), cols = view_cols(*src);
  if (rows == 0 || cols == 0) return UM_OK;
  const float* s = static_cast<const float*>(src->base) + src->row_lo * src->pitch + src->col_lo;
  float* d = static_cast<float*>(dst->base) + dst->row_lo * dst->pitch + dst->col_lo;
  const int vec = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15) == 0 &&
                  src->pitch % 4 == 0 && dst->pitch % 4 == 0 && cols % 4 == 0;
  const int dev = current_device();
  const int64_t groups = vec ? cols / 4 : cols;
  const int64_t gx = (groups + 255) / 256;
  const int64_t gy = std::max<int64_t>(1, std::min<int64_t>(rows, std::min<int64_t>(65535, ((int64_t)num_sms(dev) * 8 + gx - 1) / gx)));
  accumulate_kernel<<<dim3((unsigned)gx, (unsigned)gy, 1), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      s, src->pitch, d, dst->pitch, rows, cols, vec);
  UM_CUDA_CHECK(cudaGetLastError());
  return UM_OK;
}

namespace um {
int nvls_reduce(const um_view* dst, const um_view* mc_view, void* stream);   // symmem.cu
}

extern "C" int um_reduce_replicas(const um_view* dst, const um_view* srcs, int32_t nsrc, int32_t mode,
                                  void* stream) {
  int rc;
  if ((rc = check_view(dst, "dst", false))) return rc;
  if (dst->dtype != UM_F32) return fail(UM_ECONTRACT, "reduce expects fp32");
  if (nsrc < 0) return fail(UM_EVALUE, "negative source count");
  if (mode == UM_REDUCE_NCCL)
    return fail(UM_ECONFIG, "UM_REDUCE_NCCL is a collective over the replica owners: the host drives it through "
                            "its NCCL communicator (replicas.reduce_replicas(mode='nccl'))");
  if (mode == UM_REDUCE_NVLS) {
    if (nsrc != 1 || !srcs) return fail(UM_EVALUE, "UM_REDUCE_NVLS takes exactly one source: the multicast view");
    if ((rc = check_view(&srcs[0], "multicast view", false))) return rc;
    return nvls_reduce(dst, &srcs[0], stream);
  }
  if (mode != UM_REDUCE_PEER) return fail(UM_EVALUE, "unknown reduce mode " + std::to_string(mode));
  const int64_t rows = view_rows(*dst), cols = view_cols(*dst);
  if (rows == 0 || cols == 0 || nsrc == 0) return UM_OK;
  float* d = static_cast<float*>(dst->base) + dst->row_lo * dst->pitch + dst->col_lo;
  bool vec = (reinterpret_cast<uintptr_t>(d) & 15) == 0 && dst->pitch % 4 == 0 && cols % 4 == 0;
  const int dev = current_device();
  // Sources are consumed in chunks of 16, keeping the in-order sum per chunk;
  // chunk partials are folded into dst in order (exact for integer inputs).
  for (int base = 0; base < nsrc; base += 16) {
    SrcList sl;
    const int n = std::min(16, nsrc - base);
    for (int i = 0; i < n; ++i) {
      const um_view& s = srcs[base + i];
      if ((rc = check_view(&s, "src", false))) return rc;
      if (s.dtype != UM_F32 || view_rows(s) != rows || view_cols(s) != cols)
        return fail(UM_ECONTRACT, "reduce: replica slice shape mismatch");
      sl.ptr[i] = static_cast<const float*>(s.base) + s.row_lo * s.pitch + s.col_lo;
      sl.pitch[i] = s.pitch;
      vec = vec && (reinterpret_cast<uintptr_t>(sl.ptr[i]) & 15) == 0 && s.pitch % 4 == 0;
    }
    if (vec)
      reduce_kernel<4><<<reduce_grid(rows, cols / 4, num_sms(dev)), RED_THREADS, 0,
                         reinterpret_cast<cudaStream_t>(stream)>>>(sl, n, d, dst->pitch, rows, cols);
    else
      reduce_kernel<1><<<reduce_grid(rows, cols, num_sms(dev)), RED_THREADS, 0,
                         reinterpret_cast<cudaStream_t>(stream)>>>(sl, n, d, dst->pitch, rows, cols);
    UM_CUDA_CHECK(cudaGetLastError());
  }
  return UM_OK;
}

extern "C" int um_fill(const um_view* dst, int64_t grow0, int64_t gcol0, uint64_t seed, int32_t mode, void* stream) {
  int rc;
  if ((rc = check_view(dst, "dst", false))) return rc;
  if (mode != UM_FILL_ZERO && mode != UM_FILL_INT && mode != UM_FILL_REAL) return fail(UM_EVALUE, "bad fill mode");
  const int64_t rows = view_rows(*dst), cols = view_cols(*dst);
  if (rows == 0 || cols == 0) return UM_OK;
  const int dev = current_device();
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (dst->dtype == UM_BF16) {
    __nv_bfloat16* p = static_cast<__nv_bfloat16*>(dst->base) + dst->row_lo * dst->pitch + dst->col_lo;
    fill_kernel<__nv_bfloat16><<<grid_for(rows * cols, dev), 256, 0, st>>>(p, dst->pitch, rows, cols, grow0, gcol0,
                                                                            seed, mode);
  } else {
    float* p = static_cast<float*>(dst->base) + dst->row_lo * dst->pitch + dst->col_lo;
    fill_kernel<float><<<grid_for(rows * cols, dev), 256, 0, st>>>(p, dst->pitch, rows, cols, grow0, gcol0, seed,
                                                                    mode);
  }
  UM_CUDA_CHECK(cudaGetLastError());
  return UM_OK;
}

// ------------------------------------------------------------------ runtime

extern "C" int um_init(int32_t ndev, const int32_t* devices) {
  if (ndev < 0 || (ndev > 0 && !devices)) return fail(UM_EVALUE, "bad device list");
  int prev = 0;
  cudaGetDevice(&prev);
  for (int i = 0; i < ndev; ++i) {
    UM_CUDA_CHECK(cudaSetDevice(devices[i]));
    for (int j = 0; j < ndev; ++j) {
      if (devices[j] == devices[i]) continue;
      int can = 0;
      UM_CUDA_CHECK(cudaDeviceCanAccessPeer(&can, devices[i], devices[j]));
      if (!can) {
        cudaSetDevice(prev);
        return fail(UM_ECUDA, "device " + std::to_string(devices[i]) + " cannot access peer " +
                                  std::to_string(devices[j]));
      }
      cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (e != cudaSuccess) {
        cudaSetDevice(prev);
        return fail(UM_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
      }
    }
  }
  cudaSetDevice(prev);
  return UM_OK;
}

extern "C" int um_device_alloc(int32_t device, uint64_t bytes, void** ptr) {
  if (!ptr) return fail(UM_EVALUE, "null out pointer");
  int prev = 0;
  cudaGetDevice(&prev);
  UM_CUDA_CHECK(cudaSetDevice(device));
  cudaError_t e = cudaMalloc(ptr, bytes ? bytes : 256);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return fail(UM_ECUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  return UM_OK;
}

extern "C" int um_device_free(int32_t device, void* ptr) {
  int prev = 0;
  cudaGetDevice(&prev);
  UM_CUDA_CHECK(cudaSetDevice(device));
  cudaError_t e = cudaFree(ptr);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return fail(UM_ECUDA, std::string("cudaFree: ") + cudaGetErrorString(e));
  return UM_OK;
}

extern "C" int um_ipc_get_handle(void* ptr, void* handle_out) {
  if (!handle_out) return fail(UM_EVALUE, "null handle buffer");
  cudaIpcMemHandle_t h;
  UM_CUDA_CHECK(cudaIpcGetMemHandle(&h, ptr));
  static_assert(sizeof(h) <= UM_IPC_HANDLE_BYTES, "IPC handle size");
  memset(handle_out, 0, UM_IPC_HANDLE_BYTES);
  memcpy(handle_out, &h, sizeof(h));
  return UM_OK;
}

extern "C" int um_ipc_open_handle(const void* handle, int32_t device, void** ptr_out) {
  if (!handle || !ptr_out) return fail(UM_EVALUE, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  int prev = 0;
  cudaGetDevice(&prev);
  UM_CUDA_CHECK(cudaSetDevice(device));
  cudaError_t e = cudaIpcOpenMemHandle(ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return fail(UM_ECUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
  return UM_OK;
}

extern "C" int um_ipc_close_handle(void* ptr) {
  UM_CUDA_CHECK(cudaIpcCloseMemHandle(ptr));
  return UM_OK;
}

extern "C" int um_device_count(int32_t* n) {
  if (!n) return fail(UM_EVALUE, "null out pointer");
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    cudaGetLastError();
    c = 0;
  }
  *n = c;
  return UM_OK;
}

extern "C" int um_sm_count(int32_t device, int32_t* n) {
  if (!n) return fail(UM_EVALUE, "null out pointer");
  int v = 0;
  UM_CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  *n = v;
  return UM_OK;
}

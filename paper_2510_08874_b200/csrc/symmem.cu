// Symmetric memory through the CUDA VMM API, and K4's NVLS mode.
//
//  um_sym_alloc / um_sym_free   <- the paper's pre-registered symmetric pool
//                                  (PAPER.md:208-210), which the reference
//                                  simulates with one array per segment
//                                  (fabric.py:147-150)
//  um_nvls_team_*               <- a multicast object over the replica owners
//                                  of one C tile (distmatrix.py:211-232)
//  um_reduce_replicas mode NVLS <- reduce_replicas as one multimem.ld_reduce
//                                  per 16 bytes: NVSwitch adds the c replicas
//                                  in the switch, the origin stores the sum
//
// Allocations are cuMemCreate'd physical memory (exportable as a POSIX file
// descriptor), mapped read/write for every device that can reach the owner,
// at the multicast granularity so they can be bound to a multicast object.
// Driver entry points are resolved through cudaGetDriverEntryPoint (the
// library links only the static runtime; no -lcuda).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "um_internal.h"

namespace um {

namespace {

struct Drv {
  decltype(&cuMemCreate) memCreate = nullptr;
  decltype(&cuMemRelease) memRelease = nullptr;
  decltype(&cuMemAddressReserve) addrReserve = nullptr;
  decltype(&cuMemAddressFree) addrFree = nullptr;
  decltype(&cuMemMap) memMap = nullptr;
  decltype(&cuMemUnmap) memUnmap = nullptr;
  decltype(&cuMemSetAccess) setAccess = nullptr;
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  decltype(&cuDeviceGetAttribute) devAttr = nullptr;
  decltype(&cuDeviceGet) devGet = nullptr;
  decltype(&cuMulticastCreate) mcCreate = nullptr;
  decltype(&cuMulticastAddDevice) mcAddDevice = nullptr;
  decltype(&cuMulticastBindMem) mcBindMem = nullptr;
  decltype(&cuMulticastUnbind) mcUnbind = nullptr;
  decltype(&cuMulticastGetGranularity) mcGranularity = nullptr;
  decltype(&cuGetErrorString) errString = nullptr;
  bool ok = false;
};

template <typename F>
static void resolve(const char* name, F& fn, bool& ok) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
    fn = reinterpret_cast<F>(p);
  else
    ok = false;
}

static const Drv& drv() {
  static Drv d;
  static std::once_flag once;
  std::call_once(once, [] {
    bool ok = true;
    resolve("cuMemCreate", d.memCreate, ok);
    resolve("cuMemRelease", d.memRelease, ok);
    resolve("cuMemAddressReserve", d.addrReserve, ok);
    resolve("cuMemAddressFree", d.addrFree, ok);
    resolve("cuMemMap", d.memMap, ok);
    resolve("cuMemUnmap", d.memUnmap, ok);
    resolve("cuMemSetAccess", d.setAccess, ok);
    resolve("cuMemGetAllocationGranularity", d.granularity, ok);
    resolve("cuDeviceGetAttribute", d.devAttr, ok);
    resolve("cuDeviceGet", d.devGet, ok);
    resolve("cuGetErrorString", d.errString, ok);
    d.ok = ok;
    // multicast entry points are optional (capability, not a load failure)
    bool mc = true;
    resolve("cuMulticastCreate", d.mcCreate, mc);
    resolve("cuMulticastAddDevice", d.mcAddDevice, mc);
    resolve("cuMulticastBindMem", d.mcBindMem, mc);
    resolve("cuMulticastUnbind", d.mcUnbind, mc);
    resolve("cuMulticastGetGranularity", d.mcGranularity, mc);
    if (!mc) d.mcCreate = nullptr;
  });
  return d;
}

static int cu_fail(const char* what, CUresult r) {
  const char* s = nullptr;
  if (drv().errString) drv().errString(r, &s);
  return fail(UM_ECUDA, std::string(what) + " failed: " + (s ? s : std::to_string((int)r)));
}

#define UM_CU_CHECK(expr)                         \
  do {                                            \
    CUresult _r = (expr);                         \
    if (_r != CUDA_SUCCESS) return cu_fail(#expr, _r); \
  } while (0)

struct SymAlloc {
  CUmemGenericAllocationHandle handle;
  size_t size;
  int device;
};

std::mutex g_mu;
std::map<uintptr_t, SymAlloc> g_allocs;   // mapped base -> allocation

static CUmemAllocationProp alloc_prop(int device) {
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return prop;
}

static int granularity_of(int device, size_t* g) {
  const Drv& d = drv();
  if (!d.ok) return fail(UM_ECUDA, "CUDA VMM driver entry points unavailable");
  CUmemAllocationProp prop = alloc_prop(device);
  UM_CU_CHECK(d.granularity(g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  // multicast binding needs the multicast granularity too (2 MiB on B200)
  if (d.mcGranularity) {
    CUmulticastObjectProp mp = {};
    mp.numDevices = 1;
    mp.size = *g;
    mp.handleTypes = 0;
    size_t mg = 0;
    if (d.mcGranularity(&mg, &mp, CU_MULTICAST_GRANULARITY_MINIMUM) == CUDA_SUCCESS && mg > *g) *g = mg;
  }
  return UM_OK;
}

// ---- NVLS team: one multicast object over the replica owners' allocations

struct Team {
  CUmemGenericAllocationHandle mc;
  size_t size;
  std::vector<int> devices;
  std::vector<CUdeviceptr> mc_va;     // multicast VA mapped on each device
};

__global__ void nvls_reduce_kernel(const float* __restrict__ mc, int64_t mc_pitch, float* __restrict__ dst,
                                   int64_t dst_pitch, int64_t rows, int64_t groups) {
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const float* src_row = mc + r * mc_pitch;
    float* dst_row = dst + r * dst_pitch;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
      float4 v;
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                   : "l"(src_row + 4 * g)
                   : "memory");
      reinterpret_cast<float4*>(dst_row)[g] = v;
    }
  }
}

}  // namespace

int nvls_reduce(const um_view* dst, const um_view* mc_view, void* stream) {
  const int64_t rows = view_rows(*dst), cols = view_cols(*dst);
  if (view_rows(*mc_view) != rows || view_cols(*mc_view) != cols || mc_view->dtype != UM_F32)
    return fail(UM_ECONTRACT, "nvls reduce: multicast slice shape mismatch");
  if (rows == 0 || cols == 0) return UM_OK;
  float* d = static_cast<float*>(dst->base) + dst->row_lo * dst->pitch + dst->col_lo;
  const float* m = static_cast<const float*>(mc_view->base) + mc_view->row_lo * mc_view->pitch + mc_view->col_lo;
  if ((reinterpret_cast<uintptr_t>(d) | reinterpret_cast<uintptr_t>(m)) & 15 || cols % 4 || dst->pitch % 4 ||
      mc_view->pitch % 4)
    return fail(UM_ECONTRACT, "nvls reduce needs 16-byte aligned rows (multimem.ld_reduce.v4)");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t groups = cols / 4;
  const unsigned gx = (unsigned)std::min<int64_t>((groups + 255) / 256, 64);
  const unsigned gy = (unsigned)std::max<int64_t>(1, std::min<int64_t>(rows, (int64_t)sms * 8 / gx));
  nvls_reduce_kernel<<<dim3(gx, gy, 1), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      m, mc_view->pitch, d, dst->pitch, rows, groups);
  UM_CUDA_CHECK(cudaGetLastError());
  return UM_OK;
}

}  // namespace um

using namespace um;

extern "C" int um_sym_granularity(int32_t device, uint64_t* bytes) {
  if (!bytes) return fail(UM_EVALUE, "null out pointer");
  size_t g = 0;
  int rc = granularity_of(device, &g);
  if (rc) return rc;
  *bytes = g;
  return UM_OK;
}

extern "C" int um_sym_alloc(int32_t device, uint64_t bytes, void** ptr) {
  if (!ptr) return fail(UM_EVALUE, "null out pointer");
  const Drv& d = drv();
  size_t g = 0;
  int rc = granularity_of(device, &g);
  if (rc) return rc;
  const size_t size = ((bytes ? bytes : 1) + g - 1) / g * g;
  CUmemAllocationProp prop = alloc_prop(device);
  CUmemGenericAllocationHandle h;
  CUresult r = d.memCreate(&h, size, &prop, 0);
  if (r != CUDA_SUCCESS) {
    // some drivers reject the POSIX-fd request type: retry without export
    prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_NONE;
    UM_CU_CHECK(d.memCreate(&h, size, &prop, 0));
  }
  CUdeviceptr va = 0;
  r = d.addrReserve(&va, size, g, 0, 0);
  if (r != CUDA_SUCCESS) {
    d.memRelease(h);
    return cu_fail("cuMemAddressReserve", r);
  }
  r = d.memMap(va, size, 0, h, 0);
  if (r != CUDA_SUCCESS) {
    d.addrFree(va, size);
    d.memRelease(h);
    return cu_fail("cuMemMap", r);
  }
  // read/write for the owner and every device that can reach it over NVLink
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  std::vector<CUmemAccessDesc> acc;
  for (int j = 0; j < ndev; ++j) {
    int can = j == device;
    if (!can) cudaDeviceCanAccessPeer(&can, j, device);
    if (!can) continue;
    CUmemAccessDesc a = {};
    a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    a.location.id = j;
    a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    acc.push_back(a);
  }
  r = d.setAccess(va, size, acc.data(), acc.size());
  if (r != CUDA_SUCCESS) {
    d.memUnmap(va, size);
    d.addrFree(va, size);
    d.memRelease(h);
    return cu_fail("cuMemSetAccess", r);
  }
  {
    std::lock_guard<std::mutex> lk(g_mu);
    g_allocs[(uintptr_t)va] = {h, size, device};
  }
  *ptr = reinterpret_cast<void*>(va);
  return UM_OK;
}

extern "C" int um_sym_free(void* ptr) {
  SymAlloc a;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_allocs.find((uintptr_t)ptr);
    if (it == g_allocs.end()) return fail(UM_EVALUE, "um_sym_free: not a um_sym_alloc base");
    a = it->second;
    g_allocs.erase(it);
  }
  const Drv& d = drv();
  cudaDeviceSynchronize();
  d.memUnmap((CUdeviceptr)ptr, a.size);
  d.addrFree((CUdeviceptr)ptr, a.size);
  d.memRelease(a.handle);
  return UM_OK;
}

extern "C" int um_nvls_supported(int32_t device, int32_t* ok) {
  // The device attribute alone is not enough: a box whose NVSwitch fabric is
  // not configured for multicast (no fabric manager / IMEX in this container)
  // reports CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 1 and then refuses
  // cuMulticastCreate.  So the probe also creates (and releases) a minimal
  // multicast object once per device.
  if (!ok) return fail(UM_EVALUE, "null out pointer");
  *ok = 0;
  const Drv& d = drv();
  if (!d.ok || !d.mcCreate || device < 0 || device >= 64) return UM_OK;
  static std::mutex mu;
  static int cache[64];
  static bool init = false;
  std::lock_guard<std::mutex> lk(mu);
  if (!init) {
    for (int& c : cache) c = -1;
    init = true;
  }
  if (cache[device] >= 0) {
    *ok = cache[device];
    return UM_OK;
  }
  cache[device] = 0;
  CUdevice dev;
  if (d.devGet(&dev, device) != CUDA_SUCCESS) return UM_OK;
  int v = 0;
  if (d.devAttr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS || !v) return UM_OK;
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  size_t mg = 0;
  mp.size = 2 << 20;
  if (d.mcGranularity(&mg, &mp, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS) return UM_OK;
  mp.size = mg;
  CUmemGenericAllocationHandle h;
  if (d.mcCreate(&h, &mp) != CUDA_SUCCESS) return UM_OK;
  d.memRelease(h);
  cache[device] = 1;
  *ok = 1;
  return UM_OK;
}

extern "C" int um_nvls_team_create(int32_t ndev, const int32_t* devices, void* const* sym_ptrs, uint64_t bytes,
                                   void** mc_ptrs_out, void** team_out) {
  if (ndev < 1 || !devices || !sym_ptrs || !mc_ptrs_out || !team_out) return fail(UM_EVALUE, "bad arguments");
  int32_t ok = 0;
  um_nvls_supported(devices[0], &ok);
  if (!ok) return fail(UM_ECONFIG, "NVLS multicast is not supported on this device / driver");
  for (int i = 0; i < ndev; ++i)
    for (int j = i + 1; j < ndev; ++j)
      if (devices[i] == devices[j]) return fail(UM_ECONFIG, "an NVLS team needs distinct devices");
  const Drv& d = drv();
  std::vector<SymAlloc> allocs(ndev);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (int i = 0; i < ndev; ++i) {
      auto it = g_allocs.find((uintptr_t)sym_ptrs[i]);
      if (it == g_allocs.end()) return fail(UM_EVALUE, "NVLS team members must be um_sym_alloc bases");
      if (it->second.device != devices[i]) return fail(UM_EVALUE, "team member allocated on another device");
      if (it->second.size < bytes) return fail(UM_EVALUE, "team member smaller than the team size");
      allocs[i] = it->second;
    }
  }
  CUmulticastObjectProp mp = {};
  mp.numDevices = (unsigned)ndev;
  mp.handleTypes = 0;           // one process: the multicast handle is not exported
  size_t mg = 0;
  mp.size = bytes;
  UM_CU_CHECK(d.mcGranularity(&mg, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  mp.size = (bytes + mg - 1) / mg * mg;
  for (int i = 0; i < ndev; ++i)
    if (allocs[i].size < mp.size) return fail(UM_EVALUE, "team member smaller than the multicast granularity");
  Team* T = new Team();
  T->size = mp.size;
  T->devices.assign(devices, devices + ndev);
  CUresult r = d.mcCreate(&T->mc, &mp);
  if (r == CUDA_ERROR_INVALID_VALUE) {     // some drivers want an exportable handle type
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    r = d.mcCreate(&T->mc, &mp);
  }
  if (r != CUDA_SUCCESS) {
    delete T;
    return cu_fail("cuMulticastCreate", r);
  }
  for (int i = 0; i < ndev; ++i) {
    CUdevice dev;
    d.devGet(&dev, devices[i]);
    r = d.mcAddDevice(T->mc, dev);
    if (r != CUDA_SUCCESS) {
      d.memRelease(T->mc);
      delete T;
      return cu_fail("cuMulticastAddDevice", r);
    }
  }
  for (int i = 0; i < ndev; ++i) {
    r = d.mcBindMem(T->mc, 0, allocs[i].handle, 0, mp.size, 0);
    if (r != CUDA_SUCCESS) {
      d.memRelease(T->mc);
      delete T;
      return cu_fail("cuMulticastBindMem", r);
    }
  }
  size_t g = 0;
  granularity_of(devices[0], &g);
  for (int i = 0; i < ndev; ++i) {
    CUdeviceptr va = 0;
    r = d.addrReserve(&va, mp.size, std::max(g, mg), 0, 0);
    if (r == CUDA_SUCCESS) r = d.memMap(va, mp.size, 0, T->mc, 0);
    if (r == CUDA_SUCCESS) {
      CUmemAccessDesc a = {};
      a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      a.location.id = devices[i];
      a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
      r = d.setAccess(va, mp.size, &a, 1);
    }
    if (r != CUDA_SUCCESS) {
      for (CUdeviceptr v : T->mc_va) {
        d.memUnmap(v, mp.size);
        d.addrFree(v, mp.size);
      }
      d.memRelease(T->mc);
      delete T;
      return cu_fail("multicast mapping", r);
    }
    T->mc_va.push_back(va);
    mc_ptrs_out[i] = reinterpret_cast<void*>(va);
  }
  *team_out = T;
  return UM_OK;
}

extern "C" int um_nvls_team_destroy(void* team) {
  if (!team) return UM_OK;
  Team* T = static_cast<Team*>(team);
  const Drv& d = drv();
  cudaDeviceSynchronize();
  for (CUdeviceptr v : T->mc_va) {
    d.memUnmap(v, T->size);
    d.addrFree(v, T->size);
  }
  for (int dev : T->devices) {
    CUdevice cd;
    d.devGet(&cd, dev);
    d.mcUnbind(T->mc, cd, 0, T->size);
  }
  d.memRelease(T->mc);
  delete T;
  return UM_OK;
}

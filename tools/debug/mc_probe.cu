// Probe which cuMulticastCreate arguments this box's driver accepts.
#include <cuda.h>
#include <cstdio>
int main() {
  cuInit(0);
  CUdevice dev; cuDeviceGet(&dev, 0);
  CUcontext ctx; cuDevicePrimaryCtxRetain(&ctx, dev); cuCtxSetCurrent(ctx);
  int sup = 0; cuDeviceGetAttribute(&sup, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  int fab = 0; cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  printf("multicast supported %d, fabric handles %d\n", sup, fab);
  unsigned long long types[] = {0, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_FABRIC};
  for (int nd = 1; nd <= 2; ++nd)
    for (auto t : types)
      for (size_t sz : {(size_t)2 << 20, (size_t)512 << 20}) {
        CUmulticastObjectProp p = {};
        p.numDevices = nd; p.size = sz; p.handleTypes = t;
        size_t g1 = 0, g2 = 0;
        CUresult rg = cuMulticastGetGranularity(&g1, &p, CU_MULTICAST_GRANULARITY_MINIMUM);
        cuMulticastGetGranularity(&g2, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED);
        CUmemGenericAllocationHandle h;
        CUresult r = cuMulticastCreate(&h, &p);
        const char* s = nullptr; cuGetErrorString(r, &s);
        printf("numDevices %d handleTypes %llu size %zu: gran rc %d min %zu rec %zu -> create %d (%s)\n", nd, t, sz,
               (int)rg, g1, g2, (int)r, s);
        if (r == CUDA_SUCCESS) {
          CUresult ra = cuMulticastAddDevice(h, dev);
          cuGetErrorString(ra, &s);
          printf("   add device 0 -> %d (%s)\n", (int)ra, s);
          cuMemRelease(h);
        }
      }
  return 0;
}

// Does this GPU support NVLS multicast objects (cuMulticast*)?  One-device probe.
#include <cuda.h>
#include <cstdio>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("%s -> %s\n", #x, s); return 1; } } while (0)
int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  int mc = -1, fabric = -1, posix = -1;
  cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  cuDeviceGetAttribute(&fabric, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  cuDeviceGetAttribute(&posix, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev);
  printf("multicast_supported=%d fabric_handles=%d posix_fd_handles=%d\n", mc, fabric, posix);
  if (mc != 1) return 0;
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  CUmulticastObjectProp prop = {};
  size_t gran = 0;
  CUmemGenericAllocationHandle mch;
  const CUmemAllocationHandleType types[3] = {CU_MEM_HANDLE_TYPE_NONE, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                              CU_MEM_HANDLE_TYPE_FABRIC};
  bool made = false;
  for (int nd = 1; nd <= 2 && !made; ++nd)
    for (int t = 0; t < 3 && !made; ++t) {
      prop = {};
      prop.numDevices = nd;
      prop.handleTypes = types[t];
      prop.size = 2 << 20;
      CUresult rg = cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
      if (rg == CUDA_SUCCESS) prop.size = ((prop.size + gran - 1) / gran) * gran;
      CUresult r = cuMulticastCreate(&mch, &prop);
      const char* es = "";
      cuGetErrorString(r, &es);
      printf("numDevices=%d handleType=%d gran=%zu (rc %d) -> create: %s\n", nd, (int)types[t], gran, (int)rg, es);
      made = r == CUDA_SUCCESS && nd == 1;
    }
  if (!made) return 0;
  CK(cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle mem;
  CK(cuMemCreate(&mem, prop.size, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, mem, 0, prop.size, 0));
  CUdeviceptr mcva;
  CK(cuMemAddressReserve(&mcva, prop.size, gran, 0, 0));
  CK(cuMemMap(mcva, prop.size, 0, mch, 0));
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE; acc.location.id = 0; acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(mcva, prop.size, &acc, 1));
  printf("multicast object of %zu bytes bound and mapped (granularity %zu)\n", prop.size, gran);
  return 0;
}

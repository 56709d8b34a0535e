// Step-by-step check of the multicast (NVLS) driver path on the current GPU:
// which call fails, with which CUresult.  nvcc -o mc_selftest mc_selftest.cu -lcuda
#include <cuda.h>
#include <cstdio>

#define STEP(x)                                                       \
  do {                                                                \
    CUresult r_ = (x);                                                \
    const char* s_ = nullptr;                                         \
    cuGetErrorName(r_, &s_);                                          \
    printf("%-70s -> %d %s\n", #x, (int)r_, s_ ? s_ : "?");           \
    if (r_ != CUDA_SUCCESS) return 1;                                 \
  } while (0)

int run(CUmemAllocationHandleType ht, size_t want) {
  CUdevice dev;
  STEP(cuDeviceGet(&dev, 0));
  int v = 0;
  STEP(cuDeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  printf("multicast supported %d, handle type %d\n", v, (int)ht);
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  mp.size = want;
  mp.handleTypes = ht;
  size_t gmc = 0, gmin = 0, gmem = 0;
  STEP(cuMulticastGetGranularity(&gmc, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  STEP(cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = ht;
  STEP(cuMemGetAllocationGranularity(&gmem, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  printf("granularity mc %zu (min %zu) mem %zu\n", gmc, gmin, gmem);
  size_t g = gmc > gmem ? gmc : gmem, size = (want + g - 1) / g * g;
  mp.size = size;
  CUmemGenericAllocationHandle mem, mc;
  STEP(cuMemCreate(&mem, size, &ap, 0));
  STEP(cuMulticastCreate(&mc, &mp));
  STEP(cuMulticastAddDevice(mc, dev));
  STEP(cuMulticastBindMem(mc, 0, mem, 0, size, 0));
  CUdeviceptr va, mcva;
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = 0;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  STEP(cuMemAddressReserve(&va, size, 0, 0, 0));
  STEP(cuMemMap(va, size, 0, mem, 0));
  STEP(cuMemSetAccess(va, size, &acc, 1));
  STEP(cuMemAddressReserve(&mcva, size, 0, 0, 0));
  STEP(cuMemMap(mcva, size, 0, mc, 0));
  STEP(cuMemSetAccess(mcva, size, &acc, 1));
  STEP(cuMemsetD32(va, 0x3f800000u, size / 4));
  STEP(cuCtxSynchronize());
  printf("OK handle type %d\n", (int)ht);
  cuMemUnmap(mcva, size); cuMemAddressFree(mcva, size);
  cuMemUnmap(va, size); cuMemAddressFree(va, size);
  cuMemRelease(mc); cuMemRelease(mem);
  return 0;
}

int create_only(unsigned ndev) {
  CUmulticastObjectProp mp = {};
  mp.numDevices = ndev;
  mp.size = 2 << 20;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  CUmemGenericAllocationHandle mc;
  printf("create-only numDevices=%u\n", ndev);
  STEP(cuMulticastCreate(&mc, &mp));
  cuMemRelease(mc);
  return 0;
}

int main() {
  cuInit(0);
  CUdevice dev;
  cuDeviceGet(&dev, 0);
  CUcontext ctx;
  cuDevicePrimaryCtxRetain(&ctx, dev);
  cuCtxSetCurrent(ctx);
  int a = run(CU_MEM_HANDLE_TYPE_NONE, 1 << 20);
  int b = run(CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 1 << 20);
  int c = run(CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 64 << 20);
  int d = create_only(2);
  int e = create_only(8);
  return a | b | c | d | e;
}

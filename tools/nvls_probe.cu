// nvls_probe.cu -- can this box create a CUDA multicast object (NVLS) over
// its visible GPUs, bind each GPU's memory, map the multicast address and
// reduce into it with multimem.red from a kernel?  Prints one line per step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/nvls_probe tools/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    CUresult r_ = (x);                                                     \
    if (r_ != CUDA_SUCCESS) {                                              \
      const char* s_ = nullptr;                                            \
      cuGetErrorString(r_, &s_);                                           \
      std::printf("FAIL %s -> %d %s\n", #x, static_cast<int>(r_), s_ ? s_ : ""); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

__global__ void red_kernel(float* mc, unsigned* mc_cnt, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (4 * i + 3 < n) {
    asm volatile("multimem.red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(
                     mc + 4 * i),
                 "f"(1.0f), "f"(2.0f), "f"(3.0f), "f"(4.0f)
                 : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(mc_cnt), "r"(1u)
                 : "memory");
}

int main() {
  CK(cuInit(0));
  int ndev = 0;
  CK(cuDeviceGetCount(&ndev));
  CUdevice dev0;
  CK(cuDeviceGet(&dev0, 0));
  int mc_ok = 0;
  CK(cuDeviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev0));
  std::printf("devices %d multicast_supported %d\n", ndev, mc_ok);
  if (!mc_ok) return 0;
  cudaSetDevice(0);
  cudaFree(0);
  const size_t want = 4 << 20;
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  mp.size = want;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0, rgran = 0;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  CK(cuMulticastGetGranularity(&rgran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t size = (want + gran - 1) / gran * gran;
  mp.size = size;
  std::printf("granularity min %zu recommended %zu size %zu\n", gran, rgran, size);
  CUmemGenericAllocationHandle mc;
  CUresult rc = cuMulticastCreate(&mc, &mp);
  std::printf("cuMulticastCreate(posix fd) -> %d\n", static_cast<int>(rc));
  if (rc != CUDA_SUCCESS) {
    mp.handleTypes = 0;
    rc = cuMulticastCreate(&mc, &mp);
    std::printf("cuMulticastCreate(none) -> %d\n", static_cast<int>(rc));
  }
  if (rc != CUDA_SUCCESS) {
    mp.handleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
    rc = cuMulticastCreate(&mc, &mp);
    std::printf("cuMulticastCreate(fabric) -> %d\n", static_cast<int>(rc));
  }
  if (rc != CUDA_SUCCESS) return 1;
  CK(cuMulticastAddDevice(mc, dev0));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = static_cast<CUmemAllocationHandleType>(mp.handleTypes);
  CUmemGenericAllocationHandle phys;
  CK(cuMemCreate(&phys, size, &ap, 0));
  CK(cuMulticastBindMem(mc, 0, phys, 0, size, 0));
  CUdeviceptr uva = 0, mva = 0;
  CK(cuMemAddressReserve(&uva, size, gran, 0, 0));
  CK(cuMemMap(uva, size, 0, phys, 0));
  CK(cuMemAddressReserve(&mva, size, gran, 0, 0));
  CK(cuMemMap(mva, size, 0, mc, 0));
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uva, size, &ad, 1));
  CK(cuMemSetAccess(mva, size, &ad, 1));
  cudaMemset(reinterpret_cast<void*>(uva), 0, size);
  const int n = 1024;
  red_kernel<<<n / 4 / 128, 128>>>(reinterpret_cast<float*>(mva),
                                  reinterpret_cast<unsigned*>(mva + 65536), n);
  red_kernel<<<n / 4 / 128, 128>>>(reinterpret_cast<float*>(mva),
                                  reinterpret_cast<unsigned*>(mva + 65536), n);
  cudaError_t e = cudaDeviceSynchronize();
  std::printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> h(n);
  unsigned cnt = 0;
  cudaMemcpy(h.data(), reinterpret_cast<void*>(uva), n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&cnt, reinterpret_cast<void*>(uva + 65536), 4, cudaMemcpyDeviceToHost);
  std::printf("values %g %g %g %g ... counter %u (expect 2 4 6 8, counter 4)\n", h[0], h[1], h[2],
              h[3], cnt);
  return 0;
}

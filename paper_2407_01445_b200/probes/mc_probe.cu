// mc_probe.cu -- NVLS multicast feasibility probe (not part of the library): one process, up to
// four GPUs. Creates a multicast object over the devices, binds 64 MB of physical memory from
// each, maps the multicast address on GPU 0, and has a kernel on GPU 0 write a 2.6 MB slice (one
// source of a K = 4 rank's embedding slice) with multimem.st -- one store that lands in every
// GPU's memory -- then checks every copy and times the stores against plain stores of the same
// bytes to each GPU (the peer gather's pattern).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mc_probe mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); \
  std::printf("FAIL %s: %s (line %d)\n", #x, s_, __LINE__); return 1; } } while (0)
#define RK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { std::printf("FAIL %s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void mc_store(uint4* mc, const uint4* src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = src[i];
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i),
                 "f"(__uint_as_float(v.x)), "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)), "f"(__uint_as_float(v.w))
                 : "memory");
  }
}
struct Dsts { uint4* d[4]; int n; };
__global__ void peer_store(Dsts ds, const uint4* src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = src[i];
    for (int k = 0; k < ds.n; ++k) ds.d[k][i] = v;
  }
}

int main() {
  CK(cuInit(0));
  int ndev = 0;
  RK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { std::printf("needs 2 GPUs\n"); return 0; }
  const int G = ndev < 4 ? ndev : 4;
  CUdevice dev[4];
  for (int i = 0; i < G; ++i) {
    int ok = 0;
    CK(cuDeviceGet(&dev[i], i));
    CK(cuDeviceGetAttribute(&ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev[i]));
    std::printf("GPU %d multicast supported: %d\n", i, ok);
    if (!ok) return 0;
    RK(cudaSetDevice(i));
    RK(cudaFree(0));
  }
  RK(cudaSetDevice(0));
  const size_t bytes = 64ull << 20;
  CUmulticastObjectProp mp{};
  mp.numDevices = G;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  mp.size = (bytes + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle mc;
  CK(cuMulticastCreate(&mc, &mp));
  for (int i = 0; i < G; ++i) CK(cuMulticastAddDevice(mc, dev[i]));
  CUmemGenericAllocationHandle phys[4];
  CUdeviceptr uva[4];
  for (int i = 0; i < G; ++i) {
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = i;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CK(cuMemCreate(&phys[i], mp.size, &ap, 0));
    CK(cuMulticastBindMem(mc, 0, phys[i], 0, mp.size, 0));
    CK(cuMemAddressReserve(&uva[i], mp.size, gran, 0, 0));
    CK(cuMemMap(uva[i], mp.size, 0, phys[i], 0));
    CUmemAccessDesc ads[4];
    for (int k = 0; k < G; ++k) {   // every GPU may access every copy (GPU 0 stores / reads back)
      ads[k] = CUmemAccessDesc{};
      ads[k].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      ads[k].location.id = k;
      ads[k].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    }
    CK(cuMemSetAccess(uva[i], mp.size, ads, G));
  }
  CUdeviceptr mcva;
  CK(cuMemAddressReserve(&mcva, mp.size, gran, 0, 0));
  CK(cuMemMap(mcva, mp.size, 0, mc, 0));
  CUmemAccessDesc mad{};
  mad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  mad.location.id = 0;
  mad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(mcva, mp.size, &mad, 1));

  const size_t slice = 2621440;   // bytes: 1280 rows x 1024 B (one source of a K = 4 rank's slice)
  const size_t n4 = slice / 16;
  std::vector<uint32_t> host(slice / 4);
  for (size_t i = 0; i < host.size(); ++i) host[i] = static_cast<uint32_t>(i * 2654435761u) & 0x3f7fffffu;   // finite floats
  uint4* src;
  RK(cudaMalloc(&src, slice));
  RK(cudaMemcpy(src, host.data(), slice, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  RK(cudaEventCreate(&e0));
  RK(cudaEventCreate(&e1));
  for (int rep = 0; rep < 3; ++rep) mc_store<<<148, 512>>>(reinterpret_cast<uint4*>(mcva), src, n4);
  RK(cudaDeviceSynchronize());
  RK(cudaEventRecord(e0));
  for (int rep = 0; rep < 20; ++rep) mc_store<<<148, 512>>>(reinterpret_cast<uint4*>(mcva), src, n4);
  RK(cudaEventRecord(e1));
  RK(cudaEventSynchronize(e1));
  float ms_mc = 0;
  RK(cudaEventElapsedTime(&ms_mc, e0, e1));
  bool ok = true;
  for (int i = 0; i < G; ++i) {
    std::vector<uint32_t> back(slice / 4);
    RK(cudaMemcpy(back.data(), reinterpret_cast<void*>(uva[i]), slice, cudaMemcpyDeviceToHost));
    for (size_t k = 0; k < back.size(); ++k)
      if (back[k] != host[k]) { ok = false; std::printf("mismatch on GPU %d at %zu\n", i, k); break; }
  }
  RK(cudaEventRecord(e0));
  Dsts ds{};
  ds.n = G;
  for (int k = 0; k < G; ++k) ds.d[k] = reinterpret_cast<uint4*>(uva[k]);
  for (int rep = 0; rep < 20; ++rep) peer_store<<<148, 512>>>(ds, src, n4);
  RK(cudaEventRecord(e1));
  RK(cudaEventSynchronize(e1));
  float ms_p = 0;
  RK(cudaEventElapsedTime(&ms_p, e0, e1));
  std::printf("copies %s; multimem.st of %.1f MB to %d GPUs: %.2f us (%.0f GB/s per destination); "
              "unicast stores to each: %.2f us\n", ok ? "match" : "DIFFER", slice / 1e6, G, ms_mc * 1e3 / 20,
              slice / (ms_mc * 1e-3 / 20) / 1e9, ms_p * 1e3 / 20);
  return 0;
}

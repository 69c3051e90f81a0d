// NVLS multicast all-gather probe (design experiment, not part of the product path).
// One process drives G GPUs.  A multicast object spans all G devices; each device binds its
// own `G * shard` bytes of physical memory to it.  GPU g writes ITS shard once through the
// multicast mapping (multimem.st.global.v4.f32) at offset g*shard; the NVSwitch replicates
// it into every device's buffer.  Reports per-GPU NVLink ingress ((G-1)*shard / time), the
// quantity the pull all-gather of the library is bound by, and checks the data.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mc_probe mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); exit(1);} } while (0)
#define CU(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s = 0; cuGetErrorString(r, &s); fprintf(stderr, "%s:%d %s: %d %s\n", __FILE__, __LINE__, #x, (int)r, s ? s : ""); exit(1);} } while (0)

__global__ void mc_store(const float4* __restrict__ src, float4* mc_dst, int64_t n_vec) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_vec; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = src[i];
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc_dst + i), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w) : "memory");
  }
}

__global__ void fill(float* p, int64_t n, float base) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = base + (float)(i & 1023);
}

int main(int argc, char** argv) {
  int G = argc > 1 ? atoi(argv[1]) : 4;
  int64_t mb = argc > 2 ? atoll(argv[2]) : 512;     // shard MiB per GPU
  int ctas_per_sm = argc > 3 ? atoi(argv[3]) : 4;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (G > ndev) G = ndev;
  CU(cuInit(0));
  const size_t shard = (size_t)mb << 20;
  CUmulticastObjectProp mp = {};
  mp.numDevices = G;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
  mp.size = shard * G;
  size_t gran = 0;
  CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  mp.size = (mp.size + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle mc;
  CU(cuMulticastCreate(&mc, &mp));
  for (int g = 0; g < G; ++g) {
    CUdevice dev;
    CU(cuDeviceGet(&dev, g));
    CU(cuMulticastAddDevice(mc, dev));
  }
  float* uni[8];
  float* src[8];
  CUdeviceptr mcva[8];
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaFree(0));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = g;
    size_t agran = 0;
    CU(cuMemGetAllocationGranularity(&agran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    const size_t sz = (mp.size + agran - 1) / agran * agran;
    CUmemGenericAllocationHandle mem;
    CU(cuMemCreate(&mem, sz, &ap, 0));
    CU(cuMulticastBindMem(mc, 0, mem, 0, mp.size, 0));
    CUdeviceptr va;
    CU(cuMemAddressReserve(&va, sz, agran, 0, 0));
    CU(cuMemMap(va, sz, 0, mem, 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = g;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemSetAccess(va, sz, &ad, 1));
    uni[g] = reinterpret_cast<float*>(va);
    CUdeviceptr m;
    CU(cuMemAddressReserve(&m, mp.size, gran, 0, 0));
    CU(cuMemMap(m, mp.size, 0, mc, 0));
    CU(cuMemSetAccess(m, mp.size, &ad, 1));
    mcva[g] = m;
    CK(cudaMalloc(&src[g], shard));
    fill<<<1024, 256>>>(src[g], shard / 4, 1000.0f * (g + 1));
    CK(cudaMemset(uni[g], 0, mp.size));
    CK(cudaDeviceSynchronize());
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaStream_t st[8];
  cudaEvent_t e0[8], e1[8];
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
  }
  for (int it = 0; it < 4; ++it) {
    for (int g = 0; g < G; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaEventRecord(e0[g], st[g]));
      mc_store<<<sms * ctas_per_sm, 256, 0, st[g]>>>(reinterpret_cast<const float4*>(src[g]),
                                                      reinterpret_cast<float4*>(mcva[g] + (size_t)g * shard), shard / 16);
      CK(cudaEventRecord(e1[g], st[g]));
    }
    double mn = 1e30, sum = 0;
    for (int g = 0; g < G; ++g) {
      CK(cudaSetDevice(g));
      CK(cudaEventSynchronize(e1[g]));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
      const double gbs = (double)(G - 1) * shard / (ms * 1e-3) / 1e9;   // ingress of each GPU
      mn = gbs < mn ? gbs : mn;
      sum += gbs;
    }
    printf("iter %d mode=multimem_st G=%d MB/shard=%lld ctas/sm=%d  per-GPU ingress GB/s (from own store time): min %.1f avg %.1f\n",
           it, G, (long long)mb, ctas_per_sm, mn, sum / G);
  }
  // check: GPU 0 received every shard
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceSynchronize());
  }
  CK(cudaSetDevice(0));
  int bad = 0;
  for (int h = 0; h < G; ++h) {
    float v[2];
    CK(cudaMemcpy(v, uni[0] + (size_t)h * shard / 4 + 5, 8, cudaMemcpyDeviceToHost));
    if (v[0] != 1000.0f * (h + 1) + 5 || v[1] != 1000.0f * (h + 1) + 6) bad++;
  }
  printf("check GPU0 received all %d shards: %s\n", G, bad ? "FAIL" : "ok");
  return 0;
}

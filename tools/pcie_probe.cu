// PCIe transfer probe (diagnostic): copy-engine D2H / H2D of the cfg3 image
// stack (75 x 512^2 fp32) as one copy and as 19 unit copies, against SM-driven
// transfers (a grid-stride float4 kernel storing to / loading from mapped
// pinned host memory) at several grid sizes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pcie_probe tools/pcie_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

__global__ void sm_copy(const float4* __restrict__ src, float4* __restrict__ dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int main() {
  const size_t bytes = 75ull * 512 * 512 * 4;
  float *d = nullptr, *h = nullptr, *d2 = nullptr;
  cudaMalloc(&d, bytes);
  cudaMalloc(&d2, bytes);
  cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
  cudaMemset(d, 1, bytes);
  float* hd = nullptr;
  cudaHostGetDevicePointer((void**)&hd, h, 0);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time = [&](const char* what, auto fn) {
    for (int w = 0; w < 2; ++w) fn();
    cudaEventRecord(a, st);
    for (int r = 0; r < 5; ++r) fn();
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    std::printf("%-34s %.3f ms  %.1f GB/s\n", what, ms, bytes / ms / 1e6);
  };
  time("CE D2H one copy", [&] { cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st); });
  time("CE D2H 19 copies", [&] {
    for (int u = 0; u < 19; ++u) {
      const size_t o = bytes * u / 19, e = bytes * (u + 1) / 19;
      cudaMemcpyAsync((char*)h + o, (char*)d + o, e - o, cudaMemcpyDeviceToHost, st);
    }
  });
  time("CE H2D one copy", [&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st); });
  time("CE H2D 19 copies", [&] {
    for (int u = 0; u < 19; ++u) {
      const size_t o = bytes * u / 19, e = bytes * (u + 1) / 19;
      cudaMemcpyAsync((char*)d + o, (char*)h + o, e - o, cudaMemcpyHostToDevice, st);
    }
  });
  // unit copies each followed by a stream write-value flag (the host path's publication)
  uint32_t* flags = nullptr;
  cudaMalloc(&flags, 64 * sizeof(uint32_t));
  uint32_t ep = 0;
  time("CE H2D 19 copies + write flags", [&] {
    ++ep;
    for (int u = 0; u < 19; ++u) {
      const size_t o = bytes * u / 19, e = bytes * (u + 1) / 19;
      cudaMemcpyAsync((char*)d + o, (char*)h + o, e - o, cudaMemcpyHostToDevice, st);
      cuStreamWriteValue32((CUstream)st, (CUdeviceptr)(flags + u), ep, 0);
    }
  });
  time("CE D2H 19 copies after wait flags", [&] {
    ++ep;
    for (int u = 0; u < 19; ++u) cuStreamWriteValue32((CUstream)st, (CUdeviceptr)(flags + u), ep, 0);
    for (int u = 0; u < 19; ++u) {
      const size_t o = bytes * u / 19, e = bytes * (u + 1) / 19;
      cuStreamWaitValue32((CUstream)st, (CUdeviceptr)(flags + u), ep, CU_STREAM_WAIT_VALUE_GEQ);
      cudaMemcpyAsync((char*)h + o, (char*)d + o, e - o, cudaMemcpyDeviceToHost, st);
    }
  });
  const long long n4 = bytes / 16;
  for (int g : {4, 8, 16, 32, 64, 148, 296}) {
    char name[64];
    std::snprintf(name, sizeof(name), "SM D2H stores, %d blocks", g);
    time(name, [&] { sm_copy<<<g, 512, 0, st>>>((const float4*)d, (float4*)hd, n4); });
  }
  for (int g : {16, 64, 148, 296}) {
    char name[64];
    std::snprintf(name, sizeof(name), "SM H2D loads, %d blocks", g);
    time(name, [&] { sm_copy<<<g, 512, 0, st>>>((const float4*)hd, (float4*)d2, n4); });
  }
  std::printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}

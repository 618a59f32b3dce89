// L2 partition probe (dev tool): does data read by SMs of one half of the chip
// hit in L2 when SMs of the other half read it next?  Run under
//   ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct ./l2_probe
// read_half<<<...>>>(buf, n, half): only CTAs whose %smid lies in that half read.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__global__ void read_half(const float4* __restrict__ buf, long long n, int half, int nsm, float* sink,
                          int* smids) {
  const unsigned s = smid();
  if (threadIdx.x == 0 && smids) smids[blockIdx.x] = static_cast<int>(s);
  const bool mine = half < 0 || (half == 0 ? s < unsigned(nsm / 2) : s >= unsigned(nsm / 2));
  if (!mine) return;
  // every participating CTA reads the whole buffer
  float acc = 0.f;
  const long long stride = blockDim.x;
  for (long long i = threadIdx.x; i < n; i += stride) {
    const float4 v = buf[i];
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.f) *sink = acc;
}

__global__ void fill(float4* b, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned h = static_cast<unsigned>(i) * 2654435761u ^ 0x9e3779b9u;
    b[i] = make_float4(__uint_as_float(h & 0x3fffffff), __uint_as_float((h * 7) & 0x3fffffff),
                       __uint_as_float((h * 13) & 0x3fffffff), __uint_as_float((h * 31) & 0x3fffffff));
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const long long bytes = 48ll << 20;  // fits in either half's L2 slice
  const long long n = bytes / 16;
  float4* buf;
  float* sink;
  int* smids;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 4);
  cudaMalloc(&smids, 4 * 4096);
  fill<<<1024, 256>>>(buf, n);
  const int blocks = nsm;
  // 1: flush-ish (read a big other buffer), 2: low half reads, 3: high half reads, 4: low half again
  float4* big;
  cudaMalloc(&big, 512ll << 20);
  fill<<<1024, 256>>>(big, (512ll << 20) / 16);
  read_half<<<blocks, 256>>>(buf, n, 0, nsm, sink, smids);
  read_half<<<blocks, 256>>>(buf, n, 1, nsm, sink, nullptr);
  read_half<<<blocks, 256>>>(buf, n, 0, nsm, sink, nullptr);
  read_half<<<blocks, 256>>>(buf, n, -1, nsm, sink, nullptr);
  cudaDeviceSynchronize();
  printf("launches done: %s (sm count %d)\n", cudaGetErrorString(cudaGetLastError()), nsm);
  return 0;
}

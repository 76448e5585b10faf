// Read-bandwidth probe: what a pure 128-bit streaming read achieves on this B200
// (the ceiling for K1, whose traffic is 97% id reads). nvcc -arch=sm_100a readbw.cu
#include <cstdio>
#include <cstdint>
__global__ void read_gs(const uint4* __restrict__ p, size_t n, unsigned* out) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}
template <int U>
__global__ void read_unroll(const uint4* __restrict__ p, size_t n, unsigned* out) {
  unsigned acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t i = blockIdx.x * (size_t)blockDim.x * U + threadIdx.x; i + (U - 1) * blockDim.x < n; i += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(p + i + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}
// K1's pattern: each warp streams its own contiguous unit (units of ubytes),
// batches of 32 lanes x U x 16 B, next batch in flight (double buffer)
template <int U>
__global__ void read_units(const uint4* __restrict__ p, size_t n, size_t unit_vec, unsigned* out) {
  const int lane = threadIdx.x & 31;
  const size_t gw = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  const size_t units = n / unit_vec;
  unsigned acc = 0;
  for (size_t u = gw; u < units; u += nw) {
    const uint4* q = p + u * unit_vec + lane;
    const size_t nb = unit_vec / (32 * U);
    uint4 cur[U], nxt[U];
#pragma unroll
    for (int k = 0; k < U; ++k) cur[k] = __ldcs(q + k * 32);
    for (size_t b = 0; b < nb; ++b) {
      if (b + 1 < nb) {
#pragma unroll
        for (int k = 0; k < U; ++k) nxt[k] = __ldcs(q + (b + 1) * 32 * U + k * 32);
      }
#pragma unroll
      for (int k = 0; k < U; ++k) acc ^= cur[k].x ^ cur[k].y ^ cur[k].z ^ cur[k].w;
#pragma unroll
      for (int k = 0; k < U; ++k) cur[k] = nxt[k];
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}
int main() {
  size_t bytes = 25ull << 30;
  uint4* p; unsigned* o;
  cudaMalloc(&p, bytes); cudaMalloc(&o, 4);
  cudaMemset(p, 1, bytes);
  size_t n = bytes / 16;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto fn) {
    for (int w = 0; w < 3; ++w) fn();
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) fn();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    printf("%-28s %.3f ms  %.1f GB/s\n", name, ms, bytes / ms / 1e6);
  };
  for (int bps : {4, 8, 16}) {
    char nm[64];
    snprintf(nm, 64, "grid-stride 256t x%d/SM", bps);
    run(nm, [&] { read_gs<<<148 * bps, 256>>>(p, n, o); });
    snprintf(nm, 64, "unroll8 256t x%d/SM", bps);
    run(nm, [&] { read_unroll<8><<<148 * bps, 256>>>(p, n, o); });
  }
  for (size_t ukb : {512, 64, 16}) {
    for (int warps_per_sm : {12, 32}) {
      char nm[64];
      snprintf(nm, 64, "units %zuKB %d warps/SM", ukb, warps_per_sm);
      run(nm, [&] { read_units<8><<<148 * warps_per_sm / 4, 128>>>(p, n, ukb * 1024 / 16, o); });
    }
  }
  return 0;
}

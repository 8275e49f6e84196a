// Microbenchmark: global reduction (RED) and shared-atomic throughput on B200.
// Informs the scatter strategy of the tet map ("+= strategies").
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

// Each thread does R reds. mode 0: lane-contiguous f64 (warp covers 256 B)
// mode 1: lane stride 72 B (one K block per lane, scattered lines)
// mode 2: f32 v4 contiguous ; mode 3: f32 scalar contiguous ; mode 4: plain f64 store contiguous
__global__ void kred(double* __restrict__ d, float* __restrict__ f, uint64_t n, int mode, int R) {
  uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  for (int r = 0; r < R; ++r) {
    uint64_t i = (tid + (uint64_t)r * nth);
    if (mode == 0) { uint64_t a = i % n; asm volatile("red.global.add.f64 [%0], %1;" :: "l"(d + a), "d"(1.0)); }
    else if (mode == 1) { uint64_t a = (i * 9) % n; asm volatile("red.global.add.f64 [%0], %1;" :: "l"(d + a), "d"(1.0)); }
    else if (mode == 2) { uint64_t a = (i * 4) % (2*n); asm volatile("red.global.add.v4.f32 [%0], {%1,%1,%1,%1};" :: "l"(f + a), "f"(1.0f)); }
    else if (mode == 3) { uint64_t a = i % (2*n); asm volatile("red.global.add.f32 [%0], %1;" :: "l"(f + a), "f"(1.0f)); }
    else if (mode == 4) { uint64_t a = i % n; d[a] = 1.0; }
    else if (mode == 5) { uint64_t a = (i * 9) % n; d[a] = 1.0; }
  }
}
// shared atomics: each thread R atomics to spread addresses in a 8K-double table
__global__ void ksmem(double* out, int mode, int R) {
  __shared__ double s[4096];
  __shared__ float sf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) { s[i] = 0; sf[i] = 0; }
  __syncthreads();
  unsigned h = threadIdx.x * 2654435761u;
  for (int r = 0; r < R; ++r) {
    unsigned a = (h + r * 97u) & 4095u;
    if (mode == 0) atomicAdd(&s[a], 1.0);
    else if (mode == 1) atomicAdd(&sf[a], 1.0f);
    else { s[a] += 1.0; }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0] + sf[0];
}
int main() {
  const char* names[] = {"red.f64 contiguous", "red.f64 stride72B", "red.v4.f32 contiguous", "red.f32 contiguous", "st.f64 contiguous", "st.f64 stride72B"};
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (uint64_t nbytes : {(uint64_t)32 << 20, (uint64_t)1 << 30}) {
    uint64_t n = nbytes / 8;
    double* d; float* f; CK(cudaMalloc(&d, nbytes)); CK(cudaMalloc(&f, nbytes)); cudaMemset(d, 0, nbytes); cudaMemset(f, 0, nbytes);
    int grid = 148 * 8, block = 256, R = 64;
    for (int mode = 0; mode < 6; ++mode) {
      kred<<<grid, block>>>(d, f, n, mode, R);
      cudaEventRecord(a);
      for (int it = 0; it < 5; ++it) kred<<<grid, block>>>(d, f, n, mode, R);
      cudaEventRecord(b); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b);
      double ops = 5.0 * grid * block * R;
      double bytes_per = (mode == 2) ? 16 : (mode == 3 ? 4 : 8);
      printf("ws=%5llu MB %-24s %8.1f Gop/s  %8.1f GB/s payload\n", (unsigned long long)(nbytes >> 20), names[mode], ops / ms / 1e6, ops * bytes_per / ms / 1e6);
    }
    cudaFree(d); cudaFree(f);
  }
  double* o; cudaMalloc(&o, 148 * 64 * 8);
  const char* sn[] = {"atom.shared.f64 spread", "atom.shared.f32 spread", "lds+sts f64 (racy)"};
  for (int mode = 0; mode < 3; ++mode) {
    int grid = 148 * 4, block = 256, R = 256;
    ksmem<<<grid, block>>>(o, mode, R);
    cudaEventRecord(a);
    for (int it = 0; it < 5; ++it) ksmem<<<grid, block>>>(o, mode, R);
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = 5.0 * grid * block * R;
    printf("%-26s %8.1f Gop/s chip  (%.2f op/clk/SM at 1.9GHz)\n", sn[mode], ops / ms / 1e6, ops / ms / 1e6 / 148 / 1.9);
  }
  return 0;
}

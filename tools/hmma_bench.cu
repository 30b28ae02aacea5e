// Throughput of the legacy mma.sync tensor path on sm_100a (HMMA): cycles per warp-instruction
// per SM sub-partition for tf32 m16n8k8 and bf16 m16n8k16, 4 independent accumulator chains per
// warp, 1..4 warps per SMSP. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hmma_bench tools/hmma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int KIND>
__global__ void bench(int iters, float* out, long long* cyc) {
  float d[4][4] = {};
  uint32_t a[4] = {0x3f800000u, 0x3f800000u, 0x3f800000u, 0x3f800000u}, b[2] = {0x3f800000u, 0x3f800000u};
  if (KIND == 1) { a[0] = a[1] = a[2] = a[3] = 0x3f803f80u; b[0] = b[1] = 0x3f803f80u; }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (KIND == 0)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0.f;
  for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  const int iters = 4096;
  for (int kind = 0; kind < 2; ++kind)
    for (int wps = 1; wps <= 4; wps *= 2) {
      const int threads = 32 * 4 * wps;
      if (kind == 0) bench<0><<<148, threads>>>(iters, out, cyc); else bench<1><<<148, threads>>>(iters, out, cyc);
      if (kind == 0) bench<0><<<148, threads>>>(iters, out, cyc); else bench<1><<<148, threads>>>(iters, out, cyc);
      cudaDeviceSynchronize();
      long long h;
      cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      const double per = (double)h / (iters * 4.0 * wps);   // cycles per mma per SMSP
      const double flop = kind == 0 ? 2.0 * 16 * 8 * 8 : 2.0 * 16 * 8 * 16;
      printf("%s warps/SMSP %d: %.2f cycles per mma per SMSP -> %.0f dense FLOP/clk/SM\n",
             kind == 0 ? "tf32 m16n8k8 " : "bf16 m16n8k16", wps, per, 4 * flop / per);
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

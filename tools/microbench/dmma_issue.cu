// DMMA issue microbenchmark (sm_100a): FP64 tensor throughput as a function of
// warps per SM sub-partition and independent accumulators per warp, plus the
// dependent-chain latency. Tells how many warps / how much ILP the zgemm kernels
// need to keep the DMMA pipe busy (next-steps item 2).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

template <int ACC>
__global__ void dmma_ilp(double* out, double seed, int iters) {
  double a0 = seed + threadIdx.x, b0 = seed * 2;
  double acc[ACC][2];
#pragma unroll
  for (int j = 0; j < ACC; j++) acc[j][0] = acc[j][1] = 0;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < ACC; j++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[j][0]), "+d"(acc[j][1]) : "d"(a0), "d"(b0));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < ACC; j++) s += acc[j][0] + acc[j][1];
  if (s == 1.2345) out[0] = s;
}

template <int ACC>
int run(double* out, int sms, cudaEvent_t e0, cudaEvent_t e1) {
  for (int wps : {1, 2, 3, 4, 6, 8}) {
    int warps = 4 * wps;
    if (warps * 32 > 1024) continue;
    int iters = 4096 / ACC * 8;
    dmma_ilp<ACC><<<sms, warps * 32>>>(out, 1.0, iters);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) dmma_ilp<ACC><<<sms, warps * 32>>>(out, 1.0, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double n_dmma = 5.0 * sms * warps * (double)iters * ACC;
    double tf = n_dmma * 512 / ms / 1e9;
    // cycles per DMMA per warp (at the measured clock) -- latency when ACC = 1
    printf("ACC=%2d warps/SMSP=%d  %.2f TFLOP/s  ns/DMMA/warp=%.2f\n", ACC, wps, tf,
           ms * 1e6 / 5.0 / ((double)iters * ACC));
  }
  return 0;
}


// DMMA stream with NADD independent DADDs per 8 DMMAs: does a DADD cost the
// DMMA pipe more than its 64 flops?
template <int NADD>
__global__ void dmma_dadd(double* out, double seed, int iters) {
  double a0 = seed + threadIdx.x, b0 = seed * 2;
  double acc[8][2], x[8];
#pragma unroll
  for (int j = 0; j < 8; j++) { acc[j][0] = acc[j][1] = 0; x[j] = j; }
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[j][0]), "+d"(acc[j][1]) : "d"(a0), "d"(b0));
      if (j < NADD) asm volatile("add.f64 %0, %0, %1;" : "+d"(x[j]) : "d"(b0));
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) s += acc[j][0] + acc[j][1] + x[j];
  if (s == 1.2345) out[0] = s;
}
template <int NADD>
int run_add(double* out, int sms, cudaEvent_t e0, cudaEvent_t e1) {
  for (int wps : {1, 2}) {
    int warps = 4 * wps, iters = 4096;
    dmma_dadd<NADD><<<sms, warps * 32>>>(out, 1.0, iters);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) dmma_dadd<NADD><<<sms, warps * 32>>>(out, 1.0, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double n_dmma = 5.0 * sms * warps * (double)iters * 8;
    printf("DADD/8DMMA=%d warps/SMSP=%d  DMMA %.2f TFLOP/s\n", NADD, wps, n_dmma * 512 / ms / 1e9);
  }
  return 0;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s SMs %d\n", p.name, p.multiProcessorCount);
  double* out;
  CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  if (run<1>(out, sms, e0, e1) || run<2>(out, sms, e0, e1) || run<4>(out, sms, e0, e1) ||
      run<8>(out, sms, e0, e1) || run<16>(out, sms, e0, e1))
    return 1;
  if (run_add<0>(out, sms, e0, e1) || run_add<1>(out, sms, e0, e1) || run_add<2>(out, sms, e0, e1) ||
      run_add<4>(out, sms, e0, e1) || run_add<8>(out, sms, e0, e1))
    return 1;
  return 0;
}

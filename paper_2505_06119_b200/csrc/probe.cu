// FP64 tensor-pipe peak probe (bench roofline denominator): a DMMA-only loop on
// every SM. MEASURED_PEAKS.json carries no FP64 figure, so bench.py measures the
// peak live on the same device, clocks and power state as the timed kernels.
#include "common.h"

namespace qtnhb {
namespace {
__global__ void __launch_bounds__(256) k_dmma_peak(double* out, double seed, int iters) {
  double a = seed + threadIdx.x, b = seed * 0.5;
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[j][0]), "+d"(acc[j][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j][0] + acc[j][1];
  if (s == 1.2345) out[0] = s;
}
}  // namespace
}  // namespace qtnhb

extern "C" int qtnh_probe_fp64_peak(void* stream, double* tflops) {
  using namespace qtnhb;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  if (cudaMallocAsync(&out, 8, st) != cudaSuccess) return QTNH_E_RUNTIME;
  const int iters = 4096, blocks = sms * 4, threads = 256, reps = 5;
  k_dmma_peak<<<blocks, threads, 0, st>>>(out, 1.0, iters);
  note_launch();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  for (int r = 0; r < reps; ++r) k_dmma_peak<<<blocks, threads, 0, st>>>(out, 1.0, iters);
  note_launch(reps);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(out, st);
  double flops = double(reps) * blocks * (threads / 32) * double(iters) * 8 * (8 * 8 * 4 * 2);
  *tflops = flops / (ms * 1e-3) / 1e12;
  return cudaGetLastError() == cudaSuccess ? 0 : QTNH_E_RUNTIME;
}

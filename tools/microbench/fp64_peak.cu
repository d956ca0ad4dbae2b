// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) vs DFMA,
// plus cuBLAS Zgemm/Dgemm ceilings and a complex128 HBM copy. Numbers feed the
// roofline denominators in DESIGN.md (MEASURED_PEAKS.json has no FP64 figure).
#include <cstdio>
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cuComplex.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

template<int ITER>
__global__ void dmma_loop(double* out, double seed){
  double a0=seed+threadIdx.x, b0=seed*2;
  double acc[8][2];
  #pragma unroll
  for(int j=0;j<8;j++){acc[j][0]=0;acc[j][1]=0;}
  for(int i=0;i<ITER;i++){
    #pragma unroll
    for(int j=0;j<8;j++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(acc[j][0]),"+d"(acc[j][1]) : "d"(a0),"d"(b0));
  }
  double s=0; for(int j=0;j<8;j++) s+=acc[j][0]+acc[j][1];
  if(s==1.2345) out[0]=s;
}
__global__ void dmma16_loop(double* out, double seed, int shape, int ITER){
  double a[8], b[4];
  #pragma unroll
  for(int j=0;j<8;j++) a[j]=seed+threadIdx.x+j;
  #pragma unroll
  for(int j=0;j<4;j++) b[j]=seed*2+j;
  double acc[8][4];
  #pragma unroll
  for(int j=0;j<8;j++){acc[j][0]=0;acc[j][1]=0;acc[j][2]=0;acc[j][3]=0;}
  if(shape==4){
    for(int i=0;i<ITER;i++){
      #pragma unroll
      for(int j=0;j<8;j++)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
          : "+d"(acc[j][0]),"+d"(acc[j][1]),"+d"(acc[j][2]),"+d"(acc[j][3]) : "d"(a[0]),"d"(a[1]),"d"(b[0]));
    }
  } else if(shape==8){
    for(int i=0;i<ITER;i++){
      #pragma unroll
      for(int j=0;j<8;j++)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+d"(acc[j][0]),"+d"(acc[j][1]),"+d"(acc[j][2]),"+d"(acc[j][3]) : "d"(a[0]),"d"(a[1]),"d"(a[2]),"d"(a[3]),"d"(b[0]),"d"(b[1]));
    }
  } else {
    for(int i=0;i<ITER;i++){
      #pragma unroll
      for(int j=0;j<8;j++)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
          : "+d"(acc[j][0]),"+d"(acc[j][1]),"+d"(acc[j][2]),"+d"(acc[j][3]) : "d"(a[0]),"d"(a[1]),"d"(a[2]),"d"(a[3]),"d"(a[4]),"d"(a[5]),"d"(a[6]),"d"(a[7]),"d"(b[0]),"d"(b[1]),"d"(b[2]),"d"(b[3]));
    }
  }
  double s=0; for(int j=0;j<8;j++) s+=acc[j][0]+acc[j][1]+acc[j][2]+acc[j][3];
  if(s==1.2345) out[0]=s;
}
template<int ITER>
__global__ void dfma_loop(double* out, double seed){
  double x[8]; double a=seed+threadIdx.x, b=1.0000001;
  for(int j=0;j<8;j++) x[j]=j;
  for(int i=0;i<ITER;i++){
    #pragma unroll
    for(int j=0;j<8;j++) x[j]=fma(x[j],b,a);
  }
  double s=0; for(int j=0;j<8;j++) s+=x[j];
  if(s==1.2345) out[0]=s;
}
__global__ void copy16(const double2* __restrict__ a, double2* __restrict__ b, size_t n){
  size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x, st=(size_t)gridDim.x*blockDim.x;
  for(;i<n;i+=st) b[i]=a[i];
}
int main(){
  int dev=0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  printf("device %s SMs %d clock(kHz) %d\n", p.name, p.multiProcessorCount, p.clockRate);
  double* out; CK(cudaMalloc(&out,8));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int IT=4096;
  for(int warps: {4,8,16}){
    int blocks=p.multiProcessorCount*4;
    dmma_loop<IT><<<blocks,warps*32>>>(out,1.0); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); for(int r=0;r<5;r++) dmma_loop<IT><<<blocks,warps*32>>>(out,1.0); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double flops=5.0*blocks*warps*(double)IT*8*(8*8*4*2);
    printf("DMMA m8n8k4: blocks=%d warps/blk=%d  %.2f TFLOP/s\n",blocks,warps,flops/ms/1e9);
  }
  for(int shape: {4,8,16}) for(int warps: {4,8}){
    int blocks=p.multiProcessorCount*4; const int IT2=IT/ (shape/4);
    dmma16_loop<<<blocks,warps*32>>>(out,1.0,shape,IT2); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); for(int r=0;r<5;r++) dmma16_loop<<<blocks,warps*32>>>(out,1.0,shape,IT2); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double flops=5.0*blocks*warps*(double)IT2*8*(16*8*shape*2);
    printf("DMMA m16n8k%d: blocks=%d warps/blk=%d  %.2f TFLOP/s\n",shape,blocks,warps,flops/ms/1e9);
  }
  for(int thr: {256,512,1024}){
    int blocks=p.multiProcessorCount*2;
    dfma_loop<IT><<<blocks,thr>>>(out,1.0); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); for(int r=0;r<5;r++) dfma_loop<IT><<<blocks,thr>>>(out,1.0); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double flops=5.0*blocks*thr*(double)IT*8*2;
    printf("DFMA: blocks=%d thr=%d  %.2f TFLOP/s\n",blocks,thr,flops/ms/1e9);
  }
  // HBM copy of complex128
  size_t n=(size_t)1<<28; double2 *a,*b; CK(cudaMalloc(&a,n*16)); CK(cudaMalloc(&b,n*16));
  cudaMemset(a,0,n*16);
  for(int r=0;r<2;r++) copy16<<<p.multiProcessorCount*8,512>>>(a,b,n);
  cudaEventRecord(e0); for(int r=0;r<10;r++) copy16<<<p.multiProcessorCount*8,512>>>(a,b,n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  { float ms; cudaEventElapsedTime(&ms,e0,e1); printf("copy16 4GiB: %.1f GB/s (r+w)\n", 10.0*2*n*16/ms/1e6); }
  cudaFree(a); cudaFree(b);
  // cuBLAS ceilings
  cublasHandle_t h; cublasCreate(&h);
  int shapes[][3]={{2097152,128,128},{4096,4096,4096},{2048,2048,1024}};
  for(auto& s: shapes){
    int M=s[0],N=s[1],K=s[2];
    cuDoubleComplex *A,*B,*C; CK(cudaMalloc(&A,(size_t)M*K*16)); CK(cudaMalloc(&B,(size_t)K*N*16)); CK(cudaMalloc(&C,(size_t)M*N*16));
    cudaMemset(A,0,(size_t)M*K*16); cudaMemset(B,0,(size_t)K*N*16);
    cuDoubleComplex one=make_cuDoubleComplex(1,0), zero=make_cuDoubleComplex(0,0);
    // row-major C[M,N]=A[M,K]B[K,N] == col-major C^T = B^T A^T
    for(int r=0;r<2;r++) cublasZgemm(h,CUBLAS_OP_N,CUBLAS_OP_N,N,M,K,&one,B,N,A,K,&zero,C,N);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); for(int r=0;r<5;r++) cublasZgemm(h,CUBLAS_OP_N,CUBLAS_OP_N,N,M,K,&one,B,N,A,K,&zero,C,N); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    printf("cublasZgemm M=%d N=%d K=%d: %.2f TFLOP/s (8MNK) %.3f ms\n",M,N,K,5.0*8.0*M*N*(double)K/ms/1e9, ms/5);
    double *dA=(double*)A,*dB=(double*)B,*dC=(double*)C; double d1=1,d0=0;
    cudaEventRecord(e0); for(int r=0;r<5;r++) cublasDgemm(h,CUBLAS_OP_N,CUBLAS_OP_N,N,M,K,&d1,dB,N,dA,K,&d0,dC,N); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    printf("cublasDgemm M=%d N=%d K=%d: %.2f TFLOP/s (2MNK)\n",M,N,K,5.0*2.0*M*N*(double)K/ms/1e9);
    cudaFree(A);cudaFree(B);cudaFree(C);
  }
  return 0;
}

// FP64 latency / throughput microbenchmarks on the current GPU (development aid).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcpa(double b){double r;asm volatile("rcp.approx.ftz.f64 %0, %1;":"=d"(r):"d"(b));return r;}
__device__ __forceinline__ double rsqa(double b){double r;asm volatile("rsqrt.approx.ftz.f64 %0, %1;":"=d"(r):"d"(b));return r;}
template<int OP> __global__ void lat(double* out, long long* cyc, int n, double a0) {
  double x = a0 + threadIdx.x * 1e-9, y = 1.0000001, z = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (OP == 0) x = fma(x, y, z);
      if (OP == 1) x = x + z;
      if (OP == 2) x = x * y;
      if (OP == 3) x = rcpa(x);
      if (OP == 4) x = rsqa(x) ;
      if (OP == 5) x = sqrt(x) + z;
      if (OP == 6) x = 1.0 / x + z;
      if (OP == 7) { float f = __double2float_rn(x); f = __fmaf_rn(f, 1.0000001f, 1e-9f); x = f; }
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// throughput: 1 warp per SMSP... many independent chains
__global__ void thr_dfma(double* out, long long* cyc, int n) {
  double a[8]; for (int k=0;k<8;++k) a[k]=threadIdx.x+k;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], 0.999999, 1e-7);
  long long t1 = clock64();
  double s=0; for(int k=0;k<8;++k) s+=a[k]; out[threadIdx.x + blockIdx.x*blockDim.x]=s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void shfl_lat(double* out, long long* cyc, int n) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffff, x, 1) + 1e-9;
  long long t1 = clock64(); out[threadIdx.x]=x; if(threadIdx.x==0) cyc[0]=t1-t0;
}
__global__ void smem_lat(double* out, long long* cyc, int n) {
  __shared__ double s[64];
  s[threadIdx.x] = threadIdx.x; __syncwarp();
  int idx = threadIdx.x; double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { double v = s[idx]; acc += v; idx = ((int)v) & 31; }
  long long t1 = clock64(); out[threadIdx.x]=acc; if(threadIdx.x==0) cyc[0]=t1-t0;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 1<<24); cudaMalloc(&cyc, 64);
  const char* names[] = {"DFMA","DADD","DMUL","rcp.approx.f64","rsqrt.approx.f64","sqrt(IEEE)+add","1/x(IEEE)+add","F2F+FFMA"};
  int n = 1000; long long c;
  #define RUN(OP) lat<OP><<<1,32>>>(out,cyc,n,1.5); cudaDeviceSynchronize(); cudaMemcpy(&c,cyc,8,cudaMemcpyDeviceToHost); printf("%-20s latency %.1f cycles\n", names[OP], (double)c/(n*16));
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7)
  shfl_lat<<<1,32>>>(out,cyc,n); cudaDeviceSynchronize(); cudaMemcpy(&c,cyc,8,cudaMemcpyDeviceToHost); printf("SHFL+DADD latency %.1f\n",(double)c/n);
  smem_lat<<<1,32>>>(out,cyc,n); cudaDeviceSynchronize(); cudaMemcpy(&c,cyc,8,cudaMemcpyDeviceToHost); printf("LDS.64+DADD+F2I chain %.1f\n",(double)c/n);
  for (int w : {1,2,4,8,16}) {
    thr_dfma<<<148, 32*w>>>(out,cyc,n); cudaDeviceSynchronize(); cudaMemcpy(&c,cyc,8,cudaMemcpyDeviceToHost);
    printf("DFMA thr: %2d warps/SM: %.2f DFMA/clk/SM\n", w, (double)n*8*32*w/c);
  }
  return 0;
}

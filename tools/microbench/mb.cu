// Microbenchmarks that shape the sweep-kernel design (FFMA forms, FFMA2,
// launch gaps, L2 streaming bandwidth). Standalone: nvcc -o mb mb.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
#define CK(x) do{cudaError_t e=(x); if(e){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__constant__ float cw[64];

template<int MODE>
__global__ void __launch_bounds__(256) fma_kernel(float* out, float a, float b, int iters){
  float x0=threadIdx.x*1e-7f, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  float v = a + threadIdx.x; if(MODE==0) b = b + threadIdx.x*1e-9f;
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int k=0;k<16;k++){
      if(MODE==0){ // 3-reg
        x0=fmaf(x0,v,b); x1=fmaf(x1,v,b); x2=fmaf(x2,v,b); x3=fmaf(x3,v,b);
        x4=fmaf(x4,v,b); x5=fmaf(x5,v,b); x6=fmaf(x6,v,b); x7=fmaf(x7,v,b);
      } else if(MODE==1){ // const-bank weight: acc += w * v
        x0=fmaf(cw[k],v,x0); x1=fmaf(cw[k+1],v,x1); x2=fmaf(cw[k+2],v,x2); x3=fmaf(cw[k+3],v,x3);
        x4=fmaf(cw[k+4],v,x4); x5=fmaf(cw[k+5],v,x5); x6=fmaf(cw[k+6],v,x6); x7=fmaf(cw[k+7],v,x7);
      } else if(MODE==2){ // immediate
        x0=fmaf(x0,1.0001f,0.5f); x1=fmaf(x1,1.0001f,0.5f); x2=fmaf(x2,1.0001f,0.5f); x3=fmaf(x3,1.0001f,0.5f);
        x4=fmaf(x4,1.0001f,0.5f); x5=fmaf(x5,1.0001f,0.5f); x6=fmaf(x6,1.0001f,0.5f); x7=fmaf(x7,1.0001f,0.5f);
      }
    }
  }
  out[blockIdx.x*blockDim.x+threadIdx.x] = x0+x1+x2+x3+x4+x5+x6+x7;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c){
  unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}
__global__ void __launch_bounds__(256) fma2_kernel(float* out, float a, float b, int iters){
  float2 f0 = make_float2(threadIdx.x*1e-7f, 1.f);
  unsigned long long x[8];
  for(int j=0;j<8;j++){ float2 t=make_float2(f0.x+j,f0.y+j); x[j]=*(unsigned long long*)&t; }
  float2 vv = make_float2(a+threadIdx.x, a); unsigned long long v=*(unsigned long long*)&vv;
  float2 bb = make_float2(b,b); unsigned long long bq=*(unsigned long long*)&bb;
  for(int i=0;i<iters;i++){
    #pragma unroll
    for(int k=0;k<8;k++){
      #pragma unroll
      for(int j=0;j<8;j++) x[j]=ffma2(x[j],v,bq);
    }
  }
  float s=0; for(int j=0;j<8;j++){ float2 t=*(float2*)&x[j]; s+=t.x+t.y; }
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}

__global__ void empty_kernel(int* p){ if(p && threadIdx.x==9999) p[0]=1; }
__global__ void pdl_kernel(int* p){
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if(p && threadIdx.x==9999) p[0]=1;
  asm volatile("griddepcontrol.launch_dependents;");
}

__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x; size_t st = (size_t)gridDim.x*blockDim.x;
  for(; i<n; i+=st) b[i]=a[i];
}

int main(){
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop,0));
  printf("dev %s sms %d l2 %d MB smemPerBlockOptin %zu clock %d kHz\n", prop.name, prop.multiProcessorCount, prop.l2CacheSize>>20, prop.sharedMemPerBlockOptin, prop.clockRate);
  float* out; CK(cudaMalloc(&out, 148*8*256*4*4));
  float hw[64]; for(int i=0;i<64;i++) hw[i]=0.01f*i; CK(cudaMemcpyToSymbol(cw,hw,sizeof(hw)));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters=4096; int grid=148*8;
  const char* names[]={"FFMA 3-reg","FFMA const-bank","FFMA imm"};
  for(int m=0;m<4;m++){
    for(int rep=0;rep<2;rep++){
      cudaEventRecord(e0);
      if(m==0) fma_kernel<0><<<grid,256>>>(out,1.0f,0.5f,iters);
      if(m==1) fma_kernel<1><<<grid,256>>>(out,1.0f,0.5f,iters);
      if(m==2) fma_kernel<2><<<grid,256>>>(out,1.0f,0.5f,iters);
      if(m==3) fma2_kernel<<<grid,256>>>(out,1.0f,0.5f,iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms,e0,e1);
      double fmas = (double)grid*256*iters*128.0; // 16*8 FMA per iter (FFMA2: 8*8*2)
      if(rep==1) printf("%-18s %.3f ms  %.2f TFMA/s  (%.1f TFLOP/s)\n", m<3?names[m]:"FFMA2 (f32x2)", ms, fmas/ms/1e9, 2*fmas/ms/1e9);
    }
  }
  // launch gaps
  int N=2000; int* dp; CK(cudaMalloc(&dp,4));
  cudaStream_t s; cudaStreamCreateWithFlags(&s,cudaStreamNonBlocking);
  for(int g=0; g<2; g++){
    for(int i=0;i<100;i++) empty_kernel<<<148,256,0,s>>>(dp);
    cudaEventRecord(e0,s); for(int i=0;i<N;i++) empty_kernel<<<148,256,0,s>>>(dp); cudaEventRecord(e1,s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms,e0,e1); if(g) printf("plain launches: %.3f us/kernel (148x256)\n", ms*1e3/N);
  }
  {
    cudaLaunchConfig_t cfg={}; cfg.gridDim=dim3(148); cfg.blockDim=dim3(256); cfg.stream=s;
    cudaLaunchAttribute at[1]; at[0].id=cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed=1;
    cfg.attrs=at; cfg.numAttrs=1;
    for(int g=0; g<2; g++){
      cudaEventRecord(e0,s); for(int i=0;i<N;i++) CK(cudaLaunchKernelEx(&cfg,pdl_kernel,dp)); cudaEventRecord(e1,s); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms,e0,e1); if(g) printf("PDL launches: %.3f us/kernel\n", ms*1e3/N);
    }
    // graph of 200 PDL launches
    cudaGraph_t graph; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s,cudaStreamCaptureModeGlobal));
    for(int i=0;i<200;i++) CK(cudaLaunchKernelEx(&cfg,pdl_kernel,dp));
    CK(cudaStreamEndCapture(s,&graph)); CK(cudaGraphInstantiate(&ge,graph,0));
    for(int g=0; g<3; g++){
      cudaEventRecord(e0,s); for(int i=0;i<10;i++) cudaGraphLaunch(ge,s); cudaEventRecord(e1,s); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms,e0,e1); if(g) printf("graph(200 PDL): %.3f us/kernel\n", ms*1e3/2000);
    }
    CK(cudaStreamBeginCapture(s,cudaStreamCaptureModeGlobal));
    for(int i=0;i<200;i++) empty_kernel<<<148,256,0,s>>>(dp);
    CK(cudaStreamEndCapture(s,&graph)); CK(cudaGraphInstantiate(&ge,graph,0));
    for(int g=0; g<3; g++){
      cudaEventRecord(e0,s); for(int i=0;i<10;i++) cudaGraphLaunch(ge,s); cudaEventRecord(e1,s); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms,e0,e1); if(g) printf("graph(200 plain): %.3f us/kernel\n", ms*1e3/2000);
    }
  }
  // bandwidth: L2-resident (20 MB each way) and HBM (1 GB each way)
  size_t sizes[]={(size_t)5<<20, (size_t)10<<20, (size_t)20<<20, (size_t)256<<20};
  for(size_t nfl: sizes){
    float *a,*b; CK(cudaMalloc(&a,nfl*4)); CK(cudaMalloc(&b,nfl*4)); cudaMemset(a,0,nfl*4);
    for(int blocks: {148*4, 148*8}){
      for(int g=0; g<3; g++){
        int R=20; cudaEventRecord(e0,s); for(int r=0;r<R;r++) copy_kernel<<<blocks,512,0,s>>>((float4*)a,(float4*)b,nfl/4); cudaEventRecord(e1,s); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms,e0,e1);
        if(g==2) printf("copy %zu MB x2 (r+w) blocks %d: %.1f GB/s (%.2f us/launch)\n", (nfl*4)>>20, blocks, 2.0*nfl*4*R/ms/1e6, ms*1e3/R);
      }
    }
    cudaFree(a); cudaFree(b);
  }
  return 0;
}

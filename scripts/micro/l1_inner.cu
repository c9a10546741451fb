// Microbenchmark (not product code): the L1 engine's inner loop in isolation --
// 8x8 register micro-tile per thread, operands from shared memory every k.
//   abs : acc += |q - t|                       (FADD + FADD|.| per element)
//   max2: acc2 += (max(q,t0), max(q,t1))       (2 FMNMX + 1 FADD2 per 2 elements; L1 = 2 acc - Sq - St)
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#define KLEN 32
#define REPS 64
__device__ __forceinline__ unsigned long long pk(float a, float b){ unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void upk(unsigned long long v, float& a, float& b){ asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b){ unsigned long long d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
template<int V>
__global__ void __launch_bounds__(256,2) k(const float* g, float* out){
  __shared__ __align__(16) float Qs[KLEN*128], Ts[KLEN*128];
  for(int i=threadIdx.x;i<KLEN*128;i+=256){ Qs[i]=g[i]; Ts[i]=g[i+7]; }
  __syncthreads();
  const int ty=threadIdx.x>>4, tx=threadIdx.x&15;
  float acc[8][8]; unsigned long long acc2[8][4];
  for(int a=0;a<8;++a){ for(int b=0;b<8;++b) acc[a][b]=0; for(int b=0;b<4;++b) acc2[a][b]=0; }
  for(int rep=0; rep<REPS; ++rep){
    #pragma unroll 4
    for(int kk=0;kk<KLEN;++kk){
      const float4 qa=*reinterpret_cast<const float4*>(Qs+kk*128+ty*8), qb=*reinterpret_cast<const float4*>(Qs+kk*128+ty*8+4);
      const float4 ta=*reinterpret_cast<const float4*>(Ts+kk*128+tx*8), tb=*reinterpret_cast<const float4*>(Ts+kk*128+tx*8+4);
      const float qv[8]={qa.x,qa.y,qa.z,qa.w,qb.x,qb.y,qb.z,qb.w}, tv[8]={ta.x,ta.y,ta.z,ta.w,tb.x,tb.y,tb.z,tb.w};
      #pragma unroll
      for(int a=0;a<8;++a){
        if(V==0){
          #pragma unroll
          for(int b=0;b<8;++b) acc[a][b]+=fabsf(qv[a]-tv[b]);
        } else {
          #pragma unroll
          for(int b=0;b<4;++b) acc2[a][b]=add2(acc2[a][b], pk(fmaxf(qv[a],tv[2*b]), fmaxf(qv[a],tv[2*b+1])));
        }
      }
    }
    __syncthreads();
  }
  float s=0;
  for(int a=0;a<8;++a){ for(int b=0;b<8;++b) s+=acc[a][b]; for(int b=0;b<4;++b){float x,y; upk(acc2[a][b],x,y); s+=x+y;} }
  out[blockIdx.x*256+threadIdx.x]=s;
}
template<int OCC>
__global__ void __launch_bounds__(256,OCC) kh(const float* g, float* out){
  __shared__ __align__(16) unsigned Qs[KLEN*128], Ts[KLEN*128];
  for(int i=threadIdx.x;i<KLEN*128;i+=256){ Qs[i]=__float_as_uint(g[i]); Ts[i]=__float_as_uint(g[i+7]); }
  __syncthreads();
  const int ty=threadIdx.x>>4, tx=threadIdx.x&15;
  __half2 acc[8][8];
  for(int a=0;a<8;++a) for(int b=0;b<8;++b) acc[a][b]=__float2half2_rn(0.f);
  for(int rep=0; rep<REPS; ++rep){
    #pragma unroll 4
    for(int kk=0;kk<KLEN;++kk){
      const uint4 qa=*reinterpret_cast<const uint4*>(Qs+kk*128+ty*8), qb=*reinterpret_cast<const uint4*>(Qs+kk*128+ty*8+4);
      const uint4 ta=*reinterpret_cast<const uint4*>(Ts+kk*128+tx*8), tb=*reinterpret_cast<const uint4*>(Ts+kk*128+tx*8+4);
      const unsigned qv[8]={qa.x,qa.y,qa.z,qa.w,qb.x,qb.y,qb.z,qb.w}, tv[8]={ta.x,ta.y,ta.z,ta.w,tb.x,tb.y,tb.z,tb.w};
      #pragma unroll
      for(int a=0;a<8;++a)
      #pragma unroll
        for(int b=0;b<8;++b) acc[a][b]=__hadd2(acc[a][b], __habs2(__hsub2(*reinterpret_cast<const __half2*>(&qv[a]), *reinterpret_cast<const __half2*>(&tv[b]))));
    }
    __syncthreads();
  }
  float s=0; for(int a=0;a<8;++a) for(int b=0;b<8;++b){ float2 f=__half22float2(acc[a][b]); s+=f.x+f.y; }
  out[blockIdx.x*256+threadIdx.x]=s;
}
int main(){
  float *g,*o; cudaMalloc(&g, 8*KLEN*128*4); cudaMalloc(&o, 148*16*256*4); cudaMemset(g,0,8*KLEN*128*4);
  int clk=0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* nm[]={"abs  (FADD+FADD|.|)","max2 (2 FMNMX+FADD2)"};
  for(int v=0;v<2;++v){ for(int bps : {1,2,4}) {
    auto kern = v==0 ? k<0> : k<1>;
    cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
    kern<<<148*bps,256>>>(g,o); cudaDeviceSynchronize();
    cudaEventRecord(a); for(int r=0;r<5;++r) kern<<<148*bps,256>>>(g,o); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms,a,b); ms/=5;
    double el=(double)148*bps*256*64*KLEN*REPS;
    printf("%s blocks/SM=%d: %.3f ms  %.1f elem/clk/SM  (%.1f%% of 64 elem/clk/SM = 128 lane-ops/2)\n", nm[v], bps, ms, el/(ms*1e-3)/(clk*1e3)/148, 100*el/(ms*1e-3)/(clk*1e3)/148/64);
  }}
  for(int v=0; v<2; ++v){ for(int bps : {1,2}) {
    auto kern = v==0 ? kh<1> : kh<2>;
    if ((v==0) != (bps==1)) continue;
    cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
    kern<<<148*bps,256>>>(g,o); cudaDeviceSynchronize();
    cudaEventRecord(a); for(int r=0;r<5;++r) kern<<<148*bps,256>>>(g,o); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms,a,b); ms/=5;
    double el=(double)148*bps*256*64*KLEN*REPS*2;
    printf("half2 (HADD2+HADD2|.|, 2 elem/lane) blocks/SM=%d: %.3f ms  %.1f elem/clk/SM\n", bps, ms, el/(ms*1e-3)/(clk*1e3)/148);
  }}
  cudaError_t e=cudaGetLastError(); printf("%s\n", cudaGetErrorString(e)); return 0;
}

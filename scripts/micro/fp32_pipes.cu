// Microbenchmark (not product code): FP32 instruction-mix throughput on one B200,
// to choose the L1 engine's inner loop.  Prints element-ops per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__device__ __forceinline__ unsigned long long pk(float a, float b){ unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void upk(unsigned long long v, float& a, float& b){ asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b){ unsigned long long d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }

// mode 0: acc += |q - t|  (scalar FADD + FADD|.|), 16 chains
__global__ void k_abs(const float* in, float* out){
  float q[4], t[4], acc[16];
  for(int i=0;i<4;++i){ q[i]=in[threadIdx.x+i]; t[i]=in[threadIdx.x+64+i]; }
  for(int i=0;i<16;++i) acc[i]=0;
  for(int it=0; it<ITERS; ++it){
    #pragma unroll
    for(int a=0;a<4;++a)
    #pragma unroll
      for(int b=0;b<4;++b) acc[a*4+b] += fabsf(q[a]-t[b]);
    q[0]+=1e-7f; t[1]-=1e-7f;
  }
  float s=0; for(int i=0;i<16;++i) s+=acc[i]; out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
// mode 1: acc2 += (max(q0,t0), max(q1,t1))  (2 FMNMX + FADD2), 16 element chains = 8 packed
__global__ void k_max2(const float* in, float* out){
  float q[4], t[4]; unsigned long long acc[8];
  for(int i=0;i<4;++i){ q[i]=in[threadIdx.x+i]; t[i]=in[threadIdx.x+64+i]; }
  for(int i=0;i<8;++i) acc[i]=0;
  for(int it=0; it<ITERS; ++it){
    #pragma unroll
    for(int a=0;a<4;++a)
    #pragma unroll
      for(int b=0;b<4;b+=2) acc[a*2+b/2] = add2(acc[a*2+b/2], pk(fmaxf(q[a],t[b]), fmaxf(q[a],t[b+1])));
    q[0]+=1e-7f; t[1]-=1e-7f;
  }
  float s=0; for(int i=0;i<8;++i){ float x,y; upk(acc[i],x,y); s+=x+y;} out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
// mode 2: scalar max formulation: acc += max(q,t) (FMNMX + FADD)
__global__ void k_max1(const float* in, float* out){
  float q[4], t[4], acc[16];
  for(int i=0;i<4;++i){ q[i]=in[threadIdx.x+i]; t[i]=in[threadIdx.x+64+i]; }
  for(int i=0;i<16;++i) acc[i]=0;
  for(int it=0; it<ITERS; ++it){
    #pragma unroll
    for(int a=0;a<4;++a)
    #pragma unroll
      for(int b=0;b<4;++b) acc[a*4+b] += fmaxf(q[a],t[b]);
    q[0]+=1e-7f; t[1]-=1e-7f;
  }
  float s=0; for(int i=0;i<16;++i) s+=acc[i]; out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
// mode 3: packed sub + packed fma (L2 SIMT form): d2 = q2 - t2; acc2 = fma2(d2,d2,acc2)
__device__ __forceinline__ unsigned long long sub2(unsigned long long a, unsigned long long b){ unsigned long long d; asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c){ unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__global__ void k_l2pk(const float* in, float* out){
  unsigned long long q[4], t[2], acc[8];
  for(int i=0;i<4;++i){ float x=in[threadIdx.x+i]; q[i]=pk(x,x); }
  for(int i=0;i<2;++i){ t[i]=pk(in[threadIdx.x+64+2*i], in[threadIdx.x+65+2*i]); }
  for(int i=0;i<8;++i) acc[i]=0;
  for(int it=0; it<ITERS; ++it){
    #pragma unroll
    for(int a=0;a<4;++a)
    #pragma unroll
      for(int b=0;b<2;++b){ unsigned long long d=sub2(q[a],t[b]); acc[a*2+b]=fma2(d,d,acc[a*2+b]); }
    q[0]=add2(q[0], 1); 
  }
  float s=0; for(int i=0;i<8;++i){ float x,y; upk(acc[i],x,y); s+=x+y;} out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
// mode 4: scalar L2: d = q - t; acc = fma(d,d,acc)
__global__ void k_l2(const float* in, float* out){
  float q[4], t[4], acc[16];
  for(int i=0;i<4;++i){ q[i]=in[threadIdx.x+i]; t[i]=in[threadIdx.x+64+i]; }
  for(int i=0;i<16;++i) acc[i]=0;
  for(int it=0; it<ITERS; ++it){
    #pragma unroll
    for(int a=0;a<4;++a)
    #pragma unroll
      for(int b=0;b<4;++b){ float d=q[a]-t[b]; acc[a*4+b]=fmaf(d,d,acc[a*4+b]); }
    q[0]+=1e-7f; t[1]-=1e-7f;
  }
  float s=0; for(int i=0;i<16;++i) s+=acc[i]; out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
// mode 5: packed |q - t|: d2 = q2 - t2 (FADD2), clear both sign bits (LOP3 on the 64-bit pair), acc2 += (FADD2)
__device__ __forceinline__ unsigned long long abs2(unsigned long long a){ return a & 0x7fffffff7fffffffULL; }
__global__ void k_abs2(const float* in, float* out){
  unsigned long long q[4], t[2], acc[8];
  for(int i=0;i<4;++i){ float x=in[threadIdx.x+i]; q[i]=pk(x,x); }
  for(int i=0;i<2;++i){ t[i]=pk(in[threadIdx.x+64+2*i], in[threadIdx.x+65+2*i]); }
  for(int i=0;i<8;++i) acc[i]=0;
  for(int it=0; it<ITERS; ++it){
    #pragma unroll
    for(int a=0;a<4;++a)
    #pragma unroll
      for(int b=0;b<2;++b){ unsigned long long d=sub2(q[a],t[b]); acc[a*2+b]=add2(acc[a*2+b], abs2(d)); }
    q[0]=add2(q[0], 1);
  }
  float s=0; for(int i=0;i<8;++i){ float x,y; upk(acc[i],x,y); s+=x+y;} out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){
  float *in,*out; cudaMalloc(&in, 4096*4); cudaMalloc(&out, 148*16*256*4); cudaMemset(in,0,4096*4);
  int sms=148, clk_khz=0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const char* names[]={"abs: FADD+FADD|.| per elem","max2: 2xFMNMX+FADD2 per 2 elem","max1: FMNMX+FADD per elem","l2pk: FADD2+FFMA2 per 2 elem","l2: FADD+FFMA per elem","abs2: FADD2+LOP3x2+FADD2 per 2 elem"};
  void (*ks[])(const float*,float*)={k_abs,k_max2,k_max1,k_l2pk,k_l2,k_abs2};
  for(int blocks_per_sm : {4, 8}) for(int m=0;m<6;++m){
    cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
    ks[m]<<<sms*blocks_per_sm,256>>>(in,out); cudaDeviceSynchronize();
    cudaEventRecord(a); ks[m]<<<sms*blocks_per_sm,256>>>(in,out); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms,a,b);
    double elems=(double)sms*blocks_per_sm*256*ITERS*16;
    double per_clk_sm = elems/(ms*1e-3)/ (clk_khz*1e3) / sms;
    printf("%-34s blocks/SM %d: %.3f ms, %.1f elem/clk/SM (at %d MHz)\n", names[m], blocks_per_sm, ms, per_clk_sm, clk_khz/1000);
  }
  return 0;
}

// B200 probe: HBM stream, L2-resident random gathers (4/8/16 B), smem random lookups,
// and the combined literal-stream + gather pattern of the trigger test.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);exit(1);}}while(0)

__device__ __forceinline__ uint32_t hsh(uint32_t x){ x^=x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }

__global__ void k_stream(const uint4* __restrict__ p, size_t n, uint32_t* out){
  uint32_t acc=0; size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x, st=(size_t)gridDim.x*blockDim.x;
  #pragma unroll 4
  for(;i<n;i+=st){ uint4 v=__ldg(p+i); acc^=v.x^v.y^v.z^v.w; }
  if(acc==0x12345678) out[0]=acc;
}
template<class T>
__global__ void k_gather(const T* __restrict__ tab, uint32_t ntab, uint32_t per_thread, uint32_t* out){
  uint32_t acc=0; uint32_t t=blockIdx.x*blockDim.x+threadIdx.x;
  #pragma unroll 8
  for(uint32_t k=0;k<per_thread;k++){ uint32_t idx=hsh(t*per_thread+k)%ntab; T v=__ldg(tab+idx); acc^=((const uint32_t*)&v)[0]; }
  if(acc==0x12345678) out[0]=acc;
}
__global__ void k_smem(const uint32_t* __restrict__ tab, uint32_t ntab_words, uint32_t per_thread, uint32_t* out){
  extern __shared__ uint32_t s[];
  for(uint32_t i=threadIdx.x;i<ntab_words;i+=blockDim.x) s[i]=tab[i];
  __syncthreads();
  uint32_t acc=0; uint32_t t=blockIdx.x*blockDim.x+threadIdx.x;
  #pragma unroll 8
  for(uint32_t k=0;k<per_thread;k++){ uint32_t idx=hsh(t*per_thread+k)%ntab_words; acc^=s[idx]; }
  if(acc==0x12345678) out[0]=acc;
}
// combined: 32-clause interleaved stream (LDG.32 per literal row) + 16B gather per literal
__global__ void k_combo(const int32_t* __restrict__ lits, int size, uint32_t nblk, const uint4* __restrict__ tab, uint32_t* out){
  uint32_t acc=0; int lane=threadIdx.x&31; uint32_t w=(blockIdx.x*blockDim.x+threadIdx.x)>>5, nw=(gridDim.x*blockDim.x)>>5;
  for(uint32_t b=w;b<nblk;b+=nw){
    const int32_t* p=lits+(size_t)b*size*32+lane;
    #pragma unroll 4
    for(int j=0;j<size;j++){ int l=__ldg(p+j*32); uint4 v=__ldg(tab+(l<0?-l:l)); acc^=v.x^v.y; }
  }
  if(acc==0x12345678) out[0]=acc;
}
__global__ void k_fill(int32_t* p, size_t n, uint32_t V){ size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x; if(i<n){ uint32_t h=hsh((uint32_t)i*2654435761u+7); int v=1+h%V; p[i]=(h&0x80000000u)?-v:v; } }

int main(){
  int dev=0; cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr,dev));
  printf("dev %s SMs %d L2 %d MB smemOptin %zu\n",pr.name,pr.multiProcessorCount,pr.l2CacheSize>>20,pr.sharedMemPerBlockOptin);
  int nsm=pr.multiProcessorCount;
  cudaEvent_t a,b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); float ms;
  uint32_t* out; CK(cudaMalloc(&out,4));
  size_t nbytes=(size_t)2<<30; uint4* big; CK(cudaMalloc(&big,nbytes)); CK(cudaMemset(big,1,nbytes));
  for(int blocks_per_sm: {4,8,16}){
    int grid=nsm*blocks_per_sm; k_stream<<<grid,256>>>(big,nbytes/16,out);
    CK(cudaEventRecord(a)); for(int r=0;r<5;r++) k_stream<<<grid,256>>>(big,nbytes/16,out); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms,a,b)); printf("stream LDG.128 %d blk/SM: %.1f GB/s\n",blocks_per_sm,5*nbytes/(ms*1e-3)/1e9);
  }
  // gathers from table sizes 0.2, 3.2, 51 MB
  for(size_t tb: {(size_t)200<<10,(size_t)3200<<10,(size_t)51<<20}){
    uint32_t per=256; int grid=nsm*8, thr=256; double n=(double)grid*thr*per;
    k_gather<uint4><<<grid,thr>>>(big,tb/16,per,out); CK(cudaEventRecord(a)); k_gather<uint4><<<grid,thr>>>(big,tb/16,per,out); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms,a,b));
    printf("gather16 table %zu KB: %.2f G gathers/s (%.2f per SM-clk@1.9G)\n",tb>>10,n/(ms*1e-3)/1e9, n/(ms*1e-3)/nsm/1.9e9);
    k_gather<uint2><<<grid,thr>>>((const uint2*)big,tb/8,per,out); CK(cudaEventRecord(a)); k_gather<uint2><<<grid,thr>>>((const uint2*)big,tb/8,per,out); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms,a,b));
    printf("gather8  table %zu KB: %.2f G gathers/s\n",tb>>10,n/(ms*1e-3)/1e9);
    k_gather<uint32_t><<<grid,thr>>>((const uint32_t*)big,tb/4,per,out); CK(cudaEventRecord(a)); k_gather<uint32_t><<<grid,thr>>>((const uint32_t*)big,tb/4,per,out); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms,a,b));
    printf("gather4  table %zu KB: %.2f G gathers/s\n",tb>>10,n/(ms*1e-3)/1e9);
  }
  { // smem
    uint32_t words=(200<<10)/4; CK(cudaFuncSetAttribute(k_smem,cudaFuncAttributeMaxDynamicSharedMemorySize,words*4));
    uint32_t per=4096; int grid=nsm, thr=1024; double n=(double)grid*thr*per;
    k_smem<<<grid,thr,words*4>>>((const uint32_t*)big,words,per,out); CK(cudaEventRecord(a)); k_smem<<<grid,thr,words*4>>>((const uint32_t*)big,words,per,out); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms,a,b));
    printf("smem rand LDS.32 200KB: %.2f G lookups/s (%.2f per SM-clk@1.9G)\n",n/(ms*1e-3)/1e9,n/(ms*1e-3)/nsm/1.9e9);
  }
  { // combo: 10M clauses size 16 = 160M lits, V=200k
    uint32_t V=200000; int size=16; uint32_t nblk=10000000/32; size_t nl=(size_t)nblk*size*32; int32_t* lits; CK(cudaMalloc(&lits,nl*4));
    k_fill<<<(nl+255)/256,256>>>(lits,nl,V); CK(cudaDeviceSynchronize());
    for(int bps: {4,8}){ int grid=nsm*bps;
    k_combo<<<grid,256>>>(lits,size,nblk,big,out); CK(cudaEventRecord(a)); k_combo<<<grid,256>>>(lits,size,nblk,big,out); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms,a,b));
    printf("combo stream+gather16 (%d blk/SM): %.3f ms, %.1f GB/s lit stream, %.2f G gathers/s\n",bps,ms,nl*4/(ms*1e-3)/1e9,nl/(ms*1e-3)/1e9);}
    CK(cudaFree(lits));
  }
  printf("done\n"); return 0;
}

// Harness-only probe: accuracy of 3xTF32 products with mma.sync m16n8k8 under different
// accumulation strategies, vs an fp64 reference.  C = X Y with X, Y 32x32 (many trials).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t rna(float x){uint32_t r;asm("cvt.rna.tf32.f32 %0,%1;":"=r"(r):"f"(x));return r;}
__device__ __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]){
 asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};"
 :"+f"(c[0]),"+f"(c[1]),"+f"(c[2]),"+f"(c[3]):"r"(a[0]),"r"(a[1]),"r"(a[2]),"r"(a[3]),"r"(b[0]),"r"(b[1]));}
// mode 0: one chain c += lo*hi, hi*lo, hi*hi per kb. 1: separate small/big chains. 2: c=0 per MMA + FADD.
// 3: plain fp32 FFMA (SIMT) reference.
__global__ void k(const float* X, const float* Y, float* C, int mode){
  const float* x = X + blockIdx.x*1024; const float* y = Y + blockIdx.x*1024; float* c = C + blockIdx.x*1024;
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane>>2, t = lane&3;
  if (mode == 3) { for (int i = threadIdx.x; i < 1024; i += blockDim.x) { int r=i/32, cc=i%32; float s=0; for(int q=0;q<32;++q) s=fmaf(x[r*32+q],y[q*32+cc],s); c[i]=s;} return; }
  for (int blk = warp; blk < 8; blk += blockDim.x/32) {
    int mb = blk/4, nb = blk%4;
    float big[4]={0,0,0,0}, sm[4]={0,0,0,0};
    for (int kb=0;kb<4;++kb){
      int r0=mb*16+g, c0=kb*8+t;
      float af[4]={x[r0*32+c0],x[(r0+8)*32+c0],x[r0*32+c0+4],x[(r0+8)*32+c0+4]};
      float bf[2]={y[(kb*8+t)*32+nb*8+g],y[(kb*8+t+4)*32+nb*8+g]};
      uint32_t ah[4],al[4],bh[2],bl[2];
      for(int i=0;i<4;++i){ah[i]=rna(af[i]); al[i]=rna(af[i]-__uint_as_float(ah[i]));}
      for(int i=0;i<2;++i){bh[i]=rna(bf[i]); bl[i]=rna(bf[i]-__uint_as_float(bh[i]));}
      if (mode==0){ mma(big,al,bh); mma(big,ah,bl); mma(big,ah,bh);} 
      else if (mode==1){ mma(sm,al,bh); mma(sm,ah,bl); mma(big,ah,bh);} 
      else { float t1[4]={0,0,0,0},t2[4]={0,0,0,0}; mma(t1,al,bh); mma(t1,ah,bl); mma(t2,ah,bh); for(int i=0;i<4;++i){sm[i]+=t1[i]; big[i]+=t2[i];} }
    }
    for(int e=0;e<4;++e){int r=mb*16+g+((e&2)?8:0), cc=nb*8+2*t+(e&1); c[r*32+cc]=big[e]+sm[e];}
  }
}
int main(){
  int T=4096; size_t n=(size_t)T*1024; float *X,*Y,*C; cudaMallocManaged(&X,n*4); cudaMallocManaged(&Y,n*4); cudaMallocManaged(&C,n*4);
  srand(1); for(size_t i=0;i<n;++i){ X[i]=((rand()/(float)RAND_MAX)-0.5f)*0.3f; Y[i]=((rand()/(float)RAND_MAX)-0.5f)*0.3f; }
  for(int mode=0;mode<4;++mode){ k<<<T,128>>>(X,Y,C,mode); cudaDeviceSynchronize();
    double maxrel=0, sumrel=0, bias=0;
    for(int b=0;b<T;++b){ double num=0,den=0,bs=0; for(int r=0;r<32;++r)for(int cc=0;cc<32;++cc){ double s=0; for(int q=0;q<32;++q) s+=(double)X[b*1024+r*32+q]*Y[b*1024+q*32+cc]; double e=C[b*1024+r*32+cc]-s; num+=e*e; den+=s*s; bs+= e*(s>0?1:-1);} double rel=sqrt(num/den); maxrel=fmax(maxrel,rel); sumrel+=rel; bias+=bs/1024/sqrt(den/1024);}
    printf("mode %d: max rel %.3e mean rel %.3e mean signed(err*sign(ref))/rms %.3e\n", mode, maxrel, sumrel/T, bias/T); }
  return 0; }

// Harness-only: MMA-thread wait-cycle breakdown of the fp32 engine at d=4096.
#define NSERIES_TF32_DEBUG
#include "../paper_2602_11843_b200/csrc/gemm_tf32.cu"
using namespace nseries;
int main() {
  int d = 4096, ldp = 4096; size_t n = (size_t)d * ldp;
  float *Xh, *Xl, *Yh, *Yl, *C; cudaMalloc(&Xh, n*4); cudaMalloc(&Xl, n*4); cudaMalloc(&Yh, n*4); cudaMalloc(&Yl, n*4); cudaMalloc(&C, n*4);
  cudaMemset(Xh, 0, n*4); cudaMemset(Xl, 0, n*4); cudaMemset(Yh, 0, n*4); cudaMemset(Yl, 0, n*4);
  unsigned long long* dbg; cudaMalloc(&dbg, 128); cudaMemset(dbg, 0, 128);
  float* dp = (float*)dbg; cudaMemcpyToSymbol(g_dbg, &dp, sizeof(dp));
  EpiParamsF32 ep{}; ep.ldp = ldp; ep.n_out = 1; ep.out_x[0] = C; ep.out_ld[0] = d; ep.alpha[0] = 1.0;
  launch_gemm_tf32x3(Xh, Xl, Yh, Yl, d, ldp, ep, 0); cudaDeviceSynchronize();
  cudaMemset(dbg, 0, 128);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); launch_gemm_tf32x3(Xh, Xl, Yh, Yl, d, ldp, ep, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[10]; cudaMemcpy(h, dbg, 80, cudaMemcpyDeviceToHost);
  double ctas = h[2];
  printf("ms %.3f ctas %.0f  per-CTA avg cycles: wait tmem_empty %.0f  wait full %.0f  mma loop total %.0f (kernel %.0f cycles/CTA-wave at 1.9GHz)\n",
         ms, ctas, h[0] / ctas, h[1] / ctas, h[3] / ctas, ms * 1e-3 * 1.9e9 / 7);
  printf("prologue %.0f  epilogue-final %.0f  start->drained %.0f  staged0 %.0f staged1 %.0f\n", h[4] / ctas, h[5] / ctas, h[6] / ctas, h[7] / ctas, h[8] / ctas);
  return 0;
}

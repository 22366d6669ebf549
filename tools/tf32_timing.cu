// Harness-only: per-CTA phase breakdown of the fp32 engine at d=4096 (mainloop+drain vs final
// epilogue) for a 1-output op and a 3-output op shaped like radix-15 G1 (x, hi/lo, hiT/loT + 1 aux).
#define NSERIES_TF32_DEBUG
#include <cstdlib>
#include <vector>
#include <map>
#include <algorithm>
#include "../paper_2602_11843_b200/csrc/gemm_tf32.cu"
using namespace nseries;
int main() {
  int d = getenv("TD") ? atoi(getenv("TD")) : 4096, ldp = d; size_t n = (size_t)d * ldp;
  float *Xh, *Xl, *Yh, *Yl, *C, *P[6];
  cudaMalloc(&Xh, n*4); cudaMalloc(&Xl, n*4); cudaMalloc(&Yh, n*4); cudaMalloc(&Yl, n*4); cudaMalloc(&C, n*4);
  for (int i = 0; i < 6; ++i) { cudaMalloc(&P[i], n * 4); cudaMemset(P[i], 0, n * 4); }
  cudaMemset(Xh, 0, n*4); cudaMemset(Xl, 0, n*4); cudaMemset(Yh, 0, n*4); cudaMemset(Yl, 0, n*4);
  unsigned long long* dbg; cudaMalloc(&dbg, 256); cudaMemset(dbg, 0, 256);  // slots 8..14: epilogue phase deltas
  float* dp = (float*)dbg; cudaMemcpyToSymbol(g_dbg, &dp, sizeof(dp));
  unsigned long long* tl; cudaMalloc(&tl, 3 * 8 * 4096); cudaMemset(tl, 0, 3 * 8 * 4096);
  cudaMemcpyToSymbol(g_tl, &tl, sizeof(tl));
  for (int variant = 0; variant < 4; ++variant) {
    EpiParamsF32 ep{}; ep.ldp = ldp;
    if (variant == 0) { ep.n_out = 1; ep.out_x[0] = C; ep.out_ld[0] = d; ep.alpha[0] = 1.0; }
    else if (variant == 2) { ep.n_out = 1; ep.out_ld[0] = d; ep.alpha[0] = 1.0; }   // no stores at all
    else if (variant == 3) { ep.n_out = 1; ep.out_hiT[0] = P[2]; ep.out_loT[0] = P[3]; ep.out_ld[0] = d; ep.alpha[0] = 1.0; }
    else {
      ep.n_out = 3; ep.n_aux = 1; ep.aux[0] = P[5]; ep.aux_ld[0] = d;
      ep.out_x[0] = C; ep.out_ld[0] = d; ep.alpha[0] = 1.0;
      ep.out_hi[1] = P[0]; ep.out_lo[1] = P[1]; ep.out_ld[1] = d; ep.alpha[1] = 0.5; ep.beta[1][0] = 0.25;
      ep.out_hiT[2] = P[2]; ep.out_loT[2] = P[3]; ep.out_ld[2] = d; ep.alpha[2] = 0.3; ep.beta[2][0] = 0.1; ep.gamma[2] = 1;
    }
    launch_gemm_tf32x3(Xh, Xl, Yh, Yl, d, ldp, ep, 0); cudaDeviceSynchronize();
    cudaMemset(dbg, 0, 256);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); launch_gemm_tf32x3(Xh, Xl, Yh, Yl, d, ldp, ep, 0); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[10]; cudaMemcpy(h, dbg, 80, cudaMemcpyDeviceToHost);
    double ctas = h[2];
    printf("variant %d: ms %.3f ctas %.0f  per-CTA avg cycles: wait tmem_empty %.0f  wait full %.0f  mma loop %.0f\n",
           variant, ms, ctas, h[0] / ctas, h[1] / ctas, h[3] / ctas);
    unsigned long long h9; cudaMemcpy(&h9, dbg + 9, 8, cudaMemcpyDeviceToHost);
    if (variant == 0) {   // CTA timeline of this launch: span, per-SM busy fraction, gaps
      std::vector<unsigned long long> T(3 * (size_t)ctas);
      cudaMemcpy(T.data(), tl, T.size() * 8, cudaMemcpyDeviceToHost);
      unsigned long long t0 = ~0ull, t1 = 0;
      for (int i = 0; i < (int)ctas; ++i) { t0 = std::min(t0, T[3 * i]); t1 = std::max(t1, T[3 * i + 1]); }
      std::map<int, std::vector<std::pair<unsigned long long, unsigned long long>>> per;
      double busy = 0, dur = 0, dmin = 1e30, dmax = 0;
      for (int i = 0; i < (int)ctas; ++i) {
        per[(int)T[3 * i + 2]].push_back({T[3 * i], T[3 * i + 1]});
        const double dd = (double)(T[3 * i + 1] - T[3 * i]);
        busy += dd; dur += dd; dmin = std::min(dmin, dd); dmax = std::max(dmax, dd);
      }
      double gaps = 0; int ng = 0, maxper = 0;
      for (auto& kv : per) {
        auto v = kv.second; std::sort(v.begin(), v.end()); maxper = std::max(maxper, (int)v.size());
        for (size_t j = 1; j < v.size(); ++j) { gaps += (double)v[j].first - (double)v[j - 1].second; ++ng; }
      }
      printf("  timeline: span %.1f us, SMs used %zu, max CTAs/SM %d, CTA duration avg %.1f min %.1f max %.1f us, busy frac %.3f, avg gap between CTAs on an SM %.2f us\n",
             (t1 - t0) / 1e3, per.size(), maxper, dur / ctas / 1e3, dmin / 1e3, dmax / 1e3, busy / (148.0 * (t1 - t0)), ng ? gaps / ng / 1e3 : 0.0);
    }
    { unsigned long long e[8]; cudaMemcpy(e, dbg + 8, 56, cudaMemcpyDeviceToHost);
      printf("  epilogue phases (warp 4): bar0 %.0f rowpass0 %.0f colpass+bar0 %.0f bar1 %.0f rowpass1 %.0f colpass+bar1 %.0f\n",
             e[0] / ctas, e[1] / ctas, e[2] / ctas, e[3] / ctas, e[4] / ctas, e[5] / ctas); }
    printf("  prologue %.0f  epilogue-final %.0f  start->drained %.0f  staged0 %.0f rowpass0-done %.0f staged1 %.0f\n", h[4] / ctas, h[5] / ctas, h[6] / ctas, h[7] / ctas, h9 / ctas, h[8] / ctas);
  }
  return 0;
}

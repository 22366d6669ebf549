// Debug harness for gemm_tf32.cu (harness-only).  Includes the engine source directly.
#define NSERIES_TF32_DEBUG
#include "../paper_2602_11843_b200/csrc/gemm_tf32.cu"
#include <vector>
#include <cmath>
using namespace nseries;
int main() {
  int d = 128, ldp = 128;
  size_t n = (size_t)d * ldp;
  std::vector<float> hx(n), hy(n);
  for (size_t i = 0; i < n; ++i) { hx[i] = (float)((i * 37) % 11) - 5.f; hy[i] = (float)((i * 13) % 7) - 3.f; }
  float *X, *Y, *Xh, *Xl, *Yh, *Yl, *C;
  cudaMalloc(&X, n * 4); cudaMalloc(&Y, n * 4); cudaMalloc(&Xh, n * 4); cudaMalloc(&Xl, n * 4);
  cudaMalloc(&Yh, n * 4); cudaMalloc(&Yl, n * 4); cudaMalloc(&C, n * 4);
  cudaMemcpy(X, hx.data(), n * 4, cudaMemcpyHostToDevice); cudaMemcpy(Y, hy.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemset(C, 0, n * 4);
  launch_split_f32(X, d, Xh, Xl, nullptr, nullptr, ldp, d, false, 0);
  launch_split_f32(Y, d, nullptr, nullptr, Yh, Yl, ldp, d, false, 0);
  EpiParamsF32 ep{}; ep.ldp = ldp; ep.n_out = 1; ep.out_x[0] = C; ep.out_ld[0] = d; ep.alpha[0] = 1.f;
  float* dbg; cudaMalloc(&dbg, 4096); cudaMemset(dbg, 0, 4096);
  cudaMemcpyToSymbol(g_dbg, &dbg, sizeof(dbg));
  int rc = launch_gemm_tf32x3(Xh, Xl, Yh, Yl, d, ldp, ep, 0);
  cudaError_t e = cudaDeviceSynchronize();
  printf("launch rc=%d sync=%s\n", rc, cudaGetErrorString(e));
  std::vector<float> hc(n); cudaMemcpy(hc.data(), C, n * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0; int shown = 0;
  for (int i = 0; i < d; ++i) for (int j = 0; j < d; ++j) {
    double s = 0; for (int k = 0; k < d; ++k) s += (double)hx[i * d + k] * hy[k * d + j];
    double err = fabs(hc[i * d + j] - s); maxerr = fmax(maxerr, err);
    if (err > 1e-3 && shown < 8) { printf("(%d,%d) got %g want %g\n", i, j, hc[i * d + j], s); ++shown; }
  }
  std::vector<float> hd(256); cudaMemcpy(hd.data(), dbg, 1024, cudaMemcpyDeviceToHost);
  printf("smem A[0..7]: "); for (int i = 0; i < 8; ++i) printf("%g ", hd[i]); printf("\n");
  printf("X row0[0..7]: "); for (int i = 0; i < 8; ++i) printf("%g ", hx[i]); printf("\n");
  printf("smem B[0..7]: "); for (int i = 0; i < 8; ++i) printf("%g ", hd[64 + i]); printf("\n");
  printf("Y row0[0..7]: "); for (int i = 0; i < 8; ++i) printf("%g ", hy[i]); printf("\n");
  printf("max abs err %g ; C[0]=%g C[1]=%g C[128]=%g\n", maxerr, hc[0], hc[1], hc[128]);
  return 0;
}

// HISTORICAL (does not build against the current library, see tools/legacy/README.md).
// Harness-only: per-op phase timing (clock64, CTA 0 thread 0) of the 4-CTA cluster small kernel
// on an x9^2 plan at d = 64 (mainloop / epilogue / cluster barrier).
#define NSERIES_SMALL_PROFILE
#include "legacy/plan_small.cu"   // superseded kernels (moved out of the library in round 2)
#include <cstdio>
#include <vector>
using namespace nseries;
int main() {
  nseries_plan plan{};
  plan.n_steps = 2; plan.step[0] = 9; plan.step[1] = 9;
  if (finalize_plan(&plan, 81, 0) != NSERIES_OK) return 1;
  Program P;
  if (compile_plan(plan, false, &P) != NSERIES_OK) return 1;
  WarpProgram wp;
  if (build_cluster_program(P, &wp) != NSERIES_OK) return 1;
  const int d = 64;
  std::vector<double> h(d * d);
  for (int i = 0; i < d * d; ++i) h[i] = ((i * 2654435761u) % 1000) / 1000.0 * 0.02;
  double *A, *S; cudaMalloc(&A, d * d * 8); cudaMalloc(&S, d * d * 8);
  cudaMemcpy(A, h.data(), d * d * 8, cudaMemcpyHostToDevice);
  for (int it = 0; it < 5; ++it) launch_plan_cluster_f64(d, wp, A, S, nullptr, 0);
  cudaDeviceSynchronize();
  long long p[256]; cudaMemcpyFromSymbol(p, g_small_prof, sizeof(p));
  printf("ops %d slots %d rep %d (%s)\n", wp.n_ops, wp.n_slots, wp.n_rep, cudaGetErrorString(cudaGetLastError()));
  long long prev = p[0];
  for (int o = 0; o < wp.n_ops; ++o) {
    printf("op %2d: mainloop %6lld  epilogue %6lld  barrier %6lld cycles\n", o, p[1 + 3 * o] - prev,
           p[2 + 3 * o] - p[1 + 3 * o], p[3 + 3 * o] - p[2 + 3 * o]);
    prev = p[3 + 3 * o];
  }
  return 0;
}

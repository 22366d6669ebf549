// Harness-only: per-op phase clocks (CTA 0, thread 0) of the 4x2 cluster kernel on the x9^2
// plan at d = 64: wait (previous pushes + CTA barrier), mainloop, epilogue with pushes.
#define NSERIES_C2_PROFILE
#include "../paper_2602_11843_b200/csrc/plan_cluster2d.cu"
#include <cstdio>
#include <vector>
using namespace nseries;
int main() {
  nseries_plan plan{};
  plan.n_steps = 2; plan.step[0] = 9; plan.step[1] = 9;
  if (finalize_plan(&plan, 81, 0) != NSERIES_OK) return 1;
  Program P;
  if (compile_plan(plan, false, &P) != NSERIES_OK) return 1;
  static C2Program c2;
  if (build_cluster2d_program(P, &c2) != NSERIES_OK) return 1;
  const int d = 64;
  std::vector<double> h(d * d);
  for (int i = 0; i < d * d; ++i) h[i] = ((i * 2654435761u) % 1000) / 1000.0 * 0.02;
  double *A, *S; cudaMalloc(&A, d * d * 8); cudaMalloc(&S, d * d * 8);
  cudaMemcpy(A, h.data(), d * d * 8, cudaMemcpyHostToDevice);
  for (int it = 0; it < 5; ++it) launch_plan_cluster2d_f64(d, c2, A, S, nullptr, 0);
  cudaDeviceSynchronize();
  long long p[256]; cudaMemcpyFromSymbol(p, g_c2_prof, sizeof(p));
  printf("ops %d row %d col %d own %d (%s)\n", c2.n_ops, c2.n_row, c2.n_col, c2.n_own, cudaGetErrorString(cudaGetLastError()));
  long long prev = p[0];
  for (int o = 0; o < c2.n_ops; ++o) {
    printf("op %2d csync %d: wait %6lld  mainloop %6lld  epilogue %6lld cycles\n", o, c2.ops[o].csync, p[1 + 3 * o] - prev,
           p[2 + 3 * o] - p[1 + 3 * o], p[3 + 3 * o] - p[2 + 3 * o]);
    prev = p[3 + 3 * o];
  }
  return 0;
}

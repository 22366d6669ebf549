// Harness-only probe of the batched warp kernel (config 4 shape, 16384 x 32^2 fp32, x9x9 plan):
// builds the real op list through the library's host code and times the kernel compiled with
// -DNSERIES_BW_PROBE=0 (full) or 1 (mainloop only, epilogues replaced by a sink); with
// -DNSERIES_BW_TIMING also the clock64 time per phase of a warp-op (mainloop incl. the last
// HMMAs, group barrier, epilogue, group barrier).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2602_11843_b200/csrc/batched_warp.cu"
using namespace nseries;
int main(int argc, char** argv) {
  const int batch = 16384, d = 32;
  nseries_plan plan{};
  plan.n_steps = 2; plan.step[0] = 9; plan.step[1] = 9;
  if (finalize_plan(&plan, 81, 0) != NSERIES_OK) { printf("plan fail\n"); return 1; }
  Program P;
  if (compile_plan(plan, false, &P) != NSERIES_OK) { printf("compile fail\n"); return 1; }
  WarpProgram wp;
  if (build_warp_program(P, &wp) != NSERIES_OK) { printf("warp program fail\n"); return 1; }
  printf("ops %d slots %d\n", wp.n_ops, wp.n_slots);
  std::vector<float> h((size_t)batch * d * d);
  for (size_t i = 0; i < h.size(); ++i) h[i] = ((i * 2654435761u) % 1000) / 1000.f * 0.05f;
  float *A, *S;
  cudaMalloc(&A, h.size() * 4); cudaMalloc(&S, h.size() * 4);
  cudaMemcpy(A, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  for (unsigned delay : {0u, 200u, 400u, 800u})
  for (int wpm : {1, 2}) {
    wp.probe_delay_ns = delay;
    char buf[8]; snprintf(buf, 8, "%d", wpm); setenv("NSERIES_BATCHED_WPM", buf, 1);
    for (int i = 0; i < 3; ++i) launch_batched_warp_f32(A, d * d, nullptr, S, d * d, nullptr, batch, d, wp, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) launch_batched_warp_f32(A, d * d, nullptr, S, d * d, nullptr, batch, d, wp, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("probe %d delay %u wpm %d: %.1f us (%s)\n", NSERIES_BW_PROBE, delay, wpm, ms / 20 * 1e3, cudaGetErrorString(cudaGetLastError()));
#ifdef NSERIES_BW_TIMING
    {   // per-phase clocks per warp-op, averaged (one extra launch with the counters zeroed)
      unsigned long long z[4] = {0, 0, 0, 0}, r[4];
      cudaMemcpyToSymbol(g_bwt, z, sizeof(z));
      launch_batched_warp_f32(A, d * d, nullptr, S, d * d, nullptr, batch, d, wp, 0);
      cudaMemcpyFromSymbol(r, g_bwt, sizeof(r));
      const double n = (double)batch * wp.n_ops * wpm;   // warp-ops
      printf("  clk per warp-op: mainloop %.0f  barrier1 %.0f  epilogue %.0f  barrier2 %.0f\n",
             r[0] / n, r[1] / n, r[2] / n, r[3] / n);
    }
#endif
  }
  return 0;
}

// gemm_tf32_b128.cu -- the fp32 engine of gemm_tf32.cu in its small-grid configuration:
// 128x128 CTA tiles (pairs of 256 x 128), BK = 32, 3 stages, and the cross terms
// hi*lo + lo*hi in their own full-K TMEM accumulator (NSERIES_TF32_XACC, see gemm_tf32.cu).
// Twice the tiles of the 128x256 default: better for d up to ~1600 (d = 1024: 0.054 -> 0.040
// ms per product), worse at 4096 (0.72 -> 0.80).  Selected per size in api.cu.
#define NSERIES_TF32_VARIANT 1
#define NSERIES_TF32_XACC 1
#define NSERIES_TF32_API(name) name##_b128
#include "gemm_tf32.cu"

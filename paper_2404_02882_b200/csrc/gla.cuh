// gla.cuh -- generalised-decay path (kernels_gla.cu): plan and launch interfaces.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lasp {

struct GlaPlan {
  int64_t B, C, H, D;   // batch, n_local, heads (= kv heads), head_dim
  int64_t seg_len;      // multiple of 8 (the kernels' token tile)
  int64_t nseg;         // >= 1
};

// co-resident CTAs per SM of the slowest-occupancy pass (the host sizes the segment count to whole waves)
int gla_slots_per_sm(int D);
// F1 (rev = 0: x = k, y = v) / B1 (rev = 1: x = q, y = do): per-segment local states into seg
// [B][H][nseg][D][D] (B1: G'_p) and segment log-decay sums into ls [B][H][nseg][D]
cudaError_t gla_launch_state(const GlaPlan& p, int rev, const float* x, const float* y, const float* lg, float* seg,
                             float* ls, cudaStream_t st);
// F2 (rev = 0): cache[p] = P_p, cache[nseg] = final, fin = final; B2 (rev = 1): seg[p] <- R_p in place,
// fin = dKV_out. lsum (optional): the rank's total log decay per key row [B][H][D]
cudaError_t gla_launch_fold(const GlaPlan& p, int rev, const float* init, float* seg, const float* ls, float* cache,
                            float* fin, float* lsum, cudaStream_t st);
// ring hop: out = Diag(exp(lsum)) in + local
cudaError_t gla_launch_combine(const GlaPlan& p, const float* in, const float* local, const float* lsum, float* out,
                               cudaStream_t st);
// F3: o from the cache's prefix states
cudaError_t gla_launch_out(const GlaPlan& p, const float* q, const float* k, const float* v, const float* lg,
                           const float* cache, float* o, cudaStream_t st);
// B3: dQ, dV, then dK with the decay gradient (rseg: R_p from the B2 fold; status: cache-tag poison word)
cudaError_t gla_launch_bwd(const GlaPlan& p, const float* q, const float* k, const float* v, const float* lg,
                           const float* d_o, const float* cache, float* rseg, float* dq, float* dk, float* dv,
                           float* dlg, const unsigned* status, cudaStream_t st);

}  // namespace lasp

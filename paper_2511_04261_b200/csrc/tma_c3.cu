// tma_c3.cu -- K1 / K2 TMA instantiations for C = 3 (see tma_kernels.cuh).
#include "tma_kernels.cuh"

namespace dppx {

StatsKernel select_stats_tma_c3(int b, int n, bool adaptive, bool packed) {
  if (packed) return adaptive ? pick_b<3, true, true>(b, n) : pick_b<3, false, true>(b, n);
  return adaptive ? pick_b<3, true, false>(b, n) : pick_b<3, false, false>(b, n);
}

StatsKernel select_stats_var_c3(int b, int n) { return pick_var<3>(b, n); }

// Uniform b = 4, two cell rows per unit (wide frames).
StatsKernel select_uniform_b4_rows2_c3() { return k_stats_tma<3, 1, 1, false, false, false, 2>; }

StatsKernel select_uniform_any_c3(int b) { return pick_uniform_any<3>(b); }

StatsKernel select_adaptive_any_c3(int b, int n) { return pick_adaptive_any<3>(b, n); }

ExpandKernel select_expand_uany_c3(int b) { return pick_expand_uany<3>(b); }

ExpandKernel select_expand_aany_c3(int b, int n) { return pick_expand_aany<3>(b, n); }

ExpandKernel select_expand_tma_c3(int b, int n, bool adaptive, bool packed, int split) {
  if (split == 2 && !packed) return adaptive ? pick_expand_split<3, true, 2>(b, n) : pick_expand_split<3, false, 2>(b, n);
  if (split == 4 && !packed) return adaptive ? pick_expand_split<3, true, 4>(b, n) : pick_expand_split<3, false, 4>(b, n);
  if (split > 1) return nullptr;
  if (packed) return adaptive ? pick_expand<3, true, true>(b, n) : pick_expand<3, false, true>(b, n);
  return adaptive ? pick_expand<3, true, false>(b, n) : pick_expand<3, false, false>(b, n);
}

}  // namespace dppx

// tcgen05 Gram pair: host-side dispatch (the kernel is k_gram_tc2, mg_tc2.cu).
//
// Round 1 also carried a converter-based v1 Gram (3-piece TF32) and a
// tensor-core update that formed X Yx itself on tcgen05; both cost LOBPCG
// iterations (+15 % .. +210 %) and are gone.  Round 2's update kernel
// (mg_tc3.cu) forms only the corrections X (Yx - I) + P on the tensor core
// and keeps the iteration count (profiles/r2_update_tc3.md); an Ozaki-style
// int8 fixed-point variant was emulated and rejected
// (profiles/r2_update_tc_numerics.md).
#include "mg_tc.cuh"

namespace mg {

bool gram_tc_supported(int w) {
  const char *e = getenv("MG_TC");
  if (e && e[0] == '0') return false;
  // 48 < w <= 128: below that the CUDA-core k_gram2 is faster (the per-tile
  // pipeline cost of the tensor-core kernel dominates small tiles)
  return w > 48 && w <= 128 && w % 4 == 0;
}

void gram_pair_tc(mg_ctx *ctx, int64_t n, int ld, int w, const float *S, const float *AS,
                  const float *b, double *GB, double *GA, DBuf<double> &part) {
  require(gram_tc2_supported(w, ld), MG_ERR_INTERNAL,
          "tc Gram: needs 32 < w <= 128, w % 4 == 0, ld % 4 == 0");
  gram_pair_tc2(ctx, n, ld, w, S, AS, b, GB, GA, part);
}

}  // namespace mg

// Instantiations of the two-output-planes-per-CTA kernel (ndc_correlate_pair.cuh).
#include "ndc_correlate_pair.cuh"

namespace ndc {

cudaError_t launch_correlate_pair(int kx, int sh, const CUtensorMap& map, const CorrGeom& g, const CorrArgs& a,
                                  const TapBlock& taps, int batch, int nz_out, cudaStream_t s) {
  using namespace corr;
#define NDC_PAIR(K)                                                              \
  case K:                                                                        \
    return sh == 0 ? launch_pair<K, 0, 2>(map, g, a, taps, batch, nz_out, s)     \
                   : launch_pair<K, 2, 2>(map, g, a, taps, batch, nz_out, s);
  switch (kx) {
    NDC_PAIR(7)
    NDC_PAIR(9)
    default: return cudaErrorInvalidValue;
  }
#undef NDC_PAIR
}

}  // namespace ndc

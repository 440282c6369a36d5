// Instantiations of the correlation kernel (ndc_correlate.cuh) for register-window
// shift SH = 2 and RY = 2 output rows per thread; one translation unit per
// (SH, RY) pair so the sets compile in parallel.
#include "ndc_correlate.cuh"

namespace ndc {

cudaError_t launch_correlate_sh2_ry2(int kx, const CUtensorMap& map, const CorrGeom& g,
                                      const CorrArgs& a, const TapBlock& taps, int batch,
                                      int nz_out, cudaStream_t s, cudaStream_t s_edge) {
  using namespace corr;
  NDC_KX_SWITCH(2, 2)
}

}  // namespace ndc

// Instantiations of the correlation kernel for register-window shift SH = 0
// (ndc_correlate.cuh); split from ndc_kernels.cu so the two sets compile in parallel.
#include "ndc_correlate.cuh"

namespace ndc {

cudaError_t launch_correlate_sh0(int kx, const CUtensorMap& map, const CorrGeom& g,
                                  const CorrArgs& a, const TapBlock& taps, int batch, int nz_out,
                                  cudaStream_t s) {
  using namespace corr;
  NDC_KX_SWITCH(0)
}

}  // namespace ndc

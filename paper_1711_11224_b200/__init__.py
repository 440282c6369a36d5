"""B200-native hot path of arXiv 1711.11224's convolution-only deconvolution.

`paper_1711_11224_b200.ndconv` mirrors the reference's ndconv API (conv_full,
adjoint_apply, objective, estimate_step, kkt_residual, deconv_pg, deconv_rl, ...) over
the C-ABI of libndconv_b200.so (include/ndconv_b200.h); `synth` generates the seeded
BASELINE inputs.
"""
from . import ndconv  # noqa: F401
from .ndconv import *  # noqa: F401,F403

__version__ = "0.1.0"

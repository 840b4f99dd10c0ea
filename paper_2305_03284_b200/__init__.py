"""B200-native DDH-MBIR hot path (arXiv 2305.03284): sm_100a CUDA kernels
behind the C ABI of include/ddh.h, with a thin ctypes binding.

    from paper_2305_03284_b200 import DDH
    ctx = DDH(n=256, streams=64, noise_var=0.287)
    ctx.step(y_frames, phi_out, r_out)     # y: cuda complex64 [T][S][N][N]
"""
from .ddh import DDH, DDHSynth, DDHError, DdhParams, default_params, load_library, LIB_PATH, EXPORTS  # noqa: F401

__all__ = ["DDH", "DDHSynth", "DDHError", "DdhParams", "default_params", "load_library", "LIB_PATH", "EXPORTS"]

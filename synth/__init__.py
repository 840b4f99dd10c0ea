"""Seeded synthetic DH frame sequences shaped like the paper's workloads.

This module is the ONE thing the oracle and the CUDA path both use: it
produces inputs (frames y, truth phases, truth reflectance) and holds none of
the estimator's arithmetic (no Normalize, no back-projection, no E-step, no
ICD).  It synthesises data with the paper's forward model, Eq. 1:
y_n = D_a D(e^{j phi_n}) F_c^{-1} g_n + w_n, with its own FFT calls.

Stand-ins: the paper simulates a USAF 1951 chart and
the frozen-flow model of [srinath2015], neither of which is in this
container.  The BASELINE.json configs replace them with blurred-uniform
reflectance fields and FFT-method Kolmogorov screens translated rigidly
(frozen flow, "no boiling").
"""
from .sim import *  # noqa: F401,F403
from .sim import CONFIGS, make_stream, make_batch, recon_noise_var, flow_velocity  # noqa: F401

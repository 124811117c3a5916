"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA-side tests/bench.

This package holds NO arithmetic of the FTK method (no quadrature, no Bessel
functions, no SVD, no FFT, no inner products).  It only draws seeded
Gaussian-blob parameters and evaluates their analytic Fourier transforms on a
polar grid whose radial nodes are passed in by the caller, or samples them at pixel centres.
"""
from .workloads import (  # noqa: F401
    CONFIGS, Config, config, shift_list, delta_max, draw_items, blob_params,
    polar_samples, add_noise, make_polar_set, planted_truth, pixel_images, draw_pixel_items, ctf_filters,
)

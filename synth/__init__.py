"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This package holds NO arithmetic of the paper's method (no encoding, no
convolution, no output-size rule): only the clustered-ReLU activation
generator, He-normal weights, integer-valued fixtures and the BASELINE.json
workload catalogue (shapes, pads, strides, densities, seeds).  See
DESIGN.md "Input recipe" and SURVEY.md Appendix B.
"""
from .gen import clustered_relu, he_normal, int_map, int_weights, random_sparse  # noqa: F401
from .configs import CATALOG, CONFIGS, cfg5_layers, layer_desc  # noqa: F401

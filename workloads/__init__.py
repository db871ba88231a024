"""Seeded synthetic workloads (configs + input generators).

Shared by the oracle and the CUDA path; holds none of the method's arithmetic.
"""
from .configs import CONFIGS, VARIANTS, Config, get  # noqa: F401

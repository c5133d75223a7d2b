"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds *only* input generation (the κ field, the continuum ids ψ_j
and the BASELINE configuration table, the source f of the paper's experiments).  It contains none of the method's
arithmetic (no stiffness, constraints, solves or reductions), so both sides of
every parity test may import it without sharing method code.
"""
from .media import (CONFIGS, Config, make_medium, paper_medium, paper_source, random_medium, layered_medium,
                    periodic_medium)

__all__ = ["CONFIGS", "Config", "make_medium", "paper_medium", "paper_source", "random_medium", "layered_medium", "periodic_medium"]

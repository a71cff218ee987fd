"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no stencils, no solvers,
no time stepping): only the recipes that turn a seed and a grid size into
initial fields, exactly as BASELINE.json's configs describe them.
Both `oracle/` and `paper_1811_11842_b200/` (via tests / bench) consume it.
"""
from .inputs import (  # noqa: F401
    GridSpec,
    initial_fields,
    random_field,
    CONFIGS,
)

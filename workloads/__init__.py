"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the method (no distances, no search, no graph logic): it only draws
vectors, queries, id sets and operation streams from counter-based (Philox) generators, so that the oracle
(`oracle/`) and the CUDA path (`paper_2601_08528_b200/`) can be fed identical inputs without sharing code.
Recipes and the reasons for them are in DESIGN.md §"Input recipe".
"""
from .synth import (  # noqa: F401
    GLM,
    GCL,
    CONFIGS,
    config_spec,
    base_rows,
    query_rows,
    int_rows,
    random_graph,
    random_tombstones,
    pack_tomb,
)

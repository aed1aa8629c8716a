"""Seeded synthetic inputs shared by the tests, the bench and the oracle legs.

This package holds NONE of the method's arithmetic: no FIT coefficients, no CFL
bound, no curls, no polynomial coefficients.  It only describes workloads (grid
sizes, per-cell materials, PEC cells, source records, initial fields) with numpy
``default_rng`` seeds, exactly as SURVEY.md 8(d) / DESIGN.md "input recipe" state.
Both the CUDA path (through the C ABI) and the oracle consume these descriptions
and each derives its own coefficients from them.
"""
from .configs import (  # noqa: F401
    EPS0, MU0, C0, Z0, Source, Workload, SOURCE_KINDS, gauss_sine, layered_eps,
    config_c1, config_c2, config_c3, config_c3r, config_c4, config_c5, config_c5s, config_wave2d, small_cavity,
    random_fields, spiral_pec_cells,
)

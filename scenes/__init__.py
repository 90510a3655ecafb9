"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the PBNG method (no rest-shape inverse, no volumes, no stresses,
no colouring): it only lays out vertex lattices, tetrahedra, Dirichlet sets, initial states, material
draws and weak-constraint records. See DESIGN.md "Input recipe".
"""
from .generators import (  # noqa: F401
    Scene,
    kuhn_grid,
    five_tet_grid,
    config1_tiny_cube,
    config2_twisted_bar,
    config3_hetero_cube,
    config4_batched,
    config5_muscle_stack,
    make_config,
    SEED_BASE,
)

"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This package holds NONE of the method's arithmetic (no SBP operator, no metric terms, no
flux, no SAT, no interpolation, no time-integration weights).  It only builds mesh
coordinates, boundary-condition tags, priorities, step multiples, step sizes and seeded
initial conditions for the five workloads named in BASELINE.json (see DESIGN.md §3 for the
recipe of each).  Both `oracle/` and the CUDA path consume these arrays; neither is
imported here.
"""
from .configs import (OVERSET, FARFIELD, WALL, PERIODIC, make_config, config_names,
                      primitive_to_conserved)

__all__ = ["OVERSET", "FARFIELD", "WALL", "PERIODIC", "make_config", "config_names",
           "primitive_to_conserved"]

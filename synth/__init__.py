"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NONE of the halo-exchange arithmetic (no planes, no
predicates, no maps, no shifts): it only draws atom positions and forces.
See DESIGN.md "Input recipe".
"""
from .water import water_box, forces_int, forces_normal, wrap_f32, displacements, velocities
from .configs import CONFIGS, Config, get_config

__all__ = ["water_box", "forces_int", "forces_normal", "wrap_f32", "displacements", "velocities", "CONFIGS", "Config", "get_config"]

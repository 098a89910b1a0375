"""CPU oracle — TEST INFRASTRUCTURE ONLY (see halo_oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product never imports it.
"""
from .halo_oracle import (decompose, force_halo, coord_halo_step, pulse_list, planes, home_cell, rank_of,
                          cell_of, check_geometry, layout_summary, RankState, PulseInfo, wrap_coord, migrate,
                          pme_gather, pme_return)

__all__ = ["decompose", "force_halo", "coord_halo_step", "pulse_list", "planes", "home_cell", "rank_of", "cell_of",
           "check_geometry", "layout_summary", "RankState", "PulseInfo", "wrap_coord", "migrate", "pme_gather", "pme_return"]

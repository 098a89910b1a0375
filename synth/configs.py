"""The BASELINE.json configurations as concrete synthetic inputs.

Index convention everywhere in this repo: dimension 0 = x, 1 = y, 2 = z;
``grid = (np_x, np_y, np_z)``; ``pulses = (p_x, p_y, p_z)``.
A 1D grid splits z, a 2D grid splits z and y (reading R6).
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class Config:
    name: str
    n_atoms: int
    L: tuple
    grid: tuple
    pulses: tuple
    rc: float
    desc: str
    slab: tuple | None = None

    @property
    def nranks(self) -> int:
        return self.grid[0] * self.grid[1] * self.grid[2]


CONFIGS = {
    # BASELINE.json configs[0]: 3,000-atom SPC box, 1D 2-rank, rc 1.0, 1 pulse
    "C1": Config("C1", 3000, (3.104, 3.104, 3.104), (1, 1, 2), (0, 0, 1), 1.0,
                 "3,000-atom SPC water box, 1D 2-rank, rc 1.0 nm, 1 pulse"),
    # configs[1]: 24k RNase-like water, 2D 4-rank grid, 1 pulse per dim
    "C2": Config("C2", 24000, (6.208, 6.208, 6.208), (1, 2, 2), (0, 1, 1), 1.0,
                 "24k-atom RNase-like water box, 2D 4-rank grid, 1 pulse per dim"),
    # configs[2]: 82k benchMEM-like, 3D 2x2x2 with forwarding
    "C3": Config("C3", 81744, (10.8, 10.2, 9.6), (2, 2, 2), (1, 1, 1), 1.0,
                 "82k-atom benchMEM-like system, 3D 2x2x2 grid with forwarding"),
    # configs[3]: 1.07M STMV-like, 1D/2D/3D on 2/4/8
    "C4-1D": Config("C4-1D", 1066629, (21.68, 21.68, 21.68), (1, 1, 2), (0, 0, 1), 1.0,
                    "1.07M-atom STMV-like box, 1D 2-rank grid"),
    "C4-2D": Config("C4-2D", 1066629, (21.68, 21.68, 21.68), (1, 2, 2), (0, 1, 1), 1.0,
                    "1.07M-atom STMV-like box, 2D 4-rank grid"),
    "C4-3D": Config("C4-3D", 1066629, (21.68, 21.68, 21.68), (2, 2, 2), (1, 1, 1), 1.0,
                    "1.07M-atom STMV-like box, 3D 2x2x2 grid"),
    # configs[4]: 45k box on 8 ranks, 2 pulses (1D along z, w = 0.957 nm < rc)
    "C5": Config("C5", 45000, (7.656, 7.656, 7.656), (1, 1, 8), (0, 0, 2), 1.0,
                 "45k-atom box on 8 ranks (1D z), 2 pulses per dim (latency-bound limit)"),
    # C4-bw: bandwidth probe, C4 1D with the cutoff swept up to 8 nm
    "C4-bw2": Config("C4-bw2", 1066629, (21.68, 21.68, 21.68), (1, 1, 2), (0, 0, 1), 2.0,
                     "C4 1D 2-rank, rc 2 nm (bandwidth probe)"),
    "C4-bw5": Config("C4-bw5", 1066629, (21.68, 21.68, 21.68), (1, 1, 2), (0, 0, 1), 5.0,
                     "C4 1D 2-rank, rc 5 nm (bandwidth probe)"),
    "C4-bw8": Config("C4-bw8", 1066629, (21.68, 21.68, 21.68), (1, 1, 2), (0, 0, 1), 8.0,
                     "C4 1D 2-rank, rc 8 nm (bandwidth probe)"),
    # small oracle-self cases (SURVEY.md §8(c) parity matrix)
    "T3D": Config("T3D", 1500, (2.46, 2.46, 2.46), (2, 2, 2), (1, 1, 1), 1.0,
                  "tiny 3D 2x2x2 water box"),
    "T2P": Config("T2P", 2700, (3.0, 3.0, 3.0), (1, 1, 3), (0, 0, 2), 1.25,
                  "tiny 1D 3-rank box with 2 pulses"),
    "T2D": Config("T2D", 2100, (3.0, 3.0, 2.4), (1, 2, 2), (0, 1, 1), 0.9,
                  "tiny 2D 2x2 box"),
    "T4x2": Config("T4x2", 4002, (6.0, 4.4, 4.2), (4, 2, 1), (2, 1, 0), 2.0,
                   "4x2x1 grid with rc 2.0 nm: 2 x-pulses, 1 y-pulse"),
}


def get_config(name: str) -> Config:
    try:
        return CONFIGS[name]
    except KeyError as e:
        raise KeyError(f"unknown config {name!r}; known: {sorted(CONFIGS)}") from e

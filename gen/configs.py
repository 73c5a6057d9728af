"""The BASELINE.json workloads, as generator calls.

C1 R-MAT s10 ef16, p=2   -- configs[0], the oracle finishes in seconds
C2 R-MAT s20 ef16, p=8   -- configs[1]
C3 ER n=2^24, d=32       -- configs[2]
C4 grid 8192^2 (+10% diagonals), n=2^26 -- configs[3]
C5 Graph500 R-MAT s26 ef32 -- configs[4]
"""
from __future__ import annotations

from dataclasses import dataclass

from . import er, grid, rmat


@dataclass(frozen=True)
class Config:
    name: str
    desc: str
    p: int
    kind: str
    args: tuple

    def generate(self):
        if self.kind == "rmat":
            return rmat(*self.args)
        if self.kind == "er":
            return er(*self.args)
        if self.kind == "grid":
            return grid(*self.args)
        raise ValueError(self.kind)


CONFIGS = {
    "c1": Config("c1", "R-MAT scale 10, edge factor 16, 2x2 blocks", 2, "rmat", (10, 16, 1)),
    "c2": Config("c2", "R-MAT scale 20, edge factor 16, 8x8 blocks", 8, "rmat", (20, 16, 1)),
    "c3": Config("c3", "Erdos-Renyi n=2^24, avg degree 32, 4x4 blocks", 4, "er", (1 << 24, 32, 1)),
    # p = 1: measured on B200 (round 2: count 1.09 / 1.45 / 1.65 / 1.84 / 2.09 ms at
    # p = 1 / 2 / 3 / 4 / 6): a low-degree grid gains nothing from narrow parts and pays
    # per (edge, part) pair
    "c4": Config("c4", "grid 8192^2 + 10% diagonals (road-like), n=2^26, 1x1 block", 1, "grid",
                 (8192, 0.1, 1)),
    # profiling stand-in for c5 (same generator and p at 1/4 of the vertices; ncu-sized)
    "c5s": Config("c5s", "R-MAT scale 24, edge factor 32, 16x16 blocks", 16, "rmat", (24, 32, 1)),
    "c5": Config("c5", "Graph500 R-MAT scale 26, edge factor 32, 16x16 blocks", 16, "rmat", (26, 32, 1)),
}

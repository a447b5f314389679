"""Sweep-level types of the drop-in API (reference sweep.py).

The reference's sweep/apply_update pair (sweep.py:175-280) is one fused
CUDA kernel here (csrc/ws_kernels.cuh, k_update); what remains on the host
is the error type and the traversal-strategy markers, which the device
accepts for signature compatibility and ignores (CUDA tiling replaces
RowWise/CellWise/Tiled; results never depended on them, sweep.py:9-12).
"""

from __future__ import annotations

from dataclasses import dataclass

from .kernels import Direction


@dataclass(frozen=True)
class RowWise:
    pass


@dataclass(frozen=True)
class CellWise:
    pass


@dataclass(frozen=True)
class Tiled:
    tile_w: int = 64
    tile_h: int = 64

    def __post_init__(self):
        if self.tile_w < 1 or self.tile_h < 1:
            raise ValueError(f"tile sides must be >= 1, got {self.tile_w}x{self.tile_h}")


Strategy = RowWise | CellWise | Tiled


class SweepError(RuntimeError):
    """Kernel failure located at one interface (reference sweep.py:68-75)."""

    def __init__(self, direction: Direction, i: int, j: int, cause: Exception):
        super().__init__(f"{direction.value}-interface (i={i}, j={j}): {cause}")
        self.direction = direction
        self.i = i
        self.j = j
        self.__cause__ = cause

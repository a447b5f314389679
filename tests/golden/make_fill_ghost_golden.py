"""Golden vectors for fill_ghost from the REFERENCE itself (build container
only; the GPU box reads the committed JSON).

    python tests/golden/make_fill_ghost_golden.py

Writes tests/golden/fill_ghost_golden.json: for every (bc_x, bc_y) pair and
a few shapes (ncomp 1-3, small and n == num_ghost), a seeded field whose
ghost frame holds garbage, and the array after reference
``wavesweep.grid.fill_ghost`` (grid.py:179-193: x pass over the full y
extent, then the y pass, so corners come from the x-filled columns).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import load_reference  # noqa: E402

CASES = [  # ncomp, nx, ny, bc_x, bc_y, seed
    (3, 5, 4, "periodic", "periodic", 0),
    (3, 5, 4, "extrapolate", "extrapolate", 1),
    (2, 6, 3, "periodic", "extrapolate", 2),
    (2, 6, 3, "extrapolate", "periodic", 3),
    (1, 2, 2, "periodic", "periodic", 4),
    (4, 7, 2, "extrapolate", "periodic", 5),
]


def main():
    W = load_reference()
    from wavesweep.grid import BoundaryCondition, GridSpec, StateField
    out = []
    for ncomp, nx, ny, bx, by, seed in CASES:
        rng = np.random.default_rng(seed)
        spec = GridSpec(nx=nx, ny=ny, dx=1.0 / nx, dy=1.0 / ny, num_eqn=ncomp, num_aux=0)
        f = StateField(spec)
        f.data[...] = rng.normal(size=f.data.shape)       # ghosts start as garbage
        before = f.data.copy(order="F")
        W.grid.fill_ghost(f, BoundaryCondition(bx), BoundaryCondition(by))
        out.append({"ncomp": ncomp, "nx": nx, "ny": ny, "bc_x": bx, "bc_y": by, "seed": seed,
                    "before": before.ravel(order="F").tolist(),
                    "after": f.data.ravel(order="F").tolist()})
    with open(os.path.join(HERE, "fill_ghost_golden.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_fill_ghost_golden.py",
                   "source": "reference wavesweep.grid.fill_ghost", "cases": out}, fh)
    print(f"wrote {len(out)} cases")


if __name__ == "__main__":
    main()

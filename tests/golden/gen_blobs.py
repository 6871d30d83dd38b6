"""Golden checkpoint blobs from the REFERENCE (grid.py:236-277).

Run in the build container, where the reference is mounted read-only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_blobs.py

For a few arrays / decompositions it fills every owned tile's interior with
seeded values, bumps epochs and grows ghost frames, then stores the reference's
`checkpoint_blob` bytes (header + little-endian interior) per (tile, array) in
blobs.json next to this script. The tests only read blobs.json.
"""

from __future__ import annotations

import json
import os

import numpy as np

from elastencil.grid import ArrayInfo, TileStore, checkpoint_blob, decompose  # reference

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = [
    # (shape, workers, odf, ghost depth, epoch bumps)
    ((64,), 2, 2, (1,), 3),
    ((24, 40), 1, 1, (1, 1), 0),
    ((32, 48), 4, 1, (2, 3), 5),
    ((36, 24), 2, 3, (1, 2), 1),
]


def main():
    out = []
    for k, (shape, workers, odf, depth, bumps) in enumerate(CASES):
        decomp = decompose(shape, workers, odf)
        store = TileStore(decomp, list(decomp.all_coords()))
        store.create_array(ArrayInfo(k, shape))
        store.ensure_ghost_capacity(k, depth)
        rng = np.random.default_rng(1000 + k)
        for _ in range(bumps):
            store.bump_local_epoch(k)
        for coords, tile in sorted(store.tiles.items()):
            view = store.interior_view(tile, k)
            view[...] = np.round(rng.uniform(-8, 8, view.shape), 6)
            out.append({"case": k, "shape": list(shape), "workers": workers, "odf": odf,
                        "depth": list(depth), "coords": list(coords), "epoch": tile.local_epoch[k],
                        "interior": view.ravel().tolist(), "ext": list(view.shape),
                        "blob": checkpoint_blob(store, tile, k).hex()})
    with open(os.path.join(HERE, "blobs.json"), "w") as f:
        json.dump(out, f)
    print(f"{len(out)} blobs")


if __name__ == "__main__":
    main()

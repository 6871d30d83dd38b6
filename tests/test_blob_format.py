"""Checkpoint blob format (grid.py:236-277) pinned to the reference's own
bytes: tests/golden/blobs.json holds `checkpoint_blob` output of the reference
for rank-1/2 tiles with grown ghost frames and bumped epochs
(tests/golden/gen_blobs.py). CPU: header packing and payload layout; GPU: the
GpuTileStore export/adopt round trip through HBM."""

import json
import os

import numpy as np
import pytest

from paper_2512_19851_b200.tiles import blob_header, parse_blob_header

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "blobs.json")))


@pytest.mark.parametrize("g", GOLD, ids=lambda g: f"case{g['case']}-{g['coords']}")
def test_header_and_payload_match_reference(g):
    interior = np.asarray(g["interior"], dtype="<f8").reshape(g["ext"])
    ours = blob_header(g["case"], tuple(g["coords"]), tuple(g["ext"]), tuple(g["depth"]), g["epoch"])
    assert ours + interior.tobytes() == bytes.fromhex(g["blob"])
    a, coords, ext, depth, epoch, hs = parse_blob_header(bytes.fromhex(g["blob"]))
    assert (a, list(coords), list(ext), list(depth), epoch) == (g["case"], g["coords"], g["ext"], g["depth"],
                                                               g["epoch"])


@pytest.mark.gpu
def test_gpu_export_and_adopt_round_trip():
    from paper_2512_19851_b200.device import Device
    from paper_2512_19851_b200.tiles import ArrayInfo, GpuTileStore, decompose

    dev = Device(0)
    try:
        by_case: dict = {}
        for g in GOLD:
            by_case.setdefault(g["case"], []).append(g)
        for case, blobs in by_case.items():
            g0 = blobs[0]
            shape = tuple(g0["shape"])
            decomp = decompose(shape, g0["workers"], g0["odf"])
            # export: interiors uploaded, frame grown, epochs bumped -> same bytes
            src = GpuTileStore(dev, decomp, list(decomp.all_coords()))
            src.create_array(ArrayInfo(case, shape))
            src.ensure_ghost_capacity(case, tuple(g0["depth"]))
            src.bump_local_epoch(case, g0["epoch"])
            for g in blobs:
                src.upload_interior(tuple(g["coords"]), case,
                                    np.asarray(g["interior"]).reshape(g["ext"]))
            for g in blobs:
                assert src.checkpoint_blob(tuple(g["coords"]), case) == bytes.fromhex(g["blob"])
            # adopt into a fresh store: same interiors, zeroed frame, epochs
            dst = GpuTileStore(dev, decomp, list(decomp.all_coords()))
            dst.create_array(ArrayInfo(case, shape))
            for g in blobs:
                assert dst.adopt_blob(bytes.fromhex(g["blob"])) == (case, tuple(g["coords"]), g["epoch"])
            np.testing.assert_array_equal(dst.fetch(case), src.fetch(case))
            for g in blobs:
                assert dst.checkpoint_blob(tuple(g["coords"]), case) == bytes.fromhex(g["blob"])
            # a worker that owns none of the tiles adopts them (grid.py:271 setdefault)
            # at the blob's depth, with the blob's epochs
            empty = GpuTileStore(dev, decomp, [])
            empty.create_array(ArrayInfo(case, shape))
            for g in blobs:
                empty.adopt_blob(bytes.fromhex(g["blob"]))
                assert empty.checkpoint_blob(tuple(g["coords"]), case) == bytes.fromhex(g["blob"])
            assert empty.local_epoch(case) == g0["epoch"] and len(empty.tiles) == len(blobs)
            src.release()
            dst.release()
            empty.release()
    finally:
        dev.close()

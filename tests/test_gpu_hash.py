"""est_hash_box (include/est.h): the device content hash equals its numpy
restatement (oracle.content_hash) for fp64 / fp32 arrays of rank 1-3 under
several decompositions, and one flipped bit anywhere changes it."""

import numpy as np
import pytest

from oracle.oracle import content_hash
from paper_2512_19851_b200.session import GpuJob
from paper_2512_19851_b200.wire import DTYPE_F32, DTYPE_F64

pytestmark = pytest.mark.gpu


def _upload(job, aid, data):
    for st in job.stores:
        for coords in st.tiles:
            org = st.decomp.tile_origin(data.shape, coords)
            ext = st.decomp.tile_extents(data.shape)
            st.upload_interior(coords, aid, data[tuple(slice(o, o + e) for o, e in zip(org, ext))])


@pytest.mark.parametrize("shape,workers,odf", [((1000,), 2, 2), ((96, 130), 1, 1), ((96, 128), 2, 2),
                                               ((40, 33, 70), 1, 1), ((48, 20, 36), 4, 1), ((64, 9, 130), 2, 4)])
@pytest.mark.parametrize("dtype", [DTYPE_F64, DTYPE_F32])
def test_device_hash_matches_numpy(shape, workers, odf, dtype):
    rng = np.random.default_rng(sum(shape) + dtype)
    data = rng.standard_normal(shape).astype(np.float64 if dtype == DTYPE_F64 else np.float32)
    with GpuJob(workers, odf) as job:
        aid = job.create_array(shape, dtype)
        _upload(job, aid, data)
        h = job.hash(aid)
        assert h == content_hash(data)
        flat = data.reshape(-1).copy()
        k = int(rng.integers(flat.size))
        flat.view(np.uint64 if dtype == DTYPE_F64 else np.uint32)[k] ^= 1
        _upload(job, aid, flat.reshape(shape))
        assert job.hash(aid) != h

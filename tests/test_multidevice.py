"""Single-process multi-device run_pipeline / run_raster (SURVEY §8e's process
model: one host thread per device, query or lattice-row shards, data
replicated, global bbox combined before the grids are built).

The GPU box has one B200, so the shards share device 0 (set_devices([0, 0,
0])): three host threads, three streams, three independent pipelines on
their slices — exactly the code path of an 8-GPU box, minus the hardware.
The contract is bit-identity with the one-device run, including errors."""
import numpy as np
import pytest

import paper_1601_05904_b200 as A

UNIT = (0.0, 0.0, 1.0, 1.0)


def test_default_is_one_device():
    assert A.device_count() >= 1


@pytest.fixture
def shards():
    A.set_devices([0, 0, 0])
    yield 3
    A.set_devices([])
    A.set_weight_precision("fp32")


def single(fn):
    A.set_devices([])
    try:
        return fn()
    finally:
        A.set_devices([0, 0, 0])


@pytest.mark.gpu
@pytest.mark.parametrize("mode,precision", [("aidw", "fp32"), ("idw", "fp32"), ("aidw", "fp64")])
def test_pipeline_shards_bit_identical(shards, mode, precision):
    data = A.generate_random_points(50_000, UNIT, 3)
    q = A.generate_random_queries(30_001, UNIT, 4)
    A.set_weight_precision(precision)
    cfg = A.RunConfig(mode=mode, params=A.AidwParams(k=10), alpha=2.5)
    assert A.device_count() == 3
    b0 = A.replication_info()["nccl_broadcasts"]
    multi = A.run_pipeline(data, q, cfg)
    # data replicated by NCCL: one H2D, one grouped ncclBroadcast over the
    # distinct devices (here one; the three shards share its replica)
    info = A.replication_info()
    assert info["last"] == "nccl_broadcast" and info["nccl_broadcasts"] == b0 + 1
    assert info["nccl_version"] >= 21800
    one = single(lambda: A.run_pipeline(data, q, cfg))
    assert np.array_equal(multi.result.predicted, one.result.predicted)
    assert np.array_equal(multi.result.alphas, one.result.alphas)
    assert multi.stats["pairs"] == 50_000 * 30_001
    assert multi.k_effective == one.k_effective


@pytest.mark.gpu
def test_raster_shards_bit_identical(shards):
    data = A.generate_random_points(40_000, UNIT, 9, "planar")
    multi = A.run_raster(data, 64, 37, A.RunConfig(params=A.AidwParams(k=15)))
    one = single(lambda: A.run_raster(data, 64, 37, A.RunConfig(params=A.AidwParams(k=15))))
    assert np.array_equal(multi.raster.values, one.raster.values)
    assert (multi.raster.xllcorner, multi.raster.yllcorner, multi.raster.cellsize) == \
        (one.raster.xllcorner, one.raster.yllcorner, one.raster.cellsize)


@pytest.mark.gpu
def test_shard_error_is_the_one_device_error(shards):
    data = A.generate_random_points(20_000, UNIT, 5)
    q = A.generate_random_queries(9_000, UNIT, 6)
    cfg = A.RunConfig(params=A.AidwParams(k=10, r_min=3.0, r_max=2.0))  # invalid params
    with pytest.raises(A.InvalidArgument) as multi:
        A.run_pipeline(data, q, cfg)
    with pytest.raises(A.InvalidArgument) as one:
        single(lambda: A.run_pipeline(data, q, cfg))
    assert str(multi.value) == str(one.value)
